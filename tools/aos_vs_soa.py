"""Update time of the C2 window from SoA arrays (cbaa_update) vs interleaved pairs (cbaa_update_pairs)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, default_config
    w = W.generate(W.C2, 1, with_raw=False)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    pairs = torch.stack([src, dst], dim=1).contiguous()
    cb = Cbaa(default_config(), 0)
    res = {}
    for name, fn in (("soa", lambda: cb.update(src, dst)), ("aos", lambda: cb.update_pairs(pairs))):
        for _ in range(3):
            cb.reset()
            fn()
        torch.cuda.synchronize()
        cube = cb.cube().clone()
        ts = []
        for _ in range(10):
            cb.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = {"ms_median": sorted(ts)[5], "cube_sum": int(cube.sum())}
    res["same_cube"] = res["soa"]["cube_sum"] == res["aos"]["cube_sum"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
