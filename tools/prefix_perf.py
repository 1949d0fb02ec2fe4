"""Update time of the C2 window in inner-prefix mode (raw on-wire pairs, 16 /16 prefixes) vs normalised."""
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
    w = W.generate(W.C2, 1)
    out = {}
    for name, (s, d, prefixes) in {"normalised": (w.src, w.dst, []),
                                   "inner_prefix": (w.raw_src, w.raw_dst, w.prefixes)}.items():
        c = default_config()
        if prefixes:
            c.direction = 1
            c.n_prefixes = len(prefixes)
            for k, (pre, m) in enumerate(prefixes):
                c.inner_prefix[k], c.inner_mask[k] = pre, m
        cb = Cbaa(c, 0)
        src = torch.from_numpy(s.view(np.int32)).cuda()
        dst = torch.from_numpy(d.view(np.int32)).cuda()
        ts = []
        for k in range(8):
            cb.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cb.update(src, dst)
            b.record()
            torch.cuda.synchronize()
            if k >= 2:
                ts.append(a.elapsed_time(b))
        out[name] = {"update_ms": round(sorted(ts)[len(ts) // 2], 3), "cube_sum": int(cb.cube().sum())}
    out["same_cube"] = out["normalised"]["cube_sum"] == out["inner_prefix"]["cube_sum"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
