"""Update time for non-paper array counts (generic kernel path) vs the paper shape, C2 window."""
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
    shapes = [(3, 1, [12, 12, 12, 12], [0, 10, 20]), (3, 2, [12, 12, 12, 12, 12], [0, 10, 20]),
              (2, 1, [14, 14, 12], [0, 14]), (4, 1, [8, 8, 8, 8, 12], [0, 7, 14, 21]),
              (3, 0, [12, 12, 12], [0, 10, 20])]
    for nra, nva, cbn, clbs in shapes:
        c = default_config()
        c.num_ra, c.num_va = nra, nva
        for i in range(16):
            c.cbn[i] = cbn[i] if i < len(cbn) else 0
        for i in range(8):
            c.clbs[i] = clbs[i] if i < len(clbs) else 0
        cb = Cbaa(c, 0)
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
        print(json.dumps({"num_ra": nra, "num_va": nva, "cube_mib": cb.nbytes >> 20, "passes": cb.update_passes,
                          "update_ms": round(sorted(ts)[len(ts) // 2], 3),
                          "word_updates_per_s": round(1e8 * (nra + nva) / sorted(ts)[len(ts) // 2] / 1e6, 1)}),
              flush=True)
        cb.close()


if __name__ == "__main__":
    main()
