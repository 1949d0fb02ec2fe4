"""Update time of the C2 window in inner-prefix mode (a0: raw on-wire pairs classified by the 16 /16 inner
prefixes) vs the normalised window, with the kernels each path runs (cbaa_update_plan) and the
per-phase split; both cubes must be byte-identical."""
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
    out, cubes = {}, {}
    for name, (s, d, prefixes) in {"normalised": (w.src, w.dst, []),
                                   "inner_prefix": (w.raw_src, w.raw_dst, w.prefixes)}.items():
        c = default_config()
        if prefixes:
            c.direction = 1
            c.n_prefixes = len(prefixes)
            for k, (pre, m) in enumerate(prefixes):
                c.inner_prefix[k], c.inner_mask[k] = pre, m
        cb = Cbaa(c, 0)
        cb.set_phase_timing(True)
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
        ms, calls = cb.update_phase_ms()
        out[name] = {"update_ms": round(sorted(ts)[len(ts) // 2], 3), "plan": cb.update_plan(len(s)),
                     "phase_ms": [round(m / calls, 4) for m in ms], "skipped": cb.skipped(),
                     "pairs_per_s": len(s) / (sorted(ts)[len(ts) // 2] / 1e3)}
        cubes[name] = cb.cube().cpu().numpy()
    out["same_cube"] = bool(np.array_equal(cubes["normalised"], cubes["inner_prefix"]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
