"""Direct (test-and-set) vs binned update on one B200: ms per update for C2 and other shapes —
    python tools/binned_perf.py > gpurun_out/binned_perf.jsonl"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (default parameters only)
from paper_1901_06207_b200 import workload as W  # noqa: E402
from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict  # noqa: E402


def t_update(cb, s, d, reps=10):
    ts = []
    for _ in range(reps + 2):
        cb.reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cb.update(s, d)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[2:])), float(min(ts[2:]))


def main():
    p = O.default_params()
    cases = [("C2", W.C2, 1)]
    for name, spec, seed in cases:
        w = W.generate(spec, seed, with_raw=False)
        s = torch.from_numpy(w.src.view(np.int32)).cuda()
        d = torch.from_numpy(w.dst.view(np.int32)).cuda()
        ref = None
        for mode, staged, atoms in ((0, "1", "0"), (2, "1", "0")):
            os.environ["CBAA_APPLY_ATOMS"] = atoms
            cb = Cbaa(config_from_dict(dict(p, update_mode=mode)), 0)
            med, best = t_update(cb, s, d)
            cube = cb.cube().clone()
            same = None if ref is None else bool(torch.equal(cube, ref))
            ref = cube if ref is None else ref
            print(json.dumps({"case": name, "n": int(s.numel()), "mode": mode, "staged": staged, "apply_atoms": atoms,
                              "ms_median": round(med, 4),
                              "ms_best": round(best, 4), "gpairs_s": round(s.numel() / med / 1e6, 2),
                              "cube_equal_to_mode0": same}), flush=True)
            del cb
    # random uniform pairs (no duplicates: every pair sets fresh bits)
    for n in (10_000_000, 30_000_000, 100_000_000):
        g = torch.Generator(device="cuda").manual_seed(n)
        s = torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g)
        d = torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g)
        ref = None
        for mode in (0, 2):
            cb = Cbaa(config_from_dict(dict(p, update_mode=mode, bin_min_pairs=1)), 0)
            med, best = t_update(cb, s, d)
            cube = cb.cube().clone()
            same = None if ref is None else bool(torch.equal(cube, ref))
            ref = cube if ref is None else ref
            print(json.dumps({"case": "uniform", "n": n, "mode": mode, "ms_median": round(med, 4),
                              "ms_best": round(best, 4), "gpairs_s": round(n / med / 1e6, 2),
                              "cube_equal_to_mode0": same}), flush=True)
            del cb


if __name__ == "__main__":
    main()
