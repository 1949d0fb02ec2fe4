"""Binned update variants: tile-sort scatter with exact counts (CBAA_BIN_SAMPLE=0) or sampled region sizes
(default), write-combining scatter (CBAA_BIN_SCATTER=wc): ms per update, per-phase ms, cube equal to the direct kernel's —
    python tools/wc_ab.py > gpurun_out/wc_ab.jsonl"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (default parameters only)
from paper_1901_06207_b200 import workload as W  # noqa: E402
from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict  # noqa: E402

PH = ["count", "starts", "scatter", "apply"]
# tile scatter with exact counts / with sampled region sizes (default) / write-combining scatter
VARIANTS = [("tile-exact", {"CBAA_BIN_SAMPLE": "0"}), ("tile-sampled", {}), ("wc", {"CBAA_BIN_SCATTER": "wc"})]


def run(p, s, d, reps=10):
    cb = Cbaa(config_from_dict(p), 0)
    ts = []
    cb.set_phase_timing(True)
    for i in range(reps + 2):
        cb.reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cb.update(s, d)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        if i == 1:
            cb.update_phase_ms()   # drop the warm-up phases
    ph, calls = cb.update_phase_ms()
    cube = cb.cube().clone()
    del cb
    return float(np.median(ts[2:])), float(min(ts[2:])), [round(x / max(calls, 1), 4) for x in ph], cube


def main():
    p = O.default_params()
    cases = []
    import dataclasses
    for name, spec in (("C2", W.C2), ("C2 bursty", dataclasses.replace(W.C2, order="bursty"))):
        if len(sys.argv) > 1 and name not in sys.argv[1:]:
            continue
        w = W.generate(spec, 1, with_raw=False)
        cases.append((name, torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda()))
        del w
    g = torch.Generator(device="cuda").manual_seed(5)
    n = 100_000_000
    cases.append(("uniform", torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g),
                  torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g)))
    for name, s, d in cases:
        _, _, _, ref = run(dict(p, update_mode=0), s, d, reps=1)
        for scat, env in VARIANTS:
            for k in ("CBAA_BIN_SCATTER", "CBAA_BIN_SAMPLE"):
                os.environ.pop(k, None)
            os.environ.update(env)
            med, best, ph, cube = run(dict(p, update_mode=2, bin_min_pairs=1), s, d)
            print(json.dumps({"case": name, "n": int(s.numel()), "variant": scat, "ms_median": round(med, 4),
                              "ms_best": round(best, 4), "gpairs_s": round(s.numel() / med / 1e6, 2),
                              "phases_ms": dict(zip(PH, ph)), "cube_equal_direct": bool(torch.equal(cube, ref))}),
                  flush=True)
        for k in ("CBAA_BIN_SCATTER", "CBAA_BIN_SAMPLE"):
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()
