"""Config 5 sweep (BASELINE.json / SURVEY §8(d)): geometry (r × g × cbn) × θ ∈ {256..8192} on one
500M-pair core-network-shaped window, reporting per point: pairs/s of the update, detect latency
(p50/p99/max over repeated detects), hosts, tuples, overflow, load λ/θ, accuracy against exact truth
(FNR/FPR/FTR, Eqs. 2-3), and parity with the oracle on the WHOLE timed window:
  * cube bytes, for every cube ≤ 512 MiB (oracle update on all host threads, private cubes OR-merged);
  * the host list (ip, cs, lp, Z in order, estimates within 1e-12), wherever the oracle's Cartesian
    enumeration stays bounded (Σ tuples ≤ 2^26).

Not a pytest module (it needs tens of minutes of GPU and host time): run as
    python -m tests.sweep_c5 [--n 500000000] [--detects 200] > gpurun_out/sweep_c5.jsonl
It lives under tests/ because it uses the oracle and the exact ground truth (test infrastructure).
"""
import argparse
import json
import math
import os
import time

import numpy as np


def _hosts_equal(gh, oh):
    if len(gh) != len(oh):
        return False
    for f in ("ip", "cs", "lp", "z"):
        if not np.array_equal(gh[f], oh[f]):
            return False
    for a, b in zip(gh["estimate"], oh["estimate"]):
        if math.isinf(b):
            if not math.isinf(a):
                return False
        elif abs(a - b) > 1e-12 * max(1.0, abs(b)):
            return False
    return True


def _same_status(rc, st):
    """Library status (0, CBAA_E_TUPLE_CAP = -6, CBAA_E_CAPACITY = -5) vs the oracle's (0, 1 overflow, 2 capacity)."""
    return {0: 0, -6: 1, -5: 2}.get(rc, rc) == st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500_000_000)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--detects", type=int, default=200)
    ap.add_argument("--max-cube-mib", type=int, default=512)
    ap.add_argument("--r", type=int, default=None, help="only geometries with this r")
    args = ap.parse_args()
    import torch

    from oracle import oracle as O
    from oracle import truth
    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict

    t0 = time.time()
    spec = W.c5_spec(n=args.n)
    w = W.generate(spec, args.seed, with_raw=False)
    hosts_t, card_t, n_flows = truth.exact_cardinalities(w.src, w.dst)
    tc = dict(zip(hosts_t.tolist(), card_t.tolist()))
    print(json.dumps({"setup": "c5", "n": args.n, "flows": n_flows, "gen_s": round(time.time() - t0, 1),
                      "planted": len(w.planted), "host_threads": os.cpu_count()}), flush=True)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    for geo in W.c5_geometries():
        if args.r is not None and geo["r"] != args.r:
            continue
        p = dict(O.default_params(), **geo)
        cb = Cbaa(config_from_dict(p), 0)
        times = []
        for _ in range(4):
            cb.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cb.update(src, dst)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        upd = sorted(times)[len(times) // 2]
        ref, cube_parity = None, None
        if cb.nbytes <= (args.max_cube_mib << 20):
            th = max(1, min(os.cpu_count() or 1, (8 << 30) // cb.nbytes))   # ≤ 8 GiB of private cubes
            t1 = time.time()
            ref = O.update_parallel(p, w.src, w.dst, th)
            cube_parity = bool(np.array_equal(cb.cube().cpu().numpy(), ref))
            oracle_s = time.time() - t1
        lam = n_flows / ((1 << p["r"]) * (1 << p["cbn"][0]))
        for theta in W.C5_THETAS:
            hosts, stats, rc = cb.detect(theta, cap=1 << 22)   # first detect of this θ (graph relaunch)
            lat = []
            for _ in range(args.detects):
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                cb.detect(theta, cap=1 << 22, with_stats=False)
                lat.append(1e3 * (time.perf_counter() - t1))
            lat.sort()
            tuples = int(sum(s["tuples"] for s in stats))
            host_parity = None
            if ref is not None and sum(min(s["tuples"], p["tuple_cap"]) for s in stats) <= (1 << 26):
                st, oh, _ = O.detect(p, ref, theta, cap=1 << 22)
                host_parity = bool(_same_status(rc, st) and _hosts_equal(hosts, oh))
            m = truth.score(hosts["ip"].tolist(), tc, theta)
            print(json.dumps({"r": p["r"], "g": p["g"], "cbn": p["cbn"][0], "theta": theta,
                              "cube_mib": cb.nbytes >> 20, "update_ms": round(upd, 4),
                              "pairs_per_s": args.n / (upd / 1e3), "update_plan": cb.update_plan(args.n),
                              "detect_ms_p50": round(lat[len(lat) // 2], 4),
                              "detect_ms_p99": round(lat[min(len(lat) - 1, int(0.99 * (len(lat) - 1)))], 4),
                              "detect_ms_max": round(lat[-1], 4), "detects": len(lat),
                              "hosts": int(len(hosts)), "tuples": tuples,
                              "candidates": int(sum(s["candidates"] for s in stats)),
                              "overflow_cs": int(sum(s["overflow"] for s in stats)),
                              "lambda_over_theta": round(lam / theta, 3), "overloaded": lam > theta / 4,
                              "truth_H": m["H"], "fnr": m["fnr"], "fpr": m["fpr"], "ftr": m["ftr"],
                              "status": rc, "cube_parity_whole_window": cube_parity, "host_parity": host_parity,
                              "oracle_update_s": round(oracle_s, 1) if ref is not None else None}), flush=True)
        cb.close()
        del ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
