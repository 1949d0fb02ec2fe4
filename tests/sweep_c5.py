"""Config 5 sweep (BASELINE.json / SURVEY §8(d)): geometry (r × g × cbn) × θ ∈ {256..8192} on one
core-network-shaped window, reporting per point: pairs/s of the update, detect ms, hosts, tuples,
overflow, load λ/θ, accuracy against exact truth (FNR/FPR/FTR, Eqs. 2-3) and a bit-exact
oracle check of the cube on a 1M-pair sample (cubes ≤ 512 MiB).

Not a pytest module (it needs minutes of GPU time): run as
    python -m tests.sweep_c5 [--n 500000000] > gpurun_out/sweep_c5.jsonl
It lives under tests/ because it uses the oracle and the exact ground truth (test infrastructure).
"""
import argparse
import json
import time

import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=500_000_000)
    ap.add_argument("--seed", type=int, default=5)
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
                      "planted": len(w.planted)}), flush=True)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    sample = 1_000_000
    for geo in W.c5_geometries():
        p = dict(O.default_params(), **geo)
        cb = Cbaa(config_from_dict(p), 0)
        # sampled bit-exact check against the oracle
        parity = None
        if cb.nbytes <= (512 << 20):
            cb.reset()
            cb.update(src[:sample], dst[:sample])
            torch.cuda.synchronize()
            ref, _ = O.update(p, w.src[:sample], w.dst[:sample])
            parity = bool(np.array_equal(cb.cube().cpu().numpy(), ref))
            del ref
        # throughput of the whole window
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
        lam = n_flows / ((1 << p["r"]) * (1 << p["cbn"][0]))
        for theta in W.C5_THETAS:
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            hosts, stats, rc = cb.detect(theta, cap=1 << 22)
            det = 1e3 * (time.perf_counter() - t1)
            m = truth.score(hosts["ip"].tolist(), tc, theta)
            print(json.dumps({"r": p["r"], "g": p["g"], "cbn": p["cbn"][0], "theta": theta,
                              "cube_mib": cb.nbytes >> 20, "update_ms": round(upd, 4),
                              "pairs_per_s": args.n / (upd / 1e3), "detect_ms": round(det, 3),
                              "hosts": int(len(hosts)), "tuples": int(sum(s["tuples"] for s in stats)),
                              "candidates": int(sum(s["candidates"] for s in stats)),
                              "overflow_cs": int(sum(s["overflow"] for s in stats)),
                              "lambda_over_theta": round(lam / theta, 3), "overloaded": lam > theta / 4,
                              "truth_H": m["H"], "fnr": m["fnr"], "fpr": m["fpr"], "ftr": m["ftr"],
                              "sample_parity": parity}), flush=True)
        cb.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
