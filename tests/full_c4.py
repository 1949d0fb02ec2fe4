"""Config 4 at full size on one B200 (not a pytest module: minutes of generation) —
    python -m tests.full_c4 > gpurun_out/full_c4.jsonl

The 2B-pair window is generated as 8 router shards of 250M pairs (one flow set: 16M Zipf flows over
1.2M hosts, 50 scanners, 20 DDoS victims taking 5 % of the packets).  Checks, at full size:
  * every shard's cube equals the oracle's cube of that shard, byte for byte (oracle on all host threads);
  * shard-OR invariant: the OR-merge of the 8 router cubes equals one cube fed all 8 shards, and equals
    the OR of the 8 oracle cubes (= the oracle's cube of the whole 2B-pair window);
  * the merged window's detect (stats and host list) equals the oracle's detect of that cube;
  * every planted scanner and victim (cardinality ≥ 2θ) is detected in the merged window.
Timing of the per-shard updates and of the merged detect is reported too."""
import json
import time

import numpy as np


def main():
    import torch

    from oracle import oracle as O
    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, default_config

    p = O.default_params()
    spec = W.c4_spec()
    cfg = default_config()
    routers = [Cbaa(cfg, 0) for _ in range(8)]
    whole = Cbaa(cfg, 0)
    whole.reset()
    planted = None
    upd_ms = []
    oracle_whole = O.new_cube(p)
    for k, r in enumerate(routers):
        t0 = time.time()
        w = W.generate(spec, 4, packet_seed=k + 1, with_raw=False)
        gen_s = time.time() - t0
        planted = w.planted
        src = torch.from_numpy(w.src.view(np.int32)).cuda()
        dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
        r.reset()
        r.update(src, dst)                 # first call allocates the handle's bin scratch: untimed
        r.reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r.update(src, dst)
        b.record()
        whole.update(src, dst)
        torch.cuda.synchronize()
        upd_ms.append(a.elapsed_time(b))
        t1 = time.time()
        ref = O.update_parallel(p, w.src, w.dst)
        ok = bool(np.array_equal(r.cube().cpu().numpy(), ref))
        O.merge(oracle_whole, ref)
        print(json.dumps({"check": f"shard{k}_cube_vs_oracle", "pairs": int(w.src.size), "equal": ok,
                          "oracle_s": round(time.time() - t1, 1)}), flush=True)
        del ref
        print(json.dumps({"shard": k, "pairs": int(w.src.size), "gen_s": round(gen_s, 1),
                          "update_ms": round(upd_ms[-1], 3)}), flush=True)
        del w, src, dst
        torch.cuda.empty_cache()
    g = Cbaa(cfg, 0)
    g.reset()
    g.merge(routers)
    torch.cuda.synchronize()
    same = bool(torch.equal(g.cube(), whole.cube()))
    t0 = time.perf_counter()
    hosts, stats, rc = g.detect(1024)
    det_ms = 1e3 * (time.perf_counter() - t0)
    found = set(hosts["ip"].tolist())
    merged_vs_oracle = bool(np.array_equal(g.cube().cpu().numpy(), oracle_whole))
    st, oh, ostats = O.detect(p, oracle_whole, 1024)
    hosts_equal = bool(len(hosts) == len(oh) and all(
        np.array_equal(hosts[f], oh[f]) for f in ("ip", "cs", "lp", "z")) and all(
        (np.isinf(a) and np.isinf(b)) or abs(a - b) <= 1e-12 * max(1.0, abs(b))
        for a, b in zip(hosts["estimate"], oh["estimate"])))
    stats_equal = all(a[k_] == b[k_] for a, b in zip(stats, ostats)
                      for k_ in ("ztot", "zmax", "n_hot", "tuples", "candidates", "hits", "overflow"))
    print(json.dumps({"check": "full_c4", "pairs": 8 * spec.n, "shard_or_invariant": same,
                      "merged_cube_vs_oracle": merged_vs_oracle, "hosts_vs_oracle": hosts_equal,
                      "stats_vs_oracle": stats_equal, "oracle_status": st,
                      "planted": len(planted), "planted_detected": len(set(planted) & found),
                      "super_hosts": len(hosts), "detect_ms": round(det_ms, 3),
                      "update_ms_per_250M_shard": round(float(np.median(upd_ms)), 3),
                      "update_gpairs_s": round(spec.n / np.median(upd_ms) / 1e6, 1), "rc": rc}), flush=True)


if __name__ == "__main__":
    main()
