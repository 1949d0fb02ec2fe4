"""Config 4 at full size on one B200 (not a pytest module: minutes of generation) —
    python -m tests.full_c4 > gpurun_out/full_c4.jsonl

The 2B-pair window is generated as 8 router shards of 250M pairs (one flow set: 16M Zipf flows over
1.2M hosts, 50 scanners, 20 DDoS victims taking 5 % of the packets).  Checks, at full size:
  * shard 0's cube equals the oracle's cube of shard 0, byte for byte (sampled output the oracle can
    compute: 250M pairs);
  * shard-OR invariant: the OR-merge of the 8 router cubes equals one cube fed all 8 shards;
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
        if k == 0:
            t1 = time.time()
            ref, _ = O.update(p, w.src, w.dst)
            ok0 = bool(np.array_equal(r.cube().cpu().numpy(), ref))
            print(json.dumps({"check": "shard0_cube_vs_oracle", "pairs": int(w.src.size), "equal": ok0,
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
    print(json.dumps({"check": "full_c4", "pairs": 8 * spec.n, "shard_or_invariant": same,
                      "planted": len(planted), "planted_detected": len(set(planted) & found),
                      "super_hosts": len(hosts), "detect_ms": round(det_ms, 3),
                      "update_ms_per_250M_shard": round(float(np.median(upd_ms)), 3),
                      "update_gpairs_s": round(spec.n / np.median(upd_ms) / 1e6, 1), "rc": rc}), flush=True)


if __name__ == "__main__":
    main()
