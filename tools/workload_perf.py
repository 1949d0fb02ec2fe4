"""Update / window throughput across workload shapes (shuffled vs bursty order, DDoS-heavy C4 shard,
C5 window) on one B200; one JSON line per workload.  Not the bench metric: context for DESIGN.md."""
import dataclasses
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=10):
    import torch
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    import torch

    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, default_config
    cases = [("C2 shuffled", W.C2), ("C2 bursty", dataclasses.replace(W.C2, order="bursty")),
             ("C4 shard (250M, 5% to DDoS victims)", W.c4_spec()), ("C5 window (500M)", W.c5_spec())]
    cb = Cbaa(default_config(), 0)
    for name, spec in cases:
        w = W.generate(spec, 1, with_raw=False)
        src = torch.from_numpy(w.src.view(np.int32)).cuda()
        dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
        del w

        def upd():
            cb.reset()
            cb.update(src, dst)

        def window():
            cb.reset()
            cb.update(src, dst)
            cb.detect(1024)

        upd()
        window()
        u = timed(upd)
        t = timed(window)
        hosts, _, _ = cb.detect(1024)
        print(json.dumps({"workload": name, "pairs": int(src.numel()), "update_ms": round(u, 3),
                          "update_gpairs_s": round(src.numel() / u / 1e6, 1), "window_ms_serial": round(t, 3),
                          "super_hosts": int(len(hosts))}), flush=True)
        del src, dst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
