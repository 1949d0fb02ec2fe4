"""Same-box A/B of update variants selected by environment knobs read at handle creation
(e.g. CBAA_BIN_SCATTER=plain|wc).  Each variant: a fresh handle, 3 warm-up + 20 timed C2 updates with
per-kernel event timing; variants interleaved over 3 rounds.  Also checks every variant's cube equals the
first variant's.  Usage: python tools/ab_update.py 'CBAA_BIN_SCATTER=plain' '' ..."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1901_06207_b200 import workload as W  # noqa: E402
from paper_1901_06207_b200.cbaa import Cbaa, default_config  # noqa: E402

variants = sys.argv[1:] or ["CBAA_BIN_SCATTER=plain", ""]
w = W.generate(W.C2, 1, with_raw=False)
s = torch.from_numpy(w.src.view(np.int32)).cuda()
d = torch.from_numpy(w.dst.view(np.int32)).cuda()
res = {v: {"update": [], "phases": []} for v in variants}
ref = None
for rnd in range(3):
    for v in variants:
        env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        cb = Cbaa(default_config(), 0)
        for k, o in old.items():
            if o is None:
                os.environ.pop(k)
            else:
                os.environ[k] = o
        for _ in range(3):
            cb.reset()
            cb.update(s, d)
        torch.cuda.synchronize()
        if rnd == 0:
            cube = cb.cube().cpu().numpy()
            if ref is None:
                ref = cube
            assert np.array_equal(cube, ref), f"cube of {v!r} differs"
        cb.set_phase_timing(True)
        ts = []
        for _ in range(20):
            cb.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cb.update(s, d)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms, calls = cb.update_phase_ms()
        res[v]["update"].append(statistics.median(ts))
        res[v]["phases"].append([m / calls for m in ms])
        cb.close()
for v in variants:
    ph = np.median(np.array(res[v]["phases"]), axis=0).tolist()
    print(json.dumps({"variant": v or "default", "update_ms_median": statistics.median(res[v]["update"]),
                      "rounds": res[v]["update"], "phase_ms": dict(zip(["count", "starts", "scatter", "apply"], ph))}))
