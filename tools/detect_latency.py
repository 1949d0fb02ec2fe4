"""Where the window-end detect latency goes (C2 window): device graph time vs the C call vs the Python wrapper."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1901_06207_b200 import cbaa as cb
    from paper_1901_06207_b200 import workload as W
    w = W.generate(W.C2, 1, with_raw=False)
    h = cb.Cbaa(cb.default_config(), 0)
    h.reset()
    h.update(torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda())
    s = torch.cuda.current_stream()
    for _ in range(5):
        h.detect(1024)
    res = {}
    # Python wrapper
    ts = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.detect(1024)
        ts.append(time.perf_counter() - t0)
    res["python_detect_us"] = 1e6 * sorted(ts)[25]
    # raw C call
    out = np.empty(1 << 20, dtype=cb.HOST_DTYPE)
    n = C.c_uint64()
    ts = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cb.lib().cbaa_detect(h._h, 1024, out.ctypes.data_as(C.c_void_p), 1 << 20, C.byref(n), None,
                             C.c_void_p(s.cuda_stream))
        ts.append(time.perf_counter() - t0)
    res["c_detect_us"] = 1e6 * sorted(ts)[25]
    # device time of the graph: events around the C call
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        cb.lib().cbaa_detect(h._h, 1024, out.ctypes.data_as(C.c_void_p), 1 << 20, C.byref(n), None,
                             C.c_void_p(s.cuda_stream))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    res["event_span_us"] = sorted(ts)[25]
    res["hosts"] = int(n.value)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
