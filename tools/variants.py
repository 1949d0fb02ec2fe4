"""Time experimental update variants (tools/update_variants.cu) on the C2 window; check each cube
against the product kernel's cube.  Usage: python tools/variants.py [--n 100000000]"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build():
    out = os.path.join(ROOT, "tools", "libvariants.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), "-o", out,
                           os.path.join(ROOT, "tools", "update_variants.cu")])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_1901_06207_b200 import cbaa as cb
    from paper_1901_06207_b200 import workload as W

    path = os.path.join(ROOT, "tools", "libvariants.so")
    if not os.path.exists(path):
        path = build()
    L = C.CDLL(path)
    for name, (res, argt) in cb._SIGS.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, argt
    L.cbaa_x_update.restype = C.c_int
    L.cbaa_x_update.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
    cb._lib = L   # the binding now drives the variants library
    spec = W.C2 if args.n == W.C2.n else W.WindowSpec(n=args.n, n_hosts=600_000, n_flows=min(9_000_000, args.n // 2))
    w = W.generate(spec, 1, with_raw=False)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    h = cb.Cbaa(cb.default_config(), 0)
    s = torch.cuda.current_stream()
    ref = None
    results = []
    configs = [(0, 2, 2), (9, 2, 2), (15, 2, 2), (16, 2, 2), (15, 1, 2), (0, 2, 2)]
    for variant, passes, bps in configs:
        def run():
            h.reset()
            rc = L.cbaa_x_update(h._h, variant, passes, bps, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                 args.n, C.c_void_p(s.cuda_stream))
            assert rc == 0
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        cube = h.cube().clone()
        if ref is None:
            ref = cube
        ok = bool(torch.equal(cube, ref))
        times = []
        for _ in range(args.reps):
            h.reset()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            L.cbaa_x_update(h._h, variant, passes, bps, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                            args.n, C.c_void_p(s.cuda_stream))
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        times.sort()
        r = {"variant": variant, "passes": passes, "blocks_per_sm": bps, "ms_median": times[len(times) // 2],
             "ms_best": times[0], "gpairs": args.n / times[len(times) // 2] / 1e6, "cube_equal": ok}
        print(json.dumps(r), flush=True)
        results.append(r)


if __name__ == "__main__":
    main()
