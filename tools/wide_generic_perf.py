"""Update time of the C5 geometries on a 100M-pair C2-shaped window, per path: the handle's own choice
(auto), the generic wide binned path forced (bin_min_pairs = 1M, so small cubes bin too), the 32-bit-entry
binned path (CBAA_BIN_WIDE_GEN=0, where its tables fit) and the direct kernel (update_mode TEST_SET).
Every path's cube is checked equal to the first one's.  One JSON line per geometry."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import oracle as O
    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    w = W.generate(W.C2, 1, with_raw=False)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    n = len(w.src)
    only = sys.argv[1:]
    for geo in W.c5_geometries():
        key = f"{geo['r']},{geo['g']},{geo['cbn'][0]}"
        if only and key not in only:
            continue
        p = dict(O.default_params(), **geo)
        variants = [("auto", {}, {}), ("wide_generic", dict(bin_min_pairs=1 << 20), {}),
                    ("narrow", dict(bin_min_pairs=1 << 20), {"CBAA_BIN_WIDE_GEN": "0"}),
                    ("direct", dict(update_mode=0), {})]
        out, ref = {"r": geo["r"], "g": geo["g"], "cbn": geo["cbn"][0]}, None
        for name, kw, env in variants:
            os.environ.update(env)
            try:
                cb = Cbaa(config_from_dict(dict(p, **kw)), 0)
            finally:
                for k in env:
                    os.environ.pop(k)
            plan = cb.update_plan(n)
            if name != "auto" and any(plan == v["plan"] for v in out.values() if isinstance(v, dict)):
                out[name] = {"plan": plan, "same_as": next(k for k, v in out.items() if isinstance(v, dict) and v["plan"] == plan)}
                cb.close()
                continue
            ts = []
            for _ in range(5):
                cb.reset()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                cb.update(src, dst)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            cube = cb.cube()
            if ref is None:
                ref = cube.clone()
            same = bool(torch.equal(cube, ref))
            out[name] = {"plan": plan, "update_ms": round(statistics.median(ts[1:]), 4),
                         "gpairs_s": round(n / statistics.median(ts[1:]) / 1e6, 1), "cube_equal": same}
            cb.close()
            del cube
        del ref
        torch.cuda.empty_cache()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
