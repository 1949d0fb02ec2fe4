"""Update time vs address-range passes for large cubes (C5-shaped window).
Usage: python tools/passes_perf.py "r,g,cbn;r,g,cbn" "1,2,4" [n_pairs]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import oracle as O   # geometry dicts only
    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 500_000_000
    w = W.generate(W.c5_spec(n=n), 5, with_raw=False)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    del w
    sel = [(int(x.split(",")[0]), int(x.split(",")[1]), int(x.split(",")[2])) for x in sys.argv[1].split(";")]
    plist = [int(x) for x in sys.argv[2].split(",")]
    geos = [g for g in W.c5_geometries() if (g["r"], g["g"], g["cbn"][0]) in sel]
    for geo in geos:
        for passes in plist:
            cb = Cbaa(config_from_dict(dict(O.default_params(), update_passes=passes, **geo)), 0)
            ts = []
            for k in range(5):
                cb.reset()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                cb.update(src, dst)
                b.record()
                torch.cuda.synchronize()
                if k >= 1:
                    ts.append(a.elapsed_time(b))
            print(json.dumps({"n": n, "r": geo["r"], "g": geo["g"], "cbn": geo["cbn"][0], "cube_mib": cb.nbytes >> 20,
                              "passes": passes, "update_ms": round(sorted(ts)[len(ts) // 2], 3)}), flush=True)
            cb.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
