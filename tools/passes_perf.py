"""Update time vs address-range passes for large cubes (C5 window, 500M pairs)."""
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
    w = W.generate(W.c5_spec(), 5, with_raw=False)
    src = torch.from_numpy(w.src.view(np.int32)).cuda()
    dst = torch.from_numpy(w.dst.view(np.int32)).cuda()
    del w
    geos = [g for g in W.c5_geometries() if (g["r"], g["g"], g["cbn"][0]) in ((4, 4096, 14), (6, 4096, 12), (6, 8192, 14), (4, 4096, 12))]
    for geo in geos:
        for passes in (1, 2, 3, 4, 6, 8, 12):
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
            print(json.dumps({"r": geo["r"], "g": geo["g"], "cbn": geo["cbn"][0], "cube_mib": cb.nbytes >> 20,
                              "passes": passes, "update_ms": round(sorted(ts)[len(ts) // 2], 3)}), flush=True)
            cb.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
