"""Sparse SketchFile "CBA2" on the C2 window's cube: file size vs the dense CBA1 file, device encode and
decode times (host clock around the library calls, D2H/H2D included), round-trip equality."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, default_config
    w = W.generate(W.C2, 1, with_raw=False)
    h = Cbaa(default_config(), 0)
    h.reset()
    h.update(torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda())
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("dense", h.serialize), ("sparse", h.serialize_sparse)):
        fn()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            data = fn()
            ts.append(time.perf_counter() - t0)
        g = Cbaa(default_config(), 0)
        g.deserialize(data)
        td = []
        for _ in range(5):
            t0 = time.perf_counter()
            g.deserialize(data)
            td.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        same = bool(torch.equal(g.cube(), h.cube()))
        res[name] = {"bytes": int(data.size), "serialize_ms": 1e3 * min(ts), "deserialize_ms": 1e3 * min(td),
                     "roundtrip_equal": same}
    res["ratio"] = res["sparse"]["bytes"] / res["dense"]["bytes"]
    cube = h.cube().cpu().numpy()
    res["set_bit_fraction"] = float(np.unpackbits(cube).mean())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
