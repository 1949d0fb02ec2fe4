"""Small windows through every kernel, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool memcheck python tools/sanitize.py
Exercises update (all three modes incl. the binned kernels, aligned / misaligned / prefix), reset, merge, merge_slice, zero counts,
detect (join and Cartesian paths), SketchFile round trip and debug_map; checks the cube against the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import oracle as O
    from paper_1901_06207_b200 import workload as W
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict

    p = O.default_params()
    w = W.generate(W.WindowSpec(n=60_000, n_hosts=3000, n_flows=20000, scanners=(1500, 2500), victims=(1800,)), 3)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()
    ok = True
    for mode in (0, 1, 2):
        for extra in ({}, {"update_passes": 3}, {"direction": 1, "prefixes": w.prefixes}):
            q = dict(p, update_mode=mode, bin_min_pairs=1, **extra)
            cb = Cbaa(config_from_dict(q), 0)
            cb.reset()
            s, d = (w.raw_src, w.raw_dst) if extra.get("direction") else (w.src, w.dst)
            cb.update(dev(s)[1:], dev(d)[1:])            # misaligned start
            cb.update(dev(s[:1]), dev(d[:1]))
            hosts, stats, rc = cb.detect(1024)
            torch.cuda.synchronize()
            ref, _ = O.update(q, s, d)
            ok &= bool(np.array_equal(cb.cube().cpu().numpy(), ref))
            cb.zero_counts()
            cb.debug_map(dev(w.src[:100]), dev(w.dst[:100]))
            f = cb.serialize()
            g = Cbaa(config_from_dict(q), 0)
            g.reset()
            g.deserialize(f, merge=True)
            g.merge([cb])
            g.merge_slice([cb.cube()[: g.nbytes // 16]], 0, 1)
            g.detect(1024, cs_lo=3, cs_hi=9)
    os.environ["CBAA_FORCE_CARTESIAN"] = "1"
    cb = Cbaa(config_from_dict(p), 0)
    cb.record_candidates(True)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    cb.detect(512)
    cb.candidates()
    torch.cuda.synchronize()
    print("sanitize run", "ok" if ok else "PARITY FAILURE")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
