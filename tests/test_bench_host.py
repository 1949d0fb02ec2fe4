"""Host-side pieces of bench.py that run without a GPU: the golden self-check of the C2 window (the file
written by tools/make_golden_c2.py from the oracle) and the workload plan of every config."""
import numpy as np

import bench
from paper_1901_06207_b200.cbaa import HOST_DTYPE


def _golden_hosts():
    rows = []
    for line in open(bench.GOLDEN_C2):
        if line.startswith("#") or not line.strip():
            continue
        ip, cs, lp, z, est = line.split()
        rows.append((int(ip, 16), int(cs), int(lp), int(z), float(est)))
    out = np.zeros(len(rows), HOST_DTYPE)
    for k, (ip, cs, lp, z, est) in enumerate(rows):
        out[k] = (ip, cs, lp, z, est)
    return out


def test_golden_file_shape():
    h = _golden_hosts()
    assert len(h) == 637
    assert np.isinf(h["estimate"]).sum() >= 2
    est = np.where(np.isinf(h["estimate"]), np.inf, h["estimate"])
    assert all((est[k] > est[k + 1]) or (est[k] == est[k + 1] and h["ip"][k] < h["ip"][k + 1])
               for k in range(len(h) - 1))   # S:418 order


def test_golden_check_detects_differences():
    h = _golden_hosts()
    assert bench.golden_check(h)["match"]
    for mutate in (lambda a: a[:-1], lambda a: a[::-1]):
        assert not bench.golden_check(mutate(h.copy()))["match"]
    b = h.copy()
    k = int(np.nonzero(~np.isinf(b["estimate"]))[0][0])
    b["estimate"][k] *= 1 + 1e-9
    assert not bench.golden_check(b)["match"]
    b = h.copy()
    b["z"][5] += 1
    assert not bench.golden_check(b)["match"]


def test_plans_cover_the_configs():
    for name, world, units in (("C2", 1, 1), ("C3", 1, 4), ("C3", 2, 2), ("C4", 1, 8), ("C4", 8, 1)):
        pl = bench.Plan(name, 1, 0, world)
        assert len(pl.units) == units
    assert bench.Plan("C4", 1, 0, 2).global_pairs == 2_000_000_000
    assert bench.Plan("C3", 1, 0, 4).global_pairs == 200_000_000
