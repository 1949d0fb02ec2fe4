"""C oracle vs the pure-Python micro-oracle (oracle/micro.py) on tiny inputs.

The micro-oracle uses closed forms (rotl extraction, shift-and-mask LP assembly, set algebra for
the union column) where the C oracle uses per-bit loops over a byte string, so agreement pins both.
"""
import numpy as np
import pytest

from oracle import micro
from oracle import oracle as O
from paper_1901_06207_b200 import workload as W
from tests.geometries import random_params


def tiny_window(seed, n_hosts=300, n_flows=1500, scanners=(220, 150, 400), n=8000):
    return W.generate(W.WindowSpec(n=n, n_hosts=n_hosts, n_flows=n_flows, scanners=scanners), seed)


@pytest.mark.parametrize("union", [0, 1])
@pytest.mark.parametrize("seed", range(6))
def test_random_geometry_cube_and_detect(seed, union):
    """union = 1: the Q20 option; the C oracle thresholds Z at floor(θ_uc), the micro-oracle accepts iff the
    Thm. 2 estimate is ≥ θ (Def. 1) — two statements of the same decision."""
    p = dict(random_params(seed, max_cube_bytes=1 << 21, g_choices=(32, 64, 128)), union_threshold=union)
    w = tiny_window(seed)
    cube, _ = O.update(p, w.src, w.dst)
    m = micro.Cube(p)
    m.update(w.src.tolist(), w.dst.tolist())
    assert bytes(cube) == m.to_bytes()
    # per-pair mapping
    for k in range(0, w.src.size, 397):
        assert O.map_pair(p, int(w.src[k]), int(w.dst[k])) == micro.map_pair(p, int(w.src[k]), int(w.dst[k]))
    theta = p["g"] // 2
    st, hosts, stats = O.detect(p, cube, theta)
    mh, mstats = m.detect(theta)
    assert [(int(h["ip"]), int(h["cs"]), int(h["lp"]), int(h["z"])) for h in hosts] == [h[:4] for h in mh]
    for h, q in zip(hosts, mh):
        assert h["estimate"] == pytest.approx(q[4], rel=1e-13)
    for s, q in zip(stats, mstats):
        for k in ("ztot", "zmax", "n_hot", "tuples", "candidates", "hits", "overflow"):
            assert s[k] == q[k], (k, s, q)
        for k in ("eta", "eps", "theta_bn"):
            assert s[k] == pytest.approx(q[k], rel=1e-12, abs=1e-300)


def test_lp_from_tuple_random_geometries():
    for seed in range(20):
        p = random_params(100 + seed)
        rng = np.random.default_rng(seed)
        L = 32 - p["r"]
        for lp in rng.integers(0, 1 << L, 300):
            cols = [micro.ra_col(p, int(lp), i) for i in range(p["num_ra"])]
            assert cols == [O.ra_col(p, int(lp), i) for i in range(p["num_ra"])]
            assert O.lp_from_tuple(p, cols) == micro.lp_from_tuple(p, cols) == int(lp)
        for _ in range(300):
            cols = [int(rng.integers(0, 1 << p["cbn"][i])) for i in range(p["num_ra"])]
            assert O.lp_from_tuple(p, cols) == micro.lp_from_tuple(p, cols)


def test_paper_geometry_small_window(paper):
    """Paper geometry end to end on a small window: cube bytes and detection agree."""
    w = tiny_window(42, n_hosts=2000, n_flows=20000, scanners=(1500, 3000), n=40000)
    cube, _ = O.update(paper, w.src, w.dst)
    m = micro.Cube(paper)
    m.update(w.src.tolist(), w.dst.tolist())
    # compare only the set bits (the cube is 128 MiB; micro keeps a sparse map)
    nz = np.nonzero(cube)[0]
    mb = m.to_bytes()
    assert all(mb[i] == cube[i] for i in nz[:: max(1, nz.size // 5000)])
    assert sum(len(v) for v in m.cells.values()) == int(np.unpackbits(cube).sum())
