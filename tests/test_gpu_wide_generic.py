"""Wide entries (LP << 6 | row mod 64) for geometries other than the paper's (k_bin_scatter_w<·, NB>,
k_bin_apply_wg, k_bin_log_wg): whole cube bit-exact against the oracle (S:110 — the cube is the OR of
every pair's bits), and the full detect on the C5 sweep's own geometries (BASELINE config 5)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import workload as W

from .geometries import random_params
from .test_gpu_parity import BIN, dev, full_check, gpu_cube, handle

pytestmark = pytest.mark.gpu


def c5_geo(r, g, cbn):
    return next(dict(O.default_params(), **geo) for geo in W.c5_geometries()
                if geo["r"] == r and geo["g"] == g and geo["cbn"][0] == cbn)


def plan(cb, n):
    return cb.update_plan(n)


# (r, g, cbn) → wide bins 2^r·g/64: 256 (4, 1024), 512 (2, 8192), 1024 (6, 1024), 2048 (4, 8192), (6, 2048),
# 4096 (6, 4096); cbn = 14: Σc(i) > 16384, one apply CTA per (bin, array) (k_bin_apply_wa)
GEOS = [(4, 1024, 10), (2, 8192, 12), (6, 1024, 12), (4, 8192, 12), (6, 2048, 10), (2, 4096, 10), (6, 4096, 12),
        (4, 2048, 14), (6, 1024, 14)]


@pytest.fixture
def force_generic(monkeypatch):
    """r ≥ 5 geometries prefer the 32-bit entries (5 row bits already); =2 forces the generic wide path."""
    monkeypatch.setenv("CBAA_BIN_WIDE_GEN", "2")


@pytest.mark.parametrize("r, g, cbn", GEOS)
def test_wide_generic_c5_geometries(r, g, cbn, force_generic):
    p = c5_geo(r, g, cbn)
    spec = W.WindowSpec(n=400_000, n_hosts=4000, n_flows=60_000, scanners=(700, 1500, 3000), victims=(900,))
    w = W.generate(spec, 40 + r + g)
    cb = handle(p, **BIN)
    assert plan(cb, len(w.src)).startswith("binned-wide-generic"), plan(cb, len(w.src))
    full_check(p, w.src, w.dst, theta=512, **BIN)


@pytest.mark.parametrize("n", [1, 31, 8191, 8193, 250_001])
def test_wide_generic_ragged(n):
    p = c5_geo(4, 8192, 12)
    src, dst = W.random_pairs(n, 900 + n)
    cb = handle(p, **BIN)
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(p, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("seed", range(8))
def test_wide_generic_random_geometries(seed, force_generic):
    """2-4 RAs, 0-2 VAs, any r, g = 1024..8192: every geometry the generic wide path accepts is exact;
    the rest take the other paths and are exact too."""
    p = random_params(700 + seed, max_cube_bytes=1 << 26, g_choices=(1024, 2048, 4096, 8192))
    spec = W.WindowSpec(n=200_000, n_hosts=3000, n_flows=30000, scanners=(300, 600, 900), victims=(500,))
    w = W.generate(spec, 800 + seed)
    full_check(p, w.src, w.dst, theta=max(8, p["g"] // 8), **BIN)


@pytest.mark.parametrize("order", ["shuffled", "sorted", "bursty"])
def test_wide_generic_sampled_regions(order, monkeypatch):
    """Bin regions from the 1/64 sample (forced on a small window) with orders that defeat it: the
    excess goes to the overflow log (k_bin_log_wg) and the cube stays exact."""
    monkeypatch.setenv("CBAA_BIN_SAMPLE_MIN", "1")
    p = c5_geo(2, 8192, 12)
    src, dst = W.random_pairs(600_000, 55)
    if order == "sorted":
        o = np.argsort(src, kind="stable")
        src, dst = src[o], dst[o]
    elif order == "bursty":
        src = src.copy()
        src[100_000:400_000] = src[100_000]   # one host's burst: its bins overflow their sampled share
    cb = handle(p, **BIN)
    assert "k_bin_sample" in plan(cb, len(src))
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(p, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


def test_wide_generic_inner_prefix():
    """a0 inner-prefix mode on the generic wide scatter: cube and skip count equal the oracle's."""
    spec = W.WindowSpec(n=300_000, n_hosts=5000, n_flows=40000, victims=(3000,), scanners=(2500,))
    w = W.generate(spec, 4)
    q = dict(c5_geo(4, 8192, 12), direction=1, prefixes=w.prefixes, **BIN)
    junk_s, junk_d = W.random_pairs(1000, 9)
    raw_s = np.concatenate([w.raw_src, junk_s])
    raw_d = np.concatenate([w.raw_dst, junk_d])
    cb = handle(q)
    assert cb.update_plan(len(raw_s)).startswith("binned-wide-generic")
    cb.reset()
    cb.update(dev(raw_s), dev(raw_d))
    ref, skipped = O.update(q, raw_s, raw_d)
    assert np.array_equal(gpu_cube(cb), ref)
    assert cb.skipped() == skipped >= 1000


@pytest.mark.parametrize("r, g, cbn, auto_generic", [(6, 1024, 12, False), (4, 2048, 12, True), (2, 4096, 10, True)])
def test_wide_generic_selection(r, g, cbn, auto_generic):
    """The default choice (generic wide entries for r < 5 or where the 32-bit tables do not fit; 32-bit
    entries for r ≥ 5), forced (=2) and disabled (=0) all give the oracle's cube; small cubes bin too."""
    import os
    p = c5_geo(r, g, cbn)
    src, dst = W.random_pairs(300_000, 77)
    cb = handle(p, bin_min_pairs=0)   # the library's own choice, small-cube rule included (n ≥ bin_min)
    assert cb.update_plan(1 << 24).startswith("binned-wide-generic") == auto_generic, cb.update_plan(1 << 24)
    assert cb.update_plan(1 << 24).startswith("binned")
    cubes = []
    ref, _ = O.update(p, src, dst)
    for v in ("2", "0"):
        os.environ["CBAA_BIN_WIDE_GEN"] = v
        try:
            cb = handle(p, **BIN)
        finally:
            os.environ.pop("CBAA_BIN_WIDE_GEN")
        assert plan(cb, len(src)).startswith("binned-wide-generic") == (v == "2")
        cb.reset()
        cb.update(dev(src), dev(dst))
        cubes.append(gpu_cube(cb))
    assert np.array_equal(cubes[0], ref) and np.array_equal(cubes[1], ref)
