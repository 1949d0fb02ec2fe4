"""BASELINE.json configs 3-5 on one B200, through the C ABI, against the CPU oracle.

Config 3: four edge routers × 50M pairs, per-router cubes OR-merged (full size).
Config 4: the 8-shard window with DDoS victims and scanners, at 1/50 scale (the oracle's full 2B would
          take the better part of an hour); shards merged as 8 simulated routers.
Config 5: points of the geometry × θ sweep whose cube the oracle can scan in seconds.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import workload as W
from tests.test_gpu_parity import assert_hosts_equal, assert_stats_equal, dev, gpu_cube, handle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def merged_window(p, shards, theta):
    """k routers (handles), OR-merged into a global handle; returns (global handle, hosts, stats, rc)."""
    routers = []
    for src, dst in shards:
        h = handle(p)
        h.reset()
        h.update(dev(src), dev(dst))
        routers.append(h)
    g = handle(p)
    g.reset()
    g.merge(routers)
    hosts, stats, rc = g.detect(theta)
    return g, hosts, stats, rc


@pytest.mark.slow
def test_c3_four_routers_full_size(paper):
    shards = []
    for k in range(W.C3_ROUTERS):
        w = W.generate(W.C3_ROUTER, 3, packet_seed=k + 1, with_raw=False)
        shards.append((w.src, w.dst))
    g, hosts, stats, rc = merged_window(paper, shards, 1024)
    ref = O.new_cube(paper)
    for src, dst in shards:                       # the oracle sees the concatenated stream
        O.update(paper, src, dst, cube=ref)
    assert np.array_equal(gpu_cube(g), ref)
    st, oh, ostats = O.detect(paper, ref, 1024)
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)
    assert 550 <= len(hosts) <= 750


def test_c4_sharded_reduced(paper):
    spec = W.c4_spec(scale=0.02)
    shards, planted = [], None
    for k in range(8):
        w = W.generate(spec, 4, packet_seed=k + 1, with_raw=False)
        shards.append((w.src, w.dst))
        planted = w.planted
    g, hosts, stats, rc = merged_window(paper, shards, 1024)
    ref = O.new_cube(paper)
    for src, dst in shards:
        O.update(paper, src, dst, cube=ref)
    assert np.array_equal(gpu_cube(g), ref)
    st, oh, ostats = O.detect(paper, ref, 1024)
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)
    assert set(planted) <= set(hosts["ip"].tolist())          # every scanner and victim (d ≥ 2θ)


C5_POINTS = [dict(r=2, g=1024, cbn=10), dict(r=6, g=1024, cbn=14), dict(r=4, g=2048, cbn=12),
             dict(r=2, g=8192, cbn=12), dict(r=6, g=4096, cbn=10), dict(r=4, g=1024, cbn=14)]


@pytest.mark.parametrize("pt", C5_POINTS, ids=lambda d: f"r{d['r']}_g{d['g']}_cbn{d['cbn']}")
def test_c5_sweep_points(pt):
    geo = [x for x in W.c5_geometries() if x["r"] == pt["r"] and x["g"] == pt["g"] and x["cbn"][0] == pt["cbn"]][0]
    p = dict(O.default_params(), **geo)
    assert O.validate(p)[0] == 0
    spec = W.c5_spec(n=3_000_000)
    spec = W.WindowSpec(n=spec.n, n_hosts=60_000, n_flows=400_000, scanners=spec.scanners[:30])
    w = W.generate(spec, 5, with_raw=False)
    cb = handle(p)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    ref, _ = O.update(p, w.src, w.dst)
    assert np.array_equal(gpu_cube(cb), ref)
    for theta in (256, 1024, 4096):
        hosts, stats, rc = cb.detect(theta)
        st, oh, ostats = O.detect(p, ref, theta)
        assert_stats_equal(stats, ostats)
        assert_hosts_equal(hosts, oh)
