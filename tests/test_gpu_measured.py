"""Parity of the configuration bench.py measures: pipelined windows on two cubes created with
``detect_overlap = 1`` (window-end kernels without shared memory, hits ordered on the host per S:418),
windows of ≥ 2^24 pairs (the binned update with sampled bin regions), the reset on the detect stream —
plus the host-sort branch past kSortMax = 2048 hits, ties among +∞ estimates included, and the Q20
union-threshold option.  Every window is compared with the oracle element by element.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import workload as W
from tests.test_gpu_parity import assert_hosts_equal, assert_stats_equal, dev, gpu_cube, handle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _window(seed, n):
    # ~0.1 % super hosts and a Zipf head heavy enough that the top hosts saturate their union
    # column (Z = 0 → estimate +∞, Q21): their order is decided by the ip tie-break of S:418
    spec = W.WindowSpec(n=n, n_hosts=150_000, n_flows=1_600_000)
    return W.generate(spec, seed, with_raw=False)


def test_bench_pipeline_matches_oracle(paper):
    """The exact object bench.py times (pipeline.WindowPipeline): 3 windows of 2^24 + 12345 pairs
    (sampled bin regions, ragged tail), each window's hosts and per-CS stats == the oracle's."""
    from paper_1901_06207_b200.cbaa import config_from_dict
    from paper_1901_06207_b200.pipeline import WindowPipeline

    n = (1 << 24) + 12345
    wins = [_window(s, n) for s in (11, 12, 13)]
    pipe = WindowPipeline(config_from_dict(paper), 0, 1024, with_stats=True)
    got, keep = [], []   # device inputs stay referenced until the pipeline's streams are done
    for w in wins:
        keep.append((dev(w.src), dev(w.dst)))
        out = pipe.submit(*keep[-1])
        if out is not None:
            got.append((out, pipe.last_stats))
    got.append((pipe.flush(), pipe.last_stats))
    torch.cuda.synchronize()
    assert pipe.cbs[0].cfg.detect_overlap == 1
    n_inf = 0
    for w, (hosts, stats) in zip(wins, got):
        ref, _ = O.update(paper, w.src, w.dst)
        st, oh, ostats = O.detect(paper, ref, 1024)
        assert st == 0
        assert_stats_equal(stats, ostats)
        assert_hosts_equal(hosts, oh)
        n_inf += int(np.isinf(oh["estimate"]).sum())
    assert n_inf >= 2, "the fixture must exercise the +inf tie-break"


def _many_hits_window():
    # 2200 planted hosts of 400 distinct outer IPs (θ = 256: zmax ≈ 3847 > E[Z] ≈ 3714) and six hosts of
    # 40 000 (Z ≈ 0: +∞ estimates) → > 2048 hits, past the device sort's kSortMax
    spec = W.WindowSpec(n=2_200_000, n_hosts=60_000, n_flows=300_000, card_cap=120,
                        scanners=(400,) * 2200 + (40_000,) * 6)
    return W.generate(spec, 21, with_raw=False)


@pytest.mark.parametrize("overlap", [0, 1])
def test_host_sort_past_ksortmax(paper, overlap):
    """> 2048 hits: the host-side S:418 sort (estimate descending, ip ascending) == the oracle's order,
    standalone (past kSortMax) and with detect_overlap = 1."""
    w = _many_hits_window()
    cb = handle(paper, detect_overlap=overlap)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    hosts, stats, rc = cb.detect(256)
    ref, _ = O.update(paper, w.src, w.dst)
    assert np.array_equal(gpu_cube(cb), ref)
    st, oh, ostats = O.detect(paper, ref, 256)
    assert rc == 0 and st == 0
    assert len(oh) > 2048
    assert int(np.isinf(oh["estimate"]).sum()) >= 2
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)


@pytest.mark.parametrize("formula", [0, 1])
def test_union_threshold_thm2(paper, formula):
    """Q20 option (CBAA_UNION_THM2): Alg. 3 thresholds the union column at θ_uc = g(1−ε)e^{−θ/g};
    stats (θ_uc, zmax_uc) and hosts == the oracle's, under both θ_bn formulas and several θ."""
    w = W.generate(W.C1, 5)
    p = dict(paper, union_threshold=1, theta_formula=formula)
    cb = handle(p)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    ref, _ = O.update(p, w.src, w.dst)
    assert np.array_equal(gpu_cube(cb), ref)
    for theta in (512, 1024, 1900, 4096):
        hosts, stats, rc = cb.detect(theta)
        st, oh, ostats = O.detect(p, ref, theta)
        assert_stats_equal(stats, ostats)
        assert_hosts_equal(hosts, oh)
        # Def. 1 through Thm. 2: every output's estimate reaches θ (up to zmax_uc's floor)
        for h in hosts:
            s = stats[h["cs"]]
            assert h["z"] <= s["zmax_uc"] and s["zmax_uc"] <= s["theta_uc"]


def test_theta_change_reuses_graph(paper):
    """θ is not part of the detect graph: consecutive detects with different θ on one cube give the
    oracle's answer for each θ (the k_hot node's parameters are rewritten in place)."""
    w = W.generate(W.C1, 6)
    cb = handle(paper)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    ref, _ = O.update(paper, w.src, w.dst)
    for theta in (1024, 256, 1024, 4096, 1500, 1500):
        hosts, stats, rc = cb.detect(theta)
        st, oh, ostats = O.detect(paper, ref, theta)
        assert_stats_equal(stats, ostats)
        assert_hosts_equal(hosts, oh)


def test_pipeline_router_sets_match_oracle(paper):
    """Config 3's pipelined schedule: each window is 3 router streams into 3 router cubes, OR-merged on
    the update stream and detected beside the next window's updates; every window's hosts and
    stats == the oracle of the routers' concatenated streams."""
    from paper_1901_06207_b200.cbaa import config_from_dict
    from paper_1901_06207_b200.pipeline import WindowPipeline

    spec = W.WindowSpec(n=2_000_003, n_hosts=40_000, n_flows=300_000, scanners=(1500, 2500, 5000))
    wins = [[W.generate(spec, 31 + k, packet_seed=100 * k + r, with_raw=False) for r in range(3)] for k in range(3)]
    pipe = WindowPipeline(config_from_dict(paper), 0, 1024, with_stats=True, routers=3)
    got, keep = [], []
    for routers in wins:
        keep.append([(dev(w.src), dev(w.dst)) for w in routers])
        out = pipe.submit(keep[-1])
        if out is not None:
            got.append((out, pipe.last_stats))
    got.append((pipe.flush(), pipe.last_stats))
    torch.cuda.synchronize()
    for routers, (hosts, stats) in zip(wins, got):
        src = np.concatenate([w.src for w in routers])
        dst = np.concatenate([w.dst for w in routers])
        ref = O.update_parallel(paper, src, dst)
        st, oh, ostats = O.detect(paper, ref, 1024)
        assert_stats_equal(stats, ostats)
        assert_hosts_equal(hosts, oh)
