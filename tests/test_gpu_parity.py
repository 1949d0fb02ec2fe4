"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Bars: cube bytes, zero counts, hot-column lists, candidate sets, tuple counts, zmax and
the super-host list (ip, cs, lp, Z) are bit-exact; η, ε, θ_bn and estimates agree within 1e-12 relative.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import workload as W
from tests.geometries import random_params

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 1e-12


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def handle(p, **kw):
    from paper_1901_06207_b200.cbaa import Cbaa, config_from_dict
    return Cbaa(config_from_dict(dict(p, **kw)), 0)


def gpu_cube(cb):
    torch.cuda.synchronize()
    return cb.cube().cpu().numpy()


def assert_stats_equal(gs, os_):
    assert len(gs) == len(os_)
    for cs, (a, b) in enumerate(zip(gs, os_)):
        for k in ("ztot", "zmax", "zmax_uc", "n_hot", "tuples", "candidates", "hits", "overflow"):
            assert a[k] == b[k], (cs, k, a[k], b[k])
        for k in ("eta", "eps", "theta_bn", "theta_uc"):
            if np.isinf(b[k]) or b[k] == 0:
                assert a[k] == b[k], (cs, k)
            else:
                assert abs(a[k] - b[k]) <= RTOL * abs(b[k]), (cs, k, a[k], b[k])


def assert_hosts_equal(gh, oh):
    assert len(gh) == len(oh)
    assert [tuple(int(h[f]) for f in ("ip", "cs", "lp", "z")) for h in gh] == \
           [tuple(int(h[f]) for f in ("ip", "cs", "lp", "z")) for h in oh]
    for a, b in zip(gh["estimate"], oh["estimate"]):
        if np.isinf(b):
            assert np.isinf(a)
        else:
            assert abs(a - b) <= RTOL * max(abs(b), 1.0), (a, b)


def full_check(p, src, dst, theta, **kw):
    cb = handle(p, **kw)
    cb.reset()
    cb.update(dev(src), dev(dst))
    hosts, stats, rc = cb.detect(theta)
    cube = gpu_cube(cb)
    ref, _ = O.update(p, src, dst)
    assert np.array_equal(cube, ref)
    st, oh, ostats = O.detect(p, ref, theta)
    assert (rc == 0) == (st == 0)
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)
    return cb, ref, hosts, stats


# ------------------------------------------------------------------ mapping
def test_debug_map_matches_oracle(paper, golden):
    src, dst = W.random_pairs(20000, 1)
    for p in [paper] + [random_params(s) for s in range(4)]:
        cb = handle(p)
        cs, cols, row = cb.debug_map(dev(src), dev(dst))
        cs, cols, row = cs.cpu().numpy(), cols.cpu().numpy(), row.cpu().numpy()
        for k in range(0, src.size, 37):
            ocs, ocols, orow = O.map_pair(p, int(src[k]), int(dst[k]))
            assert (cs[k], list(cols[k]), row[k]) == (ocs, ocols, orow)
    g = {k: v[0] for k, v in golden("single_pair.txt").items()}
    cb = handle(paper)
    cs, cols, row = cb.debug_map(dev([g["iip"][0]]), dev([g["oip"][0]]))
    assert int(cs[0]) == g["cs"][0] and int(row[0]) == g["row"][0] and cols[0].tolist() == g["cols"]


# ------------------------------------------------------------------ update
def test_c1_window_paper_geometry(paper):
    """BASELINE config 1: 1M pairs, 20 planted scanners of cardinality 2000, θ = 1024."""
    w = W.generate(W.C1, 1)
    cb, ref, hosts, stats = full_check(paper, w.src, w.dst, 1024)
    assert set(w.planted) <= set(hosts["ip"].tolist())
    zc = cb.zero_counts().cpu().numpy()
    assert np.array_equal(zc.view(np.uint32), O.zero_counts_ra(paper, ref))


@pytest.mark.parametrize("seed", range(8))
def test_random_geometries(seed):
    p = random_params(seed, max_cube_bytes=1 << 24)
    spec = W.WindowSpec(n=200_000, n_hosts=3000, n_flows=30000, scanners=(300, 600, 900), victims=(500,))
    w = W.generate(spec, 100 + seed)
    full_check(p, w.src, w.dst, theta=max(8, p["g"] // 2), update_mode=seed % 2)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 7, 31, 33, 1023])
def test_small_and_ragged(paper, n, mode):
    src, dst = W.random_pairs(max(n, 1), 5 + n)
    src, dst = src[:n], dst[:n]
    cb = handle(paper, update_mode=mode)
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(paper, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("off_s, off_d", [(1, 1), (2, 2), (3, 3), (1, 2), (0, 3)])
def test_misaligned_inputs(paper, off_s, off_d):
    """Any 4-byte alignment: head/tail peeling and the scalar path (src/dst misaligned differently)."""
    src, dst = W.random_pairs(10_000, 11)
    big_s = dev(np.concatenate([np.zeros(4, np.uint32), src]))
    big_d = dev(np.concatenate([np.zeros(4, np.uint32), dst]))
    n = 9_000
    s = big_s[off_s: off_s + n]
    d = big_d[off_d: off_d + n]
    hs = big_s.cpu().numpy().view(np.uint32)[off_s: off_s + n]
    hd = big_d.cpu().numpy().view(np.uint32)[off_d: off_d + n]
    cb = handle(paper)
    cb.reset()
    cb.update(s, d)
    ref, _ = O.update(paper, hs, hd)
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("off_s, off_d", [(0, 1), (3, 1)])
def test_misaligned_inputs_larger_than_grid(paper, off_s, off_d, mode):
    """Differently aligned src/dst send every pair down the scalar path of the direct kernel; with 2M pairs
    (far more than the persistent grid's threads) the grid-stride loop must still visit all of them."""
    n = 2_000_000
    src, dst = W.random_pairs(n + 4, 12)
    big_s, big_d = dev(src), dev(dst)
    s, d = big_s[off_s: off_s + n], big_d[off_d: off_d + n]
    cb = handle(paper, update_mode=mode)
    cb.reset()
    cb.update(s, d)
    ref, _ = O.update(paper, src[off_s: off_s + n], dst[off_d: off_d + n])
    assert np.array_equal(gpu_cube(cb), ref)


def test_update_host_checks(paper):
    """update_host refuses unequal lengths and non-32-bit dtypes, and keeps converted copies alive."""
    src, dst = W.random_pairs(100_000, 13)
    cb = handle(paper)
    with pytest.raises(ValueError):
        cb.update_host(src, dst[:-1])
    with pytest.raises(TypeError):
        cb.update_host(src.astype(np.float32), dst)
    cb.reset()
    cb.update_host(src[::-1], dst[::-1].astype(np.int32))   # non-contiguous views: converted copies
    ref, _ = O.update(paper, src[::-1].copy(), dst[::-1].copy())
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("passes", [1, 2, 3, 7])
def test_update_passes(paper, passes, mode):
    """The address-range passes and the update mode (test-and-set vs plain RED) change
    only the schedule, never the cube."""
    src, dst = W.random_pairs(300_000, 3)
    cb = handle(paper, update_passes=passes, update_mode=mode)
    assert cb.update_passes == passes
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(paper, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("mode", [0, 1])
def test_hot_spot_and_duplicates(paper, mode):
    """Every pair identical (a single word hammered) and one host with 50K distinct peers."""
    n = 200_000
    cb = handle(paper, update_mode=mode)
    cb.reset()
    src = np.full(n, 0x0A000001, np.uint32)
    dst = np.full(n, 0x08080808, np.uint32)
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(paper, src[:1], dst[:1])
    assert np.array_equal(gpu_cube(cb), ref)
    dst2 = np.arange(n, dtype=np.uint32) % 50_000 + 0x20000000
    full_check(paper, src, dst2, 1024, update_mode=mode)


def test_reset_and_accumulate(paper):
    a_s, a_d = W.random_pairs(50_000, 1)
    b_s, b_d = W.random_pairs(50_000, 2)
    cb = handle(paper)
    cb.reset()
    cb.update(dev(a_s), dev(a_d))
    cb.update(dev(b_s), dev(b_d))
    ref, _ = O.update(paper, np.concatenate([a_s, b_s]), np.concatenate([a_d, b_d]))
    assert np.array_equal(gpu_cube(cb), ref)
    cb.reset()
    assert not gpu_cube(cb).any()


def test_inner_prefix_direction(paper):
    """a0: raw on-wire pairs with the prefix classifier == normalised pairs; 0/2-inner pairs skipped."""
    spec = W.WindowSpec(n=300_000, n_hosts=5000, n_flows=40000, victims=(3000,), scanners=(2500,))
    w = W.generate(spec, 4)
    q = dict(paper, direction=1, prefixes=w.prefixes)
    junk_s, junk_d = W.random_pairs(1000, 9)
    inner = np.uint32(w.prefixes[0][0]) | np.arange(1000, dtype=np.uint32)
    raw_s = np.concatenate([w.raw_src, junk_s, inner])
    raw_d = np.concatenate([w.raw_dst, junk_d, inner[::-1]])
    cb = handle(q)
    cb.reset()
    cb.update(dev(raw_s), dev(raw_d))
    ref, skipped = O.update(q, raw_s, raw_d)
    assert np.array_equal(gpu_cube(cb), ref)
    assert cb.skipped() == skipped >= 1000
    norm, _ = O.update(paper, w.src, w.dst)
    nz = np.nonzero(norm)[0]
    assert np.array_equal(np.bitwise_and(ref, norm)[nz], norm[nz])


# ------------------------------------------------------------------ detect
def test_detect_structures_c1(paper):
    """Hot-column lists (Alg. 2) and the CP-join candidate set (Alg. 3) equal the oracle's."""
    w = W.generate(W.C1, 2)
    cb = handle(paper)
    cb.record_candidates(True)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    hosts, stats, rc = cb.detect(1024)
    hc = cb.hot_columns()
    ref, _ = O.update(paper, w.src, w.dst)
    st, oh, ostats = O.detect(paper, ref, 1024)
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)
    zc = O.zero_counts_ra(paper, ref)
    c = 4096
    cand = cb.candidates()
    for cs in range(16):
        for i in range(3):
            blk = zc[(cs * 3 + i) * c: (cs * 3 + i + 1) * c]
            want = np.nonzero(blk <= ostats[cs]["zmax"])[0]
            got = hc[(cs * 3 + i) * c: (cs * 3 + i) * c + stats[cs]["n_hot"][i]]
            assert np.array_equal(got, want)
        ocand = O.candidates(paper, ref, cs, ostats[cs]["zmax"])
        gcand = np.sort((cand[(cand >> np.uint64(32)) == cs] & np.uint64(0xFFFFFFFF)).astype(np.uint32))
        assert np.array_equal(gcand, np.sort(ocand))


@pytest.mark.parametrize("theta", [256, 512, 2048, 4096, 8192])
def test_thresholds(paper, theta):
    spec = W.WindowSpec(n=600_000, n_hosts=20000, n_flows=150000, scanners=(300, 700, 1500, 3000, 6000, 12000))
    w = W.generate(spec, 3)
    full_check(paper, w.src, w.dst, theta)


def test_inverted_theta_formula(paper):
    w = W.generate(W.C1, 5)
    full_check(dict(paper, theta_formula=1), w.src, w.dst, 1024)


def test_tuple_cap_and_capacity(paper):
    spec = W.WindowSpec(n=200_000, n_hosts=3000, n_flows=40000, scanners=(3000, 2500, 4000, 5000))
    w = W.generate(spec, 6)
    p = dict(paper, tuple_cap=0)
    cb = handle(p)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    from paper_1901_06207_b200.cbaa import E_TUPLE_CAP
    hosts, stats, rc = cb.detect(1024)
    ref, _ = O.update(p, w.src, w.dst)
    st, oh, ostats = O.detect(p, ref, 1024)
    assert rc == E_TUPLE_CAP and st == 1
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)
    # capacity: ask for fewer hosts than exist
    cb2 = handle(paper)
    cb2.reset()
    cb2.update(dev(w.src), dev(w.dst))
    from paper_1901_06207_b200.cbaa import CbaaError, E_CAPACITY
    with pytest.raises(CbaaError) as ei:
        cb2.detect(1024, cap=2)
    assert ei.value.code == E_CAPACITY


def test_detect_range_matches_full(paper):
    w = W.generate(W.C1, 3)
    cb = handle(paper)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    full, fstats, _ = cb.detect(1024)
    parts, pstats = [], []
    for lo, hi in ((0, 5), (5, 6), (6, 16)):
        h, s, _ = cb.detect(1024, cs_lo=lo, cs_hi=hi)
        parts.append(h)
        pstats += s
    merged = np.concatenate(parts)
    merged = merged[np.lexsort((merged["ip"], -merged["estimate"]))]
    assert np.array_equal(merged, full)
    assert pstats == fstats


def test_empty_window(paper):
    cb = handle(paper)
    cb.reset()
    hosts, stats, rc = cb.detect(1024)
    assert rc == 0 and hosts.size == 0
    assert all(s["eta"] == 0.0 and s["eps"] == 0.0 and s["n_hot"] == [0, 0, 0] for s in stats)


# ------------------------------------------------------------------ merge / routers
@pytest.mark.parametrize("policy", ["hash-by-pair", "hash-by-inner", "round-robin"])
def test_router_merge(paper, policy):
    """Config 3 in miniature: k simulated routers (handles) OR-merged == the oracle of the whole stream."""
    w = W.generate(W.WindowSpec(n=800_000, n_hosts=20000, n_flows=100000, scanners=(2000,) * 5), 9)
    k = 4
    part = W.partition(w.src.size, k, policy, w.src, w.dst)
    routers = []
    for rr in range(k):
        sel = part == rr
        h = handle(paper)
        h.reset()
        h.update(dev(w.src[sel]), dev(w.dst[sel]))
        routers.append(h)
    g = handle(paper)
    g.reset()
    g.merge(routers)
    hosts, stats, rc = g.detect(1024)
    ref, _ = O.update(paper, w.src, w.dst)
    assert np.array_equal(gpu_cube(g), ref)
    st, oh, ostats = O.detect(paper, ref, 1024)
    assert_hosts_equal(hosts, oh)
    # slice merge of CS range [4, 12) only
    s = handle(paper)
    s.reset()
    cs_bytes = s.nbytes // 16
    s.merge_slice([r.cube()[4 * cs_bytes: 12 * cs_bytes] for r in routers], 4, 12)
    cube = gpu_cube(s)
    assert np.array_equal(cube[4 * cs_bytes: 12 * cs_bytes], ref[4 * cs_bytes: 12 * cs_bytes])
    assert not cube[: 4 * cs_bytes].any() and not cube[12 * cs_bytes:].any()


def test_update_host_pipeline(paper):
    """cbaa_update_host (pinned and pageable host arrays, > 1 staging chunk) == device update."""
    src, dst = W.random_pairs(20_000_000, 13)
    cb = handle(paper)
    cb.reset()
    ps = torch.from_numpy(src.view(np.int32)).pin_memory()
    pd = torch.from_numpy(dst.view(np.int32)).pin_memory()
    cb.update_host(ps, pd)
    a = gpu_cube(cb)
    cb.reset()
    cb.update_host(src[:5_000_001], dst[:5_000_001])
    cb.update_host(src[5_000_001:], dst[5_000_001:])
    b = gpu_cube(cb)
    cb.reset()
    cb.update(dev(src), dev(dst))
    c = gpu_cube(cb)
    assert np.array_equal(a, c) and np.array_equal(b, c)


# ------------------------------------------------------------------ full size
@pytest.mark.slow
def test_c2_full_size(paper):
    """BASELINE config 2 at full size (100M pairs, the bench workload and launch configuration):
    whole-cube bytes and the complete detection against the oracle."""
    w = W.generate(W.C2, 1, with_raw=False)
    cb, ref, hosts, stats = full_check(paper, w.src, w.dst, 1024)
    assert cb.update_passes == 2
    cb.reset()
    cb.update_host(w.src, w.dst)                 # the e2e path of bench.py, same window
    assert np.array_equal(gpu_cube(cb), ref)
    assert 550 <= len(hosts) <= 750


@pytest.mark.parametrize("seed", [1, 2])
def test_join_equals_cartesian(paper, seed, monkeypatch):
    """|RA| = 3 detect runs the sorted-run CP join (k_join3); the Cartesian enumeration (k_tuples) must
    give the same candidate set, hosts and stats (the oracle enumerates the full product)."""
    spec = W.WindowSpec(n=2_000_000, n_hosts=40000, n_flows=400000, scanners=(1100, 1500, 3000, 9000))
    w = W.generate(spec, seed)
    out = []
    for force in ("0", "1"):
        monkeypatch.setenv("CBAA_FORCE_CARTESIAN", force)
        cb = handle(paper)
        cb.record_candidates(True)
        cb.reset()
        cb.update(dev(w.src), dev(w.dst))
        for theta in (512, 1024):
            hosts, stats, rc = cb.detect(theta)
            out.append((theta, hosts, stats, np.sort(cb.candidates())))
    for (t1, h1, s1, c1), (t2, h2, s2, c2) in zip(out[:2], out[2:]):
        assert t1 == t2 and np.array_equal(h1, h2) and s1 == s2 and np.array_equal(c1, c2)
    ref, _ = O.update(paper, w.src, w.dst)
    st, oh, ostats = O.detect(paper, ref, 512)
    assert_hosts_equal(out[0][1], oh)
    assert_stats_equal(out[0][2], ostats)


def test_join_buffer_overflow_falls_back(paper):
    """More CP chains than join_capacity: the window is redone with the Cartesian enumeration and the
    result still equals the oracle's."""
    w = W.generate(W.C1, 4)
    cb, ref, hosts, stats = full_check(paper, w.src, w.dst, 1024, join_capacity=4)
    assert sum(s["candidates"] for s in stats) > 4


def test_update_host_across_streams(paper):
    """Consecutive host-ingest calls on different streams reuse the staging buffers safely."""
    src, dst = W.random_pairs(18_000_000, 17)
    cb = handle(paper)
    cb.reset()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cut = 9_000_001
    cb.update_host(src[:cut], dst[:cut], stream=s1)
    s2.wait_stream(s1)
    cb.update_host(src[cut:], dst[cut:], stream=s2)
    torch.cuda.synchronize()
    ref, _ = O.update(paper, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


def test_pipelined_windows(paper):
    """bench.py's pipelined schedule (two cubes; detect of window k on a high-priority stream while
    window k+1 resets and updates) returns each window's own super hosts."""
    wins = [W.generate(W.WindowSpec(n=400_000, n_hosts=10_000, n_flows=60_000, scanners=(2000,) * 3), 30 + k)
            for k in range(5)]
    cbs = [handle(paper), handle(paper)]
    s_upd = torch.cuda.Stream()
    s_det = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
    got, pending = [], None
    for k, w in enumerate(wins):
        c = cbs[k % 2]
        c.reset(s_upd)
        c.update(dev(w.src), dev(w.dst), s_upd)
        done = torch.cuda.Event()
        done.record(s_upd)
        if pending:
            s_det.wait_event(pending[1])
            got.append(pending[0].detect(1024, stream=s_det)[0])
        pending = (c, done)
    s_det.wait_event(pending[1])
    got.append(pending[0].detect(1024, stream=s_det)[0])
    for w, h in zip(wins, got):
        ref, _ = O.update(paper, w.src, w.dst)
        st, oh, _ = O.detect(paper, ref, 1024)
        assert_hosts_equal(h, oh)
        assert set(w.planted) <= set(h["ip"].tolist())


@pytest.mark.parametrize("no_tma", ["0", "1"])
def test_zero_count_paths(paper, no_tma, monkeypatch):
    """The TMA-streamed zero counts (g = 4096) and the register-load kernel give the oracle's counts."""
    monkeypatch.setenv("CBAA_NO_TMA", no_tma)
    w = W.generate(W.C1, 6)
    cb = handle(paper)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    ref, _ = O.update(paper, w.src, w.dst)
    assert np.array_equal(cb.zero_counts().cpu().numpy().view(np.uint32), O.zero_counts_ra(paper, ref))
    hosts, stats, rc = cb.detect(1024)
    st, oh, ostats = O.detect(paper, ref, 1024)
    assert_stats_equal(stats, ostats)
    assert_hosts_equal(hosts, oh)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n, off", [(1_000_003, 0), (1_000_003, 1), (7, 0), (9, 1), (0, 0)])
def test_update_interleaved_pairs(paper, n, off, mode):
    """cbaa_update_pairs on interleaved (src, dst) arrays: 16-B aligned, 8-B aligned (one pair peeled),
    ragged tails — same cube as the oracle."""
    src, dst = W.random_pairs(max(n, 1), 40 + n)
    src, dst = src[:n], dst[:n]
    inter = np.zeros(2 * (n + 1), np.uint32)
    inter[2 * off: 2 * off + 2 * n: 2] = src
    inter[2 * off + 1: 2 * off + 2 * n: 2] = dst
    t = dev(inter)[2 * off: 2 * off + 2 * n]
    cb = handle(paper, update_mode=mode)
    cb.reset()
    cb.update_pairs(t)
    ref, _ = O.update(paper, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


# ------------------------------------------------------------------ binned update (CBAA_UPDATE_BINNED)
BIN = dict(update_mode=2, bin_min_pairs=1)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 1023, 8191, 8192, 8193, 300_001])
def test_binned_small_and_ragged(paper, n):
    """Count → scan → scatter → apply on ragged sizes: partial scatter tiles, CTAs with empty chunks."""
    src, dst = W.random_pairs(n, 70 + n)
    cb = handle(paper, **BIN)
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(paper, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("seed", range(10))
def test_binned_random_geometries(seed):
    """Entry row bits s = min(5, r) for r = 1..8, 2-4 RAs, 0-2 VAs, g = 32..256, full detection."""
    p = random_params(200 + seed, max_cube_bytes=1 << 24)
    spec = W.WindowSpec(n=200_000, n_hosts=3000, n_flows=30000, scanners=(300, 600, 900), victims=(500,))
    w = W.generate(spec, 300 + seed)
    full_check(p, w.src, w.dst, theta=max(8, p["g"] // 2), **BIN)


@pytest.mark.parametrize("off_s, off_d", [(1, 1), (0, 3), (2, 1)])
def test_binned_misaligned(paper, off_s, off_d):
    src, dst = W.random_pairs(40_000, 12)
    big_s = dev(np.concatenate([np.zeros(4, np.uint32), src]))
    big_d = dev(np.concatenate([np.zeros(4, np.uint32), dst]))
    n = 39_001
    cb = handle(paper, **BIN)
    cb.reset()
    cb.update(big_s[off_s: off_s + n], big_d[off_d: off_d + n])
    ref, _ = O.update(paper, big_s.cpu().numpy().view(np.uint32)[off_s: off_s + n],
                      big_d.cpu().numpy().view(np.uint32)[off_d: off_d + n])
    assert np.array_equal(gpu_cube(cb), ref)


def test_binned_hot_spot_and_skew(paper):
    """One word hammered by every pair; one host with 90 % of the packets (one CS's bins take almost
    everything); a lone host with 50K distinct peers, detected like the oracle."""
    n = 400_000
    src = np.full(n, 0x0A000001, np.uint32)
    dst = np.full(n, 0x08080808, np.uint32)
    cb = handle(paper, **BIN)
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(paper, src[:1], dst[:1])
    assert np.array_equal(gpu_cube(cb), ref)
    s2, d2 = W.random_pairs(n, 13)
    s2[: 9 * n // 10] = 0x0A000002
    cb.reset()
    cb.update(dev(s2), dev(d2))
    ref, _ = O.update(paper, s2, d2)
    assert np.array_equal(gpu_cube(cb), ref)
    dst3 = np.arange(n, dtype=np.uint32) % 50_000 + 0x20000000
    full_check(paper, src, dst3, 1024, **BIN)


def test_binned_inner_prefix(paper):
    """a0 in the binned kernels: both count and scatter classify; skips are counted once."""
    spec = W.WindowSpec(n=300_000, n_hosts=5000, n_flows=40000, victims=(3000,), scanners=(2500,))
    w = W.generate(spec, 4)
    q = dict(paper, direction=1, prefixes=w.prefixes, **BIN)
    junk_s, junk_d = W.random_pairs(1000, 9)
    raw_s = np.concatenate([w.raw_src, junk_s])
    raw_d = np.concatenate([w.raw_dst, junk_d])
    cb = handle(q)
    cb.reset()
    cb.update(dev(raw_s), dev(raw_d))
    ref, skipped = O.update(q, raw_s, raw_d)
    assert np.array_equal(gpu_cube(cb), ref)
    assert cb.skipped() == skipped >= 1000


@pytest.mark.parametrize("sample", ["9", "14"])
def test_binned_inner_prefix_sampled(paper, sample, monkeypatch):
    """a0 on the wide path with sampled bin regions (forced on a small window): the sample classifies, the
    scatter classifies and counts the skips (once), regions that fall short spill to the overflow log;
    prefixes mix /16s (full bitmap) with a /24 and a /20 (partial bitmap, exact comparison)."""
    monkeypatch.setenv("CBAA_BIN_SAMPLE_MIN", "1")
    monkeypatch.setenv("CBAA_BIN_SAMPLE", sample)
    spec = W.WindowSpec(n=400_000, n_hosts=6000, n_flows=60000, victims=(3000,), scanners=(2500,))
    w = W.generate(spec, 14)
    extra = [(0xC0A80100, 0xFFFFFF00), (0x0AB00000, 0xFFF00000)]   # 192.168.1.0/24, 10.176.0.0/12-ish /20
    q = dict(paper, direction=1, prefixes=w.prefixes[:14] + extra, **BIN)
    junk_s, junk_d = W.random_pairs(20_000, 9)
    rng = np.random.default_rng(3)
    sub24 = (0xC0A80100 | rng.integers(0, 256, 5000)).astype(np.uint32)     # inner via the /24
    out24 = (0xC0A80200 | rng.integers(0, 256, 5000)).astype(np.uint32)     # same /16, outside the /24
    raw_s = np.concatenate([w.raw_src, junk_s, out24, sub24])
    raw_d = np.concatenate([w.raw_dst, junk_d, sub24, out24])
    cb = handle(q)
    cb.reset()
    cb.update(dev(raw_s), dev(raw_d))
    ref, skipped = O.update(q, raw_s, raw_d)
    assert np.array_equal(gpu_cube(cb), ref)
    assert cb.skipped() == skipped > 0
    assert cb.update_plan(len(raw_s)).startswith("binned-wide k_bin_sample")


def test_binned_chunks_and_accumulate(paper, monkeypatch):
    """Several count/scatter/apply rounds per call (small CBAA_BIN_CHUNK) and across calls, OR-ed into a
    cube that already holds bits from the direct kernel."""
    monkeypatch.setenv("CBAA_BIN_CHUNK", "100003")
    a_s, a_d = W.random_pairs(350_000, 21)
    b_s, b_d = W.random_pairs(50_000, 22)
    cb = handle(paper, update_mode=2, bin_min_pairs=100_000)
    cb.reset()
    cb.update(dev(b_s), dev(b_d))         # below bin_min_pairs: direct kernel
    cb.update(dev(a_s), dev(a_d))         # 4 binned rounds
    ref, _ = O.update(paper, np.concatenate([a_s, b_s]), np.concatenate([a_d, b_d]))
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("r, g, cbn", [(6, 4096, 12), (2, 1024, 10), (4, 4096, 14), (0, 64, 11), (2, 1024, 15)])
def test_binned_shapes(r, g, cbn):
    """r ≥ 5 (s = 5, one bin per word group), r = 2 (s = 2, 8 bins per group), r = 0 (s = 0, the entry
    is the whole mangled IP), and column counts too large for the shared-memory word group (fallback to
    the direct kernel) — all bit-exact."""
    L = 32 - r
    clbs = [0, L // 3, 2 * L // 3]
    ep = [clbs[1] - clbs[0], clbs[2] - clbs[1], L - clbs[2]]
    p = O.default_params()
    p.update(r=r, g=g, clbs=clbs, cbn=[max(ep[i], min(cbn, ep[i] + ep[(i + 1) % 3])) for i in range(3)] + [min(cbn, 14)])
    assert O.validate(p)[0] == 0, (p, O.validate(p))
    src, dst = W.random_pairs(200_000, 31 + r)
    cb = handle(p, **BIN)
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(p, src, dst)
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.slow
def test_binned_c2_full_size(paper):
    """Config 2 at full size through the binned kernels (default threshold, the bench configuration)."""
    w = W.generate(W.C2, 1, with_raw=False)
    cb, ref, hosts, stats = full_check(paper, w.src, w.dst, 1024, update_mode=2)
    assert 550 <= len(hosts) <= 750


@pytest.mark.parametrize("scatter", ["wc", "tile"])
def test_binned_scatter_variants(paper, scatter, monkeypatch):
    """Both scatters (write-combining slots with overflow re-append and back-cursor spill, and the tile
    counting sort) produce the oracle's cube: a ragged Zipf window with planted hosts, one pair repeated
    400K times (every slot overflows, the overflow list fills, the back-cursor path runs), and a window
    whose pairs fall in a handful of bins."""
    monkeypatch.setenv("CBAA_BIN_SCATTER", scatter)
    spec = W.WindowSpec(n=700_001, n_hosts=20_000, n_flows=150_000, card_cap=400, scanners=(2000, 1500),
                        victims=(2500,))
    w = W.generate(spec, 41)
    full_check(paper, w.src, w.dst, 1024, **BIN)
    n = 400_000
    src = np.full(n, 0x0A000001, np.uint32)
    dst = np.full(n, 0x08080808, np.uint32)
    cb = handle(paper, **BIN)
    cb.reset()
    cb.update(dev(src), dev(dst))
    ref, _ = O.update(paper, src[:1], dst[:1])
    assert np.array_equal(gpu_cube(cb), ref)
    s3 = np.full(n, 0x0A000003, np.uint32)
    d3 = (np.arange(n, dtype=np.uint32) % 7) + 0x30000000
    cb.reset()
    cb.update(dev(s3), dev(d3))
    ref, _ = O.update(paper, s3[:7], d3[:7])
    assert np.array_equal(gpu_cube(cb), ref)


@pytest.mark.parametrize("order, sample", [("shuffled", "9"), ("sorted", "9"), ("hot", "9"), ("shuffled", "14"),
                                           ("bursty", "14"), ("bursty", "3")])
def test_binned_sampled_regions(paper, order, sample, monkeypatch):
    """Bin regions sized from 8 of every 2^L pairs (forced on small windows): whatever the sample misses
    spills to the overflow log and still lands in the cube.  'sorted': pairs ordered by inner host;
    'hot': one host with 60 % of the pairs; L = 14 leaves most bins unsampled, so most regions
    overflow; 'bursty': each flow's packets contiguous; L = 3: every pair sampled."""
    monkeypatch.setenv("CBAA_BIN_SAMPLE_MIN", "1")
    monkeypatch.setenv("CBAA_BIN_SAMPLE", sample)
    spec = W.WindowSpec(n=400_003, n_hosts=8000, n_flows=90_000, card_cap=400, scanners=(2000, 1300),
                        victims=(1800,), order="bursty" if order == "bursty" else "shuffled")
    w = W.generate(spec, 51)
    src, dst = w.src.copy(), w.dst.copy()
    if order == "sorted":
        o = np.argsort(src, kind="stable")
        src, dst = src[o], dst[o]
    elif order == "hot":
        src[: 6 * len(src) // 10] = 0x0A000005
    full_check(paper, src, dst, 1024, **BIN)


@pytest.mark.parametrize("off_s, off_d", [(1, 1), (0, 3)])
def test_binned_sampled_misaligned(paper, off_s, off_d, monkeypatch):
    """Sampled regions on arrays that are not 16-B aligned (the sample's scalar loads, the scatter's
    per-pair path) and differently aligned src/dst."""
    monkeypatch.setenv("CBAA_BIN_SAMPLE_MIN", "1")
    src, dst = W.random_pairs(300_000, 17)
    big_s = dev(np.concatenate([np.zeros(4, np.uint32), src]))
    big_d = dev(np.concatenate([np.zeros(4, np.uint32), dst]))
    n = 290_001
    cb = handle(paper, **BIN)
    cb.reset()
    cb.update(big_s[off_s: off_s + n], big_d[off_d: off_d + n])
    ref, _ = O.update(paper, big_s.cpu().numpy().view(np.uint32)[off_s: off_s + n],
                      big_d.cpu().numpy().view(np.uint32)[off_d: off_d + n])
    assert np.array_equal(gpu_cube(cb), ref)
