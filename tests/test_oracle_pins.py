"""Pins of the CPU oracle against what the paper and mathematics fix (SURVEY §8(c) pin table).

Each test names the passage it pins and the plausible mistake it would catch.
No expected value here comes from the CUDA path.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from oracle import truth
from paper_1901_06207_b200 import workload as W


def small_params(**kw):
    """A valid small geometry: r=8 (L=24), three RAs of cbn=9 at clbs [0,8,16] -> ep [8,8,8], cp [1,1,1]."""
    p = O.default_params()
    p.update(r=8, g=256, cbn=[9, 9, 9, 8], clbs=[0, 8, 16])
    p.update(kw)
    return p


# ------------------------------------------------------------------ hashing / mangling
def test_mix32_vectors(golden):
    """S:224 definition; vectors in golden/mix32.txt.  Catches a wrong shift/constant."""
    rows = golden("mix32.txt")
    assert len(rows) == 6
    for key, vals in rows.items():
        assert O.mix32(int(key, 16)) == vals[0][0]


def test_mix32_bijection_sample():
    """mix32 is a composition of bijections (xorshift, odd multiply): no collisions on 2^16 inputs."""
    xs = [O.mix32(x * 65599) for x in range(1 << 16)]
    assert len(set(xs)) == 1 << 16


def test_mangle_inverse_constant(paper):
    """Q3: A = 0x9E3779B1 has inverse 0x0E8B2F51 mod 2^32 (A·A⁻¹ ≡ 1 checked with Python big ints)."""
    inv = O.inverse_mod32(paper["mangle_a"])
    assert inv == 0x0E8B2F51
    assert (paper["mangle_a"] * inv) % (1 << 32) == 1
    rng = np.random.default_rng(3)
    for a in rng.integers(0, 1 << 31, 200) * 2 + 1:
        assert (int(a) * O.inverse_mod32(int(a))) % (1 << 32) == 1


def test_mangle_bijection(paper):
    """unmangle∘mangle = id on a 2^16 subspace + random values; A=1,B=0 is the identity."""
    base = 0xC0A80000
    for x in range(0, 1 << 16, 7):
        assert O.unmangle(paper, O.mangle(paper, base | x)) == base | x
    rng = np.random.default_rng(1)
    for x in rng.integers(0, 1 << 32, 2000, dtype=np.uint64):
        assert O.unmangle(paper, O.mangle(paper, int(x))) == int(x)
    ident = dict(paper, mangle_a=1, mangle_b=0)
    for x in (0, 1, 0xC0A80101, 0xFFFFFFFF):
        assert O.mangle(ident, x) == x


# ------------------------------------------------------------------ config / geometry
def test_paper_geometry(golden, paper):
    """128 MB = 2^30 bits; ep [10,10,8], cp [2,2,4].  Catches a wrong size formula / EP sign."""
    g = golden("paper_geometry.txt")
    assert O.validate(paper)[0] == 0
    assert O.cube_bytes(paper) == g["cube_bytes"][0][0] == 1 << 27
    assert O.cs_bits(paper) // 8 == g["cs_bytes"][0][0]
    ep, cp = O.ep_cp(paper)
    assert ep == g["ep"][0] and cp == g["cp"][0]


@pytest.mark.parametrize("change, rule", [
    (dict(num_ra=1, clbs=[0]), 2),                       # S:66 single-RA configs are rejected
    (dict(g=48), 4),                                     # g not a power of two
    (dict(g=16), 4),                                     # g < 32 (Q28)
    (dict(mangle_a=2), 5),                               # A even -> not a bijection
    (dict(clbs=[0, 10, 28]), 7),                         # clbs >= L
    (dict(clbs=[0, 20, 10]), 8),                         # not strictly increasing
    (dict(cbn=[9, 12, 12, 12]), 10),                     # cp(0) = 9 - 10 < 0
    (dict(clbs=[0, 20, 22], cbn=[20, 12, 12, 12]), 11),  # ep [20,2,6]: cp(1) = 10 > ep(2) = 6
])
def test_validate_rules(paper, change, rule):
    """S:37-41 invariants: each violated rule is reported by number with its text."""
    code, msg = O.validate(dict(paper, **change))
    assert code == rule, msg
    assert msg


# ------------------------------------------------------------------ ip mapping
def test_extraction_worked_example(golden, paper):
    """S:180 worked example (0xA57) + hand extraction of col(0), col(1).  Catches LSB-first numbering
    (gives 0xA5E) and reading clbs as the column's LSB (gives 0x7A5), Q7."""
    g = golden("extraction.txt")
    lp = g["lp"][0][0]
    assert [O.ra_col(paper, lp, i) for i in range(3)] == g["col"][0]


def test_extraction_trivial(paper):
    """lp all-ones -> all-ones columns; lp = 0 -> 0."""
    for i in range(3):
        assert O.ra_col(paper, (1 << 28) - 1, i) == (1 << 12) - 1
        assert O.ra_col(paper, 0, i) == 0


def test_extraction_matches_rotl_closed_form(paper):
    """Per-bit loop (oracle) == closed form rotl_L(lp, clbs) >> (L - cbn)."""
    rng = np.random.default_rng(5)
    L = 28
    for lp in rng.integers(0, 1 << L, 3000):
        lp = int(lp)
        for i, c in enumerate(paper["clbs"]):
            rot = ((lp << c) | (lp >> (L - c))) & ((1 << L) - 1) if c else lp
            assert O.ra_col(paper, lp, i) == rot >> (L - 12)


def test_lp_roundtrip_exhaustive_reduced():
    """S:213 / S:602: every lp of a reduced config maps to a tuple that lpFromTuple inverts exactly,
    and flipping a CP bit makes the tuple rejected.  Exhaustive over 2^20 LPs (r = 12)."""
    p = O.default_params()
    p.update(r=12, cbn=[8, 8, 8, 8], clbs=[0, 7, 14], g=64)   # L=20, ep [7,7,6], cp [1,1,2]
    assert O.validate(p)[0] == 0
    assert O.lp_roundtrip_failures(p, 0, 1 << 20) == 0
    assert O.lp_roundtrip_failures(p, 0, 1 << 20, flip_cp=True) == 0


def test_lp_roundtrip_full_width(paper):
    """Full paper width: 2^22 consecutive + a random window of LPs round-trip; CP flips are rejected."""
    assert O.lp_roundtrip_failures(paper, 0, 1 << 22) == 0
    assert O.lp_roundtrip_failures(paper, (1 << 28) - (1 << 20), 1 << 28) == 0
    assert O.lp_roundtrip_failures(paper, 0x5A5A5A5, 0x5A5A5A5 + (1 << 20), flip_cp=True) == 0


def test_lp_from_tuple_vacuous_cp():
    """cp all zero -> every tuple passes the CP check (r=2, cbn=10 gives cp = [0,0,0])."""
    p = O.default_params()
    p.update(r=2, cbn=[10, 10, 10, 10], clbs=[0, 10, 20])
    assert O.validate(p)[0] == 0
    assert O.ep_cp(p) == ([10, 10, 10], [0, 0, 0])
    rng = np.random.default_rng(2)
    for _ in range(200):
        cols = [int(x) for x in rng.integers(0, 1024, 3)]
        lp = O.lp_from_tuple(p, cols)
        assert lp is not None and [O.ra_col(p, lp, i) for i in range(3)] == cols


def test_single_pair_vector(golden, paper):
    """One pair through Alg. 1 with the default readings (golden/single_pair.txt): mangled values, CS,
    LP, row, the 4 columns and the 4 set bits.  Catches an unmangled oip in H_bv (Q2), a VA hash on the
    IP instead of the LP (Q10), a wrong bit layout."""
    g = {k: v[0] for k, v in golden("single_pair.txt").items()}
    iip, oip = g["iip"][0], g["oip"][0]
    assert O.mangle(paper, iip) == g["m_iip"][0]
    assert O.mangle(paper, oip) == g["m_oip"][0]
    cs, cols, row = O.map_pair(paper, iip, oip)
    assert cs == g["cs"][0] and row == g["row"][0] and cols == g["cols"]
    cube, _ = O.update(paper, [iip], [oip])
    words = cube.view("<u4")
    nz = np.nonzero(words)[0]
    assert nz.tolist() == g["words"]
    assert all(int(words[w]) == g["mask"][0] for w in nz)


# ------------------------------------------------------------------ update / merge invariants
def test_update_invariants():
    """exactly |RA|+|VA| bits per pair; idempotent; order-independent."""
    p = small_params()
    src, dst = W.random_pairs(3000, 7)
    one, _ = O.update(p, src[:1], dst[:1])
    assert int(np.unpackbits(one).sum()) == 4
    a, _ = O.update(p, src, dst)
    b, _ = O.update(p, np.concatenate([src, src]), np.concatenate([dst, dst]))
    perm = np.random.default_rng(0).permutation(src.size)
    c, _ = O.update(p, src[perm], dst[perm])
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert int(np.unpackbits(a).sum()) <= 4 * 3000


def test_merge_shard_invariant():
    """P:249 / S:105-107 / S:469: OR of any partition's cubes == cube of the whole stream;
    merge identity and idempotence."""
    p = small_params()
    w = W.generate(W.WindowSpec(n=20000, n_hosts=500, n_flows=3000, scanners=(600,)), 3)
    whole, _ = O.update(p, w.src, w.dst)
    for policy in ("hash-by-pair", "hash-by-inner", "round-robin"):
        for k in (2, 4, 8):
            part = W.partition(w.src.size, k, policy, w.src, w.dst)
            acc = O.new_cube(p)
            for rr in range(k):
                sel = part == rr
                local, _ = O.update(p, w.src[sel], w.dst[sel])
                O.merge(acc, local)
            assert np.array_equal(acc, whole), (policy, k)
    x = whole.copy()
    assert np.array_equal(O.merge(x, O.new_cube(p)), whole)
    assert np.array_equal(O.merge(x, whole), whole)


def test_direction_normalisation():
    """a0 / Q25 / S:581: prefix mode keeps (inner, outer), swaps (outer, inner), skips 0- and 2-inner pairs,
    and the prefix-mode cube of raw traffic equals the normalised cube."""
    spec = W.WindowSpec(n=20000, n_hosts=400, n_flows=2000, victims=(300,), scanners=(200,))
    w = W.generate(spec, 11)
    p = small_params()
    q = dict(p, direction=1, prefixes=w.prefixes)
    a, sk_a = O.update(p, w.src, w.dst)
    b, sk_b = O.update(q, w.raw_src, w.raw_dst)
    assert sk_a == 0 and sk_b == 0 and np.array_equal(a, b)
    inner = w.prefixes[0][0] | 5
    assert O.normalize(q, inner, 0x08080808) == (inner, 0x08080808)
    assert O.normalize(q, 0x08080808, inner) == (inner, 0x08080808)
    assert O.normalize(q, inner, inner + 1) is None
    assert O.normalize(q, 0x08080808, 0x08080809) is None
    _, sk = O.update(q, [inner, 0x08080808], [inner + 1, 0x01010101])
    assert sk == 2


# ------------------------------------------------------------------ estimator closed forms
def test_eq1_closed_form(golden):
    """Eq. 1: z = g -> 0; z = g/2 -> g·ln 2; z = 0 -> +inf."""
    for z, v in golden("closed_forms.txt")["eq1"]:
        assert O.linear_estimate(4096, z) == pytest.approx(v, abs=1e-9)
    assert O.linear_estimate(4096, 2048) == pytest.approx(4096 * math.log(2), rel=1e-15)
    assert math.isinf(O.linear_estimate(4096, 0))


def test_theorem1(golden, paper):
    """Thm. 1: ε(0) = 0; single array at η = c·g -> 1 − e⁻¹; monotone; all arrays enter
    (Q14): with 4 equal arrays ε = (1 − e^{−η/(c g)})^4."""
    assert O.shared_bit_prob(paper, 0.0) == 0.0
    single = dict(paper, num_ra=1, num_va=0)   # not a valid config for the cube, only for the formula
    v = golden("closed_forms.txt")["thm1_single"][0][0]
    assert O.shared_bit_prob(single, 4096 * 4096) == pytest.approx(v, abs=1e-10)
    grid = [O.shared_bit_prob(paper, e) for e in np.linspace(0, 5e7, 50)]
    assert all(b >= a for a, b in zip(grid, grid[1:]))
    eta = 1.0e6
    assert O.shared_bit_prob(paper, eta) == pytest.approx((1 - math.exp(-eta / 2 ** 24)) ** 4, rel=1e-12)
    assert O.shared_bit_prob(paper, math.inf) == 1.0 - 2.0 ** -20   # S:333 cap


def test_theorem2():
    """Thm. 2: ε = 0 reduces to Eq. 1 bit for bit; Z = g(1−ε) -> 0; Z > g(1−ε) -> 0 (Q21);
    Z = 0 -> +inf."""
    for z in (1, 7, 100, 2048, 4095, 4096):
        assert O.corrected_estimate(z, 0.0, 4096) == O.linear_estimate(4096, z)
    assert O.corrected_estimate(4096 * 0.75, 0.25, 4096) == 0.0
    assert O.corrected_estimate(4000, 0.25, 4096) == 0.0
    assert math.isinf(O.corrected_estimate(0, 0.1, 4096))
    # the correction raises the estimate: Z_r = Z/(1−ε)
    assert O.corrected_estimate(2048, 0.1, 4096) == pytest.approx(-4096 * math.log(2048 / 4096 / 0.9), rel=1e-14)


def test_theta_bn_closed_form(golden):
    """P:261 at ε = 0: θ_bn = g·e^{−θ/g}.  Catches a sign/scale slip in the paper formula."""
    for theta, v in golden("closed_forms.txt")["theta_bn"]:
        tol = 1e-9 if theta == 1024 else 1e-4
        assert O.hot_threshold(theta, 0.0, 4096, 0) == pytest.approx(v, abs=tol)
        assert O.hot_threshold(theta, 0.0, 4096, 1) == pytest.approx(v, abs=tol)
    eps = 8.3e-4   # Q15 scratch: paper vs inverted differ by ~2 zeros
    assert O.hot_threshold(1024, eps, 4096, 0) == pytest.approx(4096 * (1 + eps) * math.exp(-0.25) - 4096 * eps)
    assert O.hot_threshold(1024, eps, 4096, 1) == pytest.approx(4096 * (1 - eps) * math.exp(-0.25))
    assert O.hot_threshold(8192, 0.9, 4096, 0) == 0.0           # (1.9)e^-2 < 0.9: clamp
    ths = [O.hot_threshold(t, 0.01, 4096) for t in range(256, 8192, 256)]
    assert all(b < a for a, b in zip(ths, ths[1:]))             # strictly decreasing in θ
    assert O.zmax(3189.968, 4096) == 3189 and O.zmax(-1.0, 4096) == 0 and O.zmax(1e9, 4096) == 4096


# ------------------------------------------------------------------ statistical pins
def _lone_host_cube(p, n, seed):
    rng = np.random.default_rng(seed)
    oips = np.unique(rng.integers(0, 1 << 32, int(n * 1.01) + 8, dtype=np.uint64).astype(np.uint32))
    oips = rng.permutation(oips)[:n]
    iip = np.full(n, 0x0A000001, np.uint32)
    cube, _ = O.update(p, iip, oips)
    cs, cols, _ = O.map_pair(p, 0x0A000001, 0)
    return cube, cs, cols


def test_eq1_accuracy_whang():
    """Linear counting vs its textbook error: relative SE ≈ sqrt(g(e^t − t − 1))/n, t = n/g
    (Whang et al.).  A lone host of n distinct oips: |estimate − n| ≤ 4σ for each seed and the median
    relative error ≤ 10%.  Catches a wrong log base / sign / row hash on unmangled oip."""
    p = O.default_params()
    p.update(r=8, g=4096, cbn=[9, 9, 9, 8], clbs=[0, 8, 16])
    g = 4096
    for n in (256, 1024, 2048):
        t = n / g
        sigma = math.sqrt(g * (math.exp(t) - t - 1))
        errs = []
        for seed in range(40):
            cube, cs, cols = _lone_host_cube(p, n, seed)
            z = O.zero_count(p, cube, cs, 0, cols[0])
            est = O.linear_estimate(g, z)
            assert abs(est - n) <= 4 * sigma, (n, seed, est)
            errs.append(abs(est - n) / n)
        assert float(np.median(errs)) <= 0.10


def test_hot_threshold_behaviour():
    """a lone host of cardinality 2θ has zeros ≤ θ_bn in ≥ 99% of seeds; θ/2 in ≤ 1% (g=4096,
    θ=1024, ε=0).  Column zero counts taken from the oracle cube."""
    p = O.default_params()
    p.update(r=8, g=4096, cbn=[9, 9, 9, 8], clbs=[0, 8, 16])
    zmax = O.zmax(O.hot_threshold(1024, 0.0, 4096), 4096)
    hi = lo = 0
    trials = 300
    for seed in range(trials):
        cube, cs, cols = _lone_host_cube(p, 2048, 1000 + seed)
        hi += O.zero_count(p, cube, cs, 0, cols[0]) <= zmax
        cube, cs, cols = _lone_host_cube(p, 512, 5000 + seed)
        lo += O.zero_count(p, cube, cs, 0, cols[0]) <= zmax
    assert hi >= 0.99 * trials and lo <= 0.01 * trials


def test_cs_load_eta():
    """empty CS -> η = 0, ε = 0; F distinct flows injected into one CS -> η within ±10%."""
    p = O.default_params()
    p.update(r=8, g=1024, cbn=[9, 9, 9, 8], clbs=[0, 8, 16])
    cube = O.new_cube(p)
    assert O.cs_load(p, cube, 3)[1:] == (0.0, 0.0)
    rng = np.random.default_rng(4)
    F = 100_000
    # inner IPs whose mangled RP selects CS 0: draw mangled values with low r bits 0 and unmangle them
    m = (rng.integers(0, 1 << 24, F, dtype=np.uint64).astype(np.uint32) << np.uint32(8))
    iip = np.array([O.unmangle(p, int(x)) for x in m], dtype=np.uint32)
    oip = rng.integers(0, 1 << 32, F, dtype=np.uint64).astype(np.uint32)
    cube, _ = O.update(p, iip, oip)
    ztot, eta, eps = O.cs_load(p, cube, 0)
    assert abs(eta - F) / F <= 0.10
    assert 0 < eps < 1
    assert O.cs_load(p, cube, 1)[1] == 0.0


def test_zero_count_brute_force():
    """S:87 / S:112: zero count + popcount of the column bytes == g, against numpy bit unpacking."""
    p = small_params()
    src, dst = W.random_pairs(20000, 9)
    cube, _ = O.update(p, src, dst)
    zc = O.zero_counts_ra(p, cube)
    g = p["g"]
    bits = np.unpackbits(cube, bitorder="little")
    k = 0
    for cs in range(1 << p["r"]):
        for i in range(3):
            for col in range(1 << p["cbn"][i]):
                base = O.bit_address(p, cs, i, col, 0)
                if k % 97 == 0:
                    assert zc[k] == g - int(bits[base: base + g].sum())
                k += 1
    assert k == zc.size


# ------------------------------------------------------------------ recovery
def test_recovery_c1_matches_exact_truth(paper):
    """Config 1 (BASELINE.json): all 20 planted scanners (|OP| = 2000 ≥ 2θ) are recovered, nothing with
    exact cardinality < θ/2 is reported, every output IP re-maps to hot columns, estimates are
    Eq. 1-consistent with their Z.  Ground truth by explicit set storage."""
    w = W.generate(W.C1, 1)
    cube, _ = O.update(paper, w.src, w.dst)
    st, hosts, stats = O.detect(paper, cube, 1024)
    assert st == 0
    hs, card, _ = truth.exact_cardinalities(w.src, w.dst)
    tc = dict(zip(hs.tolist(), card.tolist()))
    found = set(hosts["ip"].tolist())
    assert set(w.planted) <= found
    for h in hosts:
        assert tc.get(int(h["ip"]), 0) >= 512
        cs, cols, _ = O.map_pair(paper, int(h["ip"]), 0)
        assert cs == h["cs"]
        zmax = stats[cs]["zmax"]
        for i in range(3):
            assert O.zero_count(paper, cube, cs, i, cols[i]) <= zmax
        assert h["estimate"] == O.corrected_estimate(h["z"], stats[cs]["eps"], 4096)
        assert abs(h["estimate"] - 2000) < 300
    m = truth.score(found, tc, 1024)
    assert m["fnr"] == 0.0 and m["fpr"] == 0.0


def test_recovery_empty_and_order():
    """fresh cube -> no hot columns, no hosts; S:418 output order."""
    p = small_params(g=1024)
    st, hosts, stats = O.detect(p, O.new_cube(p), 256)
    assert st == 0 and hosts.size == 0
    assert all(s["n_hot"] == [0, 0, 0] and s["eta"] == 0.0 for s in stats)
    spec = W.WindowSpec(n=60000, n_hosts=2000, n_flows=8000, scanners=(1500, 900, 3000, 700, 2500))
    w = W.generate(spec, 21)
    cube, _ = O.update(p, w.src, w.dst)
    st, hosts, stats = O.detect(p, cube, 256)
    assert set(w.planted) <= set(hosts["ip"].tolist())
    key = [(-h["estimate"], h["ip"]) for h in hosts]
    assert key == sorted(key)


def test_tuple_cap_overflow():
    """S:396 / Q24: a CS whose ∏|HC(i)| exceeds the cap is skipped and flagged, others still report."""
    p = small_params(g=1024, tuple_cap=0)
    spec = W.WindowSpec(n=30000, n_hosts=500, n_flows=4000, scanners=(2000, 2000))
    w = W.generate(spec, 8)
    cube, _ = O.update(p, w.src, w.dst)
    st, hosts, stats = O.detect(p, cube, 256)
    assert st == 1 and hosts.size == 0
    assert any(s["overflow"] for s in stats)
    st2, hosts2, stats2 = O.detect(dict(p, tuple_cap=1 << 24), cube, 256)
    assert st2 == 0 and set(w.planted) <= set(hosts2["ip"].tolist())


# ------------------------------------------------------------------ Q20: union-specific threshold (f4)
def test_union_threshold_closed_form(golden):
    """θ_uc = g(1−ε)e^{−θ/g}: Thm. 2 solved for Z at estimate = θ.  Golden values evaluated with
    decimal arithmetic (tests/golden/union_threshold.txt); ε = 0 equals the Eq. 1 inverse (θ_bn pin);
    feeding θ_uc back through Thm. 2 returns θ (catches a dropped (1−ε) or a sign slip); clamp at 0."""
    for theta, eps, v in golden("union_threshold.txt")["union_thr"]:
        assert O.union_threshold(theta, eps, 4096) == pytest.approx(v, rel=1e-13), (theta, eps)
    assert O.union_threshold(1024, 0.0, 4096) == pytest.approx(golden("closed_forms.txt")["theta_bn"][2][1], abs=1e-9)
    for theta in (256, 1024, 3000, 8192):
        for eps in (0.0, 1e-4, 0.05, 0.3):
            t = O.union_threshold(theta, eps, 4096)
            assert O.corrected_estimate(t, eps, 4096) == pytest.approx(theta, rel=1e-12)
    assert O.union_threshold(1024, 1.0, 4096) == 0.0
    # against the paper's θ_bn: larger below θ = g·ln 2, smaller above (θ_bn − θ_uc = gε(2e^{−θ/g} − 1))
    eps = 0.02
    assert O.union_threshold(1024, eps, 4096) < O.hot_threshold(1024, eps, 4096, 0)
    assert O.union_threshold(4096, eps, 4096) > O.hot_threshold(4096, eps, 4096, 0)


def _loaded_window(p, seed):
    """A window loaded enough for ε to matter (λ ≈ θ/3 per column) with hosts spread around θ."""
    rng = np.random.default_rng(seed)
    sc = tuple(int(x) for x in rng.integers(120, 700, 60))
    spec = W.WindowSpec(n=260_000, n_hosts=6000, n_flows=120_000, card_cap=150, scanners=sc)
    return W.generate(spec, seed)


@pytest.mark.parametrize("theta", [256, 600])
def test_union_threshold_accepts_exactly_estimate_ge_theta(theta):
    """Q20 option: Alg. 2 (hot columns, tuples, candidates) is unchanged and Alg. 3 accepts a candidate iff
    its Thm. 2 estimate is ≥ θ (Def. 1).  Checked per CS against the full candidate list the
    oracle exposes (orc_candidates + orc_union_zeros), and against the paper option's output."""
    p = small_params(r=2, g=1024, cbn=[11, 11, 10, 10], clbs=[0, 10, 20])   # L = 30: ep [10,10,10], cp [1,1,0]
    assert O.validate(p)[0] == 0
    w = _loaded_window(p, 3)
    cube, _ = O.update(p, w.src, w.dst)
    st0, h0, s0 = O.detect(p, cube, theta)
    pu = dict(p, union_threshold=1)
    st1, h1, s1 = O.detect(pu, cube, theta)
    for a, b in zip(s0, s1):
        for k in ("ztot", "eta", "eps", "theta_bn", "zmax", "n_hot", "tuples", "candidates", "overflow"):
            assert a[k] == b[k], k
        assert a["zmax_uc"] == a["zmax"] and b["theta_uc"] == O.union_threshold(theta, b["eps"], p["g"])
    expect, rejected = [], 0
    for cs in range(1 << p["r"]):
        for lp in O.candidates(p, cube, cs, s1[cs]["zmax"]):
            cols = [O.ra_col(p, int(lp), i) for i in range(p["num_ra"])]
            z = O.union_zeros(p, cube, cs, cols, int(lp))
            est = O.corrected_estimate(z, s1[cs]["eps"], p["g"])
            if est >= theta:
                expect.append((O.unmangle(p, (int(lp) << p["r"]) | cs), z))
            else:
                rejected += 1
    assert expect and rejected   # both sides of θ are populated, so the check discriminates
    assert sorted(expect) == sorted((int(h["ip"]), int(h["z"])) for h in h1)
    assert all(h["estimate"] >= theta for h in h1)
    # θ < g·ln 2 here, so θ_uc < θ_bn: the union option drops exactly the paper output's hosts below θ
    kept = [(int(h["ip"]), int(h["z"])) for h in h0 if h["estimate"] >= theta]
    assert kept == [(int(h["ip"]), int(h["z"])) for h in h1]


def test_update_parallel_equals_update(paper):
    """The threaded oracle driver (private cubes OR-merged) is the single-threaded update."""
    src, dst = W.random_pairs(400_000, 31)
    for threads in (1, 3, 8):
        assert np.array_equal(O.update_parallel(paper, src, dst, threads), O.update(paper, src, dst)[0])
