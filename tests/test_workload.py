"""The seeded generator (paper_1901_06207_b200/workload.py): determinism and the recipe of DESIGN.md §4."""
import numpy as np

from oracle import truth
from paper_1901_06207_b200 import workload as W


def test_c1_recipe():
    w = W.generate(W.C1, 1)
    assert w.src.size == W.C1.n == 1_000_000 and w.src.dtype == np.uint32
    hosts, card, F = truth.exact_cardinalities(w.src, w.dst)
    tc = dict(zip(hosts.tolist(), card.tolist()))
    assert len(w.planted) == 20 and all(tc[h] == 2000 for h in w.planted)   # planted exactly
    assert max(c for h, c in tc.items() if h not in w.planted) <= 500        # background cap
    assert F == w.n_flows
    # inner IPs lie in the 16 /16 prefixes, outer IPs outside them
    pre = np.array([p >> 16 for p, _ in w.prefixes], dtype=np.uint32)
    assert np.isin(w.src >> np.uint32(16), pre).all()
    assert not np.isin(w.dst >> np.uint32(16), pre).any()


def test_determinism_and_packet_seed():
    spec = W.WindowSpec(n=50000, n_hosts=1000, n_flows=8000, scanners=(300,), victims=(400,))
    a, b = W.generate(spec, 5), W.generate(spec, 5)
    assert np.array_equal(a.src, b.src) and np.array_equal(a.dst, b.dst)
    c = W.generate(spec, 5, packet_seed=6)
    # same flow set (routers see the same flows), different packets
    fa = set(zip(a.src.tolist(), a.dst.tolist()))
    fc = set(zip(c.src.tolist(), c.dst.tolist()))
    assert fa == fc and not np.array_equal(a.src, c.src)


def test_victims_raw_direction():
    spec = W.WindowSpec(n=20000, n_hosts=200, n_flows=2000, victims=(500,))
    w = W.generate(spec, 2)
    (v,) = w.planted
    sel = w.src == v
    assert (w.raw_dst[sel] == v).all()          # DDoS victims are destinations on the wire
    assert ((w.raw_src == w.src) | (w.raw_dst == w.src)).all()


def test_partition_policies():
    src, dst = W.random_pairs(10000, 3)
    for pol in ("hash-by-pair", "hash-by-inner", "round-robin", "contiguous"):
        part = W.partition(src.size, 4, pol, src, dst)
        assert part.min() >= 0 and part.max() <= 3 and np.bincount(part).size == 4
    part = W.partition(src.size, 4, "hash-by-inner", src, dst)
    s2 = np.concatenate([src, src]); d2 = np.concatenate([dst, dst[::-1]])
    p2 = W.partition(s2.size, 4, "hash-by-inner", s2, d2)
    assert np.array_equal(p2[:10000], p2[10000:])     # same inner -> same router
