"""Seeded synthetic windows of core-network-shaped IPv4 traffic.

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle: it draws the input arrays and holds none of CBAA's arithmetic (no
mangling, hashing, column extraction or estimation).

The paper's own trace (CERNET, Table 1) is private and its table is
lost; the recipe below follows the structure the paper states:
  * 5-minute backbone windows, inner network NI monitored at its edge
    routers;
  * super hosts are no more than 0.1% of hosts, ~599 per window at
    θ = 1024;
  * flows may span routers, so router shards are drawn per packet.
Counter-based numpy Philox generators make every array reproducible from
(seed, packet_seed).

Layout returned: SoA uint32 arrays ``src`` (= inner IP) and ``dst`` (= outer
IP), host byte order (Q31), i.e. direction already normalised (Q25); ``raw_src``
/ ``raw_dst`` give the on-wire direction for the inner-prefix mode (a0).
"""
from __future__ import annotations

import dataclasses
import numpy as np


@dataclasses.dataclass
class WindowSpec:
    n: int                       # packets (= pairs) in the window
    n_hosts: int                 # background inner hosts
    n_flows: int                 # background flows before capping/dedup
    zipf_s: float = 1.0          # Zipf exponent of inner-host popularity per flow
    card_cap: int = 0            # cap on a background host's cardinality (0 = none)
    scanners: tuple = ()         # cardinalities of planted scanners (inner = src, 1 pkt/flow)
    victims: tuple = ()          # cardinalities of planted DDoS victims (inner = dst, 1-3 pkts/flow)
    pareto_alpha: float = 1.2    # heavy tail of extra packets per background flow
    pareto_max: float = 1.0e4    # truncation of the tail weight
    order: str = "shuffled"      # "shuffled" (primary) | "bursty" (each flow's packets contiguous)
    n_prefixes: int = 16         # random /16 prefixes forming NI
    victim_share: float = 0.0    # if > 0: fraction of the window's packets that go to the DDoS victims


# BASELINE.json configs.
C1 = WindowSpec(n=1_000_000, n_hosts=49_980, n_flows=400_000, card_cap=500, scanners=(2000,) * 20)
C2 = WindowSpec(n=100_000_000, n_hosts=600_000, n_flows=9_000_000)
# Config 3: four edge routers, 50M packets each, of one C2-like flow set (router k: packet_seed = k + 1).
C3_ROUTER = WindowSpec(n=50_000_000, n_hosts=600_000, n_flows=9_000_000)
C3_ROUTERS = 4


def c4_spec(n_shard=250_000_000, scale=1.0, seed=4):
    """Config 4: one shard (of 8) of the 2B-pair window: 16M Zipf flows over 1.2M hosts, 50 scanners
    (d ~ U[2K, 20K]), 20 DDoS victims (d ~ U[5K, 30K]) that receive ~5% of the packets.  `scale`
    shrinks hosts/flows/packets for the reduced parity test."""
    rng = np.random.Generator(np.random.Philox(seed))
    sc = tuple(int(x) for x in rng.integers(2000, 20001, 50))
    vi = tuple(int(x) for x in rng.integers(5000, 30001, 20))
    return WindowSpec(n=int(n_shard * scale), n_hosts=int(1_200_000 * scale), n_flows=int(16_000_000 * scale),
                      scanners=sc, victims=vi, victim_share=0.05, n_prefixes=32)


def c5_geometries():
    """Config 5 grid: r ∈ {2,4,6} × g ∈ {1024..8192} × cbn ∈ {10,12,14}, |RA| = 3, |VA| = 1;
    clbs = [0,10,20] at the paper point (r=4, cbn=12), else clbs(i) = round(i·L/|RA|)."""
    out = []
    for r in (2, 4, 6):
        L = 32 - r
        for cbn in (10, 12, 14):
            clbs = [0, 10, 20] if (r, cbn) == (4, 12) else [int(round(i * L / 3)) for i in range(3)]
            for g in (1024, 2048, 4096, 8192):
                out.append(dict(r=r, g=g, cbn=[cbn] * 4, clbs=clbs))
    return out


C5_THETAS = (256, 512, 1024, 2048, 4096, 8192)


def c5_spec(seed_rng: np.random.Generator | None = None, n=500_000_000):
    rng = seed_rng or np.random.Generator(np.random.Philox(5))
    d = np.exp(rng.uniform(np.log(128), np.log(32768), 200)).astype(np.int64)
    return WindowSpec(n=n, n_hosts=600_000, n_flows=8_000_000, scanners=tuple(int(x) for x in d))


@dataclasses.dataclass
class Window:
    src: np.ndarray          # uint32 inner IP per packet
    dst: np.ndarray          # uint32 outer IP per packet
    raw_src: np.ndarray      # on-wire source
    raw_dst: np.ndarray      # on-wire destination
    prefixes: list           # [(prefix, mask)] of NI
    planted: dict            # inner IP -> planted cardinality
    n_flows: int


def _rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def _outer(rng, k, pref_set):
    """k uniform IPv4 addresses outside the inner /16 prefixes."""
    out = rng.integers(0, 1 << 32, size=k, dtype=np.uint64).astype(np.uint32)
    bad = np.isin(out >> np.uint32(16), pref_set)
    while bad.any():
        out[bad] = rng.integers(0, 1 << 32, size=int(bad.sum()), dtype=np.uint64).astype(np.uint32)
        bad = np.isin(out >> np.uint32(16), pref_set)
    return out


def _distinct_outer(rng, d, pref_set):
    o = np.unique(_outer(rng, d, pref_set))
    while o.size < d:
        o = np.unique(np.concatenate([o, _outer(rng, d - o.size, pref_set)]))
    return rng.permutation(o)[:d]


def generate(spec: WindowSpec, seed: int, packet_seed: int | None = None, n: int | None = None,
             with_raw: bool = True) -> Window:
    """Draw one window.  ``seed`` fixes the address plan and the flow set;
    ``packet_seed`` (default: seed) fixes packets per flow and their order, so
    several routers can observe the same flows with different packets."""
    n = spec.n if n is None else n
    rng = _rng(seed)
    pre16 = np.sort(rng.choice(1 << 16, size=spec.n_prefixes, replace=False).astype(np.uint32))
    prefixes = [(int(p) << 16, 0xFFFF0000) for p in pre16]
    n_planted = len(spec.scanners) + len(spec.victims)
    # inner hosts drawn without replacement from NI; position = popularity rank
    inner_idx = rng.choice(spec.n_prefixes << 16, size=spec.n_hosts + n_planted, replace=False)
    inner = ((pre16[inner_idx >> 16] << np.uint32(16)) | (inner_idx & 0xFFFF).astype(np.uint32)).astype(np.uint32)
    bg_hosts, planted_hosts = inner[: spec.n_hosts], inner[spec.n_hosts:]

    # background flows: inner host per flow ~ Zipf(s) over ranks
    w = 1.0 / np.arange(1, spec.n_hosts + 1, dtype=np.float64) ** spec.zipf_s
    per_host = rng.multinomial(spec.n_flows, w / w.sum())
    if spec.card_cap:
        per_host = np.minimum(per_host, spec.card_cap)
    f_inner = np.repeat(bg_hosts, per_host)
    f_outer = _outer(rng, f_inner.size, pre16)
    key = np.sort((f_inner.astype(np.uint64) << np.uint64(32)) | f_outer)     # flows are distinct pairs
    key = key[np.concatenate([[True], key[1:] != key[:-1]])] if key.size else key
    f_inner = (key >> np.uint64(32)).astype(np.uint32)
    f_outer = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    n_bg_flows = f_inner.size

    planted = {}
    p_inner, p_outer, p_pk, p_victim = [], [], [], []
    for k, d in enumerate(spec.scanners):
        h = planted_hosts[k]
        planted[int(h)] = int(d)
        p_inner.append(np.full(d, h, np.uint32)); p_outer.append(_distinct_outer(rng, d, pre16))
        p_pk.append(np.ones(d, np.int64)); p_victim.append(np.zeros(d, bool))
    for k, d in enumerate(spec.victims):
        h = planted_hosts[len(spec.scanners) + k]
        planted[int(h)] = int(d)
        p_inner.append(np.full(d, h, np.uint32)); p_outer.append(_distinct_outer(rng, d, pre16))
        p_pk.append(None if spec.victim_share > 0 else rng.integers(1, 4, size=d).astype(np.int64))
        p_victim.append(np.ones(d, bool))

    # ---- packets: everything below depends on packet_seed only
    prng = _rng(seed if packet_seed is None else packet_seed)
    if spec.victim_share > 0 and spec.victims:
        # victims' flows share victim_share·n packets: one each, the rest multinomially (a flood)
        nv = sum(spec.victims)
        extra_v = max(0, int(spec.victim_share * n) - nv)
        vk = 1 + prng.multinomial(extra_v, np.full(nv, 1.0 / nv))
        off = 0
        for k in range(len(spec.scanners), len(p_pk)):
            d = spec.victims[k - len(spec.scanners)]
            p_pk[k] = vk[off:off + d]
            off += d
    pk_planted = np.concatenate(p_pk) if p_pk else np.zeros(0, np.int64)
    n_bg = n - int(pk_planted.sum())
    if n_bg < n_bg_flows:
        raise ValueError(f"window of {n} packets cannot carry {n_bg_flows} background flows")
    tail = np.minimum(prng.pareto(spec.pareto_alpha, n_bg_flows), spec.pareto_max)
    extra_total = n_bg - n_bg_flows
    share = tail / tail.sum() * extra_total if n_bg_flows else tail
    extra = np.floor(share).astype(np.int64)
    rem = extra_total - int(extra.sum())
    if rem > 0:   # hand the remainder to the largest fractional parts: total is exactly n
        frac = share - extra
        extra[np.argpartition(-frac, rem - 1)[:rem]] += 1
    pk = np.concatenate([1 + extra, pk_planted])

    fl_inner = np.concatenate([f_inner] + p_inner)
    fl_outer = np.concatenate([f_outer] + p_outer)
    fl_victim = np.concatenate([np.zeros(n_bg_flows, bool)] + p_victim)
    n_fl = fl_inner.size
    if spec.order == "bursty":
        forder = prng.permutation(n_fl).astype(np.int32)
        pidx = np.repeat(forder, pk[forder])
    else:
        pidx = np.repeat(np.arange(n_fl, dtype=np.int32), pk)
        prng.shuffle(pidx)
    src = fl_inner[pidx]
    dst = fl_outer[pidx]
    # on-wire direction: victims always receive (inner = dst); other packets flip a coin
    raw_src = raw_dst = None
    if with_raw:
        flip = fl_victim[pidx] | (prng.integers(0, 2, size=pidx.size, dtype=np.uint8) == 1)
        raw_src = np.where(flip, dst, src)
        raw_dst = np.where(flip, src, dst)
    return Window(src=src, dst=dst, raw_src=raw_src, raw_dst=raw_dst, prefixes=prefixes, planted=planted,
                  n_flows=n_fl)


def partition(n: int, k: int, policy: str, src=None, dst=None, seed: int = 0):
    """Router index per packet: hash-by-pair, hash-by-inner or
    round-robin.  The hash is a fixed integer mix of the raw addresses — a
    routing rule, not part of the method."""
    if policy == "round-robin":
        return (np.arange(n) % k).astype(np.int64)
    if policy == "contiguous":
        return (np.arange(n) * k // max(n, 1)).astype(np.int64)
    x = src.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    if policy == "hash-by-pair":
        x ^= dst.astype(np.uint64) * np.uint64(0xC2B2AE3D27D4EB4F)
    elif policy != "hash-by-inner":
        raise ValueError(policy)
    x ^= np.uint64(seed)
    x ^= x >> np.uint64(29)
    return (x % np.uint64(k)).astype(np.int64)


def random_pairs(n: int, seed: int):
    """Uniform random (src, dst) pairs: the unstructured edge-case input."""
    rng = _rng(seed)
    return (rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32),
            rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32))
