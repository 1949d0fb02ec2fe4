"""Pure-Python micro-oracle for tiny CBAA inputs — TEST INFRASTRUCTURE ONLY.

An independent second formulation of the same paper steps, used to check the
C oracle (oracle/cbaa_oracle.c) on tiny geometries.  Where the C oracle uses
per-bit loops, this module uses the closed forms, so the two agree only if
both are right:

* RA column (Alg. 1, Q7): col(i) = rotl_L(lp, clbs(i)) >> (L − cbn(i)).
* LP from a tuple (Alg. 3): mask-and-shift of each EP.
* The cube is a dict {(cs, array, col): set(rows)} rather than a bit string;
  zero count = g − |rows|, union = set intersection (Def. 2).

Only tests/ may import this module.
"""
from __future__ import annotations

import math

M32 = 0xFFFFFFFF


def mix32(x):
    h = x & M32
    h ^= h >> 16
    h = (h * 0x45D9F3B) & M32
    h ^= h >> 16
    h = (h * 0x45D9F3B) & M32
    h ^= h >> 16
    return h


def ep_cp(p):
    L = 32 - p["r"]
    n = p["num_ra"]
    ep = [(p["clbs"][(i + 1) % n] - p["clbs"][i]) % L for i in range(n)]
    return ep, [p["cbn"][i] - ep[i] for i in range(n)]


def rotl(x, k, L):
    k %= L
    mask = (1 << L) - 1
    return ((x << k) | (x >> (L - k))) & mask if k else x & mask


def ra_col(p, lp, i):
    L = 32 - p["r"]
    return rotl(lp, p["clbs"][i], L) >> (L - p["cbn"][i])


def va_col(p, lp, j):
    return mix32(lp ^ p["va_seeds"][j]) % (1 << p["cbn"][p["num_ra"] + j])


def mangle(p, x):
    return (p["mangle_a"] * x + p["mangle_b"]) & M32


def unmangle(p, m):
    return (pow(p["mangle_a"], -1, 1 << 32) * (m - p["mangle_b"])) & M32


def map_pair(p, iip, oip):
    mi, mo = mangle(p, iip), mangle(p, oip)
    r = p["r"]
    cs, lp = mi % (1 << r), mi >> r
    cols = [ra_col(p, lp, i) for i in range(p["num_ra"])] + [va_col(p, lp, j) for j in range(p["num_va"])]
    return cs, cols, mix32(mo ^ p["bv_seed"]) % p["g"]


def lp_from_tuple(p, cols):
    L = 32 - p["r"]
    n = p["num_ra"]
    ep, cp = ep_cp(p)
    for i in range(n):
        low = cols[i] & ((1 << cp[i]) - 1)
        nxt = (i + 1) % n
        top = cols[nxt] >> (p["cbn"][nxt] - cp[i])
        if low != top:
            return None
    lp = 0
    for i in range(n):
        e = cols[i] >> cp[i]  # EP(i): the high ep(i) bits of the column index
        # EP(i) occupies LP offsets clbs(i) .. clbs(i)+ep(i)-1 (MSB-first, mod L):
        # rotate it into place as the top bits of an L-bit word, then rotate right by clbs(i).
        placed = e << (L - ep[i])
        lp |= rotl(placed, L - p["clbs"][i], L)
    return lp


class Cube:
    def __init__(self, p):
        self.p = p
        self.cells = {}  # (cs, array, col) -> set of rows

    def update(self, src, dst):
        p = self.p
        for s, d in zip(src, dst):
            cs, cols, row = map_pair(p, int(s), int(d))
            for a, col in enumerate(cols):
                self.cells.setdefault((cs, a, col), set()).add(row)

    def to_bytes(self):
        """Bit-exact S:116 layout, for comparison with the C oracle's bytes."""
        p = self.p
        narr = p["num_ra"] + p["num_va"]
        csbits = sum((1 << p["cbn"][a]) * p["g"] for a in range(narr))
        out = bytearray((1 << p["r"]) * csbits // 8)
        for (cs, a, col), rows in self.cells.items():
            base = cs * csbits + sum((1 << p["cbn"][i]) * p["g"] for i in range(a)) + col * p["g"]
            for rw in rows:
                b = base + rw
                out[b // 8] |= 1 << (b % 8)
        return bytes(out)

    def zeros(self, cs, a, col):
        return self.p["g"] - len(self.cells.get((cs, a, col), ()))

    def detect(self, theta):
        p = self.p
        g = p["g"]
        narr = p["num_ra"] + p["num_va"]
        hosts, stats = [], []
        for cs in range(1 << p["r"]):
            c0 = 1 << p["cbn"][0]
            ztot = sum(self.zeros(cs, 0, col) for col in range(c0))
            eta = math.inf if ztot == 0 else -c0 * g * math.log(ztot / (c0 * g))
            eps = 1.0
            for i in range(narr):
                eps *= 1.0 - math.exp(-eta / ((1 << p["cbn"][i]) * g))
            eps = min(eps, 1.0 - 2.0 ** -20)
            if p.get("theta_formula", 0) == 0:
                tbn = g * (1.0 + eps) * math.exp(-theta / g) - g * eps
            else:
                tbn = g * (1.0 - eps) * math.exp(-theta / g)
            tbn = max(tbn, 0.0)
            zmax = min(max(math.floor(tbn), 0), g)
            hc = [[col for col in range(1 << p["cbn"][i]) if self.zeros(cs, i, col) <= zmax]
                  for i in range(p["num_ra"])]
            tuples = math.prod(len(h) for h in hc)
            st = dict(ztot=ztot, eta=eta, eps=eps, theta_bn=tbn, zmax=zmax, n_hot=[len(h) for h in hc],
                      tuples=tuples, candidates=0, hits=0, overflow=int(tuples > p.get("tuple_cap", 1 << 24)))
            if not st["overflow"]:
                for tup in _product(hc):
                    lp = lp_from_tuple(p, tup)
                    if lp is None:
                        continue
                    st["candidates"] += 1
                    cols = list(tup) + [va_col(p, lp, j) for j in range(p["num_va"])]
                    rows = set(range(g))
                    for a, col in enumerate(cols):
                        rows &= self.cells.get((cs, a, col), set())
                    z = g - len(rows)
                    est = math.inf if z == 0 else max(0.0, -g * math.log(z / (g - g * eps)))
                    # union option (Q20): Def. 1 directly, accept iff the Thm. 2 estimate reaches θ
                    # (the C oracle thresholds Z at floor(g(1-eps)e^(-theta/g)) instead)
                    accept = est >= theta if p.get("union_threshold", 0) else z <= zmax
                    if accept:
                        st["hits"] += 1
                        ip = unmangle(p, (lp << p["r"]) | cs)
                        hosts.append((ip, cs, lp, z, est))
            stats.append(st)
        hosts.sort(key=lambda h: (-h[4], h[0]))
        return hosts, stats


def _product(lists):
    if not lists:
        yield ()
        return
    for head in lists[0]:
        for rest in _product(lists[1:]):
            yield (head,) + rest
