"""ctypes front end of the CBAA CPU oracle (oracle/cbaa_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  The product
path (paper_1901_06207_b200/) never imports it and shares no code with it.

Configs are plain dicts with the SPEC's field names; this module
owns its own copy of the defaults so that a test can
check them against the product's ``cbaa_config_default``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cbaa_oracle.c")
LIB = os.path.join(HERE, "libcbaa_oracle.so")

MAX_ARR, MAX_RA, MAX_VA, MAX_PREFIX = 16, 8, 8, 16


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no vectorisation flags beyond -O2)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class OrcConfig(C.Structure):
    _fields_ = [
        ("r", C.c_uint32), ("num_ra", C.c_uint32), ("num_va", C.c_uint32), ("g", C.c_uint32),
        ("cbn", C.c_uint32 * MAX_ARR), ("clbs", C.c_uint32 * MAX_RA),
        ("mangle_a", C.c_uint32), ("mangle_b", C.c_uint32), ("bv_seed", C.c_uint32),
        ("va_seeds", C.c_uint32 * MAX_VA), ("theta_formula", C.c_int32), ("tuple_cap", C.c_uint64),
        ("direction", C.c_int32), ("n_prefix", C.c_uint32),
        ("prefix", C.c_uint32 * MAX_PREFIX), ("prefix_mask", C.c_uint32 * MAX_PREFIX),
        ("union_threshold", C.c_int32),
    ]


class OrcHost(C.Structure):
    _fields_ = [("ip", C.c_uint32), ("cs", C.c_uint32), ("lp", C.c_uint32), ("z", C.c_uint32),
                ("estimate", C.c_double)]


class OrcStats(C.Structure):
    _fields_ = [("ztot", C.c_uint64), ("eta", C.c_double), ("eps", C.c_double), ("theta_bn", C.c_double),
                ("zmax", C.c_uint32), ("n_hot", C.c_uint32 * MAX_RA), ("tuples", C.c_uint64),
                ("candidates", C.c_uint64), ("hits", C.c_uint64), ("overflow", C.c_int32), ("zmax_uc", C.c_uint32),
                ("theta_uc", C.c_double)]


HOST_DTYPE = np.dtype([("ip", "<u4"), ("cs", "<u4"), ("lp", "<u4"), ("z", "<u4"), ("estimate", "<f8")])


def default_params() -> dict:
    """Paper geometry (r=4, |RA|=3, |VA|=1, g=c=2^12) with the readings
    Q3 (mangling constants), Q4 (hash seeds) and Q8 (clbs = [0, 10, 20])."""
    return dict(r=4, num_ra=3, num_va=1, g=4096, cbn=[12, 12, 12, 12], clbs=[0, 10, 20],
                mangle_a=0x9E3779B1, mangle_b=0x7F4A7C15, bv_seed=0x85EBCA6B, va_seeds=[0xC2B2AE35],
                theta_formula=0, tuple_cap=1 << 24, direction=0, prefixes=[])


def to_struct(p: dict) -> OrcConfig:
    c = OrcConfig()
    c.r, c.num_ra, c.num_va, c.g = p["r"], p["num_ra"], p["num_va"], p["g"]
    for i, v in enumerate(p["cbn"]):
        c.cbn[i] = v
    for i, v in enumerate(p["clbs"]):
        c.clbs[i] = v
    c.mangle_a, c.mangle_b, c.bv_seed = p["mangle_a"], p["mangle_b"], p["bv_seed"]
    for i, v in enumerate(p["va_seeds"]):
        c.va_seeds[i] = v
    c.theta_formula = p.get("theta_formula", 0)
    c.tuple_cap = p.get("tuple_cap", 1 << 24)
    c.direction = p.get("direction", 0)
    c.union_threshold = p.get("union_threshold", 0)
    prefixes = p.get("prefixes", [])
    c.n_prefix = len(prefixes)
    for i, (pre, mask) in enumerate(prefixes):
        c.prefix[i], c.prefix_mask[i] = pre, mask
    return c


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        u32, u64, dbl, i32 = C.c_uint32, C.c_uint64, C.c_double, C.c_int32
        cfg = P(OrcConfig)
        sig = {
            "orc_mix32": (u32, [u32]),
            "orc_mangle": (u32, [cfg, u32]),
            "orc_unmangle": (u32, [cfg, u32]),
            "orc_inverse_mod32": (u32, [u32]),
            "orc_ep_cp": (None, [cfg, P(C.c_int32), P(C.c_int32)]),
            "orc_validate": (C.c_int, [cfg, C.c_char_p, C.c_int]),
            "orc_cs_bits": (u64, [cfg]),
            "orc_cube_bytes": (u64, [cfg]),
            "orc_bit_address": (u64, [cfg, u32, u32, u64, u32]),
            "orc_rp": (u32, [cfg, u32]),
            "orc_lp": (u32, [cfg, u32]),
            "orc_ra_col": (u32, [cfg, u32, u32]),
            "orc_va_col": (u32, [cfg, u32, u32]),
            "orc_row": (u32, [cfg, u32]),
            "orc_map_pair": (None, [cfg, u32, u32, P(u32), P(u32), P(u32)]),
            "orc_lp_from_tuple": (C.c_int, [cfg, P(u32), P(u32)]),
            "orc_normalize": (C.c_int, [cfg, u32, u32, P(u32), P(u32)]),
            "orc_update": (None, [cfg, C.c_void_p, C.c_void_p, C.c_void_p, u64, P(u64)]),
            "orc_merge": (None, [C.c_void_p, C.c_void_p, u64]),
            "orc_zero_count": (u32, [cfg, C.c_void_p, u32, u32, u64]),
            "orc_linear_estimate": (dbl, [dbl, dbl]),
            "orc_shared_bit_prob": (dbl, [cfg, dbl]),
            "orc_corrected_estimate": (dbl, [dbl, dbl, dbl]),
            "orc_hot_threshold": (dbl, [dbl, dbl, dbl, C.c_int]),
            "orc_union_threshold": (dbl, [dbl, dbl, dbl]),
            "orc_sparse_block_bytes": (u64, [C.c_void_p, u64, u64]),
            "orc_sparse_block_encode": (u64, [C.c_void_p, u64, u64, C.c_void_p]),
            "orc_sparse_block_decode": (C.c_int, [C.c_void_p, u64, C.c_void_p, u64, u64]),
            "orc_cs_load": (None, [cfg, C.c_void_p, u32, P(u64), P(dbl), P(dbl)]),
            "orc_zmax": (u32, [dbl, u32]),
            "orc_zero_counts_ra": (None, [cfg, C.c_void_p, C.c_void_p]),
            "orc_union_zeros": (u32, [cfg, C.c_void_p, u32, P(u32), u32]),
            "orc_detect": (C.c_int, [cfg, C.c_void_p, dbl, C.c_void_p, u64, P(u64), C.c_void_p]),
            "orc_candidates": (u64, [cfg, C.c_void_p, u32, u32, C.c_void_p, u64]),
            "orc_lp_roundtrip_failures": (u64, [cfg, u64, u64, C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- scalar API
def mix32(x: int) -> int:
    return lib().orc_mix32(x)


def mangle(p, x):
    return lib().orc_mangle(C.byref(to_struct(p)), x)


def unmangle(p, m):
    return lib().orc_unmangle(C.byref(to_struct(p)), m)


def inverse_mod32(a):
    return lib().orc_inverse_mod32(a)


def ep_cp(p):
    ep, cp = (C.c_int32 * MAX_RA)(), (C.c_int32 * MAX_RA)()
    lib().orc_ep_cp(C.byref(to_struct(p)), ep, cp)
    return list(ep[: p["num_ra"]]), list(cp[: p["num_ra"]])


def validate(p):
    buf = C.create_string_buffer(256)
    code = lib().orc_validate(C.byref(to_struct(p)), buf, 256)
    return code, buf.value.decode()


def cube_bytes(p) -> int:
    return lib().orc_cube_bytes(C.byref(to_struct(p)))


def cs_bits(p) -> int:
    return lib().orc_cs_bits(C.byref(to_struct(p)))


def bit_address(p, cs, a, col, row) -> int:
    return lib().orc_bit_address(C.byref(to_struct(p)), cs, a, col, row)


def ra_col(p, lp, i):
    return lib().orc_ra_col(C.byref(to_struct(p)), lp, i)


def va_col(p, lp, j):
    return lib().orc_va_col(C.byref(to_struct(p)), lp, j)


def row(p, moip):
    return lib().orc_row(C.byref(to_struct(p)), moip)


def map_pair(p, iip, oip):
    """(cs, [cols of all |RA|+|VA| arrays], row) of one pair (Alg. 1)."""
    cs, rw = C.c_uint32(), C.c_uint32()
    cols = (C.c_uint32 * MAX_ARR)()
    lib().orc_map_pair(C.byref(to_struct(p)), iip, oip, C.byref(cs), cols, C.byref(rw))
    return cs.value, list(cols[: p["num_ra"] + p["num_va"]]), rw.value


def lp_from_tuple(p, cols):
    arr = (C.c_uint32 * MAX_RA)(*cols)
    lp = C.c_uint32()
    ok = lib().orc_lp_from_tuple(C.byref(to_struct(p)), arr, C.byref(lp))
    return lp.value if ok else None


def normalize(p, src, dst):
    i, o = C.c_uint32(), C.c_uint32()
    ok = lib().orc_normalize(C.byref(to_struct(p)), src, dst, C.byref(i), C.byref(o))
    return (i.value, o.value) if ok else None


def linear_estimate(g, z):
    return lib().orc_linear_estimate(float(g), float(z))


def shared_bit_prob(p, eta):
    return lib().orc_shared_bit_prob(C.byref(to_struct(p)), float(eta))


def corrected_estimate(z, eps, g):
    return lib().orc_corrected_estimate(float(z), float(eps), float(g))


def hot_threshold(theta, eps, g, formula=0):
    return lib().orc_hot_threshold(float(theta), float(eps), float(g), formula)


def union_threshold(theta, eps, g):
    return lib().orc_union_threshold(float(theta), float(eps), float(g))


def zmax(theta_bn, g):
    return lib().orc_zmax(float(theta_bn), g)


# ----------------------------------------------------------------- array API
def new_cube(p) -> np.ndarray:
    return np.zeros(cube_bytes(p), dtype=np.uint8)


def update(p, src, dst, cube: np.ndarray | None = None):
    """Alg. 1 over a stream; returns (cube bytes, skipped pairs)."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    assert src.shape == dst.shape
    if cube is None:
        cube = new_cube(p)
    skipped = C.c_uint64()
    lib().orc_update(C.byref(to_struct(p)), _ptr(cube), _ptr(src), _ptr(dst), src.size, C.byref(skipped))
    return cube, skipped.value


def update_parallel(p, src, dst, threads: int | None = None):
    """Alg. 1 over a stream on `threads` host threads: each updates a private cube from a contiguous block,
    then the cubes are OR-merged (mergeCubes).  Equal to update() by the shard-OR invariant (S:105,
    pinned in tests/test_oracle_pins.py); only the wall time differs.  Returns the cube."""
    from concurrent.futures import ThreadPoolExecutor
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    threads = max(1, min(threads or os.cpu_count() or 1, max(1, src.size // 65536)))
    cuts = [src.size * t // threads for t in range(threads + 1)]
    with ThreadPoolExecutor(threads) as ex:   # ctypes drops the GIL inside orc_update
        cubes = list(ex.map(lambda t: update(p, src[cuts[t]:cuts[t + 1]], dst[cuts[t]:cuts[t + 1]])[0],
                            range(threads)))
    for c in cubes[1:]:
        merge(cubes[0], c)
    return cubes[0]


def merge(dst: np.ndarray, src: np.ndarray) -> np.ndarray:
    assert dst.size == src.size
    lib().orc_merge(_ptr(dst), _ptr(src), dst.size)
    return dst


def zero_count(p, cube, cs, a, col):
    return lib().orc_zero_count(C.byref(to_struct(p)), _ptr(cube), cs, a, col)


def cs_load(p, cube, cs):
    zt, eta, eps = C.c_uint64(), C.c_double(), C.c_double()
    lib().orc_cs_load(C.byref(to_struct(p)), _ptr(cube), cs, C.byref(zt), C.byref(eta), C.byref(eps))
    return zt.value, eta.value, eps.value


def zero_counts_ra(p, cube) -> np.ndarray:
    n = (1 << p["r"]) * sum(1 << p["cbn"][i] for i in range(p["num_ra"]))
    zc = np.zeros(n, dtype=np.uint32)
    lib().orc_zero_counts_ra(C.byref(to_struct(p)), _ptr(cube), _ptr(zc))
    return zc


def union_zeros(p, cube, cs, ra_cols, lp):
    arr = (C.c_uint32 * MAX_RA)(*ra_cols)
    return lib().orc_union_zeros(C.byref(to_struct(p)), _ptr(cube), cs, arr, lp)


def detect(p, cube, theta, cap: int = 1 << 20):
    """recoverAll: returns (status, hosts structured array, list of per-CS stats dicts)."""
    n_cs = 1 << p["r"]
    out = np.zeros(cap, dtype=HOST_DTYPE)
    stats = (OrcStats * n_cs)()
    n_out = C.c_uint64()
    st = lib().orc_detect(C.byref(to_struct(p)), _ptr(cube), float(theta), _ptr(out), cap, C.byref(n_out), stats)
    hosts = out[: min(n_out.value, cap)].copy()
    sdicts = []
    for s in stats:
        sdicts.append(dict(ztot=s.ztot, eta=s.eta, eps=s.eps, theta_bn=s.theta_bn, zmax=s.zmax,
                           theta_uc=s.theta_uc, zmax_uc=s.zmax_uc,
                           n_hot=list(s.n_hot[: p["num_ra"]]), tuples=s.tuples, candidates=s.candidates,
                           hits=s.hits, overflow=s.overflow))
    return st, hosts, sdicts


def candidates(p, cube, cs, zmax_, cap=1 << 22) -> np.ndarray:
    buf = np.zeros(cap, dtype=np.uint32)
    n = lib().orc_candidates(C.byref(to_struct(p)), _ptr(cube), cs, zmax_, _ptr(buf), cap)
    return buf[: min(n, cap)].copy()


def lp_roundtrip_failures(p, lo, hi, flip_cp=False) -> int:
    return lib().orc_lp_roundtrip_failures(C.byref(to_struct(p)), lo, hi, int(flip_cp))


# ----------------------------------------------------------------- SketchFile "CBA1"
def serialize(p, cube: np.ndarray) -> bytes:
    """SPEC's wire format, little-endian: magic "CBA1", u16 version 1, u8 r, u8 numRa, u8 numVa, u32 g,
    (numRa+numVa) × u8 cbn, numRa × u8 clbs, u32 mangleA, u32 mangleB, u32 bvSeed, numVa × u32 vaSeeds,
    u64 payload length, payload."""
    import struct
    narr = p["num_ra"] + p["num_va"]
    head = b"CBA1" + struct.pack("<HBBBI", 1, p["r"], p["num_ra"], p["num_va"], p["g"])
    head += bytes(p["cbn"][:narr]) + bytes(p["clbs"][: p["num_ra"]])
    head += struct.pack("<III", p["mangle_a"], p["mangle_b"], p["bv_seed"])
    head += struct.pack("<" + "I" * p["num_va"], *p["va_seeds"][: p["num_va"]])
    head += struct.pack("<Q", cube.size)
    return head + cube.tobytes()


def deserialize(data: bytes):
    """Inverse of serialize: (params dict of the sketch's identity, cube bytes)."""
    import struct
    if data[:4] != b"CBA1":
        raise ValueError("bad magic")
    version, r, nra, nva, g = struct.unpack_from("<HBBBI", data, 4)
    if version != 1:
        raise ValueError("bad version")
    off = 13
    cbn = list(data[off: off + nra + nva]); off += nra + nva
    clbs = list(data[off: off + nra]); off += nra
    a, b, bv = struct.unpack_from("<III", data, off); off += 12
    vs = list(struct.unpack_from("<" + "I" * nva, data, off)); off += 4 * nva
    (plen,) = struct.unpack_from("<Q", data, off); off += 8
    if len(data) - off != plen:
        raise ValueError(f"payload length {len(data) - off} != {plen}")
    p = dict(default_params(), r=r, num_ra=nra, num_va=nva, g=g, cbn=cbn, clbs=clbs, mangle_a=a, mangle_b=b,
             bv_seed=bv, va_seeds=vs)
    return p, np.frombuffer(data, dtype=np.uint8, offset=off).copy()

# ----------------------------------------------------------------- sparse SketchFile "CBA2"
SPARSE_BLOCK_BITS = 32768


def sparse_block_bytes(cube: np.ndarray, b: int) -> int:
    return lib().orc_sparse_block_bytes(_ptr(cube), cube.size, b)


def sparse_block_encode(cube: np.ndarray, b: int) -> bytes:
    buf = np.zeros(sparse_block_bytes(cube, b) + 1, np.uint8)
    n = lib().orc_sparse_block_encode(_ptr(cube), cube.size, b, _ptr(buf))
    return buf[:n].tobytes()


def serialize_sparse(p, cube: np.ndarray) -> bytes:
    """The sparse SketchFile: the CBA1 header with magic "CBA2" (its u64 = the dense cube
    length), u32 block bits (2^15), u64 block count, (blocks + 1) × u64 byte offsets of the blocks' varint
    streams, then the streams (each: LEB128 gaps between ascending set-bit positions of the block)."""
    import struct
    dense = serialize(p, cube[:0])
    head = b"CBA2" + dense[4:-8] + struct.pack("<Q", cube.size)
    nb = (cube.size * 8 + SPARSE_BLOCK_BITS - 1) // SPARSE_BLOCK_BITS
    streams = [sparse_block_encode(cube, b) for b in range(nb)]
    offs = [0]
    for st in streams:
        offs.append(offs[-1] + len(st))
    head += struct.pack("<IQ", SPARSE_BLOCK_BITS, nb) + struct.pack("<" + "Q" * (nb + 1), *offs)
    return head + b"".join(streams)


def deserialize_sparse(data: bytes, nbytes: int, header_bytes: int) -> np.ndarray:
    """The cube of a CBA2 file whose header (through the u64 dense length) is header_bytes long."""
    import struct
    bits, nb = struct.unpack_from("<IQ", data, header_bytes)
    assert bits == SPARSE_BLOCK_BITS
    offs = struct.unpack_from("<" + "Q" * (nb + 1), data, header_bytes + 12)
    base = header_bytes + 12 + 8 * (nb + 1)
    cube = np.zeros(nbytes, np.uint8)
    payload = np.frombuffer(data, np.uint8, offset=base)
    for b in range(nb):
        seg = np.ascontiguousarray(payload[offs[b]:offs[b + 1]])
        assert lib().orc_sparse_block_decode(_ptr(seg), seg.size, _ptr(cube), nbytes, b) == 0
    return cube
