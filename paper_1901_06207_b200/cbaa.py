"""Thin Python binding of libcbaa.so (include/cbaa.h): argument marshalling only.

Every step of the window path runs in the library's sm_100a kernels; this module
only converts torch tensors / numpy arrays into pointers, sizes and the current
CUDA stream.  If the library is missing the import fails loudly — there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcbaa.so")
LIB_PATH = os.environ.get("CBAA_LIB", LIB_PATH)   # A/B builds of the same sources (tools/)

MAX_RA, MAX_VA, MAX_ARRAYS, MAX_PREFIXES = 8, 8, 16, 16

OK = 0
E_CONFIG, E_ARG, E_CUDA, E_MISMATCH, E_CAPACITY, E_TUPLE_CAP, E_NOMEM = -1, -2, -3, -4, -5, -6, -7
THETA_PAPER, THETA_INVERTED = 0, 1
UNION_SAME, UNION_THM2 = 0, 1
DIR_NORMALIZED, DIR_INNER_PREFIX = 0, 1
UPDATE_TEST_SET, UPDATE_RED, UPDATE_BINNED = 0, 1, 2
SKETCH_REPLACE, SKETCH_MERGE = 0, 1


class Config(C.Structure):
    """cbaa_config (include/cbaa.h)."""
    _fields_ = [
        ("r", C.c_uint32), ("num_ra", C.c_uint32), ("num_va", C.c_uint32), ("g", C.c_uint32),
        ("cbn", C.c_uint8 * MAX_ARRAYS), ("clbs", C.c_uint8 * MAX_RA),
        ("mangle_a", C.c_uint32), ("mangle_b", C.c_uint32), ("bv_seed", C.c_uint32),
        ("va_seeds", C.c_uint32 * MAX_VA),
        ("theta_formula", C.c_int32), ("direction", C.c_int32), ("tuple_cap", C.c_uint64),
        ("n_prefixes", C.c_uint32), ("inner_prefix", C.c_uint32 * MAX_PREFIXES),
        ("inner_mask", C.c_uint32 * MAX_PREFIXES), ("update_passes", C.c_uint32), ("hit_capacity", C.c_uint32),
        ("update_mode", C.c_uint32), ("join_capacity", C.c_uint32), ("detect_overlap", C.c_uint32),
        ("bin_min_pairs", C.c_uint32), ("union_threshold", C.c_int32), ("reserved", C.c_uint32),
    ]

    def to_dict(self) -> dict:
        n = self.num_ra + self.num_va
        return dict(r=self.r, num_ra=self.num_ra, num_va=self.num_va, g=self.g, cbn=list(self.cbn[:n]),
                    clbs=list(self.clbs[: self.num_ra]), mangle_a=self.mangle_a, mangle_b=self.mangle_b,
                    bv_seed=self.bv_seed, va_seeds=list(self.va_seeds[: self.num_va]),
                    theta_formula=self.theta_formula, tuple_cap=self.tuple_cap, direction=self.direction,
                    union_threshold=self.union_threshold,
                    prefixes=[(self.inner_prefix[k], self.inner_mask[k]) for k in range(self.n_prefixes)])


class Host(C.Structure):
    _fields_ = [("ip", C.c_uint32), ("cs", C.c_uint32), ("lp", C.c_uint32), ("z", C.c_uint32),
                ("estimate", C.c_double)]


class CsStats(C.Structure):
    _fields_ = [("ztot", C.c_uint64), ("eta", C.c_double), ("eps", C.c_double), ("theta_bn", C.c_double),
                ("zmax", C.c_uint32), ("n_hot", C.c_uint32 * MAX_RA), ("tuples", C.c_uint64),
                ("candidates", C.c_uint64), ("hits", C.c_uint64), ("overflow", C.c_int32), ("zmax_uc", C.c_uint32),
                ("theta_uc", C.c_double)]


HOST_DTYPE = np.dtype([("ip", "<u4"), ("cs", "<u4"), ("lp", "<u4"), ("z", "<u4"), ("estimate", "<f8")])

# Every entry point of include/cbaa.h with its ctypes signature.
_P = C.POINTER
_h = C.c_void_p
_SIGS = {
    "cbaa_config_default": (C.c_int, [_P(Config)]),
    "cbaa_config_validate": (C.c_int, [_P(Config), C.c_char_p, C.c_uint64]),
    "cbaa_cube_bytes": (C.c_uint64, [_P(Config)]),
    "cbaa_create": (C.c_int, [_P(Config), C.c_int, _P(C.c_void_p)]),
    "cbaa_create_ext": (C.c_int, [_P(Config), C.c_int, C.c_void_p, C.c_uint64, _P(C.c_void_p)]),
    "cbaa_destroy": (None, [_h]),
    "cbaa_get_config": (C.c_int, [_h, _P(Config)]),
    "cbaa_reset": (C.c_int, [_h, C.c_void_p]),
    "cbaa_update": (C.c_int, [_h, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "cbaa_update_host": (C.c_int, [_h, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "cbaa_update_pairs": (C.c_int, [_h, C.c_void_p, C.c_uint64, C.c_void_p]),
    "cbaa_skipped": (C.c_int, [_h, _P(C.c_uint64), C.c_void_p]),
    "cbaa_merge": (C.c_int, [_h, _P(C.c_void_p), C.c_int, C.c_uint64, C.c_void_p]),
    "cbaa_merge_slice": (C.c_int, [_h, _P(C.c_void_p), C.c_int, C.c_uint32, C.c_uint32, C.c_void_p]),
    "cbaa_detect": (C.c_int, [_h, C.c_uint32, C.c_void_p, C.c_uint64, _P(C.c_uint64), C.c_void_p, C.c_void_p]),
    "cbaa_detect_range": (C.c_int, [_h, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64,
                                    _P(C.c_uint64), C.c_void_p, C.c_void_p]),
    "cbaa_cube_view": (C.c_int, [_h, _P(C.c_void_p), _P(C.c_uint64)]),
    "cbaa_zero_counts": (C.c_int, [_h, C.c_void_p, C.c_void_p]),
    "cbaa_hot_columns": (C.c_int, [_h, C.c_void_p, C.c_void_p]),
    "cbaa_set_record_candidates": (C.c_int, [_h, C.c_int, C.c_uint64]),
    "cbaa_candidates": (C.c_int, [_h, C.c_void_p, C.c_uint64, _P(C.c_uint64), C.c_void_p]),
    "cbaa_debug_map": (C.c_int, [_h, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    "cbaa_sketch_bytes": (C.c_uint64, [_h]),
    "cbaa_serialize": (C.c_int, [_h, C.c_void_p, C.c_uint64, _P(C.c_uint64), C.c_void_p]),
    "cbaa_serialize_sparse": (C.c_int, [_h, C.c_void_p, C.c_uint64, _P(C.c_uint64), C.c_void_p]),
    "cbaa_sketch_config": (C.c_int, [C.c_void_p, C.c_uint64, _P(Config), C.c_char_p, C.c_uint64]),
    "cbaa_deserialize": (C.c_int, [_h, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]),
    "cbaa_ipc_export": (C.c_int, [_h, C.c_void_p]),
    "cbaa_ipc_open": (C.c_int, [_h, C.c_void_p, _P(C.c_void_p)]),
    "cbaa_ipc_close": (C.c_int, [_h, C.c_void_p]),
    "cbaa_signal_offset": (C.c_uint64, [_h]),
    "cbaa_peer_barrier": (C.c_int, [_h, _P(C.c_void_p), C.c_int, C.c_int, C.c_uint64, C.c_void_p]),
    "cbaa_peer_status": (C.c_int, [_h, _P(C.c_uint32)]),
    "cbaa_merge_slice_zc": (C.c_int, [_h, _P(C.c_void_p), C.c_int, C.c_uint32, C.c_uint32, C.c_void_p]),
    "cbaa_merge_multicast": (C.c_int, [_h, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]),
    "cbaa_sort_hosts": (None, [C.c_void_p, C.c_uint64]),
    "cbaa_kernel_launches": (C.c_uint64, [_h]),
    "cbaa_update_passes": (C.c_uint32, [_h]),
    "cbaa_set_phase_timing": (C.c_int, [_h, C.c_int]),
    "cbaa_update_phase_ms": (C.c_int, [_h, _P(C.c_double), C.c_int, _P(C.c_uint64)]),
    "cbaa_update_plan": (C.c_int, [_h, C.c_uint64, C.c_char_p, C.c_uint64]),
    "cbaa_strerror": (C.c_char_p, [C.c_int]),
    "cbaa_last_error": (C.c_char_p, [_h]),
}

_lib = None


def lib():
    """Load libcbaa.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


class CbaaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{msg} (code {code}: {lib().cbaa_strerror(code).decode()})")
        self.code = code


def default_config() -> Config:
    c = Config()
    lib().cbaa_config_default(C.byref(c))
    return c


def config_from_dict(p: dict) -> Config:
    """Build a cbaa_config from a plain parameter dict (the SPEC's field names)."""
    c = default_config()
    c.r, c.num_ra, c.num_va, c.g = p["r"], p["num_ra"], p["num_va"], p["g"]
    for i in range(MAX_ARRAYS):
        c.cbn[i] = p["cbn"][i] if i < len(p["cbn"]) else 0
    for i in range(MAX_RA):
        c.clbs[i] = p["clbs"][i] if i < len(p["clbs"]) else 0
    c.mangle_a, c.mangle_b, c.bv_seed = p["mangle_a"], p["mangle_b"], p["bv_seed"]
    for j in range(MAX_VA):
        c.va_seeds[j] = p["va_seeds"][j] if j < len(p["va_seeds"]) else 0
    c.theta_formula = p.get("theta_formula", THETA_PAPER)
    c.tuple_cap = p.get("tuple_cap", 1 << 24)
    c.direction = p.get("direction", DIR_NORMALIZED)
    prefixes = p.get("prefixes", [])
    c.n_prefixes = len(prefixes)
    for k, (pre, mask) in enumerate(prefixes):
        c.inner_prefix[k], c.inner_mask[k] = pre, mask
    c.update_passes = p.get("update_passes", 0)
    c.hit_capacity = p.get("hit_capacity", 0)
    c.update_mode = p.get("update_mode", UPDATE_BINNED)
    c.join_capacity = p.get("join_capacity", 0)
    c.detect_overlap = p.get("detect_overlap", 0)
    c.bin_min_pairs = p.get("bin_min_pairs", 0)
    c.union_threshold = p.get("union_threshold", UNION_SAME)
    return c


def validate(cfg: Config):
    buf = C.create_string_buffer(256)
    rc = lib().cbaa_config_validate(C.byref(cfg), buf, 256)
    return rc, buf.value.decode()


def cube_bytes(cfg: Config) -> int:
    return lib().cbaa_cube_bytes(C.byref(cfg))


def sketch_config(data: bytes):
    """Geometry and seeds of a SketchFile "CBA1"; raises CbaaError naming the bad field."""
    c = Config()
    err = C.create_string_buffer(256)
    buf = C.create_string_buffer(bytes(data), len(data)) if not isinstance(data, np.ndarray) else None
    ptr = C.cast(buf, C.c_void_p) if buf is not None else C.c_void_p(data.ctypes.data)
    rc = lib().cbaa_sketch_config(ptr, len(data), C.byref(c), err, 256)
    if rc != OK:
        raise CbaaError(rc, "SketchFile: " + err.value.decode())
    return c


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dptr(t, what):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA tensor")
    if t.dtype not in (torch.int32, torch.uint32):
        raise TypeError(f"{what} must be int32/uint32 (IPv4 as 32-bit words), got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return C.c_void_p(t.data_ptr())


class Cbaa:
    """One cube of bits arrays on one GPU (a local server's CBA)."""

    def __init__(self, cfg: Config | dict | None = None, device: int = 0, cube=None):
        """cube: optional caller-owned uint8 CUDA tensor (e.g. torch symmetric memory) to hold the cube."""
        if cfg is None:
            cfg = default_config()
        elif isinstance(cfg, dict):
            cfg = config_from_dict(cfg)
        self.cfg = cfg
        self.device = device
        self._ext = cube          # keeps caller memory alive as long as the handle
        h = C.c_void_p()
        if cube is None:
            rc = lib().cbaa_create(C.byref(cfg), device, C.byref(h))
        else:
            rc = lib().cbaa_create_ext(C.byref(cfg), device, C.c_void_p(cube.data_ptr()),
                                       cube.numel() * cube.element_size(), C.byref(h))
        if rc != OK:
            raise CbaaError(rc, "cbaa_create failed: " + validate(cfg)[1])
        self._h = h
        self.n_cs = 1 << cfg.r

    def close(self):
        if getattr(self, "_h", None):
            lib().cbaa_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what, allow=()):
        if rc != OK and rc not in allow:
            raise CbaaError(rc, f"{what}: {lib().cbaa_last_error(self._h).decode()}")
        return rc

    # ---------------------------------------------------------------- window ops
    def reset(self, stream=None):
        self._check(lib().cbaa_reset(self._h, _stream(stream)), "cbaa_reset")

    def update(self, src, dst, stream=None):
        """Alg. 1 over device tensors src (inner) / dst (outer)."""
        if src.numel() != dst.numel():
            raise ValueError("src and dst differ in length")
        self._check(lib().cbaa_update(self._h, _dptr(src, "src"), _dptr(dst, "dst"), src.numel(), _stream(stream)),
                    "cbaa_update")

    def update_pairs(self, pairs, stream=None):
        """Alg. 1 over one device tensor of interleaved (src, dst) pairs, shape (n, 2) or (2n,)."""
        n = pairs.numel() // 2
        self._check(lib().cbaa_update_pairs(self._h, _dptr(pairs, "pairs"), n, _stream(stream)), "cbaa_update_pairs")

    def update_host(self, src, dst, stream=None):
        """Alg. 1 over HOST arrays (numpy or CPU tensors, ideally pinned): pipelined H2D inside the library."""
        import torch
        keep, ptrs = [], []   # converted copies stay referenced until the library call returns
        for a in (src, dst):
            if isinstance(a, torch.Tensor):
                if a.is_cuda or not a.is_contiguous() or a.dtype not in (torch.int32, torch.uint32):
                    raise TypeError("update_host needs contiguous int32/uint32 CPU tensors")
                keep.append(a)
                ptrs.append(a.data_ptr())
            else:
                a = np.ascontiguousarray(a)
                if a.dtype not in (np.dtype(np.uint32), np.dtype(np.int32)):
                    raise TypeError(f"update_host needs int32/uint32 arrays, got {a.dtype}")
                keep.append(a)
                ptrs.append(a.ctypes.data)
        if len(keep[0]) != len(keep[1]):
            raise ValueError(f"src and dst differ in length ({len(keep[0])} vs {len(keep[1])})")
        n = len(keep[0])
        self._check(lib().cbaa_update_host(self._h, C.c_void_p(ptrs[0]), C.c_void_p(ptrs[1]), n, _stream(stream)),
                    "cbaa_update_host")
        del keep

    def skipped(self, stream=None) -> int:
        v = C.c_uint64()
        self._check(lib().cbaa_skipped(self._h, C.byref(v), _stream(stream)), "cbaa_skipped")
        return v.value

    def merge(self, cubes, stream=None):
        """cube |= OR of the given device cubes (uint8 tensors of cube_bytes, or other Cbaa handles)."""
        ptrs = [(c.cube_ptr() if isinstance(c, Cbaa) else c.data_ptr()) for c in cubes]
        arr = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        self._check(lib().cbaa_merge(self._h, arr, len(ptrs), self.nbytes, _stream(stream)), "cbaa_merge")

    def merge_slice(self, slices, cs_lo, cs_hi, stream=None):
        """OR the bytes of CSs [cs_lo, cs_hi) of peer cubes into this cube: each slice is a uint8 CUDA
        tensor or a raw device address (e.g. a peer's symmetric-memory pointer, read over NVLink)."""
        ptrs = [s if isinstance(s, int) else s.data_ptr() for s in slices]
        arr = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        self._check(lib().cbaa_merge_slice(self._h, arr, len(ptrs), cs_lo, cs_hi, _stream(stream)),
                    "cbaa_merge_slice")

    def merge_slice_zc(self, slices, cs_lo, cs_hi, stream=None):
        """merge_slice fused with the window-end zero counts of [cs_lo, cs_hi) (cbaa_merge_slice_zc)."""
        ptrs = [s if isinstance(s, int) else s.data_ptr() for s in slices]
        arr = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        self._check(lib().cbaa_merge_slice_zc(self._h, arr, len(ptrs), cs_lo, cs_hi, _stream(stream)),
                    "cbaa_merge_slice_zc")

    def merge_multicast(self, mc_cube: int, cs_lo, cs_hi, stream=None):
        """NVLS OR of every rank's bytes of CSs [cs_lo, cs_hi) through a multicast address (cbaa_merge_multicast)."""
        self._check(lib().cbaa_merge_multicast(self._h, C.c_void_p(mc_cube), cs_lo, cs_hi, _stream(stream)),
                    "cbaa_merge_multicast")

    # ------------------------------------------------------------ device-side router barrier
    @property
    def signal_offset(self) -> int:
        return lib().cbaa_signal_offset(self._h)

    def peer_barrier(self, peer_cubes, world: int, rank: int, epoch: int, stream=None):
        """Stream-ordered device barrier over the peers' signal areas (cbaa_peer_barrier); peer_cubes[k] =
        rank k's cube base as mapped here (ignored for k == rank)."""
        arr = (C.c_void_p * world)(*[p or 0 for p in peer_cubes])
        self._check(lib().cbaa_peer_barrier(self._h, arr, world, rank, epoch, _stream(stream)), "cbaa_peer_barrier")

    def peer_status(self) -> int:
        v = C.c_uint32()
        self._check(lib().cbaa_peer_status(self._h, C.byref(v)), "cbaa_peer_status")
        return v.value

    def detect(self, theta: int, cap: int = 1 << 20, cs_lo: int = 0, cs_hi: int | None = None, stream=None,
               raise_on_overflow: bool = False, with_stats: bool = True):
        """Window end: returns (hosts structured array, per-CS stats list or None, status code)."""
        cs_hi = self.n_cs if cs_hi is None else cs_hi
        out = getattr(self, "_out", None)
        if out is None or out.size < max(cap, 1):
            out = self._out = np.empty(max(cap, 1), dtype=HOST_DTYPE)   # reused across windows
        stats = (CsStats * (cs_hi - cs_lo))() if with_stats else None
        n = C.c_uint64()
        rc = lib().cbaa_detect_range(self._h, theta, cs_lo, cs_hi, out.ctypes.data_as(C.c_void_p), cap,
                                     C.byref(n), stats, _stream(stream))
        allow = () if raise_on_overflow else (E_TUPLE_CAP,)
        self._check(rc, "cbaa_detect", allow=allow)
        hosts = out[: min(n.value, cap)].copy()
        if stats is None:
            return hosts, None, rc
        sd = [dict(ztot=s.ztot, eta=s.eta, eps=s.eps, theta_bn=s.theta_bn, zmax=s.zmax, zmax_uc=s.zmax_uc,
                   theta_uc=s.theta_uc,
                   n_hot=list(s.n_hot[: self.cfg.num_ra]), tuples=s.tuples, candidates=s.candidates, hits=s.hits,
                   overflow=s.overflow) for s in stats]
        return hosts, sd, rc

    # ---------------------------------------------------------------- inspection
    @property
    def nbytes(self) -> int:
        p, n = C.c_void_p(), C.c_uint64()
        self._check(lib().cbaa_cube_view(self._h, C.byref(p), C.byref(n)), "cbaa_cube_view")
        return n.value

    def cube_ptr(self) -> int:
        p, n = C.c_void_p(), C.c_uint64()
        self._check(lib().cbaa_cube_view(self._h, C.byref(p), C.byref(n)), "cbaa_cube_view")
        return p.value

    def cube(self):
        """The device cube as a torch.uint8 tensor view (no copy; valid while the handle lives)."""
        import torch
        p, n = C.c_void_p(), C.c_uint64()
        self._check(lib().cbaa_cube_view(self._h, C.byref(p), C.byref(n)), "cbaa_cube_view")
        return _wrap_device(p.value, n.value, self.device, self)

    def zero_counts(self, stream=None):
        import torch
        n = self.n_cs * sum(1 << self.cfg.cbn[i] for i in range(self.cfg.num_ra))
        out = torch.empty(n, dtype=torch.int32, device=f"cuda:{self.device}")
        self._check(lib().cbaa_zero_counts(self._h, C.c_void_p(out.data_ptr()), _stream(stream)), "cbaa_zero_counts")
        return out

    def hot_columns(self, stream=None) -> np.ndarray:
        n = self.n_cs * sum(1 << self.cfg.cbn[i] for i in range(self.cfg.num_ra))
        out = np.zeros(n, dtype=np.uint32)
        self._check(lib().cbaa_hot_columns(self._h, out.ctypes.data_as(C.c_void_p), _stream(stream)),
                    "cbaa_hot_columns")
        return out

    def record_candidates(self, enable=True, capacity=1 << 22):
        self._check(lib().cbaa_set_record_candidates(self._h, int(enable), capacity), "cbaa_set_record_candidates")

    def candidates(self, cap=1 << 22, stream=None) -> np.ndarray:
        out = np.zeros(cap, dtype=np.uint64)
        n = C.c_uint64()
        self._check(lib().cbaa_candidates(self._h, out.ctypes.data_as(C.c_void_p), cap, C.byref(n), _stream(stream)),
                    "cbaa_candidates")
        return out[: min(n.value, cap)]

    def debug_map(self, iip, oip, stream=None):
        import torch
        n = iip.numel()
        narr = self.cfg.num_ra + self.cfg.num_va
        dev = iip.device
        cs = torch.empty(n, dtype=torch.int32, device=dev)
        cols = torch.empty(n * narr, dtype=torch.int32, device=dev)
        row = torch.empty(n, dtype=torch.int32, device=dev)
        self._check(lib().cbaa_debug_map(self._h, _dptr(iip, "iip"), _dptr(oip, "oip"), n, C.c_void_p(cs.data_ptr()),
                                         C.c_void_p(cols.data_ptr()), C.c_void_p(row.data_ptr()), _stream(stream)),
                    "cbaa_debug_map")
        return cs, cols.view(n, narr), row

    # ------------------------------------------------------------ SketchFile
    def serialize(self, stream=None) -> np.ndarray:
        """The cube as a SketchFile "CBA1", uint8 numpy array."""
        n = lib().cbaa_sketch_bytes(self._h)
        out = np.empty(n, dtype=np.uint8)
        w = C.c_uint64()
        self._check(lib().cbaa_serialize(self._h, out.ctypes.data_as(C.c_void_p), n, C.byref(w), _stream(stream)),
                    "cbaa_serialize")
        return out

    def serialize_sparse(self, stream=None) -> np.ndarray:
        """The cube as a sparse SketchFile "CBA2" (cbaa_serialize_sparse), uint8 numpy array."""
        w = C.c_uint64()
        rc = lib().cbaa_serialize_sparse(self._h, None, 0, C.byref(w), _stream(stream))
        self._check(rc, "cbaa_serialize_sparse", allow=(E_CAPACITY,))
        out = np.empty(w.value, dtype=np.uint8)
        self._check(lib().cbaa_serialize_sparse(self._h, out.ctypes.data_as(C.c_void_p), w.value, C.byref(w),
                                                _stream(stream)), "cbaa_serialize_sparse")
        return out

    def deserialize(self, data, merge: bool = False, stream=None):
        """Load (or OR-merge) a SketchFile into the cube; refuses a different geometry/seeds."""
        a = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        a = np.ascontiguousarray(a)
        self._check(lib().cbaa_deserialize(self._h, a.ctypes.data_as(C.c_void_p), a.size,
                                           SKETCH_MERGE if merge else SKETCH_REPLACE, _stream(stream)),
                    "cbaa_deserialize")

    # ------------------------------------------------------------ peer cubes (CUDA IPC)
    def ipc_export(self) -> bytes:
        buf = C.create_string_buffer(64)
        self._check(lib().cbaa_ipc_export(self._h, buf), "cbaa_ipc_export")
        return buf.raw

    def ipc_open(self, handle: bytes) -> int:
        p = C.c_void_p()
        buf = C.create_string_buffer(bytes(handle), 64)
        self._check(lib().cbaa_ipc_open(self._h, buf, C.byref(p)), "cbaa_ipc_open")
        return p.value

    def ipc_close(self, ptr: int):
        self._check(lib().cbaa_ipc_close(self._h, C.c_void_p(ptr)), "cbaa_ipc_close")

    @property
    def kernel_launches(self) -> int:
        return lib().cbaa_kernel_launches(self._h)

    @property
    def update_passes(self) -> int:
        return lib().cbaa_update_passes(self._h)

    def set_phase_timing(self, enable: bool = True):
        """Event pairs around every update kernel (cbaa_set_phase_timing)."""
        self._check(lib().cbaa_set_phase_timing(self._h, int(enable)), "cbaa_set_phase_timing")

    def update_plan(self, n: int) -> str:
        """The kernels an update of n pairs launches, per phase (cbaa_update_plan)."""
        buf = C.create_string_buffer(256)
        self._check(lib().cbaa_update_plan(self._h, n, buf, 256), "cbaa_update_plan")
        return buf.value.decode()

    def update_phase_ms(self):
        """(ms per phase summed since the last query, update calls): binned [count, starts, scatter, apply],
        direct [k_update, 0, 0, 0] (cbaa_update_phase_ms; synchronizes the recorded events)."""
        ms = (C.c_double * 4)()
        calls = C.c_uint64()
        self._check(lib().cbaa_update_phase_ms(self._h, ms, 4, C.byref(calls)), "cbaa_update_phase_ms")
        return list(ms), calls.value


def sort_hosts(hosts: np.ndarray) -> np.ndarray:
    """The S:418 output order (estimate descending, ip ascending) of a host array, in the library
    (cbaa_sort_hosts); returns a sorted copy."""
    out = np.ascontiguousarray(hosts, dtype=HOST_DTYPE).copy()
    lib().cbaa_sort_hosts(out.ctypes.data_as(C.c_void_p), out.size)
    return out


def _wrap_device(ptr: int, nbytes: int, device: int, owner):
    """Zero-copy torch.uint8 view of library-owned device memory (via __cuda_array_interface__)."""
    import torch

    class _Mem:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                    "strides": None, "stream": None}

    t = torch.as_tensor(_Mem(), device=f"cuda:{device}")
    t._cbaa_owner = owner   # keep the handle alive while the view lives
    return t
