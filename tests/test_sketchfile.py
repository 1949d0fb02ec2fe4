"""SketchFile "CBA1": the cross-router transport of a local CBA.

CPU tests: the library's header parser against the oracle's serializer (written separately from S:479).
GPU tests: device cube → file bytes identical to the oracle's file; REPLACE / MERGE round trips;
globalMerge of router files == the oracle cube of the whole stream; refusals name the field."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import cbaa as cb
from paper_1901_06207_b200 import workload as W
from tests.geometries import random_params


def test_header_parse_matches_oracle_serializer(paper):
    for p in [paper] + [random_params(s) for s in range(10)]:
        data = O.serialize(p, np.zeros(O.cube_bytes(p), np.uint8))
        c = cb.sketch_config(data)
        d = c.to_dict()
        for k in ("r", "num_ra", "num_va", "g", "cbn", "clbs", "mangle_a", "mangle_b", "bv_seed", "va_seeds"):
            assert d[k] == p[k], k


def test_paper_geometry_file_size(paper):
    """the paper-config sketch is exactly 128 MiB of payload."""
    data = O.serialize(paper, np.zeros(O.cube_bytes(paper), np.uint8))
    assert len(data) - (1 << 27) == 4 + 2 + 3 + 4 + 4 + 3 + 12 + 4 + 8


@pytest.mark.parametrize("mutate, field", [
    (lambda b: b"XBA1" + b[4:], "magic"),
    (lambda b: b[:4] + b"\x02\x00" + b[6:], "version"),
    (lambda b: b[:-1], "payload truncated"),
    (lambda b: b[:20], "truncated"),
])
def test_header_errors_name_the_field(paper, mutate, field):
    p = dict(paper, r=8, g=32, cbn=[9, 9, 9, 8], clbs=[0, 8, 16])
    data = O.serialize(p, np.zeros(O.cube_bytes(p), np.uint8))
    with pytest.raises(cb.CbaaError) as e:
        cb.sketch_config(mutate(data))
    assert field in str(e.value)


def test_oracle_roundtrip(paper):
    p = dict(paper, r=8, g=64, cbn=[9, 9, 9, 8], clbs=[0, 8, 16])
    src, dst = W.random_pairs(5000, 3)
    cube, _ = O.update(p, src, dst)
    q, back = O.deserialize(O.serialize(p, cube))
    assert np.array_equal(back, cube) and q["va_seeds"] == p["va_seeds"]


@pytest.mark.gpu
def test_gpu_file_equals_oracle_file_and_global_merge(paper):
    import torch
    from tests.test_gpu_parity import dev, gpu_cube, handle
    w = W.generate(W.WindowSpec(n=400_000, n_hosts=8000, n_flows=50000, scanners=(2000,) * 3), 12)
    part = W.partition(w.src.size, 4, "hash-by-pair", w.src, w.dst)
    files = []
    for k in range(4):
        sel = part == k
        h = handle(paper)
        h.reset()
        h.update(dev(w.src[sel]), dev(w.dst[sel]))
        f = h.serialize()
        ref, _ = O.update(paper, w.src[sel], w.dst[sel])
        assert f.tobytes() == O.serialize(paper, ref)            # device file == oracle file, byte for byte
        files.append(f)
    g = handle(paper)
    g.reset()
    for f in files:
        g.deserialize(f, merge=True)                             # globalMerge
    whole, _ = O.update(paper, w.src, w.dst)
    assert np.array_equal(gpu_cube(g), whole)
    r = handle(paper)
    r.deserialize(files[0])                                      # REPLACE
    assert np.array_equal(gpu_cube(r), np.frombuffer(files[0].tobytes()[-(1 << 27):], np.uint8))
    other = handle(dict(paper, bv_seed=paper["bv_seed"] ^ 1))
    with pytest.raises(cb.CbaaError) as e:
        other.deserialize(files[0], merge=True)
    assert e.value.code == cb.E_MISMATCH and "bv_seed" in str(e.value)


ODD = dict(r=6, num_ra=2, num_va=2, g=64, cbn=[14, 13, 5, 7], clbs=[0, 13], mangle_a=0x12345679,
           mangle_b=0xDEADBEEF, bv_seed=0x01020304, va_seeds=[0xA5A5A5A5, 0x0BADF00D], theta_formula=0,
           tuple_cap=1 << 24, direction=0)


def _golden_headers(golden):
    g = golden("sketch_headers.txt")
    return {k: bytes(v[0]) for k, v in g.items()}


@pytest.mark.parametrize("name", ["paper", "odd"])
def test_header_golden_bytes(paper, golden, name):
    """The serializer's header equals the hand-assembled bytes of S:479 (tests/golden/sketch_headers.txt),
    and the library's parser reads those bytes back to the same geometry and seeds."""
    p = paper if name == "paper" else dict(paper, **ODD)
    want = _golden_headers(golden)[name]
    data = O.serialize(p, np.zeros(O.cube_bytes(p), np.uint8))
    assert data[:len(want)] == want
    assert len(data) == len(want) + O.cube_bytes(p)
    c = cb.sketch_config(want + bytes(O.cube_bytes(p))).to_dict()
    for k in ("r", "num_ra", "num_va", "g", "cbn", "clbs", "mangle_a", "mangle_b", "bv_seed", "va_seeds"):
        assert c[k] == p[k], k


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["paper", "odd"])
def test_device_file_header_golden(paper, golden, name):
    """cbaa_serialize's header from a device cube equals the hand-assembled bytes."""
    torch = pytest.importorskip("torch")
    p = paper if name == "paper" else dict(paper, **ODD)
    h = cb.Cbaa(cb.config_from_dict(p), 0)
    h.reset()
    torch.cuda.synchronize()
    want = _golden_headers(golden)[name]
    data = h.serialize()
    assert bytes(data[:len(want)]) == want and not data[len(want):].any()


# ------------------------------------------------------------------ sparse SketchFile "CBA2"
def _bits_cube(nbytes, positions):
    c = np.zeros(nbytes, np.uint8)
    for pos in positions:
        c[pos >> 3] |= np.uint8(1 << (pos & 7))
    return c


def test_sparse_block_streams_golden(golden):
    """The oracle's block encoding equals the hand-computed LEB128 gap streams (tests/golden)."""
    g = {k: bytes(v[0]) for k, v in golden("sparse_blocks.txt").items()}
    cube = _bits_cube(3 * 4096, [0, 1, 130, 32767] + [32768 + q for q in (5, 6, 127, 16384)])
    assert O.sparse_block_encode(cube, 0) == g["block0"]
    assert O.sparse_block_encode(cube, 1) == g["block1"]
    assert O.sparse_block_encode(cube, 2) == b""


@pytest.mark.parametrize("density", [0.0, 0.001, 0.034, 0.5, 1.0])
def test_sparse_roundtrip_and_size(paper, density):
    """CBA2 round trip is bit-identical; stream bytes == Σ LEB128 lengths of the gaps counted in numpy;
    a ragged last block (cube not a multiple of 4 KiB)."""
    p = dict(paper, r=2, g=64, cbn=[10, 10, 10, 6], clbs=[0, 10, 20])   # 2^2·(3·1024 + 64)·64/8 = 100352 B
    assert O.validate(p)[0] == 0
    n = O.cube_bytes(p)
    rng = np.random.default_rng(7)
    bits = rng.random(n * 8) < density
    cube = np.packbits(bits, bitorder="little")
    data = O.serialize_sparse(p, cube)
    hb = len(O.serialize(p, cube[:0]))
    assert data[:4] == b"CBA2"
    assert np.array_equal(O.deserialize_sparse(data, n, hb), cube)
    want = 0
    for b0 in range(0, n * 8, 32768):
        pos = np.nonzero(bits[b0:b0 + 32768])[0]
        gaps = np.diff(np.concatenate([[-1], pos])) - 1
        want += int(np.sum(1 + (gaps >= 128) + (gaps >= 1 << 14) + (gaps >= 1 << 21)))
    nb = -(-n * 8 // 32768)
    assert len(data) == hb + 12 + 8 * (nb + 1) + want


def test_sparse_header_parsed_by_library(paper):
    """cbaa_sketch_config reads the oracle's CBA2 header; broken offsets or streams are refused by name."""
    p = dict(paper, **ODD)
    n = O.cube_bytes(p)
    cube = np.packbits(np.random.default_rng(3).random(n * 8) < 0.01, bitorder="little")
    data = O.serialize_sparse(p, cube)
    d = cb.sketch_config(data).to_dict()
    for k in ("r", "num_ra", "num_va", "g", "cbn", "clbs", "mangle_a", "mangle_b", "bv_seed", "va_seeds"):
        assert d[k] == p[k], k
    hb = len(O.serialize(p, cube[:0]))
    for mutate, field in [(lambda b: b[:hb] + b"\x00\x40\x00\x00" + b[hb + 4:], "block bits"),
                          (lambda b: b[:hb + 12] + b"\x01" + b[hb + 13:], "offsets"),
                          (lambda b: b[:-3], "truncated")]:
        with pytest.raises(cb.CbaaError) as e:
            cb.sketch_config(mutate(data))
        assert field in str(e.value), (field, str(e.value))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["paper", "odd"])
def test_device_sparse_file_matches_oracle(paper, name):
    """cbaa_serialize_sparse on the device == the oracle's CBA2 bytes; REPLACE and MERGE of the file
    reproduce the cube; a corrupted stream is refused."""
    torch = pytest.importorskip("torch")
    p = paper if name == "paper" else dict(paper, **ODD)
    w = W.generate(W.C1, 12)
    h = cb.Cbaa(cb.config_from_dict(p), 0)
    h.reset()
    h.update(torch.from_numpy(w.src.view(np.int32)).cuda(), torch.from_numpy(w.dst.view(np.int32)).cuda())
    torch.cuda.synchronize()
    ref, _ = O.update(p, w.src, w.dst)
    data = h.serialize_sparse()
    want = O.serialize_sparse(p, ref)
    assert data.tobytes() == want
    assert len(want) < O.cube_bytes(p)            # C1 at these geometries: sparse is smaller
    g = cb.Cbaa(cb.config_from_dict(p), 0)
    g.reset()
    g.deserialize(data)
    torch.cuda.synchronize()
    assert np.array_equal(g.cube().cpu().numpy(), ref)
    g.deserialize(O.serialize(p, ref), merge=True)   # MERGE of the same bits: unchanged
    torch.cuda.synchronize()
    assert np.array_equal(g.cube().cpu().numpy(), ref)
    h.reset()
    h.deserialize(data, merge=True)
    torch.cuda.synchronize()
    assert np.array_equal(h.cube().cpu().numpy(), ref)
    bad = bytearray(want)
    bad[-1] = 0x80                                 # last varint left unterminated
    with pytest.raises(cb.CbaaError):
        g.deserialize(bytes(bad))
