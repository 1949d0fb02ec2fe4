"""CPU checks of the C ABI boundary: the library loads, exports every symbol include/cbaa.h declares, its
structs match the ctypes binding byte for byte, and its host-only logic (defaults, validation, sizes)
agrees with the oracle.  No compute call needs a GPU here."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import cbaa as cb
from tests.conftest import ROOT
from tests.geometries import random_params

HEADER = os.path.join(ROOT, "include", "cbaa.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cbaa_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 20
    L = cb.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(cb._SIGS), set(names) ^ set(cb._SIGS)
    out = subprocess.run(["nm", "-D", "--defined-only", cb.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cbaa_\w+)", out))
    assert set(names) <= exported


LAYOUT_C = r"""
#include <stddef.h>
#include <stdio.h>
#include "cbaa.h"
#define F(T, f) printf(#T " " #f " %zu\n", offsetof(T, f));
int main(void) {
  printf("cbaa_config size %zu\n", sizeof(cbaa_config));
  printf("cbaa_cs_stats size %zu\n", sizeof(cbaa_cs_stats));
  printf("cbaa_host size %zu\n", sizeof(cbaa_host));
  F(cbaa_config, cbn) F(cbaa_config, clbs) F(cbaa_config, mangle_a) F(cbaa_config, va_seeds)
  F(cbaa_config, theta_formula) F(cbaa_config, tuple_cap) F(cbaa_config, n_prefixes) F(cbaa_config, inner_mask)
  F(cbaa_config, update_passes) F(cbaa_config, hit_capacity) F(cbaa_config, union_threshold)
  F(cbaa_cs_stats, zmax) F(cbaa_cs_stats, n_hot) F(cbaa_cs_stats, tuples) F(cbaa_cs_stats, overflow)
  F(cbaa_cs_stats, zmax_uc) F(cbaa_cs_stats, theta_uc)
  F(cbaa_host, z) F(cbaa_host, estimate)
  return 0;
}
"""


def test_struct_layout_matches_binding():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(src, "w").write(LAYOUT_C)
        subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-o", exe, src])
        lines = subprocess.check_output([exe], text=True).split("\n")
    types = {"cbaa_config": cb.Config, "cbaa_cs_stats": cb.CsStats, "cbaa_host": cb.Host}
    for line in filter(None, lines):
        t, f, v = line.split()
        if f == "size":
            assert C.sizeof(types[t]) == int(v), line
        else:
            assert getattr(types[t], f).offset == int(v), line


def test_defaults_agree_with_oracle():
    """Both sides state Q3/Q4/Q8 and P:437 independently; they must agree."""
    d = cb.default_config().to_dict()
    o = O.default_params()
    for k in ("r", "num_ra", "num_va", "g", "cbn", "clbs", "mangle_a", "mangle_b", "bv_seed", "va_seeds",
              "theta_formula", "tuple_cap", "direction"):
        assert d[k] == o[k], k
    assert cb.cube_bytes(cb.default_config()) == O.cube_bytes(o) == 1 << 27


def test_validation_agrees_with_oracle():
    rng = np.random.default_rng(0)
    n_bad = 0
    for seed in range(300):
        p = random_params(seed, max_cube_bytes=1 << 30)
        # perturb half of them into (possibly) invalid configs
        if seed % 2:
            k = int(rng.integers(0, 5))
            if k == 0:
                p["clbs"] = [int(x) for x in rng.integers(0, 32 - p["r"] + 2, p["num_ra"])]
            elif k == 1:
                p["cbn"] = [int(x) for x in rng.integers(1, 16, p["num_ra"] + p["num_va"])]
            elif k == 2:
                p["g"] = int(rng.choice([16, 24, 32, 48, 64]))
            elif k == 3:
                p["mangle_a"] = int(rng.integers(0, 1 << 32))
            else:
                p["r"] = int(rng.integers(0, 20))
        c = cb.config_from_dict(p)
        rc, msg = cb.validate(c)
        orc, omsg = O.validate(p)
        if orc == 0 and (O.cube_bytes(p) >> p["r"]) % 16:
            # the GPU build's one extra rule (16-byte CS slices); the oracle is generic
            assert rc == cb.E_CONFIG and "multiple of 16" in msg, (p, msg)
            n_bad += 1
            continue
        assert (rc == 0) == (orc == 0), (p, msg, omsg)
        if rc:
            n_bad += 1
            assert msg
        else:
            assert cb.cube_bytes(c) == O.cube_bytes(p)
    assert n_bad > 50


def test_strerror_and_create_without_gpu():
    assert cb.lib().cbaa_strerror(cb.E_CONFIG).decode() == "invalid config"
    bad = cb.default_config()
    bad.g = 48
    with pytest.raises(cb.CbaaError):
        cb.Cbaa(bad, 0)
