"""The C ABI used from plain C (examples/cbaa_window.c: no Python, no torch) on a C1 window."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1901_06207_b200 import workload as W
from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_program_window(tmp_path, paper):
    exe = os.path.join(ROOT, "examples", "cbaa_window")
    if not os.path.exists(exe):
        pytest.fail("examples/cbaa_window not built: run __graft_entry__.build()")
    w = W.generate(W.C1, 11)
    path = tmp_path / "pairs.bin"
    np.concatenate([w.src, w.dst]).astype("<u4").tofile(path)
    out = subprocess.run([exe, str(path), "1024"], capture_output=True, text=True, check=True).stdout
    lines = [l.split() for l in out.splitlines() if l and not l.startswith("#")]
    got = [(sum(int(x) << (24 - 8 * k) for k, x in enumerate(ip.split("."))), float(est)) for ip, est in lines]
    cube, _ = O.update(paper, w.src, w.dst)
    st, ref, _ = O.detect(paper, cube, 1024)
    assert [g[0] for g in got] == ref["ip"].tolist()
    assert np.allclose([g[1] for g in got], ref["estimate"], atol=5e-4)
    assert set(w.planted) <= {g[0] for g in got}
