"""Accuracy harness on the CUDA path: the paper's evaluation — FNR / FPR / FTR of the
detected super hosts against exact truth (Eqs. 2-3; averages P:421) — scored on the GPU
detector's output, with the GPU output first proven identical to the oracle's on the same window.

* a reduced config-5 sweep: 8 geometries (r, g, cbn) × 3 thresholds on a 10M-pair window with 200 planted
  hosts of log-uniform cardinality (BASELINE config 5's recipe at 1/50 of its length): whole cube, per-CS
  stats and host list == oracle; FNR/FPR/FTR vs truth.exact_cardinalities;
* SPEC's acceptance 3: paper configuration, θ = 1024, 50 planted hosts of cardinality
  U[2048, 16384] over 10^5 background hosts of cardinality ≤ 100, 20 seeds: median FTR ≤ 5 %, median
  FNR ≤ 1 % for the GPU detector (two seeds also checked against the oracle element by element).
Set CBAA_ACCURACY_OUT=<path> to append the per-point scores as JSON lines.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import truth
from paper_1901_06207_b200 import workload as W
from tests.test_gpu_parity import assert_hosts_equal, assert_stats_equal, dev, gpu_cube, handle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

# (r, g, cbn) points of the config-5 grid: the paper point, both ends of r and cbn, and g from 1024 to 8192
SWEEP = [(4, 4096, 12), (2, 1024, 10), (2, 4096, 14), (4, 1024, 12), (4, 8192, 10), (6, 2048, 12),
         (6, 4096, 10), (4, 2048, 14)]
THETAS = (512, 1024, 4096)


def _emit(rec):
    path = os.environ.get("CBAA_ACCURACY_OUT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.fixture(scope="module")
def c5_small():
    spec = W.c5_spec(n=10_000_000)
    spec = W.WindowSpec(n=spec.n, n_hosts=200_000, n_flows=1_500_000, scanners=spec.scanners)
    w = W.generate(spec, 5, with_raw=False)
    hs, card, n_flows = truth.exact_cardinalities(w.src, w.dst)
    return w, dict(zip(hs.tolist(), card.tolist())), n_flows


@pytest.mark.parametrize("r, g, cbn", SWEEP)
def test_reduced_c5_sweep(paper, c5_small, r, g, cbn):
    w, tc, n_flows = c5_small
    geo = next(x for x in W.c5_geometries() if (x["r"], x["g"], x["cbn"][0]) == (r, g, cbn))
    p = dict(paper, **geo)
    cb = handle(p)
    cb.reset()
    cb.update(dev(w.src), dev(w.dst))
    ref = O.update_parallel(p, w.src, w.dst)
    assert np.array_equal(gpu_cube(cb), ref)
    lam = n_flows / ((1 << r) * (1 << cbn))
    for theta in THETAS:
        hosts, stats, rc = cb.detect(theta, cap=1 << 22)
        st, oh, ostats = O.detect(p, ref, theta, cap=1 << 22)
        assert {0: 0, -6: 1, -5: 2}.get(rc, rc) == st   # library vs oracle status codes
        assert_stats_equal(stats, ostats)
        assert_hosts_equal(hosts, oh)
        m = truth.score(hosts["ip"].tolist(), tc, theta)
        _emit({"test": "reduced_c5", "r": r, "g": g, "cbn": cbn, "theta": theta, "n": int(w.src.size),
               "lambda_over_theta": lam / theta, "overloaded": lam > theta / 4, "hosts": int(len(hosts)),
               "overflow_cs": int(sum(s["overflow"] for s in stats)), **m})
        # the load rule of SURVEY §8(d) (λ ≤ θ/4), no skipped CS and wide enough columns: the detector
        # finds the super hosts (loose bound: the table itself is the result, recorded above)
        if lam <= theta / 4 and rc == 0 and g >= 2048 and m["H"]:
            assert m["fnr"] <= 0.10, m


def _s599_window(seed):
    rng = np.random.default_rng(300 + seed)
    d = tuple(int(x) for x in rng.integers(2048, 16385, 50))
    spec = W.WindowSpec(n=6_500_000, n_hosts=100_000, n_flows=6_000_000, card_cap=100, scanners=d)
    return W.generate(spec, 400 + seed, with_raw=False)


def test_s599_acceptance_on_gpu(paper):
    """SPEC acceptance 3 on the CUDA path, all 20 seeds."""
    ftr, fnr = [], []
    cb = handle(paper)
    for seed in range(20):
        w = _s599_window(seed)
        cb.reset()
        cb.update(dev(w.src), dev(w.dst))
        hosts, stats, rc = cb.detect(1024)
        assert rc == 0
        if seed < 2:   # the scored output is the oracle's output
            ref = O.update_parallel(paper, w.src, w.dst)
            assert np.array_equal(gpu_cube(cb), ref)
            st, oh, ostats = O.detect(paper, ref, 1024)
            assert_stats_equal(stats, ostats)
            assert_hosts_equal(hosts, oh)
        hs, card, _ = truth.exact_cardinalities(w.src, w.dst)
        m = truth.score(hosts["ip"].tolist(), dict(zip(hs.tolist(), card.tolist())), 1024)
        ftr.append(m["ftr"])
        fnr.append(m["fnr"])
        _emit({"test": "s599", "seed": seed, **m})
    assert np.median(ftr) <= 0.05 and np.median(fnr) <= 0.01, (np.median(ftr), np.median(fnr))
