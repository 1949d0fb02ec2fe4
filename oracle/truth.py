"""Exact ground truth — TEST INFRASTRUCTURE ONLY.

The paper's own baseline stores every host's opposite points in an STL map
and counts them.  Here: the distinct (iip, oip) flows of a window and
|OP(iip)| per inner IP, by explicit set storage (numpy unique on the
packed 64-bit pair).  Used only for accuracy checks, never for parity.
"""
from __future__ import annotations

import numpy as np


def exact_cardinalities(iip: np.ndarray, oip: np.ndarray):
    """Returns (hosts, cardinalities, flow_count) with |FLW| = Σ|OP(iip)|."""
    iip = np.asarray(iip, dtype=np.uint64)
    oip = np.asarray(oip, dtype=np.uint64)
    if iip.size == 0:
        return np.zeros(0, np.uint32), np.zeros(0, np.int64), 0
    flows = np.unique((iip << np.uint64(32)) | oip)
    hosts, card = np.unique((flows >> np.uint64(32)).astype(np.uint32), return_counts=True)
    return hosts, card.astype(np.int64), int(flows.size)


def super_hosts(iip, oip, theta):
    """H = {h : |OP(h)| ≥ θ} (Def. 1) as a dict ip → cardinality."""
    hosts, card, _ = exact_cardinalities(iip, oip)
    sel = card >= theta
    return dict(zip(hosts[sel].tolist(), card[sel].tolist()))


def score(detected_ips, truth_card: dict, theta):
    """FNR / FPR / FTR per Eqs. 2-3 with the literal Ĥ+ (≤ θ, Q30).
    truth_card maps every inner IP that appears to its exact cardinality."""
    H = {h for h, c in truth_card.items() if c >= theta}
    Hhat = set(detected_ips)
    miss = H - Hhat
    spurious = {h for h in Hhat if truth_card.get(h, 0) <= theta}
    if not H:
        return dict(fnr=None, fpr=None, ftr=None, H=0, detected=len(Hhat), missed=0, spurious=len(spurious))
    fnr = len(miss) / len(H)
    fpr = len(spurious) / len(H)
    return dict(fnr=fnr, fpr=fpr, ftr=fnr + fpr, H=len(H), detected=len(Hhat), missed=len(miss),
                spurious=len(spurious))
