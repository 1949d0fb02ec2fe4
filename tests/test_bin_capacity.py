"""Host logic of the binned update's sampled region sizing (cbaa.cu update_binned, binned.cuh bin_cap):
the scratch allocated for a chunk must hold the regions k_bin_starts lays out for ANY sampled histogram,
or the scatter would write past the buffer.  The device formula is restated here (float32 sqrt like
sqrtf) and checked against the host bound on adversarial histograms."""
import math

import numpy as np
import pytest

NBINS = 4096
UNIT = 8   # pairs per sample unit (kSampleUnit)


def bin_cap(c, slack, L):
    est = (int(c) << L) // UNIT
    sd = int(np.sqrt(np.float32(est) * np.float32(1 << L), dtype=np.float32))
    return (est + est // 4 + 2 * sd + 64 + slack + 7) & ~7


def want(m, L, slack):
    sm = float(m + (1 << L))
    return max(m + (slack + 8) * NBINS,
               int(1.25 * sm + 2.0 * math.sqrt(NBINS * (1 << L) * sm)) + (slack + 80) * NBINS + 64)


def sampled_pairs(m, L):
    """Upper bound of Σ counts: every unit [u·2^L, u·2^L + 8) that starts inside the chunk, full."""
    return UNIT * ((m + (1 << L) - 1) >> L)


@pytest.mark.parametrize("L", [3, 6, 9, 12, 16])
@pytest.mark.parametrize("m", [1 << 24, 100_000_000, (1 << 28) - 3])
def test_capacity_bound_holds(L, m):
    total = sampled_pairs(m, L)
    rng = np.random.default_rng(L * 1000 + m % 997)
    cases = {
        "one_bin": np.bincount([0], minlength=NBINS) * total,
        "uniform": np.full(NBINS, total // NBINS) + (np.arange(NBINS) < total % NBINS),
        "zipf": np.bincount(np.minimum(rng.zipf(1.3, total if total < 2_000_000 else 2_000_000), NBINS) - 1,
                            minlength=NBINS),
    }
    if total >= 2_000_000:   # rescale the Zipf shape to the full sampled count
        z = cases["zipf"].astype(np.float64)
        cases["zipf"] = np.floor(z / z.sum() * total).astype(np.int64)
    for name, counts in cases.items():
        assert counts.sum() <= total, name
        s = sum(bin_cap(c, 0, L) for c in counts)
        assert s <= want(m, L, 0), (name, s, want(m, L, 0))


def test_exact_count_bound():
    m = 12_345_679
    counts = np.full(NBINS, m // NBINS)
    counts[: m % NBINS] += 1
    slack = 8 * 148
    s = sum(((int(c) + slack + 7) & ~7) for c in counts)
    assert s <= want(m, 9, slack)
