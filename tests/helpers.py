"""Comparison helpers for GPU-vs-oracle parity tests (no method arithmetic here)."""
import numpy as np


def tie_adjusted_overlap(gi, gd, oi, od, rel=1e-5):
    """Fraction of GPU ids that are in the oracle's top-K, where an id outside it still counts if
    its distance ties the oracle's K-th distance within `rel` (R22: several results are correct)."""
    tot = good = 0
    for q in range(gi.shape[0]):
        oset = set(oi[q][oi[q] >= 0].tolist())
        kth = od[q][oi[q] >= 0].max() if (oi[q] >= 0).any() else np.inf
        for i, d in zip(gi[q], gd[q]):
            if i < 0:
                continue
            tot += 1
            if i in oset or abs(float(d) - kth) <= rel * max(kth, 1e-30):
                good += 1
    return good / max(tot, 1)


def raw_overlap(gi, oi):
    tot = good = 0
    for q in range(gi.shape[0]):
        s = set(oi[q][oi[q] >= 0].tolist())
        for i in gi[q]:
            if i >= 0:
                tot += 1
                good += i in s
    return good / max(tot, 1)


def rel_err(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    m = np.isfinite(b)
    assert np.array_equal(np.isfinite(a), m)
    return float(np.max(np.abs(a[m] - b[m]) / np.maximum(np.abs(b[m]), 1e-30))) if m.any() else 0.0
