"""Pins for the oracle's DADE search (O5)."""
import numpy as np
import pytest

from oracle import dade_oracle as O
from datagen import synth


def test_epoch_bounds_hand():
    assert O.epoch_bounds(1000, 10) == [0, 40, 80, 160, 320, 640, 1000]
    assert O.epoch_bounds(30, 10) == [0, 30]
    assert O.epoch_bounds(0, 10) == [0]


@pytest.fixture(scope="module")
def ivf_case():
    cfg = synth.config("c2", n=6000, nlist=24, nq=25, n_cal=60)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    cent = O.kmeans(X, cfg.nlist, iters=4)
    idx = O.build_index(X, cent, mean, R)
    idx["cal"] = O.calibrate(X, idx, synth.cal_queries(cfg), cfg.k, n_neg=50, nprobe_neg=4, seed=0)
    return cfg, X, idx, synth.queries(cfg)


def test_alpha0_equals_exact_ivf(ivf_case):
    cfg, X, idx, Q = ivf_case
    ids, d, st = O.search(idx, Q, 10, 5, 16, 0.0)
    ei, ed = O.exact_ivf(idx, X, Q, 10, 5)
    assert np.array_equal(ids, ei)
    np.testing.assert_allclose(d, ed, rtol=1e-12)
    assert st["dims_scanned"] == st["tested"] * X.shape[1]


def test_alpha0_full_probe_equals_brute_force(ivf_case):
    cfg, X, idx, Q = ivf_case
    ids, d, _ = O.search(idx, Q[:8], 10, cfg.nlist, 16, 0.0)
    bi, bd = O.brute_force_knn(X, Q[:8], 10)
    assert np.array_equal(ids, bi)
    np.testing.assert_allclose(d, bd, rtol=1e-12)


def test_delta_d_equal_D_is_exact(ivf_case):
    cfg, X, idx, Q = ivf_case
    ids, d, _ = O.search(idx, Q[:8], 10, 4, X.shape[1], 0.3)
    ei, ed = O.exact_ivf(idx, X, Q[:8], 10, 4)
    assert np.array_equal(ids, ei)


def test_pruned_decisions_and_exact_distances(ivf_case):
    cfg, X, idx, Q = ivf_case
    ids, d, st = O.search(idx, Q, 10, 6, 16, 0.005, log=True)
    for (_q, _id, step, val, tau) in st["decisions"]:
        assert val > tau and np.isfinite(tau)
    for qn in range(Q.shape[0]):  # at d = D the estimator is the exact distance
        ex = O.sqdist_seq(X[ids[qn]], Q[qn])
        np.testing.assert_allclose(d[qn], ex, rtol=1e-12)
    assert st["survivors"] + int(st["pruned_at_step"].sum()) == st["tested"]
    ei, _ = O.exact_ivf(idx, X, Q, 10, 6)
    bi, _ = O.brute_force_knn(X, Q, 10)
    assert O.recall_at_k(ids, bi, 10) >= O.recall_at_k(ei, bi, 10) - 0.01
    assert st["dims_scanned"] < 0.6 * st["tested"] * X.shape[1]  # pruning actually happens


def test_sequential_vs_epoch(ivf_case):
    cfg, X, idx, Q = ivf_case
    a, _, sa = O.search(idx, Q[:10], 10, 6, 16, 0.005, mode="epoch")
    b, _, sb = O.search(idx, Q[:10], 10, 6, 16, 0.005, mode="sequential")
    bi, _ = O.brute_force_knn(X, Q[:10], 10)
    assert abs(O.recall_at_k(a, bi, 10) - O.recall_at_k(b, bi, 10)) <= 0.02


def test_sharded_merge_alpha0(ivf_case):
    cfg, X, idx, Q = ivf_case
    S, n = 3, X.shape[0]
    parts = []
    for s in range(S):
        lo, hi = s * n // S, (s + 1) * n // S
        sidx = O.build_index(X[lo:hi], idx["centroids"], idx["mean"], idx["R"], idx["cal"], id_base=lo)
        i, d, _ = O.search(sidx, Q[:6], 10, 5, 16, 0.0)
        parts.append((i, d))
    mi, md = O.merge_shards(parts, 10)
    ei, ed = O.exact_ivf(idx, X, Q[:6], 10, 5)
    assert np.array_equal(mi, ei)
