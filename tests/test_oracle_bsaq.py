"""Pins for the oracle's BSA-q (NEXT-3, §V-B): PQ encoding, ADC look-up tables, the
Procrustes step of OPQ, OPQ training, the multi-feature logistic fit, the calibrated classifier's
held-out quantile and the search — against brute force, closed forms, an independent optimiser
and a hand-worked case."""
import itertools

import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O


def test_pq_encode_brute_force_and_ties():
    rng = np.random.default_rng(0)
    m, ds = 3, 4
    C = rng.integers(-3, 4, size=(m, O.PQ_K, ds)).astype(np.float32)
    C[1, 7] = C[1, 200]                                    # duplicated codeword: ties go to code 7
    X = rng.integers(-3, 4, size=(40, m * ds)).astype(np.float32)
    X[5, ds:2 * ds] = C[1, 200]
    codes, e = O.pq_encode(X, C)
    for i in range(X.shape[0]):                            # pure-Python loops
        err = 0.0
        for j in range(m):
            best, arg = None, None
            for c in range(O.PQ_K):
                d = sum((float(X[i, j * ds + t]) - float(C[j, c, t])) ** 2 for t in range(ds))
                if best is None or d < best:
                    best, arg = d, c
            assert codes[i, j] == arg
            err += best
        assert e[i] == err
    assert codes[5, 1] == 7


def test_adc_table_and_distance():
    rng = np.random.default_rng(1)
    m, ds = 4, 4
    C = rng.standard_normal((m, O.PQ_K, ds)).astype(np.float32)
    q = rng.standard_normal(m * ds)
    lut = O.adc_lut(q, C)
    for j, c in itertools.product(range(m), (0, 17, 255)):
        assert abs(lut[j, c] - sum((float(C[j, c, t]) - q[j * ds + t]) ** 2 for t in range(ds))) < 1e-12
    codes = rng.integers(0, O.PQ_K, size=(25, m)).astype(np.uint8)
    # a row equal to its reconstruction: ADC = the exact distance, reconstruction error = 0
    X = np.concatenate([C[j][codes[:, j]] for j in range(m)], axis=1)
    np.testing.assert_allclose(O.adc(lut, codes), np.sum((X.astype(np.float64) - q) ** 2, axis=1), rtol=1e-12)
    c2, e2 = O.pq_encode(X, C)
    assert np.array_equal(c2, codes) and np.all(e2 == 0)


def test_procrustes_recovers_a_known_rotation():
    # rows y = Q x for a known orthogonal Q: the least-squares orthogonal map is Q itself
    rng = np.random.default_rng(2)
    X = rng.standard_normal((300, 12))
    Q = synth.haar_basis(12, rng)
    R = O.procrustes(X, X @ Q.T)
    np.testing.assert_allclose(R, Q, atol=1e-10)


@pytest.fixture(scope="module")
def word_like():
    # a flat-spectrum mixture (where the paper says BSA-q wins)
    cfg = synth.config("c1", n=3000, d=32, nlist=8, nq=30, n_cal=60, spectrum=0.2)
    X = synth.base(cfg)
    return cfg, X


def test_opq_training_orthogonal_and_beats_pq_on_pca(word_like):
    cfg, X = word_like
    m = O.pq_subspaces(cfg.d)
    mean, R, C = O.opq_train(X, m, n_train=3000, iters=4, km_iters=3, final_iters=4)
    np.testing.assert_allclose(R @ R.T, np.eye(cfg.d), atol=1e-12)
    assert C.shape == (m, O.PQ_K, cfg.d // m) and C.dtype == np.float32
    m0, R0, C0 = O.opq_train(X, m, n_train=3000, iters=0, final_iters=4)    # PQ on the PCA basis
    d_opq = O.pq_encode(O.rotate(X, mean, R), C)[1].mean()
    d_pca = O.pq_encode(O.rotate(X, m0, R0), C0)[1].mean()
    assert d_opq <= d_pca * 1.001, (d_opq, d_pca)
    assert np.array_equal(m0, mean)                                            # same sample mean


def test_logistic_multi_k1_equals_logistic_irls():
    rng = np.random.default_rng(3)
    n = 400
    P = rng.gamma(3.0, 2.0, n); tau = rng.gamma(4.0, 1.5, n)
    y = (rng.random(n) < 1 / (1 + np.exp(-(1.3 * P - 1.8 * tau + 0.5)))).astype(float)
    m1, b1, ok1 = O.logistic_irls(P, tau, y)
    mv, b2, ok2 = O.logistic_irls_multi(P[:, None], tau, y)
    assert ok1 and ok2 and abs(mv[0] - m1) <= 1e-9 * abs(m1) and abs(b2 - b1) <= 1e-9 * max(1, abs(b1))


def test_logistic_multi_vs_bfgs():
    from scipy.optimize import minimize
    rng = np.random.default_rng(4)
    n = 600
    F = np.stack([rng.gamma(3.0, 2.0, n), rng.gamma(2.0, 0.5, n)], axis=1)
    tau = rng.gamma(4.0, 1.5, n)
    z = 1.1 * F[:, 0] + 0.7 * F[:, 1] - 1.5 * tau + 0.3
    y = (rng.random(n) < 1 / (1 + np.exp(-z))).astype(float)
    mv, beta, ok = O.logistic_irls_multi(F, tau, y, ridge=0.0)

    def bce(w):
        t = w[0] + F @ w[1:3] + w[3] * tau
        return float(np.sum(np.logaddexp(0.0, t) - y * t))
    w = minimize(bce, np.zeros(4), method="BFGS", options={"gtol": 1e-10, "maxiter": 20000}).x
    assert ok
    np.testing.assert_allclose(mv, -w[1:3] / w[3], rtol=2e-4)
    assert abs(beta - (-w[0] / w[3])) <= 2e-3 * max(1.0, abs(beta))


def test_logistic_multi_flags_wrong_slope():
    # label falls with the ADC distance: m_0 <= 0 → flagged, (e_0, 0, False)
    rows = []
    for t in (1.0, 2.0, 3.0):
        for p in (1.0, 2.0, 3.0):
            n1 = int(9 - t - p)
            rows += [(p, 1.0, t, 1.0)] * n1 + [(p, 1.0, t, 0.0)] * (9 - n1)
    P, E, tau, y = (np.array(c) for c in zip(*rows))
    mv, beta, ok = O.logistic_irls_multi(np.stack([P, E], axis=1), tau, y)
    assert not ok and mv.tolist() == [1.0, 0.0] and beta == 0.0


# ---------------------------------------------------------------- hand-worked search (D = 16, m = 2)
def _hand_q():
    D, ds = 16, 8
    C = np.zeros((2, O.PQ_K, ds), np.float32)
    C[:, :, 0] = np.arange(O.PQ_K)                       # codeword c = (c, 0, ..., 0): lut[j, c] = c² at q̃ = 0
    rows = [  # (a, b): x̃ = (a, 0 x 7, b, 0 x 7)
        (3.0, 0.0), (2.0, 1.0), (1.0, 1.0), (0.0, 2.0),   # epoch 0 (c0 = 4K = 4): τ = ∞; dists 9 5 2 4 → τ_1 = 2
        (1.25, 0.0),   # id 4: code (1, 0), ADC 1, e 1/16: 1 + 4/16 + 1 = 2.25 > 2 → pruned (exact dist 1.5625)
        (0.0, 1.0),    # id 5: ADC 1, e 0: 2 > 2? no → exact 1
        (1.0, 0.0),    # id 6: 2 ≤ 2 → exact 1 (ties id 5: lower id first)
        (0.0, 1.5),    # id 7: 1.5 ties codes 1 and 2 → code 1, ADC 1, e 1/4: 1 + 1 + 1 = 3 > 2 → pruned
        (0.0, 0.0),    # id 8: epoch 2, τ_2 = 1: ADC 0 → 1 > 1? no → exact 0
        (1.0, 0.0),    # id 9: 1 + 0 + 1 = 2 > 1 → pruned
    ]
    X = np.zeros((len(rows), D), np.float32)
    for i, (a, b) in enumerate(rows):
        X[i, 0], X[i, 8] = a, b
    idx = O.build_index_q(X, np.zeros((1, D), np.float32), np.zeros(D), np.eye(D), C)
    # m = (1, 4); v sorted descending (n0 = 4): α = 0.3 → k = ⌈0.7·4⌉ = 3 → β' = v[2] = 1
    idx["calq"] = {"m": np.array([1.0, 4.0]), "v": np.array([5.0, 3.0, 1.0, -1.0]), "n0": 4, "K": 1}
    return X, idx


def test_hand_worked_bsaq_search():
    X, idx = _hand_q()
    assert idx["codes"].tolist()[4] == [1, 0] and idx["codes"].tolist()[7] == [0, 1]
    assert idx["pq_err"].tolist()[4] == 0.0625 and idx["pq_err"].tolist()[7] == 0.25
    ids, d, st = O.search_q(idx, np.zeros((1, 16), np.float32), 1, 1, 0.3, log=True)
    assert ids.tolist() == [[8]] and d.tolist() == [[0.0]]
    assert st["tested"] == 10 and st["survivors"] == 7 and st["pruned"] == 3     # ids 4, 7, 9 pruned
    q_, i_, dims, margin = (np.concatenate(c) for c in zip(*st["candidates"]))
    assert dims.tolist() == [16, 16, 16, 16, 0, 16, 16, 0, 16, 0]
    # id 5: |2 − 2| = 0; id 4: |2.25 − 2| / (1.25 + 1 + 2) = 1/17
    assert margin[5] == 0.0 and abs(margin[4] - 1 / 17) < 1e-15
    ids, d, st = O.search_q(idx, np.zeros((1, 16), np.float32), 2, 1, 0.0)      # α = 0: exact
    assert ids.tolist() == [[8, 5]] and st["pruned"] == 0


@pytest.fixture(scope="module")
def q_index(word_like):
    cfg, X = word_like
    m = O.pq_subspaces(cfg.d)
    mean, R, C = O.opq_train(X, m, n_train=3000, iters=3, km_iters=3, final_iters=4)
    cent = O.kmeans(X, cfg.nlist, iters=3)
    idx = O.build_index_q(X, cent, mean, R, C)
    idx["calq"] = O.calibrate_q(X, idx, synth.cal_queries(cfg), cfg.k, n_neg=50, nprobe_neg=3, seed=0)
    return cfg, X, idx


def test_bsaq_alpha0_is_exact_and_distances_exact(q_index):
    cfg, X, idx = q_index
    Q = synth.queries(cfg)
    ids, d, st = O.search_q(idx, Q, cfg.k, 3, 0.0)
    ei, ed = O.exact_ivf(idx, X, Q, cfg.k, 3)
    assert np.array_equal(ids, ei)
    ids, d, st = O.search_q(idx, Q, cfg.k, 3, 0.005)
    for q in range(Q.shape[0]):
        np.testing.assert_allclose(d[q], O.sqdist_seq(X[ids[q]], Q[q]), rtol=1e-9)
    assert O.recall_at_k(ids, ei, cfg.k) >= 0.98
    assert st["pruned"] > 0.3 * st["tested"]                                      # the ADC test prunes


def test_bsaq_heldout_quantile(q_index):
    # the calibrated classifier prunes held-out Label-0 pairs at about the target rate α
    cfg, X, idx = q_index
    cal = idx["calq"]
    alpha = 0.2
    beta = O.beta_from_v(cal["v"], alpha)
    Qh = synth.heldout_queries(cfg, 80)
    qi, ids, lab, tau = O.calibration_pairs(X, idx, Qh, cfg.k, 0, 3, 0)
    Qr = O.rotate(Qh, idx["mean"], idx["R"])
    dis = np.array([O.adc(O.adc_lut(Qr[q], idx["pq"]), idx["codes"][i:i + 1])[0] for q, i in zip(qi, ids)])
    score = cal["m"][0] * dis + cal["m"][1] * idx["pq_err"][ids] + beta
    frac = float(np.mean(score[lab == 0] > tau[lab == 0]))
    n0, nh = cal["n0"], int(np.sum(lab == 0))
    band = np.sqrt(np.log(2 / 0.05) / (2 * n0)) + 3 * np.sqrt(alpha * (1 - alpha) / nh)
    assert abs(frac - alpha) <= band, (frac, band)
