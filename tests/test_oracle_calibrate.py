"""Pins for the oracle's calibration (§V-A; cascade P:L582-586)."""
import json
import math
import os

import numpy as np
import pytest
from scipy.optimize import minimize

from oracle import dade_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vectors():
    g = json.load(open(os.path.join(GOLD, "splitmix64_vectors.json")))
    for s, o in zip(g["states"], g["outputs"]):
        assert int(O.splitmix64(np.uint64(int(s, 16)))) == int(o, 16)


def test_cascade_recall_example():
    g = json.load(open(os.path.join(GOLD, "cascade_recall_example.json")))
    assert abs(O.step_recall(g["r"], g["D"], g["delta_d"]) - g["r_i"]) < 1e-15
    assert g["D"] // g["delta_d"] - 1 == g["n_classifiers"]


def _recall0(v, beta):
    # Label-0 recall of sign(m1·P + β > τ): a Label-0 pair is kept iff β ≤ τ − m1·P = v
    return np.mean(v >= beta)


@pytest.mark.parametrize("seed", range(4))
def test_beta_equals_bisection(seed):
    # P:L551 "A binary search on β′ ... to ensure the model achieves the target recall r for Label 0"
    rng = np.random.default_rng(seed)
    n0 = int(rng.integers(5, 400))
    v = np.sort(rng.standard_normal(n0) * 10)[::-1]
    for r in (0.5, 0.9, 0.99, 0.995, 1.0):
        got = O.beta_from_v(v, 1.0 - r)
        lo, hi = v.min() - 100.0, v.max() + 100.0  # recall(lo) = 1 ≥ r > recall(hi) = 0
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if _recall0(v, mid) >= r:
                lo = mid
            else:
                hi = mid
        # the largest feasible β′ lies in [got, next order statistic); bisection converges to it
        assert _recall0(v, got) >= r
        assert abs(lo - got) <= 1e-9 * max(1.0, abs(got))


@pytest.mark.parametrize("seed", range(3))
def test_beta_monotonicity_lemmas(seed):
    # recall of Label 0 non-increasing in β; pruning rate η non-decreasing in β
    rng = np.random.default_rng(seed)
    m1 = 1.3
    P0, P1 = rng.random(200) * 5, rng.random(600) * 10 + 2
    tau0, tau1 = rng.random(200) * 6, rng.random(600) * 6
    betas = np.sort(rng.standard_normal(50) * 5)
    rec = [np.mean(m1 * P0 + b <= tau0) for b in betas]
    eta = [np.mean(m1 * P1 + b > tau1) for b in betas]
    assert all(rec[i + 1] <= rec[i] for i in range(49))
    assert all(eta[i + 1] >= eta[i] for i in range(49))


def _bce(wfull, A, y):
    z = A @ wfull
    return np.sum(np.logaddexp(0.0, z) - y * z)


@pytest.mark.parametrize("seed", range(3))
def test_logistic_matches_independent_optimiser(seed):
    # the slope must be the BCE minimiser; compare against scipy's BFGS on raw features
    rng = np.random.default_rng(seed)
    n = 3000
    tau = rng.random(n) * 4 + 1
    P = rng.random(n) * 8
    logit = 2.5 * P - 3.0 * tau + 0.7 + rng.logistic(size=n) * 0.0
    y = (rng.random(n) < 1 / (1 + np.exp(-logit))).astype(float)
    m1, beta, ok = O.logistic_irls(P, tau, y, ridge=0.0)
    A = np.stack([np.ones(n), P, tau], axis=1)
    res = minimize(_bce, np.zeros(3), args=(A, y), method="BFGS", options={"gtol": 1e-10, "maxiter": 10000})
    b0, wP, wt = res.x
    assert ok
    assert abs(m1 - (-wP / wt)) <= 2e-4 * abs(m1)
    assert abs(beta - (-b0 / wt)) <= 2e-3 * max(1, abs(beta))
    # and it recovers the generating model within sampling error
    assert abs(m1 - 2.5 / 3.0) < 0.15


def test_logistic_flag_rule_w_tau_nonnegative():
    # R3 flag rule, case w_τ ≥ 0: the label rises with τ (and does not depend on P), so the fitted
    # τ-weight is positive — the model "prune iff m1·P + β > τ" does not exist — and the fit must
    # return exactly (m1, β, ok) = (1, 0, False). Non-separable: each τ level carries both labels.
    tau = np.repeat(np.arange(1.0, 11.0), 20)            # 10 τ levels x 20 pairs
    P = np.tile(np.arange(20.0), 10)                     # P uncorrelated with y
    y = np.zeros(200)
    for lvl in range(10):                                # label-1 count grows with τ: 2 + lvl of 20
        y[lvl * 20: lvl * 20 + 2 + lvl] = 1.0
    m1, beta, ok = O.logistic_irls(P, tau, y)
    assert (m1, beta, ok) == (1.0, 0.0, False)


def test_logistic_flag_rule_m1_nonpositive():
    # R3 flag rule, case m1 ≤ 0: w_τ < 0 (label 1 more likely at small τ, as the model expects) but
    # w_P < 0 too (label 1 more likely at SMALL partial distances), so m1 = −w_P/w_τ < 0: flagged,
    # exactly (1, 0, False). Hand-built, non-separable counts.
    rows = []
    for t in (1.0, 2.0, 3.0, 4.0):
        for p in (1.0, 2.0, 3.0, 4.0):
            n1 = int(10 - t - p)                          # label-1 count falls with both τ and P
            rows += [(p, t, 1.0)] * n1 + [(p, t, 0.0)] * (10 - n1)
    P, tau, y = (np.array(c) for c in zip(*rows))
    m1, beta, ok = O.logistic_irls(P, tau, y)
    assert (m1, beta, ok) == (1.0, 0.0, False)


def test_logistic_flag_rule_accepts_the_expected_sign():
    # control for the two flag tests: label 1 rises with P and falls with τ (the model's shape)
    # → ok, m1 > 0 (the same hand-built counts with P reversed)
    rows = []
    for t in (1.0, 2.0, 3.0, 4.0):
        for p in (1.0, 2.0, 3.0, 4.0):
            n1 = int(10 - t - (5.0 - p))
            rows += [(p, t, 1.0)] * n1 + [(p, t, 0.0)] * (10 - n1)
    P, tau, y = (np.array(c) for c in zip(*rows))
    m1, beta, ok = O.logistic_irls(P, tau, y)
    assert ok and m1 > 0
    # symmetric counts in (P, 5 − τ): the fitted weights are equal and opposite → m1 = 1 exactly
    assert abs(m1 - 1.0) < 1e-9


def test_step_table_alpha_zero_disables_pruning():
    cal = {"m1": np.array([1.1, 1.2, 1.3]), "v": np.zeros((3, 10)), "block": 16}
    m, b = O.step_table(cal, 64, 16, 0.0)
    assert np.all(np.isneginf(b)) and m.tolist() == [1.1, 1.2, 1.3]
    m, b = O.step_table(cal, 64, 32, 0.01)  # Δd = 32 uses the d = 32 entry (index 1)
    assert m.tolist() == [1.2]


@pytest.fixture(scope="module")
def c1_index():
    from datagen import synth
    cfg = synth.config("c1", n=4000)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    cent = X[:1].copy()
    idx = O.build_index(X, cent, mean, R)
    return cfg, X, idx


def test_calibration_pairs_labels(c1_index):
    from datagen import synth
    cfg, X, idx = c1_index
    Qc = synth.cal_queries(cfg, 20)
    qi, ids, lab, tau = O.calibration_pairs(X, idx, Qc, 10, 30, 0, seed=0)
    assert np.sum(lab == 0) == 20 * 10 and np.sum(lab == 1) == 20 * 30
    for q in range(20):
        d = O.sqdist_seq(X[ids[qi == q]], Qc[q])
        l = lab[qi == q]
        assert np.all(d[l == 0] <= tau[qi == q][0])          # Label 0 = the K NN (dis ≤ τ)
        assert np.all(d[l == 1] >= tau[qi == q][0])          # Label 1 = the rest
        assert len(set(ids[qi == q].tolist())) == 40


def test_heldout_quantile(c1_index):
    # north_star: calibrated thresholds hit their target quantile on held-out samples.
    # DKW band on the empirical quantile of n0 calibration pairs + binomial noise of n_h held-out pairs.
    from datagen import synth
    cfg, X, idx = c1_index
    K, D, dd = 10, X.shape[1], 16
    cal = O.calibrate(X, idx, synth.cal_queries(cfg, 100), K, n_neg=50, nprobe_neg=0, seed=0, block=16)
    H = synth.heldout_queries(cfg, 100)
    hid, hd = O.brute_force_knn(X, H, K)
    Hr = O.rotate(H, idx["mean"], idx["R"])
    Xr = idx["Xr"]
    P = np.cumsum((Xr[hid.reshape(-1)] - np.repeat(Hr, K, axis=0)) ** 2, axis=1)
    tau = np.repeat(hd[:, K - 1], K)
    n0, nh = cal["n0"], len(tau)
    for alpha in (0.05, 0.2):
        m, b = O.step_table(cal, D, dd, alpha)
        a_s = alpha * dd / D
        band = math.sqrt(math.log(2 / 0.05) / (2 * n0)) + 3 * math.sqrt(a_s * (1 - a_s) / nh)
        for s in range(len(m)):
            d = (s + 1) * dd
            frac = np.mean(m[s] * P[:, d - 1] + b[s] > tau)
            assert abs(frac - a_s) <= band, (alpha, d, frac, a_s, band)


def test_step_table_uses_the_row_of_its_prefix_length():
    # the classifier at step s (d = s*Δd) must use the calibration row fitted on
    # prefix length d: rows are made distinguishable (value = d) and the slope row likewise
    D, n0 = 128, 50
    cls_d = np.arange(1, D // 16) * 16                      # prefixes 16, 32, ..., 112
    cal = {"block": 16, "m1": cls_d.astype(float) / 1000.0,
           "v": np.repeat(cls_d[:, None].astype(float), n0, axis=1)}
    for dd in (16, 32, 64):
        m, b = O.step_table(cal, D, dd, 0.01)
        d = np.arange(1, D // dd) * dd
        assert np.array_equal(b, d.astype(float))
        assert np.allclose(m, d / 1000.0)
