"""Pins of the oracle's NEXT-1 corrections (the paper's other two DCOs on the same scan loop):
ADSampling on a random orthogonal projection and BSA-res (Alg. 2, P:L434-470;
Eq. 2-3). Each pin checks against what the paper or the mathematics fixes — a closed
form, a Monte Carlo property with a binomial tolerance, or the reduction to exact search."""
import math

import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O


def _haar(d, seed):
    return synth.haar_basis(d, np.random.default_rng(seed))


def test_decomposition_identity_eq2():
    # ‖x−q‖² = P_d + ‖x_r‖² + ‖q_r‖² − 2⟨q_r, x_r⟩ (Eq. 2): the terms BSA-res keeps and drops
    rng = np.random.default_rng(0)
    for d in (0, 5, 16, 31, 32):
        x, q = rng.standard_normal(32), rng.standard_normal(32)
        P = np.sum((x[:d] - q[:d]) ** 2)
        lhs = P + np.sum(x[d:] ** 2) + np.sum(q[d:] ** 2) - 2 * np.dot(q[d:], x[d:])
        assert abs(lhs - np.sum((x - q) ** 2)) <= 1e-12 * np.sum((x - q) ** 2)


@pytest.mark.parametrize("m", [1.0, 2.0])
def test_bsa_res_error_quantile_is_gaussian(m):
    # x ~ N(0, diag(λ)) (data already in its PCA basis): for a fixed q the estimate error
    # dis' − dis = 2⟨q_r, x_r⟩ is N(0, σ²) with σ² = 4 Σ_{i≥d} q_i² λ_i (Eq. 3), so the BSA-res
    # test dis' − mσ > dis fires with probability 1 − Φ(m)
    rng = np.random.default_rng(1)
    D, d, n = 48, 16, 200_000
    lam = 1.0 / np.arange(1, D + 1)
    q = rng.standard_normal(D)
    X = rng.standard_normal((n, D)) * np.sqrt(lam)
    c = O.bsa_res_consts(q, lam, d, m)[0]               # step d = Δd: ‖q_r‖² − mσ
    P = np.sum((X[:, :d] - q[:d]) ** 2, axis=1)
    score = P + np.sum(X[:, d:] ** 2, axis=1) + c       # P_d + ‖x_r‖² + ‖q_r‖² − mσ
    dis = np.sum((X - q) ** 2, axis=1)
    frac = np.mean(score > dis)
    p = 0.5 * math.erfc(m / math.sqrt(2.0))
    assert abs(frac - p) <= 4 * math.sqrt(p * (1 - p) / n)


def test_adsampling_estimate_is_unbiased_and_concentrated():
    # JL scaling (Lemma 1): after a random orthogonal rotation, (D/d)·P_d is an
    # unbiased estimate of the squared distance; with ε = ε₀/√d the test (D/d)P_d > (1+ε)²·dis
    # rarely fires (significance 2e^{-c0 ε0²})
    rng = np.random.default_rng(2)
    D, d, trials = 64, 16, 4000
    m1, b = O.adsampling_table(D, d, 0.0)               # ε₀ = 0: the bare JL scaling D/d
    assert np.allclose(m1, D / (np.arange(1, D // d) * d)) and np.all(b == 0)
    m21, _ = O.adsampling_table(D, d, 2.1)
    x = rng.standard_normal(D) * 3
    ratios, fires = [], 0
    for t in range(trials):
        R = _haar(D, 100 + t)
        y = R @ x
        est = m1[0] * np.sum(y[:d] ** 2)
        ratios.append(est / np.sum(x ** 2))
        fires += m21[0] * np.sum(y[:d] ** 2) > np.sum(x ** 2)
    ratios = np.array(ratios)
    assert abs(ratios.mean() - 1.0) <= 4 * ratios.std() / math.sqrt(trials)
    assert fires / trials < 0.01


@pytest.fixture(scope="module")
def small():
    cfg = synth.config("c2", n=6000, nlist=24, nq=12, n_cal=40)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    cent = O.kmeans(X, cfg.nlist, iters=3)
    idx = O.build_index(X, cent, mean, R, lam=lam)
    ridx = O.build_index(X, cent, mean, _haar(cfg.d, 7), lam=lam)   # random rotation (ADSampling)
    return cfg, X, idx, ridx


def test_next1_methods_reduce_to_exact_ivf(small):
    # a correction that can never fire (ε₀, m → ∞) leaves exact IVF; α = 0 disables every method
    cfg, X, idx, ridx = small
    Q = synth.queries(cfg)
    ei, ed = O.exact_ivf(idx, X, Q, 10, 6)
    for ix, kw in ((ridx, dict(method="adsampling", eps0=1e9)), (idx, dict(method="bsa_res", m_res=1e9)),
                   (ridx, dict(method="adsampling", eps0=2.1, alpha=0.0)), (idx, dict(method="bsa_res", alpha=0.0))):
        alpha = kw.pop("alpha", 0.005)
        oi, od, st = O.search(ix, Q, 10, 6, 16, alpha, **kw)
        assert np.array_equal(oi, ei)
        assert np.allclose(od, ed, rtol=1e-12)
        assert st["dims_scanned"] == st["tested"] * cfg.d


@pytest.mark.parametrize("method,kw,which", [("adsampling", dict(eps0=2.1), "r"), ("bsa_res", dict(m_res=8.0), "p")])
def test_next1_methods_prune_and_stay_exact(small, method, kw, which):
    # the paper's defaults (ε₀ = 2.1, m = 8) prune, every returned distance is the
    # exact distance of that id (d = D), every logged prune re-evaluates true, recall ~ exact IVF
    cfg, X, idx, ridx = small
    ix = ridx if which == "r" else idx
    Q = synth.queries(cfg)
    oi, od, st = O.search(ix, Q, 10, 6, 16, 0.005, method=method, log=True, **kw)
    assert st["dims_scanned"] < st["tested"] * cfg.d
    for q in range(Q.shape[0]):
        ok = oi[q] >= 0
        ex = np.sum((ix["Xr"][oi[q][ok]] - O.rotate(Q[q:q + 1], ix["mean"], ix["R"])[0]) ** 2, axis=1)
        assert np.allclose(od[q][ok], ex, rtol=1e-12)
    for (_, _, _, score, tau) in st["decisions"]:
        assert score > tau
    ei, _ = O.exact_ivf(idx, X, Q, 10, 6)
    assert O.recall_at_k(oi, ei, 10) >= 0.97
