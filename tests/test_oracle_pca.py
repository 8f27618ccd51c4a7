"""Pins for the oracle's PCA rotation (Theorem 1; proof P:L4067-4096)."""
import json
import os

import numpy as np
import pytest

from oracle import dade_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_example_2d():
    # points (±a,0), (0,±b): mean 0, Σ = diag(a²/2, b²/2) with divisor n
    a, b = 3.0, 1.0
    X = np.array([[a, 0], [-a, 0], [0, b], [0, -b]], np.float32)
    mean, R, lam = O.fit_rotation(X)
    np.testing.assert_allclose(mean, [0, 0], atol=0)
    np.testing.assert_allclose(lam, [a * a / 2, b * b / 2], rtol=1e-14)
    np.testing.assert_allclose(R, np.eye(2), atol=1e-14)
    # rotated by 90°: the principal direction is now the y axis
    mean, R, lam = O.fit_rotation(X[:, ::-1].copy())
    np.testing.assert_allclose(R, [[0, 1], [1, 0]], atol=1e-14)


def test_closed_form_known_covariance():
    # X = sqrt(n)·Z·diag(sqrt λ)·Qᵀ + μ with Z orthonormal, zero-mean columns ⇒ Σ = Q diag(λ) Qᵀ exactly
    rng = np.random.default_rng(0)
    n, D = 500, 8
    G = rng.standard_normal((n, D))
    G -= G.mean(axis=0)
    Z, _ = np.linalg.qr(G)
    Z -= Z.mean(axis=0)  # keep columns zero-mean (QR of centred G already ~ is)
    Q, _ = np.linalg.qr(rng.standard_normal((D, D)))
    lam = np.array([9.0, 7.0, 5.0, 3.0, 2.0, 1.0, 0.5, 0.25])
    mu = rng.standard_normal(D)
    X = (np.sqrt(n) * Z * np.sqrt(lam)) @ Q.T + mu
    mean, R, got = O.fit_rotation(X.astype(np.float64))
    np.testing.assert_allclose(got, lam, rtol=1e-9)
    np.testing.assert_allclose(mean, mu, atol=1e-12)
    for i in range(D):  # each row is ± the i-th column of Q
        assert abs(abs(R[i] @ Q[:, i]) - 1.0) < 1e-9


@pytest.fixture(scope="module")
def c1_small():
    from datagen import synth
    cfg = synth.config("c1", n=3000)
    return synth.base(cfg)


def test_orthogonality_isometry_and_sign(c1_small):
    X = c1_small
    mean, R, lam = O.fit_rotation(X)
    assert np.max(np.abs(R @ R.T - np.eye(R.shape[0]))) <= 1e-12
    assert np.all(np.diff(lam) <= 0)
    for row in R:  # R18 sign rule
        j = int(np.argmax(np.abs(row)))
        assert row[j] > 0
    # north_star: rotation preserves all pairwise distances (≤1e-6 rel in float64)
    Xr = O.rotate(X[:200], mean, R)
    for i in range(0, 200, 7):
        for j in range(1, 200, 11):
            d0 = O.sqdist_seq(X[i:i + 1], X[j])[0]
            if d0 > 1e-9:
                d1 = float(np.sum((Xr[i] - Xr[j]) ** 2))
                assert abs(d1 - d0) <= 1e-6 * d0


def test_eigen_residual(c1_small):
    X = c1_small.astype(np.float64)
    mean, R, lam = O.fit_rotation(X)
    # covariance formed independently (two loops over dims, population divisor)
    Y = X - X.mean(axis=0)
    cov = np.einsum("ni,nj->ij", Y, Y) / X.shape[0]
    for i in range(X.shape[1]):
        assert np.linalg.norm(cov @ R[i] - lam[i] * R[i]) <= 1e-10 * np.linalg.norm(cov)


def test_theorem1_pca_minimises_residual_variance(c1_small):
    # Theorem 1: Σ_{i>d} var under PCA ≤ the same under any orthogonal rotation, every d
    X = c1_small.astype(np.float64)
    mean, R, lam = O.fit_rotation(X)
    rng = np.random.default_rng(1)
    for trial in range(3):
        Qr, _ = np.linalg.qr(rng.standard_normal((X.shape[1], X.shape[1])))
        var_rand = ((X - mean) @ Qr).var(axis=0)
        var_pca = O.rotate(X, mean, R).var(axis=0)
        for d in range(1, X.shape[1]):
            assert var_pca[d:].sum() <= var_rand[d:].sum() + 1e-9


def test_eq3_error_variance():
    g = json.load(open(os.path.join(GOLD, "sigma_suffix_example.json")))
    for d, v in zip(g["d"], g["var"]):
        assert O.err_variance(np.array(g["q"], float), np.array(g["sigma2"], float), d) == v
    # Monte Carlo: Var(-2<q_r,x_r>) for x ~ N(0, diag σ²) within 10%
    rng = np.random.default_rng(2)
    sig2 = np.array([4.0, 3.0, 2.0, 1.0, 0.5, 0.25])
    q = rng.standard_normal(6)
    x = rng.standard_normal((40000, 6)) * np.sqrt(sig2)
    for d in (1, 3, 5):
        emp = np.var(-2.0 * x[:, d:] @ q[d:])
        assert abs(emp - O.err_variance(q, sig2, d)) <= 0.1 * O.err_variance(q, sig2, d)
