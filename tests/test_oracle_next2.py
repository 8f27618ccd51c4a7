"""Pins of the oracle's NEXT-2 Exp-7 estimators (R27): a hand-worked example, the
d = D special case (the estimate IS the distance: the ranking equals brute force), Eq. 2's
decomposition (exact = residual estimate − 2⟨q_r, x_r⟩), and the paper's Table III ordering
(BSA-res ≥ PCA ≥ Rand in recall@100) on anisotropic data (S:L611 criterion 7)."""
import numpy as np

from oracle import dade_oracle as O


def _index(X, R=None):
    mean, Rp, _ = O.fit_rotation(X)
    return O.build_index(X, X[:1].copy(), mean, Rp if R is None else R)


def test_hand_example():
    # x~ = (3, 4), q~ = (1, 1), d = 1: P_1 = (3-1)^2 = 4; residual = 4 + 4^2 + 1^2 = 21;
    # exact = 4 + (4-1)^2 = 13 = 21 - 2*1*4
    Xr = np.array([[3.0, 4.0]])
    q = np.array([1.0, 1.0])
    assert O.estimate_dists(Xr, q, 1, "partial")[0] == 4.0
    assert O.estimate_dists(Xr, q, 1, "residual")[0] == 21.0
    assert O.estimate_dists(Xr, q, 2, "partial")[0] == 13.0
    assert O.estimate_dists(Xr, q, 2, "residual")[0] == 13.0


def test_full_dimension_equals_brute_force():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((600, 16)).astype(np.float32)
    Q = rng.standard_normal((5, 16)).astype(np.float32)
    idx = _index(X)
    gt, gd = O.brute_force_knn(X, Q, 20)
    for est in ("partial", "residual"):
        ids, e = O.estimate_knn(idx, Q, 16, 20, est)
        assert np.array_equal(ids, gt)
        np.testing.assert_allclose(e, gd, rtol=1e-9)


def test_residual_estimate_drops_only_the_cross_term():
    rng = np.random.default_rng(2)
    Xr = rng.standard_normal((200, 24))
    q = rng.standard_normal(24)
    exact = O.sqdist_seq(Xr, q)
    for d in (1, 8, 16, 23):
        cross = -2.0 * (Xr[:, d:] @ q[d:])
        np.testing.assert_allclose(O.estimate_dists(Xr, q, d, "residual") + cross, exact, rtol=1e-10, atol=1e-10)
        # the partial estimate is the prefix of the sequential sum
        np.testing.assert_allclose(O.estimate_dists(Xr, q, d, "partial"), O.sqdist_seq(Xr[:, :d], q[:d]),
                                   rtol=1e-12)


def test_table3_ordering_on_anisotropic_data():
    rng = np.random.default_rng(7)
    n, D = 20000, 64
    lam = np.arange(1, D + 1) ** -1.0
    lam *= D / lam.sum()
    B, _ = np.linalg.qr(rng.standard_normal((D, D)))

    def draw(m):
        return ((rng.standard_normal((m, D)) * np.sqrt(lam)) @ B.T).astype(np.float32)

    X, Q = draw(n), draw(30)
    gt, _ = O.brute_force_knn(X, Q, 100)
    idx = _index(X)
    H, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((D, D)))
    idr = _index(X, R=np.ascontiguousarray(H.T))
    for d in (16, 32):
        pca = O.recall_at_k(O.estimate_knn(idx, Q, d, 100, "partial")[0], gt, 100)
        res = O.recall_at_k(O.estimate_knn(idx, Q, d, 100, "residual")[0], gt, 100)
        rnd = O.recall_at_k(O.estimate_knn(idr, Q, d, 100, "partial")[0], gt, 100)
        assert res >= pca >= rnd and res - rnd >= 0.02, (d, res, pca, rnd)
