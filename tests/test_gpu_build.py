"""GPU parity: PCA rotation, k-means, IVF lists and the rotated blocked layout."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import build, Index
    build.build()
    cfg = synth.config("c2", n=20000, nlist=64, nq=50, n_cal=100)
    X = synth.base(cfg)
    return torch, Index, cfg, X


def test_fit_rotation_vs_oracle(env):
    torch, Index, cfg, X = env
    ix = Index(cfg.d)
    ix.fit_rotation(torch.from_numpy(X).cuda(), sample_size=15000)
    m, R, lam = ix.get_rotation()
    om, oR, olam = O.fit_rotation(X, sample_size=15000)
    np.testing.assert_allclose(m, om, rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(lam, olam, rtol=1e-9, atol=1e-9 * olam[0])
    assert np.max(np.abs(R @ R.T - np.eye(cfg.d))) < 1e-12
    gap = np.abs(np.diff(olam))
    for i in range(cfg.d):      # well-separated eigenvalues: same direction, same sign (R18)
        g = min(gap[i - 1] if i > 0 else np.inf, gap[i] if i < cfg.d - 1 else np.inf)
        if g > 1e-3 * olam[0]:
            assert abs(R[i] @ oR[i] - 1.0) < 1e-6, i


def test_kmeans_and_lists_bit_exact(env):
    torch, Index, cfg, X = env
    ix = Index(cfg.d)
    om, oR, olam = O.fit_rotation(X)
    ix.set_rotation(om, oR, olam)
    Xd = torch.from_numpy(X).cuda()
    ix.build_ivf(Xd, cfg.nlist, kmeans_iters=3)
    off, row_id, assign, cent = ix.get_ivf()
    ocent = O.kmeans(X, cfg.nlist, iters=3)
    assert np.array_equal(cent, ocent)                       # same exact assignments + same fp64 means
    oa, ooff, orow = O.build_ivf(X, ocent)
    assert np.array_equal(assign, oa) and np.array_equal(off, ooff) and np.array_equal(row_id, orow)
    lay = ix.get_layout()
    ref = O.rotate(X[orow], om, oR)
    err = np.max(np.abs(lay - ref)) / np.max(np.abs(ref))
    assert err < 1e-6


def test_sharded_pca_partials_equal_single(env):
    torch, Index, cfg, X = env
    n = X.shape[0]
    ix = Index(cfg.d)
    S = 3
    parts = [(s * n // S, (s + 1) * n // S) for s in range(S)]
    sums, cnt = np.zeros(cfg.d), 0
    for lo, hi in parts:
        s, c = ix.pca_mean_partial(torch.from_numpy(X[lo:hi]).cuda(), lo, n, sample_size=7000)
        sums += s; cnt += c
    mean = sums / cnt
    cov = np.zeros((cfg.d, cfg.d))
    for lo, hi in parts:
        cov += ix.pca_cov_partial(torch.from_numpy(X[lo:hi]).cuda(), lo, n, mean, sample_size=7000)
    ix.set_rotation_from_cov(mean, cov, cnt)
    m, R, lam = ix.get_rotation()
    om, oR, olam = O.fit_rotation(X, sample_size=7000)
    assert cnt == 7000
    np.testing.assert_allclose(lam, olam, rtol=1e-9, atol=1e-9 * olam[0])


def test_kmeans_partial_logical_shards_equal_single():
    # sharded k-means through the C-ABI (dade_kmeans_partial): S logical shards of one base on one
    # GPU, their fp64 partial sums / counts added (what the all-reduce does) == the single-index
    # k-means on the whole base (centroids up to the fp64 summation order) and the oracle's
    import torch
    from paper_2404_16322_b200 import Index, build
    build.build()
    cfg = synth.config("c4", n=20000, nlist=48)
    X = synth.base(cfg)
    Xd = torch.from_numpy(X).cuda()
    mean, R, lam = O.fit_rotation(X)
    full = Index(cfg.d)
    full.set_rotation(mean, R, lam)
    full.build_ivf(Xd, cfg.nlist, kmeans_iters=3)
    cent_single = full.get_ivf()[3]
    S = 3
    shards = []
    for s in range(S):
        lo, hi = s * cfg.n // S, (s + 1) * cfg.n // S
        ix = Index(cfg.d)
        ix.set_rotation(mean, R, lam)
        shards.append((ix, Xd[lo:hi].contiguous(), lo))
    parts = [ix.kmeans_partial(Xs, lo, cfg.n, cfg.nlist) for ix, Xs, lo in shards]
    cent = sum(p[0] for p in parts).astype(np.float32)
    assert np.array_equal(sum(p[1] for p in parts), np.ones(cfg.nlist, np.int64))
    for _ in range(3):
        parts = [ix.kmeans_partial(Xs, lo, cfg.n, cfg.nlist, cent) for ix, Xs, lo in shards]
        sums, counts = sum(p[0] for p in parts), sum(p[1] for p in parts)
        nz = counts > 0
        cent = cent.copy()
        cent[nz] = (sums[nz] / counts[nz, None]).astype(np.float32)
    assert np.allclose(cent, cent_single, rtol=1e-6, atol=1e-6)
    assert np.allclose(cent, O.kmeans(X, cfg.nlist, iters=3), rtol=1e-6, atol=1e-6)
