"""GPU parity of the PCA covariance on the int8 tensor cores (pca.cu Gram mode of rotate.cu,
DADE_OPT_PCA_TC = 1, the default): Sigma_sum = sum over the strided sample of (x - mu)(x - mu)^T
(R17) against the fp64 definition computed here with numpy (the oracle's O1 formula),
entry-wise within the exact-split bound's scale, on GIST-like D = 960 data whose sample spans
several 16,384-row chunks with a ragged last one, on integer-valued SIFT-like data, and on a D = 96
set; the CUDA-core fp64 path (DADE_OPT_PCA_TC = 0) must agree too, and fit_rotation's eigenpairs
must match the oracle's at the tolerances of tests/test_gpu_build.py."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import build
    build.build()
    return torch


def _cov_ref(X, ns, mean):
    Xs = X[O.strided_ids(X.shape[0], ns)].astype(np.float64)
    Y = Xs - mean
    return Y.T @ Y, np.max(np.abs(Y), axis=0)


@pytest.mark.parametrize("cfgname,n,ns", [("c3", 40000, 37000), ("c2", 30000, 30000), ("c4", 50000, 20000)])
def test_covariance_tensor_cores_vs_fp64(torch_cuda, cfgname, n, ns):
    torch = torch_cuda
    from paper_2404_16322_b200 import Index
    cfg = synth.config(cfgname, n=n, nlist=8)
    X = synth.base(cfg)
    Xd = torch.from_numpy(X).cuda()
    ix = Index(cfg.d)
    s, cnt = ix.pca_mean_partial(Xd, 0, n, sample_size=ns)
    assert cnt == ns
    mean = s / cnt
    ref, ymax = _cov_ref(X, ns, mean)
    scale = np.sqrt(np.outer(np.diag(ref), np.diag(ref))) + 1e-300
    # the exact-split bound (rotate.cu, R36) summed over the chunks: 9 K 2^-42 2^(e_a + e_b) per
    # chunk with 2^e < 2 max|y|  ->  36 ns 2^-42 max|y_a| max|y_b|, plus fp64 rounding of the sums
    bound = 36.0 * ns * 2.0 ** -42 * np.outer(ymax, ymax) + 1e-13 * scale
    out = {}
    for tc in (1, 0):
        ix.set_option("pca_tc", tc)
        cov = ix.pca_cov_partial(Xd, 0, n, mean, sample_size=ns)
        out[tc] = cov
        assert np.array_equal(cov, cov.T) or tc == 0  # the Gram mode is exactly symmetric
        assert np.all(np.abs(cov - ref) <= bound), (tc, np.max(np.abs(cov - ref) / bound))
        assert np.max(np.abs(cov - ref) / scale) < 1e-9, tc
    ix.set_option("pca_tc", 1)


def test_fit_rotation_tensor_core_covariance_vs_oracle(torch_cuda):
    torch = torch_cuda
    from paper_2404_16322_b200 import Index
    cfg = synth.config("c3", n=20000, nlist=8)
    X = synth.base(cfg)
    ix = Index(cfg.d)
    ix.set_option("pca_tc", 1)
    ix.fit_rotation(torch.from_numpy(X).cuda(), sample_size=18000)
    m, R, lam = ix.get_rotation()
    om, oR, olam = O.fit_rotation(X, sample_size=18000)
    np.testing.assert_allclose(m, om, rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(lam, olam, rtol=1e-9, atol=1e-9 * olam[0])
    assert np.max(np.abs(R @ R.T - np.eye(cfg.d))) < 1e-12
