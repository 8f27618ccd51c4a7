"""GPU parity of the d_hat writer on fp16 operands (gemm_tf32.cu k_l2_tc with kind::f16,
DADE_OPT_DHAT_H16 = 1 / 2 / 3 on the d_hat path, DADE_OPT_KNN_PATH 1): probes bit-exact against the
oracle's fp64 definition (R20) on the bench's centroid-set shapes (C2 / C4 widths),
ragged tiles, integer ties, k up to 64 and the fp16 edge cases (power-of-two scales far outside
fp16's range, rows spanning its subnormal range, a zero operand row), and equal to the tf32
writer's probes on every row."""
import numpy as np
import pytest

from oracle import dade_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import build
    build.build()
    return torch


H16 = 1   # 1: 128 x 128 tiles (default), 2: 128 x 256 tiles, 3: cooperative cp.async operand loads


@pytest.fixture(autouse=True, params=[1, 2, 3])
def _tiles(request):
    global H16
    H16 = request.param
    yield


def _index(torch, X, cent):
    from paper_2404_16322_b200 import Index
    ix = Index(X.shape[1])
    ix.set_option("knn_path", 1)
    ix.set_option("probe_passes", 1)
    ix.set_option("dhat_h16", H16)
    mean, R, lam = O.fit_rotation(X)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), cent.shape[0], centroids=torch.from_numpy(cent).cuda())
    return ix


def _check(torch, ix, Q, cent, nprobe, step=1):
    Qd = torch.from_numpy(Q).cuda()
    pr = ix.probe(Qd, nprobe).cpu().numpy()
    for q in range(0, Q.shape[0], step):
        assert pr[q].tolist() == O.probe(Q[q], cent, nprobe).tolist(), f"query {q}"
    ix.set_option("dhat_h16", 0)          # the tf32 writer returns the same probes on every row
    pt = ix.probe(Qd, nprobe).cpu().numpy()
    ix.set_option("dhat_h16", H16)
    assert np.array_equal(pr, pt)


@pytest.mark.parametrize("D,C,nprobe", [(128, 4096, 8), (96, 16384, 8), (256, 20000, 8), (96, 3000, 64),
                                        (32, 777, 2), (256, 1000, 31), (48, 6000, 64)])
def test_h16_mixture_bit_exact(torch_cuda, D, C, nprobe):
    # Gaussian-mixture data like the bench's; ragged last column tiles (3000, 777, 20000, 1000)
    torch = torch_cuda
    rng = np.random.default_rng(D * 7 + C)
    centers = rng.standard_normal((64, D)).astype(np.float32) * 2
    X = (centers[rng.integers(0, 64, 2 * C)] + rng.standard_normal((2 * C, D)).astype(np.float32)).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent)
    Q = (centers[rng.integers(0, 64, 300)] + rng.standard_normal((300, D)).astype(np.float32)).astype(np.float32)
    _check(torch, ix, Q, cent, nprobe, step=3)


@pytest.mark.parametrize("nprobe", [2, 16, 64])
def test_h16_integer_ties(torch_cuda, nprobe):
    # small-integer data: massive exact distance ties, duplicated centroids (ties go to the lower id)
    torch = torch_cuda
    rng = np.random.default_rng(nprobe)
    D, C = 64, 5000
    X = rng.integers(0, 4, size=(3 * C, D)).astype(np.float32)
    cent = X[rng.choice(3 * C, C, replace=False)].copy()
    cent[4000] = cent[7]
    cent[4001] = cent[7]
    ix = _index(torch, X, cent)
    Q = rng.integers(0, 4, size=(257, D)).astype(np.float32)
    _check(torch, ix, Q, cent, nprobe, step=2)


@pytest.mark.parametrize("scale", [1e-18, 1.0, 3e15])
def test_h16_scales(torch_cuda, scale):
    # magnitudes far outside fp16's range: the power-of-two scales must map them in and out exactly
    torch = torch_cuda
    rng = np.random.default_rng(3)
    D, C = 96, 2000
    X = (rng.standard_normal((2 * C, D)) * scale).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent)
    Q = (rng.standard_normal((200, D)) * scale).astype(np.float32)
    _check(torch, ix, Q, cent, 8)


def test_h16_dynamic_range_and_zero_rows(torch_cuda):
    # rows whose coordinates span ~40 binades (many land in fp16's subnormal range after the row
    # scale), a query equal to the centring vector (a zero operand row), duplicated queries
    torch = torch_cuda
    rng = np.random.default_rng(5)
    D, C = 128, 3000
    mags = np.exp2(rng.uniform(-30, 10, size=(1, D))).astype(np.float32)
    X = (rng.standard_normal((2 * C, D)) * mags).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent)
    Q = (rng.standard_normal((130, D)) * mags).astype(np.float32)
    Q[0] = cent.astype(np.float64).mean(axis=0).astype(np.float32)
    Q[1] = Q[2]
    Q[129] = 0.0
    _check(torch, ix, Q, cent, 12)


def test_h16_many_rows(torch_cuda):
    # several 128-row tiles with a ragged last one (1000 = 7 x 128 + 104) on C4's centroid shape
    torch = torch_cuda
    rng = np.random.default_rng(9)
    D, C = 96, 16384
    X = rng.standard_normal((C + 5000, D)).astype(np.float32)
    cent = X[:C].copy()
    ix = _index(torch, X, cent)
    Q = rng.standard_normal((1000, D)).astype(np.float32)
    _check(torch, ix, Q, cent, 8, step=37)
