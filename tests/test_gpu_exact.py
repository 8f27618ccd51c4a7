"""GPU parity: exact KNN / probe / assignment (bit-exact ids vs the oracle's fp64 definition)."""
import numpy as np
import pytest

from oracle import dade_oracle as O

pytestmark = pytest.mark.gpu


_OPTS = {}  # dade_set_option values applied to every index a test creates


@pytest.fixture(autouse=True, params=[1, 2, 4, 5, 6], ids=["dhat-matrix", "fused-filter", "fz-fp16", "fz-tf32", "int8-split"])
def knn_path(request):
    # every selection path: the d_hat-matrix select (exact.cu), the fused filter GEMM with
    # in-epilogue candidate tracking (probe_tc.cu) and the throughput fused filter on fp16 / tf32
    # operands (probe_fz.cu; 1-pass filters only, the others fall back); each must be bit-exact
    _OPTS.clear()
    _OPTS["knn_path"] = request.param
    yield request.param
    _OPTS.clear()


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import build
    build.build()
    return torch


def _idx(torch, D):
    from paper_2404_16322_b200 import Index
    ix = Index(D)
    for k, v in _OPTS.items():
        ix.set_option(k, v)
    return ix


@pytest.mark.parametrize("n,D,K", [(1000, 16, 1), (3001, 48, 10), (777, 128, 100), (5000, 64, 257)])
def test_bruteforce_knn_bit_exact(torch_cuda, n, D, K):
    torch = torch_cuda
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, D)).astype(np.float32)
    Q = rng.standard_normal((37, D)).astype(np.float32)
    ix = _idx(torch, D)
    gi, gd = ix.bruteforce_knn(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), K, id_base=5)
    oi, od = O.brute_force_knn(X, Q, K, id_base=5)
    assert np.array_equal(gi.cpu().numpy(), oi)
    assert np.array_equal(gd.cpu().numpy(), od.astype(np.float32))  # fp32 rounding of the exact fp64 value


def test_bruteforce_knn_integer_ties(torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(1)
    X = rng.integers(0, 4, size=(4000, 32)).astype(np.float32)   # massive exact ties
    Q = rng.integers(0, 4, size=(20, 32)).astype(np.float32)
    ix = _idx(torch, 32)
    gi, gd = ix.bruteforce_knn(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), 50)
    oi, od = O.brute_force_knn(X, Q, 50)
    assert np.array_equal(gi.cpu().numpy(), oi)


@pytest.fixture(params=[1, 3], ids=["1-pass", "3-pass"])
def probe_passes(request):
    # the probe's tensor-core filter runs 1-pass (hi parts, wide window) or 3-pass (split); both
    # must certify the same exact answer
    _OPTS["probe_passes"] = request.param
    return request.param


def test_probe_and_assign_bit_exact(torch_cuda, probe_passes):
    torch = torch_cuda
    rng = np.random.default_rng(2)
    D, n, C = 64, 6000, 200
    X = rng.integers(0, 6, size=(n, D)).astype(np.float32)
    cent = X[rng.choice(n, C, replace=False)].copy()
    cent[17] = cent[3]                                           # duplicated centroid -> tie to 3
    cent[:50] += rng.standard_normal((50, D)).astype(np.float32) * 0.5
    ix = _idx(torch, D)
    mean, R, lam = O.fit_rotation(X)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), C, centroids=torch.from_numpy(cent).cuda())
    off, row_id, assign, c2 = ix.get_ivf()
    oa, ooff, orow = O.build_ivf(X, cent)
    assert np.array_equal(assign, oa)
    assert np.array_equal(off, ooff) and np.array_equal(row_id, orow)
    Q = rng.integers(0, 6, size=(25, D)).astype(np.float32)
    pr = ix.probe(torch.from_numpy(Q).cuda(), 31).cpu().numpy()
    for q in range(25):
        assert pr[q].tolist() == O.probe(Q[q], cent, 31).tolist()


@pytest.mark.parametrize("nprobe", [1, 7, 64])
@pytest.mark.parametrize("C", [3000, 20000, 40000])
def test_probe_wide_ragged_bit_exact(torch_cuda, nprobe, C, probe_passes):
    # several column tiles per split and a ragged last tile (3000 = 23 x 128 + 56; 20000 = 625
    # 32-column groups), integer data with exact distance ties; both selection paths must return
    # the oracle's probes exactly
    torch = torch_cuda
    rng = np.random.default_rng(7)
    D, n = 96, 3 * C
    X = rng.integers(0, 5, size=(n, D)).astype(np.float32)
    cent = X[rng.choice(n, C, replace=False)].copy()
    cent[1000] = cent[10]
    ix = _idx(torch, D)
    mean, R, lam = O.fit_rotation(X)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), C, centroids=torch.from_numpy(cent).cuda())
    Q = rng.integers(0, 5, size=(300, D)).astype(np.float32)
    pr = ix.probe(torch.from_numpy(Q).cuda(), nprobe).cpu().numpy()
    for q in range(0, 300, 7):
        assert pr[q].tolist() == O.probe(Q[q], cent, nprobe).tolist()


@pytest.mark.parametrize("ares", [0, 1])
def test_probe_wide_d256_resident_a(torch_cuda, ares):
    # the wide-row d_hat writers at D = 256 (the C5 shape; nkc = 16 chunks of A resident in
    # shared memory for "1"), 1-pass filter, 64-column groups, ragged last tile: probes must equal
    # the oracle's exactly with either writer
    torch = torch_cuda
    _OPTS["probe_passes"] = 1
    _OPTS["dhat_ares"] = ares
    rng = np.random.default_rng(11)
    D, C = 256, 33000
    X = rng.integers(0, 5, size=(2 * C, D)).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    cent[20000] = cent[30]
    ix = _idx(torch, D)
    mean, R, lam = O.fit_rotation(X)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), C, centroids=torch.from_numpy(cent).cuda())
    Q = rng.integers(0, 5, size=(200, D)).astype(np.float32)
    pr = ix.probe(torch.from_numpy(Q).cuda(), 8).cpu().numpy()
    for q in range(0, 200, 9):
        assert pr[q].tolist() == O.probe(Q[q], cent, 8).tolist()
