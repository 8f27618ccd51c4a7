"""GPU parity of the throughput fused probe filter (probe_fz.cu, DADE_OPT_KNN_PATH 4 = fp16
operands, 5 = tf32): probes bit-exact against the oracle's fp64 definition (R20) on the
shapes the bench runs (C2/C4/C5-shard widths), ragged tiles, integer ties, k up to 64, and the
fp16 edge cases — rows that span fp16's subnormal range after scaling, a query equal to the
centring vector (zero row), tiny and huge magnitudes (the power-of-two scales)."""
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


def _index(torch, X, cent, path):
    from paper_2404_16322_b200 import Index
    D = X.shape[1]
    ix = Index(D)
    ix.set_option("knn_path", path)
    ix.set_option("probe_passes", 1)
    mean, R, lam = O.fit_rotation(X)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), cent.shape[0], centroids=torch.from_numpy(cent).cuda())
    return ix


def _check(torch, ix, Q, cent, nprobe, step=1):
    pr = ix.probe(torch.from_numpy(Q).cuda(), nprobe).cpu().numpy()
    for q in range(0, Q.shape[0], step):
        assert pr[q].tolist() == O.probe(Q[q], cent, nprobe).tolist(), f"query {q}"
    return pr


@pytest.mark.parametrize("path", [4, 5])
@pytest.mark.parametrize("D,C,nprobe", [(128, 4096, 8), (96, 16384, 8), (256, 20000, 8), (96, 3000, 64),
                                        (32, 777, 1), (256, 1000, 33)])
def test_fz_mixture_bit_exact(torch_cuda, path, D, C, nprobe):
    # Gaussian-mixture data like the bench's: centroids are noisy data points, queries from the
    # same mixture; ragged last column tiles (3000, 777, 20000 = 156 x 128 + 32, 1000)
    torch = torch_cuda
    rng = np.random.default_rng(D * 7 + C)
    centers = rng.standard_normal((64, D)).astype(np.float32) * 2
    X = (centers[rng.integers(0, 64, 2 * C)] + rng.standard_normal((2 * C, D)).astype(np.float32)).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent, path)
    Q = (centers[rng.integers(0, 64, 300)] + rng.standard_normal((300, D)).astype(np.float32)).astype(np.float32)
    _check(torch, ix, Q, cent, nprobe, step=3)


@pytest.mark.parametrize("path", [4, 5])
@pytest.mark.parametrize("nprobe", [1, 16, 64])
def test_fz_integer_ties(torch_cuda, path, nprobe):
    # small-integer data: massive exact distance ties, duplicated centroids (ties go to the lower id)
    torch = torch_cuda
    rng = np.random.default_rng(nprobe)
    D, C = 64, 5000
    X = rng.integers(0, 4, size=(3 * C, D)).astype(np.float32)
    cent = X[rng.choice(3 * C, C, replace=False)].copy()
    cent[4000] = cent[7]
    cent[4001] = cent[7]
    ix = _index(torch, X, cent, path)
    Q = rng.integers(0, 4, size=(257, D)).astype(np.float32)
    _check(torch, ix, Q, cent, nprobe, step=2)


@pytest.mark.parametrize("scale", [1e-18, 1.0, 3e15])
def test_fz_fp16_scales(torch_cuda, scale):
    # magnitudes far outside fp16's range: the power-of-two scales must map them in and out exactly
    torch = torch_cuda
    rng = np.random.default_rng(3)
    D, C = 96, 2000
    X = (rng.standard_normal((2 * C, D)) * scale).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent, 4)
    Q = (rng.standard_normal((200, D)) * scale).astype(np.float32)
    _check(torch, ix, Q, cent, 8)


def test_fz_fp16_dynamic_range_and_zero_rows(torch_cuda):
    # rows whose coordinates span ~40 binades (many land in fp16's subnormal range after the row
    # scale: the slack's absolute term must cover them), a query equal to the centring vector
    # (the centroids' mean: a zero operand row), and duplicated queries
    torch = torch_cuda
    rng = np.random.default_rng(5)
    D, C = 128, 3000
    mags = np.exp2(rng.uniform(-30, 10, size=(1, D))).astype(np.float32)
    X = (rng.standard_normal((2 * C, D)) * mags).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent, 4)
    Q = (rng.standard_normal((130, D)) * mags).astype(np.float32)
    Q[0] = cent.astype(np.float64).mean(axis=0).astype(np.float32)
    Q[1] = Q[2]
    Q[129] = 0.0
    _check(torch, ix, Q, cent, 12)


@pytest.mark.parametrize("path", [4, 5])
@pytest.mark.parametrize("k", [32, 64])
def test_fz_large_k(torch_cuda, path, k):
    torch = torch_cuda
    rng = np.random.default_rng(k)
    D, C = 48, 6000
    X = rng.standard_normal((2 * C, D)).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent, path)
    Q = rng.standard_normal((200, D)).astype(np.float32)
    _check(torch, ix, Q, cent, k, step=5)


def test_fz_many_rows_chunks(torch_cuda):
    # more query rows than one 128-row tile wave, ragged last row tile (1000 = 7 x 128 + 104)
    torch = torch_cuda
    rng = np.random.default_rng(9)
    D, C = 96, 16384
    X = rng.standard_normal((C + 5000, D)).astype(np.float32)
    cent = X[:C].copy()
    ix = _index(torch, X, cent, 4)
    Q = rng.standard_normal((1000, D)).astype(np.float32)
    _check(torch, ix, Q, cent, 8, step=37)
    # every path agrees on every row
    pr4 = ix.probe(torch.from_numpy(Q).cuda(), 8).cpu().numpy()
    ix.set_option("knn_path", 1)
    pr1 = ix.probe(torch.from_numpy(Q).cuda(), 8).cpu().numpy()
    assert np.array_equal(pr4, pr1)


@pytest.mark.parametrize("D,C,nprobe,nq", [(256, 20000, 8, 300), (96, 16384, 8, 1000), (128, 4096, 8, 257),
                                           (64, 5000, 16, 129), (32, 777, 1, 40), (256, 1000, 33, 513)])
@pytest.mark.parametrize("rows,cols", [(2, 1), (1, 2), (2, 2)])
def test_fz_row_tile_pairs(torch_cuda, D, C, nprobe, nq, rows, cols):
    # DADE_OPT_FZ_ROWS = 2: two resident 128-row A tiles share every B chunk (two accumulators, one
    # epilogue group per half); ragged pairs (nq = 300, 257, 129, 40, 513: the second tile of the
    # last pair partly or wholly past the rows). DADE_OPT_FZ_COLS = 2: two epilogue groups drain
    # each accumulator (64 columns each, separate per-row windows and lists, united by the select
    # pass and the finish). Bit-exact vs the oracle and equal to the default kernel on every row;
    # integer data adds exact ties.
    if rows * cols == 4 and D > 128:
        pytest.skip("two A tiles + four epilogue groups exceed shared memory at D > 128")
    torch = torch_cuda
    rng = np.random.default_rng(D + C + nq)
    if D == 64:
        X = rng.integers(0, 4, size=(2 * C, D)).astype(np.float32)
        Q = rng.integers(0, 4, size=(nq, D)).astype(np.float32)
    else:
        centers = rng.standard_normal((64, D)).astype(np.float32) * 2
        X = (centers[rng.integers(0, 64, 2 * C)] + rng.standard_normal((2 * C, D)).astype(np.float32)).astype(np.float32)
        Q = (centers[rng.integers(0, 64, nq)] + rng.standard_normal((nq, D)).astype(np.float32)).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    ix = _index(torch, X, cent, 4)
    ix.set_option("fz_rows", rows)
    ix.set_option("fz_cols", cols)
    pr2 = _check(torch, ix, Q, cent, nprobe, step=3)
    ix.set_option("fz_rows", 0)
    ix.set_option("fz_cols", 0)
    pr1 = ix.probe(torch.from_numpy(Q).cuda(), nprobe).cpu().numpy()
    assert np.array_equal(pr2, pr1)


@pytest.mark.parametrize("D,C,nprobe", [(960, 4096, 64), (512, 3000, 16), (960, 777, 8)])
def test_int8_split_filter_gist_like(torch_cuda, D, C, nprobe):
    # the int8 exact-split filter (knn_path 6; DADE_OPT_KNN_I8 for D >= 512): GIST-like
    # data in [0, 1] with a decaying spectrum (dense near-ties at D = 960), ragged column tiles;
    # probes bit-exact against the oracle and equal to the 3-pass tf32 path's
    torch = torch_cuda
    from paper_2404_16322_b200 import Index
    rng = np.random.default_rng(D + C)
    lam = np.arange(1, D + 1, dtype=np.float64) ** -1.5
    basis = np.linalg.qr(rng.standard_normal((D, D)))[0]
    X = ((rng.standard_normal((2 * C, D)) * np.sqrt(lam)) @ basis.T)
    X = ((X - X.min()) / (X.max() - X.min())).astype(np.float32)
    cent = X[rng.choice(2 * C, C, replace=False)].copy()
    cent[C - 1] = cent[3]
    ix = Index(D)
    mean, R, lam_ = O.fit_rotation(X)
    ix.set_rotation(mean, R, lam_)
    ix.build_ivf(torch.from_numpy(X).cuda(), C, centroids=torch.from_numpy(cent).cuda())
    Q = np.clip(((rng.standard_normal((200, D)) * np.sqrt(lam)) @ basis.T - X.min()) / (X.max() - X.min()), 0, 1)
    Q = Q.astype(np.float32)
    Q[5] = cent[3]
    ix.set_option("probe_passes", 3)
    ix.set_option("knn_path", 6)
    pr = _check(torch, ix, Q, cent, nprobe, step=4)
    ix.set_option("knn_path", 1)
    ix.set_option("knn_i8", 0)
    pr3 = ix.probe(torch.from_numpy(Q).cuda(), nprobe).cpu().numpy()
    assert np.array_equal(pr, pr3)
