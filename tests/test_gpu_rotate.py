"""GPU parity of the tensor-core rotation (a1 database rows, a4 queries; rotate.cu: tcgen05
kind::i8 with a 6-way split, exact int32 levels combined in fp64) against the oracle's fp64
rotation x~ = R(x - mu). Every stored coordinate must be within its own fp32
rounding (2^-24 |x~_i|) plus the split's bound 9 D 2^-42 2^(e_v + e_i) (2^e_v > max|v| of the row,
2^e_i > max|r_i|; rotate.cu header), and almost all of them equal the correctly rounded fp64
value. Ragged tiles (n = 1, 129), D = 16 .. 960, zero rows (x = mu) and extreme scales."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O

pytestmark = pytest.mark.gpu


def _lib():
    import torch
    assert torch.cuda.is_available()
    from paper_2404_16322_b200 import Index, build
    build.build()
    return torch, Index


def _bound(V, R, ref):
    """|gpu - ref| allowed per coordinate: half an fp32 ulp of ref + the split error bound."""
    D = V.shape[1]
    ev = np.frexp(np.max(np.abs(V), axis=1))[1].astype(np.float64)      # max|v| < 2^ev
    er = np.frexp(np.max(np.abs(R), axis=1))[1].astype(np.float64)
    split = 9.0 * D * 2.0 ** (-42) * np.exp2(ev[:, None] + er[None, :])
    return np.abs(ref) * 2.0 ** -24 + split + 1e-13 * np.abs(ref)


def _rotation(D, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((D, D)))
    return Q


def _check(gpu, ref, V, R):
    gpu = gpu.astype(np.float64)
    bound = _bound(V, R, ref)
    err = np.abs(gpu - ref)
    assert np.all(err <= bound), (np.max(err / bound), np.unravel_index(np.argmax(err / bound), err.shape))
    same = np.mean(gpu == ref.astype(np.float32).astype(np.float64))
    return same


@pytest.mark.parametrize("cfg_name,D,n", [("c2", 128, 3000), ("c4", 96, 129), ("c3", 960, 300),
                                          ("c1", 16, 1), ("c2", 256, 1000)])
def test_layout_rotation_matches_fp64(cfg_name, D, n):
    torch, Index = _lib()
    cfg = synth.config(cfg_name, n=n, d=D, nq=4)
    X = synth.base(cfg)
    mu = X.mean(axis=0, dtype=np.float64)
    R = _rotation(D, 1)
    ix = Index(D)
    ix.set_rotation(mu, R, np.ones(D))
    ix.build_ivf(torch.from_numpy(X).cuda(), 1, centroids=torch.from_numpy(X[:1].copy()).cuda())
    off, row_id, _, _ = ix.get_ivf()
    lay = ix.get_layout()
    V = X[row_id].astype(np.float64) - mu
    ref = O.rotate(X[row_id], mu, R)
    same = _check(lay, ref, V, R)
    assert same >= 0.99, same


@pytest.mark.parametrize("scale", [1.0, 1e-20, 1e20])
def test_query_rotation_matches_fp64(scale):
    torch, Index = _lib()
    D = 128
    cfg = synth.config("c2", n=600, nq=300, nlist=4)
    X = (synth.base(cfg) * np.float32(scale)).astype(np.float32)
    Q = (synth.queries(cfg) * np.float32(scale)).astype(np.float32)
    Q[5] = X[0]                       # a query with v = x - mu of mixed magnitudes
    mu = X.mean(axis=0, dtype=np.float64)
    Q[7] = mu.astype(np.float32)      # v ~ 0 (only the fp32 rounding of mu survives)
    R = _rotation(D, 2)
    ix = Index(D)
    ix.set_rotation(mu, R, np.ones(D))
    ix.build_ivf(torch.from_numpy(X).cuda(), 4, kmeans_iters=1)
    qrot, _ = ix.prepare(torch.from_numpy(Q).cuda(), 2)
    V = Q.astype(np.float64) - mu
    ref = O.rotate(Q, mu, R)
    same = _check(qrot.cpu().numpy(), ref, V, R)
    assert same >= 0.99, same


def test_zero_rows():
    # rows equal to mu rotate to exactly 0 (exponent 0, all slices 0); their neighbours are unaffected
    torch, Index = _lib()
    D = 32
    rng = np.random.default_rng(3)
    X = rng.standard_normal((200, D)).astype(np.float32)
    mu = X[0].astype(np.float64)
    X[7] = X[0]
    R = _rotation(D, 4)
    ix = Index(D)
    ix.set_rotation(mu, R, np.ones(D))
    ix.build_ivf(torch.from_numpy(X).cuda(), 1, centroids=torch.zeros((1, D), device="cuda"))
    off, row_id, _, _ = ix.get_ivf()
    lay = ix.get_layout()
    for z in (0, 7):
        assert np.all(lay[np.where(row_id == z)[0][0]] == 0.0)
    V = X[row_id].astype(np.float64) - mu
    _check(lay, O.rotate(X[row_id], mu, R), V, R)
