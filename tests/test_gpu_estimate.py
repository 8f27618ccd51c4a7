"""GPU parity of NEXT-2's Exp-7 flat estimate scan (`dade_estimate_knn`, R27) against
the oracle: the K smallest estimates agree value by value within the north_star's 1e-5 relative,
the ids within the tie-adjusted overlap; every estimator, d in {16, 32, D}, K in {1, 100, 256},
a random orthogonal basis ("Rand"), a ragged row count, D = 960, and the argument errors."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.helpers import rel_err, tie_adjusted_overlap

pytestmark = pytest.mark.gpu


def _setup(cfg, R=None):
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import build, Index
    build.build()
    X = synth.base(cfg)
    mean, Rp, lam = O.fit_rotation(X)
    R = Rp if R is None else R
    cent = O.kmeans(X, cfg.nlist, iters=2)
    oidx = O.build_index(X, cent, mean, R)
    ix = Index(cfg.d)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), cfg.nlist, centroids=torch.from_numpy(cent).cuda())
    return torch, ix, oidx, X


@pytest.fixture(scope="module")
def sift_est():
    cfg = synth.config("c2", n=30001, nlist=64, nq=24)   # ragged: not a multiple of the 1,024-row sweep
    return cfg, _setup(cfg)


def _check(torch, ix, oidx, Q, d, K, est):
    gi, ge = ix.estimate_knn(torch.from_numpy(Q).cuda(), d, K, est)
    gi, ge = gi.cpu().numpy(), ge.cpu().numpy()
    oi, oe = O.estimate_knn(oidx, Q, d, K, est)
    assert rel_err(ge, oe) <= 1e-5
    assert tie_adjusted_overlap(gi, ge, oi, oe) >= 0.999
    assert np.all(np.diff(ge, axis=1) >= 0)


@pytest.mark.parametrize("est", ["partial", "residual"])
@pytest.mark.parametrize("d", [16, 32, 128])
@pytest.mark.parametrize("K", [1, 100, 256])
def test_estimate_parity_sift_shaped(sift_est, est, d, K):
    cfg, (torch, ix, oidx, X) = sift_est
    _check(torch, ix, oidx, synth.queries(cfg), d, K, est)


def test_full_dimension_is_exact_knn(sift_est):
    cfg, (torch, ix, oidx, X) = sift_est
    Q = synth.queries(cfg)
    gi, ge = ix.estimate_knn(torch.from_numpy(Q).cuda(), cfg.d, 10, "partial")
    bi, bd = ix.bruteforce_knn(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), 10)
    oi, od = O.brute_force_knn(X, Q, 10)
    assert tie_adjusted_overlap(gi.cpu().numpy(), ge.cpu().numpy(), oi, od) >= 0.999
    assert rel_err(ge.cpu().numpy(), od) <= 1e-5


def test_random_rotation_column():
    cfg = synth.config("c4", n=20000, nlist=32, nq=16)
    H = synth.haar_basis(cfg.d, np.random.default_rng(12345)).T.copy()
    torch, ix, oidx, X = _setup(cfg, R=H)
    _check(torch, ix, oidx, synth.queries(cfg), 32, 100, "partial")


def test_gist_shaped_d32():
    cfg = synth.config("c3", n=6000, nlist=16, nq=8)
    torch, ix, oidx, X = _setup(cfg)
    for est in ("partial", "residual"):
        _check(torch, ix, oidx, synth.queries(cfg), 32, 100, est)


def test_estimate_errors(sift_est):
    cfg, (torch, ix, oidx, X) = sift_est
    Q = torch.from_numpy(synth.queries(cfg)).cuda()
    from paper_2404_16322_b200.dade import DadeError
    for d, K in ((8, 10), (cfg.d + 16, 10), (0, 10), (16, 0), (16, 257)):
        with pytest.raises(DadeError):
            ix.estimate_knn(Q, d, K, "partial")
    Qn = Q.clone()
    Qn[3, 5] = float("nan")
    with pytest.raises(DadeError):
        ix.estimate_knn(Qn, 16, 10, "partial")
    ids, est = ix.estimate_knn(Q[:0], 16, 10, "residual")
    assert ids.shape == (0, 10)
