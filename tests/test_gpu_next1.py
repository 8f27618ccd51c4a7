"""GPU parity for NEXT-1: the paper's other two distance corrections on the same
scan kernel — ADSampling on a random orthogonal rotation and BSA-res (Alg. 2,
P:L434-470) — against the oracle on the same seeded inputs: identical candidate counts, returned
distances within 1e-5 of the exact distance of each id, tie-adjusted ID overlap >= 0.999, and the
number of dimensions read within 1% (decisions identical outside R21's tie band)."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.helpers import rel_err, tie_adjusted_overlap

pytestmark = pytest.mark.gpu


def _setup(cfg, random_rotation):
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import Index, build
    build.build()
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    if random_rotation:  # ADSampling's projection: a Haar-random orthogonal matrix
        R = synth.haar_basis(cfg.d, np.random.default_rng(11)).T.copy()
    cent = O.kmeans(X, cfg.nlist, iters=3)
    oidx = O.build_index(X, cent, mean, R, lam=lam)
    ix = Index(cfg.d)
    ix.set_rotation(mean, R, lam)
    ix.build_ivf(torch.from_numpy(X).cuda(), cfg.nlist, centroids=torch.from_numpy(cent).cuda())
    return torch, ix, oidx, X


def _compare(torch, ix, oidx, Q, cfg, nprobe, method, param):
    K = cfg.k
    gi, gd, st = ix.search_method(torch.from_numpy(Q).cuda(), K, nprobe, cfg.delta_d, method, param, stats=True)
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    kw = {"eps0": param} if method == "adsampling" else {"m_res": param}
    oi, od, ost = O.search(oidx, Q, K, nprobe, cfg.delta_d, 0.005, method=method, **kw)
    assert st["tested"] == ost["tested"]
    assert tie_adjusted_overlap(gi, gd, oi, od) >= 0.999
    Qr = O.rotate(Q, oidx["mean"], oidx["R"])
    for q in range(Q.shape[0]):
        ok = gi[q] >= 0
        ex = np.sum((oidx["Xr"][gi[q][ok] - oidx["id_base"]] - Qr[q]) ** 2, axis=1)
        assert rel_err(gd[q][ok], ex) <= 1e-5
    assert abs(st["dims_scanned"] - ost["dims_scanned"]) <= 0.01 * ost["dims_scanned"] + 64
    assert st["dims_scanned"] < st["tested"] * cfg.d        # the test prunes
    assert st["tested"] == sum(st["pruned_at_step"]) + st["survivors"]
    return st, ost


@pytest.mark.parametrize("name,kw,nprobe", [("c2", dict(n=30000, nlist=120, nq=40, n_cal=10), 6),
                                            ("c4", dict(n=30000, nlist=96, nq=40, n_cal=10), 8),
                                            ("c5", dict(n=16000, nlist=48, nq=12, n_cal=10), 5)])
@pytest.mark.parametrize("method,param", [("adsampling", 2.1), ("bsa_res", 8.0), ("bsa_res", 2.0)])
def test_next1_parity(name, kw, nprobe, method, param):
    cfg = synth.config(name, **kw)
    torch, ix, oidx, X = _setup(cfg, random_rotation=(method == "adsampling"))
    _compare(torch, ix, oidx, synth.queries(cfg), cfg, nprobe, method, param)


def test_next1_errors():
    cfg = synth.config("c2", n=3000, nlist=12, nq=4, n_cal=10)
    torch, ix, oidx, X = _setup(cfg, random_rotation=False)
    from paper_2404_16322_b200 import DadeError
    Q = torch.from_numpy(synth.queries(cfg)).cuda()
    with pytest.raises(DadeError):
        ix.search_method(Q, 10, 4, 16, "adsampling", 0.0)   # eps0 must be positive
    with pytest.raises(DadeError):
        ix.search_method(Q, 10, 4, 16, "bsa_res", -1.0)     # m must be positive
