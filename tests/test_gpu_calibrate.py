"""GPU calibration vs the oracle's (same rotation / centroids injected)."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O

pytestmark = pytest.mark.gpu


def test_calibration_table_matches_oracle():
    import torch
    assert torch.cuda.is_available()
    from paper_2404_16322_b200 import build, Index
    build.build()
    cfg = synth.config("c2", n=20000, nlist=64, nq=10, n_cal=150)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    cent = O.kmeans(X, cfg.nlist, iters=3)
    oidx = O.build_index(X, cent, mean, R)
    Qc = synth.cal_queries(cfg)
    ocal = O.calibrate(X, oidx, Qc, cfg.k, n_neg=50, nprobe_neg=6, seed=7)
    ix = Index(cfg.d)
    ix.set_rotation(mean, R, lam)
    Xd = torch.from_numpy(X).cuda()
    ix.build_ivf(Xd, cfg.nlist, centroids=torch.from_numpy(cent).cuda())
    ix.calibrate(Xd, torch.from_numpy(Qc).cuda(), cfg.k, n_neg=50, nprobe_neg=6, seed=7)
    gcal = ix.get_calibration()
    assert gcal["n0"] == ocal["n0"] == 150 * cfg.k
    np.testing.assert_allclose(gcal["m1"], ocal["m1"], rtol=1e-4)
    for alpha in (0.005, 0.05):
        gm, gb = O.step_table(gcal, cfg.d, 16, alpha)
        om, ob = O.step_table(ocal, cfg.d, 16, alpha)
        scale = np.median(np.abs(ocal["v"]))
        assert np.max(np.abs(gb - ob)) <= 1e-4 * scale + 1e-3


def test_sharded_calibration_equals_single():
    # the sharded calibration protocol (sharded.py: per-shard K-NN / negatives / pair features,
    # merged and summed as the all-gathers and all-reduce would) installs exactly the table an
    # unsharded dade_calibrate computes on the same base, centroids and rotation
    import torch
    from paper_2404_16322_b200 import Index, build, dade
    build.build()
    cfg = synth.config("c2", n=24000, nlist=64, nq=10, n_cal=40)
    X = synth.base(cfg)
    Qc = torch.from_numpy(synth.cal_queries(cfg)).cuda()
    Xd = torch.from_numpy(X).cuda()
    mean, R, lam = O.fit_rotation(X)
    cent = torch.from_numpy(O.kmeans(X, cfg.nlist, iters=2)).cuda()
    full = Index(cfg.d)
    full.set_rotation(mean, R, lam)
    full.build_ivf(Xd, cfg.nlist, centroids=cent)
    full.calibrate(Xd, Qc, cfg.k, n_neg=cfg.n_neg, nprobe_neg=6, seed=3)
    ref = full.get_calibration()
    S = 3
    shards = []
    for s in range(S):
        lo, hi = s * cfg.n // S, (s + 1) * cfg.n // S
        ix = Index(cfg.d)
        ix.set_rotation(mean, R, lam)
        ix.build_ivf(Xd[lo:hi].contiguous(), cfg.nlist, centroids=cent, id_base=lo)
        shards.append((ix, Xd[lo:hi].contiguous()))
    kl = [ix.calib_knn(Xs, Qc, cfg.k) for ix, Xs in shards]
    knn_ids, knn_d = dade.merge_knn(np.stack([k[0] for k in kl]), np.stack([k[1] for k in kl]), cfg.k)
    ng = [ix.calib_negatives(Qc, cfg.k, knn_ids, cfg.n_neg, 6, 3) for ix, _ in shards]
    pq, pid, tau, y = dade.calibration_pairs(knn_ids, knn_d, np.stack([g[0] for g in ng]),
                                                np.stack([g[1] for g in ng]), np.stack([g[2] for g in ng]), cfg.n_neg)
    F = sum(ix.pair_features(Qc, pq, pid) for ix, _ in shards)
    shards[0][0].fit_calibration(cfg.k, F, tau, y)
    got = shards[0][0].get_calibration()
    assert got["n0"] == ref["n0"] and got["K"] == ref["K"]
    assert np.array_equal(got["m1"], ref["m1"]) and np.array_equal(got["v"], ref["v"])
