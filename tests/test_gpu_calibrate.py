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
