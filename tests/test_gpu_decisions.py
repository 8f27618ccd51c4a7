"""Per-candidate decision parity (SURVEY §8(c) "decisions identical outside R21's tie band"):
the GPU's decision log (dade_search_log: every tested candidate's (query, id, dims read)) against
the oracle's per-candidate log on the same inputs and artefacts; pruned_at_step compared exactly;
the hand-worked prune case of tests/test_oracle_search_pins.py reproduced on the GPU; Δd values
that are multiples of 16 other than 16/32/64."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.helpers import rel_err, tie_adjusted_overlap
from tests.stage_parity import compare_decisions, step_histogram
from tests.test_gpu_search import _setup
from tests.test_oracle_search_pins import CAL, D as HD, hand_case

pytestmark = pytest.mark.gpu


def _check(torch, ix, oidx, Q, K, nprobe, dd, alpha, max_flag_frac=0.02):
    D = Q.shape[1]
    gi, gd, glog = ix.search_log(torch.from_numpy(Q).cuda(), K, nprobe, dd, alpha)
    gi, gd, glog = gi.cpu().numpy(), gd.cpu().numpy(), glog.cpu().numpy()
    oi, od, ost = O.search(oidx, Q, K, nprobe, dd, alpha, log=True)
    flagged, oq, odims, gdims = compare_decisions(glog, ost["candidates"])
    assert len(flagged) <= max(1, int(max_flag_frac * Q.shape[0])), flagged
    # outside the flagged queries: identical decisions -> identical histograms and results
    h_o = step_histogram(oq, odims, D, dd, flagged)
    h_g = step_histogram(oq, gdims, D, dd, flagged)
    assert np.array_equal(h_o, h_g)
    keep = [q for q in range(Q.shape[0]) if q not in flagged]
    assert tie_adjusted_overlap(gi[keep], gd[keep], oi[keep], od[keep]) == 1.0
    same = gi[keep] == oi[keep]
    assert rel_err(gd[keep][same], od[keep][same]) <= 1e-5
    # the plain search's counters equal the log's (all queries)
    _, _, st = ix.search(torch.from_numpy(Q).cuda(), K, nprobe, dd, alpha, stats=True)
    h_all = step_histogram(oq, gdims, D, dd)
    assert st["pruned_at_step"][:len(h_all)] == h_all.tolist()
    assert st["dims_scanned"] == int(gdims.sum()) and st["tested"] == len(gdims)
    return flagged, h_g


def test_hand_worked_case_on_gpu():
    """tests/test_oracle_search_pins.py's hand-derived case through the C-ABI: identity rotation,
    one list, K = 1, m1 = (2, 1), beta' = (1, 3) — ids, distances and every candidate's dims read."""
    import torch
    from paper_2404_16322_b200 import Index, build
    build.build()
    X, _ = hand_case()
    ix = Index(HD)
    ix.set_rotation(np.zeros(HD), np.eye(HD), np.ones(HD))
    ix.build_ivf(torch.from_numpy(X).cuda(), 1, centroids=torch.zeros((1, HD), device="cuda"))
    ix.set_calibration(1, CAL["m1"], CAL["v"])
    Q = torch.zeros((1, HD), device="cuda")
    gi, gd, log = ix.search_log(Q, 1, 1, 16, 0.1)
    assert gi.tolist() == [[4]] and gd.tolist() == [[1.0]]
    log = sorted(map(tuple, log.cpu().numpy().tolist()))
    assert log == [(0, i, d) for i, d in enumerate([48, 48, 48, 48, 48, 32, 48, 16, 32, 16])]
    _, _, st = ix.search(Q, 1, 1, 16, 0.1, stats=True)
    assert st["pruned_at_step"][:3] == [0, 2, 2] and st["dims_scanned"] == 384 and st["survivors"] == 6
    for G in (1, 2, 8):   # the warp split never changes a decision
        ix.set_option("scan_warps", G)
        _, _, s2 = ix.search(Q, 1, 1, 16, 0.1, stats=True)
        assert s2["pruned_at_step"] == st["pruned_at_step"]


def test_decisions_c1_flat():
    cfg = synth.config("c1")
    torch, ix, oidx, X, Xd = _setup(cfg)
    flagged, h = _check(torch, ix, oidx, synth.queries(cfg), cfg.k, 1, cfg.delta_d, 0.005)
    assert h[1:].sum() > 0                                   # pruning happens


@pytest.fixture(scope="module")
def sift_small():
    cfg = synth.config("c2", n=30000, nlist=128, nq=60, n_cal=200)
    return cfg, _setup(cfg, nprobe_neg=8)


@pytest.mark.parametrize("nprobe,dd", [(4, 16), (16, 16), (8, 32), (8, 64), (8, 128)])
def test_decisions_sift_shaped(sift_small, nprobe, dd):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    _check(torch, ix, oidx, synth.queries(cfg), cfg.k, nprobe, dd, 0.005)


def test_decisions_alpha_sweep(sift_small):
    # larger significance = more aggressive beta': decisions still identical
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    for alpha in (0.05, 0.2):
        _check(torch, ix, oidx, synth.queries(cfg)[:30], cfg.k, 8, 16, alpha)


def test_decisions_gist_shaped_k100():
    cfg = synth.config("c3", n=6000, d=256, nlist=32, nq=20, n_cal=60)
    torch, ix, oidx, X, Xd = _setup(cfg, nprobe_neg=4)
    _check(torch, ix, oidx, synth.queries(cfg), 100, 6, 32, 0.005)


@pytest.mark.parametrize("D,dd", [(96, 48), (144, 48), (160, 80), (192, 96)])
def test_delta_d_general_multiples_of_16(D, dd):
    # Δd any multiple of 16 dividing D: staged in 16-dim blocks, classifier every
    # dd/16 blocks — decisions identical to the oracle's
    cfg = synth.config("c1", n=6000, d=D, nlist=16, nq=24, n_cal=40, delta_d=dd)
    torch, ix, oidx, X, Xd = _setup(cfg, kmeans_iters=2)
    flagged, h = _check(torch, ix, oidx, synth.queries(cfg), cfg.k, 4, dd, 0.05)
    assert len(h) == D // dd


def test_adsampling_decisions(sift_small):
    # NEXT-1 ADSampling table (R8) through the same log: identical decisions
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = synth.queries(cfg)[:30]
    gi, gd, glog = ix.search_log(torch.from_numpy(Q).cuda(), cfg.k, 8, 16, 2.1, method="adsampling")
    oi, od, ost = O.search(oidx, Q, cfg.k, 8, 16, 0.005, method="adsampling", eps0=2.1, log=True)
    flagged, *_ = compare_decisions(glog.cpu().numpy(), ost["candidates"])
    assert len(flagged) <= 1
