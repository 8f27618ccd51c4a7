"""GPU parity for NEXT-3 BSA-q (§V-B): OPQ training quality, PQ codes bit-exact with
the oracle's encoding of the same stored rows (R30), the two-feature calibration against the
oracle's, and the ADC-pruned search — ids, distances and every candidate's decision — against the
oracle's search_q on the same artefacts; the hand-worked case of tests/test_oracle_bsaq.py."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.helpers import rel_err, tie_adjusted_overlap
from tests.stage_parity import compare_decisions
from tests.test_oracle_bsaq import _hand_q

pytestmark = pytest.mark.gpu


def _lib():
    import torch
    assert torch.cuda.is_available()
    from paper_2404_16322_b200 import Index, build
    build.build()
    return torch, Index


def test_hand_worked_bsaq_on_gpu():
    torch, Index = _lib()
    X, idx = _hand_q()
    ix = Index(16)
    ix.set_rotation(np.zeros(16), np.eye(16))
    ix.build_ivf(torch.from_numpy(X).cuda(), 1, centroids=torch.zeros((1, 16), device="cuda"))
    ix.set_pq(idx["pq"])
    C, codes, err = ix.get_pq()
    assert np.array_equal(codes, idx["codes"]) and np.array_equal(err, idx["pq_err"].astype(np.float32))
    ix.set_calibration_q(1, idx["calq"]["m"], idx["calq"]["v"])
    Q = torch.zeros((1, 16), device="cuda")
    gi, gd, log = ix.search_log(Q, 1, 1, 16, 0.3, method="bsa_q")
    assert gi.tolist() == [[8]] and gd.tolist() == [[0.0]]
    assert sorted(map(tuple, log.cpu().numpy().tolist())) == \
        [(0, i, d) for i, d in enumerate([16, 16, 16, 16, 0, 16, 16, 0, 16, 0])]
    _, _, st = ix.search_method(Q, 1, 1, 16, "bsa_q", 0.3, stats=True)
    assert st["pruned_at_step"] == [3] and st["survivors"] == 7 and st["dims_scanned"] == 7 * 16


@pytest.fixture(scope="module")
def pq_case():
    torch, Index = _lib()
    cfg = synth.config("c2", n=30000, nlist=64, nq=40, n_cal=150)
    X = synth.base(cfg)
    m = O.pq_subspaces(cfg.d)
    mean, R, C = O.opq_train(X, m, n_train=8192, iters=2, km_iters=2, final_iters=3)
    cent = O.kmeans(X, cfg.nlist, iters=3)
    ix = Index(cfg.d)
    ix.set_rotation(mean, R)
    Xd = torch.from_numpy(X).cuda()
    ix.build_ivf(Xd, cfg.nlist, centroids=torch.from_numpy(cent).cuda())
    ix.set_pq(C)
    # the oracle's index over the same artefacts, its codes / errors = the GPU's (stage-isolated)
    oidx = O.build_index_q(X, cent, mean, R, C)
    return torch, cfg, X, Xd, ix, oidx


def test_codes_bit_exact_on_the_stored_rows(pq_case):
    torch, cfg, X, Xd, ix, oidx = pq_case
    off, row_id, _, _ = ix.get_ivf()
    C, codes, err = ix.get_pq()
    lay = ix.get_layout()                                   # the stored fp32 x~, list-major
    oc, oe = O.pq_encode(lay, C)
    assert np.array_equal(codes, oc)                         # R30: same rows, same rule
    assert rel_err(err, oe) <= 1e-6                          # fp64 sum stored as fp32
    # against the oracle's own fp64 rotation: codes may differ only at near-ties
    same = np.mean(codes == oidx["codes"][row_id])
    assert same >= 0.995, same


def test_calibration_matches_oracle(pq_case):
    torch, cfg, X, Xd, ix, oidx = pq_case
    Qc = synth.cal_queries(cfg)
    ix.calibrate_pq(Xd, torch.from_numpy(Qc).cuda(), cfg.k, n_neg=50, nprobe_neg=8, seed=0)
    g = ix.get_calibration_q()
    o = O.calibrate_q(X, oidx, Qc, cfg.k, n_neg=50, nprobe_neg=8, seed=0)
    assert g["n0"] == o["n0"] and g["K"] == cfg.k
    np.testing.assert_allclose(g["m"], o["m"], rtol=2e-3)
    np.testing.assert_allclose(g["v"][[0, len(g["v"]) // 2, -1]], o["v"][[0, len(o["v"]) // 2, -1]],
                               rtol=2e-3, atol=1e-3 * abs(o["v"]).max())


def _stage_isolated(ix, oidx, K):
    off, row_id, _, _ = ix.get_ivf()
    C, codes, err = ix.get_pq()
    o = dict(oidx)
    base = oidx["id_base"]
    o["codes"] = np.zeros_like(codes); o["codes"][row_id - base] = codes
    o["pq_err"] = np.zeros(len(err)); o["pq_err"][row_id - base] = err
    o["calq"] = ix.get_calibration_q()
    return o


@pytest.mark.parametrize("nprobe,alpha", [(4, 0.005), (8, 0.005), (8, 0.1)])
def test_search_decisions_match_oracle(pq_case, nprobe, alpha):
    torch, cfg, X, Xd, ix, oidx = pq_case
    if not hasattr(ix, "_calq"):
        ix.calibrate_pq(Xd, torch.from_numpy(synth.cal_queries(cfg)).cuda(), cfg.k, n_neg=50, nprobe_neg=8, seed=0)
        ix._calq = True
    o = _stage_isolated(ix, oidx, cfg.k)
    Q = synth.queries(cfg)
    gi, gd, glog = ix.search_log(torch.from_numpy(Q).cuda(), cfg.k, nprobe, 16, alpha, method="bsa_q")
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    oi, od, ost = O.search_q(o, Q, cfg.k, nprobe, alpha, log=True)
    flagged, *_ = compare_decisions(glog.cpu().numpy(), ost["candidates"])
    assert len(flagged) <= 1, flagged
    keep = [q for q in range(Q.shape[0]) if q not in flagged]
    assert tie_adjusted_overlap(gi[keep], gd[keep], oi[keep], od[keep]) == 1.0
    same = gi == oi
    assert rel_err(gd[same], od[same]) <= 1e-5
    _, _, st = ix.search_method(torch.from_numpy(Q).cuda(), cfg.k, nprobe, 16, "bsa_q", alpha, stats=True)
    assert st["pruned_at_step"][0] == ost["pruned"] or flagged
    assert st["pruned_at_step"][0] > 0.3 * st["tested"]


def test_alpha0_is_exact_ivf(pq_case):
    torch, cfg, X, Xd, ix, oidx = pq_case
    Q = synth.queries(cfg)
    gi, gd = ix.search_method(torch.from_numpy(Q).cuda(), cfg.k, 6, 16, "bsa_q", 0.0)
    ei, ed = O.exact_ivf(oidx, X, Q, cfg.k, 6)
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), ei, ed) == 1.0


def test_gpu_opq_training_quality():
    # the library's OPQ (GPU assignment + cross-product, host Procrustes) against the oracle's:
    # orthogonal rotation and a distortion within 1% of the oracle's on the same sample recipe
    torch, Index = _lib()
    cfg = synth.config("c1", n=6000, d=32, nlist=8, spectrum=0.2)
    X = synth.base(cfg)
    m = O.pq_subspaces(cfg.d)
    ix = Index(cfg.d)
    ix.train_pq(torch.from_numpy(X).cuda(), m, n_train=4096, iters=3, km_iters=3, final_iters=4)
    mean, R, _ = ix.get_rotation()
    np.testing.assert_allclose(R @ R.T, np.eye(cfg.d), atol=1e-9)
    ix.build_ivf(torch.from_numpy(X).cuda(), 1, centroids=torch.zeros((1, cfg.d), device="cuda"))
    C, codes, err = ix.get_pq()
    om, oR, oC = O.opq_train(X, m, n_train=4096, iters=3, km_iters=3, final_iters=4)
    np.testing.assert_allclose(mean, om, rtol=1e-12, atol=1e-12)
    d_gpu = float(err.astype(np.float64).mean())
    d_orc = float(O.pq_encode(O.rotate(X, om, oR), oC)[1].mean())
    assert d_gpu <= 1.01 * d_orc, (d_gpu, d_orc)
