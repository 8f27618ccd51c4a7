"""GPU parity for NEXT-4 (graph refinement with the DCO, R33-R35): the hand-worked search of
tests/test_oracle_graph.py, the plain (alpha = 0) traversal, per-node decisions against the
oracle's graph_search on the same (injected) graph and calibration, and the library's graph
builder against the oracle's."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.helpers import rel_err, tie_adjusted_overlap
from tests.stage_parity import BAND
from tests.test_oracle_graph import _hand_graph
from tests.test_oracle_search_pins import CAL, D as HD

pytestmark = pytest.mark.gpu


def _lib():
    import torch
    assert torch.cuda.is_available()
    from paper_2404_16322_b200 import Index, build
    build.build()
    return torch, Index


def test_hand_worked_graph_search_on_gpu():
    torch, Index = _lib()
    X, idx = _hand_graph()
    ix = Index(HD)
    ix.set_rotation(np.zeros(HD), np.eye(HD), np.ones(HD))
    ix.build_ivf(torch.from_numpy(X).cuda(), 1, centroids=torch.zeros((1, HD), device="cuda"))
    ix.set_graph(idx["nbrs"], idx["entry"])
    nb, e = ix.get_graph()
    assert np.array_equal(nb, idx["nbrs"]) and e == 0
    ix.set_calibration(2, CAL["m1"], CAL["v"])                   # the step table, calibrated K = ef = 2
    gi, gd, st, log = ix.graph_search(torch.zeros((1, HD), device="cuda"), 1, 2, 16, 0.1, stats=True, log=True)
    assert gi.tolist() == [[3]] and gd.tolist() == [[0.25]]
    assert sorted(map(tuple, log.cpu().numpy().tolist())) == [(0, 0, 48), (0, 1, 48), (0, 2, 48), (0, 3, 48), (0, 4, 32)]
    assert st["pruned_at_step"][:3] == [0, 0, 1] and st["n_epochs"] == 3 and st["dims_scanned"] == 4 * 48 + 32


@pytest.fixture(scope="module")
def graph_case():
    torch, Index = _lib()
    cfg = synth.config("c2", n=3000, nlist=8, nq=30, n_cal=80)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    nbrs, entry = O.build_graph(X, 32, 64)
    ef = 32
    oidx = O.build_index(X, X[:1].copy(), mean, R)
    oidx["nbrs"], oidx["entry"] = nbrs, entry
    oidx["cal"] = O.calibrate(X, oidx, synth.cal_queries(cfg), ef, n_neg=50, nprobe_neg=0, seed=0)
    ix = Index(cfg.d)
    ix.set_rotation(mean, R, lam)
    Xd = torch.from_numpy(X).cuda()
    ix.build_ivf(Xd, 1, centroids=torch.from_numpy(X[:1].copy()).cuda())
    ix.set_graph(nbrs, entry)
    ix.set_calibration(ef, oidx["cal"]["m1"], oidx["cal"]["v"])
    return torch, cfg, X, Xd, ix, oidx, ef


def test_graph_search_alpha0_matches_oracle(graph_case):
    # no DCO (alpha = 0), wide queue: the same traversal as the oracle's, near-exact results
    torch, cfg, X, Xd, ix, oidx, ef = graph_case
    Q = synth.queries(cfg)[:10]
    gi, gd = ix.graph_search(torch.from_numpy(Q).cuda(), 10, 256, 16, 0.0)[:2]
    oi, od, _ = O.graph_search(oidx, Q, 10, 256, 16, 0.0)
    bi, bd = O.brute_force_knn(X, Q, 10)
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), oi, od) == 1.0
    assert O.recall_at_k(oi, bi, 10) >= 0.99


def _graph_decisions(glog, ocands):
    """Per query, walk the oracle's tested nodes in order; at the first node whose GPU decision
    differs (or that the GPU did not test) the oracle's closest call must be inside the band — the
    traversal may then diverge, so the rest of that query is not compared."""
    g = {}
    for q, i, d in np.asarray(glog, np.int64).tolist():
        assert (q, i) not in g, "a node was tested twice"
        g[(q, i)] = d
    flagged = set()
    done = set()
    n_cmp = 0
    for oq, oi, od, om in ocands:
        for q, i, d, m in zip(oq.tolist(), oi.tolist(), od.tolist(), om.tolist()):
            if q in flagged:
                continue
            n_cmp += 1
            if g.get((q, i)) != d:
                assert m <= BAND, (q, i, d, g.get((q, i)), m)
                flagged.add(q)
            done.add((q, i))
    # outside the flagged queries the GPU tested exactly the oracle's nodes
    extra = [k for k in g if k[0] not in flagged and k not in done]
    assert not extra, extra[:5]
    return flagged, n_cmp


@pytest.mark.parametrize("alpha,dd", [(0.005, 16), (0.05, 32)])
def test_graph_decisions_match_oracle(graph_case, alpha, dd):
    torch, cfg, X, Xd, ix, oidx, ef = graph_case
    Q = synth.queries(cfg)
    gi, gd, st, log = ix.graph_search(torch.from_numpy(Q).cuda(), 10, ef, dd, alpha, stats=True, log=True)
    oi, od, ost = O.graph_search(oidx, Q, 10, ef, dd, alpha, log=True)
    flagged, n_cmp = _graph_decisions(log.cpu().numpy(), ost["candidates"])
    assert len(flagged) <= 1 and n_cmp > 1000
    keep = [q for q in range(Q.shape[0]) if q not in flagged]
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    assert tie_adjusted_overlap(gi[keep], gd[keep], oi[keep], od[keep]) == 1.0
    same = gi == oi
    assert rel_err(gd[same], od[same]) <= 1e-5
    if not flagged:
        assert st["tested"] == ost["tested"] and st["dims_scanned"] == ost["dims_scanned"]
        assert st["n_epochs"] == ost["expansions"]
    assert sum(st["pruned_at_step"]) > 0.2 * st["tested"]                  # the DCO prunes


def test_library_graph_builder_matches_oracle(graph_case):
    torch, cfg, X, Xd, ix, oidx, ef = graph_case
    from paper_2404_16322_b200 import Index
    iy = Index(cfg.d)
    mean, R, lam = ix.get_rotation()
    iy.set_rotation(mean, R, lam)
    iy.build_ivf(Xd, 1, centroids=torch.from_numpy(X[:1].copy()).cuda())
    iy.build_graph(Xd, M0=32, P=64)                                      # exact pools (every list)
    nb, entry = iy.get_graph()
    assert entry == oidx["entry"]
    same_rows = np.mean([np.array_equal(a, b) for a, b in zip(nb, oidx["nbrs"])])
    assert same_rows >= 0.98, same_rows                                   # fp32 vs fp64 near-ties only
    Q = synth.queries(cfg)
    gi, gd = iy.graph_search(torch.from_numpy(Q).cuda(), 10, 64, 16, 0.0)[:2]
    bi, _ = O.brute_force_knn(X, Q, 10)
    assert O.recall_at_k(gi.cpu().numpy(), bi, 10) >= 0.95


def test_graph_decisions_with_ivf_entry(graph_case):
    # nlist > 1: the entry point of each query is the lowest-id node of its nearest non-empty list
    # (R33); the same decisions as the oracle's on the same graph and calibration
    torch, cfg, X, Xd, ix, oidx, ef = graph_case
    from paper_2404_16322_b200 import Index
    cent = O.kmeans(X, 16, iters=2)
    mean, R, lam = ix.get_rotation()
    iz = Index(cfg.d)
    iz.set_rotation(mean, R, lam)
    iz.build_ivf(Xd, 16, centroids=torch.from_numpy(cent).cuda())
    iz.set_graph(oidx["nbrs"], oidx["entry"])
    iz.set_calibration(ef, oidx["cal"]["m1"], oidx["cal"]["v"])
    o16 = O.build_index(X, cent, mean, R, oidx["cal"])
    o16["nbrs"], o16["entry"] = oidx["nbrs"], oidx["entry"]
    Q = synth.queries(cfg)
    gi, gd, log = iz.graph_search(torch.from_numpy(Q).cuda(), 10, ef, 16, 0.005, log=True)
    oi, od, ost = O.graph_search(o16, Q, 10, ef, 16, 0.005, log=True)
    flagged, n_cmp = _graph_decisions(log.cpu().numpy(), ost["candidates"])
    assert len(flagged) <= 1
    keep = [q for q in range(Q.shape[0]) if q not in flagged]
    assert tie_adjusted_overlap(gi.cpu().numpy()[keep], gd.cpu().numpy()[keep], oi[keep], od[keep]) == 1.0
