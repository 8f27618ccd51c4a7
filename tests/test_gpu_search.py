"""GPU parity for the DADE search (north_star tolerances): returned distances within 1e-5
relative of the oracle's, tie-adjusted ID overlap >= 0.999, identical candidate counts; edge
cases (empty lists, K larger than the candidate stream, nprobe = nlist, delta_d = D, ragged tails)."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.helpers import rel_err, tie_adjusted_overlap

pytestmark = pytest.mark.gpu


def _setup(cfg, kmeans_iters=4, cal=True, nprobe_neg=None, cent=None):
    import torch
    assert torch.cuda.is_available(), "GPU test run without a GPU"
    from paper_2404_16322_b200 import build, Index
    build.build()
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    if cent is None:
        cent = O.kmeans(X, cfg.nlist, iters=kmeans_iters) if cfg.nlist > 1 else X[:1].copy()
    oidx = O.build_index(X, cent, mean, R)
    if cal:
        npn = cfg.nprobe_neg if nprobe_neg is None else nprobe_neg
        oidx["cal"] = O.calibrate(X, oidx, synth.cal_queries(cfg), cfg.k, n_neg=cfg.n_neg,
                                  nprobe_neg=npn, seed=0)
    ix = Index(cfg.d)
    ix.set_rotation(mean, R, lam)
    Xd = torch.from_numpy(X).cuda()
    ix.build_ivf(Xd, cfg.nlist, centroids=torch.from_numpy(cent).cuda())
    if cal:
        ix.set_calibration(cfg.k, oidx["cal"]["m1"], oidx["cal"]["v"])
    return torch, ix, oidx, X, Xd


def _compare(torch, ix, oidx, Q, K, nprobe, dd, alpha, min_overlap=0.999):
    gi, gd, st = ix.search(torch.from_numpy(Q).cuda(), K, nprobe, dd, alpha, stats=True)
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    oi, od, ost = O.search(oidx, Q, K, nprobe, dd, alpha)
    assert st["tested"] == ost["tested"]
    ov = tie_adjusted_overlap(gi, gd, oi, od)
    assert ov >= min_overlap, ov
    # every returned GPU distance is the exact distance of that id (R21 fp32 tolerance)
    ok = gi >= 0
    assert np.array_equal(ok, oi >= 0)
    Xr = oidx["Xr"]
    Qr = O.rotate(Q, oidx["mean"], oidx["R"])
    for q in range(Q.shape[0]):
        ids = gi[q][ok[q]] - oidx["id_base"]
        ex = np.sum((Xr[ids] - Qr[q]) ** 2, axis=1)
        assert rel_err(gd[q][ok[q]], ex) <= 1e-5
    both = (gi == oi)
    if both.any():
        assert rel_err(gd[both], od[both]) <= 1e-5
    # scan-rate agreement (decisions identical outside the tau tie band)
    assert abs(st["dims_scanned"] - ost["dims_scanned"]) <= 0.01 * ost["dims_scanned"] + 64
    return gi, gd, st, oi, od, ost


def test_c1_flat_parity():
    cfg = synth.config("c1")  # configs[0] as stated: 10k x 128, K=10, Δd=32, 1,000 calibration pairs
    torch, ix, oidx, X, Xd = _setup(cfg)
    Q = synth.queries(cfg)
    gi, gd, st, oi, od, ost = _compare(torch, ix, oidx, Q, cfg.k, 1, cfg.delta_d, 0.005)
    assert st["dims_scanned"] < 0.5 * st["tested"] * cfg.d   # pruning happens (paper: 25-35% scan)


@pytest.fixture(scope="module")
def sift_small():
    cfg = synth.config("c2", n=30000, nlist=128, nq=60, n_cal=200)
    return cfg, _setup(cfg, nprobe_neg=8)


@pytest.mark.parametrize("nprobe", [4, 16])
def test_ivf_parity_sift_shaped(sift_small, nprobe):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = synth.queries(cfg)
    _compare(torch, ix, oidx, Q, cfg.k, nprobe, cfg.delta_d, 0.005)


def test_alpha0_equals_exact_ivf_and_bruteforce(sift_small):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = synth.queries(cfg)[:20]
    gi, gd = ix.search(torch.from_numpy(Q).cuda(), 10, 8, 16, 0.0)
    ei, ed = O.exact_ivf(oidx, X, Q, 10, 8)
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), ei, ed) == 1.0
    assert rel_err(gd.cpu().numpy(), ed) <= 1e-5
    gi, gd = ix.search(torch.from_numpy(Q).cuda(), 10, cfg.nlist, 16, 0.0)
    bi, bd = O.brute_force_knn(X, Q, 10)
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd) == 1.0


def test_delta_d_equal_D_and_32(sift_small):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = synth.queries(cfg)[:20]
    _compare(torch, ix, oidx, Q, cfg.k, 8, 128, 0.005)
    _compare(torch, ix, oidx, Q, cfg.k, 8, 32, 0.005)
    _compare(torch, ix, oidx, Q, cfg.k, 8, 64, 0.005)


def test_k_larger_than_stream_and_empty_lists():
    # many lists relative to n: some lists are tiny or empty; K exceeds a 1-list stream
    cfg = synth.config("c1", n=1000, nlist=200, nq=10, n_cal=20)
    X = synth.base(cfg)
    cent = O.kmeans(X, cfg.nlist, iters=2)
    cent[[7, 50, 199]] = 1e3                      # three centroids far from every row: empty lists
    torch, ix, oidx, X, Xd = _setup(cfg, cal=False, cent=cent)
    off, *_ = ix.get_ivf()
    assert (np.diff(off)[[7, 50, 199]] == 0).all()
    Q = synth.queries(cfg)
    gi, gd = ix.search(torch.from_numpy(Q).cuda(), 50, 1, 32, 0.0)
    oi, od, _ = O.search(oidx, Q, 50, 1, 32, 0.0)
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    assert np.array_equal(gi < 0, oi < 0)          # padding slots: id -1, dist +inf
    assert np.all(np.isinf(gd[gi < 0]))
    assert tie_adjusted_overlap(gi, gd, oi, od) == 1.0
    # every list probed: the empty lists sit inside the candidate stream
    gi, gd = ix.search(torch.from_numpy(Q).cuda(), 50, cfg.nlist, 32, 0.0)
    oi, od, _ = O.search(oidx, Q, 50, cfg.nlist, 32, 0.0)
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), oi, od) == 1.0


def test_gist_shaped_k100_dd32():
    cfg = synth.config("c3", n=6000, d=256, nlist=32, nq=20, n_cal=60)
    torch, ix, oidx, X, Xd = _setup(cfg, nprobe_neg=4)
    Q = synth.queries(cfg)
    _compare(torch, ix, oidx, Q, 100, 6, 32, 0.005)


def test_zero_queries_and_errors(sift_small):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    from paper_2404_16322_b200 import DadeError
    Q = torch.zeros((0, cfg.d), dtype=torch.float32, device="cuda")
    ix.search(Q, 10, 4, 16, 0.005)
    Q = torch.from_numpy(synth.queries(cfg)[:2]).cuda()
    with pytest.raises(DadeError):
        ix.search(Q, 10, 0, 16, 0.005)        # nprobe < 1
    with pytest.raises(DadeError):
        ix.search(Q, 10, 4, 24, 0.005)        # Δd not a multiple of 16
    with pytest.raises(DadeError):
        ix.search(Q, 10, 4, 16, 1.0)          # significance not in [0,1)
    with pytest.raises(DadeError):
        ix.search(Q, 7, 4, 16, 0.005)         # K differs from the calibrated K
    bad = Q.clone(); bad[0, 0] = float("nan")
    with pytest.raises(DadeError):
        ix.calibrate(Xd, bad, 10)


def test_sharded_logical_shards_match_oracle(sift_small):
    # G3: S logical shards on one GPU + the merge kernel == the sharded oracle (alpha=0: == exact)
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    from paper_2404_16322_b200 import Index
    Q = synth.queries(cfg)[:16]
    S, n = 3, X.shape[0]
    gids, gds, parts = [], [], []
    for s in range(S):
        lo, hi = s * n // S, (s + 1) * n // S
        sh = Index(cfg.d)
        sh.set_rotation(oidx["mean"], oidx["R"])
        sh.build_ivf(Xd[lo:hi].contiguous(), cfg.nlist, centroids=torch.from_numpy(oidx["centroids"]).cuda(),
                     id_base=lo)
        i, d = sh.search(torch.from_numpy(Q).cuda(), 10, 6, 16, 0.0)
        gids.append(i); gds.append(d)
        so = O.build_index(X[lo:hi], oidx["centroids"], oidx["mean"], oidx["R"], id_base=lo)
        parts.append(O.search(so, Q, 10, 6, 16, 0.0)[:2])
    mi, md = ix.merge_topk(torch.stack(gids), torch.stack(gds))
    oi, od = O.merge_shards(parts, 10)
    assert tie_adjusted_overlap(mi.cpu().numpy(), md.cpu().numpy(), oi, od) == 1.0
    ei, ed = O.exact_ivf(oidx, X, Q, 10, 6)
    assert np.array_equal(oi, ei)


def test_search_host_matches_device(sift_small):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = synth.queries(cfg)[:30]
    a, b = ix.search(torch.from_numpy(Q).cuda(), 10, 8, 16, 0.005)
    c, d = ix.search_host(Q, 10, 8, 16, 0.005)
    assert np.array_equal(a.cpu().numpy(), c) and np.array_equal(b.cpu().numpy(), d)


@pytest.mark.parametrize("chunks,prep", [(1, 1), (3, 1), (7, 1), (1, 2), (1, 3)])
def test_search_host_pipeline_chunks(sift_small, chunks, prep):
    """The H2D / search / D2H pipeline of dade_search_host (pinned buffers, ragged chunks; search
    chunks or rotation + probe chunks ahead of one scan) returns exactly the device-buffer
    search's results."""
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = synth.queries(cfg, n=1001)
    a, b = ix.search(torch.from_numpy(Q).cuda(), 10, 8, 16, 0.005)
    ix.set_option("host_chunks", chunks)
    ix.set_option("host_prep_chunks", prep)
    Qh = torch.from_numpy(Q).pin_memory()
    ih = torch.empty((1001, 10), dtype=torch.int64).pin_memory()
    dh = torch.empty((1001, 10), dtype=torch.float32).pin_memory()
    ix.search_host(Qh, 10, 8, 16, 0.005, ids=ih, dists=dh)
    ix.set_option("host_chunks", 1)
    ix.set_option("host_prep_chunks", 0)
    assert np.array_equal(a.cpu().numpy(), ih.numpy()) and np.array_equal(b.cpu().numpy(), dh.numpy())


@pytest.mark.parametrize("mode", [1, 2])
def test_scan_query_order_invariance(sift_small, mode):
    """DADE_OPT_SCAN_ORDER = 1 (queries scanned grouped by nearest probed list) returns exactly the
    default order's results and counters: each query's scan depends only on its own stream."""
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = torch.from_numpy(synth.queries(cfg, n=700)).cuda()
    ix.set_option("scan_order", 0)      # as given
    a, b, sa = ix.search(Q, 10, 8, 16, 0.005, stats=True)
    ix.set_option("scan_order", mode)   # 1: grouped by nearest list, 2: longest stream first
    c, d, sc = ix.search(Q, 10, 8, 16, 0.005, stats=True)
    ix.set_option("scan_order", 2)
    assert torch.equal(a, c) and torch.equal(b, d)
    assert sa["tested"] == sc["tested"] and sa["dims_scanned"] == sc["dims_scanned"]


@pytest.mark.parametrize("tail", [1, 300])
def test_scan_tail_split_invariance(sift_small, tail):
    """DADE_OPT_SCAN_TAIL (the last queries scanned by a concurrent 4-warps-per-query launch) returns
    exactly the single launch's results and counters."""
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = torch.from_numpy(synth.queries(cfg, n=700)).cuda()
    ix.set_option("scan_order", 0)      # the tail split applies to the as-given order
    a, b, sa = ix.search(Q, 10, 8, 16, 0.005, stats=True)
    ix.set_option("scan_tail", tail)
    c, d, sc = ix.search(Q, 10, 8, 16, 0.005, stats=True)
    ix.set_option("scan_tail", 0)
    ix.set_option("scan_order", 2)
    assert torch.equal(a, c) and torch.equal(b, d)
    assert sa["tested"] == sc["tested"] and sa["dims_scanned"] == sc["dims_scanned"]


def test_save_load_roundtrip(sift_small, tmp_path):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    from paper_2404_16322_b200 import Index
    p = str(tmp_path / "idx.bin")
    ix.save(p)
    iy = Index(cfg.d)
    iy.load(p)
    Q = torch.from_numpy(synth.queries(cfg)[:10]).cuda()
    a, b = ix.search(Q, 10, 8, 16, 0.005)
    c, d = iy.search(Q, 10, 8, 16, 0.005)
    assert torch.equal(a, c) and torch.equal(b, d)


def test_nonfinite_query_reported(sift_small):
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    from paper_2404_16322_b200 import DadeError
    Q = torch.from_numpy(synth.queries(cfg)[:4]).cuda()
    Q[1, 3] = float("inf")
    with pytest.raises(DadeError):
        ix.search(Q, 10, 4, 16, 0.005, stats=True)   # a synchronising call reports it
    ix.search(Q[:1].contiguous(), 10, 4, 16, 0.005, stats=True)  # the latch is cleared


def test_prepare_then_search_prepared_equals_search(sift_small):
    # the split used by the query-partitioned multi-GPU path: a4 + a5 (prepare) and a6-a8
    # (search_prepared) give bit-identical results to one dade_search, for every method; queries
    # prepared in blocks (as ranks would) and concatenated give the same too
    cfg, (torch, ix, oidx, X, Xd) = sift_small
    Q = torch.from_numpy(synth.queries(cfg)[:30]).cuda()
    qrot, probes = ix.prepare(Q, 8)
    a, b = ix.search(Q, 10, 8, 16, 0.005)
    c, d = ix.search_prepared(qrot, probes, 10, 16, "bsa_p", 0.005)
    assert torch.equal(a, c) and torch.equal(b, d)
    parts = [ix.prepare(Q[i:i + 7].contiguous(), 8) for i in range(0, 30, 7)]
    qr2 = torch.cat([p[0] for p in parts]); pr2 = torch.cat([p[1] for p in parts])
    assert torch.equal(qr2, qrot) and torch.equal(pr2, probes)
    e, f = ix.search_method(Q, 10, 8, 16, "bsa_res", 8.0)
    g, h = ix.search_prepared(qrot, probes, 10, 16, "bsa_res", 8.0)
    assert torch.equal(e, g) and torch.equal(f, h)
    z = ix.prepare(Q[:0].contiguous(), 8)                      # an empty block (more ranks than queries)
    assert z[0].shape == (0, cfg.d) and z[1].shape == (0, 8)


@pytest.mark.parametrize("D,K,dd", [(16, 1, 16), (32, 7, 16), (128, 256, 32)])
def test_extreme_shapes(D, K, dd):
    # D = 16 (one block, a single step: never a classifier), K = 1, and K = 256 (DADE_MAX_K: eight
    # register keys per lane); exact search (alpha = 0) over every list equals brute force and
    # the calibrated search loses at most 1% recall against exact IVF
    cfg = synth.config("c1", n=4000, d=D, nlist=16, nq=16, n_cal=20, k=K, delta_d=dd)
    torch, ix, oidx, X, Xd = _setup(cfg, kmeans_iters=2, cal=False)
    Q = synth.queries(cfg)
    gi, gd = ix.search(torch.from_numpy(Q).cuda(), K, cfg.nlist, dd, 0.0)
    bi, bd = O.brute_force_knn(X, Q, K)
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd) == 1.0
    assert rel_err(gd.cpu().numpy(), bd) <= 1e-5
    from paper_2404_16322_b200 import DadeError
    with pytest.raises(DadeError):
        ix.search(torch.from_numpy(Q).cuda(), 257, 4, dd, 0.0)   # K > DADE_MAX_K


@pytest.mark.parametrize("dd", [16, 32, 64])
def test_list_major_stage1_option(dd):
    # DADE_OPT_SCAN_P1 = 1 (p1.cu): stage 1 from the list-major precompute (the first step's
    # block sums of every (query, candidate), each probed list read once) — the same oracle
    # parity as the row-reading stage 1, on a SIFT-shaped index with lists shared by many queries;
    # staging units 1, 2 and 4 blocks (delta_d 16 / 32 / 64)
    cfg = synth.config("c2", n=20000, nlist=32, nq=120, n_cal=60)
    torch, ix, oidx, X, Xd = _setup(cfg)
    Q = synth.queries(cfg)
    ix.set_option("scan_p1", 1)
    gi, gd, st, oi, od, ost = _compare(torch, ix, oidx, Q, cfg.k, 6, dd, 0.005)
    ix.set_option("scan_p1", 0)
    gi0, gd0, st0 = ix.search(torch.from_numpy(Q).cuda(), cfg.k, 6, dd, 0.005, stats=True)
    assert tie_adjusted_overlap(gi, gd, gi0.cpu().numpy(), gd0.cpu().numpy()) >= 0.999
    assert st["tested"] == st0["tested"]
