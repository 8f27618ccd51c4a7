"""The library-owned NCCL path (dade_set_comm) on one GPU: a group of one rank runs the collective
schedules — the sharded build (fp64 all-reduces, k-means, merged calibration) and the collective
search (query-partitioned prepare, all-gathers, merge kernel) — and must return exactly what the
single-GPU calls return. (More ranks need more GPUs; the process-group schedule with 2 ranks is
covered on CPU by tests/test_sharded_gloo.py with the same host combination steps.)"""
import numpy as np
import pytest

from datagen import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    import torch
    assert torch.cuda.is_available()
    from paper_2404_16322_b200 import Index, build
    build.build()
    cfg = synth.config("c2", n=40000, nlist=64, nq=300, n_cal=64)
    X = torch.from_numpy(synth.base(cfg)).cuda()
    Qc = torch.from_numpy(synth.cal_queries(cfg)).cuda()
    a = Index(cfg.d)
    a.fit_rotation(X)
    a.build_ivf(X, cfg.nlist, kmeans_iters=4)
    a.calibrate(X, Qc, cfg.k, n_neg=30, nprobe_neg=8, seed=3)
    b = Index(cfg.d)
    b.set_comm(None, 1, 0)
    b.fit_rotation_dist(X, 0, cfg.n)
    b.build_ivf_dist(X, 0, cfg.n, cfg.nlist, kmeans_iters=4)
    b.calibrate_dist(X, Qc, cfg.k, n_neg=30, nprobe_neg=8, seed=3)
    return torch, cfg, a, b


def test_sharded_build_equals_single_gpu_build(pair):
    torch, cfg, a, b = pair
    for x, y in zip(a.get_rotation(), b.get_rotation()):
        assert np.array_equal(x, y)
    for x, y in zip(a.get_ivf(), b.get_ivf()):
        assert np.array_equal(x, y)
    ca, cb = a.get_calibration(), b.get_calibration()
    assert np.array_equal(ca["m1"], cb["m1"]) and np.array_equal(ca["v"], cb["v"])


def test_collective_search_equals_search(pair):
    torch, cfg, a, b = pair
    Q = torch.from_numpy(synth.queries(cfg)).cuda()
    for nprobe, alpha in ((4, 0.005), (8, 0.0), (64, 0.005)):
        i1, d1, s1 = a.search(Q, cfg.k, nprobe, 16, alpha, stats=True)
        i2, d2, s2 = b.search(Q, cfg.k, nprobe, 16, alpha, stats=True)
        assert torch.equal(i1, i2) and torch.equal(d1, d2)
        assert s1["dims_scanned"] == s2["dims_scanned"] and s1["pruned_at_step"] == s2["pruned_at_step"]
    i1, d1 = a.search_method(Q, cfg.k, 8, 16, "adsampling", 2.1)
    i2, d2 = b.search_method(Q, cfg.k, 8, 16, "adsampling", 2.1)
    assert torch.equal(i1, i2) and torch.equal(d1, d2)
    Qh = synth.queries(cfg)
    h1 = a.search_host(Qh, cfg.k, 8, 16, 0.005)
    h2 = b.search_host(Qh, cfg.k, 8, 16, 0.005)
    assert np.array_equal(h1[0], h2[0]) and np.array_equal(h1[1], h2[1])
    z = b.search(Q[:0].contiguous(), cfg.k, 8, 16, 0.005)       # no queries: nothing to gather
    assert z[0].shape == (0, cfg.k)


@pytest.mark.parametrize("E", [0, 1, 3])
def test_collective_phases_equal_search(pair, E):
    # R32's phased schedule (epochs 0..E-1 one launch each, queue carried over, exchanged K-th as a
    # tau bound) in a group of one: every phase boundary must be invisible — results and counters
    # equal the single-launch search, for one warp per query and for several (G > 1 epoch merges)
    torch, cfg, a, b = pair
    Q = torch.from_numpy(synth.queries(cfg)).cuda()
    b.set_option("shard_exchanges", E)
    for G in (1, 4):
        a.set_option("scan_warps", G); b.set_option("scan_warps", G)
        i1, d1, s1 = a.search(Q, cfg.k, 8, 16, 0.005, stats=True)
        i2, d2, s2 = b.search(Q, cfg.k, 8, 16, 0.005, stats=True)
        assert torch.equal(i1, i2) and torch.equal(d1, d2)
        assert s1["tested"] == s2["tested"] and s1["dims_scanned"] == s2["dims_scanned"]
        assert s1["pruned_at_step"] == s2["pruned_at_step"]
        i1, d1 = a.search(Q, 100, 8, 32, 0.0)                 # K = 100: four keys per lane
        i2, d2 = b.search(Q, 100, 8, 32, 0.0)
        assert torch.equal(i1, i2) and torch.equal(d1, d2)
    a.set_option("scan_warps", 0); b.set_option("scan_warps", 0)
    b.set_option("shard_exchanges", 2)


def test_comm_errors(pair):
    torch, cfg, a, b = pair
    from paper_2404_16322_b200 import DadeError
    with pytest.raises(DadeError):
        a.fit_rotation_dist(torch.zeros((16, cfg.d), device="cuda"), 0, 16)   # no communicator: STATE
    with pytest.raises(DadeError):
        a.set_comm(None, 2, 0)                                              # 2 ranks need the shared id
    with pytest.raises(DadeError):
        a.set_comm(None, 1, 1)                                              # rank out of range
