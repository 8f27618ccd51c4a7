"""GPU parity at the shapes of every BASELINE.json config (configs[0..4]): the same generators,
D, K, delta_d and value distributions, at base sizes the oracle finishes in seconds that still
span several scan tiles per list and ragged tails. The north_star tolerances apply: returned
distances within 1e-5 relative of the exact distance of that id, tie-adjusted ID overlap with
the oracle's DADE result >= 0.999, and identical candidate counts (same probes, same lists).
configs[0] (c1) at its full stated size lives in test_gpu_search.py."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.test_gpu_search import _compare, _setup

pytestmark = pytest.mark.gpu


def _run(cfg, nprobes, nprobe_neg, alphas=(0.005,)):
    torch, ix, oidx, X, Xd = _setup(cfg, nprobe_neg=nprobe_neg)
    Q = synth.queries(cfg)
    for npb in nprobes:
        for a in alphas:
            _compare(torch, ix, oidx, Q, cfg.k, npb, cfg.delta_d, a)
    # alpha = 0: the search is exact IVF at the same nprobe (north_star: pruning disabled
    # reduces to the textbook routine)
    gi, gd = ix.search(torch.from_numpy(Q).cuda(), cfg.k, nprobes[0], cfg.delta_d, 0.0)
    ei, ed = O.exact_ivf(oidx, X, Q, cfg.k, nprobes[0])
    from tests.helpers import rel_err, tie_adjusted_overlap
    assert tie_adjusted_overlap(gi.cpu().numpy(), gd.cpu().numpy(), ei, ed) == 1.0
    assert rel_err(gd.cpu().numpy(), ed) <= 1e-5
    return torch, ix, oidx, X


def test_c2_shape_integer_data_ties():
    # configs[1] shape: integer-valued [0,255] SIFT-like data produces exact distance ties
    cfg = synth.config("c2", n=40_000, nlist=160, nq=40, n_cal=120)
    _run(cfg, (3, 12), nprobe_neg=6, alphas=(0.005, 0.05))


def test_c3_shape_gist_d960_k100():
    # configs[2] shape: D = 960 (60 blocks, 30 steps of delta_d = 32), K = 100, values in [0,1]
    cfg = synth.config("c3", n=9_000, nlist=24, nq=12, n_cal=30)
    _run(cfg, (4,), nprobe_neg=3)


def test_c4_shape_deep_d96():
    # configs[3] shape: D = 96 (6 steps of 16), unit-norm vectors, K = 10
    cfg = synth.config("c4", n=30_000, nlist=96, nq=40, n_cal=150)
    _run(cfg, (6, 20), nprobe_neg=6)


def test_c5_shape_d256_k100():
    # configs[4] shape: D = 256 (8 steps of 32), K = 100, 4096-component mixture
    cfg = synth.config("c5", n=24_000, nlist=64, nq=12, n_cal=30)
    _run(cfg, (5,), nprobe_neg=4)


def test_c5_shape_logical_shards_alpha():
    # configs[4] runs sharded: S logical shards on one GPU (global centroids, rotation and
    # calibration replicated) + the merge kernel == the sharded oracle, with pruning on
    cfg = synth.config("c5", n=16_000, nlist=48, nq=8, n_cal=20)
    torch, ix, oidx, X, Xd = _setup(cfg, nprobe_neg=4)
    from paper_2404_16322_b200 import Index
    from tests.helpers import tie_adjusted_overlap
    Q = synth.queries(cfg)
    S, n = 4, X.shape[0]
    gids, gds, parts = [], [], []
    for s in range(S):
        lo, hi = s * n // S, (s + 1) * n // S
        sh = Index(cfg.d)
        sh.set_rotation(oidx["mean"], oidx["R"])
        sh.build_ivf(Xd[lo:hi].contiguous(), cfg.nlist, centroids=torch.from_numpy(oidx["centroids"]).cuda(),
                     id_base=lo)
        sh.set_calibration(cfg.k, oidx["cal"]["m1"], oidx["cal"]["v"])
        i, d = sh.search(torch.from_numpy(Q).cuda(), cfg.k, 5, cfg.delta_d, 0.005)
        gids.append(i); gds.append(d)
        so = O.build_index(X[lo:hi], oidx["centroids"], oidx["mean"], oidx["R"], id_base=lo,
                           cal=oidx["cal"])
        parts.append(O.search(so, Q, cfg.k, 5, cfg.delta_d, 0.005)[:2])
    mi, md = ix.merge_topk(torch.stack(gids), torch.stack(gds))
    oi, od = O.merge_shards(parts, cfg.k)
    assert tie_adjusted_overlap(mi.cpu().numpy(), md.cpu().numpy(), oi, od) >= 0.999


_G_CFGS = {"c4": dict(n=20_000, nlist=64, nq=24, n_cal=100), "c5": dict(n=16_000, nlist=40, nq=10, n_cal=30)}


@pytest.fixture(scope="module", params=["c4", "c5"])
def g_setup(request):
    cfg = synth.config(request.param, **_G_CFGS[request.param])
    return cfg, _setup(cfg, nprobe_neg=6)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_warps_per_query_do_not_change_results(g_setup, G):
    # the scan deals a query's tiles to G warps with tau frozen per epoch (R13) and merges the
    # warps' top-K lists exactly at each epoch end: decisions and results must not depend on G
    # (K = 10: one key per lane; K = 100: four keys per lane)
    cfg, (torch, ix, oidx, X, Xd) = g_setup
    Q = torch.from_numpy(synth.queries(cfg)).cuda()
    ix.set_option("scan_warps", 1)
    ri, rd, rs = ix.search(Q, cfg.k, 10, cfg.delta_d, 0.005, stats=True)
    ix.set_option("scan_warps", G)
    gi, gd, gs = ix.search(Q, cfg.k, 10, cfg.delta_d, 0.005, stats=True)
    ix.set_option("scan_warps", 0)
    assert torch.equal(ri, gi) and torch.equal(rd, gd)
    assert rs["tested"] == gs["tested"] and rs["dims_scanned"] == gs["dims_scanned"]
    assert rs["pruned_at_step"] == gs["pruned_at_step"]
    _compare(torch, ix, oidx, synth.queries(cfg), cfg.k, 10, cfg.delta_d, 0.005)
