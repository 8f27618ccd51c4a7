"""Pins for the sharded oracle with the cross-shard τ exchange (R32): S = 1 is the
plain search; α = 0 is exact IVF for any S; a hand-worked two-shard case where the exchanged
K-th distance prunes candidates the shard's own τ would keep; and the pruning it buys back: the
2-shard scan rate within 4% of the single index (unseeded: +7.8%)."""
import numpy as np
import pytest

from datagen import synth
from oracle import dade_oracle as O
from tests.test_oracle_search_pins import CAL, D


def test_one_shard_seeded_is_plain_search():
    cfg = synth.config("c2", n=6000, nlist=24, nq=20, n_cal=60)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    cent = O.kmeans(X, cfg.nlist, iters=3)
    idx = O.build_index(X, cent, mean, R)
    idx["cal"] = O.calibrate(X, idx, synth.cal_queries(cfg), cfg.k, n_neg=50, nprobe_neg=4, seed=0)
    Q = synth.queries(cfg)
    a, ad, ast = O.search(idx, Q, cfg.k, 5, 16, 0.005)
    b, bd, bst = O.search_sharded([idx], Q, cfg.k, 5, 16, 0.005)
    assert np.array_equal(a, b) and np.array_equal(ad, bd)
    for k in ("tested", "dims_scanned", "survivors"):
        assert ast[k] == bst[0][k]
    assert np.array_equal(ast["pruned_at_step"], bst[0]["pruned_at_step"])


def test_hand_worked_two_shard_seed():
    # D = 48, K = 1, m1 = (2, 1), beta' = (1, 3) (the hand case of test_oracle_search_pins); S = 2 so
    # the per-shard c0 = ceil(4K/S) = 2: shard epochs [0,2), [2,4), [4,8); exchanges after epochs 0, 1.
    # phase 0 (tau = inf): shard 0 ids 0 (9), 1 (0.25); shard 1 ids 4 (9), 5 (16) -> merged K-th 0.25
    # phase 1, tau = min(own, 0.25) = 0.25 on both shards:
    #   id 2 = (0, 0, .25) d16 2*0 + 1 = 1 > .25 pruned (a false prune: dist 0.0625); id 3 = (3,0,0) pruned
    #   id 6 = (.5, 0, 0) d16 1.5 > .25 pruned; id 7 = (0, 0, 1) d16 1 > .25 pruned
    # exchange 2: merged K-th still 0.25; phase 2 (shard 1 ids 8 = (0,0,0), 9 = (4,0,0)): both d16 > .25
    rows = [(3, 0, 0), (0, 0, 0.5), (0, 0, 0.25), (3, 0, 0), (3, 0, 0), (4, 0, 0), (0.5, 0, 0), (0, 0, 1),
            (0, 0, 0), (4, 0, 0)]
    X = np.zeros((10, D), np.float32)
    for i, (a, b, c) in enumerate(rows):
        X[i, 0], X[i, 16], X[i, 32] = a, b, c
    cent = np.zeros((1, D), np.float32)
    sh = [O.build_index(X[:4], cent, np.zeros(D), np.eye(D), CAL, id_base=0),
          O.build_index(X[4:], cent, np.zeros(D), np.eye(D), CAL, id_base=4)]
    Q = np.zeros((1, D), np.float32)
    ids, d, st = O.search_sharded(sh, Q, 1, 1, 16, 0.1, seed=True)
    assert ids.tolist() == [[1]] and d.tolist() == [[0.25]]
    assert st[0]["pruned_at_step"].tolist() == [0, 2, 0] and st[0]["survivors"] == 2
    assert st[1]["pruned_at_step"].tolist() == [0, 4, 0] and st[1]["survivors"] == 2 and st[1]["tested"] == 6
    # unseeded (c0 = 4K = 4 per shard, own tau only): shard 0's epoch 0 is all four ids -> id 2 (0.0625)
    # survives; shard 1: ids 4-7 survive (tau = inf), then 8, 9 are pruned against its own 0.25 (id 6)
    ids, d, st = O.search_sharded(sh, Q, 1, 1, 16, 0.1, seed=False)
    assert ids.tolist() == [[2]] and d.tolist() == [[0.0625]]
    assert st[1]["pruned_at_step"].tolist() == [0, 2, 0] and st[1]["survivors"] == 4


@pytest.fixture(scope="module")
def sift_shards():
    cfg = synth.config("c2", n=40000, nlist=96, nq=40, n_cal=120)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    cent = O.kmeans(X, cfg.nlist, iters=3)
    full = O.build_index(X, cent, mean, R)
    full["cal"] = O.calibrate(X, full, synth.cal_queries(cfg), cfg.k, n_neg=50, nprobe_neg=8, seed=0)
    return cfg, X, cent, mean, R, full


def _shards(X, cent, mean, R, cal, S):
    n = X.shape[0]
    return [O.build_index(X[s * n // S:(s + 1) * n // S], cent, mean, R, cal, id_base=s * n // S) for s in range(S)]


def test_alpha0_any_S_is_exact(sift_shards):
    cfg, X, cent, mean, R, full = sift_shards
    Q = synth.queries(cfg)[:10]
    ei, ed = O.exact_ivf(full, X, Q, cfg.k, 6)
    for S in (2, 3):
        ids, d, _ = O.search_sharded(_shards(X, cent, mean, R, full["cal"], S), Q, cfg.k, 6, 16, 0.0)
        assert np.array_equal(ids, ei)


def test_two_shard_scan_rate_close_to_one(sift_shards):
    cfg, X, cent, mean, R, full = sift_shards
    Q = synth.queries(cfg)
    _, _, s1 = O.search(full, Q, cfg.k, 8, 16, 0.005)
    rate1 = s1["dims_scanned"] / s1["tested"]
    sh = _shards(X, cent, mean, R, full["cal"], 2)
    i2, _, st = O.search_sharded(sh, Q, cfg.k, 8, 16, 0.005, seed=True)
    rate2 = sum(x["dims_scanned"] for x in st) / sum(x["tested"] for x in st)
    _, _, su = O.search_sharded(sh, Q, cfg.k, 8, 16, 0.005, seed=False)
    rate_u = sum(x["dims_scanned"] for x in su) / sum(x["tested"] for x in su)
    # measured (R32): unseeded +7.8%, the default schedule (2 exchanges) +3.3% at S = 2
    assert rate2 <= rate1 * 1.04, (rate2, rate1, rate_u)
    assert rate_u > rate2 * 1.03
    ei, _ = O.exact_ivf(full, X, Q, cfg.k, 8)
    assert O.recall_at_k(i2, ei, cfg.k) >= 0.99
