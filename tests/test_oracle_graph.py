"""Pins for the oracle's NEXT-4 graph refinement (HNSW base layer with the DCO, R33-R35):
HNSW's neighbour-selection heuristic on a hand example, the exact candidate pools and entry point,
exhaustive search (ef = n) ≡ brute force, and a hand-worked search whose τ is frozen per expansion."""
import numpy as np

from datagen import synth
from oracle import dade_oracle as O
from tests.test_oracle_search_pins import CAL, D


def test_neighbor_heuristic_hand_example():
    # points on a line (dim 0): node 0 at 0; 1 at 1; 2 at -1; 3 at 2; 4 at 3
    X = np.zeros((5, 16), np.float32)
    X[:, 0] = [0, 1, -1, 2, 3]
    # node 0's pool by distance: 1 (1), 2 (1), 3 (4), 4 (9)
    pool = np.array([[1, 2, 3, 4]]); pool_d = np.array([[1.0, 1.0, 4.0, 9.0]])
    # keep 1; 2: d(2,0) = 1 < d(2,1) = 4 -> keep; 3: d(3,0) = 4 < d(3,1) = 1? no -> drop; 4 likewise
    assert O.graph_neighbors(X, pool, pool_d, M0=2).tolist() == [[1, 2]]
    # M0 = 3: the nearest dropped candidate (3) fills the list
    assert O.graph_neighbors(X, pool, pool_d, M0=3).tolist() == [[1, 2, 3]]
    # M0 = 5 > pool: padded with -1
    assert O.graph_neighbors(X, pool, pool_d, M0=5).tolist() == [[1, 2, 3, 4, -1]]


def test_build_graph_pools_and_entry():
    X = np.zeros((6, 16), np.float32)
    X[:, 0] = [0, 1, 2, 3, 4, 10]                         # mean 3.33 -> entry = node 3
    nbrs, entry = O.build_graph(X, M0=2, P=3)
    assert entry == 3
    # node 5 (at 10): pool 4 (36), 3 (49), 2 (64): keep 4; 3: d(3,5) = 49 < d(3,4) = 1? no -> dropped
    assert nbrs[5].tolist() == [4, 3]
    # node 2 (at 2): pool 1 (1), 3 (1), 0 (4): keep 1; 3: d(3,2) = 1 < d(3,1) = 4 -> keep
    assert nbrs[2].tolist() == [1, 3]


def test_exhaustive_graph_search_is_brute_force():
    cfg = synth.config("c1", n=600, d=32, nq=12)
    X = synth.base(cfg)
    mean, R, lam = O.fit_rotation(X)
    idx = O.build_index(X, X[:1].copy(), mean, R)
    idx["nbrs"], idx["entry"] = O.build_graph(X, M0=16, P=32)
    Q = synth.queries(cfg)
    ids, d, st = O.graph_search(idx, Q, 10, X.shape[0], 16, 0.0)   # ef = n: every reachable node
    bi, bd = O.brute_force_knn(X, Q, 10)
    assert np.array_equal(ids, bi)
    np.testing.assert_allclose(d, bd, rtol=1e-9)


def _hand_graph():
    # q = 0, identity rotation; (a, b, c) at dims (0, 16, 32); m1 = (2, 1), beta' = (1, 3)
    rows = [(2, 0, 0), (1, 0, 0), (0, 2, 0), (0, 0, 0.5), (1, 1, 0), (0, 0, 0)]
    X = np.zeros((6, D), np.float32)
    for i, (a, b, c) in enumerate(rows):
        X[i, 0], X[i, 16], X[i, 32] = a, b, c
    idx = O.build_index(X, np.zeros((1, D), np.float32), np.zeros(D), np.eye(D), CAL)
    idx["nbrs"] = np.array([[1, 2], [3, 4], [5, -1], [-1, -1], [5, -1], [-1, -1]])
    idx["entry"] = 0
    return X, idx


def test_hand_worked_graph_search():
    # ef = 2: W = {(4, 0)}; expand 0 (tau = inf): 1 -> 1, 2 -> 4; (1, 1) enters, (4, 2) does not
    # (W full, not below max (4, 0)). Expand 1 with tau = max W = 4 FROZEN: 3 = (0,0,.5): d16 1, d32
    # 3 <= 4 -> exact 0.25; 4 = (1,1,0): d16 3 <= 4, d32 2 + 3 = 5 > 4 -> pruned at 32 (with tau
    # refreshed to 1 after 3 entered it would have been pruned at 16). Expand 3: no neighbours.
    X, idx = _hand_graph()
    ids, d, st = O.graph_search(idx, np.zeros((1, D), np.float32), 1, 2, 16, 0.1, log=True)
    assert ids.tolist() == [[3]] and d.tolist() == [[0.25]]
    assert st["tested"] == 5 and st["survivors"] == 4 and st["expansions"] == 3
    assert st["pruned_at_step"].tolist() == [0, 0, 1]
    assert st["dims_scanned"] == 4 * 48 + 32
    q_, u_, dims, _ = (np.concatenate(c) for c in zip(*st["candidates"]))
    assert list(zip(u_.tolist(), dims.tolist())) == [(0, 48), (1, 48), (2, 48), (3, 48), (4, 32)]
    ids, d, st = O.graph_search(idx, np.zeros((1, D), np.float32), 2, 2, 16, 0.0)   # no DCO
    assert ids.tolist() == [[3, 1]] and st["pruned_at_step"].sum() == 0
