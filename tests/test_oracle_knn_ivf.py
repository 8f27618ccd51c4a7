"""Pins for the oracle's distance / brute-force / IVF functions (no GPU).

Each test checks the oracle against something other than itself: the SPEC worked
example, pure-Python double loops on tiny inputs, exact integer arithmetic, or a
constructed configuration whose answer is known in closed form."""
import json
import os

import numpy as np
import pytest

from oracle import dade_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _py_sqdist(a, b):
    return sum((float(x) - float(y)) ** 2 for x, y in zip(a, b))


def test_spec_worked_example():
    g = json.load(open(os.path.join(GOLD, "spec_knn_example.json")))
    ids, d = O.brute_force_knn(np.array(g["base"], np.float32), np.array([g["query"]], np.float32), g["K"])
    assert ids[0].tolist() == g["ids"]
    np.testing.assert_allclose(d[0], g["dists"], rtol=1e-6)  # 0.9 is not exact in fp32


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_brute_force_vs_double_loop(seed):
    rng = np.random.default_rng(seed)
    n, D, K = int(rng.integers(20, 200)), int(rng.integers(1, 16)), 7
    X = rng.standard_normal((n, D)).astype(np.float32)
    Q = rng.standard_normal((5, D)).astype(np.float32)
    ids, d = O.brute_force_knn(X, Q, K)
    for qi in range(5):
        ref = sorted((_py_sqdist(X[i], Q[qi]), i) for i in range(n))[:K]
        assert ids[qi].tolist() == [i for _, i in ref]
        np.testing.assert_allclose(d[qi], [x for x, _ in ref], rtol=1e-12)


def test_integer_data_is_exact_and_ties_to_lower_id():
    # integer-valued data: every distance is an exact integer; equal distances tie to lower id
    X = np.array([[3, 0], [0, 3], [1, 1], [5, 5], [-3, 0]], np.float32)
    ids, d = O.brute_force_knn(X, np.zeros((1, 2), np.float32), 4)
    assert d[0].tolist() == [2.0, 9.0, 9.0, 9.0]
    assert ids[0].tolist() == [2, 0, 1, 4]
    # a query equal to a base point returns it at distance 0
    ids, d = O.brute_force_knn(X, X[3:4], 1)
    assert ids[0, 0] == 3 and d[0, 0] == 0.0


def test_sqdist_seq_matches_python_fsum_order():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((30, 9)).astype(np.float32)
    v = rng.standard_normal(9).astype(np.float32)
    got = O.sqdist_seq(X, v)
    for i in range(30):
        acc = 0.0
        for j in range(9):  # sequential Python-float (IEEE double) loop = the stated definition
            t = float(X[i, j]) - float(v[j])
            acc += t * t
        assert got[i] == acc  # bit-identical: same operations in the same order


@pytest.mark.parametrize("seed", [0, 1])
def test_assign_vs_brute_force_and_tie(seed):
    rng = np.random.default_rng(seed)
    X = rng.integers(-3, 4, size=(60, 5)).astype(np.float32)
    C = rng.integers(-3, 4, size=(7, 5)).astype(np.float32)
    C[5] = C[2]  # duplicated centroid: the lower id (2) must win every tie
    a = O.assign(X, C)
    for i in range(60):
        dd = [_py_sqdist(X[i], C[c]) for c in range(7)]
        assert a[i] == min(range(7), key=lambda c: (dd[c], c))
        assert a[i] != 5


def test_build_ivf_partition_and_order():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((300, 4)).astype(np.float32)
    C = X[:9].copy()
    a, off, row_id = O.build_ivf(X, C, id_base=1000)
    assert off[0] == 0 and off[-1] == 300 and np.all(np.diff(off) >= 0)
    assert sorted(row_id.tolist()) == list(range(1000, 1300))  # every id exactly once
    for l in range(9):
        members = row_id[off[l]:off[l + 1]]
        assert np.all(np.diff(members) > 0)  # ascending ids inside a list
        assert np.all(a[members - 1000] == l)
    a1, off1, row1 = O.build_ivf(X, C[:1])  # nlist = 1: one list holding everything
    assert off1.tolist() == [0, 300] and row1.tolist() == list(range(300))


def test_probe_order():
    rng = np.random.default_rng(4)
    C = rng.integers(0, 3, size=(40, 3)).astype(np.float32)  # many exact ties
    q = np.array([1, 1, 1], np.float32)
    p = O.probe(q, C, 12)
    ref = sorted(range(40), key=lambda c: (_py_sqdist(C[c], q), c))[:12]
    assert p.tolist() == ref


def test_kmeans_recovers_separated_clusters():
    # C tight clusters, rows interleaved so the strided sample's first C rows hit every cluster
    rng = np.random.default_rng(7)
    C, D, per = 6, 3, 20
    centres = 100.0 * rng.standard_normal((C, D))
    X = np.empty((C * per, D), np.float32)
    for i in range(C * per):
        X[i] = centres[i % C] + rng.standard_normal(D)
    cent = O.kmeans(X, C, iters=5)
    for c in range(C):
        members = X[c::C].astype(np.float64)
        ref = np.array([sum(members[:, j].tolist()) / per for j in range(D)])
        np.testing.assert_allclose(cent[c], ref, rtol=1e-6, atol=1e-4)


def test_kmeans_objective_non_increasing():
    rng = np.random.default_rng(8)
    X = rng.standard_normal((400, 6)).astype(np.float32)
    objs = []
    for it in range(0, 6):
        cent = O.kmeans(X, 10, iters=it)
        a = O.assign(X, cent)
        objs.append(sum(_py_sqdist(X[i], cent[a[i]]) for i in range(400)))
    assert all(objs[i + 1] <= objs[i] * (1 + 1e-6) for i in range(len(objs) - 1))


def test_strided_ids():
    assert O.strided_ids(10, 4).tolist() == [0, 2, 5, 7]
    assert O.strided_ids(5, 5).tolist() == [0, 1, 2, 3, 4]


def test_recall_at_k_spec_example():
    # T={1,2,3,4}, G={1,2,5,6} -> 0.5
    assert O.recall_at_k(np.array([[1, 2, 3, 4]]), np.array([[1, 2, 5, 6]]), 4) == 0.5
