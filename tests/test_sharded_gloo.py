"""World-size-2 gloo tests of the multi-rank path on CPU (no GPU): shard ranges, the PCA
all-reduce, and the all-gather + merge of local top-K lists. The per-shard engine here is the
oracle (test infrastructure); in production it is the C-ABI library on each GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from datagen import synth
from oracle import dade_oracle as O
from paper_2404_16322_b200 import sharded


class OracleEngine:
    """Per-shard engine over the oracle (CPU tensors), same interface as dade.Index."""

    def __init__(self, X, id_base, centroids=None, mean=None, R=None):
        self.X, self.id_base = X, id_base
        self.idx = None if centroids is None else O.build_index(X, centroids, mean, R, id_base=id_base)

    def pca_mean_partial(self, X, id_base, n_total, sample_size=0):
        ns = min(n_total, 1_000_000) if sample_size <= 0 else min(n_total, sample_size)
        g = O.strided_ids(n_total, ns)
        mine = g[(g >= id_base) & (g < id_base + len(self.X))] - id_base
        return self.X[mine].astype(np.float64).sum(axis=0), len(mine)

    def pca_cov_partial(self, X, id_base, n_total, mean, sample_size=0):
        ns = min(n_total, 1_000_000) if sample_size <= 0 else min(n_total, sample_size)
        g = O.strided_ids(n_total, ns)
        Y = self.X[g[(g >= id_base) & (g < id_base + len(self.X))] - id_base].astype(np.float64) - mean
        return Y.T @ Y

    def kmeans_partial(self, X, id_base, n_total, nlist, centroids=None):
        nkm = min(n_total, 64 * nlist)
        g = O.strided_ids(n_total, nkm)
        own = (g >= id_base) & (g < id_base + len(self.X))
        ks, rows = np.nonzero(own)[0], g[own] - id_base
        D = self.X.shape[1]
        sums, counts = np.zeros((nlist, D)), np.zeros(nlist, np.int64)
        if centroids is None:
            sel = ks < nlist
            sums[ks[sel]] = self.X[rows[sel]].astype(np.float64)
            counts[ks[sel]] = 1
            return sums, counts
        a = O.assign(self.X[rows], centroids)
        np.add.at(sums, a, self.X[rows].astype(np.float64))
        counts += np.bincount(a, minlength=nlist)
        return sums, counts

    def set_rotation_from_cov(self, mean, cov, cnt):
        lam, V = np.linalg.eigh(cov / cnt)
        self.rot = (mean, lam[::-1])

    def search(self, Q, K, nprobe, dd, alpha):
        i, d, _ = O.search(self.idx, Q.numpy(), K, nprobe, dd, alpha)
        return torch.from_numpy(i), torch.from_numpy(d)

    # split search: "q~" here is the raw query (the oracle rotates inside search); the probes the
    # ranks computed must be the ones this shard's own search would use
    def prepare(self, Q, nprobe):
        Qn = Q.numpy()
        pr = np.stack([O.probe(q, self.idx["centroids"], nprobe) for q in Qn]) if len(Qn) else \
            np.zeros((0, nprobe), np.int64)
        return torch.from_numpy(Qn.copy()), torch.from_numpy(pr.astype(np.int32))

    def search_prepared(self, qrot, probes, K, dd, method, param):
        Qn = qrot.numpy()
        for q in range(len(Qn)):
            assert probes[q].tolist() == O.probe(Qn[q], self.idx["centroids"], probes.shape[1]).tolist()
        i, d, _ = O.search(self.idx, Qn, K, probes.shape[1], dd, param if method == "bsa_p" else 0.0)
        return torch.from_numpy(i), torch.from_numpy(d)

    # calibration pieces (dade_calib_knn / _negatives / dade_pair_features / dade_fit_calibration)
    def calib_knn(self, X, Qc, K):
        return O.brute_force_knn(self.X, Qc, K, id_base=self.id_base)

    def calib_negatives(self, Qc, K, knn_ids, n_neg, nprobe_neg, seed):
        nq = Qc.shape[0]
        keys = np.zeros((nq, n_neg), np.uint64); ids = np.zeros((nq, n_neg), np.int64)
        cnt = np.zeros(nq, np.int32)
        off, row_id, cent = self.idx["off"], self.idx["row_id"], self.idx["centroids"]
        for q in range(nq):
            pr = O.probe(Qc[q], cent, nprobe_neg)
            cand = np.concatenate([row_id[off[l]:off[l + 1]] for l in pr])
            cand = np.setdiff1d(cand, knn_ids[q])
            h = O.neg_hash(seed, q, cand)
            o = np.lexsort((cand, h))[:n_neg]
            keys[q, :len(o)], ids[q, :len(o)], cnt[q] = h[o], cand[o], len(o)
        return keys, ids, cnt

    def pair_features(self, Qc, pq, pid):
        qr = O.rotate(Qc, self.idx["mean"], self.idx["R"])
        D = qr.shape[1]
        F = np.zeros((len(pq), D // 16))
        for i, (q, g) in enumerate(zip(pq, pid)):
            if self.id_base <= g < self.id_base + len(self.X):
                diff2 = (self.idx["Xr"][g - self.id_base] - qr[q]) ** 2
                F[i] = np.cumsum(diff2)[15::16]
        return F

    def fit_calibration(self, K, F, tau, y):
        self.fit_args = (K, F, tau, y)

    def merge_topk(self, g_ids, g_d):
        i, d = O.merge_shards([(g_ids[s].numpy(), g_d[s].numpy()) for s in range(g_ids.shape[0])],
                              g_ids.shape[2])
        return torch.from_numpy(i), torch.from_numpy(d)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config("c2", n=6000, nlist=24, nq=12)
        X = synth.base(cfg)
        Q = synth.queries(cfg)
        lo, hi = sharded.shard_range(cfg.n, rank, world)
        # a0 over the sharded base
        eng = OracleEngine(X[lo:hi], lo)
        mean, cnt = sharded.fit_rotation_sharded(eng, None, lo, cfg.n, sample_size=3000)
        om, _, olam = O.fit_rotation(X, sample_size=3000)
        assert cnt == 3000 and np.allclose(mean, om, rtol=1e-12)
        assert np.allclose(eng.rot[1], olam, rtol=1e-9)
        # k-means over the sharded base (fp64 sums all-reduced) == the oracle's k-means on the whole
        # base (up to the summation order of the fp64 sums)
        cent_s = sharded.kmeans_sharded(eng, None, lo, cfg.n, cfg.nlist, iters=3)
        cent_o = O.kmeans(X, cfg.nlist, iters=3)
        assert np.allclose(cent_s, cent_o, rtol=1e-6, atol=1e-6), "sharded k-means differs"
        # search on the shard + all-gather + merge == unsharded exact IVF (alpha = 0)
        mean, R, lam = O.fit_rotation(X)
        cent = O.kmeans(X, cfg.nlist, iters=2)
        eng = OracleEngine(X[lo:hi], lo, cent, mean, R)
        ids, d = sharded.ShardedSearch(eng).search(torch.from_numpy(Q), 10, 5, 16, 0.0)
        full = O.build_index(X, cent, mean, R)
        ei, ed = O.exact_ivf(full, X, Q, 10, 5)
        assert np.array_equal(ids.numpy(), ei), "sharded merge differs from unsharded exact IVF"
        # query-partitioned split search (each rank prepares a block of queries; 12 queries over
        # 2 ranks, and 11 so that the last block is ragged) == the same exact IVF
        for nq in (12, 11):
            ids, d = sharded.QueryPartitionedSearch(eng).search(torch.from_numpy(Q[:nq]), 10, 5, 16, "bsa_p", 0.0)
            assert np.array_equal(ids.numpy(), ei[:nq]), "query-partitioned search differs"
        # sharded calibration: merged K-NN, merged negatives and summed pair features give the
        # single-index calibration pairs (R14-R16) in the same order with the same features
        Qc = synth.cal_queries(cfg)[:8]
        sharded.calibrate_sharded(eng, None, Qc, 10, n_neg=20, nprobe_neg=4, seed=5)
        K_, F, tau, y = eng.fit_args
        oq, oid, olab, otau = O.calibration_pairs(X, full, Qc, 10, 20, 4, 5)
        assert K_ == 10 and np.array_equal(y, olab) and np.allclose(tau, otau, rtol=1e-12)
        qr = O.rotate(Qc, mean, R)
        Fo = np.stack([np.cumsum((full["Xr"][i] - qr[q]) ** 2)[15::16] for q, i in zip(oq, oid)])
        assert np.allclose(F, Fo, rtol=1e-12), "sharded pair features differ"
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_ranges_partition():
    for n in (1, 7, 100, 1_000_003):
        for w in (1, 2, 3, 8):
            rs = [sharded.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
