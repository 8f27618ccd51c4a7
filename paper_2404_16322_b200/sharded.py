"""Multi-GPU plumbing for the DADE path.

The database is sharded by contiguous global-id ranges, one shard per rank (one process per GPU).
Replicated state (μ, R, centroids, calibration) is computed from fp64 partials all-reduced over
the process group; a search runs on every shard and the local top-K lists are combined by an
all-gather followed by the library's merge kernel (`dade_merge_topk`). The collective is NCCL
(`torch.distributed`, backend "nccl") on GPUs; the same code runs over gloo in the CPU tests.

`engine` is the per-shard object: `paper_2404_16322_b200.Index` in production. It must provide
search(Q, K, nprobe, delta_d, alpha) -> (ids, dists), merge_topk(ids[S,nq,K], dists[S,nq,K]),
pca_mean_partial / pca_cov_partial / set_rotation_from_cov.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int):
    """Rows [lo, hi) owned by `rank`: contiguous id ranges, sizes differing by at most 1."""
    return rank * n // world, (rank + 1) * n // world


def _all_gather(t, group=None):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out.view(-1), t.contiguous().view(-1), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), t.contiguous(), group=group)
    return out


def fit_rotation_sharded(engine, X_shard, id_base: int, n_total: int, sample_size: int = 0, group=None):
    """a0 over a sharded base: fp64 sum and count of the owned strided-sample rows, all-reduce,
    mean; fp64 centred cross products, all-reduce; every rank then runs the same eigensolve."""
    import torch
    import torch.distributed as dist
    dev = X_shard.device if X_shard is not None and hasattr(X_shard, "device") else torch.device("cpu")
    s, c = engine.pca_mean_partial(X_shard, id_base, n_total, sample_size)
    t = torch.tensor(np.r_[s, c], dtype=torch.float64, device=dev)
    dist.all_reduce(t, group=group)
    t = t.cpu().numpy()
    cnt = int(round(t[-1]))
    mean = t[:-1] / cnt
    cov = torch.from_numpy(engine.pca_cov_partial(X_shard, id_base, n_total, mean, sample_size)).to(dev)
    dist.all_reduce(cov, group=group)
    engine.set_rotation_from_cov(mean, cov.cpu().numpy(), cnt)
    return mean, cnt


def kmeans_sharded(engine, X_shard, id_base: int, n_total: int, nlist: int, iters: int = 10, group=None):
    """k-means over a sharded base: the global strided sample, init = its first
    nlist rows, `iters` Lloyd steps whose per-cluster fp64 sums and counts are all-reduced across
    ranks; centroid = sum / count rounded to fp32, an empty cluster keeps its centroid. Every rank
    ends with the same centroids (nlist x D fp32, host)."""
    import torch
    import torch.distributed as dist

    def allreduce(a, dtype):
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dtype)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, group=group)
        return t.cpu().numpy()

    sums, counts = engine.kmeans_partial(X_shard, id_base, n_total, nlist, None)
    cent = allreduce(sums, torch.float64).astype(np.float32)
    for _ in range(iters):
        sums, counts = engine.kmeans_partial(X_shard, id_base, n_total, nlist, cent)
        sums = allreduce(sums, torch.float64)
        counts = allreduce(counts, torch.int64)
        nz = counts > 0
        cent = cent.copy()
        cent[nz] = (sums[nz] / counts[nz, None]).astype(np.float32)
    return cent


def _gather_np(a, group=None):
    """All-gather a host numpy array (same shape on every rank) -> [world, ...] numpy."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    return _all_gather(t, group).cpu().numpy()


def merge_knn_lists(ids_g, d_g, K: int):
    """[S, nq, K] per-shard K-NN lists (global ids, fp64 dists) -> the global K-NN by (dist, id)."""
    S, nq, _ = ids_g.shape
    knn_ids, knn_d = np.zeros((nq, K), np.int64), np.zeros((nq, K))
    for q in range(nq):
        ci, cd = ids_g[:, q, :].ravel(), d_g[:, q, :].ravel()
        o = np.lexsort((ci, cd))[:K]
        knn_ids[q], knn_d[q] = ci[o], cd[o]
    return knn_ids, knn_d


def calibration_pairs(knn_ids, knn_d, keys_g, nids_g, cnt_g, n_neg: int):
    """The calibration pairs in dade_calibrate's order: per query its K nearest (Label 0, in (dist,
    id) order) then the n_neg smallest (hash, id) negatives over all shards (Label 1); tau = the
    query's K-th distance. keys_g / nids_g: [S, nq, n_neg], cnt_g: [S, nq]."""
    nq, K = knn_ids.shape
    pq, pid, tau, y = [], [], [], []
    for q in range(nq):
        t = knn_d[q, K - 1]
        pq += [q] * K; pid += knn_ids[q].tolist(); tau += [t] * K; y += [0.0] * K
        kk = np.concatenate([keys_g[s, q, :cnt_g[s, q]] for s in range(keys_g.shape[0])]).astype(np.uint64)
        ii = np.concatenate([nids_g[s, q, :cnt_g[s, q]] for s in range(keys_g.shape[0])])
        o = np.lexsort((ii, kk))[:n_neg]
        pq += [q] * len(o); pid += ii[o].tolist(); tau += [t] * len(o); y += [1.0] * len(o)
    return np.array(pq, np.int32), np.array(pid, np.int64), np.array(tau), np.array(y)


def calibrate_sharded(engine, X_shard, Qc, K: int, n_neg: int = 50, nprobe_neg: int = 0, seed: int = 0,
                      group=None):
    """dade_calibrate over a sharded base: every rank runs each step on its shard
    and the steps are combined exactly as the single-GPU calibration defines them — the K nearest
    neighbours are the shards' lists merged by (fp64 dist, id) (R14), the negatives the n_neg
    smallest (hash, id) over the shards' candidates (R15/R16), the pair features P_d (held by the
    rank owning the row) summed over ranks — so the installed table equals an unsharded
    dade_calibrate on the same base, centroids and rotation."""
    import torch
    import torch.distributed as dist
    ids_l, d_l = engine.calib_knn(X_shard, Qc, K)
    knn_ids, knn_d = merge_knn_lists(_gather_np(ids_l, group), _gather_np(d_l, group), K)
    keys_l, nids_l, cnt_l = engine.calib_negatives(Qc, K, knn_ids, n_neg, nprobe_neg, seed)
    keys_g = _gather_np(keys_l.view(np.int64), group).view(np.uint64)
    pq, pid, tau, y = calibration_pairs(knn_ids, knn_d, keys_g, _gather_np(nids_l, group),
                                        _gather_np(cnt_l, group), n_neg)
    t = torch.from_numpy(engine.pair_features(Qc, pq, pid))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, group=group)
    engine.fit_calibration(K, t.cpu().numpy(), tau, y)


class ShardedSearch:
    """search() on this rank's shard, then all-gather of the local top-K and the merge (a9)."""

    def __init__(self, engine, group=None):
        self.engine, self.group = engine, group

    def search(self, Q, K: int, nprobe: int, delta_d: int, significance: float):
        ids, dists = self.engine.search(Q, K, nprobe, delta_d, significance)[:2]
        g_ids = _all_gather(ids, self.group)
        g_d = _all_gather(dists, self.group)
        return self.engine.merge_topk(g_ids, g_d)


def _gather_rows(t, rows_per_rank: int, nq: int, group=None):
    """All-gather equal-size row blocks (padded to rows_per_rank) and return the first nq rows in
    rank order (rank r prepared queries [r*rows_per_rank, (r+1)*rows_per_rank))."""
    import torch
    pad = rows_per_rank - t.shape[0]
    if pad:
        t = torch.cat([t, torch.zeros((pad,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)])
    g = _all_gather(t, group)
    return g.reshape((-1,) + tuple(t.shape[1:]))[:nq].contiguous()


class QueryPartitionedSearch:
    """Multi-GPU search that also splits the per-query fixed costs: rank r rotates
    and probes only its block of queries (a4 + a5, `engine.prepare`), the blocks are all-gathered
    (q~ and probe lists, ~D*4 + nprobe*4 bytes per query), every rank scans ALL queries on its own
    shard (a6-a8, `engine.search_prepared`), and the local top-K lists are all-gathered and merged
    (a9). μ, R and the centroids are replicated, so any rank's prepared queries are valid on every
    shard and the result equals ShardedSearch's."""

    def __init__(self, engine, group=None):
        self.engine, self.group = engine, group

    def search(self, Q, K: int, nprobe: int, delta_d: int, method: str = "bsa_p", param: float = 0.005):
        import torch.distributed as dist
        world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        nq = Q.shape[0]
        per = (nq + world - 1) // world
        lo, hi = min(rank * per, nq), min((rank + 1) * per, nq)
        qrot, probes = self.engine.prepare(Q[lo:hi].contiguous(), nprobe)
        qrot = _gather_rows(qrot, per, nq, self.group)
        probes = _gather_rows(probes, per, nq, self.group)
        ids, dists = self.engine.search_prepared(qrot, probes, K, delta_d, method, param)[:2]
        return self.engine.merge_topk(_all_gather(ids, self.group), _all_gather(dists, self.group))
