"""Multi-GPU plumbing for the DADE path. Moves buffers only: every
step of the method, including the combination of the shards' partial results, runs in libdade.so.

The database is sharded by contiguous global-id ranges, one shard per rank (one process per GPU).
Two ways to drive a group of ranks:

* `attach_comm(index)` (production, bench.py): rank 0 creates the NCCL unique id, the process
  group broadcasts it, and every rank joins the library's own NCCL communicator
  (`dade_set_comm`). From then on the library runs the collectives itself: the sharded build
  (`Index.fit_rotation_dist / build_ivf_dist / calibrate_dist`) and the collective search
  (`Index.search*`: query-partitioned rotate + probe, all-gather, local scan, all-gather + merge).
* the process-group functions below (`fit_rotation_sharded`, `kmeans_sharded`,
  `calibrate_sharded`, `ShardedSearch`, `QueryPartitionedSearch`): torch.distributed moves the
  partial results between ranks and the library's host steps (`dade_kmeans_update`,
  `dade_merge_knn`, `dade_calibration_pairs`) and merge kernel combine them. The CPU tests run
  these over gloo with the oracle as the per-shard engine.

`engine` is the per-shard object: `paper_2404_16322_b200.Index` in production.
"""
from __future__ import annotations

import numpy as np

from . import dade


def shard_range(n: int, rank: int, world: int):
    """Rows [lo, hi) owned by `rank`: contiguous id ranges, sizes differing by at most 1."""
    return rank * n // world, (rank + 1) * n // world


def attach_comm(engine, group=None):
    """Join the library's NCCL communicator (collective over the process group): rank 0 creates
    the unique id, the group broadcasts it, every rank calls dade_set_comm."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    obj = [dade.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    engine.set_comm(obj[0], world, rank)


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


def _to_group(t, group=None):
    import torch.distributed as dist
    return t.cuda() if dist.get_backend(group) == "nccl" else t


def _all_reduce_np(a, dtype, group=None):
    import torch
    import torch.distributed as dist
    t = _to_group(torch.from_numpy(np.ascontiguousarray(a)).to(dtype), group)
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def _gather_np(a, group=None):
    """All-gather a host numpy array (same shape on every rank) -> [world, ...] numpy."""
    import torch
    t = _to_group(torch.from_numpy(np.ascontiguousarray(a)), group)
    return _all_gather(t, group).cpu().numpy()


def fit_rotation_sharded(engine, X_shard, id_base: int, n_total: int, sample_size: int = 0, group=None):
    """a0 over a sharded base: fp64 sum and count of the owned strided-sample rows (all-reduced),
    mean; fp64 centred cross products (all-reduced); every rank runs the same eigensolve."""
    import torch
    s, c = engine.pca_mean_partial(X_shard, id_base, n_total, sample_size)
    t = _all_reduce_np(np.r_[s, c], torch.float64, group)
    cnt = int(round(t[-1]))
    mean = t[:-1] / cnt
    cov = _all_reduce_np(engine.pca_cov_partial(X_shard, id_base, n_total, mean, sample_size), torch.float64, group)
    engine.set_rotation_from_cov(mean, cov, cnt)
    return mean, cnt


def kmeans_sharded(engine, X_shard, id_base: int, n_total: int, nlist: int, iters: int = 10, group=None):
    """k-means over a sharded base: the global strided sample, init = its first
    nlist rows, `iters` Lloyd steps whose per-cluster fp64 sums and counts are all-reduced; the
    update (dade_kmeans_update) runs on every rank. Returns the nlist x D fp32 centroids (host)."""
    import torch
    sums, counts = engine.kmeans_partial(X_shard, id_base, n_total, nlist, None)
    cent = _all_reduce_np(sums, torch.float64, group).astype(np.float32)
    for _ in range(iters):
        sums, counts = engine.kmeans_partial(X_shard, id_base, n_total, nlist, cent)
        cent = dade.kmeans_update(_all_reduce_np(sums, torch.float64, group),
                                  _all_reduce_np(counts, torch.int64, group), cent.copy())
    return cent


def calibrate_sharded(engine, X_shard, Qc, K: int, n_neg: int = 50, nprobe_neg: int = 0, seed: int = 0,
                      group=None):
    """dade_calibrate over a sharded base: each step on every shard, combined as the
    single-GPU calibration defines them — K-NN lists merged by (fp64 dist, id) (dade_merge_knn,
    R14), negatives the n_neg smallest (hash, id) over the shards (dade_calibration_pairs,
    R15/R16), pair features summed over ranks — so the installed table equals an unsharded
    dade_calibrate on the same base, centroids and rotation."""
    import torch
    ids_l, d_l = engine.calib_knn(X_shard, Qc, K)
    knn_ids, knn_d = dade.merge_knn(_gather_np(ids_l, group), _gather_np(d_l, group), K)
    keys_l, nids_l, cnt_l = engine.calib_negatives(Qc, K, knn_ids, n_neg, nprobe_neg, seed)
    keys_g = _gather_np(keys_l.view(np.int64), group).view(np.uint64)
    pq, pid, tau, y = dade.calibration_pairs(knn_ids, knn_d, keys_g, _gather_np(nids_l, group),
                                             _gather_np(cnt_l, group), n_neg)
    F = _all_reduce_np(engine.pair_features(Qc, pq, pid), torch.float64, group)
    engine.fit_calibration(K, F, tau, y)


class ShardedSearch:
    """search() on this rank's shard, then all-gather of the local top-K and the merge (a9)."""

    def __init__(self, engine, group=None):
        self.engine, self.group = engine, group

    def search(self, Q, K: int, nprobe: int, delta_d: int, significance: float):
        ids, dists = self.engine.search(Q, K, nprobe, delta_d, significance)[:2]
        return self.engine.merge_topk(_all_gather(ids, self.group), _all_gather(dists, self.group))


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
    """The collective search's schedule over a torch.distributed group (the library's own NCCL
    path, `attach_comm` + `Index.search`, runs the same schedule inside dade_search): rank r
    rotates and probes only its block of queries (a4 + a5, `engine.prepare`), the blocks are
    all-gathered, every rank scans ALL queries on its shard (a6-a8, `engine.search_prepared`), and
    the local top-K lists are all-gathered and merged (a9)."""

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
