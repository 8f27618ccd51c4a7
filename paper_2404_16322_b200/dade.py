"""Thin ctypes binding over the C ABI in include/dade.h (argument marshalling only).

Every computation runs in libdade.so (hand-written sm_100a CUDA kernels + host C++). PyTorch
is used for device memory and streams only. There is no CPU fallback: if the library is not
built, or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DADE_LIB", os.path.join(_HERE, "libdade.so"))
MAX_STEPS = 64
MAX_K = 256

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_SHAPE", 3: "ERR_STATE", 4: "ERR_NONFINITE", 5: "ERR_OOM",
          6: "ERR_CUDA", 7: "ERR_NCCL", 8: "ERR_UNSUPPORTED"}
# dade_set_option (include/dade.h DADE_OPT_*)
OPTIONS = {"knn_path": 1, "probe_passes": 2, "scan_warps": 3, "scan_order": 4, "scan_tail": 5,
           "host_chunks": 6, "host_prep_chunks": 7, "dhat_ares": 8, "shard_exchanges": 9,
           "fz_stages": 10, "fz_groups": 11, "fz_cps": 12, "fz_debug": 13, "fz_cpc": 14, "pca_tc": 15, "scan_p1": 17, "dhat_chunk_mb": 18, "knn_i8": 19, "gmin_ratio": 20, "fz_seed_stride": 21, "fz_rows": 22, "fz_cols": 23, "dhat_h16": 24}


class DadeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Stats(C.Structure):
    _fields_ = [("tested", C.c_int64), ("survivors", C.c_int64), ("dims_scanned", C.c_int64),
                ("pruned_at_step", C.c_int64 * MAX_STEPS), ("n_steps", C.c_int32),
                ("n_epochs", C.c_int32), ("ms_rotate", C.c_float), ("ms_probe", C.c_float),
                ("ms_scan", C.c_float), ("ms_total", C.c_float)]

    def as_dict(self) -> dict:
        return {"tested": self.tested, "survivors": self.survivors, "dims_scanned": self.dims_scanned,
                "pruned_at_step": list(self.pruned_at_step[: self.n_steps]), "n_steps": self.n_steps,
                "n_epochs": self.n_epochs, "ms_rotate": self.ms_rotate, "ms_probe": self.ms_probe,
                "ms_scan": self.ms_scan, "ms_total": self.ms_total}


_lib = None
P = C.c_void_p
I64, I32, DBL = C.c_int64, C.c_int, C.c_double
_SIGS = {
    "dade_create": [I32, P, I32, C.POINTER(P)],
    "dade_destroy": [P],
    "dade_fit_rotation": [P, P, I64, I64],
    "dade_pca_mean_partial": [P, P, I64, I64, I64, I64, P, P],
    "dade_pca_cov_partial": [P, P, I64, I64, I64, I64, P, P],
    "dade_set_rotation_from_cov": [P, P, P, I64],
    "dade_get_rotation": [P, P, P, P],
    "dade_set_rotation": [P, P, P, P],
    "dade_build_ivf": [P, P, I64, I64, I32, P, I32],
    "dade_get_ivf": [P, P, P, P, P],
    "dade_get_sizes": [P, P, P],
    "dade_get_layout": [P, P],
    "dade_calibrate": [P, P, P, I32, I32, I32, I32, C.c_uint64],
    "dade_get_calibration": [P, P, P, P, P, P],
    "dade_set_calibration": [P, I32, I32, I32, P, P],
    "dade_search": [P, P, I32, I32, I32, I32, DBL, P, P, P],
    "dade_search_host": [P, P, I32, I32, I32, I32, DBL, P, P, P],
    "dade_search_method": [P, P, I32, I32, I32, I32, I32, DBL, P, P, P],
    "dade_prepare": [P, P, I32, I32, P, P],
    "dade_kmeans_partial": [P, P, I64, I64, I64, I32, P, P, P],
    "dade_calib_knn": [P, P, P, I32, I32, P, P],
    "dade_calib_negatives": [P, P, I32, I32, P, I32, I32, C.c_uint64, P, P, P],
    "dade_pair_features": [P, P, I32, I32, P, P, P],
    "dade_fit_calibration": [P, I32, I32, P, P, P],
    "dade_set_timing": [P, I32],
    "dade_get_timing": [P, P],
    "dade_search_prepared": [P, P, P, I32, I32, I32, I32, I32, DBL, P, P, P],
    "dade_probe": [P, P, I32, I32, P],
    "dade_estimate_knn": [P, P, I32, I32, I32, I32, P, P],
    "dade_bruteforce_knn": [P, P, I64, I64, P, I32, I32, P, P],
    "dade_merge_topk": [P, P, P, I32, I32, I32, P, P],
    "dade_set_ivf": [P, P, I64, I64, P, P, I32, P],
    "dade_set_option": [P, I32, I64],
    "dade_search_log": [P, P, I32, I32, I32, I32, I32, DBL, P, P, P, I64, P],
    "dade_train_pq": [P, P, I64, I32, I64, I32, I32, I32],
    "dade_set_pq": [P, I32, P],
    "dade_get_pq": [P, P, P, P, P],
    "dade_calibrate_pq": [P, P, P, I32, I32, I32, I32, C.c_uint64],
    "dade_get_calibration_q": [P, P, P, P, P],
    "dade_set_calibration_q": [P, I32, I32, P, P],
    "dade_build_graph": [P, P, I32, I32, I32],
    "dade_set_graph": [P, P, I32, I64],
    "dade_get_graph": [P, P, P, P],
    "dade_graph_search": [P, P, I32, I32, I32, I32, DBL, P, P, P, P, I64, P],
    "dade_comm_unique_id": [P],
    "dade_set_comm": [P, P, I32, I32],
    "dade_fit_rotation_dist": [P, P, I64, I64, I64, I64],
    "dade_build_ivf_dist": [P, P, I64, I64, I64, I32, I32],
    "dade_calibrate_dist": [P, P, P, I32, I32, I32, I32, C.c_uint64],
    "dade_kmeans_update": [I32, I32, P, P, P],
    "dade_merge_knn": [I32, I32, I32, P, P, P, P],
    "dade_calibration_pairs": [I32, I32, I32, I32, P, P, P, P, P, P, P, P, P, P],
    "dade_save": [P, C.c_char_p],
    "dade_load": [P, C.c_char_p],
}


def lib():
    """Load libdade.so (built in-tree by paper_2404_16322_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2404_16322_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.dade_last_error.restype = C.c_char_p
        L.dade_last_error.argtypes = []
        _lib = L
    return _lib


def _ck(st: int):
    if st != 0:
        raise DadeError(st, lib().dade_last_error().decode())


def _ptr(t) -> int:
    """Device (torch CUDA tensor) or host (numpy / torch CPU) pointer of a contiguous array."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    assert t.is_contiguous(), "tensor must be contiguous"
    return t.data_ptr()


def _dev(t, dtype):
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous(), \
        f"expected a contiguous CUDA {dtype} tensor"
    return t


# ---------------------------------------------------------------- host steps of the sharded build
def comm_unique_id() -> bytes:
    """128-byte NCCL unique id for dade_set_comm (created on one rank, shared with the others)."""
    buf = C.create_string_buffer(128)
    _ck(lib().dade_comm_unique_id(C.cast(buf, P)))
    return buf.raw


def kmeans_update(sums, counts, centroids):
    """dade_kmeans_update: centroid = fp32(sum / count) where count > 0 (in place on `centroids`)."""
    sums = np.ascontiguousarray(sums, np.float64); counts = np.ascontiguousarray(counts, np.int64)
    assert centroids.dtype == np.float32 and centroids.flags["C_CONTIGUOUS"]
    _ck(lib().dade_kmeans_update(centroids.shape[0], centroids.shape[1], _ptr(sums), _ptr(counts), _ptr(centroids)))
    return centroids


def merge_knn(ids_g, d_g, K: int):
    """dade_merge_knn: [S, nq, K] shard K-NN lists (global ids, fp64) -> the global K-NN by (dist, id)."""
    ids_g = np.ascontiguousarray(ids_g, np.int64); d_g = np.ascontiguousarray(d_g, np.float64)
    S, nq, _ = ids_g.shape
    oi = np.zeros((nq, K), np.int64); od = np.zeros((nq, K))
    _ck(lib().dade_merge_knn(S, nq, K, _ptr(ids_g), _ptr(d_g), _ptr(oi), _ptr(od)))
    return oi, od


def calibration_pairs(knn_ids, knn_d, keys_g, nids_g, cnt_g, n_neg: int):
    """dade_calibration_pairs: (pair_q, pair_id, tau, y) in dade_calibrate's order."""
    knn_ids = np.ascontiguousarray(knn_ids, np.int64); knn_d = np.ascontiguousarray(knn_d, np.float64)
    keys_g = np.ascontiguousarray(keys_g, np.uint64); nids_g = np.ascontiguousarray(nids_g, np.int64)
    cnt_g = np.ascontiguousarray(cnt_g, np.int32)
    S, nq, w = keys_g.shape
    K = knn_ids.shape[1]
    cap = nq * (K + w)
    pq = np.zeros(cap, np.int32); pid = np.zeros(cap, np.int64); tau = np.zeros(cap); y = np.zeros(cap)
    npairs = np.zeros(1, np.int64)
    _ck(lib().dade_calibration_pairs(S, nq, K, w, _ptr(knn_ids), _ptr(knn_d), _ptr(keys_g), _ptr(nids_g),
                                     _ptr(cnt_g), _ptr(pq), _ptr(pid), _ptr(tau), _ptr(y), _ptr(npairs)))
    n = int(npairs[0])
    return pq[:n], pid[:n], tau[:n], y[:n]


class Index:
    """One shard of a DADE index on one GPU (wraps `dade_index*`)."""

    def __init__(self, D: int, device: int = 0, stream=None):
        import torch
        self.D = D
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = P()
        _ck(lib().dade_create(device, P(self.stream.cuda_stream), D, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().dade_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------- a0
    def fit_rotation(self, X, sample_size: int = 0):
        import torch
        X = _dev(X, torch.float32)
        _ck(lib().dade_fit_rotation(self.h, _ptr(X), X.shape[0], sample_size))

    def pca_mean_partial(self, X, id_base: int, n_total: int, sample_size: int = 0):
        s = np.zeros(self.D); cnt = np.zeros(1, np.int64)
        n = 0 if X is None else X.shape[0]
        _ck(lib().dade_pca_mean_partial(self.h, _ptr(X), n, id_base, n_total, sample_size, _ptr(s), _ptr(cnt)))
        return s, int(cnt[0])

    def pca_cov_partial(self, X, id_base: int, n_total: int, mean, sample_size: int = 0):
        mean = np.ascontiguousarray(mean, np.float64)
        cov = np.zeros((self.D, self.D))
        n = 0 if X is None else X.shape[0]
        _ck(lib().dade_pca_cov_partial(self.h, _ptr(X), n, id_base, n_total, sample_size, _ptr(mean), _ptr(cov)))
        return cov

    def set_rotation_from_cov(self, mean, cov_sum, count: int):
        mean = np.ascontiguousarray(mean, np.float64); cov_sum = np.ascontiguousarray(cov_sum, np.float64)
        _ck(lib().dade_set_rotation_from_cov(self.h, _ptr(mean), _ptr(cov_sum), count))

    def get_rotation(self):
        D = self.D
        m, R, l = np.zeros(D), np.zeros((D, D)), np.zeros(D)
        _ck(lib().dade_get_rotation(self.h, _ptr(m), _ptr(R), _ptr(l)))
        return m, R, l

    def set_rotation(self, mean, R, eigvals=None):
        mean = np.ascontiguousarray(mean, np.float64); R = np.ascontiguousarray(R, np.float64)
        ev = None if eigvals is None else np.ascontiguousarray(eigvals, np.float64)
        _ck(lib().dade_set_rotation(self.h, _ptr(mean), _ptr(R), _ptr(ev)))

    # -------------------------------------------------- a1 + a2
    def build_ivf(self, X, nlist: int, centroids=None, kmeans_iters: int = 10, id_base: int = 0):
        import torch
        X = _dev(X, torch.float32)
        if centroids is not None:
            centroids = _dev(centroids, torch.float32)
        _ck(lib().dade_build_ivf(self.h, _ptr(X), X.shape[0], id_base, nlist, _ptr(centroids), kmeans_iters))

    def sizes(self):
        n = np.zeros(1, np.int64); nl = np.zeros(1, np.int32)
        _ck(lib().dade_get_sizes(self.h, _ptr(n), _ptr(nl)))
        return int(n[0]), int(nl[0])

    def get_ivf(self):
        n, nlist = self.sizes()
        off = np.zeros(nlist + 1, np.int64); row_id = np.zeros(n, np.int64)
        assign = np.zeros(n, np.int32); cent = np.zeros((nlist, self.D), np.float32)
        _ck(lib().dade_get_ivf(self.h, _ptr(off), _ptr(row_id), _ptr(assign), _ptr(cent)))
        return off, row_id, assign, cent

    def set_ivf(self, Xrot, row_id, off, centroids, id_base: int = 0):
        """Inject a ready layout in the current rotation's basis: Xrot CUDA [n, D] fp32 rotated
        rows in list-major order, row_id / off host int64 (as get_ivf returns them), centroids
        CUDA [nlist, D] fp32 raw-space."""
        import torch
        Xrot = _dev(Xrot, torch.float32); centroids = _dev(centroids, torch.float32)
        rid = np.ascontiguousarray(row_id, np.int64); off = np.ascontiguousarray(off, np.int64)
        _ck(lib().dade_set_ivf(self.h, _ptr(Xrot), Xrot.shape[0], id_base, _ptr(rid), _ptr(off),
                               len(off) - 1, _ptr(centroids)))

    def set_option(self, name: str, value: int):
        """Tuning option of this index (dade_set_option): knn_path, probe_passes, scan_warps,
        scan_order, scan_tail, host_chunks, host_prep_chunks, dhat_ares."""
        _ck(lib().dade_set_option(self.h, OPTIONS[name], int(value)))

    def get_layout(self):
        n, _ = self.sizes()
        out = np.zeros((n, self.D), np.float32)
        _ck(lib().dade_get_layout(self.h, _ptr(out)))
        return out

    # -------------------------------------------------- a3
    def calibrate(self, X, Qc, K: int, n_neg: int = 50, nprobe_neg: int = 0, seed: int = 0):
        import torch
        X = _dev(X, torch.float32); Qc = _dev(Qc, torch.float32)
        _ck(lib().dade_calibrate(self.h, _ptr(X), _ptr(Qc), Qc.shape[0], K, n_neg, nprobe_neg, seed))

    def get_calibration(self):
        K, n0, nc = (np.zeros(1, np.int32) for _ in range(3))
        _ck(lib().dade_get_calibration(self.h, _ptr(K), _ptr(n0), _ptr(nc), None, None))
        m1 = np.zeros(int(nc[0])); v = np.zeros((int(nc[0]), int(n0[0])))
        _ck(lib().dade_get_calibration(self.h, None, None, None, _ptr(m1), _ptr(v)))
        return {"K": int(K[0]), "n0": int(n0[0]), "m1": m1, "v": v, "block": 16}

    def set_calibration(self, K: int, m1, v):
        m1 = np.ascontiguousarray(m1, np.float64); v = np.ascontiguousarray(v, np.float64)
        _ck(lib().dade_set_calibration(self.h, K, v.shape[1], v.shape[0], _ptr(m1), _ptr(v)))

    # -------------------------------------------------- a4..a8
    def search(self, Q, K: int, nprobe: int, delta_d: int, significance: float, ids=None, dists=None,
               stats: bool = False):
        import torch
        Q = _dev(Q, torch.float32)
        nq = Q.shape[0]
        if ids is None:
            ids = torch.empty((nq, K), dtype=torch.int64, device=Q.device)
        if dists is None:
            dists = torch.empty((nq, K), dtype=torch.float32, device=Q.device)
        st = Stats() if stats else None
        _ck(lib().dade_search(self.h, _ptr(Q), nq, K, nprobe, delta_d, float(significance), _ptr(ids),
                              _ptr(dists), C.byref(st) if st is not None else None))
        return (ids, dists, st.as_dict()) if stats else (ids, dists)

    METHODS = {"bsa_p": 0, "adsampling": 1, "bsa_res": 2, "bsa_q": 3}

    def search_method(self, Q, K: int, nprobe: int, delta_d: int, method: str, param: float, ids=None,
                      dists=None, stats: bool = False):
        """NEXT-1: the same scan with another per-step test. method "bsa_p" (param = significance),
        "adsampling" (param = eps0; install a random orthogonal rotation first), "bsa_res"
        (param = multiplier m)."""
        import torch
        Q = _dev(Q, torch.float32)
        nq = Q.shape[0]
        if ids is None:
            ids = torch.empty((nq, K), dtype=torch.int64, device=Q.device)
        if dists is None:
            dists = torch.empty((nq, K), dtype=torch.float32, device=Q.device)
        st = Stats() if stats else None
        _ck(lib().dade_search_method(self.h, _ptr(Q), nq, K, nprobe, delta_d, self.METHODS[method], float(param),
                                     _ptr(ids), _ptr(dists), C.byref(st) if st is not None else None))
        return (ids, dists, st.as_dict()) if stats else (ids, dists)

    def search_log(self, Q, K: int, nprobe: int, delta_d: int, param: float, method: str = "bsa_p",
                   cap: int = 0):
        """Parity run: the search plus its decision log — per tested candidate (query, global id,
        dims read) as an int32 [count, 3] CUDA tensor (unordered). Returns (ids, dists, log)."""
        import torch
        Q = _dev(Q, torch.float32)
        nq = Q.shape[0]
        ids = torch.empty((nq, K), dtype=torch.int64, device=Q.device)
        dists = torch.empty((nq, K), dtype=torch.float32, device=Q.device)
        cap = cap or max(1, nq * 4096)
        log = torch.empty((cap, 3), dtype=torch.int32, device=Q.device)
        cnt = np.zeros(1, np.int64)
        _ck(lib().dade_search_log(self.h, _ptr(Q), nq, K, nprobe, delta_d, self.METHODS[method], float(param),
                                  _ptr(ids), _ptr(dists), _ptr(log), cap, _ptr(cnt)))
        n = int(cnt[0])
        if n > cap:
            return self.search_log(Q, K, nprobe, delta_d, param, method, cap=n)
        return ids, dists, log[:n]

    def kmeans_partial(self, X, id_base: int, n_total: int, nlist: int, centroids=None):
        """This shard's fp64 sums / counts of one Lloyd step over the global strided sample
        (centroids: host nlist x D fp32, None = the init step). Returns (sums, counts)."""
        import torch
        X = _dev(X, torch.float32)
        sums = np.zeros((nlist, self.D)); counts = np.zeros(nlist, np.int64)
        c = None if centroids is None else np.ascontiguousarray(centroids, np.float32)
        _ck(lib().dade_kmeans_partial(self.h, _ptr(X), X.shape[0], id_base, n_total, nlist,
                                      None if c is None else _ptr(c), _ptr(sums), _ptr(counts)))
        return sums, counts

    # ---- sharded calibration steps (sharded.calibrate_sharded combines them across ranks)
    def calib_knn(self, X, Qc, K: int):
        import torch
        X = _dev(X, torch.float32); Qc = _dev(Qc, torch.float32)
        nq = Qc.shape[0]
        ids = np.zeros((nq, K), np.int64); d = np.zeros((nq, K))
        _ck(lib().dade_calib_knn(self.h, _ptr(X), _ptr(Qc), nq, K, _ptr(ids), _ptr(d)))
        return ids, d

    def calib_negatives(self, Qc, K: int, knn_ids, n_neg: int, nprobe_neg: int, seed: int):
        import torch
        Qc = _dev(Qc, torch.float32)
        nq = Qc.shape[0]
        knn = np.ascontiguousarray(knn_ids, np.int64)
        keys = np.zeros((nq, max(n_neg, 1)), np.uint64); ids = np.zeros((nq, max(n_neg, 1)), np.int64)
        cnt = np.zeros(nq, np.int32)
        _ck(lib().dade_calib_negatives(self.h, _ptr(Qc), nq, K, _ptr(knn), n_neg, nprobe_neg, seed, _ptr(keys),
                                       _ptr(ids), _ptr(cnt)))
        return keys, ids, cnt

    def pair_features(self, Qc, pair_q, pair_id):
        import torch
        Qc = _dev(Qc, torch.float32)
        pq = np.ascontiguousarray(pair_q, np.int32); pid = np.ascontiguousarray(pair_id, np.int64)
        F = np.zeros((len(pq), self.D // 16))
        _ck(lib().dade_pair_features(self.h, _ptr(Qc), Qc.shape[0], len(pq), _ptr(pq), _ptr(pid), _ptr(F)))
        return F

    def fit_calibration(self, K: int, F, tau, y):
        F = np.ascontiguousarray(F, np.float64); tau = np.ascontiguousarray(tau, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        _ck(lib().dade_fit_calibration(self.h, K, len(tau), _ptr(F), _ptr(tau), _ptr(y)))

    def set_timing(self, on: bool):
        """Record stage events on every search (no synchronisation); read them with get_timing."""
        _ck(lib().dade_set_timing(self.h, int(bool(on))))

    def get_timing(self):
        """{'rotate', 'probe', 'scan'} ms of the last search (waits for its events)."""
        ms = np.zeros(3, np.float32)
        _ck(lib().dade_get_timing(self.h, _ptr(ms)))
        return {"rotate": float(ms[0]), "probe": float(ms[1]), "scan": float(ms[2])}

    def prepare(self, Q, nprobe: int):
        """a4 + a5 only: (q~ = R(q - mu) [nq, D] fp32, probes [nq, nprobe] int32) on the device."""
        import torch
        Q = _dev(Q, torch.float32)
        nq = Q.shape[0]
        qrot = torch.empty((nq, self.D), dtype=torch.float32, device=Q.device)
        probes = torch.empty((nq, nprobe), dtype=torch.int32, device=Q.device)
        _ck(lib().dade_prepare(self.h, _ptr(Q), nq, nprobe, _ptr(qrot), _ptr(probes)))
        return qrot, probes

    def search_prepared(self, qrot, probes, K: int, delta_d: int, method: str, param: float, ids=None,
                        dists=None, stats: bool = False):
        """a6-a8 on this shard for prepared queries (see prepare)."""
        import torch
        qrot = _dev(qrot, torch.float32)
        probes = _dev(probes, torch.int32)
        nq, nprobe = probes.shape
        if ids is None:
            ids = torch.empty((nq, K), dtype=torch.int64, device=qrot.device)
        if dists is None:
            dists = torch.empty((nq, K), dtype=torch.float32, device=qrot.device)
        st = Stats() if stats else None
        _ck(lib().dade_search_prepared(self.h, _ptr(qrot), _ptr(probes), nq, K, nprobe, delta_d,
                                       self.METHODS[method], float(param), _ptr(ids), _ptr(dists),
                                       C.byref(st) if st is not None else None))
        return (ids, dists, st.as_dict()) if stats else (ids, dists)

    def search_host(self, Q, K: int, nprobe: int, delta_d: int, significance: float, ids=None, dists=None,
                    stats: bool = False):
        """Q, ids, dists in HOST memory (numpy or pinned torch CPU tensors); H2D/D2H inside."""
        nq = Q.shape[0]
        if ids is None:
            ids = np.empty((nq, K), np.int64)
        if dists is None:
            dists = np.empty((nq, K), np.float32)
        st = Stats() if stats else None
        _ck(lib().dade_search_host(self.h, _ptr(Q), nq, K, nprobe, delta_d, float(significance), _ptr(ids),
                                   _ptr(dists), C.byref(st) if st is not None else None))
        return (ids, dists, st.as_dict()) if stats else (ids, dists)

    def probe(self, Q, nprobe: int):
        import torch
        Q = _dev(Q, torch.float32)
        out = torch.empty((Q.shape[0], nprobe), dtype=torch.int32, device=Q.device)
        _ck(lib().dade_probe(self.h, _ptr(Q), Q.shape[0], nprobe, _ptr(out)))
        return out

    # -------------------------------------------------- tools
    ESTIMATORS = {"partial": 0, "residual": 1}

    def estimate_knn(self, Q, d: int, K: int, estimator: str = "partial"):
        """NEXT-2 (Exp-7 / Table III): per query the K rows with the smallest d-dim distance
        estimate over the whole index ("partial" = P_d, "residual" = P_d + ||x_r||^2 + ||q_r||^2)."""
        import torch
        Q = _dev(Q, torch.float32)
        nq = Q.shape[0]
        ids = torch.empty((nq, K), dtype=torch.int64, device=Q.device)
        est = torch.empty((nq, K), dtype=torch.float32, device=Q.device)
        _ck(lib().dade_estimate_knn(self.h, _ptr(Q), nq, d, self.ESTIMATORS[estimator], K, _ptr(ids), _ptr(est)))
        return ids, est

    def bruteforce_knn(self, X, Q, K: int, id_base: int = 0):
        import torch
        X = _dev(X, torch.float32); Q = _dev(Q, torch.float32)
        ids = torch.empty((Q.shape[0], K), dtype=torch.int64, device=Q.device)
        d = torch.empty((Q.shape[0], K), dtype=torch.float32, device=Q.device)
        _ck(lib().dade_bruteforce_knn(self.h, _ptr(X), X.shape[0], id_base, _ptr(Q), Q.shape[0], K, _ptr(ids), _ptr(d)))
        return ids, d

    def merge_topk(self, ids_in, dists_in):
        """ids_in/dists_in: CUDA tensors S x nq x K (as all_gather_into_tensor lays them out)."""
        import torch
        ids_in = _dev(ids_in, torch.int64); dists_in = _dev(dists_in, torch.float32)
        S, nq, K = ids_in.shape
        ids = torch.empty((nq, K), dtype=torch.int64, device=ids_in.device)
        d = torch.empty((nq, K), dtype=torch.float32, device=ids_in.device)
        _ck(lib().dade_merge_topk(self.h, _ptr(ids_in), _ptr(dists_in), S, nq, K, _ptr(ids), _ptr(d)))
        return ids, d

    # -------------------------------------------------- NEXT-3 BSA-q (OPQ + PQ codes + ADC test)
    def train_pq(self, X, m: int, n_train: int = 0, iters: int = 8, km_iters: int = 4, final_iters: int = 10):
        """OPQ training (installs the OPQ rotation and the codebooks; build_ivf afterwards)."""
        import torch
        X = _dev(X, torch.float32)
        _ck(lib().dade_train_pq(self.h, _ptr(X), X.shape[0], m, n_train, iters, km_iters, final_iters))

    def set_pq(self, codebooks):
        C = np.ascontiguousarray(codebooks, np.float32)
        _ck(lib().dade_set_pq(self.h, C.shape[0], _ptr(C)))

    def get_pq(self, with_codes: bool = True):
        """(codebooks [m, 256, D/m] fp32, codes [n, m] uint8 list-major, err [n] fp32)."""
        mm = np.zeros(1, np.int32)
        _ck(lib().dade_get_pq(self.h, _ptr(mm), None, None, None))
        m = int(mm[0])
        C = np.zeros((m, 256, self.D // m), np.float32)
        n, _ = self.sizes()
        codes = np.zeros((n, m), np.uint8) if with_codes else None
        err = np.zeros(n, np.float32) if with_codes else None
        _ck(lib().dade_get_pq(self.h, None, _ptr(C), _ptr(codes), _ptr(err)))
        return C, codes, err

    def calibrate_pq(self, X, Qc, K: int, n_neg: int = 50, nprobe_neg: int = 0, seed: int = 0):
        import torch
        X = _dev(X, torch.float32); Qc = _dev(Qc, torch.float32)
        _ck(lib().dade_calibrate_pq(self.h, _ptr(X), _ptr(Qc), Qc.shape[0], K, n_neg, nprobe_neg, seed))

    def get_calibration_q(self):
        K, n0 = np.zeros(1, np.int32), np.zeros(1, np.int32)
        _ck(lib().dade_get_calibration_q(self.h, _ptr(K), _ptr(n0), None, None))
        m = np.zeros(2); v = np.zeros(int(n0[0]))
        _ck(lib().dade_get_calibration_q(self.h, None, None, _ptr(m), _ptr(v)))
        return {"K": int(K[0]), "n0": int(n0[0]), "m": m, "v": v}

    def set_calibration_q(self, K: int, m, v):
        m = np.ascontiguousarray(m, np.float64); v = np.ascontiguousarray(v, np.float64)
        _ck(lib().dade_set_calibration_q(self.h, K, len(v), _ptr(m), _ptr(v)))

    # -------------------------------------------------- NEXT-4 graph refinement with the DCO
    def build_graph(self, X, M0: int = 32, P: int = 64, nprobe_pool: int = 0):
        """Base-layer graph over this index's rows (X = the raw rows given to build_ivf);
        nprobe_pool = 0: every list (exact pools)."""
        import torch
        X = _dev(X, torch.float32)
        _, nlist = self.sizes()
        _ck(lib().dade_build_graph(self.h, _ptr(X), M0, P, nprobe_pool or nlist))

    def set_graph(self, nbrs, entry: int):
        nb = np.ascontiguousarray(nbrs, np.int64)
        _ck(lib().dade_set_graph(self.h, _ptr(nb), nb.shape[1], int(entry)))

    def get_graph(self):
        m0 = np.zeros(1, np.int32); e = np.zeros(1, np.int64)
        _ck(lib().dade_get_graph(self.h, _ptr(m0), None, _ptr(e)))
        n, _ = self.sizes()
        nb = np.zeros((n, int(m0[0])), np.int64)
        _ck(lib().dade_get_graph(self.h, None, _ptr(nb), None))
        return nb, int(e[0])

    def graph_search(self, Q, K: int, ef: int, delta_d: int, significance: float, stats: bool = False,
                     log: bool = False, cap: int = 0):
        """HNSW base-layer refinement with the DCO. Returns (ids, dists[, stats][, log])."""
        import torch
        Q = _dev(Q, torch.float32)
        nq = Q.shape[0]
        ids = torch.empty((nq, K), dtype=torch.int64, device=Q.device)
        dists = torch.empty((nq, K), dtype=torch.float32, device=Q.device)
        st = Stats() if stats else None
        lg, cnt = None, np.zeros(1, np.int64)
        if log:
            cap = cap or max(1, nq * 4 * ef * 32)
            lg = torch.empty((cap, 3), dtype=torch.int32, device=Q.device)
        _ck(lib().dade_graph_search(self.h, _ptr(Q), nq, K, ef, delta_d, float(significance), _ptr(ids), _ptr(dists),
                                    C.byref(st) if st is not None else None, _ptr(lg) if log else None,
                                    cap if log else 0, _ptr(cnt) if log else None))
        out = [ids, dists]
        if stats:
            out.append(st.as_dict())
        if log:
            n = int(cnt[0])
            if n > cap:
                return self.graph_search(Q, K, ef, delta_d, significance, stats, log, cap=n)
            out.append(lg[:n])
        return tuple(out)

    # -------------------------------------------------- multi-rank (the library owns NCCL)
    def set_comm(self, uid, nranks: int, rank: int):
        """Join the NCCL group (collective). uid: the 128-byte id from comm_unique_id() (None for a
        group of one). Afterwards search / search_method / search_host are collective."""
        buf = None if uid is None else C.create_string_buffer(bytes(uid), 128)
        _ck(lib().dade_set_comm(self.h, None if buf is None else C.cast(buf, P), nranks, rank))

    def fit_rotation_dist(self, X, id_base: int, n_total: int, sample_size: int = 0):
        import torch
        X = _dev(X, torch.float32)
        _ck(lib().dade_fit_rotation_dist(self.h, _ptr(X), X.shape[0], id_base, n_total, sample_size))

    def build_ivf_dist(self, X, id_base: int, n_total: int, nlist: int, kmeans_iters: int = 10):
        import torch
        X = _dev(X, torch.float32)
        _ck(lib().dade_build_ivf_dist(self.h, _ptr(X), X.shape[0], id_base, n_total, nlist, kmeans_iters))

    def calibrate_dist(self, X, Qc, K: int, n_neg: int = 50, nprobe_neg: int = 0, seed: int = 0):
        import torch
        X = _dev(X, torch.float32); Qc = _dev(Qc, torch.float32)
        _ck(lib().dade_calibrate_dist(self.h, _ptr(X), _ptr(Qc), Qc.shape[0], K, n_neg, nprobe_neg, seed))

    def save(self, path: str):
        _ck(lib().dade_save(self.h, path.encode()))

    def load(self, path: str):
        _ck(lib().dade_load(self.h, path.encode()))
