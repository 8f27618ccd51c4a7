"""CPU ORACLE for the DADE hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, float64 NumPy restatement of what arxiv 2404.16322
computes on the path BASELINE.json's `north_star` names: PCA rotation,
IVF build/probe, the §V data-driven linear correction calibrated per Δd step,
and the epoch-frozen-τ progressive search. It shares no code with the CUDA
library (paper_2404_16322_b200/) and neither imports the other. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it; the product path never does.

Citations: `P:L<n>` = /root/reference/PAPER.md line n; `R<n>` = the reading
numbered n in DESIGN.md §3 (copied from SURVEY.md §8(c)).

Parity pins: every public function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py against a closed form, a hand-worked example, brute
force on tiny inputs or a property the paper states (DESIGN.md §4 lists which).
No function here is "parity unpinned".
"""
from __future__ import annotations

import math
import numpy as np

F64 = np.float64
U64 = np.uint64
MASK64 = (1 << 64) - 1


# ----------------------------------------------------------------------------- helpers
def strided_ids(n: int, m: int) -> np.ndarray:
    """Portable sample ⌊k·n/m⌋, k = 0..m-1 (R17/R19: integer rule both sides can compute)."""
    return (np.arange(m, dtype=np.int64) * n) // m


def sqdist_seq(rows: np.ndarray, v: np.ndarray) -> np.ndarray:
    """dis(p, q) = ||p - q||^2, evaluated in float64 as the SEQUENTIAL sum over
    j = 0..D-1 of (p_j - q_j)^2 (R20: the exact rule assignment/probe/brute force share).
    `rows` n x D, `v` D; the difference of two fp32 numbers is formed in fp64."""
    rows = np.asarray(rows)
    v = np.asarray(v, dtype=F64)
    acc = np.zeros(rows.shape[0], dtype=F64)
    for j in range(rows.shape[1]):
        t = rows[:, j].astype(F64) - v[j]
        acc += t * t
    return acc


def order_by_dist_id(dist: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Permutation sorting by (dist, id) ascending (R12 tie rule: lower id first)."""
    return np.lexsort((ids, dist))


# ----------------------------------------------------------------------------- O1 fit_rotation
def fit_rotation(X: np.ndarray, sample_size: int = 0):
    """PCA rotation (Theorem 1; proof P:L4067-4096: principal directions are the
    eigenvectors of the covariance Σ, ordered by eigenvalue). Data are centred (P:L305
    footnote). Sample: strided ids, n_s = min(N, 1,000,000) when sample_size == 0 (P:L3105,
    R17). Σ = (X_s-μ)^T(X_s-μ)/n_s (divisor as P:L4074). Eigenvectors sorted by λ
    descending; sign: largest-|component| positive, lowest index on ties (R18).
    Returns (mean[D], R[D,D] rows = directions, lam[D])."""
    X = np.asarray(X)
    n = X.shape[0]
    ns = min(n, 1_000_000) if sample_size <= 0 else min(n, sample_size)
    Xs = X[strided_ids(n, ns)].astype(F64)
    mean = Xs.mean(axis=0)
    Y = Xs - mean
    cov = (Y.T @ Y) / ns
    lam, V = np.linalg.eigh(cov)
    order = np.argsort(-lam, kind="stable")
    lam, V = lam[order], V[:, order]
    for i in range(V.shape[1]):
        j = int(np.argmax(np.abs(V[:, i])))          # argmax returns the lowest index on ties
        if V[j, i] < 0:
            V[:, i] = -V[:, i]
    return mean, np.ascontiguousarray(V.T), lam


def rotate(X: np.ndarray, mean: np.ndarray, R: np.ndarray) -> np.ndarray:
    """x̃ = R(x - μ) in float64 (x_D = R x, after centring P:L305)."""
    return (np.asarray(X, dtype=F64) - mean) @ np.asarray(R, dtype=F64).T


def err_variance(q_rot: np.ndarray, sigma2: np.ndarray, d: int) -> float:
    """Eq. 3: Var(−2⟨q_r, x_r⟩) = 4·Σ_{i>d} (q_i σ_i)^2 over the residual dims
    (0-based: dims d..D-1). Context for the PCA choice; used by the NEXT-1 BSA-res test."""
    q = np.asarray(q_rot, F64)
    return float(4.0 * np.sum(q[d:] ** 2 * np.asarray(sigma2, F64)[d:]))


# ----------------------------------------------------------------------------- O3 IVF
def assign(X: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    """IVF bucket of each point = its nearest centroid, raw space, exact
    sequential fp64 sum (R20), ties to the lower centroid id (R12)."""
    X = np.asarray(X)
    best = np.full(X.shape[0], np.inf)
    arg = np.zeros(X.shape[0], dtype=np.int64)
    for c in range(centroids.shape[0]):
        d = sqdist_seq(X, centroids[c])
        upd = d < best                                  # strict: lower c wins ties
        best[upd] = d[upd]
        arg[upd] = c
    return arg


def kmeans(X: np.ndarray, nlist: int, iters: int = 10) -> np.ndarray:
    """k-means clustering for the IVF buckets ("uses the k-means algorithm";
    details are R19): strided sample of min(N, 64·C) rows, init = first C sampled rows,
    `iters` Lloyd iterations with exact assignment, centroid = fp64 mean rounded to fp32,
    empty cluster keeps its centroid. Returns float32 centroids."""
    X = np.asarray(X, dtype=np.float32)
    n = X.shape[0]
    sample = X[strided_ids(n, min(n, 64 * nlist))]
    cent = sample[:nlist].copy()
    for _ in range(iters):
        a = assign(sample, cent)
        sums = np.zeros((nlist, X.shape[1]), dtype=F64)
        np.add.at(sums, a, sample.astype(F64))
        cnt = np.bincount(a, minlength=nlist)
        nz = cnt > 0
        cent[nz] = (sums[nz] / cnt[nz, None]).astype(np.float32)
    return cent


def build_ivf(X: np.ndarray, centroids: np.ndarray, id_base: int = 0):
    """Buckets: every id in exactly one list; lists hold ids ascending.
    Returns (assign[n], off[nlist+1], row_id[n]) with row_id = global ids, list-major."""
    a = assign(X, centroids)
    nlist = centroids.shape[0]
    cnt = np.bincount(a, minlength=nlist)
    off = np.zeros(nlist + 1, dtype=np.int64)
    off[1:] = np.cumsum(cnt)
    row_id = np.argsort(a, kind="stable").astype(np.int64) + id_base
    return a, off, row_id


def probe(q: np.ndarray, centroids: np.ndarray, nprobe: int) -> np.ndarray:
    """The N^probe nearest centroids of q, raw space, exact fp64 sequential sums,
    ordered by (dist, centroid id) (R12, R20)."""
    d = sqdist_seq(centroids, q)
    return order_by_dist_id(d, np.arange(len(d)))[:nprobe]


# ----------------------------------------------------------------------------- O6 brute force
def brute_force_knn(X: np.ndarray, Q: np.ndarray, K: int, id_base: int = 0):
    """Exact KNN under squared L2, fp64 sequential sums, (dist, id) order
    (R12). Returns ids (nq x K int64) and dists (nq x K float64)."""
    Q = np.atleast_2d(Q)
    ids = np.empty((Q.shape[0], K), dtype=np.int64)
    dists = np.empty((Q.shape[0], K), dtype=F64)
    gid = np.arange(X.shape[0], dtype=np.int64) + id_base
    for i, q in enumerate(Q):
        d = sqdist_seq(X, q)
        o = order_by_dist_id(d, gid)[:K]
        ids[i], dists[i] = gid[o], d[o]
    return ids, dists


# ----------------------------------------------------------------------------- O4 calibrate
def splitmix64(x) -> np.ndarray:
    """SplitMix64 output for state `x` (one step: x += golden gamma, then the finaliser).
    Counter-based: both the oracle and the library evaluate it on (seed ⊕ (q<<32 | id))."""
    z = (np.asarray(x, dtype=U64) + U64(0x9E3779B97F4A7C15))
    with np.errstate(over="ignore"):
        z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
    return z ^ (z >> U64(31))


def neg_hash(seed: int, qi: int, ids: np.ndarray) -> np.ndarray:
    key = (U64(qi) << U64(32)) | np.asarray(ids, dtype=U64)
    return splitmix64(U64(seed) ^ key)


def logistic_irls(P: np.ndarray, tau: np.ndarray, y: np.ndarray, ridge: float = 1e-8,
                  max_iter: int = 100, tol: float = 1e-12):
    """Logistic regression with cross-entropy loss on features (dis', τ)
    (P:L529), label y = 1 ⇔ dis > τ. R3: the BCE minimiser, computed by damped
    Newton/IRLS on standardised features, ridge on the non-intercept weights.
    Returns (m1, beta, ok): the model in the form sign(m1·dis' + β > τ)."""
    P = np.asarray(P, F64); tau = np.asarray(tau, F64); y = np.asarray(y, F64)
    mP, sP = P.mean(), P.std()
    mt, st = tau.mean(), tau.std()
    sP = sP if sP > 0 else 1.0
    st = st if st > 0 else 1.0
    A = np.stack([np.ones_like(P), (P - mP) / sP, (tau - mt) / st], axis=1)
    reg = np.array([0.0, ridge, ridge])

    def loss(w):
        z = A @ w
        return float(np.sum(np.logaddexp(0.0, z) - y * z) + 0.5 * np.sum(reg * w * w))

    w = np.zeros(3)
    cur = loss(w)
    for _ in range(max_iter):
        z = A @ w
        p = 0.5 * (1.0 + np.tanh(0.5 * z))           # logistic σ(z), overflow-free
        g = A.T @ (y - p) - reg * w
        H = (A * (p * (1 - p))[:, None]).T @ A + np.diag(reg)
        step = np.linalg.solve(H, g)
        t = 1.0
        for _h in range(30):                            # damping: halve until the loss does not grow
            nw = w + t * step
            nl = loss(nw)
            if nl <= cur:
                break
            t *= 0.5
        w, cur = nw, nl
        if np.max(np.abs(t * step)) < tol:
            break
    wP, wt = w[1] / sP, w[2] / st
    b = w[0] - w[1] * mP / sP - w[2] * mt / st
    # w_P·P + w_τ·τ + b > 0  ⇔  (−w_P/w_τ)·P + (−b/w_τ) > τ  when w_τ < 0
    if not (wt < 0) or not np.isfinite(wP) or not np.isfinite(wt):
        return 1.0, 0.0, False
    m1 = -wP / wt
    if not (m1 > 0) or not np.isfinite(m1):
        return 1.0, 0.0, False
    return float(m1), float(-b / wt), True


def calibration_pairs(X, index, Qc, K, n_neg, nprobe_neg, seed):
    """Training samples (R14-R16): per calibration query the exact K NN over
    the whole base are Label 0 and τ_q is the K-th NN distance; Label 1 =
    the n_neg non-KNN candidates of q's nprobe_neg probed lists (whole base if 0 or flat)
    with the smallest SplitMix64(seed ⊕ (q<<32 | id)).
    Returns (qi[], id[], label[], tau_of_pair[])."""
    off, row_id, cent = index["off"], index["row_id"], index["centroids"]
    nlist = len(off) - 1
    knn_ids, knn_d = brute_force_knn(X, Qc, K)
    qi_l, id_l, lab_l, tau_l = [], [], [], []
    for qi in range(Qc.shape[0]):
        tau = knn_d[qi, K - 1]
        if nprobe_neg <= 0 or nlist == 1:
            cand = np.arange(X.shape[0], dtype=np.int64)
        else:
            pr = probe(Qc[qi], cent, nprobe_neg)
            cand = np.concatenate([row_id[off[l]:off[l + 1]] for l in pr])
        cand = np.setdiff1d(cand, knn_ids[qi])
        h = neg_hash(seed, qi, cand)
        negs = cand[np.lexsort((cand, h))[:n_neg]]
        for i in knn_ids[qi]:
            qi_l.append(qi); id_l.append(i); lab_l.append(0); tau_l.append(tau)
        for i in negs:
            qi_l.append(qi); id_l.append(i); lab_l.append(1); tau_l.append(tau)
    return (np.array(qi_l), np.array(id_l, dtype=np.int64), np.array(lab_l), np.array(tau_l))


def calibrate(X, index, Qc, K, n_neg=50, nprobe_neg=0, seed=0, block=16):
    """§V-A data-driven correction in its incremental form: one
    linear classifier per projected dimension d ∈ {16, 32, …, D-16}. For each d: the slope
    m1_d from the logistic fit on (P_d, τ) (R3), then the sorted array
    v_d = sort_desc(τ − m1_d·P_d) over Label-0 pairs, from which search derives β'_d (R4).
    P_d = Σ_{i<d}(x̃_i − q̃_i)^2 is BSA-p's plain PCA projected distance (R2).
    Returns dict(m1[ns], v[ns, n0], ok[ns], n0, K)."""
    D = X.shape[1]
    qi, ids, lab, tau = calibration_pairs(X, index, Qc, K, n_neg, nprobe_neg, seed)
    Xr = rotate(X[ids], index["mean"], index["R"])
    Qr = rotate(Qc, index["mean"], index["R"])[qi]
    Pcum = np.cumsum((Xr - Qr) ** 2, axis=1)            # sequential prefix sums over dims
    ns = D // block - 1
    n0 = int(np.sum(lab == 0))
    m1 = np.ones(ns); ok = np.zeros(ns, dtype=bool); v = np.empty((ns, n0))
    for s in range(ns):
        d = (s + 1) * block
        P = Pcum[:, d - 1]
        m1[s], _, ok[s] = logistic_irls(P, tau, lab)
        v[s] = np.sort(tau[lab == 0] - m1[s] * P[lab == 0])[::-1]
    return {"m1": m1, "v": v, "ok": ok, "n0": n0, "K": K, "block": block}


def step_recall(r: float, D: int, delta_d: int) -> float:
    """Per-classifier target recall r_i = 1 − (1 − r)/(D/Δd) (R5)."""
    return 1.0 - (1.0 - r) / (D / delta_d)


def beta_from_v(v_d: np.ndarray, alpha_s: float) -> float:
    """β'_d: the LARGEST intercept whose Label-0 recall on the calibration set is ≥ 1−α_s
    (R4). With v = sort_desc(τ − m1·P), recall(β') = #{v ≥ β'}/n0, so the answer
    is v[k−1], k = clamp(⌈(1−α_s)·n0⌉, 1, n0)."""
    n0 = len(v_d)
    k = min(max(int(math.ceil((1.0 - alpha_s) * n0)), 1), n0)
    return float(v_d[k - 1])


def step_table(cal: dict, D: int, delta_d: int, alpha: float):
    """Per-step (m1, β') used by search at d = Δd, 2Δd, …, D−Δd. α_s = (α·Δd)/D (R5);
    α = 0 disables pruning (β' = −∞, R26)."""
    block = cal["block"]
    ns = D // delta_d
    alpha_s = (alpha * delta_d) / D
    m = np.empty(ns - 1); b = np.empty(ns - 1)
    for s in range(1, ns):
        idx = (s * delta_d) // block - 1
        m[s - 1] = cal["m1"][idx]
        b[s - 1] = -np.inf if alpha == 0 else beta_from_v(cal["v"][idx], alpha_s)
    return m, b


# ----------------------------------------------------------------------------- O5 search
def epoch_bounds(total: int, K: int, c0: int | None = None):
    """R13 epoch schedule: positions 0, c0, 2c0, 4c0, … (c0 = 4K); τ frozen per epoch."""
    c0 = 4 * K if c0 is None else c0
    b = [0]
    nxt = c0
    while b[-1] < total:
        b.append(min(nxt, total))
        nxt *= 2
    return b


def build_index(X, centroids, mean=None, R=None, cal=None, id_base=0, lam=None):
    """Bundle the artefacts search needs (fp64 rotated base, lists, rotation, calibration;
    lam = per-dimension variances σ_i² of the rotated data, for BSA-res)."""
    a, off, row_id = build_ivf(X, centroids, id_base)
    return {"centroids": np.asarray(centroids, np.float32), "assign": a, "off": off,
            "row_id": row_id, "mean": mean, "R": R, "cal": cal, "id_base": id_base, "lam": lam,
            "Xr": None if mean is None else rotate(X, mean, R)}


# ----------------------------------------------------------------------------- NEXT-1 corrections
def adsampling_table(D: int, delta_d: int, eps0: float):
    """ADSampling's hypothesis test as a linear classifier: after d
    randomly projected dims the estimate (D/d)·P_d (JL scaling, Lemma 1) prunes iff
    it exceeds (1 + ε)²·τ with ε = ε₀/√d (R8: squared distances). Returned as the per-step
    (m1, β') of the BSA-p form: m1_d = (D/d)/(1 + ε₀/√d)², β' = 0."""
    ns = D // delta_d
    d = np.arange(1, ns) * delta_d
    return (D / d) / (1.0 + eps0 / np.sqrt(d)) ** 2, np.zeros(ns - 1)


def bsa_res_consts(q_rot: np.ndarray, lam: np.ndarray, delta_d: int, m: float) -> np.ndarray:
    """Per-step query constants of the BSA-res test (Alg. 2; incremental form
    P:L455-470; R6): with P_d the partial distance and N_d = ‖x_{:d}‖², the estimate is
    dis'_d = C1 − C2 = P_d + ‖x_r‖² + ‖q_r‖² (Eq. 2: the dropped term is the error
    −2⟨q_r, x_r⟩), σ_d² = 4·Σ_{i≥d} q_i² σ_i² (Eq. 3, σ_i² = λ_i for the PCA
    basis), and the test prunes iff dis'_d − m·σ_d > τ. Returns c_d = ‖q_r‖² −
    m·σ_d for d = Δd, 2Δd, …, D − Δd; the test is P_d + (‖x‖² − N_d) + c_d > τ."""
    q = np.asarray(q_rot, F64)
    D = q.shape[0]
    ns = D // delta_d
    out = np.empty(ns - 1)
    for s in range(1, ns):
        d = s * delta_d
        out[s - 1] = float(np.sum(q[d:] ** 2)) - m * math.sqrt(err_variance(q, lam, d))
    return out


def search(index, Q, K, nprobe, delta_d, alpha, c0=None, mode="epoch", log=False, method="bsa_p",
           eps0=2.1, m_res=8.0, epochs=None, init_top=None, tau_cap=None):
    """IVF search with the per-step data-driven correction (O5).
    Refinement: result queue of size K, τ = its K-th distance (R11: +∞ until full).
    Candidates = the probed lists in probe order. For each candidate, the partial
    squared distance P_d over the first d rotated dims is accumulated in Δd steps
    (Alg. 2 loop, R9) and the cascade classifier for d prunes iff
    m1_d·P_d + β'_d > τ. Survivors reach d = D, where P_D is the exact distance
    (R10), and enter the queue. mode="epoch": τ frozen per epoch (R13, the parity
    target); mode="sequential": τ refreshed after every survivor (P:L42-43 literal).
    method (NEXT-1, the paper's other corrections on the same loop): "bsa_p" (above, α =
    significance), "adsampling" (adsampling_table(ε₀); use a random orthogonal R), "bsa_res"
    (bsa_res_consts(m_res); needs index["lam"]). α = 0 disables pruning for every method.
    Cross-shard τ seed (R32, epoch mode, used by search_sharded): `epochs` = (first, end) runs only
    those epochs of the stream; `init_top` = (ids, dists) per query starts the result queue (the
    shard's own epoch-0 results); `tau_cap` per query bounds τ_e from above (τ_e = min(K-th of the
    queue, tau_cap[q]))."""
    Q = np.atleast_2d(Q)
    D = Q.shape[1]
    ns = D // delta_d
    if alpha == 0:
        m, b = np.ones(ns - 1), np.full(ns - 1, -np.inf)
    elif method == "bsa_p":
        m, b = step_table(index["cal"], D, delta_d, alpha)
    elif method == "adsampling":
        m, b = adsampling_table(D, delta_d, eps0)
    elif method == "bsa_res":
        m, b = np.ones(ns - 1), np.zeros(ns - 1)
    else:
        raise ValueError(method)
    res = method == "bsa_res" and alpha > 0
    off, row_id, Xr = index["off"], index["row_id"], index["Xr"]
    base = index["id_base"]                          # Xr rows are in id order: row = id - id_base
    out_ids = np.full((Q.shape[0], K), -1, dtype=np.int64)
    out_d = np.full((Q.shape[0], K), np.inf)
    st = {"tested": 0, "dims_scanned": 0, "survivors": 0, "pruned_at_step": np.zeros(ns, np.int64),
          "n_epochs": 0, "decisions": [], "candidates": []}
    Qr = rotate(Q, index["mean"], index["R"])
    steps = np.arange(1, ns) * delta_d
    for qn in range(Q.shape[0]):
        pr = probe(Q[qn], index["centroids"], nprobe)
        qc = bsa_res_consts(Qr[qn], index["lam"], delta_d, m_res) if res else None
        cand = np.concatenate([row_id[off[l]:off[l + 1]] for l in pr]) if len(pr) else np.zeros(0, np.int64)
        top_d = np.zeros(0); top_i = np.zeros(0, dtype=np.int64)
        if init_top is not None:
            ok = init_top[0][qn] >= 0
            top_d, top_i = np.asarray(init_top[1][qn], F64)[ok], np.asarray(init_top[0][qn], np.int64)[ok]
        if mode == "epoch":
            bounds = epoch_bounds(len(cand), K, c0)
            e_first, e_end = (0, len(bounds) - 1) if epochs is None else (epochs[0], min(epochs[1], len(bounds) - 1))
            last = len(bounds) - 1
            st["tested"] += bounds[min(max(e_end, e_first), last)] - bounds[min(e_first, last)]
            st["n_epochs"] = max(st["n_epochs"], len(bounds) - 1)
            for e in range(e_first, e_end):
                tau = top_d[K - 1] if len(top_d) >= K else np.inf
                if tau_cap is not None:
                    tau = min(tau, float(tau_cap[qn]))
                ids = cand[bounds[e]:bounds[e + 1]]
                P = np.cumsum((Xr[ids - base] - Qr[qn]) ** 2, axis=1)
                keep = np.ones(len(ids), dtype=bool)
                dims = np.full(len(ids), D)
                margin = np.full(len(ids), np.inf)
                if np.isfinite(tau) and ns > 1:
                    score = m[None, :] * P[:, steps - 1] + b[None, :]
                    if res:  # P_d + ‖x_r‖² + c_d, ‖x_r‖² = ‖x‖² − N_d
                        N = np.cumsum(Xr[ids - base] ** 2, axis=1)
                        score = score + (N[:, D - 1:D] - N[:, steps - 1]) + qc[None, :]
                    test = score > tau
                    anyp = test.any(axis=1)
                    first = np.argmax(test, axis=1)
                    keep = ~anyp
                    dims[anyp] = steps[first[anyp]]
                    np.add.at(st["pruned_at_step"], first[anyp] + 1, 1)
                    if log:
                        for i in np.nonzero(anyp)[0]:
                            s = first[i]
                            st["decisions"].append((qn, int(ids[i]), int(steps[s]),
                                                    float(score[i, s]), float(tau)))
                        # closest call of each candidate over the tests it went through (up to and
                        # including the deciding one): |score − τ| / (|m1·P| + |β'| + τ) — a decision
                        # taken in another rounding (fp32 on the GPU, R21) can only differ where it is tiny
                        scale = np.abs(m[None, :] * P[:, steps - 1]) + np.abs(b[None, :]) + tau
                        rel = np.abs(score - tau) / scale
                        last = np.where(anyp, first, ns - 2)
                        upto = np.arange(ns - 1)[None, :] <= last[:, None]
                        margin = np.where(upto, rel, np.inf).min(axis=1)
                if log:
                    st["candidates"].append((np.full(len(ids), qn), ids.copy(), dims.copy(), margin))
                st["dims_scanned"] += int(dims.sum())
                st["survivors"] += int(keep.sum())
                cd = np.concatenate([top_d, P[keep, D - 1]])
                ci = np.concatenate([top_i, ids[keep]])
                o = order_by_dist_id(cd, ci)[:K]
                top_d, top_i = cd[o], ci[o]
        else:
            st["tested"] += len(cand)
            for idn in cand:
                tau = top_d[K - 1] if len(top_d) >= K else np.inf
                P = np.cumsum((Xr[idn - base] - Qr[qn]) ** 2)
                N = np.cumsum(Xr[idn - base] ** 2)
                pruned_at = 0
                if np.isfinite(tau):
                    for si, d in enumerate(steps):
                        sc = m[si] * P[d - 1] + b[si]
                        if res:
                            sc += (N[D - 1] - N[d - 1]) + qc[si]
                        if sc > tau:
                            pruned_at = d
                            st["pruned_at_step"][si + 1] += 1
                            break
                st["dims_scanned"] += pruned_at if pruned_at else D
                if pruned_at:
                    continue
                st["survivors"] += 1
                cd = np.append(top_d, P[D - 1]); ci = np.append(top_i, idn)
                o = order_by_dist_id(cd, ci)[:K]
                top_d, top_i = cd[o], ci[o]
        out_ids[qn, :len(top_i)] = top_i
        out_d[qn, :len(top_d)] = top_d
    return out_ids, out_d, st


def search_sharded(shards, Q, K, nprobe, delta_d, alpha, seed=True, exchanges=2, method="bsa_p", **kw):
    """The database split over S shards: every shard searches its own sub-lists of
    the same probed lists with the same calibration, and the local top-K lists are merged by
    (dist, id). seed=True is R32's schedule: per-shard c0 = ⌈4K/S⌉ (the shards' epoch-0 prefixes
    together are as long as the single index's); the shards run epoch 0, then epoch 1, …, epoch
    `exchanges`−1 as separate phases and, after each, exchange their top-K lists (all-gather +
    merge): from epoch 1 on every shard tests against τ_e = min(its own K-th, the merged K-th of
    the last exchange); the remaining epochs run as one last phase. The merged K-th is the K-th
    distance of a subset of the candidates the search has seen, so it bounds the global queue's
    τ from above. seed=False: independent shards (each τ is its own K-th, c0 = 4K). S = 1 with
    seed reduces to `search`. Returns (ids, dists, per-shard stats)."""
    S = len(shards)
    if not seed:
        parts, sts = [], []
        for sh in shards:
            i, d, st = search(sh, Q, K, nprobe, delta_d, alpha, method=method, **kw)
            parts.append((i, d)); sts.append(st)
        return (*merge_shards(parts, K), sts)
    c0 = -(-4 * K // S)
    edges = list(range(exchanges + 1)) + [1 << 30]
    tops, cap, sts = [None] * S, None, [None] * S
    for a, b in zip(edges[:-1], edges[1:]):
        for s, sh in enumerate(shards):
            i, d, st = search(sh, Q, K, nprobe, delta_d, alpha, c0=c0, method=method, epochs=(a, b),
                              init_top=tops[s], tau_cap=cap, **kw)
            tops[s] = (i, d)
            if sts[s] is None:
                sts[s] = st
            else:
                for k in ("tested", "dims_scanned", "survivors"):
                    sts[s][k] += st[k]
                sts[s]["pruned_at_step"] = sts[s]["pruned_at_step"] + st["pruned_at_step"]
        if b < (1 << 30):  # exchange: merged K-th of the shards' queues
            mi, md = merge_shards(tops, K)
            cap = np.where(mi[:, K - 1] >= 0, md[:, K - 1], np.inf)
    return (*merge_shards(tops, K), sts)


def exact_ivf(index, X, Q, K, nprobe):
    """IVF without any DCO: exact raw-space distances of every candidate of the probed lists
    (P:L174-175), (dist, id) order. Used to pin search(α=0)."""
    Q = np.atleast_2d(Q)
    off, row_id = index["off"], index["row_id"]
    ids = np.full((Q.shape[0], K), -1, dtype=np.int64); ds = np.full((Q.shape[0], K), np.inf)
    for qn, q in enumerate(Q):
        pr = probe(q, index["centroids"], nprobe)
        cand = np.concatenate([row_id[off[l]:off[l + 1]] for l in pr])
        d = sqdist_seq(X[cand - index["id_base"]], q)
        o = order_by_dist_id(d, cand)[:K]
        ids[qn, :len(o)], ds[qn, :len(o)] = cand[o], d[o]
    return ids, ds


def merge_shards(parts, K):
    """Combine per-shard top-K lists by (dist, id) (local top-K → all-gather →
    merge). parts: list of (ids[nq,K], dists[nq,K])."""
    nq = parts[0][0].shape[0]
    ids = np.full((nq, K), -1, dtype=np.int64); ds = np.full((nq, K), np.inf)
    for q in range(nq):
        ci = np.concatenate([p[0][q] for p in parts]); cd = np.concatenate([p[1][q] for p in parts])
        valid = ci >= 0
        ci, cd = ci[valid], cd[valid]
        o = order_by_dist_id(cd, ci)[:K]
        ids[q, :len(o)], ds[q, :len(o)] = ci[o], cd[o]
    return ids, ds


def recall_at_k(found: np.ndarray, truth: np.ndarray, K: int) -> float:
    """recall@K = |T ∩ G| / K averaged over queries."""
    tot = 0
    for f, g in zip(found, truth):
        tot += len(set(f[:K].tolist()) & set(g[:K].tolist()))
    return tot / (K * len(found))


# ----------------------------------------------------------------------------- NEXT-2 Exp-7
def estimate_dists(Xr: np.ndarray, q_rot: np.ndarray, d: int, estimator: str = "partial") -> np.ndarray:
    """Exp-7 / Table III's estimates of every row's squared distance from its first d rotated
    dims (R27). "partial": P_d = Σ_{i<d} (x_i − q_i)² — the "PCA" column in the
    PCA basis, the "Rand" column in a random orthogonal basis (its (D/d) JL scale, is
    a constant factor and does not change the ranking). "residual": the BSA-res estimate of Eq. 2
    (P:L289-297), dis'_d = P_d + ‖x_r‖² + ‖q_r‖² with x_r, q_r the dims i ≥ d — the exact distance
    minus the dropped cross term −2⟨q_r, x_r⟩ (Eq. 3's m·σ margin is per query: no effect on a
    ranking). fp64."""
    Xr = np.asarray(Xr, F64)
    q = np.asarray(q_rot, F64)
    e = np.sum((Xr[:, :d] - q[:d]) ** 2, axis=1)
    if estimator == "residual":
        e = e + np.sum(Xr[:, d:] ** 2, axis=1) + float(np.sum(q[d:] ** 2))
    elif estimator != "partial":
        raise ValueError(estimator)
    return e


def estimate_knn(index, Q: np.ndarray, d: int, K: int, estimator: str = "partial"):
    """Flat scan by the d-dim estimate (Exp-7): per query the K rows with the smallest estimate,
    (estimate, id) order (R12). Uses the index's rotation and fp64 rotated base."""
    Q = np.atleast_2d(Q)
    Qr = rotate(Q, index["mean"], index["R"])
    gid = np.arange(index["Xr"].shape[0], dtype=np.int64) + index["id_base"]
    ids = np.empty((Q.shape[0], K), dtype=np.int64)
    est = np.empty((Q.shape[0], K), dtype=F64)
    for i, q in enumerate(Qr):
        e = estimate_dists(index["Xr"], q, d, estimator)
        o = order_by_dist_id(e, gid)[:K]
        ids[i], est[i] = gid[o], e[o]
    return ids, est


# ----------------------------------------------------------------------------- NEXT-3 BSA-q (§V-B)
# The data-driven correction on a QUANTIZATION distance: dis' = the asymmetric
# distance (ADC) from the query to the product-quantized candidate, OPQ rotation, one
# extra feature = the candidate's distance to its own quantized reconstruction.
# Readings R28-R30: OPQ trained on a strided sample of 65,536 rows,
# PCA-initialised, alternating per-subspace k-means and orthogonal Procrustes; m = D/4 subspaces
# (D/8 for GIST-like data), 8-bit codes; one classifier (PQ has no incremental
# refinement: survivors get the exact distance), target recall r (α_s = α).
PQ_K = 256  # 2^nbits codewords per subspace, nbits = 8


def pq_subspaces(D: int, gist_like: bool = False) -> int:
    """m = D/8 for GIST, D/4 for the other datasets."""
    return D // 8 if gist_like else D // 4


def pq_kmeans(Z: np.ndarray, iters: int, init: np.ndarray | None = None) -> np.ndarray:
    """One subspace's codebook: k-means with 256 centroids on the rows of Z (R28): init = the first
    256 rows (the sample is strided, so they are spread over the base) unless `init` is given,
    `iters` Lloyd iterations with exact assignment (`assign`: fp64 sequential sums, lower code on
    ties), centroid = fp64 mean rounded to fp32, an empty cell keeps its centroid."""
    C = (np.asarray(Z[:PQ_K], np.float64) if init is None else np.asarray(init, np.float64)).astype(np.float32)
    for _ in range(iters):
        a = assign(Z, C)
        sums = np.zeros((PQ_K, Z.shape[1]))
        np.add.at(sums, a, np.asarray(Z, np.float64))
        cnt = np.bincount(a, minlength=PQ_K)
        nz = cnt > 0
        C[nz] = (sums[nz] / cnt[nz, None]).astype(np.float32)
    return C


def pq_encode(Xr: np.ndarray, C: np.ndarray):
    """PQ code of each rotated row: per subspace j the nearest codeword of C[j]
    (256 x D/m), exact fp64 sequential sums, ties to the lower code (R30); and the row's distance
    to its reconstruction e = ||x − x̂||² (the extra feature), fp64.
    Returns codes (n x m uint8), e (n fp64)."""
    Xr = np.asarray(Xr)
    m, _, ds = C.shape
    codes = np.zeros((Xr.shape[0], m), np.uint8)
    e = np.zeros(Xr.shape[0])
    for j in range(m):
        Z = Xr[:, j * ds:(j + 1) * ds]
        a = assign(Z, C[j])
        codes[:, j] = a
        diff = np.asarray(Z, np.float64) - C[j][a].astype(np.float64)
        e += np.sum(diff * diff, axis=1)
    return codes, e


def procrustes(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Orthogonal R minimising Σ_rows ||R x − y||² (OPQ's rotation step): with
    M = Σ x yᵀ = U S Vᵀ, R = V Uᵀ."""
    M = np.asarray(X, np.float64).T @ np.asarray(Y, np.float64)
    U, _, Vt = np.linalg.svd(M)
    return Vt.T @ U.T


def opq_train(X: np.ndarray, m: int, n_train: int = 65536, iters: int = 8, km_iters: int = 4,
              final_iters: int = 10):
    """OPQ on a strided sample of min(N, 65,536) rows, R28: centred on the
    sample mean; R initialised to the sample's PCA rotation (fit_rotation); `iters` rounds of
    {per-subspace k-means (`km_iters` Lloyd iterations, warm-started), R ← procrustes(x − μ,
    reconstruction)}; then `final_iters` Lloyd iterations of the codebooks on the final rotation.
    Returns (mean[D], R[D,D] rows = directions, C[m, 256, D/m] fp32)."""
    X = np.asarray(X)
    n, D = X.shape
    ds = D // m
    S = X[strided_ids(n, min(n, n_train))]
    mean, R, _ = fit_rotation(S, sample_size=S.shape[0])
    Xc = S.astype(np.float64) - mean
    C = None
    for _ in range(iters):
        Z = Xc @ R.T
        C = np.stack([pq_kmeans(Z[:, j * ds:(j + 1) * ds], km_iters, None if C is None else C[j])
                      for j in range(m)])
        codes, _ = pq_encode(Z, C)
        Y = np.concatenate([C[j][codes[:, j]].astype(np.float64) for j in range(m)], axis=1)
        R = procrustes(Xc, Y)
    Z = Xc @ R.T
    C = np.stack([pq_kmeans(Z[:, j * ds:(j + 1) * ds], final_iters, None if C is None else C[j])
                  for j in range(m)])
    return mean, R, C


def adc_lut(q_rot: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Asymmetric distance look-up table: lut[j, c] = ||q_j − C[j, c]||², fp64."""
    m, _, ds = C.shape
    q = np.asarray(q_rot, np.float64)
    lut = np.zeros((m, PQ_K))
    for j in range(m):
        d = C[j].astype(np.float64) - q[j * ds:(j + 1) * ds]
        lut[j] = np.sum(d * d, axis=1)
    return lut


def adc(lut: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """ADC distance of coded rows: Σ_j lut[j, code_j] (m table look-ups)."""
    return lut[np.arange(lut.shape[0])[None, :], np.asarray(codes, np.int64)].sum(axis=1)


def logistic_irls_multi(F: np.ndarray, tau: np.ndarray, y: np.ndarray, ridge: float = 1e-8,
                        max_iter: int = 100, tol: float = 1e-12):
    """logistic_irls with several approximate-distance features (ADC distance and the
    distance to the quantized centroid, plus τ): the BCE minimiser by damped Newton/IRLS on
    standardised features (R3). Returns (m[k], β, ok): the model m·f + β > τ, m_i = −w_i/w_τ.
    Flag (R29): w_τ ≥ 0, a non-finite weight, or m_0 (the ADC slope) ≤ 0 → (e_0, 0, False)."""
    F = np.atleast_2d(np.asarray(F, F64).T).T
    n, k = F.shape
    tau = np.asarray(tau, F64); y = np.asarray(y, F64)
    mf, sf = F.mean(axis=0), F.std(axis=0)
    sf = np.where(sf > 0, sf, 1.0)
    mt, st = tau.mean(), tau.std()
    st = st if st > 0 else 1.0
    A = np.concatenate([np.ones((n, 1)), (F - mf) / sf, ((tau - mt) / st)[:, None]], axis=1)
    reg = np.r_[0.0, np.full(k + 1, ridge)]

    def loss(w):
        z = A @ w
        return float(np.sum(np.logaddexp(0.0, z) - y * z) + 0.5 * np.sum(reg * w * w))

    w = np.zeros(k + 2)
    cur = loss(w)
    for _ in range(max_iter):
        z = A @ w
        p = 0.5 * (1.0 + np.tanh(0.5 * z))
        g = A.T @ (y - p) - reg * w
        H = (A * (p * (1 - p))[:, None]).T @ A + np.diag(reg)
        step = np.linalg.solve(H, g)
        t = 1.0
        for _h in range(30):
            nw = w + t * step
            nl = loss(nw)
            if nl <= cur:
                break
            t *= 0.5
        w, cur = nw, nl
        if np.max(np.abs(t * step)) < tol:
            break
    wf, wt = w[1:k + 1] / sf, w[k + 1] / st
    b = w[0] - np.sum(w[1:k + 1] * mf / sf) - w[k + 1] * mt / st
    unit = np.r_[1.0, np.zeros(k - 1)]
    if not (wt < 0) or not np.all(np.isfinite(wf)) or not np.isfinite(wt):
        return unit, 0.0, False
    mv = -wf / wt
    if not (mv[0] > 0) or not np.all(np.isfinite(mv)):
        return unit, 0.0, False
    return mv, float(-b / wt), True


def build_index_q(X, centroids, mean, R, C, id_base=0):
    """build_index plus the PQ encoding of the rotated base (codes, reconstruction errors)."""
    idx = build_index(X, centroids, mean, R, id_base=id_base)
    idx["pq"] = np.asarray(C, np.float32)
    idx["codes"], idx["pq_err"] = pq_encode(idx["Xr"], idx["pq"])
    return idx


def calibrate_q(X, index, Qc, K, n_neg=50, nprobe_neg=0, seed=0):
    """§V-A correction on the ADC distance (BSA-q): the calibration pairs of
    `calibration_pairs` (R14-R16), features (ADC dis', e) and τ, the logistic fit (R3/R29), and
    v = sort_desc(τ − m_1·dis' − m_2·e) over the Label-0 pairs, from which search derives β'."""
    qi, ids, lab, tau = calibration_pairs(X, index, Qc, K, n_neg, nprobe_neg, seed)
    Qr = rotate(Qc, index["mean"], index["R"])
    rows = ids - index["id_base"]
    dis = np.array([adc(adc_lut(Qr[q], index["pq"]), index["codes"][r:r + 1])[0] for q, r in zip(qi, rows)])
    e = index["pq_err"][rows]
    mv, _, ok = logistic_irls_multi(np.stack([dis, e], axis=1), tau, lab)
    v = np.sort(tau[lab == 0] - mv[0] * dis[lab == 0] - mv[1] * e[lab == 0])[::-1]
    return {"m": mv, "v": v, "ok": ok, "n0": int(np.sum(lab == 0)), "K": K}


def search_q(index, Q, K, nprobe, alpha, c0=None, log=False):
    """IVF search with the quantization-distance correction (BSA-q, O5 with one classifier):
    per candidate of the probed lists (probe order), dis' = ADC(q̃, code), prune iff τ_e < ∞ and
    m_1·dis' + m_2·e + β' > τ_e with β' = v[k−1], k = clamp(⌈(1−α)·n0⌉, 1, n0) (R4; one classifier,
    α_s = α, R29); survivors get the exact distance P_D over the rotated vectors and enter
    the top-K; τ frozen per epoch (R13). α = 0 disables pruning. Logged dims: 0 for an ADC prune
    (only the code was read), D for a survivor."""
    Q = np.atleast_2d(Q)
    D = Q.shape[1]
    cal = index["calq"]
    beta = -np.inf if alpha == 0 else beta_from_v(cal["v"], alpha)
    m1, m2 = cal["m"]
    off, row_id, Xr, base = index["off"], index["row_id"], index["Xr"], index["id_base"]
    codes, err = index["codes"], index["pq_err"]
    out_ids = np.full((Q.shape[0], K), -1, dtype=np.int64)
    out_d = np.full((Q.shape[0], K), np.inf)
    st = {"tested": 0, "survivors": 0, "pruned": 0, "n_epochs": 0, "candidates": []}
    Qr = rotate(Q, index["mean"], index["R"])
    for qn in range(Q.shape[0]):
        pr = probe(Q[qn], index["centroids"], nprobe)
        cand = np.concatenate([row_id[off[l]:off[l + 1]] for l in pr])
        lut = adc_lut(Qr[qn], index["pq"])
        top_d = np.zeros(0); top_i = np.zeros(0, dtype=np.int64)
        st["tested"] += len(cand)
        bounds = epoch_bounds(len(cand), K, c0)
        st["n_epochs"] = max(st["n_epochs"], len(bounds) - 1)
        for e in range(len(bounds) - 1):
            tau = top_d[K - 1] if len(top_d) >= K else np.inf
            ids = cand[bounds[e]:bounds[e + 1]]
            rows = ids - base
            keep = np.ones(len(ids), dtype=bool)
            margin = np.full(len(ids), np.inf)
            if np.isfinite(tau) and np.isfinite(beta):
                score = m1 * adc(lut, codes[rows]) + m2 * err[rows] + beta
                keep = ~(score > tau)
                scale = np.abs(score - beta) + abs(beta) + tau
                margin = np.abs(score - tau) / scale
            st["pruned"] += int((~keep).sum())
            st["survivors"] += int(keep.sum())
            dis = np.sum((Xr[rows[keep]] - Qr[qn]) ** 2, axis=1)
            if log:
                st["candidates"].append((np.full(len(ids), qn), ids.copy(), np.where(keep, D, 0), margin))
            cd = np.concatenate([top_d, dis])
            ci = np.concatenate([top_i, ids[keep]])
            o = order_by_dist_id(cd, ci)[:K]
            top_d, top_i = cd[o], ci[o]
        out_ids[qn, :len(top_i)] = top_i
        out_d[qn, :len(top_d)] = top_d
    return out_ids, out_d, st


# ----------------------------------------------------------------------------- NEXT-4 graph refinement
# HNSW (M = 16, efConstruction = 500) with the DCO in its base-layer
# refinement. Readings R33-R35: the base layer is a fixed-degree graph of M0 = 2M =
# 32 neighbours per node chosen from the node's nearest candidates by HNSW's neighbour-selection
# heuristic; the upper layers only supply the entry point, read as the node nearest to the mean;
# the search is HNSW's best-first base-layer search with a result queue of size ef (N^{ef}), the
# DCO tests a neighbour against τ = the queue's max, frozen while one node is expanded.
def graph_neighbors(X: np.ndarray, pool: np.ndarray, pool_d: np.ndarray, M0: int = 32) -> np.ndarray:
    """HNSW's neighbour-selection heuristic (R33): walk each node's candidate pool in (dist, id)
    order and keep a candidate e iff it is closer to the node than to every kept neighbour r
    (dist(e, node) < dist(e, r)); then fill up to M0 with the nearest discarded candidates (HNSW's
    keepPrunedConnections). pool / pool_d: n x P candidate ids (exact nearest first, the node
    itself excluded) and their distances to the node. Returns n x M0 int64 (−1 padded)."""
    n = pool.shape[0]
    out = np.full((n, M0), -1, dtype=np.int64)
    for i in range(n):
        cand = [(int(e), float(de)) for e, de in zip(pool[i], pool_d[i]) if e >= 0]
        if not cand:
            continue
        ce = np.array([e for e, _ in cand])
        # distances among the pool members: sequential fp64 sums over the dims (R20's rule)
        A = np.asarray(X[ce], F64)
        pair = np.zeros((len(ce), len(ce)))
        for j in range(A.shape[1]):
            t = A[:, j][:, None] - A[:, j][None, :]
            pair += t * t
        kept, dropped = [], []
        for a, (e, de) in enumerate(cand):
            if len(kept) < M0 and all(de < pair[a, r] for r in kept):
                kept.append(a)
            else:
                dropped.append(a)
        sel = [int(ce[a]) for a in (kept + dropped)[:M0]]
        out[i, :len(sel)] = sel
    return out


def build_graph(X: np.ndarray, M0: int = 32, P: int = 64):
    """The base-layer graph (R33) from EXACT candidate pools: each node's P nearest other nodes
    (fp64, (dist, id) order), the heuristic, and the entry point = the node nearest to the mean
    of the base (ties → lower id). Returns (nbrs n x M0, entry)."""
    n = X.shape[0]
    P = min(P, n - 1)
    ids, d = brute_force_knn(X, X, P + 1)
    pool = np.zeros((n, P), np.int64); pool_d = np.zeros((n, P))
    for i in range(n):
        keep = ids[i] != i
        pool[i], pool_d[i] = ids[i][keep][:P], d[i][keep][:P]
    mu = np.asarray(X, F64).mean(axis=0)
    entry = int(order_by_dist_id(sqdist_seq(X, mu), np.arange(n))[0])
    return graph_neighbors(X, pool, pool_d, M0), entry


def graph_search(index, Q, K, ef, delta_d, alpha, log=False):
    """HNSW base-layer refinement with the DCO (R34): result queue W of size ef, candidate queue C;
    start at the entry point (exact distance); repeatedly take the nearest unexpanded c of C, stop
    once W holds ef entries and dist(c) > max W; expand c: every unvisited neighbour u is tested
    with the BSA-p cascade against τ = max W (∞ while |W| < ef), FROZEN during this expansion
    (prune iff m1_d·P_d + β'_d > τ at d = Δd, 2Δd, …); a survivor's exact
    distance P_D enters C and W (in (dist, id) order) if |W| < ef or it is below max W; W keeps its
    ef best. Returns the first K of W (ids, dists) and counters. α = 0: no pruning (plain HNSW
    refinement). index: build_index(...) over the rows in id order plus "nbrs", "entry". The
    entry point (R33): with an IVF (nlist > 1) the lowest-id node of the query's nearest non-empty
    list — the coarse quantizer stands in for HNSW's upper layers — else index["entry"]."""
    Q = np.atleast_2d(Q)
    D = Q.shape[1]
    ns = D // delta_d
    if alpha == 0:
        m, b = np.ones(ns - 1), np.full(ns - 1, -np.inf)
    else:
        m, b = step_table(index["cal"], D, delta_d, alpha)
    steps = np.arange(1, ns) * delta_d
    Xr, nbrs, base = index["Xr"], index["nbrs"], index["id_base"]
    Qr = rotate(Q, index["mean"], index["R"])
    out_i = np.full((Q.shape[0], K), -1, np.int64); out_d = np.full((Q.shape[0], K), np.inf)
    st = {"tested": 0, "dims_scanned": 0, "survivors": 0, "expansions": 0,
          "pruned_at_step": np.zeros(ns, np.int64), "candidates": []}
    nlist = len(index["off"]) - 1
    for qn in range(Q.shape[0]):
        q = Qr[qn]
        e0 = index["entry"]
        if nlist > 1:  # R33: the entry is the lowest-id node of the query's nearest non-empty IVF list
            for l in probe(Q[qn], index["centroids"], min(nlist, 8)):
                if index["off"][l + 1] > index["off"][l]:
                    e0 = int(index["row_id"][index["off"][l]])
                    break
        d0 = float(np.sum((Xr[e0 - base] - q) ** 2))
        visited = {e0}
        W = [(d0, e0)]
        C = [(d0, e0)]
        st["tested"] += 1; st["dims_scanned"] += D; st["survivors"] += 1
        if log:
            st["candidates"].append((np.array([qn]), np.array([e0]), np.array([D]), np.array([np.inf])))
        while C:
            c = min(C)
            C.remove(c)
            if len(W) >= ef and c[0] > max(W)[0]:
                break
            st["expansions"] += 1
            tau = max(W)[0] if len(W) >= ef else np.inf
            us = [int(u) for u in nbrs[c[1] - base] if u >= 0 and int(u) not in visited]
            for u in us:
                visited.add(u)
            if not us:
                continue
            U = np.array(us, np.int64)
            P = np.cumsum((Xr[U - base] - q) ** 2, axis=1)
            dims = np.full(len(U), D)
            keep = np.ones(len(U), bool)
            margin = np.full(len(U), np.inf)
            if np.isfinite(tau) and ns > 1:
                score = m[None, :] * P[:, steps - 1] + b[None, :]
                test = score > tau
                anyp = test.any(axis=1)
                first = np.argmax(test, axis=1)
                keep = ~anyp
                dims[anyp] = steps[first[anyp]]
                np.add.at(st["pruned_at_step"], first[anyp] + 1, 1)
                if log:
                    scale = np.abs(m[None, :] * P[:, steps - 1]) + np.abs(b[None, :]) + tau
                    rel = np.abs(score - tau) / scale
                    last = np.where(anyp, first, ns - 2)
                    upto = np.arange(ns - 1)[None, :] <= last[:, None]
                    margin = np.where(upto, rel, np.inf).min(axis=1)
            st["tested"] += len(U); st["dims_scanned"] += int(dims.sum()); st["survivors"] += int(keep.sum())
            if log:
                st["candidates"].append((np.full(len(U), qn), U.copy(), dims.copy(), margin))
            for du, u in sorted(zip(P[keep, D - 1].tolist(), U[keep].tolist())):
                if len(W) < ef or (du, u) < max(W):
                    C.append((du, u))
                    W.append((du, u))
                    if len(W) > ef:
                        W.remove(max(W))
        W.sort()
        for j, (dd, u) in enumerate(W[:K]):
            out_i[qn, j], out_d[qn, j] = u, dd
    return out_i, out_d, st
