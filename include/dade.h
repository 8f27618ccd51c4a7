/*
 * dade.h — C ABI of the B200-native DADE hot path (arxiv 2404.16322, "Effective and General
 * Distance Computation for Approximate Nearest Neighbor Search"; PAPER.md = /root/reference/PAPER.md).
 *
 * What the library computes (citations are PAPER.md lines, "R<n>" = DESIGN.md §3 readings):
 *   - KNN under squared Euclidean distance dis(p,q) = ||p-q||^2
 *   - IVF: k-means buckets, query probes the N^probe nearest centroids
 *   - PCA rotation x~ = R(x - mu) (Theorem 1)
 *   - refinement with result queue Q of size K, tau = its max
 *   - BSA-p estimator dis'_d = partial PCA distance over the first d dims
 *   - data-driven correction: prune iff m1_d * dis'_d + beta'_d > tau
 *     one classifier per projected dimension d (cascade)
 *     beta'_d calibrated to Label-0 recall r_i = 1 - (1-r)/(D/Delta_d)
 *   - tau frozen within geometric epochs of the candidate stream (R13)
 *
 * Conventions for every entry point
 *   - Return: dade_status; DADE_OK (0) on success. On error the index state is unchanged and
 *     dade_last_error() returns a thread-local message. No C++ exception crosses the ABI.
 *   - Pointers are plain: "device" = CUDA device memory of the index's device, "host" = host memory.
 *     Arrays are dense, row-major, 0-based. Inputs are borrowed for the duration of the call;
 *     the library copies everything it keeps. Outputs are caller-allocated.
 *   - All device work is ordered on the stream given to dade_create. Build calls (fit/build/
 *     calibrate) and calls returning host data synchronise before returning; dade_search is
 *     asynchronous unless `stats` is non-NULL.
 *   - One host thread per dade_index at a time.
 *   - Global ids are int64 in the ABI and must be < 2^31 (kernels carry 32-bit ids).
 *   - D must be a multiple of 16 (the layout block width B_L = 16 dims = 64 B rows); else
 *     DADE_ERR_UNSUPPORTED.
 */
#ifndef DADE_H
#define DADE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dade_index dade_index; /* opaque; owns the device memory of ONE GPU (one shard) */

typedef enum {
  DADE_OK = 0,
  DADE_ERR_ARG = 1,        /* bad scalar argument (K, nprobe, delta_d, significance, NULL ptr) */
  DADE_ERR_SHAPE = 2,      /* dimension mismatch */
  DADE_ERR_STATE = 3,      /* call order violated (e.g. search before build, alpha>0 without calibration) */
  DADE_ERR_NONFINITE = 4,  /* NaN/Inf in an input array */
  DADE_ERR_OOM = 5,        /* device allocation failed */
  DADE_ERR_CUDA = 6,       /* CUDA runtime error */
  DADE_ERR_NCCL = 7,       /* NCCL error (multi-rank calls after dade_set_comm), or libnccl missing */
  DADE_ERR_UNSUPPORTED = 8 /* valid but outside what the kernels implement (D%16, K>256, ...) */
} dade_status;

#define DADE_MAX_STEPS 64
#define DADE_MAX_K 256

/* Per-search counters (P:L3964-3974 pruning rate; Exp-6 "dimensions scanned"). */
typedef struct {
  int64_t tested;                         /* candidates entering the DCO (sum of probed list sizes) */
  int64_t survivors;                      /* candidates that reached d = D (exact distance computed) */
  int64_t dims_scanned;                   /* sum over tested candidates of dims read (d at prune, else D) */
  int64_t pruned_at_step[DADE_MAX_STEPS]; /* [s] = pruned by the classifier at d = s*delta_d, s>=1 */
  int32_t n_steps;                        /* D / delta_d */
  int32_t n_epochs;                       /* epochs of the longest candidate stream */
  float ms_rotate, ms_probe, ms_scan, ms_total; /* CUDA-event times of the stages */
} dade_stats;

/* Thread-local message describing the last failing call ("" if none). */
const char* dade_last_error(void);

/* Create an index for dimension D on CUDA `device`; `cuda_stream` is a cudaStream_t (NULL =
 * the legacy default stream). Errors: ARG (D<=0), UNSUPPORTED (D%16 != 0 or D > 4096), CUDA. */
dade_status dade_create(int device, void* cuda_stream, int D, dade_index** out);
dade_status dade_destroy(dade_index* idx);

/* ---------------------------------------------------------------- a0 fit_rotation
 * PCA of the rows of X (device, n x D fp32): strided sample ids floor(k*n/ns), k < ns,
 * ns = min(n, sample_size>0 ? sample_size : 1,000,000) (R17); mu = sample mean,
 * Sigma = (Xs-mu)^T(Xs-mu)/ns (fp64 on the GPU), eigendecomposition in fp64 on the host;
 * R rows = eigenvectors by descending eigenvalue, sign: largest-|component| positive (R18).
 * Errors: ARG, NONFINITE, CUDA. */
dade_status dade_fit_rotation(dade_index* idx, const float* X, int64_t n, int64_t sample_size);

/* Multi-rank form of fit_rotation (each rank owns global ids [id_base, id_base+n) of a base of
 * n_total rows; the caller all-reduces the fp64 partials between the calls):
 *   1. dade_pca_mean_partial  -> sum[D] (host), count (host) of the sampled rows this rank owns
 *   2. dade_pca_cov_partial   -> cov_sum[D*D] (host) = sum over owned sampled rows of (x-mean)(x-mean)^T
 *   3. dade_set_rotation_from_cov(mean, cov_sum, count) -> eigendecomposition as above. */
dade_status dade_pca_mean_partial(dade_index* idx, const float* X, int64_t n, int64_t id_base,
                                  int64_t n_total, int64_t sample_size, double* sum, int64_t* count);
dade_status dade_pca_cov_partial(dade_index* idx, const float* X, int64_t n, int64_t id_base,
                                 int64_t n_total, int64_t sample_size, const double* mean,
                                 double* cov_sum);
dade_status dade_set_rotation_from_cov(dade_index* idx, const double* mean, const double* cov_sum,
                                       int64_t count);

/* Host copies of the rotation: mean[D], R[D*D] (row-major, rows = directions), eigvals[D].
 * dade_set_rotation installs a rotation (host arrays; eigvals may be NULL: then BSA-res, which
 * needs them, returns STATE). Installing a rotation — by either setter or by fit — discards the
 * IVF layout and the calibration built in the previous basis (build_ivf / set_ivf again).
 * Errors: ARG (NULL), NONFINITE. */
dade_status dade_get_rotation(const dade_index* idx, double* mean, double* R, double* eigvals);
dade_status dade_set_rotation(dade_index* idx, const double* mean, const double* R,
                              const double* eigvals);

/* ---------------------------------------------------------------- a1+a2 build_ivf
 * X: device n x D fp32 raw rows with global ids [id_base, id_base+n). Requires a rotation.
 * centroids: device nlist x D fp32 raw-space centroids, or NULL -> k-means (R19: strided sample
 * of min(n, 64*nlist) rows, init = first nlist sampled rows, `kmeans_iters` Lloyd iterations).
 * assign(i) = argmin_c sum_j (x_ij - c_cj)^2 evaluated EXACTLY as an fp64 sequential sum, ties to
 * the lower c (R20; fp32 tile filter + fp64 certification). Lists hold ids ascending. The rotated
 * rows x~ = R(x - mu) (fp64 accumulation, stored fp32) are written dimension-blocked and
 * list-major: block b (dims 16b..16b+15) is an n x 16 matrix whose row p is list-major position p.
 * Errors: ARG (nlist<1 or nlist>n), STATE (no rotation), NONFINITE, OOM, CUDA. */
dade_status dade_build_ivf(dade_index* idx, const float* X, int64_t n, int64_t id_base, int nlist,
                           const float* centroids_or_null, int kmeans_iters);

/* Host copies of the IVF: off[nlist+1] list offsets, row_id[n] global id of list-major position p,
 * assign[n] (by local row i = id - id_base), centroids[nlist*D]. Any pointer may be NULL. */
dade_status dade_get_ivf(const dade_index* idx, int64_t* off, int64_t* row_id, int32_t* assign,
                         float* centroids);
/* Sizes: *n rows, *nlist lists (either may be NULL). */
dade_status dade_get_sizes(const dade_index* idx, int64_t* n, int* nlist);
/* Host copy of the blocked layout as list-major rows: Xrot[n*D] (row p = x~ of row_id[p]). */
dade_status dade_get_layout(const dade_index* idx, float* Xrot);
/* Inject a ready IVF + layout (parity tests, or an index built elsewhere) in the
 * CURRENT rotation's basis: Xrot device n x D fp32 ROTATED rows x~ = R(x - mu) in list-major order
 * (row p = x~ of row_id[p]; copied into the blocked layout); row_id host n int64 global ids,
 * off host nlist+1 int64 list offsets (lists hold ids ascending, ids = a permutation of
 * [id_base, id_base+n), as dade_get_ivf returns them); centroids device nlist x D fp32 raw-space
 * (the probe's space). Discards the calibration. Errors: STATE (no rotation), ARG
 * (inconsistent off / row_id, ids >= 2^31), NONFINITE, OOM, CUDA. */
dade_status dade_set_ivf(dade_index* idx, const float* Xrot, int64_t n, int64_t id_base, const int64_t* row_id,
                         const int64_t* off, int nlist, const float* centroids);

/* ---------------------------------------------------------------- a3 calibrate
 * X: device n x D, the raw rows given to dade_build_ivf (the index keeps only the rotated layout).
 * Qc: device nq x D raw calibration queries. For each: exact K NN over this index's base
 * (Label 0; tau_q = K-th NN distance, R14); Label 1 = the n_neg non-KNN candidates of
 * its nprobe_neg probed lists (whole base if 0 or nlist==1) with the smallest
 * SplitMix64(seed ^ (q<<32 | id)) (R16). For d = 16, 32, ..., D-16: m1_d from the logistic
 * (BCE) fit on (P_d, tau) (R3) and v_d = sort_desc(tau - m1_d*P_d) over Label-0 pairs.
 * Errors: ARG (K<1, K>n, K>DADE_MAX_K, n_neg<0), STATE (no IVF), NONFINITE, CUDA. */
dade_status dade_calibrate(dade_index* idx, const float* X, const float* Qc, int nq, int K,
                           int n_neg, int nprobe_neg, uint64_t seed);
/* Host copy of the calibration table: m1[n_cls], v[n_cls*n0] (row s = d = 16(s+1)), n_cls = D/16-1.
 * Pass NULL arrays to query K, n0, n_cls only. */
dade_status dade_get_calibration(const dade_index* idx, int* K, int* n0, int* n_cls, double* m1,
                                 double* v);
dade_status dade_set_calibration(dade_index* idx, int K, int n0, int n_cls, const double* m1,
                                 const double* v);

/* ---------------------------------------------------------------- a4..a8 search
 * Q: device nq x D raw queries; ids (int64) / dists (fp32 squared L2) device nq x K, ascending by
 * (dist, id); missing slots -> id -1, dist +inf. delta_d: any positive multiple of 16 dividing D
 * (D / delta_d <= DADE_MAX_STEPS).
 * significance alpha in [0,1): alpha = 0 disables pruning (exact IVF); alpha > 0 uses
 * beta'_d = v_d[k-1], k = clamp(ceil((1 - alpha*delta_d/D) * n0), 1, n0) (R4, R5).
 * Per query: q~ = R(q-mu) (fp64 accumulation), exact probes (fp64-certified, ties to lower id),
 * candidate stream = probed lists in probe order, epochs [0,4K),[4K,8K),[8K,16K),... with tau
 * frozen per epoch, prune iff m1_d*P_d + beta'_d > tau, survivors' exact P_D enter the top-K.
 * stats may be NULL (then the call is asynchronous on the stream).
 * Errors: ARG, STATE (no IVF; alpha>0 without calibration; K != calibrated K), UNSUPPORTED
 * (K > DADE_MAX_K, D/delta_d > DADE_MAX_STEPS), CUDA. */
dade_status dade_search(dade_index* idx, const float* Q, int nq, int K, int nprobe, int delta_d,
                        double significance, int64_t* ids, float* dists, dade_stats* stats);

/* ---------------------------------------------------------------- NEXT-1: the paper's other DCOs
 * Same scan, different per-step test:
 *   DADE_METHOD_BSA_P      param = significance alpha (== dade_search).
 *   DADE_METHOD_ADSAMPLING param = eps0 > 0: prune iff (D/d) P_d > (1 + eps0/sqrt(d))^2 tau — the
 *       ADSampling hypothesis test (linear form P:L3937; R8). Meaningful on a RANDOM
 *       orthogonal rotation (install it with dade_set_rotation); eps0 = 2.1 in the paper.
 *   DADE_METHOD_BSA_RES    param = multiplier m > 0: prune iff P_d + ||x_r||^2 + ||q_r||^2 - m sigma_d
 *       > tau, sigma_d^2 = 4 sum_{i>=d} q~_i^2 lambda_i (Alg. 2, Eq. 3, R6);
 *       lambda = the rotation's eigenvalues; m = 8 in the paper.
 * Errors: as dade_search; ARG if param <= 0 for ADSAMPLING / BSA_RES or method unknown. */
#define DADE_METHOD_BSA_P 0
#define DADE_METHOD_ADSAMPLING 1
#define DADE_METHOD_BSA_RES 2
#define DADE_METHOD_BSA_Q 3   /* NEXT-3, see the BSA-q section below; param = significance alpha */
dade_status dade_search_method(dade_index* idx, const float* Q, int nq, int K, int nprobe, int delta_d,
                               int method, double param, int64_t* ids, float* dists, dade_stats* stats);

/* Stage timing without synchronisation: with timing on, every search records CUDA events around
 * a4 (rotation), a5 (probe) and a6-a8 (scan) on the index's stream(s); dade_get_timing waits for
 * the last search's events and returns ms3 = {rotate, probe (both from the search start, they
 * run concurrently), scan} in milliseconds. Errors: STATE (no search recorded), CUDA. */
dade_status dade_set_timing(dade_index* idx, int on);
dade_status dade_get_timing(dade_index* idx, float* ms3);

/* Sharded k-means (R19): this rank's part of one Lloyd step over the GLOBAL strided
 * sample floor(k*n_total/n_km), n_km = min(n_total, 64*nlist). X: device rows [id_base, id_base+n)
 * of the base. centroids: HOST nlist x D fp32 — the sampled rows this rank owns are assigned
 * exactly (R20, lower id on ties) and their fp64 sums / counts are written to sums (host
 * nlist x D) and counts (host nlist); the caller all-reduces them and sets centroid = sum / count
 * rounded to fp32 (empty: keep). centroids == NULL: the init step — sampled rows with sample index
 * < nlist are written to sums[k] (counts[k] = 1), so an all-reduce yields the first nlist sampled
 * rows. Errors: ARG (bad range, nlist), CUDA. */
dade_status dade_kmeans_partial(dade_index* idx, const float* X, int64_t n, int64_t id_base, int64_t n_total,
                                int nlist, const float* centroids, double* sums, int64_t* counts);

/* Sharded calibration: dade_calibrate's steps, each over this rank's shard, for a
 * driver that combines them across ranks (paper_2404_16322_b200/sharded.py):
 *   dade_calib_knn        exact K nearest rows of THIS shard for each calibration query (X: device
 *                         raw rows of the shard), ids global (host nq x K int64), fp64 distances
 *                         (host nq x K) — the caller merges the shards' lists by (dist, id) (R14);
 *   dade_calib_negatives  Label-1 candidates of this shard (R15/R16: rows of the query's nprobe_neg
 *                         probed lists, or the whole shard if 0, not among the GLOBAL knn_ids) with
 *                         the n_neg smallest (SplitMix64(seed ^ (q << 32 | id)), id): keys / ids host
 *                         nq x n_neg, counts host nq — the caller keeps the n_neg smallest overall;
 *   dade_pair_features    P_d at every 16-dim prefix (fp64, from the stored rotated rows) for the
 *                         pairs (pair_q, global pair_id) whose id lies in this shard, zero rows for
 *                         the others: F host npairs x D/16 — the caller sums F over ranks;
 *   dade_fit_calibration  the per-step logistic slope (R3) and sorted thresholds (R4) from the
 *                         pairs' features, tau and labels y (0 = a K-NN, 1 = a negative); installs
 *                         the calibration exactly as dade_calibrate does.
 * dade_calibrate is these four steps on one shard. Errors: ARG, STATE, NONFINITE, CUDA. */
dade_status dade_calib_knn(dade_index* idx, const float* X, const float* Qc, int nq, int K, int64_t* ids,
                           double* dists);
dade_status dade_calib_negatives(dade_index* idx, const float* Qc, int nq, int K, const int64_t* knn_ids,
                                 int n_neg, int nprobe_neg, uint64_t seed, uint64_t* keys, int64_t* ids,
                                 int32_t* counts);
dade_status dade_pair_features(dade_index* idx, const float* Qc, int nq, int npairs, const int32_t* pair_q,
                               const int64_t* pair_id, double* F);
dade_status dade_fit_calibration(dade_index* idx, int K, int npairs, const double* F, const double* tau,
                                 const double* y);

/* Split search (multi-GPU query partitioning): dade_prepare runs a4 + a5 for a block
 * of queries — qrot (device nq x D fp32, q~ = R(q - mu)) and probes (device nq x nprobe int32,
 * exact, ordered by (dist, id)); dade_search_prepared runs a6-a8 on this index's shard for
 * queries prepared anywhere (e.g. on another rank with the same replicated mu, R, centroids,
 * then all-gathered). Results are identical to dade_search / dade_search_method on the same
 * queries. Errors: as dade_search. */
dade_status dade_prepare(dade_index* idx, const float* Q, int nq, int nprobe, float* qrot, int32_t* probes);
dade_status dade_search_prepared(dade_index* idx, const float* qrot, const int32_t* probes, int nq, int K,
                                 int nprobe, int delta_d, int method, double param, int64_t* ids,
                                 float* dists, dade_stats* stats);

/* Same as dade_search with HOST Q/ids/dists: the H2D copy of Q and the D2H copy of the results
 * are part of the call (synchronous; returns when ids/dists are written). The copies run on two
 * copy streams; with DADE_OPT_HOST_CHUNKS = c (default 1) the batch is cut into c chunks pipelined so
 * that chunk c's H2D overlaps the search of chunk c-1 and its D2H the search of chunk c+1 (not
 * the default: measured slower on C2). Each query's result is independent of
 * the chunking. Unchunked batches of >= 4,096 queries copy Q in two halves and rotate + probe
 * each half as it lands (DADE_OPT_HOST_PREP_CHUNKS overrides), then scan once. Pinned host memory
 * gives asynchronous copies;
 * pageable memory works but serialises them. With stats != NULL the batch runs unchunked.
 * Used for the end-to-end (e2e) measurement. Errors: as dade_search. */
dade_status dade_search_host(dade_index* idx, const float* Q_host, int nq, int K, int nprobe,
                             int delta_d, double significance, int64_t* ids_host, float* dists_host,
                             dade_stats* stats);

/* NEXT-2, Exp-7 / Table III: standalone approximation accuracy. A flat scan of the
 * whole index in which each row's distance is ESTIMATED from its first d rotated dimensions
 * (R27): DADE_EST_PARTIAL  est = P_d = ||x~_{:d} - q~_{:d}||^2 (the table's "PCA" column in the
 * PCA basis; its "Rand" column after dade_set_rotation with a random orthogonal R before
 * dade_build_ivf); DADE_EST_RESIDUAL  est = P_d + ||x~_r||^2 + ||q~_r||^2, the BSA-res estimate
 * of Eq. 2 without the per-query m*sigma margin, which does not change the
 * ranking. Returns, per query, the K rows with the smallest estimate, ordered by (fp32 est, id):
 * ids[nq*K] int64 (global ids), est[nq*K] fp32, device. Q: device nq x D fp32 (raw).
 * fp32 arithmetic with the scan's block association (R21); the residual estimate is clamped
 * at 0. Errors: STATE (no IVF / rotation), ARG (d not a multiple of 16 in [16, D], K not in
 * [1, min(n, DADE_MAX_K)], unknown estimator, NULL), NONFINITE, UNSUPPORTED (n >= 2^31). */
#define DADE_EST_PARTIAL 0
#define DADE_EST_RESIDUAL 1
dade_status dade_estimate_knn(dade_index* idx, const float* Q, int nq, int d, int method, int K, int64_t* ids,
                              float* est);

/* Parity run of the search (SURVEY §8(c) "decisions identical outside R21's tie band"): the same
 * search (one warp per query; decisions and results do not depend on the warp split), plus a
 * decision log: for every tested candidate one record of 3 int32 {query, global id, dims read}
 * (dims = s * delta_d if the classifier at step s pruned it, D if it reached the exact distance),
 * in no particular order. log: device log_cap x 3 int32; *log_count (host) = records produced
 * (> log_cap: the rest were dropped). method BSA_P or ADSAMPLING. Synchronous.
 * Errors: as dade_search_method; UNSUPPORTED for BSA_RES. */
dade_status dade_search_log(dade_index* idx, const float* Q, int nq, int K, int nprobe, int delta_d, int method,
                            double param, int64_t* ids, float* dists, int32_t* log, int64_t log_cap,
                            int64_t* log_count);

/* Tuning options of one index (defaults are the measured best; the alternatives exist for A/B
 * measurement and for tests proving every path returns identical results). Errors: ARG (unknown
 * option or value). */
#define DADE_OPT_KNN_PATH 1        /* exact-KNN filter: 0 auto, 1 d_hat matrix, 2 fused (no d_hat), 3 group minima,
                                      4 throughput fused filter on fp16 operands, 5 the same on tf32 (probe_fz.cu),
                                      6 int8 exact-split filter + group-minima select (rotate.cu distance mode) */
#define DADE_OPT_PROBE_PASSES 2    /* tf32 passes of the probe filter: 0 auto (1 if D < 512, else 3), 1, 3 */
#define DADE_OPT_SCAN_WARPS 3      /* warps per query in the scan: 0 auto, 1, 2, 4, 8 */
#define DADE_OPT_SCAN_ORDER 4      /* scan order: 2 (default) longest candidate stream first, 1 grouped by nearest list, 0 as given */
#define DADE_OPT_SCAN_TAIL 5       /* X > 0: last X queries in a concurrent 4-warps-per-query scan */
#define DADE_OPT_HOST_CHUNKS 6     /* dade_search_host: chunks pipelined with the copies (default 1) */
#define DADE_OPT_HOST_PREP_CHUNKS 7 /* dade_search_host: rotation+probe chunks ahead of one scan (0 auto) */
#define DADE_OPT_DHAT_ARES 8       /* 1: A-resident d_hat writer for very wide probe rows */
#define DADE_OPT_SHARD_EXCHANGES 9 /* collective search: top-K exchanges after epochs 0..E-1 (R32; default 2, 0 = none) */
#define DADE_OPT_FZ_STAGES 10      /* fused probe filter (knn_path 4/5): B ring stages (0 auto) */
#define DADE_OPT_FZ_GROUPS 11      /* fused probe filter: epilogue groups of 4 warps (0 auto, 1, 2) */
#define DADE_OPT_FZ_DEBUG 13       /* measurement only: 1/2 add a pipeline-only launch of the fused filter */
#define DADE_OPT_FZ_CPC 14         /* fused probe filter: 8 KB operand chunks per TMA copy (0 auto) */
#define DADE_OPT_PCA_TC 15         /* PCA covariance: 1 (default) int8 tensor cores (exact levels), 0 fp64 CUDA cores (process-wide) */
#define DADE_OPT_SCAN_P1 17        /* 1: scan stage 1 list-major (first-step rows read once per probed list; p1.cu); 0 (default) off */
#define DADE_OPT_DHAT_CHUNK_MB 18  /* probe d_hat matrix chunk size in MB (0 = 2 GiB) */
#define DADE_OPT_KNN_I8 19         /* exact KNN for D >= 512: 1 int8 exact-split filter, 0 (default) the 3-pass tf32 filter */
#define DADE_OPT_GMIN_RATIO 20     /* exact KNN: group-minima select only when k * ratio <= 32-column groups (default 1) */
#define DADE_OPT_FZ_SEED_STRIDE 21 /* fused probe filter: seed pass column-tile stride (0 auto) */
#define DADE_OPT_FZ_ROWS 22        /* fused probe filter: 128-row A tiles per CTA sharing the B stream (0 auto, 1, 2) */
#define DADE_OPT_FZ_COLS 23        /* fused probe filter: epilogue groups per accumulator (column shares; 0 auto, 1, 2) */
#define DADE_OPT_DHAT_H16 24       /* probe d_hat writer (1-pass filter): 1 (default) fp16 operands (kind::f16), 2 the same with 128 x 256 tiles, 3 with cooperative cp.async operand loads (measurement), 0 tf32 hi parts */
#define DADE_OPT_FZ_CPS 12         /* fused probe filter: persistent CTAs per SM (0 auto = 1, 2 with 1 group) */
dade_status dade_set_option(dade_index* idx, int option, int64_t value);

/* Exact probes (a5 alone): probes[nq*nprobe] int32 device, ordered by (exact fp64 dist, id). */
dade_status dade_probe(dade_index* idx, const float* Q, int nq, int nprobe, int32_t* probes);

/* ---------------------------------------------------------------- tools
 * Exact KNN (K12): X device n x D (global ids id_base+i), Q device nq x D -> ids/dists device
 * nq x K ascending by (exact fp64 dist rounded to fp32, id). fp32 tile filter + fp64 re-rank. */
dade_status dade_bruteforce_knn(dade_index* idx, const float* X, int64_t n, int64_t id_base,
                                const float* Q, int nq, int K, int64_t* ids, float* dists);

/* a9 shard merge: ids_in/dists_in device S x nq x K (rank-major, as an all-gather lays them
 * out) -> ids_out/dists_out device nq x K, first K by (dist, id) over the S lists; id -1 slots
 * are ignored. */
dade_status dade_merge_topk(dade_index* idx, const int64_t* ids_in, const float* dists_in, int S,
                            int nq, int K, int64_t* ids_out, float* dists_out);

/* ---------------------------------------------------------------- NEXT-3: BSA-q (§V-B)
 * The data-driven correction on a QUANTIZATION distance: dis' = the asymmetric distance (ADC) of
 * the query to the candidate's product-quantization code (m subspaces of D/m dims, 256 codewords
 * each: nbits = 8; m = D/4, D/8 for GIST-like data), OPQ rotation, and the
 * candidate's distance to its own reconstruction e = ||x~ - x^||^2 as a second feature.
 * One classifier (R29): prune iff m1 * dis' + m2 * e + beta' > tau; survivors get the exact
 * distance and enter the top-K; tau frozen per epoch (R13) as in dade_search.
 *   dade_train_pq   OPQ on a strided sample of min(n, n_train ? n_train : 65,536) rows (P:L3105,
 *                   R28): PCA init, `iters` rounds of per-subspace k-means (km_iters Lloyd
 *                   iterations) + orthogonal Procrustes, then final_iters Lloyd iterations.
 *                   X: device n x D raw rows. INSTALLS the OPQ rotation as the index rotation
 *                   (discarding a built IVF: build_ivf afterwards) and the codebooks.
 *   dade_set_pq     install codebooks (host m x 256 x D/m fp32, row-major) in the CURRENT rotation's
 *                   basis; the layout (if built) is encoded at once.
 *   dade_get_pq     *m, codebooks (host, may be NULL), codes (host n x m, list-major rows) and err
 *                   (host n fp32 reconstruction errors) of the layout (may be NULL).
 *   Codes (R30): per subspace the argmin over the 256 codewords of the fp64 sequential sum of
 *   (x~_i - c_i)^2 over the subspace's dims of the STORED fp32 x~, ties to the lower code.
 *   dade_calibrate_pq  as dade_calibrate (same Label 0/1 pairs, R14-R16) with features (ADC dis', e):
 *                   two-feature logistic fit (R3, R29) -> m1, m2; v = sort_desc(tau - m1 dis' - m2 e)
 *                   over Label-0 pairs; a search with significance alpha uses beta' = v[k-1],
 *                   k = clamp(ceil((1 - alpha) n0), 1, n0).
 *   dade_get/set_calibration_q  K, n0, m[2] = {m1, m2}, v[n0] (host).
 * Search: dade_search_method(..., DADE_METHOD_BSA_Q, alpha, ...); stats->pruned_at_step[0] counts
 * the ADC prunes (0 dims read), n_steps = 1. PQ state is not saved by dade_save.
 * Errors: ARG (m does not divide D, D/m > 32, < 256 training rows), STATE (order), NONFINITE, CUDA. */
dade_status dade_train_pq(dade_index* idx, const float* X, int64_t n, int m, int64_t n_train, int iters,
                          int km_iters, int final_iters);
dade_status dade_set_pq(dade_index* idx, int m, const float* codebooks);
dade_status dade_get_pq(const dade_index* idx, int* m, float* codebooks, uint8_t* codes, float* err);
dade_status dade_calibrate_pq(dade_index* idx, const float* X, const float* Qc, int nq, int K, int n_neg,
                              int nprobe_neg, uint64_t seed);
dade_status dade_get_calibration_q(const dade_index* idx, int* K, int* n0, double* m, double* v);
dade_status dade_set_calibration_q(dade_index* idx, int K, int n0, const double* m, const double* v);

/* ---------------------------------------------------------------- NEXT-4: graph refinement with the DCO
 * HNSW (M = 16 -> base-layer degree M0 = 32) searched with the same
 * classifier-pruned progressive distances. Readings R33-R35:
 *   graph       a base-layer graph over this index's rows: each row's M0 neighbours chosen from its
 *               P nearest other rows by HNSW's neighbour-selection heuristic (keep e iff e is closer
 *               to the row than to every kept neighbour; fill from the dropped ones); the upper
 *               layers only supply the entry point: with an IVF (nlist > 1) the lowest-id row of
 *               the query's nearest non-empty list (the coarse quantizer stands in for them), in a
 *               flat index the row nearest to the rotation's mean.
 *   search      HNSW's best-first base-layer search: result queue W of size ef (N^{ef}), candidate
 *               queue C; pop the nearest c, stop when |W| = ef and dist(c) > max W; every unvisited
 *               neighbour is tested against tau = max W (inf while |W| < ef), FROZEN for the
 *               expansion; survivors' exact distances enter C and W in (dist, id) order; the first
 *               K of W are returned. The BSA-p step table comes from dade_calibrate with K = ef.
 *   dade_build_graph   pools from exact IVF searches of the rows themselves at nprobe_pool lists
 *                      (nprobe_pool = nlist: the exact P nearest), X = the raw rows (device);
 *                      1 <= M0 <= 32, M0 <= P <= 128.
 *   dade_set_graph / dade_get_graph   host n x M0 global ids (row i = id id_base + i, -1 pads), entry id.
 *   dade_graph_search  Q device nq x D raw; ids / dists device nq x K; K <= ef <= DADE_MAX_K; alpha
 *                      = 0: no pruning. stats (may be NULL): tested = nodes whose distance was
 *                      started, survivors = exact distances, dims_scanned, pruned_at_step,
 *                      n_epochs = node expansions. log (device log_cap x 3 int32, may be NULL): one
 *                      record {query, id, dims read} per tested node; *log_count = records produced.
 * A new IVF / rotation discards the graph. Errors: ARG, STATE (no IVF / graph / calibration with
 * K = ef), NONFINITE, UNSUPPORTED (D, ef too large for shared memory), CUDA. */
dade_status dade_build_graph(dade_index* idx, const float* X, int M0, int P, int nprobe_pool);
dade_status dade_set_graph(dade_index* idx, const int64_t* nbrs, int M0, int64_t entry);
dade_status dade_get_graph(const dade_index* idx, int* M0, int64_t* nbrs, int64_t* entry);
dade_status dade_graph_search(dade_index* idx, const float* Q, int nq, int K, int ef, int delta_d, double alpha,
                              int64_t* ids, float* dists, dade_stats* stats, int32_t* log, int64_t log_cap,
                              int64_t* log_count);

/* ---------------------------------------------------------------- multi-rank
 * The database is sharded by contiguous global-id ranges, one index (one process, one GPU) per
 * shard; mu, R, the centroids and the calibration table are replicated. The library owns the NCCL
 * communicator (libnccl.so.2 is loaded at run time; absent -> DADE_ERR_NCCL).
 *   dade_comm_unique_id  one rank creates the 128-byte NCCL unique id (host); the caller
 *                        distributes it to the other ranks (any out-of-band channel).
 *   dade_set_comm        every rank joins the group (collective; blocks until all have joined).
 *                        id may be NULL when nranks == 1. Replaces a previous communicator.
 * With a communicator (any nranks), dade_search / dade_search_method / dade_search_host are
 * COLLECTIVE: every rank passes the same queries; rank r rotates and probes its block of
 * ceil(nq/S) queries, the q~ and probe blocks are all-gathered (ncclAllGather), every rank scans all
 * queries over its shard, and the local top-K lists are all-gathered and merged by (dist, id); every
 * rank receives the full result. Pruning across shards (R32): per-shard c0 = ceil(4K/S); the scan
 * runs in E + 1 phases (epochs 0, ..., E-1 one by one, then the rest; E = DADE_OPT_SHARD_EXCHANGES,
 * default 2) and after each of the first E phases the shards' queues are all-gathered and merged:
 * from then on every shard prunes against tau_e = min(its own K-th, the merged K-th) — the merged
 * K-th bounds the global queue's tau from above, so a shard prunes no more aggressively than the
 * single-index search does at the same stream position. alpha = 0 gives exactly the unsharded
 * exact IVF. A group of one rank runs the same schedule and equals dade_search.
 * The sharded build (collective; X = this rank's rows, global ids [id_base, id_base+n) of n_total):
 *   dade_fit_rotation_dist  a0 on the GLOBAL strided sample (fp64 moments all-reduced);
 *   dade_build_ivf_dist     k-means on the global strided sample (R19; per-iteration fp64 sums and
 *                           counts all-reduced), then this shard's lists for all nlist centroids;
 *   dade_calibrate_dist     a3: shard K-NN lists merged, negatives merged, pair features summed —
 *                           the same table as an unsharded dade_calibrate on the whole base.
 * Errors: NCCL, STATE (no communicator for the _dist calls), and as the single-GPU calls. */
dade_status dade_comm_unique_id(void* id128);
dade_status dade_set_comm(dade_index* idx, const void* id128, int nranks, int rank);
dade_status dade_fit_rotation_dist(dade_index* idx, const float* X, int64_t n, int64_t id_base, int64_t n_total,
                                   int64_t sample_size);
dade_status dade_build_ivf_dist(dade_index* idx, const float* X, int64_t n, int64_t id_base, int64_t n_total,
                                int nlist, int kmeans_iters);
dade_status dade_calibrate_dist(dade_index* idx, const float* X, const float* Qc, int nq, int K, int n_neg,
                                int nprobe_neg, uint64_t seed);
/* Host combination steps of the sharded build (HOST arrays, no index, no GPU; the steps
 * dade_*_dist run between collectives, exported for drivers that move the buffers themselves):
 *   dade_kmeans_update      centroid[c] = fp32(sums[c] / counts[c]) where counts[c] > 0 (R19);
 *   dade_merge_knn          ids/dists S x nq x K (rank-major) -> the first K by (fp64 dist, id) (R14);
 *   dade_calibration_pairs  per query: its K nearest (Label 0) then the n_neg smallest (hash, id)
 *                           over the S shards' negative candidates keys/neg_ids S x nq x n_neg,
 *                           counts S x nq (Label 1), tau = the K-th distance (R15/R16); outputs
 *                           sized nq*(K+n_neg), *npairs = pairs written. */
dade_status dade_kmeans_update(int nlist, int D, const double* sums, const int64_t* counts, float* centroids);
dade_status dade_merge_knn(int S, int nq, int K, const int64_t* ids, const double* dists, int64_t* out_ids,
                           double* out_dists);
dade_status dade_calibration_pairs(int S, int nq, int K, int n_neg, const int64_t* knn_ids, const double* knn_dists,
                                   const uint64_t* keys, const int64_t* neg_ids, const int32_t* counts,
                                   int32_t* pair_q, int64_t* pair_id, double* tau, double* y, int64_t* npairs);

/* Persistence of {rotation, IVF, layout, calibration} (little-endian binary). */
dade_status dade_save(const dade_index* idx, const char* path);
dade_status dade_load(dade_index* idx, const char* path);

#ifdef __cplusplus
}
#endif
#endif /* DADE_H */
