// Internal declarations shared by the C-ABI layer (dade_api.cu) and the kernel TUs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dade.h"

namespace dade {

// A dade_status-carrying exception used inside the library only; converted at the ABI edge.
struct Error : std::runtime_error {
  dade_status st;
  Error(dade_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define DADE_CK(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::dade::Error(e_ == cudaErrorMemoryAllocation ? DADE_ERR_OOM : DADE_ERR_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));           \
  } while (0)
#define DADE_REQUIRE(cond, st, msg) \
  do {                              \
    if (!(cond)) throw ::dade::Error(st, msg); \
  } while (0)

// Owning device buffer (grows, never shrinks).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), cap(o.cap) { o.p = nullptr; o.cap = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; cap = o.cap;
      o.p = nullptr; o.cap = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }  // scoped scratch (e.g. inside dade_train_pq) is freed on every exit path
  void reserve(size_t n) {
    if (n <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (n == 0) return;
    DADE_CK(cudaMalloc(&p, n * sizeof(T)));
    cap = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

constexpr int kBlk = 16;  // layout block width B_L (dims per 64-B row)
#ifndef DADE_SCAN_PQ_LA  // BSA-q gather rounds: blocks per lane; 0 = chosen per D (scan.cu launch_k)
#define DADE_SCAN_PQ_LA 0
#endif
// lanes per survivor in a BSA-q gather round of LA blocks per lane: the fewest (a power of two,
// at most 32) that cover all nblk blocks in one round trip
inline int pq_gather_lanes(int nblk, int la) {
  int lanes = 1;
  while (lanes < 32 && lanes * la < nblk) lanes *= 2;
  return lanes;
}

// --------------------------------------------------------------------- kernel launchers
// exact.cu : fp32 tile distances + fp64-certified selection (assign / probe / KNN)
// d_hat[i*n + j] = fp32 sum_k fma((a_ik - b_jk)^2) for a block of rows of A against all rows of B.
void launch_l2_tile(const float* A, int64_t m, const float* B, int64_t n, int D, float* out,
                    cudaStream_t st);
// For each row i of the m x n matrix d_hat: the k nearest columns under the EXACT fp64
// sequential-sum distance between A[i] and B[col], ordered by (dist, col). Writes
// out_idx[i*k..] (column indices), out_d64[i*k..] (fp64 distances, may be null). Returns via
// *d_flag a nonzero value if a candidate buffer overflowed (caller reports an error).
void launch_select_exact(const float* d_hat, int64_t m, int64_t n, int k, const float* A,
                         const float* B, int D, int32_t* out_idx, double* out_d64,
                         int32_t* cand_buf, int cand_cap, int* d_flag, cudaStream_t st,
                         const float* slack = nullptr);
// Argmin (k = 1) specialisation for assignment: out[i] = argmin_c exact(A[i], B[c]).
void launch_argmin_exact(const float* d_hat, int64_t m, int64_t n, const float* A, const float* B,
                         int D, int32_t* out, int* d_flag, cudaStream_t st,
                         const float* slack = nullptr);
// gemm_tf32.cu : tensor-core (tcgen05 kind::tf32, 3-pass split) distance filter tiles
int64_t tc_rows_pad(int64_t rows);
int tc_nkc(int D);
float tc_gamma(int D, int passes = 3);
// center (nullable, fp32 D): operands are split from fl(x - center)
void launch_split_tf32(const float* X, int64_t rows, int D, const float* center, float* hi, float* lo,
                       float* norm, cudaStream_t st);
// out[j] = fp32(mean_r X[r, j]) (fp64 sums in scratch[D])
void launch_col_mean(const float* X, int64_t n, int D, double* scratch, float* out, cudaStream_t st);
void launch_slack(const float* an, int64_t m, float bmax, int D, float* slack, cudaStream_t st,
                  int passes = 3);
void launch_l2_tc(const float* Ahi, const float* Alo, const float* an, int64_t m, const float* Bhi,
                  const float* Blo, const float* bn, int64_t n, int D, float* out, int64_t ldo,
                  cudaStream_t st, float* gmin = nullptr, int passes = 3, int gshift = 5,
                  const float* ahs = nullptr, float bhs = 1.f,  // ahs: fp16 operands (per-row 1/scale of A, bhs = B's)
                  int nt = 1);  // nt = 2: 128 x 256 tiles (1-pass)
// warp-per-row exact select using the GEMM's 32-column group minima (k <= ceil(n/32) <= 256)
void launch_select_gmin(const float* d_hat, const float* gmin, int gshift, int64_t m, int64_t n, int k,
                        const float* A, const float* B, int D, int32_t* out_idx, double* out_d64,
                        int* d_flag, const float* slack, int* ovf_n, int32_t* ovf_rows,
                        cudaStream_t st);
// k nearest columns from the filter GEMM's 32-column group minima only (no d_hat matrix):
// exact fp64 distances for every column of the groups inside the certified window (k <= 512)
void launch_select_groups(const float* gmin, int64_t m, int64_t n, int k, const float* A, const float* B,
                          int D, int32_t* out_idx, double* out_d64, const float* slack, cudaStream_t st);
// probe_tc.cu: fused filter GEMM + candidate tracking (no d_hat matrix) + exact finish, k <= 64.
// cand: m * nsplit * probe_tc_cap(k) * 2 int32 scratch, ccount: m * nsplit int32 scratch.
int probe_tc_cap(int k);
// d_hat matrix + group minima with the warp-specialised pipeline of probe_tc.cu (same contract as
// launch_l2_tc with out != nullptr)
void launch_dhat_tc(const float* Ahi, const float* Alo, const float* an, int64_t m, const float* Bhi,
                    const float* Blo, const float* bn, int64_t n, int D, float* out, int64_t ldo, float* gmin,
                    int gshift, int passes, cudaStream_t st);
int probe_tc_splits(int64_t m, int64_t n, int sms);
bool dhat_ares_ok(int D, int passes);
void launch_dhat_ares(const float* Ahi, const float* an, int64_t m, const float* Bhi, const float* bn, int64_t n,
                      int D, float* out, int64_t ldo, float* gmin, int gshift, cudaStream_t st);
void launch_probe_tc(const float* Ahi, const float* Alo, const float* an, int64_t m, const float* Bhi,
                     const float* Blo, const float* bn, int64_t n, int D, int k, const float* slack,
                     const float* A, const float* B, int32_t* cand, int32_t* ccount, int nsplit,
                     int32_t* out_idx, double* out_d64, cudaStream_t st, int passes = 3);
void launch_max_nonneg(const float* v, int64_t n, float* out_dev, cudaStream_t st);
// exact finish of the fused filters: union of nlists candidate lists per row, fp64 re-rank
void launch_probe_finish(const int32_t* cand, const int32_t* ccount, int nlists, int C, int64_t m, int64_t n, int k,
                         const float* A, const float* B, int D, const float* slack, int32_t* out_idx, double* out_d64,
                         cudaStream_t st);
// probe_fz.cu: throughput fused filter (A tile resident, B ring, 2G TMEM accumulators, skip test)
// kind 1 = fp16 operands (kind::f16, power-of-two scales), 0 = tf32 hi parts (kind::tf32)
int fz_nkc(int D, int kind);
int fz_cap(int k);
size_t fz_smem(int D, int kind, int k, int G, int S, int cpc, int RP = 1, int CS = 1);
int64_t fz_rows_pad(int64_t rows);
bool fz_config(int D, int kind, int k, int* G, int* S, int* cps, int* RP);
int fz_lists_per_row(int64_t m, int64_t n, int P, int cstride = 1, int RP = 1);
void fz_seed_plan(int64_t m, int64_t n, int k, int P, int force, int* cstride, int* P1, int* maxL1, int RP = 1);
// gscale > 0: one matrix scale; else per-row power-of-two scales (inv_scale[r] = 1/s_r, +inf if unbounded)
void launch_split_h16(const float* X, int64_t rows, int D, const float* center, uint16_t* h, float* norm,
                      float* inv_scale, float gscale, cudaStream_t st);
void launch_slack_h16(const float* an, const float* ainv, int64_t m, float bmax, float binv, int D, float* slack,
                      cudaStream_t st);
void launch_probe_fz(int kind, const void* Aop, const float* an, const float* ainv, int64_t m, const void* Bop,
                     const float* bn, float binv, float bmax, int64_t n, int D, int k, const float* slack,
                     const float* A, const float* B, float* seeds, int32_t* cand, int32_t* ccount, int P, int maxL,
                     int G, int S, int cpc, int cstride, int P1, int maxL1, int32_t* out_idx, double* out_d64,
                     cudaStream_t st, int RP = 1, int CS = 1);

// rotate.cu : x~ = R (x - mu) on the tensor cores (tcgen05 kind::i8, kRotSlices-way split with
// exact int32 levels combined in fp64), stored fp32.
//  rowmajor_out != null: out[p*D + i]; blocked_out != null: out[(b*n_out + p)*16 + i%16].
//  src_rows != null: input row of output p is X[src_rows[p]] (gather) else X[p].
constexpr int kRotSlices = 6;
constexpr int kRotMaxD = 16384;
struct RotOp {  // R's rows, split (rot_prepare; once per rotation)
  DBuf<int8_t> bs;
  DBuf<int32_t> be;
  int D = 0;
  void release() { bs.release(); be.release(); D = 0; }
};
struct RotWs {  // slice scratch of the rotated rows (one per stream that rotates)
  DBuf<int8_t> as;
  DBuf<int32_t> ae;
  void release() { as.release(); ae.release(); }
};
void rot_prepare(RotOp& op, const double* R, int D, cudaStream_t st);
void launch_rotate(const RotOp& op, RotWs& ws, const float* X, const int32_t* src_rows, int64_t n_out,
                   const double* mu, float* rowmajor_out, float* blocked_out, cudaStream_t st);

// pca.cu : strided-sample moments in fp64
void launch_pca_sum(const float* X, int64_t n, int64_t id_base, int64_t n_total, int64_t ns,
                    int D, double* sum_dev, int64_t* cnt_host, cudaStream_t st);
void launch_pca_cov(const float* X, int64_t n, int64_t id_base, int64_t n_total, int64_t ns, int D,
                    const double* mean_dev, double* cov_dev, double* scratch, int64_t scratch_elems,
                    cudaStream_t st);
int64_t pca_cov_scratch_elems(int64_t n_owned, int D);
extern int g_pca_tc;  // 1 (default): covariance on the int8 tensor cores; 0: fp64 CUDA cores
// rotate.cu: acc[a][b] += sum_k Y[a][k] Y[b][k] (rows x K fp64 Y, K % 64 == 0, K <= 16384, rmax = row max bits)

// calib.cu : per-pair prefix partial distances in fp64 from the fp32 layout
void launch_pair_prefix(const float* layout, int64_t n_rows, int D, const float* qrot,
                        const int32_t* pair_q, const int32_t* pair_row, int npairs, double* out,
                        cudaStream_t st);
// scan.cu
struct ScanParams {
  const float* qrot;      // nq x D
  const int32_t* probes;  // nq x nprobe
  const int32_t* off;     // nlist + 1
  const int32_t* row_id;  // n global ids (list-major)
  const float* layout;    // D/16 blocks of n x 16
  int64_t n;
  int D, nq, nprobe, K, dd, nsteps, c0;  // dd = classifier spacing in 16-dim blocks (delta_d / 16)
  int prune;              // 0: no classifier can prune (alpha = 0 or one step)
  float m1[DADE_MAX_STEPS];
  float beta[DADE_MAX_STEPS];
  int64_t* out_ids;
  float* out_d;
  unsigned long long* counters;  // [0]=tested [1]=survivors [2]=dims [3]=max epochs [4..4+64) pruned_at_step
  int* work_counter;             // zeroed before the launch; persistent warps take queries from it
  // residual test (BSA-res, NEXT-1): prune iff P_d + (‖x‖² − N_d) + qconst[q][s-1] > tau
  int residual;
  const float* xnorm;   // n: ‖x~‖² per list-major row (residual only)
  const float* qconst;  // nq x (nsteps - 1): ‖q_r‖² − m·σ_d per step (residual only)
  int64_t avg_stream;   // expected candidates per query (nprobe * n / nlist): picks warps per query
  const int32_t* order; // nq: processing order of the queries (null = 0..nq-1); results stay at q
  int g_force;          // warps per query (0 = the scan_group heuristic)
  unsigned dd_magic;    // ceil(2^32 / dd), set by launch_scan
  // BSA-q (NEXT-3): stage 1 reads the candidates' PQ code rows (codes | fp32
  // reconstruction error, pq_stride bytes per list-major row) and prunes iff
  // pq_m1 * ADC + pq_m2 * err + pq_beta > tau; survivors get the exact distance over all blocks
  int pq;
  const uint8_t* pq_codes;
  int pq_stride, pq_eo, pq_m, pq_ds;
  const float* pq_C;       // m x 256 x ds codebooks
  float pq_m1, pq_m2, pq_beta;
  int pq_lg;               // log2 lanes per survivor in the exact-distance gather rounds
  // phases of a sharded search (R32): epochs [ep_first, ep_end) of each query's stream; the
  // previous phase's queue (init_*: nq x K, null = empty) and the exchanged merged queue whose
  // K-th distance bounds tau from above (cap_*: nq x K, null = no bound)
  int ep_first, ep_end;
  const int64_t* init_ids;
  const float* init_d;
  const int64_t* cap_ids;
  const float* cap_d;
  // stage 1 from the list-major precompute (p1.cu; null = read the rows): p1[p1_base[q] + t] is
  // the first step's partial distance of candidate t of query q's stream (BSA-p / ADSampling)
  const float* p1;
  const int* p1_base;
  const long long* p1_total;  // the streams' total length (device); p1 is used only if <= p1_cap
  long long p1_cap;
  // decision log (parity runs; null = off): per tested candidate (query, global id, dims read)
  int32_t* dlog;
  int64_t dlog_cap;              // records
  unsigned long long* dlog_n;    // records written (may exceed dlog_cap: the caller sees the overflow)
};
void launch_scan(const ScanParams& p, cudaStream_t st);
// p1.cu: the first step's partial distances of every (query, candidate) pair, list-major (each
// probed list's first-step rows read once for all queries probing it). dd_unit = the scan's
// staging unit in blocks (1, 2, 4); scratch: p1_scratch_ints ints; qbase_out: nq ints; p1: the
// sum of the queries' stream lengths (+ 4) floats.
size_t p1_scratch_ints(int nq, int nprobe, int nlist);
void p1_launch(const float* layout, int64_t n, const int32_t* off, int nlist, const int32_t* probes, int nq,
               int nprobe, const float* qrot, int D, int dd_unit, int* scratch, int* qbase_out, float* p1,
               int64_t p1_cap, long long* total, cudaStream_t st);
// misc.cu: the scan's query order — a counting sort of the queries by their nearest probed list
// (probes[q][0]), so queries that share lists are scanned close in time (L2 reuse of their
// tiles). cnt: nlist ints of scratch; order: nq ints.
void launch_query_order(const int32_t* probes, int nq, int nprobe, int nlist, int* cnt, int32_t* order,
                        cudaStream_t st);
// the scan's query order, longest candidate stream first (scratch: 1024 + nq ints)
void launch_query_order_lpt(const int32_t* probes, int nq, int nprobe, const int32_t* off, int64_t avg_stream,
                            int* scratch, int32_t* order, cudaStream_t st);
// ‖x~‖² of every list-major row of the blocked layout (fp64 sums, stored fp32)
void launch_row_norms(const float* layout, int64_t n, int D, float* out, cudaStream_t st);
// estimate.cu (NEXT-2, Exp-7): top-K by the d-dim estimate over the whole layout; xnorm != null
// adds the residual terms ||x_r||^2 + ||q_r||^2 (Eq. 2)
#define DADE_EST_MAX_D 4096
void launch_estimate_topk(const float* layout, const int32_t* row_id, const float* xnorm, int64_t n, int D, int d,
                          const float* qrot, int nq, int K, float* est, int64_t* ids, cudaStream_t st);
// BSA-res per-step query constants c_s = sum_{i>=d} q_i^2 - m sqrt(4 sum_{i>=d} q_i^2 lam_i), d = s*delta_d
void launch_res_consts(const float* qrot, int nq, int D, int delta_d, const double* lam, double m,
                       float* out, cudaStream_t st);
// merge.cu
void launch_merge_topk(const int64_t* ids_in, const float* d_in, int S, int nq, int K,
                       int64_t* ids_out, float* d_out, cudaStream_t st);
void launch_check_finite(const float* X, int64_t n, int* flag, cudaStream_t st, int code = 1);
// row-major n x D -> dimension-blocked layout (block b = n x 16, rows in the same order)
void launch_to_blocked(const float* X, int64_t n, int D, float* out, cudaStream_t st);
void launch_gather_rows(const float* X, const int32_t* rows, int64_t m, int D, float* out,
                        cudaStream_t st);

// comm.cpp : the index's NCCL communicator (dlopen'd libnccl) and the sharded build's host steps
struct Comm;
enum class CommType { F64, I64 };
void comm_unique_id(void* out128);
Comm* comm_create(const void* id128, int nranks, int rank);
void comm_destroy(Comm* c);
int comm_size(const Comm* c);
int comm_rank(const Comm* c);
// in-place sum over ranks of a DEVICE buffer, on `st`
void comm_allreduce_sum(Comm* c, void* buf, size_t count, CommType t, cudaStream_t st);
// DEVICE all-gather: recv = rank 0's bytes, rank 1's, ... (in place when send == recv + rank * bytes)
void comm_allgather(Comm* c, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st);
void kmeans_update(int nlist, int D, const double* sums, const int64_t* counts, float* cent);
void merge_knn(int S, int nq, int K, const int64_t* ids, const double* d, int64_t* out_ids, double* out_d);
int64_t calibration_pairs(int S, int nq, int K, int n_neg, const int64_t* knn_ids, const double* knn_d,
                          const uint64_t* keys, const int64_t* nids, const int32_t* cnt, int32_t* pq,
                          int64_t* pid, double* tau, double* y);

// pq.cu (NEXT-3 BSA-q)
void launch_pq_assign(const float* X, bool blocked, int64_t n, int D, int m, const float* C, uint8_t* codes,
                      int stride, cudaStream_t st);
void launch_pq_err(const float* layout, int64_t n, int D, int m, const float* C, uint8_t* codes, int stride, int eo,
                   cudaStream_t st);
void launch_pq_pair_feat(const uint8_t* codes, int stride, int eo, int m, int D, const float* C, const float* qrot,
                         const int32_t* pq, const int32_t* pr, int npairs, double* out, cudaStream_t st);
void launch_pq_cross(const float* X, const double* mu, int64_t n, int D, int m, const float* C, const uint8_t* codes,
                     double* M, cudaStream_t st);

// graph.cu (NEXT-4): HNSW base-layer refinement with the DCO
struct GraphParams {  // one graph search launch (graph.cu)
  const float* qrot;        // nq x D
  const float* layout;      // blocked
  const int32_t* row_id;    // list-major position -> global id
  const int32_t* adj;       // n x M0 positions (-1 pad)
  int64_t n;
  int D, nq, K, ef, M0, entry, dd, nsteps;
  // per-query entry (R33): the first row of the query's nearest non-empty list among `eprobe`
  // probes (null: the index-wide entry)
  const int32_t* eprobes;
  int eprobe;
  const int32_t* off;
  float m1[DADE_MAX_STEPS], beta[DADE_MAX_STEPS];
  int64_t* out_ids;
  float* out_d;
  unsigned* visited;        // per warp slot: ceil(n / 32) words, zero between queries
  int32_t* vlist;           // per warp slot: vcap positions set in the bitmap
  int vcap;
  int* work;
  unsigned long long* counters;  // [0] tested [1] survivors [2] expansions [3] unused [4 + s] pruned at step s
  int32_t* dlog;
  int64_t dlog_cap;
  unsigned long long* dlog_n;
};


size_t graph_smem(int D, int ef);
int graph_slots(int sms);
void launch_graph_search(const GraphParams& p, int sms, cudaStream_t st);
// HNSW's neighbour-selection heuristic per node over its candidate pool (positions, ascending by
// (dist, id)); out: n x M0 positions (-1 pad)
void launch_graph_prune(const float* layout, int64_t n, int D, const int32_t* pool, const float* pool_d, int P,
                        int M0, int32_t* out, cudaStream_t st);

// host_eig.cpp : symmetric eigendecomposition (Householder tridiagonalisation + implicit QL)
void sym_eig(int n, const double* A, double* eigval, double* eigvec_colmajor);
// host_calib.cpp
bool logistic_irls(const std::vector<double>& P, const std::vector<double>& tau,
                   const std::vector<double>& y, double ridge, int max_iter, double tol,
                   double* m1, double* beta);
bool logistic_irls_multi(const std::vector<double>& F, int k, const std::vector<double>& tau,
                         const std::vector<double>& y, double ridge, int max_iter, double tol,
                         std::vector<double>& m_out, double* beta_out);
uint64_t splitmix64(uint64_t x);

// rotate.cu, the int8 filter of exact_knn (distance mode): B slices (centred on mu, fp64),
// fp64 centred norms, per-row slack, and the d_hat matrix + 32-column group minima (float bits)
void prepare_i8_b(const float* B, int64_t n, int D, const double* mu, RotOp& ob, cudaStream_t st);
void launch_cnorm64(const float* X, int64_t n, int64_t rows_pad, int D, const double* mu, double* out,
                    cudaStream_t st);
void launch_slack_i8(const double* an, const int32_t* ea, int64_t m, const int* e_bmax,
                     const unsigned long long* bmax_bits, int D, float* slack, cudaStream_t st);
// B side of the int8 filter, all on the device: mu64 = the fp32 centre, the slices, fp64 norms
// (bn64: n rounded up to 32 entries), the largest slice exponent and the largest norm
void launch_i8_bprep(const float* B, int64_t n, int D, const float* center, double* mu64, RotOp& ob, double* bn64,
                     int* emax, unsigned long long* bmax_bits, cudaStream_t st);
void launch_dist_i8(const float* A, int64_t m, int D, const double* mu, const double* an64, RotWs& wa,
                    const RotOp& ob, const double* bn64, int64_t n, float* dist, unsigned* gmin, int64_t ldg,
                    cudaStream_t st);
void launch_gram_i8(const double* Y, int rows, int64_t K, const unsigned long long* rmax, RotWs& wa, RotOp& wb,
                    double* acc, cudaStream_t st);
}  // namespace dade
