// C-ABI of the DADE library: index state, orchestration of the kernels, error mapping.
// Every entry point follows include/dade.h; citations there.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <type_traits>
#include <vector>

#include "dade_internal.h"

namespace dade { extern int g_fz_debug; }
using namespace dade;

// A matrix pre-split for the tensor-core distance filter (gemm_tf32.cu): tf32 hi/lo parts in the
// UMMA tiled layout, fp32 squared norms, and the largest norm (for the error bound).
struct TcOp {
  DBuf<float> hi, lo, norm, maxn, center;
  DBuf<double> csum;
  DBuf<uint16_t> h16;  // fp16 operand (probe_fz.cu), K-major tiles of 32 halves per row per chunk
  DBuf<float> hinv;    // per-row 1 / scale of the fp16 operand (A side)
  int64_t rows = 0;
  float maxnorm = 0.f;
  float hinv_b = 0.f;  // 1 / matrix scale of the fp16 operand (B side)
  bool h16_ok = false;
  // int8 exact-split filter (rotate.cu distance mode), B side: slices, fp64 centre and norms,
  // largest slice exponent and norm (device)
  RotOp i8b;
  DBuf<double> mu64, bn64;
  DBuf<int> i8e;
  DBuf<unsigned long long> i8bmax;
  bool i8_ok = false;
  void release() {
    hi.release(); lo.release(); norm.release(); maxn.release(); center.release(); csum.release();
    h16.release(); hinv.release();
    i8b.release(); mu64.release(); bn64.release(); i8e.release(); i8bmax.release();
    rows = 0;
    h16_ok = false;
    i8_ok = false;
  }
};

// Tuning options (dade_set_option): every default is the measured best; the others exist for
// A/B measurement and for the tests that prove each path returns identical results.
struct Options {
  int knn_path = 0;         // exact KNN filter: 0 auto, 1 d_hat matrix, 2 fused (no d_hat), 3 group minima,
                            // 4 throughput fused filter on fp16 operands, 5 the same on tf32 hi parts
  int probe_passes = 0;     // tf32 passes of the probe filter: 0 auto (1 if D < 512 else 3), 1, 3
  int scan_warps = 0;       // warps per query in k_scan: 0 auto, 1, 2, 4, 8
  int scan_order = 2;       // 0: as given, 1: grouped by nearest probed list, 2: longest stream first
  int scan_tail = 0;        // last X queries scanned by a concurrent 4-warps-per-query launch
  int host_chunks = 1;      // dade_search_host: searches pipelined with the copies
  int host_prep_chunks = 0; // dade_search_host: rotation + probe chunks ahead of one scan (0 auto)
  int dhat_ares = 0;        // 1: A-resident d_hat writer for very wide rows (1-pass filter)
  int dhat_h16 = 1;         // 1 (default): the d_hat writer's 1-pass filter on fp16 operands (kind::f16), 0: tf32 hi parts
  int dhat_chunk_mb = 0;    // d_hat matrix chunk in MB (0: 2 GiB); measurement option
  int gmin_ratio = 1;       // exact_knn: group-minima select only when k * ratio <= number of 32-column groups
  int knn_i8 = 0;           // exact_knn: 1 = int8 exact-split filter for D >= 512; 0 (default) the 3-pass tf32 one
  int scan_p1 = 0;          // stage 1 list-major (p1.cu): 1 on; 0 (default) off — measured slower
  int shard_exchanges = 2;  // collective search: top-K exchanges after epochs 0 .. E-1 (R32)
  int fz_stages = 0;        // probe_fz.cu: B ring stages (0 auto)
  int fz_groups = 0;        // probe_fz.cu: epilogue groups of 4 warps (0 auto, 1, 2)
  int fz_cps = 0;           // probe_fz.cu: persistent CTAs per SM (0 auto = 1; 2 needs 1 group and smem <= 113 KB)
  int fz_seed_stride = 0;   // probe_fz.cu: seed pass column-tile stride (0 auto: >= 16 k group minima, <= 16)
  int fz_cpc = 0;           // probe_fz.cu: 8 KB operand chunks per TMA copy (0 auto = 1)
  int fz_rows = 0;          // probe_fz.cu: 128-row A tiles per CTA sharing the B stream (0 auto, 1, 2)
  int fz_cols = 0;          // probe_fz.cu: epilogue groups per accumulator, column shares (0 auto, 1, 2)
};

struct dade_index {
  int device = 0;
  Options opt;
  cudaStream_t stream = nullptr;
  int D = 0;
  // rotation (a0)
  bool has_rot = false;
  bool has_lam = false;  // eigenvalues known (fit_rotation, or given to set_rotation): BSA-res needs them
  std::vector<double> mean, R, lam;
  DBuf<double> R_d, mean_d;
  RotOp rot_op;              // R split for the tensor-core rotation (rotate.cu)
  RotWs rot_ws, rot_ws_side;  // slice scratch: main stream / side stream (query rotation ∥ probe)
  // IVF + layout (a1, a2)
  bool has_ivf = false;
  int nlist = 0;
  int64_t n = 0, id_base = 0;
  DBuf<float> cent, layout;
  TcOp cent_tc;  // centroids, pre-split for the tensor-core probe filter
  DBuf<int32_t> off_d, row_id_d;
  std::vector<int64_t> off_h, row_id_h;
  std::vector<int32_t> assign_h, pos_of_h;  // pos_of_h[local id] = list-major position
  // calibration (a3)
  bool has_cal = false;
  int calK = 0, n0 = 0, ncls = 0;
  std::vector<double> m1, v;
  // scratch
  DBuf<float> qrot, dmat, qbuf, slack, gmin, fzseed, p1;
  DBuf<double> an64;  // int8 filter: fp64 centred query norms
  DBuf<int> p1_base, p1_scr;
  DBuf<long long> p1_total;
  TcOp a_tc;  // scratch: query-side operand of the filter GEMM
  DBuf<int32_t> probes, cand, idx32;
  DBuf<double> d64;
  DBuf<int> flag, fflag, work, ovf;
  DBuf<unsigned long long> counters, dlog_n;
  DBuf<int64_t> ids_tmp;
  DBuf<int> ordcnt;      // scan query order: per-list counts / cursors
  DBuf<int32_t> order;
  DBuf<float> dists_tmp;
  // NEXT-1 BSA-res: per-row ‖x~‖² (list-major, computed on first use), eigenvalues, query constants
  DBuf<float> xnorm, qconst;
  DBuf<double> lam_d;
  bool xnorm_ok = false;
  cudaEvent_t ev[5] = {};
  bool timing = false;  // record the stage events on every search (dade_set_timing)
  // a4 (rotation) runs on a side stream concurrently with a5 (probe): fork/join events
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // dade_search_host: copy streams and per-chunk events of the H2D / search / D2H pipeline
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> hev;
  // NEXT-3 BSA-q: PQ codebooks (m x 256 x D/m, in the current rotation's basis), the code rows of
  // the layout (list-major; codes | fp32 reconstruction error | pad, pq_stride bytes), calibration
  bool has_pq = false;
  int pq_m = 0, pq_stride = 0, pq_eo = 0;
  std::vector<float> pq_C;
  DBuf<float> pq_Cd;
  DBuf<uint8_t> pq_codes;
  bool pq_codes_ok = false;
  bool has_calq = false;
  int calqK = 0, n0q = 0;
  double mq[2] = {1.0, 0.0};
  std::vector<double> vq;
  // NEXT-4 graph refinement: base-layer adjacency (n x M0 layout positions), entry position,
  // per-warp-slot visited bitmaps and lists
  bool has_graph = false;
  int g_M0 = 0, g_entry = 0;
  DBuf<int32_t> g_adj, g_vlist;
  DBuf<unsigned> g_vis;
  int64_t g_slots = 0;
  // multi-rank (dade_set_comm): the NCCL communicator of this shard's group
  Comm* comm = nullptr;
  DBuf<int64_t> gids, cap_ids;    // collective search: all-gathered local top-K ids / dists, the
  DBuf<float> gdists, cap_d;      // merged queue of the last exchange (R32)
  DBuf<double> red;      // device staging of host partials for all-reduce
};

// ------------------------------------------------------------------ error plumbing
static thread_local std::string g_err;
#define API_BEGIN try {
#define API_END                                  \
  g_err.clear();                                 \
  return DADE_OK;                                \
  }                                              \
  catch (const Error& e) {                       \
    g_err = e.what();                            \
    return e.st;                                 \
  }                                              \
  catch (const std::bad_alloc&) {                \
    g_err = "host allocation failed";            \
    return DADE_ERR_OOM;                         \
  }                                              \
  catch (const std::exception& e) {              \
    g_err = e.what();                            \
    return DADE_ERR_CUDA;                        \
  }

extern "C" const char* dade_last_error(void) { return g_err.c_str(); }

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) DADE_CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void need(const void* p, const char* what) {
  DADE_REQUIRE(p != nullptr, DADE_ERR_ARG, std::string("NULL pointer: ") + what);
}

void check_finite(dade_index* x, const float* X, int64_t count, const char* what) {
  x->fflag.reserve(1);
  DADE_CK(cudaMemsetAsync(x->fflag.p, 0, sizeof(int), x->stream));
  launch_check_finite(X, count, x->fflag.p, x->stream);
  int h = 0;
  DADE_CK(cudaMemcpyAsync(&h, x->fflag.p, sizeof(int), cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  DADE_REQUIRE(h == 0, DADE_ERR_NONFINITE, std::string("non-finite value in ") + what);
}

// Errors of the exact selection (candidate buffers overflowed) latch in x->flag and are reported
// at the next synchronising call.
void check_knn_flag(dade_index* x) {
  if (!x->flag.p) return;
  int h = 0;
  DADE_CK(cudaMemcpyAsync(&h, x->flag.p, sizeof(int), cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  if (h != 0) {
    DADE_CK(cudaMemsetAsync(x->flag.p, 0, sizeof(int), x->stream));
    if (h == 3) throw Error(DADE_ERR_NONFINITE, "non-finite value in the queries of a previous search");
    throw Error(DADE_ERR_UNSUPPORTED, "exact selection: more than 4096 near-tied candidates for one row");
  }
}

// need_max: B operand (computes its column mean = the centre both operands use, and the largest
// centred norm); else A operand, centred on `center` (the B operand's).
void tc_prepare(dade_index* x, const float* B, int64_t n, TcOp& op, bool need_max, const float* center = nullptr) {
  const int D = x->D;
  const int64_t rp = tc_rows_pad(n);
  const size_t elems = (size_t)rp * tc_nkc(D) * 32;
  op.hi.reserve(elems);
  op.lo.reserve(elems);
  op.norm.reserve(rp);
  if (need_max) {
    op.center.reserve(D);
    op.csum.reserve(D);
    launch_col_mean(B, n, D, op.csum.p, op.center.p, x->stream);
    center = op.center.p;
  }
  launch_split_tf32(B, n, D, center, op.hi.p, op.lo.p, op.norm.p, x->stream);
  op.rows = n;
  if (need_max) {
    op.maxn.reserve(1);
    launch_max_nonneg(op.norm.p, n, op.maxn.p, x->stream);
    DADE_CK(cudaMemcpyAsync(&op.maxnorm, op.maxn.p, sizeof(float), cudaMemcpyDeviceToHost, x->stream));
    DADE_CK(cudaStreamSynchronize(x->stream));
  }
  op.h16_ok = false;  // the fp16 copy (probe_fz.cu) is made on first use: tc_prepare_h16
  op.i8_ok = false;   // so is the int8 split (tc_prepare_i8)
}

// int8 exact-split copy of a prepared B operand (the wide-row filter of exact_knn), on first use
void tc_prepare_i8(dade_index* x, const float* B, TcOp& op) {
  if (op.i8_ok) return;
  const int D = x->D;
  const int64_t rp = (op.rows + 31) / 32 * 32;
  op.mu64.reserve((size_t)D);
  op.bn64.reserve((size_t)rp);
  op.i8e.reserve(1);
  op.i8bmax.reserve(1);
  launch_i8_bprep(B, op.rows, D, op.center.p, op.mu64.p, op.i8b, op.bn64.p, op.i8e.p, op.i8bmax.p, x->stream);
  op.i8_ok = true;
}

// fp16 copy of a prepared B operand for the fused probe filter (probe_fz.cu), made once per
// preparation: one power-of-two scale from the largest centred norm, ||b'||_inf <=
// sqrt(maxnorm (1 + 2^-20)) < 2^E, s = 2^(14 - E). Leaves h16_ok false when the operand is too
// wide for the kernel or the scale would clamp.
void tc_prepare_h16(dade_index* x, const float* B, TcOp& op) {
  if (op.h16_ok) return;
  const int D = x->D;
  if (fz_nkc(D, 1) * 8192 > 64 * 1024) return;
  int E = 0;
  const double bnd = std::sqrt((double)op.maxnorm * (1.0 + 9.5367431640625e-07));
  if (bnd > 0.0) std::frexp(bnd, &E);
  const int e = std::min(60, 14 - E);
  if (e < -60) return;
  const float sc = std::ldexp(1.f, e);
  op.h16.reserve((size_t)fz_rows_pad(op.rows) * fz_nkc(D, 1) * 32);  // 32 halves per row per chunk
  launch_split_h16(B, op.rows, D, op.center.p, op.h16.p, nullptr, nullptr, sc, x->stream);
  op.hinv_b = 1.f / sc;
  op.h16_ok = true;
}

// Exact k nearest rows of B for every row of A: tensor-core distance filter (tcgen05 kind::tf32,
// 3-pass split; bop = B pre-split by tc_prepare) with a rigorous absolute error bound, then fp64
// re-rank of every column inside the certified window (exact.cu). Bit-exact with the fp64
// sequential-sum definition (R20). out_idx: device m x k int32; out_d64: device m x k or null.
void exact_knn(dade_index* x, const float* A, int64_t m, const float* B, int64_t n, int k,
               int32_t* out_idx, double* out_d64, const TcOp& bop, bool sync = true, int passes = 3) {
  const int D = x->D;
  DADE_REQUIRE(k >= 1 && k <= n, DADE_ERR_ARG, "exact_knn: k out of range");
  DADE_REQUIRE(k <= 4096, DADE_ERR_UNSUPPORTED, "exact_knn: k > 4096");
  DADE_REQUIRE(bop.rows == n, DADE_ERR_STATE, "exact_knn: operand not prepared");
  if (!x->flag.p) {
    x->flag.reserve(1);
    DADE_CK(cudaMemsetAsync(x->flag.p, 0, sizeof(int), x->stream));
  }
  // fused path only for very wide rows, where the d_hat matrix would not fit the group-minima
  // select (> 1024 groups; measured at 16,384 columns: d_hat path 0.31 ms, fused 0.61 ms);
  // DADE_OPT_KNN_PATH forces a path (tests cover each)
  const int path = x->opt.knn_path;
  // throughput fused filter (probe_fz.cu): the 1-pass probe filter on fp16 (4) or tf32 (5)
  // operands with the A tile resident in shared memory; where it does not apply (3-pass filters,
  // k > 64, n < 256, A tiles wider than shared memory) paths 4/5 fall back to the d_hat matrix
  {
    const int kind = path == 5 ? 0 : 1;
    int G = 0, S = 0;
    if (kind == 1 && passes == 1 && k <= 32 && n >= 256 && (path ? path == 4 : n > 32768))
      tc_prepare_h16(x, B, const_cast<TcOp&>(bop));  // the operand cache (cent_tc) gains its fp16 copy
    // auto: only for very wide rows (> 32,768 columns, the C5 shard's 65,536 lists) — measured
    // (tools/exp_probe_fz.py): C5 shard 1.42 -> 0.95 ms, but slower than the d_hat path at 4,096
    // and 16,384 columns (C2, C4), where the d_hat matrix is small
    int cps = 1, RP = 1, CS = 1;
    bool fz = passes == 1 && k <= 32 && n >= 256 && (path ? (path == 4 || path == 5) : n > 32768) &&
              (kind == 0 || bop.h16_ok) && fz_config(D, kind, k, &G, &S, &cps, &RP);
    int cpc = 1;
    if (fz && (x->opt.fz_groups || x->opt.fz_stages || x->opt.fz_cps || x->opt.fz_cpc || x->opt.fz_rows ||
               x->opt.fz_cols)) {
      // measurement overrides
      if (x->opt.fz_groups) G = x->opt.fz_groups;
      if (x->opt.fz_stages) S = x->opt.fz_stages;
      if (x->opt.fz_cps) cps = x->opt.fz_cps;
      if (x->opt.fz_cpc) cpc = x->opt.fz_cpc;
      if (x->opt.fz_rows) RP = x->opt.fz_rows;
      if (x->opt.fz_cols) CS = x->opt.fz_cols;
      if (RP == 2 || CS == 2) {  // row-tile pairs: one group, one CTA per SM, the deepest ring that fits
        if (!x->opt.fz_groups) G = 1;
        if (!x->opt.fz_cps) cps = 1;
        if (!x->opt.fz_stages)
          for (S = 12; S > 3 && fz_smem(D, kind, k, G, S, cpc, RP, CS) * cps > 226 * 1024; --S) {}
      }
      DADE_REQUIRE(fz_smem(D, kind, k, G, S, cpc, RP, CS) * cps <= 226 * 1024 && (cps == 1 || G == 1) &&
                       (RP == 1 || (kind == 1 && G == 1)) && (CS == 1 || kind == 1) && G * RP * CS * cps <= 4,
                   DADE_ERR_UNSUPPORTED, "fz options: shared memory or TMEM does not fit");
    }
    if (fz) {
      int sms = 0;
      DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->device));
      const int64_t chunk = std::min<int64_t>(tc_rows_pad(m), 65536);
      // persistent: one CTA per SM (at most one per (row tile, column tile) pair)
      auto ctas = [&](int64_t rows) {
        return (int)std::min<int64_t>((int64_t)sms * cps, ((rows + 128 * RP - 1) / (128 * RP)) * ((n + 127) / 128));
      };
      const int64_t last = m - (m - 1) / chunk * chunk;  // rows of the last chunk
      const size_t nl = (size_t)G * CS * std::max((size_t)chunk * fz_lists_per_row(chunk, n, ctas(chunk), 1, RP),
                                             (size_t)last * fz_lists_per_row(last, n, ctas(last), 1, RP));
      const int C = fz_cap(k);
      x->slack.reserve((size_t)chunk);
      x->cand.reserve(nl * C * 2 + nl);
      auto seed_plan = [&](int64_t rows, int* cs, int* P1, int* L1) {
        fz_seed_plan(rows, n, k, ctas(rows), x->opt.fz_seed_stride, cs, P1, L1, RP);
      };
      size_t nseed = 0;
      for (int64_t rows : {chunk, last}) {
        int cs, P1, L1;
        seed_plan(rows, &cs, &P1, &L1);
        nseed = std::max(nseed, (size_t)rows * L1 * G * CS);
      }
      // (>= 4,096 floats: the pipeline-only measurement build records its timeline there)
      x->fzseed.reserve(std::max<size_t>(std::max(nl, nseed) * k, 4096));
      for (int64_t r0 = 0; r0 < m; r0 += chunk) {
        const int64_t mm = std::min(chunk, m - r0);
        const void* Aop;
        const float* ainv = nullptr;
        if (kind == 1) {
          const int64_t rp = fz_rows_pad(mm);
          x->a_tc.h16.reserve((size_t)rp * fz_nkc(D, 1) * 32);  // 32 halves per row per chunk
          x->a_tc.hinv.reserve((size_t)rp);
          x->a_tc.norm.reserve((size_t)rp);
          launch_split_h16(A + r0 * D, mm, D, bop.center.p, x->a_tc.h16.p, x->a_tc.norm.p, x->a_tc.hinv.p, 0.f,
                           x->stream);
          launch_slack_h16(x->a_tc.norm.p, x->a_tc.hinv.p, mm, bop.maxnorm, bop.hinv_b, D, x->slack.p, x->stream);
          Aop = x->a_tc.h16.p;
          ainv = x->a_tc.hinv.p;
        } else {
          tc_prepare(x, A + r0 * D, mm, x->a_tc, false, bop.center.p);
          launch_slack(x->a_tc.norm.p, mm, bop.maxnorm, D, x->slack.p, x->stream, 1);
          Aop = x->a_tc.hi.p;
        }
        int cs1, P1, L1;
        seed_plan(mm, &cs1, &P1, &L1);
        launch_probe_fz(kind, Aop, x->a_tc.norm.p, ainv, mm, kind == 1 ? (const void*)bop.h16.p : (const void*)bop.hi.p,
                        bop.norm.p, bop.hinv_b, bop.maxnorm, n, D, k, x->slack.p, A + r0 * D, B, x->fzseed.p, x->cand.p,
                        x->cand.p + nl * C * 2, ctas(mm), fz_lists_per_row(mm, n, ctas(mm), 1, RP), G, S, cpc, cs1,
                        P1, L1, out_idx + r0 * k, out_d64 ? out_d64 + r0 * k : nullptr, x->stream, RP, CS);
      }
      if (sync) check_knn_flag(x);
      return;
    }
  }
  const bool fused = k <= 64 && n >= 256 && (path ? path == 2 : (n + 63) / 64 > 1024);
  if (fused) {
    // fused filter GEMM + candidate tracking (probe_tc.cu): no m x n d_hat matrix
    int sms = 0;
    DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->device));
    const int64_t chunk = std::min<int64_t>(tc_rows_pad(m), 65536);
    const int nsplit = probe_tc_splits(chunk, n, sms);
    const int C = probe_tc_cap(k);
    x->slack.reserve((size_t)chunk);
    x->cand.reserve((size_t)chunk * nsplit * C * 2 + (size_t)chunk * nsplit);
    for (int64_t r0 = 0; r0 < m; r0 += chunk) {
      const int64_t mm = std::min(chunk, m - r0);
      tc_prepare(x, A + r0 * D, mm, x->a_tc, false, bop.center.p);
      launch_slack(x->a_tc.norm.p, mm, bop.maxnorm, D, x->slack.p, x->stream, passes);
      launch_probe_tc(x->a_tc.hi.p, x->a_tc.lo.p, x->a_tc.norm.p, mm, bop.hi.p, bop.lo.p, bop.norm.p, n, D, k,
                      x->slack.p, A + r0 * D, B, x->cand.p, x->cand.p + (size_t)chunk * nsplit * C * 2, nsplit,
                      out_idx + r0 * k, out_d64 ? out_d64 + r0 * k : nullptr, x->stream, passes);
    }
    if (sync) check_knn_flag(x);
    return;
  }
  const int64_t ng = (n + 31) / 32;
  // group-minima-only path (no d_hat matrix): measured slower than the d_hat path at k <= 32
  // (32 exact fp64 columns per candidate group, uncoalesced); kept for very wide rows
  if (k <= 512 && (int64_t)k * 4 <= ng && (path ? path == 3 : n > (int64_t)1 << 20)) {
    // the GEMM writes only 32-column group minima; exact fp64 distances for the columns of the
    // groups inside the certified window (no m x n d_hat matrix)
    int64_t chunk = std::max<int64_t>(128, ((int64_t)1 << 27) / ng / 128 * 128);
    chunk = std::min<int64_t>(chunk, tc_rows_pad(m));
    x->slack.reserve((size_t)chunk);
    x->gmin.reserve((size_t)chunk * ng);
    for (int64_t r0 = 0; r0 < m; r0 += chunk) {
      const int64_t mm = std::min(chunk, m - r0);
      tc_prepare(x, A + r0 * D, mm, x->a_tc, false, bop.center.p);
      launch_l2_tc(x->a_tc.hi.p, x->a_tc.lo.p, x->a_tc.norm.p, mm, bop.hi.p, bop.lo.p, bop.norm.p, n, D,
                   nullptr, 0, x->stream, x->gmin.p);
      launch_slack(x->a_tc.norm.p, mm, bop.maxnorm, D, x->slack.p, x->stream);
      launch_select_groups(x->gmin.p, mm, n, k, A + r0 * D, B, D, out_idx + r0 * k,
                           out_d64 ? out_d64 + r0 * k : nullptr, x->slack.p, x->stream);
    }
    if (sync) check_knn_flag(x);
    return;
  }
  // int8 exact-split filter (rotate.cu distance mode) for long rows, where the 3-pass tf32 window
  // (gamma_3 ~ 6 Dp 2^-23 of the norms) holds hundreds of near-ties: the exact split bounds the
  // dot product to 9 D 2^-42 of the slice scales, so the window is the fp32 rounding of d_hat and
  // the fp64 certification sees ~k columns (knn_path 6 forces it; DADE_OPT_KNN_I8 = 1 uses it for
  // D >= 512 with the group-minima select). Off by default: measured on C3 (1,000 x 4,096 x 960,
  // k = 64) the probe takes 0.334 ms against the 3-pass tf32 filter's 0.285 — the group-minima
  // select (0.27 ms) does not shrink with the window, and the int8 split + GEMM (0.23 ms) costs
  // more than the tf32 split + 3-pass GEMM (0.14 ms)
  {
    const int64_t ngr = (n + 31) / 32;
    const bool i8 = k > 1 && k <= ngr && ngr <= 1024 && D % 16 == 0 && D <= kRotMaxD &&
                    (path ? path == 6 : (passes == 3 && D >= 512 && x->opt.knn_i8));
    if (i8) {
      tc_prepare_i8(x, B, const_cast<TcOp&>(bop));
      const int64_t budget = (int64_t)1 << 29;
      int64_t chunk = std::max<int64_t>(128, budget / std::max<int64_t>(n, 1) / 128 * 128);
      chunk = std::min<int64_t>(std::min<int64_t>(chunk, 16384), tc_rows_pad(m));
      x->dmat.reserve((size_t)chunk * n);
      x->gmin.reserve((size_t)chunk * ngr);
      x->slack.reserve((size_t)chunk);
      x->an64.reserve((size_t)chunk);
      x->ovf.reserve((size_t)chunk + 1);
      if (!x->flag.p) {
        x->flag.reserve(1);
        DADE_CK(cudaMemsetAsync(x->flag.p, 0, sizeof(int), x->stream));
      }
      for (int64_t r0 = 0; r0 < m; r0 += chunk) {
        const int64_t mm = std::min(chunk, m - r0);
        launch_cnorm64(A + r0 * D, mm, mm, D, bop.mu64.p, x->an64.p, x->stream);
        DADE_CK(cudaMemsetAsync(x->gmin.p, 0x7f, sizeof(float) * (size_t)mm * ngr, x->stream));
        launch_dist_i8(A + r0 * D, mm, D, bop.mu64.p, x->an64.p, x->rot_ws, bop.i8b, bop.bn64.p, n, x->dmat.p,
                       reinterpret_cast<unsigned*>(x->gmin.p), ngr, x->stream);
        launch_slack_i8(x->an64.p, x->rot_ws.ae.p, mm, bop.i8e.p, bop.i8bmax.p, D, x->slack.p, x->stream);
        launch_select_gmin(x->dmat.p, x->gmin.p, 5, mm, n, k, A + r0 * D, B, D, out_idx + r0 * k,
                           out_d64 ? out_d64 + r0 * k : nullptr, x->flag.p, x->slack.p, x->ovf.p, x->ovf.p + 1,
                           x->stream);
      }
      if (sync) check_knn_flag(x);
      return;
    }
  }
  // floats of d_hat per chunk (2 GiB; DADE_OPT_DHAT_CHUNK_MB overrides, e.g. an L2-sized chunk)
  const int64_t budget = x->opt.dhat_chunk_mb ? (int64_t)x->opt.dhat_chunk_mb << 18 : (int64_t)1 << 29;
  int64_t chunk = std::max<int64_t>(128, budget / std::max<int64_t>(n, 1) / 128 * 128);
  const int cand_cap = 4096;
  if (k > 1 || out_d64) {
    chunk = std::min<int64_t>(chunk, 16384);
    x->cand.reserve((size_t)std::min(chunk, tc_rows_pad(m)) * cand_cap);
  }
  chunk = std::min<int64_t>(chunk, tc_rows_pad(m));
  x->dmat.reserve((size_t)chunk * n);
  x->slack.reserve((size_t)chunk);
  // group minima over 32 columns (64 beyond 32,768 columns, so a row has <= 1024 groups)
  const int gshift = (n + 31) / 32 > 1024 ? 6 : 5;
  const int64_t ngrp = (n + (1 << gshift) - 1) >> gshift;
  x->gmin.reserve((size_t)chunk * ngrp);
  if (!x->flag.p) {
    x->flag.reserve(1);
    DADE_CK(cudaMemsetAsync(x->flag.p, 0, sizeof(int), x->stream));
  }
  // fp16 operands for the d_hat writer (DADE_OPT_DHAT_H16; 1-pass filter + group-minima select):
  // the same power-of-two scaled operands, d_hat formula and slack as the fused fp16 filter
  // (probe_fz.cu MODE 1), half the operand bytes and half the MMAs of the tf32 hi x hi filter
  const bool h16_want = x->opt.dhat_h16 && passes == 1 && k > 1 && n <= 32768 &&
                        (int64_t)k * x->opt.gmin_ratio <= ngrp && ngrp <= 1024;
  if (h16_want) tc_prepare_h16(x, B, const_cast<TcOp&>(bop));
  const bool h16 = h16_want && bop.h16_ok;
  for (int64_t r0 = 0; r0 < m; r0 += chunk) {
    const int64_t mm = std::min(chunk, m - r0);
    if (h16) {
      const int64_t rp = fz_rows_pad(mm);
      x->a_tc.h16.reserve((size_t)rp * fz_nkc(D, 1) * 32);
      x->a_tc.hinv.reserve((size_t)rp);
      x->a_tc.norm.reserve((size_t)rp);
      launch_split_h16(A + r0 * D, mm, D, bop.center.p, x->a_tc.h16.p, x->a_tc.norm.p, x->a_tc.hinv.p, 0.f,
                       x->stream);
      launch_l2_tc(reinterpret_cast<const float*>(x->a_tc.h16.p), nullptr, x->a_tc.norm.p, mm,
                   reinterpret_cast<const float*>(bop.h16.p), nullptr, bop.norm.p, n, D, x->dmat.p, n, x->stream,
                   x->gmin.p, 1, gshift, x->a_tc.hinv.p, bop.hinv_b, x->opt.dhat_h16 >= 2 ? x->opt.dhat_h16 : 1);
      launch_slack_h16(x->a_tc.norm.p, x->a_tc.hinv.p, mm, bop.maxnorm, bop.hinv_b, D, x->slack.p, x->stream);
      x->ovf.reserve((size_t)chunk + 1);
      launch_select_gmin(x->dmat.p, x->gmin.p, gshift, mm, n, k, A + r0 * D, B, D, out_idx + r0 * k,
                         out_d64 ? out_d64 + r0 * k : nullptr, x->flag.p, x->slack.p, x->ovf.p,
                         x->ovf.p + 1, x->stream);
      continue;
    }
    tc_prepare(x, A + r0 * D, mm, x->a_tc, false, bop.center.p);
    // the group-minima select bounds the k-th smallest d_hat by the k-th smallest GROUP minimum,
    // loose when k nears the number of groups (C3: k = 64 of 128); the histogram select
    // (k_select_small, DADE_OPT_GMIN_RATIO > 1 moves rows to it) measured slower even there
    // (C3 probe 0.28 -> 0.45 ms, C2 at nprobe 64 0.555 -> 0.61 ms)
    const bool use_gmin = k > 1 && (int64_t)k * x->opt.gmin_ratio <= ngrp && ngrp <= 1024;
    // the warp-specialised d_hat writer pays off for very wide rows (measured on C5, 65,536
    // columns: 1.42 -> 1.19 ms); up to 16,384 columns the one-tile-per-CTA kernel with 3 CTAs/SM
    // is faster (C2 68 vs 97 us, C4 222 vs 358 us, C3 36 vs 42 us)
    if (use_gmin && n > 32768 && x->opt.dhat_ares && dhat_ares_ok(D, passes))
      launch_dhat_ares(x->a_tc.hi.p, x->a_tc.norm.p, mm, bop.hi.p, bop.norm.p, n, D, x->dmat.p, n, x->gmin.p,
                       gshift, x->stream);
    else if (use_gmin && n > 32768)
      launch_dhat_tc(x->a_tc.hi.p, x->a_tc.lo.p, x->a_tc.norm.p, mm, bop.hi.p, bop.lo.p, bop.norm.p, n, D,
                     x->dmat.p, n, x->gmin.p, gshift, passes, x->stream);
    else
      launch_l2_tc(x->a_tc.hi.p, x->a_tc.lo.p, x->a_tc.norm.p, mm, bop.hi.p, bop.lo.p, bop.norm.p, n, D,
                   x->dmat.p, n, x->stream, use_gmin ? x->gmin.p : nullptr, passes, gshift);
    launch_slack(x->a_tc.norm.p, mm, bop.maxnorm, D, x->slack.p, x->stream, passes);
    if (use_gmin) {
      x->ovf.reserve((size_t)chunk + 1);
      launch_select_gmin(x->dmat.p, x->gmin.p, gshift, mm, n, k, A + r0 * D, B, D, out_idx + r0 * k,
                         out_d64 ? out_d64 + r0 * k : nullptr, x->flag.p, x->slack.p, x->ovf.p,
                         x->ovf.p + 1, x->stream);
      continue;
    }
    if (k == 1 && !out_d64)
      launch_argmin_exact(x->dmat.p, mm, n, A + r0 * D, B, D, out_idx + r0, x->flag.p, x->stream,
                          x->slack.p);
    else
      launch_select_exact(x->dmat.p, mm, n, k, A + r0 * D, B, D, out_idx + r0 * k,
                          out_d64 ? out_d64 + r0 * k : nullptr, x->cand.p, cand_cap, x->flag.p,
                          x->stream, x->slack.p);
  }
  if (sync) check_knn_flag(x);
}

void exact_knn(dade_index* x, const float* A, int64_t m, const float* B, int64_t n, int k,
               int32_t* out_idx, double* out_d64) {
  TcOp bop;
  tc_prepare(x, B, n, bop, true);
  exact_knn(x, A, m, B, n, k, out_idx, out_d64, bop);
  bop.release();
}

// passes of the probe's tensor-core filter: 1 (tf32 hi parts only: 1/3 of the MMAs and 1/2 of the
// operand bytes, a ~40x wider but still rigorous certified window; the fp64 re-rank keeps the
// result exact) unless DADE_OPT_PROBE_PASSES = 3
// tf32 passes of the probe filter: 1 (hi x hi) with its wider certified window, or 3 (split
// precision) when the rows are long — at D = 960 the 1-pass window holds so many near-ties that
// the fp64 certification dominates (measured C3 step 1.95 -> 1.83 ms with 3 passes; C2, C4 and
// the C5 shard, D <= 256, are faster with 1). DADE_OPT_PROBE_PASSES overrides.
int probe_passes(const dade_index* x) {
  return x->opt.probe_passes ? x->opt.probe_passes : (x->D >= 512 ? 3 : 1);
}

// Installs x->mean / x->R on the device. A new rotation invalidates everything built in the old
// basis: the rotated layout (and the IVF that owns it), the calibration table and the row norms.
void upload_rotation(dade_index* x) {
  const int D = x->D;
  x->has_ivf = false;
  x->has_cal = false;
  x->xnorm_ok = false;
  x->has_pq = false;  // codebooks live in the old basis
  x->has_graph = false;
  x->pq_codes_ok = false;
  x->has_calq = false;
  x->R_d.reserve((size_t)D * D);
  x->mean_d.reserve(D);
  DADE_CK(cudaMemcpyAsync(x->R_d.p, x->R.data(), sizeof(double) * D * D, cudaMemcpyHostToDevice, x->stream));
  DADE_CK(cudaMemcpyAsync(x->mean_d.p, x->mean.data(), sizeof(double) * D, cudaMemcpyHostToDevice, x->stream));
  rot_prepare(x->rot_op, x->R_d.p, D, x->stream);  // R's slices for the tensor-core rotation
  DADE_CK(cudaStreamSynchronize(x->stream));
  x->has_rot = true;
}

// PQ code rows of the current layout (R30): codes | fp32 reconstruction error, stride bytes
void pq_encode_layout(dade_index* x) {
  x->pq_codes_ok = false;
  x->has_calq = false;
  if (!x->has_pq || !x->has_ivf) return;
  x->pq_codes.reserve((size_t)x->n * x->pq_stride);
  DADE_CK(cudaMemsetAsync(x->pq_codes.p, 0, (size_t)x->n * x->pq_stride, x->stream));
  launch_pq_assign(x->layout.p, true, x->n, x->D, x->pq_m, x->pq_Cd.p, x->pq_codes.p, x->pq_stride, x->stream);
  launch_pq_err(x->layout.p, x->n, x->D, x->pq_m, x->pq_Cd.p, x->pq_codes.p, x->pq_stride, x->pq_eo, x->stream);
  DADE_CK(cudaStreamSynchronize(x->stream));
  x->pq_codes_ok = true;
}

void install_pq(dade_index* x, int m, const float* C) {
  const int D = x->D;
  DADE_REQUIRE(m >= 1 && D % m == 0 && D / m <= 32, DADE_ERR_ARG, "pq: m must divide D with D/m <= 32");
  for (size_t i = 0; i < (size_t)D * 256; ++i) DADE_REQUIRE(std::isfinite(C[i]), DADE_ERR_NONFINITE, "pq: non-finite codebook");
  x->pq_m = m;
  x->pq_eo = (m + 3) & ~3;
  x->pq_stride = (x->pq_eo + 4 + 15) & ~15;
  DADE_REQUIRE(x->pq_stride <= 256, DADE_ERR_UNSUPPORTED, "pq: more than 248 subspaces");
  x->pq_C.assign(C, C + (size_t)D * 256);
  x->pq_Cd.reserve((size_t)D * 256);
  DADE_CK(cudaMemcpyAsync(x->pq_Cd.p, x->pq_C.data(), sizeof(float) * D * 256, cudaMemcpyHostToDevice, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  x->has_pq = true;
  pq_encode_layout(x);
}

// R from a covariance (eigenvectors by descending eigenvalue, sign rule R18)
void rotation_from_cov(int D, std::vector<double> cov, std::vector<double>& R, std::vector<double>& lam) {
  std::vector<double> ev(D), V((size_t)D * D);
  for (int a = 0; a < D; ++a)
    for (int b = a + 1; b < D; ++b) cov[(size_t)b * D + a] = cov[(size_t)a * D + b];
  sym_eig(D, cov.data(), ev.data(), V.data());
  std::vector<int> order(D);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ev[a] > ev[b]; });
  R.assign((size_t)D * D, 0.0);
  lam.assign(D, 0.0);
  for (int i = 0; i < D; ++i) {
    const double* col = &V[(size_t)order[i] * D];
    int jm = 0;
    for (int j = 1; j < D; ++j)
      if (std::fabs(col[j]) > std::fabs(col[jm])) jm = j;
    const double sg = col[jm] < 0 ? -1.0 : 1.0;
    for (int j = 0; j < D; ++j) R[(size_t)i * D + j] = sg * col[j];
    lam[i] = ev[order[i]];
  }
}

int64_t sample_count(int64_t n_total, int64_t sample_size) {
  return std::min<int64_t>(n_total, sample_size > 0 ? sample_size : 1000000);
}

__global__ void k_ids_from_idx(const int32_t* idx, const double* d64, int64_t cnt, int64_t id_base,
                               int64_t* ids, float* dists) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = idx[i];
    ids[i] = c < 0 ? -1 : id_base + c;
    dists[i] = c < 0 ? INFINITY : (float)d64[i];
  }
}

// a4 + a5: q~ = R(q - mu) (side stream) and the exact probes (main stream), joined on the main
// stream. qrot: device nq x D, probes: device nq x nprobe.
void ensure_side(dade_index* x) {
  if (!x->side) {
    DADE_CK(cudaStreamCreateWithFlags(&x->side, cudaStreamNonBlocking));
    DADE_CK(cudaEventCreateWithFlags(&x->fork, cudaEventDisableTiming));
    DADE_CK(cudaEventCreateWithFlags(&x->join, cudaEventDisableTiming));
  }
}

void prepare(dade_index* x, const float* Q, int nq, int nprobe, float* qrot, int32_t* probes, bool stats) {
  const int D = x->D;
  cudaStream_t st = x->stream;
  // non-finite queries latch error 3 in the flag (reported at the next synchronising call)
  if (!x->flag.p) {
    x->flag.reserve(1);
    DADE_CK(cudaMemsetAsync(x->flag.p, 0, sizeof(int), st));
  }
  ensure_side(x);
  DADE_CK(cudaEventRecord(x->fork, st));
  DADE_CK(cudaStreamWaitEvent(x->side, x->fork, 0));
  launch_check_finite(Q, (int64_t)nq * D, x->flag.p, x->side, 3);
  launch_rotate(x->rot_op, x->rot_ws_side, Q, nullptr, nq, x->mean_d.p, qrot, nullptr, x->side);
  if (stats) DADE_CK(cudaEventRecord(x->ev[1], x->side));
  DADE_CK(cudaEventRecord(x->join, x->side));
  if (x->nlist == 1) {
    DADE_CK(cudaMemsetAsync(probes, 0, sizeof(int32_t) * nq, st));
  } else {
    exact_knn(x, Q, nq, x->cent.p, x->nlist, nprobe, probes, nullptr, x->cent_tc, false, probe_passes(x));
  }
  DADE_CK(cudaStreamWaitEvent(st, x->join, 0));
}

// qrot_in / probes_in (device, optional): queries already rotated and probed (dade_prepare, e.g.
// on another rank) — only the scan runs.
#ifndef DADE_C0_MULT  // R13: c0 = 4K (experiment builds may change it)
#define DADE_C0_MULT 4
#endif

// dade_search_host's pipeline depth (DADE_OPT_HOST_CHUNKS, default 1): on C2
// (tools/e2e_breakdown.py) a search cut in two costs 0.19 ms more on the device (the scan's
// per-launch tail: 0.36 ms at 5,000 queries vs 0.55 ms at 10,000) while the H2D it could hide is
// 0.20 ms, so chunking does not pay at these batch sizes.
// DADE_OPT_SCAN_TAIL = X: the last X queries of a batch are scanned by a concurrent second launch
// with 4 warps per query. Measured on C2: X = 500 -0.7% (noise), 1,000 +4%, 2,000 +13%; C4 X =
// 1,000 -0.5% — the one-warp scan is throughput-bound, not tail-bound, so it stays off.
// DADE_OPT_SCAN_ORDER: the order in which the persistent scan takes the queries (results do not
// depend on it). 2 (default): longest candidate stream first (a counting sort on the stream length,
// launch_query_order_lpt) — the last wave of the persistent grid then holds the shortest queries;
// measured (profiles/r02_scan_order_c{2,4}.jsonl): C4 scan 1.196 -> 1.103 ms, step 1.460 -> 1.384;
// C2 scan 0.553 -> 0.500, step 0.700 -> 0.664. 1: grouped by nearest probed list (C2 scan unchanged,
// C4 -3.6%, +20 us of ordering kernels). 0: as given.
int scan_tail(const dade_index* x, int nq) { return std::max(0, std::min(x->opt.scan_tail, nq)); }
bool scan_order(const dade_index* x, int nq) { return x->opt.scan_order != 0 && nq > 0; }
// dade_search_host's rotation + probe chunks when the search itself is not chunked (default 2 for
// batches of >= 4,096 queries)
int host_prep_chunks(const dade_index* x, int nq) {
  if (x->opt.host_prep_chunks > 0) return std::max(1, std::min(x->opt.host_prep_chunks, std::max(nq, 1)));
  return nq >= 4096 ? 2 : 1;
}
int host_chunks(const dade_index* x, int nq) { return std::max(1, std::min(x->opt.host_chunks, std::max(nq, 1))); }

// One phase of a sharded search (R32): the epochs it runs, the queue it starts from, the exchanged
// queue bounding tau, the per-shard c0; counters are zeroed by the first phase and read by the last.
struct Phase {
  int ep_first = 0, ep_end = 1 << 30;
  const int64_t* init_ids = nullptr;
  const float* init_d = nullptr;
  const int64_t* cap_ids = nullptr;
  const float* cap_d = nullptr;
  int c0 = 0;
  bool first = true, last = true;
};

struct DecisionLog {
  int32_t* buf = nullptr;  // device, cap x 3 int32
  int64_t cap = 0;
  int64_t* count = nullptr;  // host out
};

void do_search(dade_index* x, const float* Q, int nq, int K, int nprobe, int delta_d, double alpha,
               int64_t* ids, float* dists, dade_stats* stats, int method = DADE_METHOD_BSA_P,
               const float* qrot_in = nullptr, const int32_t* probes_in = nullptr,
               const DecisionLog* dlog = nullptr, const Phase* phase = nullptr) {
  const Phase ph0;
  const Phase& ph = phase ? *phase : ph0;
  const int D = x->D;
  DADE_REQUIRE(x->has_ivf && x->has_rot, DADE_ERR_STATE, "search before build_ivf");
  DADE_REQUIRE(nq >= 0, DADE_ERR_ARG, "nq < 0");
  if (nq > 0) {
    if (!qrot_in) need(Q, "Q");
    else need(probes_in, "probes");
    need(ids, "ids"); need(dists, "dists");
  }
  DADE_REQUIRE(K >= 1, DADE_ERR_ARG, "K < 1");
  DADE_REQUIRE(K <= DADE_MAX_K, DADE_ERR_UNSUPPORTED, "K > DADE_MAX_K");
  DADE_REQUIRE(nprobe >= 1 && nprobe <= x->nlist, DADE_ERR_ARG, "nprobe not in [1, nlist]");
  DADE_REQUIRE(delta_d >= 16 && delta_d % 16 == 0 && D % delta_d == 0, DADE_ERR_ARG,
               "delta_d must be a positive multiple of 16 dividing D");
  DADE_REQUIRE(method == DADE_METHOD_BSA_P || method == DADE_METHOD_ADSAMPLING || method == DADE_METHOD_BSA_RES ||
               method == DADE_METHOD_BSA_Q, DADE_ERR_ARG, "unknown method");
  const bool pqm = method == DADE_METHOD_BSA_Q;
  if (method == DADE_METHOD_BSA_P || pqm)
    DADE_REQUIRE(alpha >= 0.0 && alpha < 1.0, DADE_ERR_ARG, "significance not in [0,1)");
  else
    DADE_REQUIRE(alpha > 0.0 && std::isfinite(alpha), DADE_ERR_ARG, "eps0 / m must be positive");
  if (method == DADE_METHOD_BSA_RES)
    DADE_REQUIRE(x->has_lam, DADE_ERR_STATE, "BSA-res needs the rotation's eigenvalues");
  const int nsteps = D / delta_d;
  DADE_REQUIRE(nsteps <= DADE_MAX_STEPS, DADE_ERR_UNSUPPORTED, "D/delta_d > DADE_MAX_STEPS");
  const int dd = delta_d / 16;
  const bool prune = alpha > 0.0 && (pqm || nsteps > 1);
  if (pqm) {
    DADE_REQUIRE(x->has_pq && x->pq_codes_ok, DADE_ERR_STATE, "BSA-q needs PQ codebooks (dade_train_pq / dade_set_pq)");
    if (prune) {
      DADE_REQUIRE(x->has_calq, DADE_ERR_STATE, "BSA-q with significance > 0 requires dade_calibrate_pq");
      DADE_REQUIRE(x->calqK == K, DADE_ERR_STATE, "K differs from the PQ-calibrated K");
    }
  }
  if (prune && method == DADE_METHOD_BSA_P) {
    DADE_REQUIRE(x->has_cal, DADE_ERR_STATE, "significance > 0 requires calibration");
    DADE_REQUIRE(x->calK == K, DADE_ERR_STATE, "K differs from the calibrated K");
  }
  if (nq == 0) return;
  cudaStream_t st = x->stream;
  const bool evs = stats || x->timing;  // stage events (no synchronisation unless stats)
  if (evs) {
    for (auto& e : x->ev)
      if (!e) DADE_CK(cudaEventCreate(&e));
    DADE_CK(cudaEventRecord(x->ev[0], st));
  }
  const float* qrot = qrot_in;
  const int32_t* probes = probes_in;
  if (!qrot_in) {
    x->qrot.reserve((size_t)nq * D);
    x->probes.reserve((size_t)nq * nprobe);
    prepare(x, Q, nq, nprobe, x->qrot.p, x->probes.p, evs);
    qrot = x->qrot.p;
    probes = x->probes.p;
  } else if (evs) {
    DADE_CK(cudaEventRecord(x->ev[1], st));
  }
  // the scan's query order (counted with the probe stage, so the scan's events time k_scan alone)
  const int32_t* order = nullptr;
  if (scan_order(x, nq)) {
    x->order.reserve((size_t)nq);
    if (x->opt.scan_order == 2) {  // longest candidate stream first
      x->ordcnt.reserve((size_t)1024 + nq);
      launch_query_order_lpt(probes, nq, nprobe, x->off_d.p, (int64_t)nprobe * x->n / std::max(1, x->nlist),
                             x->ordcnt.p, x->order.p, st);
    } else {
      x->ordcnt.reserve((size_t)x->nlist);
      launch_query_order(probes, nq, nprobe, x->nlist, x->ordcnt.p, x->order.p, st);
    }
    order = x->order.p;
  }
  if (evs) DADE_CK(cudaEventRecord(x->ev[2], st));
  // step table (R4, R5): alpha_s = alpha*delta_d/D, k = clamp(ceil((1-alpha_s)*n0), 1, n0)
  ScanParams p{};
  p.qrot = qrot; p.probes = probes; p.off = x->off_d.p; p.row_id = x->row_id_d.p;
  p.layout = x->layout.p; p.n = x->n; p.D = D; p.nq = nq; p.nprobe = nprobe; p.K = K;
  // alpha = 0 (or a single step): nothing can be pruned; the kernel then runs with 16-dim
  // steps (no classifier fires: m1 = 1, beta' = -inf), which serves every delta_d | D.
  p.dd = prune ? dd : 1; p.nsteps = prune ? nsteps : D / 16; p.c0 = DADE_C0_MULT * K; p.prune = prune ? 1 : 0;
  if (ph.c0 > 0) p.c0 = ph.c0;
  p.ep_first = ph.ep_first;
  p.ep_end = ph.ep_end;
  p.init_ids = ph.init_ids;
  p.init_d = ph.init_d;
  p.cap_ids = ph.cap_ids;
  p.cap_d = ph.cap_d;
  if (pqm) {
    // BSA-q: one classifier on the ADC distance in stage 1 (R29), then exact distances — no
    // classifier in the gather rounds (spacing = all blocks, one step)
    p.dd = D / 16;
    p.nsteps = 1;
    p.pq = 1;
    p.pq_codes = x->pq_codes.p;
    p.pq_stride = x->pq_stride;
    p.pq_eo = x->pq_eo;
    p.pq_m = x->pq_m;
    p.pq_ds = D / x->pq_m;
    p.pq_C = x->pq_Cd.p;
    p.pq_m1 = (float)x->mq[0];
    p.pq_m2 = (float)x->mq[1];
    if (prune) {  // beta' = v[k-1], k = clamp(ceil((1 - alpha) n0), 1, n0): one classifier, alpha_s = alpha
      long k = (long)std::ceil((1.0 - alpha) * (double)x->n0q);
      k = std::min<long>(std::max<long>(k, 1), x->n0q);
      p.pq_beta = (float)x->vq[(size_t)(k - 1)];
    } else {
      p.pq_beta = -INFINITY;
    }
    p.pq_lg = 0;  // lanes per survivor of the gather rounds: set with the kernel's LA (scan.cu launch_k)
  }
  p.avg_stream = (int64_t)nprobe * x->n / std::max(1, x->nlist);
  for (int s = 1; s < p.nsteps; ++s) {
    if (prune && method == DADE_METHOD_ADSAMPLING) {  // m1_d = (D/d)/(1 + eps0/sqrt(d))^2, beta = 0
      const double d = (double)s * delta_d;
      p.m1[s - 1] = (float)((D / d) / ((1.0 + alpha / std::sqrt(d)) * (1.0 + alpha / std::sqrt(d))));
      p.beta[s - 1] = 0.f;
    } else if (prune && method == DADE_METHOD_BSA_RES) {  // the residual test uses qconst instead
      p.m1[s - 1] = 1.f;
      p.beta[s - 1] = 0.f;
    } else if (prune) {
      const int idx = (s * delta_d) / 16 - 1;
      const double alpha_s = (alpha * delta_d) / D;
      long k = (long)std::ceil((1.0 - alpha_s) * (double)x->n0);
      k = std::min<long>(std::max<long>(k, 1), x->n0);
      p.m1[s - 1] = (float)x->m1[idx];
      p.beta[s - 1] = (float)x->v[(size_t)idx * x->n0 + (k - 1)];
    } else {
      p.m1[s - 1] = 1.f;
      p.beta[s - 1] = -INFINITY;
    }
  }
  p.out_ids = ids; p.out_d = dists;
  if (stats) {
    x->counters.reserve(4 + DADE_MAX_STEPS + 8);
    if (ph.first)
      DADE_CK(cudaMemsetAsync(x->counters.p, 0, sizeof(unsigned long long) * (4 + DADE_MAX_STEPS + 8), st));
    p.counters = x->counters.p;
  }
  if (prune && method == DADE_METHOD_BSA_RES) {
    if (!x->xnorm_ok) {
      x->xnorm.reserve((size_t)std::max<int64_t>(x->n, 1));
      launch_row_norms(x->layout.p, x->n, D, x->xnorm.p, st);
      x->xnorm_ok = true;
    }
    x->lam_d.reserve(D);
    DADE_CK(cudaMemcpyAsync(x->lam_d.p, x->lam.data(), sizeof(double) * D, cudaMemcpyHostToDevice, st));
    x->qconst.reserve((size_t)nq * (nsteps - 1) + 1);
    launch_res_consts(qrot, nq, D, delta_d, x->lam_d.p, alpha, x->qconst.p, st);
    p.residual = 1;
    p.xnorm = x->xnorm.p;
    p.qconst = x->qconst.p;
  }
  // work counters: [0] the main scan, [1] the tail scan; reserved (and zeroed) before any pointer
  // into the buffer is taken
  x->work.reserve(2);
  DADE_CK(cudaMemsetAsync(x->work.p, 0, 2 * sizeof(int), st));
  p.work_counter = x->work.p;
  p.order = order;
  p.g_force = x->opt.scan_warps;
  // stage 1 list-major (p1.cu, DADE_OPT_SCAN_P1 = 1): each probed list's first-step rows read once
  // for every query that probes it (BSA-p / ADSampling). Off by default: measured on C4 it halves
  // the scan's DRAM bytes (5.20 -> 2.59 GB) but the scan is bound by its survivors' gather round
  // trips (1.68 -> 1.44 ms under ncu) and the precompute costs more than that (0.95 ms)
  {
    const int unit = p.pq ? 0 : (p.dd % 4 == 0 ? 4 : p.dd % 2 == 0 ? 2 : 1);  // the scan's staging unit
    const bool want = x->opt.scan_p1 == 1;
    if (want && unit && !p.residual && !p.pq && x->nlist > 1) {
      const int64_t avg = std::max<int64_t>(1, x->n / std::max(1, x->nlist));
      const int64_t cap = std::min<int64_t>((int64_t)nq * nprobe * avg * 2 + 65536, (int64_t)1 << 31);
      x->p1.reserve((size_t)cap + 4);
      x->p1_base.reserve((size_t)nq + 1);
      x->p1_scr.reserve(p1_scratch_ints(nq, nprobe, x->nlist));
      x->p1_total.reserve(1);
      p1_launch(x->layout.p, x->n, x->off_d.p, x->nlist, probes, nq, nprobe, qrot, D, unit, x->p1_scr.p,
                x->p1_base.p, x->p1.p, cap, x->p1_total.p, st);
      p.p1 = x->p1.p;
      p.p1_base = x->p1_base.p;
      p.p1_total = x->p1_total.p;
      p.p1_cap = cap;
    }
  }
  if (dlog) {
    x->dlog_n.reserve(1);
    DADE_CK(cudaMemsetAsync(x->dlog_n.p, 0, sizeof(unsigned long long), st));
    p.dlog = dlog->buf;
    p.dlog_cap = dlog->cap;
    p.dlog_n = x->dlog_n.p;
  }
  const int tail = dlog ? 0 : scan_tail(x, nq);
  if (tail > 0 && tail < nq && !order) {
    // the last `tail` queries run as a second scan with 4 warps per query on the side stream:
    // its CTAs take the SM slots the first scan's warps free as they run out of queries, so the
    // first scan's tail is filled and the second's is 4x shorter
    const int q0 = nq - tail;
    ScanParams p2 = p;
    p.nq = q0;
    p2.nq = tail;
    p2.qrot += (size_t)q0 * D;
    p2.probes += (size_t)q0 * nprobe;
    p2.out_ids += (size_t)q0 * K;
    p2.out_d += (size_t)q0 * K;
    if (p2.p1_base) p2.p1_base += q0;
    if (p2.qconst) p2.qconst += (size_t)q0 * (nsteps - 1);
    p2.work_counter = x->work.p + 1;
    p2.g_force = 4;
    ensure_side(x);
    DADE_CK(cudaEventRecord(x->fork, st));
    DADE_CK(cudaStreamWaitEvent(x->side, x->fork, 0));
    launch_scan(p, st);
    launch_scan(p2, x->side);
    DADE_CK(cudaEventRecord(x->join, x->side));
    DADE_CK(cudaStreamWaitEvent(st, x->join, 0));
  } else {
    launch_scan(p, st);
  }
  if (evs && !stats) DADE_CK(cudaEventRecord(x->ev[3], st));
  if (dlog) {
    unsigned long long cnt = 0;
    DADE_CK(cudaMemcpyAsync(&cnt, x->dlog_n.p, sizeof(cnt), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    *dlog->count = (int64_t)cnt;
  }
  if (stats && ph.last) {
    DADE_CK(cudaEventRecord(x->ev[3], st));
    unsigned long long c[4 + DADE_MAX_STEPS + 8];
    DADE_CK(cudaMemcpyAsync(c, x->counters.p, sizeof(c), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    check_knn_flag(x);
    memset(stats, 0, sizeof(*stats));
    stats->tested = (int64_t)c[0];
    stats->survivors = (int64_t)c[1];
    // dims read: a candidate pruned at step s read s*delta_d dims; a survivor read all D
    int64_t dims = (int64_t)c[1] * D;
    for (int s = 1; s < DADE_MAX_STEPS; ++s) dims += (int64_t)c[4 + s] * s * (p.dd * 16);
    stats->dims_scanned = dims;
    stats->n_epochs = (int32_t)c[3];
    for (int s = 0; s < DADE_MAX_STEPS; ++s) stats->pruned_at_step[s] = (int64_t)c[4 + s];
    stats->n_steps = pqm ? 1 : nsteps;
    cudaEventElapsedTime(&stats->ms_rotate, x->ev[0], x->ev[1]);  // concurrent with the probe
    cudaEventElapsedTime(&stats->ms_probe, x->ev[0], x->ev[2]);
    cudaEventElapsedTime(&stats->ms_scan, x->ev[2], x->ev[3]);
    cudaEventElapsedTime(&stats->ms_total, x->ev[0], x->ev[3]);
  }
}

// Collective search (dade_set_comm with nranks > 1): every rank passes the same
// queries. Rank r rotates and probes its block of ceil(nq / S) queries (a4 + a5), the blocks of
// q~ and probe lists are all-gathered in place, every rank scans ALL queries over its own shard
// (a6-a8), and the local top-K lists are all-gathered and merged by (dist, id) (a9, k_merge_topk).
// mu, R and the centroids are replicated, so a query's q~ and probes are the same whichever rank
// prepared them; with alpha = 0 the result equals the unsharded search.
void do_search_collective(dade_index* x, const float* Q, int nq, int K, int nprobe, int delta_d, double alpha,
                          int64_t* ids, float* dists, dade_stats* stats, int method) {
  const int S = comm_size(x->comm), r = comm_rank(x->comm);
  const int D = x->D;
  cudaStream_t st = x->stream;
  DADE_REQUIRE(x->has_ivf && x->has_rot, DADE_ERR_STATE, "search before build_ivf");
  DADE_REQUIRE(nq >= 0, DADE_ERR_ARG, "nq < 0");
  DADE_REQUIRE(nprobe >= 1 && nprobe <= x->nlist, DADE_ERR_ARG, "nprobe not in [1, nlist]");
  DADE_REQUIRE(K >= 1 && K <= DADE_MAX_K, DADE_ERR_ARG, "K not in [1, DADE_MAX_K]");
  if (nq == 0) return;
  need(Q, "Q"); need(ids, "ids"); need(dists, "dists");
  const int per = (nq + S - 1) / S;
  const int lo = std::min(r * per, nq), hi = std::min(lo + per, nq);
  x->qrot.reserve((size_t)S * per * D);
  x->probes.reserve((size_t)S * per * nprobe);
  float* qr = x->qrot.p + (size_t)r * per * D;
  int32_t* pr = x->probes.p + (size_t)r * per * nprobe;
  if (hi > lo) prepare(x, Q + (size_t)lo * D, hi - lo, nprobe, qr, pr, false);
  comm_allgather(x->comm, qr, x->qrot.p, sizeof(float) * per * D, st);
  comm_allgather(x->comm, pr, x->probes.p, sizeof(int32_t) * per * nprobe, st);
  x->gids.reserve((size_t)S * nq * K);
  x->gdists.reserve((size_t)S * nq * K);
  int64_t* li = x->gids.p + (size_t)r * nq * K;
  float* ld = x->gdists.p + (size_t)r * nq * K;
  // the local scan over this shard in E + 1 phases (R32): epochs 0, 1, ..., E-1 one by one, then
  // the rest; after each of the first E phases the shards' queues are all-gathered and merged and
  // the merged K-th distance bounds every shard's tau from then on. Per-shard c0 = ceil(4K / S).
  // Each phase starts from this shard's own queue (init = its previous output, in place: a
  // query's queue is read at its start and written at its end by the same CTA).
  const int E = x->opt.shard_exchanges;
  Phase P;
  P.c0 = E > 0 ? (DADE_C0_MULT * K + S - 1) / S : DADE_C0_MULT * K;
  x->cap_ids.reserve((size_t)nq * K);
  x->cap_d.reserve((size_t)nq * K);
  for (int e = 0; e <= E; ++e) {
    P.ep_first = e;
    P.ep_end = e < E ? e + 1 : (1 << 30);
    P.first = e == 0;
    P.last = e == E;
    P.init_ids = e > 0 ? li : nullptr;
    P.init_d = e > 0 ? ld : nullptr;
    P.cap_ids = e > 0 ? x->cap_ids.p : nullptr;
    P.cap_d = e > 0 ? x->cap_d.p : nullptr;
    // scratch q~ / probes are the gathered buffers: the scan reads them in place
    do_search(x, nullptr, nq, K, nprobe, delta_d, alpha, li, ld, stats, method, x->qrot.p, x->probes.p, nullptr, &P);
    comm_allgather(x->comm, li, x->gids.p, sizeof(int64_t) * nq * K, st);
    comm_allgather(x->comm, ld, x->gdists.p, sizeof(float) * nq * K, st);
    if (e < E) launch_merge_topk(x->gids.p, x->gdists.p, S, nq, K, x->cap_ids.p, x->cap_d.p, st);
  }
  launch_merge_topk(x->gids.p, x->gdists.p, S, nq, K, ids, dists, st);
  if (stats) DADE_CK(cudaStreamSynchronize(st));
}

// any communicator makes the searches collective (a group of one runs the same schedule: the
// all-gathers are copies and the merge sorts one list — the single-GPU test of this path)
bool collective(const dade_index* x) { return x->comm != nullptr; }

// all-reduce (sum) of a HOST array over the index's communicator, staged through the device
template <typename T>
void allreduce_host(dade_index* x, T* a, size_t count) {
  if (!x->comm || count == 0) return;
  static_assert(sizeof(T) == 8, "fp64 / int64 only");
  x->red.reserve(count);
  DADE_CK(cudaMemcpyAsync(x->red.p, a, 8 * count, cudaMemcpyHostToDevice, x->stream));
  comm_allreduce_sum(x->comm, x->red.p, count, std::is_same<T, double>::value ? CommType::F64 : CommType::I64,
                     x->stream);
  DADE_CK(cudaMemcpyAsync(a, x->red.p, 8 * count, cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
}

// all-gather of a HOST array (same size on every rank) -> out[S * count]
template <typename T>
void allgather_host(dade_index* x, const T* a, size_t count, T* out) {
  const int S = comm_size(x->comm), r = comm_rank(x->comm);
  if (count == 0) return;
  const size_t words = (count * sizeof(T) + 7) / 8;
  x->red.reserve((size_t)S * words);
  char* base = reinterpret_cast<char*>(x->red.p);
  DADE_CK(cudaMemcpyAsync(base + (size_t)r * words * 8, a, sizeof(T) * count, cudaMemcpyHostToDevice, x->stream));
  comm_allgather(x->comm, base + (size_t)r * words * 8, base, words * 8, x->stream);
  for (int s = 0; s < S; ++s)
    DADE_CK(cudaMemcpyAsync(out + (size_t)s * count, base + (size_t)s * words * 8, sizeof(T) * count,
                            cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
}

}  // namespace

// ================================================================== lifecycle
extern "C" dade_status dade_create(int device, void* cuda_stream, int D, dade_index** out) {
  API_BEGIN
  need(out, "out");
  DADE_REQUIRE(D > 0, DADE_ERR_ARG, "D must be positive");
  DADE_REQUIRE(D % 16 == 0 && D <= 4096, DADE_ERR_UNSUPPORTED, "D must be a multiple of 16, <= 4096");
  int ndev = 0;
  DADE_CK(cudaGetDeviceCount(&ndev));
  DADE_REQUIRE(device >= 0 && device < ndev, DADE_ERR_ARG, "bad device ordinal");
  DeviceGuard g(device);
  auto* x = new dade_index();
  x->device = device;
  x->stream = (cudaStream_t)cuda_stream;
  x->D = D;
  *out = x;
  API_END
}

extern "C" dade_status dade_destroy(dade_index* x) {
  API_BEGIN
  if (!x) { g_err.clear(); return DADE_OK; }
  DeviceGuard g(x->device);
  cudaStreamSynchronize(x->stream);
  x->R_d.release(); x->mean_d.release(); x->cent.release(); x->layout.release();
  x->rot_op.release(); x->rot_ws.release(); x->rot_ws_side.release();
  x->off_d.release(); x->row_id_d.release(); x->qrot.release(); x->dmat.release();
  x->qbuf.release(); x->probes.release(); x->cand.release(); x->idx32.release();
  x->d64.release(); x->flag.release(); x->fflag.release(); x->work.release(); x->ovf.release(); x->counters.release(); x->dlog_n.release(); x->ids_tmp.release(); x->ordcnt.release(); x->order.release(); x->xnorm.release(); x->qconst.release(); x->lam_d.release();
  x->dists_tmp.release();
  x->cent_tc.release(); x->a_tc.release(); x->slack.release(); x->gmin.release(); x->fzseed.release();
  x->p1.release(); x->p1_base.release(); x->p1_scr.release(); x->p1_total.release(); x->an64.release();
  for (auto& e : x->ev)
    if (e) cudaEventDestroy(e);
  if (x->side) {
    cudaStreamSynchronize(x->side);
    cudaStreamDestroy(x->side);
    cudaEventDestroy(x->fork);
    cudaEventDestroy(x->join);
  }
  for (cudaStream_t s2 : {x->h2d, x->d2h})
    if (s2) {
      cudaStreamSynchronize(s2);
      cudaStreamDestroy(s2);
    }
  for (auto e : x->hev) cudaEventDestroy(e);
  x->gids.release(); x->gdists.release(); x->cap_ids.release(); x->cap_d.release(); x->red.release(); x->pq_Cd.release(); x->pq_codes.release();
  x->g_adj.release(); x->g_vlist.release(); x->g_vis.release();
  comm_destroy(x->comm);
  delete x;
  API_END
}

// ================================================================== a0 rotation
extern "C" dade_status dade_pca_mean_partial(dade_index* x, const float* X, int64_t n,
                                             int64_t id_base, int64_t n_total, int64_t sample_size,
                                             double* sum, int64_t* count) {
  API_BEGIN
  need(x, "index"); need(sum, "sum"); need(count, "count");
  DADE_REQUIRE(n >= 0 && id_base >= 0 && id_base + n <= n_total && n_total > 0, DADE_ERR_ARG,
               "bad row range");
  if (n > 0) need(X, "X");
  DeviceGuard g(x->device);
  const int D = x->D;
  if (n > 0) check_finite(x, X, n * D, "X");
  DBuf<double> s;
  s.reserve(D);
  int64_t cnt = 0;
  if (n > 0) {
    launch_pca_sum(X, n, id_base, n_total, sample_count(n_total, sample_size), D, s.p, &cnt, x->stream);
  } else {
    DADE_CK(cudaMemsetAsync(s.p, 0, sizeof(double) * D, x->stream));
  }
  DADE_CK(cudaMemcpyAsync(sum, s.p, sizeof(double) * D, cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  s.release();
  *count = cnt;
  API_END
}

extern "C" dade_status dade_pca_cov_partial(dade_index* x, const float* X, int64_t n,
                                            int64_t id_base, int64_t n_total, int64_t sample_size,
                                            const double* mean, double* cov_sum) {
  API_BEGIN
  need(x, "index"); need(mean, "mean"); need(cov_sum, "cov_sum");
  DADE_REQUIRE(n >= 0 && id_base >= 0 && id_base + n <= n_total && n_total > 0, DADE_ERR_ARG,
               "bad row range");
  DeviceGuard g(x->device);
  const int D = x->D;
  DBuf<double> mu, cov, scratch;
  mu.reserve(D);
  cov.reserve((size_t)D * D);
  DADE_CK(cudaMemcpyAsync(mu.p, mean, sizeof(double) * D, cudaMemcpyHostToDevice, x->stream));
  if (n > 0) {
    need(X, "X");
    const int64_t ns = sample_count(n_total, sample_size);
    const int64_t sc = pca_cov_scratch_elems(std::min(ns, n) + 1, D);
    scratch.reserve((size_t)sc);
    launch_pca_cov(X, n, id_base, n_total, ns, D, mu.p, cov.p, scratch.p, sc, x->stream);
  } else {
    DADE_CK(cudaMemsetAsync(cov.p, 0, sizeof(double) * D * D, x->stream));
  }
  DADE_CK(cudaMemcpyAsync(cov_sum, cov.p, sizeof(double) * D * D, cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  API_END
}

extern "C" dade_status dade_set_rotation_from_cov(dade_index* x, const double* mean,
                                                  const double* cov_sum, int64_t count) {
  API_BEGIN
  need(x, "index"); need(mean, "mean"); need(cov_sum, "cov_sum");
  DADE_REQUIRE(count > 0, DADE_ERR_ARG, "count must be positive");
  DeviceGuard g(x->device);
  const int D = x->D;
  std::vector<double> cov(cov_sum, cov_sum + (size_t)D * D), ev(D), V((size_t)D * D);
  for (auto& c : cov) c /= (double)count;                       // divisor n_s
  for (int a = 0; a < D; ++a)                                   // exact symmetry
    for (int b = a + 1; b < D; ++b) cov[(size_t)b * D + a] = cov[(size_t)a * D + b];
  sym_eig(D, cov.data(), ev.data(), V.data());                  // V column-major
  std::vector<int> order(D);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ev[a] > ev[b]; });
  std::vector<double> R((size_t)D * D), lam(D);
  for (int i = 0; i < D; ++i) {
    const double* col = &V[(size_t)order[i] * D];
    int jm = 0;
    for (int j = 1; j < D; ++j)
      if (std::fabs(col[j]) > std::fabs(col[jm])) jm = j;      // lowest index on ties (R18)
    const double sg = col[jm] < 0 ? -1.0 : 1.0;
    for (int j = 0; j < D; ++j) R[(size_t)i * D + j] = sg * col[j];
    lam[i] = ev[order[i]];
  }
  x->mean.assign(mean, mean + D);
  x->R = std::move(R);
  x->lam = std::move(lam);
  x->has_lam = true;
  upload_rotation(x);
  API_END
}

extern "C" dade_status dade_fit_rotation(dade_index* x, const float* X, int64_t n,
                                         int64_t sample_size) {
  API_BEGIN
  need(x, "index"); need(X, "X");
  DADE_REQUIRE(n >= 1, DADE_ERR_ARG, "n must be >= 1");
  const int D = x->D;
  std::vector<double> sum(D), cov((size_t)D * D);
  int64_t cnt = 0;
  dade_status s = dade_pca_mean_partial(x, X, n, 0, n, sample_size, sum.data(), &cnt);
  if (s != DADE_OK) throw Error(s, g_err);
  std::vector<double> mean(D);
  for (int j = 0; j < D; ++j) mean[j] = sum[j] / (double)cnt;
  s = dade_pca_cov_partial(x, X, n, 0, n, sample_size, mean.data(), cov.data());
  if (s != DADE_OK) throw Error(s, g_err);
  s = dade_set_rotation_from_cov(x, mean.data(), cov.data(), cnt);
  if (s != DADE_OK) throw Error(s, g_err);
  API_END
}

extern "C" dade_status dade_get_rotation(const dade_index* x, double* mean, double* R, double* ev) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_rot, DADE_ERR_STATE, "no rotation");
  const int D = x->D;
  if (mean) memcpy(mean, x->mean.data(), sizeof(double) * D);
  if (R) memcpy(R, x->R.data(), sizeof(double) * D * D);
  if (ev) memcpy(ev, x->lam.data(), sizeof(double) * D);
  API_END
}

extern "C" dade_status dade_set_rotation(dade_index* x, const double* mean, const double* R,
                                         const double* ev) {
  API_BEGIN
  need(x, "index"); need(mean, "mean"); need(R, "R");
  DeviceGuard g(x->device);
  const int D = x->D;
  for (int64_t i = 0; i < (int64_t)D * D; ++i)
    DADE_REQUIRE(std::isfinite(R[i]), DADE_ERR_NONFINITE, "non-finite R");
  for (int i = 0; i < D; ++i) DADE_REQUIRE(std::isfinite(mean[i]), DADE_ERR_NONFINITE, "non-finite mean");
  if (ev)
    for (int i = 0; i < D; ++i) DADE_REQUIRE(std::isfinite(ev[i]), DADE_ERR_NONFINITE, "non-finite eigenvalues");
  x->mean.assign(mean, mean + D);
  x->R.assign(R, R + (size_t)D * D);
  if (ev) x->lam.assign(ev, ev + D); else x->lam.assign(D, 0.0);
  x->has_lam = ev != nullptr;
  upload_rotation(x);
  API_END
}

// ================================================================== a1 + a2 IVF
extern "C" dade_status dade_build_ivf(dade_index* x, const float* X, int64_t n, int64_t id_base,
                                      int nlist, const float* centroids, int kmeans_iters) {
  API_BEGIN
  need(x, "index"); need(X, "X");
  DADE_REQUIRE(x->has_rot, DADE_ERR_STATE, "build_ivf needs a rotation (fit or set it first)");
  DADE_REQUIRE(n >= 1 && id_base >= 0 && id_base + n < ((int64_t)1 << 31), DADE_ERR_ARG,
               "bad row range (ids must be < 2^31)");
  DADE_REQUIRE(nlist >= 1 && nlist <= n, DADE_ERR_ARG, "nlist not in [1, n]");
  DADE_REQUIRE(kmeans_iters >= 0, DADE_ERR_ARG, "kmeans_iters < 0");
  DeviceGuard g(x->device);
  const int D = x->D;
  cudaStream_t st = x->stream;
  check_finite(x, X, n * D, "X");
  DBuf<float> cent;
  cent.reserve((size_t)nlist * D);
  if (centroids) {
    check_finite(x, centroids, (int64_t)nlist * D, "centroids");
    DADE_CK(cudaMemcpyAsync(cent.p, centroids, sizeof(float) * nlist * D, cudaMemcpyDeviceToDevice, st));
  } else {
    // k-means (R19): strided sample, init = first nlist sampled rows, exact assignment,
    // centroid = fp64 mean (sample order) rounded to fp32, empty cluster keeps its centroid.
    const int64_t nkm = std::min<int64_t>(n, (int64_t)64 * nlist);
    std::vector<int32_t> sid(nkm);
    for (int64_t k = 0; k < nkm; ++k) sid[k] = (int32_t)(((__int128)k * n) / nkm);
    DBuf<int32_t> sid_d;
    sid_d.reserve(nkm);
    DBuf<float> S;
    S.reserve((size_t)nkm * D);
    DADE_CK(cudaMemcpyAsync(sid_d.p, sid.data(), sizeof(int32_t) * nkm, cudaMemcpyHostToDevice, st));
    launch_gather_rows(X, sid_d.p, nkm, D, S.p, st);
    std::vector<float> Sh((size_t)nkm * D);
    DADE_CK(cudaMemcpyAsync(Sh.data(), S.p, sizeof(float) * nkm * D, cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaMemcpyAsync(cent.p, S.p, sizeof(float) * nlist * D, cudaMemcpyDeviceToDevice, st));
    DADE_CK(cudaStreamSynchronize(st));
    std::vector<float> ch(Sh.begin(), Sh.begin() + (size_t)nlist * D);
    DBuf<int32_t> a_d;
    a_d.reserve(nkm);
    std::vector<int32_t> a(nkm);
    std::vector<double> sums((size_t)nlist * D);
    std::vector<int64_t> cnt(nlist);
    for (int it = 0; it < kmeans_iters; ++it) {
      exact_knn(x, S.p, nkm, cent.p, nlist, 1, a_d.p, nullptr);
      DADE_CK(cudaMemcpyAsync(a.data(), a_d.p, sizeof(int32_t) * nkm, cudaMemcpyDeviceToHost, st));
      DADE_CK(cudaStreamSynchronize(st));
      check_knn_flag(x);
      for (int64_t k = 0; k < nkm; ++k)
        DADE_REQUIRE(a[k] >= 0 && a[k] < nlist, DADE_ERR_CUDA, "k-means: invalid list id from the assignment");
      std::fill(sums.begin(), sums.end(), 0.0);
      std::fill(cnt.begin(), cnt.end(), 0);
      for (int64_t k = 0; k < nkm; ++k) {
        double* sr = &sums[(size_t)a[k] * D];
        const float* xr = &Sh[(size_t)k * D];
        for (int j = 0; j < D; ++j) sr[j] += (double)xr[j];
        ++cnt[a[k]];
      }
      for (int c = 0; c < nlist; ++c)
        if (cnt[c] > 0)
          for (int j = 0; j < D; ++j) ch[(size_t)c * D + j] = (float)(sums[(size_t)c * D + j] / (double)cnt[c]);
      DADE_CK(cudaMemcpyAsync(cent.p, ch.data(), sizeof(float) * nlist * D, cudaMemcpyHostToDevice, st));
    }
    DADE_CK(cudaStreamSynchronize(st));
    S.release(); sid_d.release(); a_d.release();
  }
  // exact assignment of every row (R20)
  std::vector<int32_t> assign(n);
  {
    DBuf<int32_t> a_d;
    a_d.reserve(n);
    if (nlist == 1) DADE_CK(cudaMemsetAsync(a_d.p, 0, sizeof(int32_t) * n, st));
    else exact_knn(x, X, n, cent.p, nlist, 1, a_d.p, nullptr);
    DADE_CK(cudaMemcpyAsync(assign.data(), a_d.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    check_knn_flag(x);
    for (int64_t i = 0; i < n; ++i)
      DADE_REQUIRE(assign[i] >= 0 && assign[i] < nlist, DADE_ERR_CUDA, "build_ivf: invalid list id from the assignment");
  }
  // counting sort by (list, id): lists hold ids ascending
  std::vector<int64_t> off(nlist + 1, 0);
  for (int64_t i = 0; i < n; ++i) ++off[assign[i] + 1];
  for (int c = 0; c < nlist; ++c) off[c + 1] += off[c];
  std::vector<int64_t> fill(off.begin(), off.end() - 1), row_id(n);
  std::vector<int32_t> pos_of(n), src(n), off32(nlist + 1), rid32(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t p = fill[assign[i]]++;
    row_id[p] = id_base + i;
    pos_of[i] = (int32_t)p;
    src[p] = (int32_t)i;
  }
  for (int c = 0; c <= nlist; ++c) off32[c] = (int32_t)off[c];
  for (int64_t p = 0; p < n; ++p) rid32[p] = (int32_t)row_id[p];
  // rotated, dimension-blocked, list-major layout (a1)
  DBuf<float> layout;
  layout.reserve((size_t)n * D);
  DBuf<int32_t> off_d, rid_d, src_d;
  off_d.reserve(nlist + 1); rid_d.reserve(n); src_d.reserve(n);
  DADE_CK(cudaMemcpyAsync(off_d.p, off32.data(), sizeof(int32_t) * (nlist + 1), cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(rid_d.p, rid32.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(src_d.p, src.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
  launch_rotate(x->rot_op, x->rot_ws, X, src_d.p, n, x->mean_d.p, nullptr, layout.p, st);
  DADE_CK(cudaStreamSynchronize(st));
  src_d.release();
  // commit (state unchanged on any earlier error)
  std::swap(x->cent, cent); cent.release();
  tc_prepare(x, x->cent.p, nlist, x->cent_tc, true);
  std::swap(x->layout, layout); layout.release();
  std::swap(x->off_d, off_d); off_d.release();
  std::swap(x->row_id_d, rid_d); rid_d.release();
  x->off_h = std::move(off);
  x->row_id_h = std::move(row_id);
  x->assign_h = std::move(assign);
  x->pos_of_h = std::move(pos_of);
  x->nlist = nlist;
  x->n = n;
  x->id_base = id_base;
  x->has_ivf = true;
  x->xnorm_ok = false;
  x->has_cal = false;
  pq_encode_layout(x);  // BSA-q: codes of the new layout (if codebooks are installed)
  x->has_graph = false;
  API_END
}

// Sharded k-means: this rank's contribution to one Lloyd step over the GLOBAL
// strided sample ⌊k·n_total/n_km⌋, n_km = min(n_total, 64·nlist) (R19). Rows of the sample in
// [id_base, id_base + n) are assigned exactly to `centroids` (host nlist x D fp32; R20) and their
// fp64 sums / counts added to sums (host nlist x D) / counts (host nlist). centroids == NULL:
// the init step — the sampled rows with sample index < nlist are written into sums (row = sample
// index) and counts[k] = 1 for them.
extern "C" dade_status dade_kmeans_partial(dade_index* x, const float* X, int64_t n, int64_t id_base,
                                           int64_t n_total, int nlist, const float* centroids, double* sums,
                                           int64_t* counts) {
  API_BEGIN
  need(x, "index"); need(sums, "sums"); need(counts, "counts");
  DADE_REQUIRE(nlist >= 1 && nlist <= n_total, DADE_ERR_ARG, "nlist not in [1, n_total]");
  DADE_REQUIRE(n >= 0 && id_base >= 0 && id_base + n <= n_total, DADE_ERR_ARG, "bad row range");
  DeviceGuard g(x->device);
  const int D = x->D;
  cudaStream_t st = x->stream;
  std::fill(sums, sums + (size_t)nlist * D, 0.0);
  std::fill(counts, counts + nlist, (int64_t)0);
  const int64_t nkm = std::min<int64_t>(n_total, (int64_t)64 * nlist);
  std::vector<int32_t> sid;     // local row of each owned sample
  std::vector<int64_t> sidx;    // its sample index k
  for (int64_t k = 0; k < nkm; ++k) {
    const int64_t gid = (int64_t)(((__int128)k * n_total) / nkm);
    if (gid >= id_base && gid < id_base + n) { sid.push_back((int32_t)(gid - id_base)); sidx.push_back(k); }
  }
  if (centroids == nullptr) {  // init: the first nlist sampled rows
    std::vector<int32_t> rows; std::vector<int64_t> ks;
    for (size_t i = 0; i < sid.size(); ++i)
      if (sidx[i] < nlist) { rows.push_back(sid[i]); ks.push_back(sidx[i]); }
    if (!rows.empty()) {
      need(X, "X");
      DBuf<int32_t> r_d; DBuf<float> S;
      r_d.reserve(rows.size()); S.reserve(rows.size() * D);
      DADE_CK(cudaMemcpyAsync(r_d.p, rows.data(), 4 * rows.size(), cudaMemcpyHostToDevice, st));
      launch_gather_rows(X, r_d.p, (int64_t)rows.size(), D, S.p, st);
      std::vector<float> Sh(rows.size() * D);
      DADE_CK(cudaMemcpyAsync(Sh.data(), S.p, 4 * Sh.size(), cudaMemcpyDeviceToHost, st));
      DADE_CK(cudaStreamSynchronize(st));
      for (size_t i = 0; i < rows.size(); ++i) {
        for (int j = 0; j < D; ++j) sums[(size_t)ks[i] * D + j] = (double)Sh[i * D + j];
        counts[ks[i]] = 1;
      }
      r_d.release(); S.release();
    }
    g_err.clear();
    return DADE_OK;
  }
  if (sid.empty()) { g_err.clear(); return DADE_OK; }
  need(X, "X");
  const int64_t m = (int64_t)sid.size();
  DBuf<int32_t> sid_d, a_d; DBuf<float> S, C;
  sid_d.reserve(m); a_d.reserve(m); S.reserve((size_t)m * D); C.reserve((size_t)nlist * D);
  DADE_CK(cudaMemcpyAsync(sid_d.p, sid.data(), 4 * m, cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(C.p, centroids, sizeof(float) * nlist * D, cudaMemcpyHostToDevice, st));
  launch_gather_rows(X, sid_d.p, m, D, S.p, st);
  exact_knn(x, S.p, m, C.p, nlist, 1, a_d.p, nullptr);
  std::vector<int32_t> a(m);
  std::vector<float> Sh((size_t)m * D);
  DADE_CK(cudaMemcpyAsync(a.data(), a_d.p, 4 * m, cudaMemcpyDeviceToHost, st));
  DADE_CK(cudaMemcpyAsync(Sh.data(), S.p, 4 * Sh.size(), cudaMemcpyDeviceToHost, st));
  DADE_CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < m; ++i) {  // sample order within the shard (R19: fp64 sums)
    DADE_REQUIRE(a[i] >= 0 && a[i] < nlist, DADE_ERR_CUDA, "k-means: invalid list id from the assignment");
    double* sr = &sums[(size_t)a[i] * D];
    const float* xr = &Sh[(size_t)i * D];
    for (int j = 0; j < D; ++j) sr[j] += (double)xr[j];
    ++counts[a[i]];
  }
  sid_d.release(); a_d.release(); S.release(); C.release();
  API_END
}

extern "C" dade_status dade_get_ivf(const dade_index* x, int64_t* off, int64_t* row_id,
                                    int32_t* assign, float* centroids) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_ivf, DADE_ERR_STATE, "no IVF");
  if (off) memcpy(off, x->off_h.data(), sizeof(int64_t) * (x->nlist + 1));
  if (row_id) memcpy(row_id, x->row_id_h.data(), sizeof(int64_t) * x->n);
  if (assign) memcpy(assign, x->assign_h.data(), sizeof(int32_t) * x->n);
  if (centroids) {
    DeviceGuard g(x->device);
    DADE_CK(cudaMemcpyAsync(centroids, x->cent.p, sizeof(float) * x->nlist * x->D, cudaMemcpyDeviceToHost, x->stream));
    DADE_CK(cudaStreamSynchronize(x->stream));
  }
  API_END
}

extern "C" dade_status dade_get_sizes(const dade_index* x, int64_t* n, int* nlist) {
  API_BEGIN
  need(x, "index");
  if (n) *n = x->has_ivf ? x->n : 0;
  if (nlist) *nlist = x->has_ivf ? x->nlist : 0;
  API_END
}

extern "C" dade_status dade_get_layout(const dade_index* x, float* Xrot) {
  API_BEGIN
  need(x, "index"); need(Xrot, "Xrot");
  DADE_REQUIRE(x->has_ivf, DADE_ERR_STATE, "no IVF");
  DeviceGuard g(x->device);
  const int D = x->D;
  const int64_t n = x->n;
  std::vector<float> blk((size_t)n * D);
  DADE_CK(cudaMemcpyAsync(blk.data(), x->layout.p, sizeof(float) * n * D, cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  for (int b = 0; b < D / 16; ++b)
    for (int64_t p = 0; p < n; ++p)
      memcpy(Xrot + p * D + b * 16, &blk[((size_t)b * n + p) * 16], 64);
  API_END
}

// ================================================================== a3 calibration
// ---- calibration building blocks (single-GPU dade_calibrate and the sharded protocol share them)
namespace {
// exact K nearest rows of this index's base X (raw, id order) for every query, fp64 distances
void calib_knn(dade_index* x, const float* X, const float* Qc, int nq, int K, std::vector<int64_t>& ids,
               std::vector<double>& d) {
  DBuf<int32_t> knn_i;
  DBuf<double> knn_d;
  knn_i.reserve((size_t)nq * K);
  knn_d.reserve((size_t)nq * K);
  exact_knn(x, Qc, nq, X, x->n, K, knn_i.p, knn_d.p);
  std::vector<int32_t> ki((size_t)nq * K);
  d.resize((size_t)nq * K);
  DADE_CK(cudaMemcpyAsync(ki.data(), knn_i.p, sizeof(int32_t) * ki.size(), cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaMemcpyAsync(d.data(), knn_d.p, sizeof(double) * d.size(), cudaMemcpyDeviceToHost, x->stream));
  DADE_CK(cudaStreamSynchronize(x->stream));
  ids.resize(ki.size());
  for (size_t i = 0; i < ki.size(); ++i) ids[i] = x->id_base + ki[i];
}

// Label-1 candidates of this shard (R15/R16): the rows of the query's nprobe_neg probed lists (the
// whole shard if 0 or flat) that are not among its K nearest (knn_ids: global ids, nq x K), the
// n_neg smallest by (SplitMix64(seed ^ (q << 32 | id)), id). Outputs per query, ascending.
void calib_negatives(dade_index* x, const float* Qc, int nq, int K, const int64_t* knn_ids, int n_neg,
                     int nprobe_neg, uint64_t seed, std::vector<std::vector<std::pair<uint64_t, int64_t>>>& out) {
  const bool whole = nprobe_neg == 0 || x->nlist == 1;
  std::vector<int32_t> pr;
  if (!whole) {
    DBuf<int32_t> pd;
    pd.reserve((size_t)nq * nprobe_neg);
    exact_knn(x, Qc, nq, x->cent.p, x->nlist, nprobe_neg, pd.p, nullptr, x->cent_tc);
    pr.resize((size_t)nq * nprobe_neg);
    DADE_CK(cudaMemcpyAsync(pr.data(), pd.p, sizeof(int32_t) * pr.size(), cudaMemcpyDeviceToHost, x->stream));
    DADE_CK(cudaStreamSynchronize(x->stream));
  }
  out.assign(nq, {});
  std::vector<std::pair<uint64_t, int64_t>> cand;
  for (int qi = 0; qi < nq; ++qi) {
    std::vector<int64_t> kn(knn_ids + (size_t)qi * K, knn_ids + (size_t)qi * K + K);
    std::sort(kn.begin(), kn.end());
    cand.clear();
    auto consider = [&](int64_t id) {
      if (std::binary_search(kn.begin(), kn.end(), id)) return;
      const uint64_t key = ((uint64_t)(uint32_t)qi << 32) | (uint64_t)id;
      cand.emplace_back(splitmix64(seed ^ key), id);
    };
    if (whole) {
      for (int64_t i = 0; i < x->n; ++i) consider(x->id_base + i);
    } else {
      for (int j = 0; j < nprobe_neg; ++j) {
        const int l = pr[(size_t)qi * nprobe_neg + j];
        for (int64_t p = x->off_h[l]; p < x->off_h[l + 1]; ++p) consider(x->row_id_h[p]);
      }
    }
    const size_t take = std::min<size_t>((size_t)n_neg, cand.size());
    std::partial_sort(cand.begin(), cand.begin() + take, cand.end());
    out[qi].assign(cand.begin(), cand.begin() + take);
  }
}

// P_d at every 16-dim prefix for the pairs whose id lies in this shard (fp64 from the stored fp32
// rotated rows); rows of other shards' pairs are zero. F: npairs x (D/16).
void pair_features(dade_index* x, const float* Qc, int nq, int npairs, const int32_t* pq, const int64_t* pid,
                   std::vector<double>& F) {
  const int D = x->D, nblk = D / 16;
  F.assign((size_t)npairs * nblk, 0.0);
  std::vector<int32_t> q_own, row_own, which;
  for (int i = 0; i < npairs; ++i) {
    const int64_t loc = pid[i] - x->id_base;
    if (loc < 0 || loc >= x->n) continue;
    q_own.push_back(pq[i]); row_own.push_back(x->pos_of_h[loc]); which.push_back(i);
  }
  const int m = (int)which.size();
  if (m == 0) return;
  cudaStream_t st = x->stream;
  DBuf<float> qr;
  qr.reserve((size_t)nq * D);
  launch_rotate(x->rot_op, x->rot_ws, Qc, nullptr, nq, x->mean_d.p, qr.p, nullptr, st);
  DBuf<int32_t> pq_d, pr_d;
  DBuf<double> feat;
  pq_d.reserve(m); pr_d.reserve(m); feat.reserve((size_t)m * nblk);
  DADE_CK(cudaMemcpyAsync(pq_d.p, q_own.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(pr_d.p, row_own.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
  launch_pair_prefix(x->layout.p, x->n, D, qr.p, pq_d.p, pr_d.p, m, feat.p, st);
  std::vector<double> Fm((size_t)m * nblk);
  DADE_CK(cudaMemcpyAsync(Fm.data(), feat.p, sizeof(double) * Fm.size(), cudaMemcpyDeviceToHost, st));
  DADE_CK(cudaStreamSynchronize(st));
  for (int i = 0; i < m; ++i)
    std::copy(Fm.begin() + (size_t)i * nblk, Fm.begin() + (size_t)(i + 1) * nblk, F.begin() + (size_t)which[i] * nblk);
}

// per-step logistic slope (R3) and sorted thresholds v_d = sort_desc(tau - m1 P_d) over Label 0 (R4)
void fit_calibration(dade_index* x, int K, int npairs, const double* F, const double* ptau_, const double* py_) {
  const int nblk = x->D / 16, ncls = nblk - 1;
  std::vector<double> ptau(ptau_, ptau_ + npairs), py(py_, py_ + npairs);
  int n0 = 0;
  for (double y : py) n0 += y == 0.0;
  DADE_REQUIRE(n0 >= 1, DADE_ERR_ARG, "calibration needs Label-0 pairs");
  std::vector<double> m1(ncls, 1.0), v((size_t)ncls * n0), P(npairs);
  for (int s = 0; s < ncls; ++s) {
    for (int i = 0; i < npairs; ++i) P[i] = F[(size_t)i * nblk + s];
    double m, b;
    logistic_irls(P, ptau, py, 1e-8, 100, 1e-12, &m, &b);
    m1[s] = m;
    std::vector<double> vv;
    vv.reserve(n0);
    for (int i = 0; i < npairs; ++i)
      if (py[i] == 0.0) vv.push_back(ptau[i] - m * P[i]);
    std::sort(vv.begin(), vv.end(), std::greater<double>());
    std::copy(vv.begin(), vv.end(), v.begin() + (size_t)s * n0);
  }
  x->m1 = std::move(m1);
  x->v = std::move(v);
  x->calK = K;
  x->n0 = n0;
  x->ncls = ncls;
  x->has_cal = true;
}

void calib_checks(dade_index* x, const float* Qc, int nq, int K, int n_neg, int nprobe_neg) {
  DADE_REQUIRE(x->has_ivf, DADE_ERR_STATE, "calibrate needs build_ivf first");
  DADE_REQUIRE(nq >= 1, DADE_ERR_ARG, "nq < 1");
  DADE_REQUIRE(K >= 1 && K <= DADE_MAX_K, DADE_ERR_ARG, "K not in [1, DADE_MAX_K]");
  DADE_REQUIRE(n_neg >= 0, DADE_ERR_ARG, "n_neg < 0");
  DADE_REQUIRE(nprobe_neg >= 0 && nprobe_neg <= x->nlist, DADE_ERR_ARG, "nprobe_neg not in [0, nlist]");
  check_finite(x, Qc, (int64_t)nq * x->D, "Qc");
}
}  // namespace

extern "C" dade_status dade_calibrate(dade_index* x, const float* X, const float* Qc, int nq, int K,
                                      int n_neg, int nprobe_neg, uint64_t seed) {
  API_BEGIN
  need(x, "index"); need(X, "X"); need(Qc, "Qc");
  DeviceGuard g(x->device);
  calib_checks(x, Qc, nq, K, n_neg, nprobe_neg);
  DADE_REQUIRE(K <= x->n, DADE_ERR_ARG, "K not in [1, n]");
  // exact KNN over the whole base (Label 0, tau_q) — P:L3930, R14
  std::vector<int64_t> ki;
  std::vector<double> kd;
  calib_knn(x, X, Qc, nq, K, ki, kd);
  // Label 1 = n_neg non-KNN candidates with the smallest hash (R15, R16)
  std::vector<std::vector<std::pair<uint64_t, int64_t>>> neg;
  calib_negatives(x, Qc, nq, K, ki.data(), n_neg, nprobe_neg, seed, neg);
  std::vector<int32_t> pq;
  std::vector<int64_t> pid;
  std::vector<double> ptau, py;
  for (int qi = 0; qi < nq; ++qi) {
    const double tau = kd[(size_t)qi * K + K - 1];
    for (int j = 0; j < K; ++j) { pq.push_back(qi); pid.push_back(ki[(size_t)qi * K + j]); ptau.push_back(tau); py.push_back(0.0); }
    for (const auto& c : neg[qi]) { pq.push_back(qi); pid.push_back(c.second); ptau.push_back(tau); py.push_back(1.0); }
  }
  std::vector<double> F;
  pair_features(x, Qc, nq, (int)pq.size(), pq.data(), pid.data(), F);
  fit_calibration(x, K, (int)pq.size(), F.data(), ptau.data(), py.data());
  API_END
}

// ---- sharded calibration: the same steps split across ranks (sharded.py)
extern "C" dade_status dade_calib_knn(dade_index* x, const float* X, const float* Qc, int nq, int K,
                                      int64_t* ids, double* dists) {
  API_BEGIN
  need(x, "index"); need(X, "X"); need(Qc, "Qc"); need(ids, "ids"); need(dists, "dists");
  DeviceGuard g(x->device);
  calib_checks(x, Qc, nq, K, 0, 0);
  DADE_REQUIRE(K <= x->n, DADE_ERR_ARG, "K > shard size");
  std::vector<int64_t> ki;
  std::vector<double> kd;
  calib_knn(x, X, Qc, nq, K, ki, kd);
  std::copy(ki.begin(), ki.end(), ids);
  std::copy(kd.begin(), kd.end(), dists);
  API_END
}

extern "C" dade_status dade_calib_negatives(dade_index* x, const float* Qc, int nq, int K, const int64_t* knn_ids,
                                            int n_neg, int nprobe_neg, uint64_t seed, uint64_t* keys, int64_t* ids,
                                            int32_t* counts) {
  API_BEGIN
  need(x, "index"); need(Qc, "Qc"); need(knn_ids, "knn_ids"); need(counts, "counts");
  if (n_neg > 0) { need(keys, "keys"); need(ids, "ids"); }
  DeviceGuard g(x->device);
  calib_checks(x, Qc, nq, K, n_neg, nprobe_neg);
  std::vector<std::vector<std::pair<uint64_t, int64_t>>> neg;
  calib_negatives(x, Qc, nq, K, knn_ids, n_neg, nprobe_neg, seed, neg);
  for (int qi = 0; qi < nq; ++qi) {
    counts[qi] = (int32_t)neg[qi].size();
    for (size_t j = 0; j < neg[qi].size(); ++j) {
      keys[(size_t)qi * n_neg + j] = neg[qi][j].first;
      ids[(size_t)qi * n_neg + j] = neg[qi][j].second;
    }
  }
  API_END
}

extern "C" dade_status dade_pair_features(dade_index* x, const float* Qc, int nq, int npairs, const int32_t* pair_q,
                                          const int64_t* pair_id, double* F) {
  API_BEGIN
  need(x, "index"); need(Qc, "Qc"); need(F, "F");
  if (npairs > 0) { need(pair_q, "pair_q"); need(pair_id, "pair_id"); }
  DADE_REQUIRE(x->has_ivf, DADE_ERR_STATE, "pair features need build_ivf first");
  DeviceGuard g(x->device);
  std::vector<double> Fv;
  pair_features(x, Qc, nq, npairs, pair_q, pair_id, Fv);
  std::copy(Fv.begin(), Fv.end(), F);
  API_END
}

extern "C" dade_status dade_fit_calibration(dade_index* x, int K, int npairs, const double* F, const double* tau,
                                            const double* y) {
  API_BEGIN
  need(x, "index"); need(F, "F"); need(tau, "tau"); need(y, "y");
  DADE_REQUIRE(K >= 1 && K <= DADE_MAX_K && npairs >= 1, DADE_ERR_ARG, "bad K / npairs");
  fit_calibration(x, K, npairs, F, tau, y);
  API_END
}

extern "C" dade_status dade_get_calibration(const dade_index* x, int* K, int* n0, int* ncls,
                                            double* m1, double* v) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_cal, DADE_ERR_STATE, "no calibration");
  if (K) *K = x->calK;
  if (n0) *n0 = x->n0;
  if (ncls) *ncls = x->ncls;
  if (m1) memcpy(m1, x->m1.data(), sizeof(double) * x->ncls);
  if (v) memcpy(v, x->v.data(), sizeof(double) * x->v.size());
  API_END
}

extern "C" dade_status dade_set_calibration(dade_index* x, int K, int n0, int ncls,
                                            const double* m1, const double* v) {
  API_BEGIN
  need(x, "index"); need(m1, "m1"); need(v, "v");
  DADE_REQUIRE(K >= 1 && K <= DADE_MAX_K && n0 >= 1, DADE_ERR_ARG, "bad K / n0");
  DADE_REQUIRE(ncls == x->D / 16 - 1, DADE_ERR_SHAPE, "n_cls must be D/16 - 1");
  x->m1.assign(m1, m1 + ncls);
  x->v.assign(v, v + (size_t)ncls * n0);
  x->calK = K;
  x->n0 = n0;
  x->ncls = ncls;
  x->has_cal = true;
  API_END
}

// ================================================================== a4..a8 search
extern "C" dade_status dade_search(dade_index* x, const float* Q, int nq, int K, int nprobe,
                                   int delta_d, double significance, int64_t* ids, float* dists,
                                   dade_stats* stats) {
  API_BEGIN
  need(x, "index");
  DeviceGuard g(x->device);
  if (collective(x)) do_search_collective(x, Q, nq, K, nprobe, delta_d, significance, ids, dists, stats, DADE_METHOD_BSA_P);
  else do_search(x, Q, nq, K, nprobe, delta_d, significance, ids, dists, stats);
  API_END
}

extern "C" dade_status dade_search_method(dade_index* x, const float* Q, int nq, int K, int nprobe,
                                          int delta_d, int method, double param, int64_t* ids,
                                          float* dists, dade_stats* stats) {
  API_BEGIN
  need(x, "index");
  DeviceGuard g(x->device);
  if (collective(x)) do_search_collective(x, Q, nq, K, nprobe, delta_d, param, ids, dists, stats, method);
  else do_search(x, Q, nq, K, nprobe, delta_d, param, ids, dists, stats, method);
  API_END
}

extern "C" dade_status dade_set_timing(dade_index* x, int on) {
  API_BEGIN
  need(x, "index");
  x->timing = on != 0;
  API_END
}

extern "C" dade_status dade_get_timing(dade_index* x, float* ms3) {
  API_BEGIN
  need(x, "index"); need(ms3, "ms3");
  DeviceGuard g(x->device);
  DADE_REQUIRE(x->ev[3] != nullptr, DADE_ERR_STATE, "no timed search yet");
  DADE_CK(cudaEventSynchronize(x->ev[3]));
  DADE_CK(cudaEventElapsedTime(&ms3[0], x->ev[0], x->ev[1]));
  DADE_CK(cudaEventElapsedTime(&ms3[1], x->ev[0], x->ev[2]));
  DADE_CK(cudaEventElapsedTime(&ms3[2], x->ev[2], x->ev[3]));
  API_END
}

extern "C" dade_status dade_prepare(dade_index* x, const float* Q, int nq, int nprobe, float* qrot,
                                    int32_t* probes) {
  API_BEGIN
  need(x, "index");
  DeviceGuard g(x->device);
  DADE_REQUIRE(x->has_ivf && x->has_rot, DADE_ERR_STATE, "prepare before build_ivf");
  DADE_REQUIRE(nq >= 0, DADE_ERR_ARG, "nq < 0");
  DADE_REQUIRE(nprobe >= 1 && nprobe <= x->nlist, DADE_ERR_ARG, "nprobe not in [1, nlist]");
  if (nq == 0) { g_err.clear(); return DADE_OK; }
  need(Q, "Q"); need(qrot, "qrot"); need(probes, "probes");
  prepare(x, Q, nq, nprobe, qrot, probes, false);
  API_END
}

extern "C" dade_status dade_search_prepared(dade_index* x, const float* qrot, const int32_t* probes, int nq,
                                            int K, int nprobe, int delta_d, int method, double param,
                                            int64_t* ids, float* dists, dade_stats* stats) {
  API_BEGIN
  need(x, "index");
  DeviceGuard g(x->device);
  if (nq > 0) need(qrot, "qrot");
  do_search(x, nullptr, nq, K, nprobe, delta_d, param, ids, dists, stats, method, qrot, probes);
  API_END
}

extern "C" dade_status dade_search_host(dade_index* x, const float* Qh, int nq, int K, int nprobe,
                                        int delta_d, double significance, int64_t* ids_h,
                                        float* dists_h, dade_stats* stats) {
  API_BEGIN
  need(x, "index"); need(Qh, "Q"); need(ids_h, "ids"); need(dists_h, "dists");
  DeviceGuard g(x->device);
  const int D = x->D;
  cudaStream_t st = x->stream;
  x->qbuf.reserve((size_t)std::max(nq, 1) * D);
  x->ids_tmp.reserve((size_t)std::max(nq, 1) * K);
  x->dists_tmp.reserve((size_t)std::max(nq, 1) * K);
  // Pipeline: the batch is cut into chunks; chunk c's H2D (copy stream) overlaps the search of
  // chunk c-1 (library stream), whose results' D2H (second copy stream) overlaps chunk c's search.
  // Stats need one search over the whole batch, so they run unchunked.
  if (collective(x)) {  // H2D, the collective search (NCCL inside), D2H
    if (nq > 0) {
      DADE_CK(cudaMemcpyAsync(x->qbuf.p, Qh, sizeof(float) * nq * D, cudaMemcpyHostToDevice, st));
      do_search_collective(x, x->qbuf.p, nq, K, nprobe, delta_d, significance, x->ids_tmp.p, x->dists_tmp.p, stats,
                           DADE_METHOD_BSA_P);
      DADE_CK(cudaMemcpyAsync(ids_h, x->ids_tmp.p, sizeof(int64_t) * nq * K, cudaMemcpyDeviceToHost, st));
      DADE_CK(cudaMemcpyAsync(dists_h, x->dists_tmp.p, sizeof(float) * nq * K, cudaMemcpyDeviceToHost, st));
    }
    DADE_CK(cudaStreamSynchronize(st));
    check_knn_flag(x);
    g_err.clear();
    return DADE_OK;
  }
  int nch = host_chunks(x, nq);
  if (stats || nq <= 0) nch = 1;
  if (!x->h2d) {
    DADE_CK(cudaStreamCreateWithFlags(&x->h2d, cudaStreamNonBlocking));
    DADE_CK(cudaStreamCreateWithFlags(&x->d2h, cudaStreamNonBlocking));
  }
  while ((int)x->hev.size() < 2 * nch + 1) {
    cudaEvent_t e;
    DADE_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    x->hev.push_back(e);
  }
  DADE_CK(cudaEventRecord(x->hev[0], st));  // the copies start after earlier work on the stream
  DADE_CK(cudaStreamWaitEvent(x->h2d, x->hev[0], 0));
  DADE_CK(cudaStreamWaitEvent(x->d2h, x->hev[0], 0));
  const int npc_copy = nch == 1 && !stats && nq > 0 ? host_prep_chunks(x, nq) : 1;
  while ((int)x->hev.size() < npc_copy + 3) {
    cudaEvent_t e;
    DADE_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    x->hev.push_back(e);
  }
  if (npc_copy > 1) {
    for (int c = 0; c < npc_copy; ++c) {
      const int q0 = (int)((int64_t)nq * c / npc_copy), q1 = (int)((int64_t)nq * (c + 1) / npc_copy);
      DADE_CK(cudaMemcpyAsync(x->qbuf.p + (size_t)q0 * D, Qh + (size_t)q0 * D, sizeof(float) * (q1 - q0) * D,
                              cudaMemcpyHostToDevice, x->h2d));
      DADE_CK(cudaEventRecord(x->hev[3 + c], x->h2d));
    }
  } else {
    for (int c = 0; c < nch; ++c) {
      const int q0 = (int)((int64_t)nq * c / nch), q1 = (int)((int64_t)nq * (c + 1) / nch);
      DADE_CK(cudaMemcpyAsync(x->qbuf.p + (size_t)q0 * D, Qh + (size_t)q0 * D, sizeof(float) * (q1 - q0) * D,
                              cudaMemcpyHostToDevice, x->h2d));
      DADE_CK(cudaEventRecord(x->hev[1 + 2 * c], x->h2d));
    }
  }
  // one search: its rotation + probe (a4, a5) run per H2D chunk, so the copy of chunk c+1
  // overlaps the probe of chunk c; the scan (a6-a8) then runs once over the whole batch
  const int npc = nch == 1 && !stats && nq > 0 ? host_prep_chunks(x, nq) : 1;
  if (npc > 1) {
    DADE_REQUIRE(x->has_ivf && x->has_rot, DADE_ERR_STATE, "search before build_ivf");
    DADE_REQUIRE(nprobe >= 1 && nprobe <= x->nlist, DADE_ERR_ARG, "nprobe not in [1, nlist]");
    while ((int)x->hev.size() < npc + 3) {
      cudaEvent_t e;
      DADE_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      x->hev.push_back(e);
    }
    x->qrot.reserve((size_t)nq * D);
    x->probes.reserve((size_t)nq * nprobe);
    for (int c = 0; c < npc; ++c) {
      const int q0 = (int)((int64_t)nq * c / npc), q1 = (int)((int64_t)nq * (c + 1) / npc);
      DADE_CK(cudaStreamWaitEvent(st, x->hev[3 + c], 0));
      prepare(x, x->qbuf.p + (size_t)q0 * D, q1 - q0, nprobe, x->qrot.p + (size_t)q0 * D,
              x->probes.p + (size_t)q0 * nprobe, false);
    }
    do_search(x, nullptr, nq, K, nprobe, delta_d, significance, x->ids_tmp.p, x->dists_tmp.p, nullptr,
              DADE_METHOD_BSA_P, x->qrot.p, x->probes.p);
    DADE_CK(cudaEventRecord(x->hev[2], st));
    DADE_CK(cudaStreamWaitEvent(x->d2h, x->hev[2], 0));
    DADE_CK(cudaMemcpyAsync(ids_h, x->ids_tmp.p, sizeof(int64_t) * nq * K, cudaMemcpyDeviceToHost, x->d2h));
    DADE_CK(cudaMemcpyAsync(dists_h, x->dists_tmp.p, sizeof(float) * nq * K, cudaMemcpyDeviceToHost, x->d2h));
    nch = 0;  // done: skip the per-chunk searches below
  }
  for (int c = 0; c < nch; ++c) {
    const int q0 = (int)((int64_t)nq * c / nch), q1 = (int)((int64_t)nq * (c + 1) / nch);
    DADE_CK(cudaStreamWaitEvent(st, x->hev[1 + 2 * c], 0));
    do_search(x, x->qbuf.p + (size_t)q0 * D, q1 - q0, K, nprobe, delta_d, significance,
              x->ids_tmp.p + (size_t)q0 * K, x->dists_tmp.p + (size_t)q0 * K, stats);
    DADE_CK(cudaEventRecord(x->hev[2 + 2 * c], st));
    DADE_CK(cudaStreamWaitEvent(x->d2h, x->hev[2 + 2 * c], 0));
    DADE_CK(cudaMemcpyAsync(ids_h + (size_t)q0 * K, x->ids_tmp.p + (size_t)q0 * K, sizeof(int64_t) * (q1 - q0) * K,
                            cudaMemcpyDeviceToHost, x->d2h));
    DADE_CK(cudaMemcpyAsync(dists_h + (size_t)q0 * K, x->dists_tmp.p + (size_t)q0 * K,
                            sizeof(float) * (q1 - q0) * K, cudaMemcpyDeviceToHost, x->d2h));
  }
  DADE_CK(cudaEventRecord(x->hev[0], x->d2h));  // the library stream resumes after the last D2H
  DADE_CK(cudaStreamWaitEvent(st, x->hev[0], 0));
  DADE_CK(cudaStreamSynchronize(st));
  check_knn_flag(x);
  API_END
}

// NEXT-2: Exp-7 / Table III standalone approximation accuracy (flat scan by a d-dim estimate)
extern "C" dade_status dade_estimate_knn(dade_index* x, const float* Q, int nq, int d, int method, int K,
                                         int64_t* ids, float* est) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_ivf && x->has_rot, DADE_ERR_STATE, "estimate before build_ivf");
  DADE_REQUIRE(nq >= 0, DADE_ERR_ARG, "nq < 0");
  DADE_REQUIRE(d >= 16 && d % 16 == 0 && d <= x->D, DADE_ERR_ARG, "d must be a positive multiple of 16, <= D");
  DADE_REQUIRE(K >= 1 && K <= DADE_MAX_K && K <= x->n, DADE_ERR_ARG, "K not in [1, min(n, DADE_MAX_K)]");
  DADE_REQUIRE(method == DADE_EST_PARTIAL || method == DADE_EST_RESIDUAL, DADE_ERR_ARG, "unknown estimator");
  DADE_REQUIRE(x->n < ((int64_t)1 << 31), DADE_ERR_UNSUPPORTED, "n >= 2^31");
  if (nq == 0) { g_err.clear(); return DADE_OK; }
  need(Q, "Q"); need(ids, "ids"); need(est, "est");
  DeviceGuard g(x->device);
  const int D = x->D;
  cudaStream_t st = x->stream;
  check_finite(x, Q, (int64_t)nq * D, "Q");
  x->qrot.reserve((size_t)nq * D);
  launch_rotate(x->rot_op, x->rot_ws, Q, nullptr, nq, x->mean_d.p, x->qrot.p, nullptr, st);
  if (method == DADE_EST_RESIDUAL && !x->xnorm_ok) {
    x->xnorm.reserve((size_t)std::max<int64_t>(x->n, 1));
    launch_row_norms(x->layout.p, x->n, D, x->xnorm.p, st);
    x->xnorm_ok = true;
  }
  launch_estimate_topk(x->layout.p, x->row_id_d.p, method == DADE_EST_RESIDUAL ? x->xnorm.p : nullptr, x->n, D, d,
                       x->qrot.p, nq, K, est, ids, st);
  API_END
}

extern "C" dade_status dade_probe(dade_index* x, const float* Q, int nq, int nprobe, int32_t* probes) {
  API_BEGIN
  need(x, "index"); need(Q, "Q"); need(probes, "probes");
  DADE_REQUIRE(x->has_ivf, DADE_ERR_STATE, "no IVF");
  DADE_REQUIRE(nprobe >= 1 && nprobe <= x->nlist, DADE_ERR_ARG, "nprobe not in [1, nlist]");
  DeviceGuard g(x->device);
  if (nq > 0) exact_knn(x, Q, nq, x->cent.p, x->nlist, nprobe, probes, nullptr, x->cent_tc, true, probe_passes(x));
  API_END
}

// ================================================================== tools
extern "C" dade_status dade_bruteforce_knn(dade_index* x, const float* X, int64_t n, int64_t id_base,
                                           const float* Q, int nq, int K, int64_t* ids, float* dists) {
  API_BEGIN
  need(x, "index"); need(X, "X"); need(Q, "Q"); need(ids, "ids"); need(dists, "dists");
  DADE_REQUIRE(K >= 1 && K <= n, DADE_ERR_ARG, "K not in [1, n]");
  DADE_REQUIRE(n < ((int64_t)1 << 31), DADE_ERR_UNSUPPORTED, "n >= 2^31");
  DeviceGuard g(x->device);
  if (nq <= 0) { g_err.clear(); return DADE_OK; }
  x->idx32.reserve((size_t)nq * K);
  x->d64.reserve((size_t)nq * K);
  exact_knn(x, Q, nq, X, n, K, x->idx32.p, x->d64.p);
  k_ids_from_idx<<<256, 256, 0, x->stream>>>(x->idx32.p, x->d64.p, (int64_t)nq * K, id_base, ids, dists);
  DADE_CK(cudaGetLastError());
  DADE_CK(cudaStreamSynchronize(x->stream));
  API_END
}

extern "C" dade_status dade_merge_topk(dade_index* x, const int64_t* ids_in, const float* dists_in,
                                       int S, int nq, int K, int64_t* ids_out, float* dists_out) {
  API_BEGIN
  need(x, "index"); need(ids_in, "ids_in"); need(dists_in, "dists_in");
  need(ids_out, "ids_out"); need(dists_out, "dists_out");
  DADE_REQUIRE(S >= 1 && K >= 1 && nq >= 0, DADE_ERR_ARG, "bad S / K / nq");
  DeviceGuard g(x->device);
  launch_merge_topk(ids_in, dists_in, S, nq, K, ids_out, dists_out, x->stream);
  API_END
}

// ================================================================== persistence
namespace {
const uint64_t kMagic = 0x3130454441444144ull;  // "DADADE01"
void wr(FILE* f, const void* p, size_t b) {
  DADE_REQUIRE(fwrite(p, 1, b, f) == b, DADE_ERR_ARG, "write failed");
}
void rd(FILE* f, void* p, size_t b) {
  DADE_REQUIRE(fread(p, 1, b, f) == b, DADE_ERR_ARG, "read failed / truncated file");
}
}  // namespace

extern "C" dade_status dade_save(const dade_index* x, const char* path) {
  API_BEGIN
  need(x, "index"); need(path, "path");
  DADE_REQUIRE(x->has_rot && x->has_ivf, DADE_ERR_STATE, "save needs rotation + IVF");
  DeviceGuard g(x->device);
  FILE* f = fopen(path, "wb");
  DADE_REQUIRE(f, DADE_ERR_ARG, std::string("cannot open ") + path);
  struct Closer { FILE* f; ~Closer() { fclose(f); } } cl{f};
  const int D = x->D;
  const int64_t hdr[6] = {(int64_t)kMagic, D, x->nlist, x->n, x->id_base, x->has_cal ? 1 : 0};
  wr(f, hdr, sizeof(hdr));
  wr(f, x->mean.data(), 8 * D); wr(f, x->R.data(), 8 * (size_t)D * D); wr(f, x->lam.data(), 8 * D);
  std::vector<float> cent((size_t)x->nlist * D), lay((size_t)x->n * D);
  DADE_CK(cudaMemcpy(cent.data(), x->cent.p, 4 * cent.size(), cudaMemcpyDeviceToHost));
  DADE_CK(cudaMemcpy(lay.data(), x->layout.p, 4 * lay.size(), cudaMemcpyDeviceToHost));
  wr(f, cent.data(), 4 * cent.size());
  wr(f, x->off_h.data(), 8 * x->off_h.size());
  wr(f, x->row_id_h.data(), 8 * x->row_id_h.size());
  wr(f, x->assign_h.data(), 4 * x->assign_h.size());
  wr(f, lay.data(), 4 * lay.size());
  if (x->has_cal) {
    const int64_t c[3] = {x->calK, x->n0, x->ncls};
    wr(f, c, sizeof(c));
    wr(f, x->m1.data(), 8 * x->m1.size());
    wr(f, x->v.data(), 8 * x->v.size());
  }
  API_END
}

// IVF/layout consistency shared by dade_load and dade_set_ivf: off monotone from 0 to n, row ids a
// permutation of [id_base, id_base + n) ascending inside each list (lists hold ids
// ascending). Fills assign (local id -> list) and pos_of (local id -> list-major position).
static void check_ivf(int64_t n, int64_t id_base, int nlist, const std::vector<int64_t>& off,
               const std::vector<int64_t>& rid, std::vector<int32_t>& assign, std::vector<int32_t>& pos_of) {
  DADE_REQUIRE(n >= 1 && nlist >= 1 && nlist <= n, DADE_ERR_ARG, "ivf: nlist not in [1, n]");
  DADE_REQUIRE(id_base >= 0 && id_base + n < ((int64_t)1 << 31), DADE_ERR_ARG, "ivf: ids must be < 2^31");
  DADE_REQUIRE(off[0] == 0 && off[nlist] == n, DADE_ERR_ARG, "ivf: off must run from 0 to n");
  for (int c = 0; c < nlist; ++c) DADE_REQUIRE(off[c] <= off[c + 1], DADE_ERR_ARG, "ivf: off not monotone");
  assign.assign(n, -1);
  pos_of.assign(n, 0);
  for (int c = 0; c < nlist; ++c)
    for (int64_t p = off[c]; p < off[c + 1]; ++p) {
      const int64_t loc = rid[p] - id_base;
      DADE_REQUIRE(loc >= 0 && loc < n, DADE_ERR_ARG, "ivf: row id outside [id_base, id_base + n)");
      DADE_REQUIRE(assign[loc] < 0, DADE_ERR_ARG, "ivf: row id listed twice");
      DADE_REQUIRE(p == off[c] || rid[p] > rid[p - 1], DADE_ERR_ARG, "ivf: ids not ascending inside a list");
      assign[loc] = c;
      pos_of[loc] = (int32_t)p;
    }
}

extern "C" dade_status dade_load(dade_index* x, const char* path) {
  API_BEGIN
  need(x, "index"); need(path, "path");
  DeviceGuard g(x->device);
  FILE* f = fopen(path, "rb");
  DADE_REQUIRE(f, DADE_ERR_ARG, std::string("cannot open ") + path);
  struct Closer { FILE* f; ~Closer() { fclose(f); } } cl{f};
  int64_t hdr[6];
  rd(f, hdr, sizeof(hdr));
  DADE_REQUIRE(hdr[0] == (int64_t)kMagic, DADE_ERR_ARG, "not a DADE index file");
  DADE_REQUIRE(hdr[1] == x->D, DADE_ERR_SHAPE, "file D differs from the index D");
  const int D = x->D;
  // header ranges before any allocation sized by them
  DADE_REQUIRE(hdr[3] >= 1 && hdr[3] < ((int64_t)1 << 31), DADE_ERR_ARG, "file: n out of range");
  DADE_REQUIRE(hdr[2] >= 1 && hdr[2] <= hdr[3], DADE_ERR_ARG, "file: nlist out of range");
  DADE_REQUIRE(hdr[4] >= 0 && hdr[4] + hdr[3] < ((int64_t)1 << 31), DADE_ERR_ARG, "file: id_base out of range");
  DADE_REQUIRE(hdr[5] == 0 || hdr[5] == 1, DADE_ERR_ARG, "file: bad calibration flag");
  const int nlist = (int)hdr[2];
  const int64_t n = hdr[3];
  std::vector<double> mean(D), R((size_t)D * D), lam(D);
  rd(f, mean.data(), 8 * D); rd(f, R.data(), 8 * R.size()); rd(f, lam.data(), 8 * D);
  std::vector<float> cent((size_t)nlist * D), lay((size_t)n * D);
  std::vector<int64_t> off(nlist + 1), rid(n);
  std::vector<int32_t> asg(n);
  rd(f, cent.data(), 4 * cent.size()); rd(f, off.data(), 8 * off.size());
  rd(f, rid.data(), 8 * rid.size()); rd(f, asg.data(), 4 * asg.size());
  rd(f, lay.data(), 4 * lay.size());
  std::vector<double> m1, v;
  int64_t c[3] = {0, 0, 0};
  if (hdr[5]) {
    rd(f, c, sizeof(c));
    DADE_REQUIRE(c[0] >= 1 && c[0] <= DADE_MAX_K && c[1] >= 1 && c[1] <= ((int64_t)1 << 31) && c[2] == D / 16 - 1,
                 DADE_ERR_ARG, "file: bad calibration header");
    m1.resize(c[2]); v.resize((size_t)c[2] * c[1]);
    rd(f, m1.data(), 8 * m1.size()); rd(f, v.data(), 8 * v.size());
  }
  // contents: the same checks as a build, before any state changes
  std::vector<int32_t> asg_chk, pos_of;
  check_ivf(n, hdr[4], nlist, off, rid, asg_chk, pos_of);
  DADE_REQUIRE(asg_chk == asg, DADE_ERR_ARG, "file: assign does not match the lists");
  for (double t : mean) DADE_REQUIRE(std::isfinite(t), DADE_ERR_NONFINITE, "file: non-finite mean");
  for (double t : R) DADE_REQUIRE(std::isfinite(t), DADE_ERR_NONFINITE, "file: non-finite R");
  for (float t : cent) DADE_REQUIRE(std::isfinite(t), DADE_ERR_NONFINITE, "file: non-finite centroids");
  for (float t : lay) DADE_REQUIRE(std::isfinite(t), DADE_ERR_NONFINITE, "file: non-finite layout");
  DBuf<float> cent_d, lay_d;
  DBuf<int32_t> off_d, rid_d;
  cent_d.reserve(cent.size()); lay_d.reserve(lay.size()); off_d.reserve(nlist + 1); rid_d.reserve(n);
  std::vector<int32_t> off32(off.begin(), off.end()), rid32(rid.begin(), rid.end());
  DADE_CK(cudaMemcpy(cent_d.p, cent.data(), 4 * cent.size(), cudaMemcpyHostToDevice));
  DADE_CK(cudaMemcpy(lay_d.p, lay.data(), 4 * lay.size(), cudaMemcpyHostToDevice));
  DADE_CK(cudaMemcpy(off_d.p, off32.data(), 4 * off32.size(), cudaMemcpyHostToDevice));
  DADE_CK(cudaMemcpy(rid_d.p, rid32.data(), 4 * rid32.size(), cudaMemcpyHostToDevice));
  // commit
  x->mean = mean; x->R = R; x->lam = lam; x->has_lam = true;
  upload_rotation(x);
  std::swap(x->cent, cent_d); std::swap(x->layout, lay_d); std::swap(x->off_d, off_d); std::swap(x->row_id_d, rid_d);
  cent_d.release(); lay_d.release(); off_d.release(); rid_d.release();
  x->off_h = off; x->row_id_h = rid; x->assign_h = asg; x->pos_of_h = std::move(pos_of);
  x->nlist = nlist; x->n = n; x->id_base = hdr[4]; x->has_ivf = true; x->xnorm_ok = false;
  tc_prepare(x, x->cent.p, nlist, x->cent_tc, true);
  x->has_cal = hdr[5] != 0;
  if (x->has_cal) { x->calK = (int)c[0]; x->n0 = (int)c[1]; x->ncls = (int)c[2]; x->m1 = m1; x->v = v; }
  API_END
}

// ================================================================== injection of a ready layout
extern "C" dade_status dade_set_ivf(dade_index* x, const float* Xrot, int64_t n, int64_t id_base,
                                    const int64_t* row_id, const int64_t* off, int nlist,
                                    const float* centroids) {
  API_BEGIN
  need(x, "index"); need(Xrot, "Xrot"); need(row_id, "row_id"); need(off, "off"); need(centroids, "centroids");
  DADE_REQUIRE(x->has_rot, DADE_ERR_STATE, "set_ivf needs the rotation the layout was made with");
  DADE_REQUIRE(n >= 1 && n < ((int64_t)1 << 31), DADE_ERR_ARG, "n out of range");
  DADE_REQUIRE(nlist >= 1 && nlist <= n, DADE_ERR_ARG, "nlist not in [1, n]");
  DeviceGuard g(x->device);
  const int D = x->D;
  cudaStream_t st = x->stream;
  std::vector<int64_t> offv(off, off + nlist + 1), rid(row_id, row_id + n);
  std::vector<int32_t> asg, pos_of;
  check_ivf(n, id_base, nlist, offv, rid, asg, pos_of);
  check_finite(x, Xrot, n * D, "Xrot");
  check_finite(x, centroids, (int64_t)nlist * D, "centroids");
  DBuf<float> cent, lay;
  DBuf<int32_t> off_d, rid_d;
  cent.reserve((size_t)nlist * D); lay.reserve((size_t)n * D); off_d.reserve(nlist + 1); rid_d.reserve(n);
  std::vector<int32_t> off32(offv.begin(), offv.end()), rid32(rid.begin(), rid.end());
  DADE_CK(cudaMemcpyAsync(cent.p, centroids, sizeof(float) * nlist * D, cudaMemcpyDeviceToDevice, st));
  DADE_CK(cudaMemcpyAsync(off_d.p, off32.data(), 4 * off32.size(), cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(rid_d.p, rid32.data(), 4 * rid32.size(), cudaMemcpyHostToDevice, st));
  launch_to_blocked(Xrot, n, D, lay.p, st);
  DADE_CK(cudaStreamSynchronize(st));
  std::swap(x->cent, cent); std::swap(x->layout, lay); std::swap(x->off_d, off_d); std::swap(x->row_id_d, rid_d);
  cent.release(); lay.release(); off_d.release(); rid_d.release();
  x->off_h = std::move(offv); x->row_id_h = std::move(rid); x->assign_h = std::move(asg); x->pos_of_h = std::move(pos_of);
  x->nlist = nlist; x->n = n; x->id_base = id_base;
  tc_prepare(x, x->cent.p, nlist, x->cent_tc, true);
  x->has_ivf = true; x->has_cal = false; x->xnorm_ok = false; x->has_graph = false;
  pq_encode_layout(x);
  API_END
}

// ================================================================== options
extern "C" dade_status dade_set_option(dade_index* x, int option, int64_t value) {
  API_BEGIN
  need(x, "index");
  Options& o = x->opt;
  auto in = [&](std::initializer_list<int64_t> ok) {
    for (int64_t v : ok) if (v == value) return;
    throw Error(DADE_ERR_ARG, "option value not allowed");
  };
  switch (option) {
    case DADE_OPT_KNN_PATH: in({0, 1, 2, 3, 4, 5, 6}); o.knn_path = (int)value; break;
    case DADE_OPT_PROBE_PASSES: in({0, 1, 3}); o.probe_passes = (int)value; break;
    case DADE_OPT_SCAN_WARPS: in({0, 1, 2, 4, 8}); o.scan_warps = (int)value; break;
    case DADE_OPT_SCAN_ORDER: in({0, 1, 2}); o.scan_order = (int)value; break;
    case DADE_OPT_SCAN_TAIL:
      DADE_REQUIRE(value >= 0 && value < ((int64_t)1 << 31), DADE_ERR_ARG, "scan tail out of range");
      o.scan_tail = (int)value; break;
    case DADE_OPT_HOST_CHUNKS:
      DADE_REQUIRE(value >= 1 && value <= 1024, DADE_ERR_ARG, "host chunks not in [1, 1024]");
      o.host_chunks = (int)value; break;
    case DADE_OPT_HOST_PREP_CHUNKS:
      DADE_REQUIRE(value >= 0 && value <= 64, DADE_ERR_ARG, "prep chunks not in [0, 64]");
      o.host_prep_chunks = (int)value; break;
    case DADE_OPT_DHAT_ARES: in({0, 1}); o.dhat_ares = (int)value; break;
    case DADE_OPT_DHAT_H16: in({0, 1, 2, 3}); o.dhat_h16 = (int)value; break;
    case DADE_OPT_SHARD_EXCHANGES:
      DADE_REQUIRE(value >= 0 && value <= 16, DADE_ERR_ARG, "shard exchanges not in [0, 16]");
      o.shard_exchanges = (int)value; break;
    case DADE_OPT_FZ_STAGES: DADE_REQUIRE(value >= 0 && value <= 16, DADE_ERR_ARG, "fz stages not in [0, 16]");
      o.fz_stages = (int)value; break;
    case DADE_OPT_FZ_GROUPS: in({0, 1, 2}); o.fz_groups = (int)value; break;
    case DADE_OPT_FZ_CPS: in({0, 1, 2}); o.fz_cps = (int)value; break;
    case DADE_OPT_FZ_DEBUG: in({0, 1, 2}); g_fz_debug = (int)value; break;
    case DADE_OPT_PCA_TC: in({0, 1}); g_pca_tc = (int)value; break;
    case DADE_OPT_SCAN_P1: in({0, 1}); o.scan_p1 = (int)value; break;
    case DADE_OPT_KNN_I8: in({0, 1}); o.knn_i8 = (int)value; break;
    case DADE_OPT_FZ_SEED_STRIDE: DADE_REQUIRE(value >= 0 && value <= 64, DADE_ERR_ARG, "fz seed stride not in [0, 64]");
      o.fz_seed_stride = (int)value; break;
    case DADE_OPT_FZ_ROWS: in({0, 1, 2}); o.fz_rows = (int)value; break;
    case DADE_OPT_FZ_COLS: in({0, 1, 2}); o.fz_cols = (int)value; break;
    case DADE_OPT_GMIN_RATIO: DADE_REQUIRE(value >= 1 && value <= 1024, DADE_ERR_ARG, "gmin ratio not in [1, 1024]");
      o.gmin_ratio = (int)value; break;
    case DADE_OPT_DHAT_CHUNK_MB: DADE_REQUIRE(value >= 0 && value <= 8192, DADE_ERR_ARG, "dhat chunk not in [0, 8192] MB");
      o.dhat_chunk_mb = (int)value; break;
    case DADE_OPT_FZ_CPC: DADE_REQUIRE(value >= 0 && value <= 64, DADE_ERR_ARG, "fz cpc not in [0, 64]");
      o.fz_cpc = (int)value; break;
    default: throw Error(DADE_ERR_ARG, "unknown option");
  }
  API_END
}

// ================================================================== decision log (parity)
extern "C" dade_status dade_search_log(dade_index* x, const float* Q, int nq, int K, int nprobe, int delta_d,
                                       int method, double param, int64_t* ids, float* dists, int32_t* log,
                                       int64_t log_cap, int64_t* log_count) {
  API_BEGIN
  need(x, "index"); need(log_count, "log_count");
  DADE_REQUIRE(log_cap >= 0, DADE_ERR_ARG, "log_cap < 0");
  if (log_cap > 0) need(log, "log");
  DADE_REQUIRE(method != DADE_METHOD_BSA_RES, DADE_ERR_UNSUPPORTED, "decision log: BSA-p and ADSampling only");
  DeviceGuard g(x->device);
  DecisionLog dl;
  dl.buf = log; dl.cap = log_cap; dl.count = log_count;
  *log_count = 0;
  do_search(x, Q, nq, K, nprobe, delta_d, param, ids, dists, nullptr, method, nullptr, nullptr, &dl);
  API_END
}

// ================================================================== multi-rank
extern "C" dade_status dade_comm_unique_id(void* id128) {
  API_BEGIN
  need(id128, "id");
  comm_unique_id(id128);
  API_END
}

extern "C" dade_status dade_set_comm(dade_index* x, const void* id128, int nranks, int rank) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, DADE_ERR_ARG, "bad nranks / rank");
  DeviceGuard g(x->device);
  unsigned char own[128];
  if (!id128) {
    DADE_REQUIRE(nranks == 1, DADE_ERR_ARG, "a group of more than one rank needs the shared unique id");
    comm_unique_id(own);
    id128 = own;
  }
  Comm* c = comm_create(id128, nranks, rank);
  comm_destroy(x->comm);
  x->comm = c;
  API_END
}

// a0 over a sharded base: fp64 partial moments of the owned strided-sample rows, all-reduced
extern "C" dade_status dade_fit_rotation_dist(dade_index* x, const float* X, int64_t n, int64_t id_base,
                                              int64_t n_total, int64_t sample_size) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->comm, DADE_ERR_STATE, "dade_fit_rotation_dist needs dade_set_comm");
  DeviceGuard g(x->device);
  const int D = x->D;
  std::vector<double> sum(D + 1), cov((size_t)D * D);
  int64_t cnt = 0;
  dade_status s = dade_pca_mean_partial(x, X, n, id_base, n_total, sample_size, sum.data(), &cnt);
  if (s != DADE_OK) throw Error(s, g_err);
  sum[D] = (double)cnt;                                   // exact: counts < 2^53
  allreduce_host(x, sum.data(), sum.size());
  const int64_t tot = (int64_t)sum[D];
  DADE_REQUIRE(tot > 0, DADE_ERR_ARG, "empty PCA sample");
  std::vector<double> mean(D);
  for (int j = 0; j < D; ++j) mean[j] = sum[j] / (double)tot;
  s = dade_pca_cov_partial(x, X, n, id_base, n_total, sample_size, mean.data(), cov.data());
  if (s != DADE_OK) throw Error(s, g_err);
  allreduce_host(x, cov.data(), cov.size());
  s = dade_set_rotation_from_cov(x, mean.data(), cov.data(), tot);
  if (s != DADE_OK) throw Error(s, g_err);
  API_END
}

// a2 over a sharded base: k-means (R19) on the GLOBAL strided sample — the init rows and every
// Lloyd step's fp64 per-cluster sums / counts all-reduced, the update on every rank — then this
// rank's sub-lists for all nlist global centroids (a1 + a2 on the shard)
extern "C" dade_status dade_build_ivf_dist(dade_index* x, const float* X, int64_t n, int64_t id_base,
                                           int64_t n_total, int nlist, int kmeans_iters) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->comm, DADE_ERR_STATE, "dade_build_ivf_dist needs dade_set_comm");
  DADE_REQUIRE(kmeans_iters >= 0, DADE_ERR_ARG, "kmeans_iters < 0");
  DeviceGuard g(x->device);
  const int D = x->D;
  std::vector<double> sums((size_t)nlist * D);
  std::vector<int64_t> counts(nlist);
  std::vector<float> cent((size_t)nlist * D);
  dade_status s = dade_kmeans_partial(x, X, n, id_base, n_total, nlist, nullptr, sums.data(), counts.data());
  if (s != DADE_OK) throw Error(s, g_err);
  allreduce_host(x, sums.data(), sums.size());
  for (size_t i = 0; i < cent.size(); ++i) cent[i] = (float)sums[i];   // the first nlist sampled rows
  for (int it = 0; it < kmeans_iters; ++it) {
    s = dade_kmeans_partial(x, X, n, id_base, n_total, nlist, cent.data(), sums.data(), counts.data());
    if (s != DADE_OK) throw Error(s, g_err);
    allreduce_host(x, sums.data(), sums.size());
    allreduce_host(x, counts.data(), counts.size());
    kmeans_update(nlist, D, sums.data(), counts.data(), cent.data());
  }
  DBuf<float> cd;
  cd.reserve(cent.size());
  DADE_CK(cudaMemcpyAsync(cd.p, cent.data(), 4 * cent.size(), cudaMemcpyHostToDevice, x->stream));
  s = dade_build_ivf(x, X, n, id_base, nlist, cd.p, 0);
  cd.release();
  if (s != DADE_OK) throw Error(s, g_err);
  API_END
}

// a3 over a sharded base (R14-R16): merged K-NN, merged negatives, summed pair features, then the
// same fit on every rank — the table equals an unsharded dade_calibrate on the whole base
extern "C" dade_status dade_calibrate_dist(dade_index* x, const float* X, const float* Qc, int nq, int K,
                                           int n_neg, int nprobe_neg, uint64_t seed) {
  API_BEGIN
  need(x, "index"); need(X, "X"); need(Qc, "Qc");
  DADE_REQUIRE(x->comm, DADE_ERR_STATE, "dade_calibrate_dist needs dade_set_comm");
  DeviceGuard g(x->device);
  calib_checks(x, Qc, nq, K, n_neg, nprobe_neg);
  DADE_REQUIRE(K <= x->n, DADE_ERR_ARG, "K > shard size");
  const int S = comm_size(x->comm);
  std::vector<int64_t> ki;
  std::vector<double> kd;
  calib_knn(x, X, Qc, nq, K, ki, kd);
  std::vector<int64_t> gi((size_t)S * nq * K), mi((size_t)nq * K);
  std::vector<double> gd((size_t)S * nq * K), md((size_t)nq * K);
  allgather_host(x, ki.data(), ki.size(), gi.data());
  allgather_host(x, kd.data(), kd.size(), gd.data());
  merge_knn(S, nq, K, gi.data(), gd.data(), mi.data(), md.data());
  std::vector<std::vector<std::pair<uint64_t, int64_t>>> neg;
  calib_negatives(x, Qc, nq, K, mi.data(), n_neg, nprobe_neg, seed, neg);
  const size_t w = std::max(n_neg, 1);
  std::vector<uint64_t> keys((size_t)nq * w, 0), gk((size_t)S * nq * w);
  std::vector<int64_t> nid((size_t)nq * w, 0), gn((size_t)S * nq * w);
  std::vector<int32_t> cnt(nq), gc((size_t)S * nq);
  for (int q = 0; q < nq; ++q) {
    cnt[q] = (int32_t)neg[q].size();
    for (size_t j = 0; j < neg[q].size(); ++j) { keys[q * w + j] = neg[q][j].first; nid[q * w + j] = neg[q][j].second; }
  }
  allgather_host(x, keys.data(), keys.size(), gk.data());
  allgather_host(x, nid.data(), nid.size(), gn.data());
  allgather_host(x, cnt.data(), cnt.size(), gc.data());
  const size_t cap = (size_t)nq * (K + n_neg);
  std::vector<int32_t> pq(cap);
  std::vector<int64_t> pid(cap);
  std::vector<double> tau(cap), y(cap);
  const int64_t np = calibration_pairs(S, nq, K, (int)w, mi.data(), md.data(), gk.data(), gn.data(), gc.data(),
                                       pq.data(), pid.data(), tau.data(), y.data());
  std::vector<double> F;
  pair_features(x, Qc, nq, (int)np, pq.data(), pid.data(), F);
  allreduce_host(x, F.data(), F.size());
  fit_calibration(x, K, (int)np, F.data(), tau.data(), y.data());
  API_END
}

// host combination steps of the sharded build (no index, no GPU): the process-group driver
// (sharded.py) moves the buffers and calls these
extern "C" dade_status dade_kmeans_update(int nlist, int D, const double* sums, const int64_t* counts,
                                          float* centroids) {
  API_BEGIN
  need(sums, "sums"); need(counts, "counts"); need(centroids, "centroids");
  DADE_REQUIRE(nlist >= 1 && D >= 1, DADE_ERR_ARG, "bad nlist / D");
  kmeans_update(nlist, D, sums, counts, centroids);
  API_END
}

extern "C" dade_status dade_merge_knn(int S, int nq, int K, const int64_t* ids, const double* dists,
                                      int64_t* out_ids, double* out_dists) {
  API_BEGIN
  need(ids, "ids"); need(dists, "dists"); need(out_ids, "out_ids"); need(out_dists, "out_dists");
  DADE_REQUIRE(S >= 1 && nq >= 0 && K >= 1, DADE_ERR_ARG, "bad S / nq / K");
  merge_knn(S, nq, K, ids, dists, out_ids, out_dists);
  API_END
}

extern "C" dade_status dade_calibration_pairs(int S, int nq, int K, int n_neg, const int64_t* knn_ids,
                                              const double* knn_dists, const uint64_t* keys, const int64_t* neg_ids,
                                              const int32_t* counts, int32_t* pair_q, int64_t* pair_id,
                                              double* tau, double* y, int64_t* npairs) {
  API_BEGIN
  need(knn_ids, "knn_ids"); need(knn_dists, "knn_dists"); need(counts, "counts"); need(npairs, "npairs");
  need(pair_q, "pair_q"); need(pair_id, "pair_id"); need(tau, "tau"); need(y, "y");
  DADE_REQUIRE(S >= 1 && nq >= 0 && K >= 1 && n_neg >= 1, DADE_ERR_ARG, "bad S / nq / K / n_neg");
  *npairs = calibration_pairs(S, nq, K, n_neg, knn_ids, knn_dists, keys, neg_ids, counts, pair_q, pair_id, tau, y);
  API_END
}

// ================================================================== NEXT-3 BSA-q (§V-B)
// OPQ on a strided sample of min(n, n_train) rows (R28): PCA-initialised,
// `iters` rounds of {per-subspace k-means (km_iters Lloyd iterations, warm-started), orthogonal
// Procrustes R = V U^T of M = sum (x - mu) y^T = U S V^T (computed as (M^T M)^(-1/2) M^T)}, then
// final_iters Lloyd iterations on the final rotation. Installs (mu, R) as the index rotation
// (discarding a built IVF) and the codebooks.
extern "C" dade_status dade_train_pq(dade_index* x, const float* X, int64_t n, int m, int64_t n_train, int iters,
                                     int km_iters, int final_iters) {
  API_BEGIN
  need(x, "index"); need(X, "X");
  const int D = x->D;
  DADE_REQUIRE(m >= 1 && D % m == 0 && D / m <= 32, DADE_ERR_ARG, "m must divide D with D/m <= 32");
  DADE_REQUIRE(iters >= 0 && km_iters >= 0 && final_iters >= 0, DADE_ERR_ARG, "negative iteration count");
  const int64_t ns = std::min<int64_t>(n, n_train > 0 ? n_train : 65536);
  DADE_REQUIRE(ns >= 256, DADE_ERR_ARG, "OPQ needs at least 256 training rows");
  DeviceGuard g(x->device);
  cudaStream_t st = x->stream;
  check_finite(x, X, n * D, "X");
  const int ds = D / m;
  // the strided sample (row-major ns x D)
  std::vector<int32_t> sid(ns);
  for (int64_t k = 0; k < ns; ++k) sid[k] = (int32_t)(((__int128)k * n) / ns);
  DBuf<int32_t> sid_d;
  DBuf<float> Xs, Z, Cd;
  DBuf<double> mu_d, R_d, M_d;
  DBuf<uint8_t> codes;
  RotOp rop;
  RotWs rws;
  sid_d.reserve(ns); Xs.reserve((size_t)ns * D); Z.reserve((size_t)ns * D); Cd.reserve((size_t)D * 256);
  mu_d.reserve(D); R_d.reserve((size_t)D * D); M_d.reserve((size_t)D * D); codes.reserve((size_t)ns * m);
  DADE_CK(cudaMemcpyAsync(sid_d.p, sid.data(), 4 * ns, cudaMemcpyHostToDevice, st));
  launch_gather_rows(X, sid_d.p, ns, D, Xs.p, st);
  // PCA of the sample (its mean centres everything)
  std::vector<double> sum(D), cov((size_t)D * D), mean(D), R, lam;
  int64_t cnt = 0;
  dade_status s = dade_pca_mean_partial(x, Xs.p, ns, 0, ns, ns, sum.data(), &cnt);
  if (s != DADE_OK) throw Error(s, g_err);
  for (int j = 0; j < D; ++j) mean[j] = sum[j] / (double)cnt;
  s = dade_pca_cov_partial(x, Xs.p, ns, 0, ns, ns, mean.data(), cov.data());
  if (s != DADE_OK) throw Error(s, g_err);
  for (auto& c : cov) c /= (double)cnt;
  rotation_from_cov(D, cov, R, lam);
  DADE_CK(cudaMemcpyAsync(mu_d.p, mean.data(), 8 * D, cudaMemcpyHostToDevice, st));
  std::vector<float> C((size_t)D * 256), Zh((size_t)ns * D);
  std::vector<uint8_t> ch((size_t)ns * m);
  bool have_C = false;
  auto rotate_sample = [&]() {
    DADE_CK(cudaMemcpyAsync(R_d.p, R.data(), 8 * R.size(), cudaMemcpyHostToDevice, st));
    rot_prepare(rop, R_d.p, D, st);
    launch_rotate(rop, rws, Xs.p, nullptr, ns, mu_d.p, Z.p, nullptr, st);
    DADE_CK(cudaMemcpyAsync(Zh.data(), Z.p, 4 * Zh.size(), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    if (!have_C) {  // init: the first 256 sampled rows' sub-vectors (R28)
      for (int j = 0; j < m; ++j)
        for (int c = 0; c < 256; ++c)
          for (int i = 0; i < ds; ++i) C[((size_t)j * 256 + c) * ds + i] = Zh[(size_t)c * D + j * ds + i];
      have_C = true;
    }
  };
  auto assign_all = [&]() {
    DADE_CK(cudaMemcpyAsync(Cd.p, C.data(), 4 * C.size(), cudaMemcpyHostToDevice, st));
    launch_pq_assign(Z.p, false, ns, D, m, Cd.p, codes.p, m, st);
    DADE_CK(cudaMemcpyAsync(ch.data(), codes.p, ch.size(), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
  };
  std::vector<double> sums((size_t)D * 256);
  std::vector<int64_t> cnts((size_t)m * 256);
  auto lloyd = [&](int its) {  // centroid = fp64 mean (sample order) rounded to fp32; empty keeps
    for (int it = 0; it < its; ++it) {
      assign_all();
      std::fill(sums.begin(), sums.end(), 0.0);
      std::fill(cnts.begin(), cnts.end(), (int64_t)0);
      for (int64_t r = 0; r < ns; ++r)
        for (int j = 0; j < m; ++j) {
          const int c = ch[(size_t)r * m + j];
          ++cnts[(size_t)j * 256 + c];
          double* sr = &sums[((size_t)j * 256 + c) * ds];
          const float* zr = &Zh[(size_t)r * D + j * ds];
          for (int i = 0; i < ds; ++i) sr[i] += (double)zr[i];
        }
      for (int j = 0; j < m; ++j)
        for (int c = 0; c < 256; ++c) {
          const int64_t k = cnts[(size_t)j * 256 + c];
          if (k > 0)
            for (int i = 0; i < ds; ++i)
              C[((size_t)j * 256 + c) * ds + i] = (float)(sums[((size_t)j * 256 + c) * ds + i] / (double)k);
        }
    }
  };
  std::vector<double> M((size_t)D * D), MtM((size_t)D * D), ev(D), V((size_t)D * D), T((size_t)D * D);
  for (int t = 0; t < iters; ++t) {
    rotate_sample();
    lloyd(km_iters);
    assign_all();  // codes of the updated codebooks -> reconstructions y
    DADE_CK(cudaMemcpyAsync(Cd.p, C.data(), 4 * C.size(), cudaMemcpyHostToDevice, st));
    launch_pq_cross(Xs.p, mu_d.p, ns, D, m, Cd.p, codes.p, M_d.p, st);
    DADE_CK(cudaMemcpyAsync(M.data(), M_d.p, 8 * M.size(), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    // R = V S^-1 V^T M^T with M^T M = V S^2 V^T (the polar factor: R = V U^T for M = U S V^T)
    for (int a = 0; a < D; ++a)
      for (int b = a; b < D; ++b) {
        double acc = 0;
        for (int k = 0; k < D; ++k) acc += M[(size_t)k * D + a] * M[(size_t)k * D + b];
        MtM[(size_t)a * D + b] = MtM[(size_t)b * D + a] = acc;
      }
    sym_eig(D, MtM.data(), ev.data(), V.data());  // V column-major: V[k * D + a] = V_a,k
    for (int k = 0; k < D; ++k) {
      DADE_REQUIRE(ev[k] > 0, DADE_ERR_ARG, "OPQ: singular cross-product (degenerate training data)");
      const double inv = 1.0 / std::sqrt(ev[k]);
      for (int b = 0; b < D; ++b) {  // T[k][b] = (V^T M^T)[k][b] / s_k = sum_c V_c,k M[b][c] / s_k
        double acc = 0;
        for (int c = 0; c < D; ++c) acc += V[(size_t)k * D + c] * M[(size_t)b * D + c];
        T[(size_t)k * D + b] = acc * inv;
      }
    }
    for (int a = 0; a < D; ++a)
      for (int b = 0; b < D; ++b) {
        double acc = 0;
        for (int k = 0; k < D; ++k) acc += V[(size_t)k * D + a] * T[(size_t)k * D + b];
        R[(size_t)a * D + b] = acc;
      }
  }
  rotate_sample();
  lloyd(final_iters);
  // install: the OPQ rotation becomes the index rotation (invalidates a built IVF), then codebooks
  x->mean = mean;
  x->R = R;
  x->lam.assign(D, 0.0);
  x->has_lam = false;
  upload_rotation(x);
  install_pq(x, m, C.data());
  API_END
}

extern "C" dade_status dade_set_pq(dade_index* x, int m, const float* codebooks) {
  API_BEGIN
  need(x, "index"); need(codebooks, "codebooks");
  DADE_REQUIRE(x->has_rot, DADE_ERR_STATE, "set_pq needs the rotation the codebooks live in");
  DeviceGuard g(x->device);
  install_pq(x, m, codebooks);
  API_END
}

extern "C" dade_status dade_get_pq(const dade_index* x, int* m, float* codebooks, uint8_t* codes, float* err) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_pq, DADE_ERR_STATE, "no PQ codebooks");
  if (m) *m = x->pq_m;
  if (codebooks) memcpy(codebooks, x->pq_C.data(), sizeof(float) * x->pq_C.size());
  if (codes || err) {
    DADE_REQUIRE(x->pq_codes_ok, DADE_ERR_STATE, "no PQ codes (build the IVF)");
    DeviceGuard g(x->device);
    std::vector<uint8_t> rows((size_t)x->n * x->pq_stride);
    DADE_CK(cudaMemcpyAsync(rows.data(), x->pq_codes.p, rows.size(), cudaMemcpyDeviceToHost, x->stream));
    DADE_CK(cudaStreamSynchronize(x->stream));
    for (int64_t p = 0; p < x->n; ++p) {
      const uint8_t* r = &rows[(size_t)p * x->pq_stride];
      if (codes) memcpy(codes + (size_t)p * x->pq_m, r, x->pq_m);
      if (err) memcpy(err + p, r + x->pq_eo, 4);
    }
  }
  API_END
}

// §V-A correction on the ADC distance (BSA-q; R29): the calibration pairs of
// dade_calibrate (R14-R16), features (ADC dis', reconstruction error e) in fp64 from the stored
// codes and the GPU-rotated queries, the two-feature logistic fit, v = sort_desc(tau - m1 dis' - m2 e)
// over the Label-0 pairs
extern "C" dade_status dade_calibrate_pq(dade_index* x, const float* X, const float* Qc, int nq, int K, int n_neg,
                                         int nprobe_neg, uint64_t seed) {
  API_BEGIN
  need(x, "index"); need(X, "X"); need(Qc, "Qc");
  DeviceGuard g(x->device);
  calib_checks(x, Qc, nq, K, n_neg, nprobe_neg);
  DADE_REQUIRE(x->has_pq && x->pq_codes_ok, DADE_ERR_STATE, "calibrate_pq needs PQ codes");
  DADE_REQUIRE(K <= x->n, DADE_ERR_ARG, "K not in [1, n]");
  const int D = x->D;
  cudaStream_t st = x->stream;
  std::vector<int64_t> ki;
  std::vector<double> kd;
  calib_knn(x, X, Qc, nq, K, ki, kd);
  std::vector<std::vector<std::pair<uint64_t, int64_t>>> neg;
  calib_negatives(x, Qc, nq, K, ki.data(), n_neg, nprobe_neg, seed, neg);
  std::vector<int32_t> pq, prow;
  std::vector<double> ptau, py;
  for (int qi = 0; qi < nq; ++qi) {
    const double tau = kd[(size_t)qi * K + K - 1];
    for (int j = 0; j < K; ++j) {
      pq.push_back(qi); prow.push_back(x->pos_of_h[ki[(size_t)qi * K + j] - x->id_base]);
      ptau.push_back(tau); py.push_back(0.0);
    }
    for (const auto& c : neg[qi]) {
      pq.push_back(qi); prow.push_back(x->pos_of_h[c.second - x->id_base]); ptau.push_back(tau); py.push_back(1.0);
    }
  }
  const int np = (int)pq.size();
  DBuf<float> qr;
  DBuf<int32_t> pq_d, pr_d;
  DBuf<double> feat;
  qr.reserve((size_t)nq * D); pq_d.reserve(np); pr_d.reserve(np); feat.reserve((size_t)2 * np);
  launch_rotate(x->rot_op, x->rot_ws, Qc, nullptr, nq, x->mean_d.p, qr.p, nullptr, st);
  DADE_CK(cudaMemcpyAsync(pq_d.p, pq.data(), 4 * np, cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(pr_d.p, prow.data(), 4 * np, cudaMemcpyHostToDevice, st));
  launch_pq_pair_feat(x->pq_codes.p, x->pq_stride, x->pq_eo, x->pq_m, D, x->pq_Cd.p, qr.p, pq_d.p, pr_d.p, np,
                      feat.p, st);
  std::vector<double> F((size_t)2 * np);
  DADE_CK(cudaMemcpyAsync(F.data(), feat.p, 8 * F.size(), cudaMemcpyDeviceToHost, st));
  DADE_CK(cudaStreamSynchronize(st));
  std::vector<double> mv;
  double beta;
  logistic_irls_multi(F, 2, ptau, py, 1e-8, 100, 1e-12, mv, &beta);
  std::vector<double> v;
  for (int i = 0; i < np; ++i)
    if (py[i] == 0.0) v.push_back(ptau[i] - mv[0] * F[2 * (size_t)i] - mv[1] * F[2 * (size_t)i + 1]);
  std::sort(v.begin(), v.end(), std::greater<double>());
  x->mq[0] = mv[0];
  x->mq[1] = mv[1];
  x->vq = std::move(v);
  x->n0q = (int)x->vq.size();
  x->calqK = K;
  x->has_calq = true;
  API_END
}

extern "C" dade_status dade_get_calibration_q(const dade_index* x, int* K, int* n0, double* m2, double* v) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_calq, DADE_ERR_STATE, "no PQ calibration");
  if (K) *K = x->calqK;
  if (n0) *n0 = x->n0q;
  if (m2) { m2[0] = x->mq[0]; m2[1] = x->mq[1]; }
  if (v) memcpy(v, x->vq.data(), sizeof(double) * x->vq.size());
  API_END
}

extern "C" dade_status dade_set_calibration_q(dade_index* x, int K, int n0, const double* m2, const double* v) {
  API_BEGIN
  need(x, "index"); need(m2, "m"); need(v, "v");
  DADE_REQUIRE(K >= 1 && K <= DADE_MAX_K && n0 >= 1, DADE_ERR_ARG, "bad K / n0");
  DADE_REQUIRE(x->has_pq, DADE_ERR_STATE, "set_calibration_q needs PQ codebooks");
  x->mq[0] = m2[0];
  x->mq[1] = m2[1];
  x->vq.assign(v, v + n0);
  x->n0q = n0;
  x->calqK = K;
  x->has_calq = true;
  API_END
}

// ================================================================== NEXT-4 graph refinement
namespace {
void install_graph(dade_index* x, const std::vector<int32_t>& adj_pos, int M0, int entry_pos) {
  x->g_adj.reserve(adj_pos.size());
  DADE_CK(cudaMemcpyAsync(x->g_adj.p, adj_pos.data(), 4 * adj_pos.size(), cudaMemcpyHostToDevice, x->stream));
  int sms = 0;
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->device));
  x->g_slots = graph_slots(sms);
  const size_t words = (size_t)((x->n + 31) / 32);
  x->g_vis.reserve((size_t)x->g_slots * words);
  DADE_CK(cudaMemsetAsync(x->g_vis.p, 0, 4 * (size_t)x->g_slots * words, x->stream));
  x->g_vlist.reserve((size_t)x->g_slots * 8192);
  DADE_CK(cudaStreamSynchronize(x->stream));
  x->g_M0 = M0;
  x->g_entry = entry_pos;
  x->has_graph = true;
}
}  // namespace

// Inject a base-layer graph (R33): nbrs host n x M0 global ids (row i = global id id_base + i; -1
// pads), entry = global id of the entry point. The graph lives over this index's rows.
extern "C" dade_status dade_set_graph(dade_index* x, const int64_t* nbrs, int M0, int64_t entry) {
  API_BEGIN
  need(x, "index"); need(nbrs, "nbrs");
  DADE_REQUIRE(x->has_ivf, DADE_ERR_STATE, "set_graph needs the index's rows (build_ivf)");
  DADE_REQUIRE(M0 >= 1 && M0 <= 32, DADE_ERR_ARG, "M0 not in [1, 32]");
  DADE_REQUIRE(entry >= x->id_base && entry < x->id_base + x->n, DADE_ERR_ARG, "entry outside the index");
  DeviceGuard g(x->device);
  std::vector<int32_t> adj((size_t)x->n * M0, -1);
  for (int64_t i = 0; i < x->n; ++i)
    for (int j = 0; j < M0; ++j) {
      const int64_t u = nbrs[(size_t)i * M0 + j];
      if (u < 0) continue;
      DADE_REQUIRE(u >= x->id_base && u < x->id_base + x->n, DADE_ERR_ARG, "neighbour id outside the index");
      adj[(size_t)x->pos_of_h[i] * M0 + j] = x->pos_of_h[u - x->id_base];
    }
  install_graph(x, adj, M0, x->pos_of_h[entry - x->id_base]);
  API_END
}

extern "C" dade_status dade_get_graph(const dade_index* x, int* M0, int64_t* nbrs, int64_t* entry) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_graph, DADE_ERR_STATE, "no graph");
  if (M0) *M0 = x->g_M0;
  if (entry) *entry = x->row_id_h[x->g_entry];
  if (nbrs) {
    DeviceGuard g(x->device);
    std::vector<int32_t> adj((size_t)x->n * x->g_M0);
    DADE_CK(cudaMemcpyAsync(adj.data(), x->g_adj.p, 4 * adj.size(), cudaMemcpyDeviceToHost, x->stream));
    DADE_CK(cudaStreamSynchronize(x->stream));
    for (int64_t i = 0; i < x->n; ++i)
      for (int j = 0; j < x->g_M0; ++j) {
        const int32_t pv = adj[(size_t)x->pos_of_h[i] * x->g_M0 + j];
        nbrs[(size_t)i * x->g_M0 + j] = pv < 0 ? -1 : x->row_id_h[pv];
      }
  }
  API_END
}

// Build the base-layer graph (R33): each row's P nearest other rows from an exact IVF search of
// the row itself at nprobe_pool lists (nprobe_pool = nlist: the exact P nearest), HNSW's heuristic
// down to M0 on the GPU, entry = the row nearest to the rotation's mean (min ||x~||^2, lower id on
// ties). X: device n x D raw rows of this index (the IVF's input).
extern "C" dade_status dade_build_graph(dade_index* x, const float* X, int M0, int P, int nprobe_pool) {
  API_BEGIN
  need(x, "index"); need(X, "X");
  DADE_REQUIRE(x->has_ivf && x->has_rot, DADE_ERR_STATE, "build_graph needs build_ivf");
  DADE_REQUIRE(M0 >= 1 && M0 <= 32 && P >= M0 && P <= 128 && P < x->n, DADE_ERR_ARG, "need 1 <= M0 <= 32, M0 <= P <= 128, P < n");
  DADE_REQUIRE(nprobe_pool >= 1 && nprobe_pool <= x->nlist, DADE_ERR_ARG, "nprobe_pool not in [1, nlist]");
  DeviceGuard g(x->device);
  const int64_t n = x->n;
  const int K = P + 1;
  cudaStream_t st = x->stream;
  std::vector<int32_t> pool((size_t)n * P, -1);
  std::vector<float> pool_d((size_t)n * P, INFINITY);
  const int64_t chunk = 65536;
  DBuf<int64_t> ids;
  DBuf<float> ds;
  ids.reserve((size_t)chunk * K);
  ds.reserve((size_t)chunk * K);
  std::vector<int64_t> hi((size_t)chunk * K);
  std::vector<float> hd((size_t)chunk * K);
  for (int64_t r0 = 0; r0 < n; r0 += chunk) {
    const int m = (int)std::min(chunk, n - r0);
    do_search(x, X + r0 * x->D, m, K, nprobe_pool, 16, 0.0, ids.p, ds.p, nullptr);
    DADE_CK(cudaMemcpyAsync(hi.data(), ids.p, 8 * (size_t)m * K, cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaMemcpyAsync(hd.data(), ds.p, 4 * (size_t)m * K, cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    for (int i = 0; i < m; ++i) {
      const int64_t gid = x->id_base + r0 + i;
      const size_t row = (size_t)x->pos_of_h[r0 + i] * P;
      int c = 0;
      for (int j = 0; j < K && c < P; ++j) {
        const int64_t u = hi[(size_t)i * K + j];
        if (u < 0 || u == gid) continue;
        pool[row + c] = x->pos_of_h[u - x->id_base];
        pool_d[row + c] = hd[(size_t)i * K + j];
        ++c;
      }
    }
  }
  ids.release(); ds.release();
  DBuf<int32_t> pool_dev, adj_dev;
  DBuf<float> pd_dev;
  pool_dev.reserve(pool.size()); pd_dev.reserve(pool_d.size()); adj_dev.reserve((size_t)n * M0);
  DADE_CK(cudaMemcpyAsync(pool_dev.p, pool.data(), 4 * pool.size(), cudaMemcpyHostToDevice, st));
  DADE_CK(cudaMemcpyAsync(pd_dev.p, pool_d.data(), 4 * pool_d.size(), cudaMemcpyHostToDevice, st));
  launch_graph_prune(x->layout.p, n, x->D, pool_dev.p, pd_dev.p, P, M0, adj_dev.p, st);
  std::vector<int32_t> adj((size_t)n * M0);
  DADE_CK(cudaMemcpyAsync(adj.data(), adj_dev.p, 4 * adj.size(), cudaMemcpyDeviceToHost, st));
  // entry: min ||x~||^2 (the row nearest to mu), ties to the lower id
  if (!x->xnorm_ok) {
    x->xnorm.reserve((size_t)std::max<int64_t>(n, 1));
    launch_row_norms(x->layout.p, n, x->D, x->xnorm.p, st);
    x->xnorm_ok = true;
  }
  std::vector<float> nrm(n);
  DADE_CK(cudaMemcpyAsync(nrm.data(), x->xnorm.p, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
  DADE_CK(cudaStreamSynchronize(st));
  int entry = 0;
  for (int64_t p = 1; p < n; ++p)
    if (nrm[p] < nrm[entry] || (nrm[p] == nrm[entry] && x->row_id_h[p] < x->row_id_h[entry])) entry = (int)p;
  install_graph(x, adj, M0, entry);
  API_END
}

// HNSW base-layer refinement with the DCO (R34): Q device nq x D raw; result queue of size ef,
// tau = its max frozen per expansion; BSA-p step table from the calibration (calibrated with K =
// ef; alpha = 0: no pruning); the first K of the queue -> ids / dists (device nq x K). stats may be
// NULL; log (device, log_cap x 3 int32: query, id, dims read per tested node) may be NULL.
extern "C" dade_status dade_graph_search(dade_index* x, const float* Q, int nq, int K, int ef, int delta_d,
                                         double alpha, int64_t* ids, float* dists, dade_stats* stats, int32_t* log,
                                         int64_t log_cap, int64_t* log_count) {
  API_BEGIN
  need(x, "index");
  DADE_REQUIRE(x->has_graph, DADE_ERR_STATE, "graph search needs a graph (dade_build_graph / dade_set_graph)");
  DADE_REQUIRE(nq >= 0, DADE_ERR_ARG, "nq < 0");
  DADE_REQUIRE(K >= 1 && ef >= K && ef <= DADE_MAX_K, DADE_ERR_ARG, "need 1 <= K <= ef <= DADE_MAX_K");
  const int D = x->D;
  DADE_REQUIRE(delta_d >= 16 && delta_d % 16 == 0 && D % delta_d == 0, DADE_ERR_ARG,
               "delta_d must be a positive multiple of 16 dividing D");
  DADE_REQUIRE(alpha >= 0.0 && alpha < 1.0, DADE_ERR_ARG, "significance not in [0,1)");
  const int nsteps = D / delta_d;
  const bool prune = alpha > 0.0 && nsteps > 1;
  if (prune) {
    DADE_REQUIRE(x->has_cal, DADE_ERR_STATE, "significance > 0 requires calibration (with K = ef)");
    DADE_REQUIRE(x->calK == ef, DADE_ERR_STATE, "the calibration's K differs from ef");
  }
  if (log) DADE_REQUIRE(log_count != nullptr && log_cap >= 0, DADE_ERR_ARG, "log needs log_count");
  if (nq == 0) { if (log_count) *log_count = 0; g_err.clear(); return DADE_OK; }
  need(Q, "Q"); need(ids, "ids"); need(dists, "dists");
  DeviceGuard g(x->device);
  cudaStream_t st = x->stream;
  check_finite(x, Q, (int64_t)nq * D, "Q");
  x->qrot.reserve((size_t)nq * D);
  launch_rotate(x->rot_op, x->rot_ws, Q, nullptr, nq, x->mean_d.p, x->qrot.p, nullptr, st);
  GraphParams p{};
  if (x->nlist > 1) {  // R33: entry = first row of the query's nearest non-empty list (exact probes)
    p.eprobe = std::min(x->nlist, 8);
    x->probes.reserve((size_t)nq * p.eprobe);
    exact_knn(x, Q, nq, x->cent.p, x->nlist, p.eprobe, x->probes.p, nullptr, x->cent_tc, false, probe_passes(x));
    p.eprobes = x->probes.p;
    p.off = x->off_d.p;
  }
  p.qrot = x->qrot.p; p.layout = x->layout.p; p.row_id = x->row_id_d.p; p.adj = x->g_adj.p; p.n = x->n;
  p.D = D; p.nq = nq; p.K = K; p.ef = ef; p.M0 = x->g_M0; p.entry = x->g_entry;
  p.dd = prune ? delta_d / 16 : 1;
  p.nsteps = prune ? nsteps : D / 16;
  for (int s2 = 1; s2 < p.nsteps; ++s2) {
    if (prune) {  // the scan's step table (R4, R5)
      const int idx = (s2 * delta_d) / 16 - 1;
      const double alpha_s = (alpha * delta_d) / D;
      long k = (long)std::ceil((1.0 - alpha_s) * (double)x->n0);
      k = std::min<long>(std::max<long>(k, 1), x->n0);
      p.m1[s2 - 1] = (float)x->m1[idx];
      p.beta[s2 - 1] = (float)x->v[(size_t)idx * x->n0 + (k - 1)];
    } else {
      p.m1[s2 - 1] = 1.f;
      p.beta[s2 - 1] = -INFINITY;
    }
  }
  p.out_ids = ids; p.out_d = dists;
  p.visited = x->g_vis.p; p.vlist = x->g_vlist.p; p.vcap = 8192;
  x->work.reserve(2);
  DADE_CK(cudaMemsetAsync(x->work.p, 0, sizeof(int), st));
  p.work = x->work.p;
  if (stats) {
    x->counters.reserve(4 + DADE_MAX_STEPS + 8);
    DADE_CK(cudaMemsetAsync(x->counters.p, 0, sizeof(unsigned long long) * (4 + DADE_MAX_STEPS + 8), st));
    p.counters = x->counters.p;
  }
  if (log) {
    x->dlog_n.reserve(1);
    DADE_CK(cudaMemsetAsync(x->dlog_n.p, 0, sizeof(unsigned long long), st));
    p.dlog = log; p.dlog_cap = log_cap; p.dlog_n = x->dlog_n.p;
  }
  int sms = 0;
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->device));
  if (stats) DADE_CK(cudaEventRecord(x->ev[0] ? x->ev[0] : (cudaEventCreate(&x->ev[0]), x->ev[0]), st));
  launch_graph_search(p, sms, st);
  if (log) {
    unsigned long long c = 0;
    DADE_CK(cudaMemcpyAsync(&c, x->dlog_n.p, sizeof(c), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    *log_count = (int64_t)c;
  }
  if (stats) {
    if (!x->ev[3]) DADE_CK(cudaEventCreate(&x->ev[3]));
    DADE_CK(cudaEventRecord(x->ev[3], st));
    unsigned long long c[4 + DADE_MAX_STEPS + 8];
    DADE_CK(cudaMemcpyAsync(c, x->counters.p, sizeof(c), cudaMemcpyDeviceToHost, st));
    DADE_CK(cudaStreamSynchronize(st));
    memset(stats, 0, sizeof(*stats));
    stats->tested = (int64_t)c[0];
    stats->survivors = (int64_t)c[1];
    int64_t dims = (int64_t)c[1] * D;
    for (int s2 = 1; s2 < DADE_MAX_STEPS; ++s2) dims += (int64_t)c[4 + s2] * s2 * (p.dd * 16);
    stats->dims_scanned = dims;
    stats->n_epochs = (int32_t)std::min<unsigned long long>(c[2], 0x7fffffffull);  // expansions
    for (int s2 = 0; s2 < DADE_MAX_STEPS; ++s2) stats->pruned_at_step[s2] = (int64_t)c[4 + s2];
    stats->n_steps = p.nsteps;
    cudaEventElapsedTime(&stats->ms_total, x->ev[0], x->ev[3]);
    stats->ms_scan = stats->ms_total;
  }
  API_END
}
