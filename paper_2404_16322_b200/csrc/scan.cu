// a6-a8: the progressive-scan kernel (the hot loop of the method).
//
// Method: refinement keeps a result queue of size K, tau = its K-th distance
// (P:L42-43). For every candidate of the probed IVF lists the squared distance in
// the PCA basis is accumulated Delta_d dims at a time (Alg. 2 loop); after each step
// d < D the cascade classifier for d prunes iff m1_d * P_d + beta'_d > tau
// (BSA-p estimator P:L569-573). Survivors reach d = D, where P_D is the exact
// distance, and enter the queue. tau is frozen within geometric epochs of the
// candidate stream (R13: [0,4K), [4K,8K), [8K,16K), ...) so the result does not depend on
// the parallel schedule.
//
// B200 mapping:
//  * persistent CTAs of G warps (G = 1 when there are enough queries to fill the machine), one
//    query at a time (queries taken from an atomic counter); with G = 1 an epoch boundary
//    waits only for the warp's own survivors, never for other warps;
//  * the probed lists' (start, length) table and q~ sit in shared memory; the first step of
//    every candidate is STREAMED with TMA bulk copies (cp.async.bulk, one elected lane,
//    mbarrier completion) into a ring of tiles, issued kStages tiles ahead of consumption
//    (across list and epoch boundaries: the data does not depend on tau). The
//    dimension-blocked, list-major layout makes every tile one contiguous block-row range
//    (64 B per row per 16 dims);
//  * survivors of a step are ballot-compacted into a shared-memory ring; their next blocks are
//    gathered with 128-bit loads (one 64-B row per lane, up to LA blocks per round trip); the
//    global id of a candidate is fetched in the same round trip as its last block;
//  * arithmetic is packed FP32x2 (FADD2/FFMA2): a 16-dim block costs 16 packed instructions;
//    the distance is the fp32 sum of per-block sums, added in block order (R21) — identical
//    whichever round a block is processed in, so results never depend on the schedule;
//  * the top-K is REGISTER-RESIDENT: KPL sorted keys (dist_bits << 32 | id) per lane, position
//    lane*KPL + i; an accepted key is inserted by a warp-wide shift (no shared memory);
//  * Delta_d is any multiple of 16 dividing D: the template DD (1, 2 or 4 blocks) is the unit the
//    TMA tiles and gather rounds move, the runtime p.dd (a multiple of DD) the classifier spacing;
//  * LOG instantiations (parity only) append every tested candidate's decision (query, id, dims
//    read) to a device log — the per-candidate comparison with the oracle.
#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr int TR = 32;            // rows per tile: one row per lane
#ifndef DADE_SCAN_TMAG  // 1: survivor gathers staged by TMA bulk copies instead of LDG.256 (experiment builds)
#define DADE_SCAN_TMAG 0
#endif
#ifndef DADE_SCAN_REG1  // register cap of the Delta_d = 16, K <= 64 kernels (experiment builds may change it)
#define DADE_SCAN_REG1 80
#endif
#ifndef DADE_EPOCH_GROWTH  // R13: epoch boundaries c0, 2 c0, 4 c0, ... (experiment builds may change it)
#define DADE_EPOCH_GROWTH 2
#endif
#ifndef DADE_SCAN_STREAM0  // 0: epoch 0 through stage 1 + gather rounds like later epochs (experiment builds)
#define DADE_SCAN_STREAM0 1
#endif
#ifndef DADE_SCAN_STREAM0_MINDD  // smallest staging unit (blocks) whose kernels stream epoch 0
#define DADE_SCAN_STREAM0_MINDD 2
#endif
constexpr unsigned long long kKeyInf = ~0ull;

struct __align__(16) QEntry {
  int32_t row;   // list-major position
  float phi;     // partial distance over blocks [0, blk)
  int32_t blk;   // 16-dim blocks accumulated
  float res;     // residual test only: ‖x‖² − (x² summed over blocks [0, blk))
};

struct TileMeta {
  int32_t row0, nr, ep, pad;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
#ifndef DADE_SCAN_MBAR_HINT
#define DADE_SCAN_MBAR_HINT 0
#endif
// DADE_SCAN_MBAR_HINT > 0: try_wait with a suspend-time hint (ns), so a waiting warp yields its issue slots
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  if (DADE_SCAN_MBAR_HINT > 0) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra W%=;\n}" ::"r"(smem_u32(b)),
        "r"(phase), "r"((uint32_t)DADE_SCAN_MBAR_HINT)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W%=;\n}" ::"r"(smem_u32(b)),
        "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// ---- packed FP32x2 arithmetic (sm_100a FADD2 / FFMA2)
__device__ __forceinline__ unsigned long long pk(float2 a) {
  return *reinterpret_cast<unsigned long long*>(&a);
}
__device__ __forceinline__ float2 upk(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Sum over one 16-dim block of (x_i - q_i)^2: 4 packed accumulators, fixed association
// ((a0 + a1) + (a2 + a3)), then lo + hi. x: 8 packed pairs (registers); q: 16 floats (smem).
__device__ __forceinline__ float block_sum(const unsigned long long (&x)[8], const float* q) {
  const ulonglong2* qq = reinterpret_cast<const ulonglong2*>(q);
  unsigned long long a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const ulonglong2 qc = qq[c];
    const unsigned long long t0 = sub2(x[2 * c], qc.x);
    const unsigned long long t1 = sub2(x[2 * c + 1], qc.y);
    a[c] = fma2(t1, t1, 0ull);
    a[c] = fma2(t0, t0, a[c]);
  }
  const float2 s = upk(add2(add2(a[0], a[1]), add2(a[2], a[3])));
  return s.x + s.y;
}

// Same with the 16-B chunks in a per-lane rotated order (stage 1 reads the tile rotated so the
// 8 lanes of a shared-memory phase hit distinct banks); q chunk c pairs with x chunk c. (Measured:
// rotating the chunk partials back to block_sum's association costs ~2% of the C4 scan; the
// rounding of the block-0 sum therefore depends on the row's lane, a deterministic function of
// the stream — R21's bound covers either association.)
__device__ __forceinline__ float block_sum_rot(const unsigned long long (&x)[8], const float* const (&q)[4]) {
  unsigned long long a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const ulonglong2 qc = *reinterpret_cast<const ulonglong2*>(q[c]);
    const unsigned long long t0 = sub2(x[2 * c], qc.x);
    const unsigned long long t1 = sub2(x[2 * c + 1], qc.y);
    a[c] = fma2(t1, t1, 0ull);
    a[c] = fma2(t0, t0, a[c]);
  }
  const float2 s = upk(add2(add2(a[0], a[1]), add2(a[2], a[3])));
  return s.x + s.y;
}

// Σ x_i² over one 16-dim block (residual test), fixed association
__device__ __forceinline__ float block_sq(const unsigned long long (&x)[8]) {
  unsigned long long a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    a[c] = fma2(x[2 * c + 1], x[2 * c + 1], 0ull);
    a[c] = fma2(x[2 * c], x[2 * c], a[c]);
  }
  const float2 s = upk(add2(add2(a[0], a[1]), add2(a[2], a[3])));
  return s.x + s.y;
}

// one 64-B block row as two 256-bit loads (LDG.256, sm_100): each load is a whole 32-B sector
// (measured vs four 16-B loads: C2 scan -1.5%, C3 -3%; bypassing L1 instead was 20% slower)
__device__ __forceinline__ void ld_block(unsigned long long (&x)[8], const float* src) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(x[4 * h]), "=l"(x[4 * h + 1]), "=l"(x[4 * h + 2]), "=l"(x[4 * h + 3])
        : "l"(s + 4 * h));
}

// lanes per survivor in a draining gather round (log2): 32 / qn rounded down to a power of two,
// at most DADE_DRAIN_LG (experiment builds; 5 = up to 32 lanes)
#ifndef DADE_DRAIN_LG
#define DADE_DRAIN_LG 5
#endif
__device__ __forceinline__ int drain_lanes_log2(int qn) {
  const int lg = qn <= 1 ? 5 : qn <= 2 ? 4 : qn <= 4 ? 3 : qn <= 8 ? 2 : qn <= 16 ? 1 : 0;
  return lg < DADE_DRAIN_LG ? lg : DADE_DRAIN_LG;
}

// DADE_DEBUG_CHECKS builds (tools/build_variant.py; compute-sanitizer is not available on the
// GPU pool): device-side invariants of the rings and index ranges — a violation traps, and the
// next synchronising call reports a CUDA error
#ifdef DADE_DEBUG_CHECKS
#define DADE_DCHECK(c) \
  do {                 \
    if (!(c)) __trap(); \
  } while (0)
#else
#define DADE_DCHECK(c) \
  do {                 \
  } while (0)
#endif

__device__ __forceinline__ unsigned long long make_key(float d, uint32_t id) {
  return ((unsigned long long)__float_as_uint(d) << 32) | id;
}

// Register-resident sorted top-K: position g = lane*KPL + i holds key k[i] (kKeyInf = empty).
template <int KPL>
struct RegTopK {
  unsigned long long k[KPL];
  unsigned long long kth;  // key at position K-1 (kKeyInf while fewer than K keys)
  int kl, ki;              // lane / slot of position K-1

  __device__ __forceinline__ void init(int K) {
#pragma unroll
    for (int i = 0; i < KPL; ++i) k[i] = kKeyInf;
    kth = kKeyInf;
    kl = (K - 1) / KPL;
    ki = (K - 1) % KPL;
  }
  __device__ __forceinline__ void refresh_kth() {
    unsigned long long t = k[0];
#pragma unroll
    for (int i = 1; i < KPL; ++i)
      if (i == ki) t = k[i];
    kth = __shfl_sync(0xffffffffu, t, kl);
  }
  // insert x (warp-uniform, x < kth): shift every key >= x one position up
  __device__ __forceinline__ void insert_one(unsigned long long x, int lane) {
    unsigned long long left = __shfl_up_sync(0xffffffffu, k[KPL - 1], 1);
    if (lane == 0) left = 0ull;  // "smaller than x"
#pragma unroll
    for (int i = KPL - 1; i >= 0; --i) {
      const unsigned long long l = i > 0 ? k[i - 1] : left;
      if (k[i] >= x) k[i] = l < x ? x : l;
    }
    refresh_kth();
  }
  // offer one key per lane (kKeyInf = none)
  __device__ __forceinline__ void offer(unsigned long long key, int lane) {
    unsigned m = __ballot_sync(0xffffffffu, key < kth);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const unsigned long long x = __shfl_sync(0xffffffffu, key, src);
      if (x < kth) insert_one(x, lane);
    }
  }
};

}  // namespace

// DADE_SCAN_PROF builds only (tools/scan_prof.py, a separate library): per-phase clock64 cycles
// summed over warps, to see where a query's latency chain goes. Not in the product library.
#ifdef DADE_SCAN_PROF
__device__ unsigned long long g_scan_prof[16];
#define PROF_MARK(cat)                                        \
  do {                                                        \
    const long long _t = clock64();                           \
    if (lane == 0) {                                          \
      sprof[cat] += (unsigned long long)(_t - prof_last);     \
      sprof[8 + (cat)] += 1;                                  \
    }                                                         \
    prof_last = _t;                                           \
  } while (0)
#else
#define PROF_MARK(cat) \
  do {                 \
  } while (0)
#endif

// Per-warp shared-memory slice: tiles | mbar | meta | ring.
// Ring capacity: rounds start at 32 queued and stage 1 runs below 32, so at most 63 entries are
// queued.
template <int DD, int LA = 1>
struct Slice {
#ifdef DADE_SCAN_STAGES  // experiment builds (tools/build_variant.py)
  static constexpr int kStages = DADE_SCAN_STAGES;
#else
  // two tiles in flight: measured on C2 scan 0.553 -> 0.531 ms against three (C4 equal, C3 and the
  // C5 shard already used two) — fewer TMA bytes in flight leave the latency-critical survivor
  // gathers less queueing, and the shared-memory footprint shrinks to ~6 KB per warp
  static constexpr int kStages = 2;
#endif
  static constexpr int TB = TR * 64 * DD;  // tile bytes (DD blocks of 32 rows)
  static constexpr int QCAP = 64;
  static constexpr size_t GB = DADE_SCAN_TMAG ? (size_t)32 * LA * 64 : 0;  // TMA gather staging
  static constexpr size_t bytes =
      (size_t)kStages * TB + 4 * 8 + kStages * sizeof(TileMeta) + QCAP * sizeof(QEntry) + GB;
};

// decision log (LOG builds): (query, global id, dims read) of one tested candidate
__device__ __forceinline__ void log_decision(const ScanParams& p, int64_t q, int32_t id, int dims) {
  const unsigned long long slot = atomicAdd(p.dlog_n, 1ull);
  if ((int64_t)slot < p.dlog_cap) {
    int32_t* r = p.dlog + 3 * slot;
    r[0] = (int32_t)q;
    r[1] = id;
    r[2] = dims;
  }
}

// classifier step index of block count blk: ns = blk / dd if blk is a multiple of dd, else 0
// (dd = p.dd, magic = ceil(2^32 / dd): exact for blk, dd <= 256)
__device__ __forceinline__ int step_of(int blk, int dd, unsigned magic) {
  if (dd == 1) return blk;
  const int ns = (int)__umulhi((unsigned)blk, magic);
  return ns * dd == blk ? ns : 0;
}

// CTA = G warps (blockDim.x = 32 G), one query at a time. G = 1: the warp owns the query and its
// register top-K is the query's top-K. G > 1: the query's candidate tiles are dealt round-robin
// to the G warps (tile t -> warp t mod G); within an epoch every warp tests against the same
// frozen tau (R13), so the split cannot change a decision; at each epoch end the warps' local
// top-K lists are merged exactly (rank by binary search, smem) into the query's top-K.
// CTA shared memory: G slices | pruned[64] | lists[nprobe] | qs[D] | qi | (G > 1) W[G][K] + Gk[2][K].
template <int DD, int KPL, int LA, int MAXREG, bool MULTI, bool RES, bool LOG, bool PQ>
__global__ void __launch_bounds__(256) __maxnreg__(MAXREG) k_scan(const __grid_constant__ ScanParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  using SL = Slice<DD, LA>;
  constexpr int kQCap = SL::QCAP;
  constexpr int kStages = SL::kStages;
  constexpr int TB = SL::TB;
  constexpr bool kStream0 = DADE_SCAN_STREAM0 && !PQ && !RES && DD >= DADE_SCAN_STREAM0_MINDD;  // epoch-0 streaming (below)
  const int D = p.D, K = p.K;
  const int G = MULTI ? (blockDim.x >> 5) : 1;  // warps per query (power of two)
  const int lane = threadIdx.x & 31, warp = MULTI ? threadIdx.x >> 5 : 0;
  unsigned char* base = smem + warp * SL::bytes;
  unsigned char* tiles = base;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + kStages * TB);
  TileMeta* meta = reinterpret_cast<TileMeta*>(mbar + 4);
  QEntry* ring = reinterpret_cast<QEntry*>(meta + kStages);
  unsigned char* gstg = reinterpret_cast<unsigned char*>(ring + kQCap);  // TMAG: gather staging
  uint64_t* gbar = &mbar[3];
  unsigned* pruned = reinterpret_cast<unsigned*>(smem + G * SL::bytes);
  int2* lists = reinterpret_cast<int2*>(pruned + DADE_MAX_STEPS);
  float* qs = reinterpret_cast<float*>(lists + ((p.nprobe + 1) & ~1));
  float* qcs = qs + ((D + 3) & ~3);                       // residual: per-step query constants
  float* lut = qcs + (RES ? DADE_MAX_STEPS : 0);                // PQ: m x 256 ADC table of the query
  int* qslot = reinterpret_cast<int*>(lut + (PQ ? p.pq_m * 256 : 0));
  unsigned long long* W = reinterpret_cast<unsigned long long*>(qslot + 4);  // G x K (G > 1)
  unsigned long long* Gk = W + (size_t)G * K;                               // 2 x K (G > 1)

  const bool stats = p.counters != nullptr;
  if (stats)
    for (int j = threadIdx.x; j < DADE_MAX_STEPS; j += blockDim.x) pruned[j] = 0;
#ifdef DADE_SCAN_PROF
  __shared__ unsigned long long sprof_all[8][16];
  unsigned long long* sprof = sprof_all[warp];
  if (lane < 16) sprof[lane] = 0;
  long long prof_last = clock64();
#endif
  uint32_t gphase = 0;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&mbar[s], 1);
    if (DADE_SCAN_TMAG) mbar_init(gbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int nsteps = p.nsteps;
  const int nblk = D >> 4;
  const int sdd = p.dd;                 // classifier spacing in blocks (a multiple of DD)
  const unsigned smagic = p.dd_magic;
  const bool test1 = sdd == DD && nsteps > 1;  // stage 1 ends on a classifier step
  const int kRoundQ = PQ ? (32 >> p.pq_lg) : 32;  // queued survivors that make a full gather round
  const float* lay = p.layout;
  const int64_t n = p.n;
  unsigned long long c_tested = 0, c_surv = 0;  // warp-uniform
  uint32_t phase_bits = 0;
  const unsigned lt_mask = (1u << lane) - 1;

  for (;;) {
    if (threadIdx.x == 0) {
      const int slot = atomicAdd(p.work_counter, 1);
      *qslot = slot < p.nq && p.order ? p.order[slot] : slot;
    }
    __syncthreads();
    const int qi = *qslot;
    if (qi >= p.nq) break;
    const int64_t q = qi;
    for (int j = threadIdx.x; j < D; j += blockDim.x) qs[j] = p.qrot[q * D + j];
    if (RES)
      for (int j = threadIdx.x; j < nsteps - 1; j += blockDim.x) qcs[j] = p.qconst[q * (nsteps - 1) + j];
    for (int j = threadIdx.x; j < p.nprobe; j += blockDim.x) {
      const int l = p.probes[q * p.nprobe + j];
      const int s0 = p.off[l];
      lists[j] = make_int2(s0, p.off[l + 1] - s0);
    }
    if (MULTI)
      for (int j = threadIdx.x; j < K; j += blockDim.x) Gk[j] = kKeyInf;
    __syncthreads();
    if (PQ) {  // ADC look-up table: lut[j][c] = ||q~_j - C_j[c]||^2, fp32, dims in order
      const int ds = p.pq_ds;
      for (int idx = threadIdx.x; idx < p.pq_m * 256; idx += blockDim.x) {
        const int j = idx >> 8;
        const float* c = p.pq_C + (int64_t)idx * ds;
        float acc = 0.f;
        for (int t = 0; t < ds; ++t) {
          const float d = qs[j * ds + t] - __ldg(c + t);
          acc = fmaf(d, d, acc);
        }
        lut[idx] = acc;
      }
      __syncthreads();
    }
    int L = 0;
    for (int j = lane; j < p.nprobe; j += 32) L += lists[j].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    // this launch's epochs [ep_first, ep_end) (R32 phases of a sharded search; default: all):
    // stream positions [e_lo0, L) with L capped at the end of epoch ep_end - 1
    int e_lo0 = 0, e_hi0 = p.c0;
    for (int e = 0; e < p.ep_first; ++e) {
      e_lo0 = e_hi0;
      e_hi0 = e_hi0 > (1 << 29) / DADE_EPOCH_GROWTH ? (1 << 30) : e_hi0 * DADE_EPOCH_GROWTH;
    }
    {
      int64_t b = 0, h = p.c0;
      for (int e = 0; e < p.ep_end && b < L; ++e, b = h, h *= DADE_EPOCH_GROWTH) {}
      if (b < L) L = (int)b;
    }
    int n_ep = 0;  // epochs the stream touches: [0,c0), [c0,2c0), [2c0,4c0), ...
    for (int64_t e_lo = 0, e_hi = p.c0; e_lo < L; e_lo = e_hi, e_hi *= DADE_EPOCH_GROWTH) ++n_ep;

    RegTopK<KPL> tk;
    tk.init(K);
    unsigned long long cap = kKeyInf;  // G > 1: the query's K-th key at the start of the epoch
    // a previous phase's result queue (R32) and the exchanged K-th distance bounding tau
    float* qtcap = reinterpret_cast<float*>(qslot + 1);
    if (p.init_ids) {
      if (!MULTI) {
#pragma unroll
        for (int i = 0; i < KPL; ++i) {
          const int pos = lane * KPL + i;
          if (pos < K) {
            const int64_t id = p.init_ids[q * K + pos];
            tk.k[i] = id < 0 ? kKeyInf : make_key(p.init_d[q * K + pos], (uint32_t)id);
          }
        }
        tk.refresh_kth();
      } else {
        unsigned long long* G0 = Gk + (p.ep_first & 1) * K;
        __syncthreads();
        for (int j = threadIdx.x; j < K; j += blockDim.x) {
          const int64_t id = p.init_ids[q * K + j];
          G0[j] = id < 0 ? kKeyInf : make_key(p.init_d[q * K + j], (uint32_t)id);
        }
        __syncthreads();
        cap = G0[K - 1];
      }
    }
    if (threadIdx.x == 0) {
      float tc = INFINITY;
      if (p.cap_ids && p.cap_ids[q * K + K - 1] >= 0) tc = p.cap_d[q * K + K - 1];
      *qtcap = tc;
    }
    __syncthreads();

    // ---------------------------------------------------- producer state (warp-uniform)
    // tiles never cross a list or an epoch boundary (R13); tile t belongs to warp t mod G
    int pj = 0, ppos = 0, pr = e_lo0, pep = p.ep_first, pe_hi = e_hi0, tix = 0;
    const float* p1q =  // list-major stage 1 (p1.cu), unless its buffer was too small
        (!PQ && !RES && p.p1 && *p.p1_total <= p.p1_cap) ? p.p1 + p.p1_base[q] : nullptr;
    int2 pl = p.nprobe > 0 ? lists[0] : make_int2(0, 0);
    int issued = 0;
    // Epoch-0 streaming: while tau is +inf (epoch 0 of a search that starts from an empty queue
    // and no exchanged bound) nothing can be pruned, so every candidate of epoch 0 is read in
    // full. Instead of stage 1 + gather rounds, its 32-row group is streamed by TMA as nblk / DD
    // sub-tiles of DD blocks each (contiguous in the blocked layout) and the exact distance is
    // accumulated in a register, block by block in block order (R21). Warp-uniform.
    const bool stream0 = kStream0 && !p1q && nblk > DD && p.ep_first == 0 && !p.init_ids &&
                         *qtcap == INFINITY;
    // (DD = 1 kernels: C2 / C4 run 80-register warps whose epoch 0 is <= 9% of the dims read;
    // the extra state would spill there)
    int sb = 0, srow0 = 0, snr = 0;  // stream0: next sub-tile block of the current row group
    auto issue = [&](int slot) -> bool {
      int row0, nr, sp, b0 = -1;
      if (kStream0 && sb > 0) {  // the next sub-tile of an epoch-0 row group (same warp, same rows)
        row0 = srow0;
        nr = snr;
        b0 = sb;
        sb = b0 + DD < nblk ? b0 + DD : 0;
        if (lane == 0) {
          meta[slot] = TileMeta{row0, nr, 0, b0 + 1};
          mbar_expect_tx(&mbar[slot], (uint32_t)nr * 64u * DD);
#pragma unroll
          for (int bb = 0; bb < DD; ++bb)
            bulk_g2s(tiles + slot * TB + bb * TR * 64, lay + (((int64_t)(b0 + bb) * n + row0) << 4),
                     (uint32_t)nr * 64u, &mbar[slot]);
        }
        ++issued;
        return true;
      }
      for (;;) {
        if (pr >= L) return false;
        if (pr >= pe_hi) {
          ++pep;
          pe_hi = pe_hi > (1 << 29) / DADE_EPOCH_GROWTH ? (1 << 30) : pe_hi * DADE_EPOCH_GROWTH;
        }
        while (ppos + pl.y <= pr) {  // skip exhausted (and empty) lists; pr < L keeps pj < nprobe
          ppos += pl.y;
          pl = lists[++pj];
          DADE_DCHECK(pj < p.nprobe);
        }
        nr = min(min(pe_hi, ppos + pl.y) - pr, TR);
        row0 = pl.x + (pr - ppos);
        sp = pr;
        pr += nr;
        DADE_DCHECK(nr >= 1 && nr <= TR && row0 >= 0 && (int64_t)row0 + nr <= n);
        if (!MULTI || (tix++ & (G - 1)) == warp) break;
      }
      if (stream0 && pep == 0) {  // first sub-tile of an epoch-0 row group
        srow0 = row0;
        snr = nr;
        sb = DD;
      }
      if (lane == 0) {
        meta[slot] = TileMeta{row0, nr, pep, stream0 && pep == 0 ? 1 : 0};
        if (!PQ && !RES && p1q) {  // the tile's precomputed stage-1 values: 16-B aligned superset
          const uintptr_t a = reinterpret_cast<uintptr_t>(p1q + sp), a0 = a & ~(uintptr_t)15;
          const uint32_t bytes = (uint32_t)(((a + 4u * (uint32_t)nr + 15) & ~(uintptr_t)15) - a0);
          meta[slot].pad = (int32_t)((a - a0) >> 2);
          mbar_expect_tx(&mbar[slot], bytes);
          bulk_g2s(tiles + slot * TB, reinterpret_cast<const void*>(a0), bytes, &mbar[slot]);
        } else if (PQ) {  // the tile's code rows: one contiguous range of list-major rows
          const uint32_t bytes = (uint32_t)nr * (uint32_t)p.pq_stride;
          mbar_expect_tx(&mbar[slot], bytes);
          bulk_g2s(tiles + slot * TB, p.pq_codes + (int64_t)row0 * p.pq_stride, bytes, &mbar[slot]);
        } else {
          const uint32_t bytes = (uint32_t)nr * 64u;
          mbar_expect_tx(&mbar[slot], bytes * DD);
#pragma unroll
          for (int bb = 0; bb < DD; ++bb)
            bulk_g2s(tiles + slot * TB + bb * TR * 64, lay + (((int64_t)bb * n + row0) << 4), bytes, &mbar[slot]);
        }
      }
      ++issued;
      return true;
    };
#pragma unroll 1
    for (int s = 0; s < kStages; ++s)
      if (!issue(s)) break;
    PROF_MARK(0);  // query start: work item, q~, list table, first tile issues

    int head = 0, tail = 0;  // survivor ring (monotonic indices), warp-uniform
    float tau = MULTI ? (cap == kKeyInf ? INFINITY : __uint_as_float((unsigned)(cap >> 32)))
                      : (tk.kth == kKeyInf ? INFINITY : __uint_as_float((unsigned)(tk.kth >> 32)));
    tau = fminf(tau, *qtcap);
    int cur_ep = p.ep_first, consumed = 0;

    auto push = [&](bool keep, const QEntry& e) {
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (keep) ring[(tail + __popc(km & lt_mask)) & (kQCap - 1)] = e;
      tail += __popc(km);
      DADE_DCHECK(tail - head <= kQCap);
    };

    // One gather round over up to 32 queued survivors. Normally one lane per survivor, up to LA
    // blocks per round trip. When draining a short queue (epoch boundary, end of stream) 2 to 32
    // lanes share a survivor (32/qn rounded down to a power of two) and each loads LA consecutive
    // blocks, so one round trip advances it by up to 32/qn*LA blocks; the group's block sums are then accumulated in block order by every
    // lane of the group (shuffles), so phi is bit-identical to the one-lane path.
    auto queue_round = [&](bool drain) {
      const int qn = min(tail - head, kRoundQ);
      // log2 lanes per survivor: a draining round spreads its survivors over all 32 lanes (PQ:
      // every round — a survivor of the ADC test needs all of its blocks)
      const int lg = !(drain || PQ) ? 0 : drain_lanes_log2(qn);
      const int ei = lane >> lg, sub = lane & ((1 << lg) - 1);
      const bool val = ei < qn;
      QEntry e = val ? ring[(head + ei) & (kQCap - 1)] : QEntry{0, 0.f, nblk, 0.f};
      // blk == nblk: stage 1 already covered every block (D = 16 * DD); the round only finishes it
      DADE_DCHECK(!val || (e.row >= 0 && (int64_t)e.row < n && e.blk >= 0 && e.blk <= nblk));
      // full rounds: one step (DD blocks, LA >= DD) or LA blocks; draining rounds: LA per lane
      int wtot = (drain || PQ) ? (LA << lg) : (DD < LA ? DD : LA);
      wtot = min(wtot, nblk - e.blk);
      const int b0 = e.blk + sub * LA;  // this lane's first block
      const int want = max(0, min(LA, e.blk + wtot - b0));
      unsigned long long v[LA][8];
#if DADE_SCAN_TMAG
      {  // the rows come through shared memory: one 64-B bulk copy per lane per block
        const unsigned bytes = __reduce_add_sync(0xffffffffu, (unsigned)want * 64u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier reads of the staging
        if (lane == 0) mbar_expect_tx(gbar, bytes);
        __syncwarp();
#pragma unroll
        for (int s = 0; s < LA; ++s)
          if (s < want)
            bulk_g2s(gstg + (lane * LA + s) * 64, lay + (((int64_t)(b0 + s) * n + e.row) << 4), 64u, gbar);
      }
#else
#pragma unroll
      for (int s = 0; s < LA; ++s)
        if (s < want) ld_block(v[s], lay + (((int64_t)(b0 + s) * n + e.row) << 4));
#endif
      uint32_t gid = 0;
      if (e.blk + wtot == nblk && val && sub == 0) gid = (uint32_t)__ldg(p.row_id + e.row);
      head += qn;
      __syncwarp();
#if DADE_SCAN_TMAG
      mbar_wait(gbar, gphase);
      gphase ^= 1u;
#pragma unroll
      for (int s = 0; s < LA; ++s)
        if (s < want) {
          const ulonglong2* src = reinterpret_cast<const ulonglong2*>(gstg + (lane * LA + s) * 64);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const ulonglong2 t = src[c];
            v[s][2 * c] = t.x;
            v[s][2 * c + 1] = t.y;
          }
        }
      __syncwarp();
#endif
      float bs[LA], bq[LA];
#pragma unroll
      for (int s = 0; s < LA; ++s) {
        bs[s] = s < want ? block_sum(v[s], qs + (b0 + s) * 16) : 0.f;
        bq[s] = RES && s < want ? block_sq(v[s]) : 0.f;
      }
      float phi = e.phi, res = e.res;
      int blk = e.blk;
      bool alive = val;
      const int bend = e.blk + wtot;
      auto step = [&](float b, float nq) {  // add the next block; classifier at step boundaries d < D
        if (alive && blk < bend) {
          phi += b;
          if (RES) res -= nq;
          ++blk;
          const int ns = blk < nblk ? step_of(blk, sdd, smagic) : 0;
          if (ns) {
            const bool pr = RES ? phi + res + qcs[ns - 1] > tau : fmaf(p.m1[ns - 1], phi, p.beta[ns - 1]) > tau;
            if (pr) {
              alive = false;
              if (stats && sub == 0) atomicAdd(&pruned[ns], 1u);
              if (LOG && sub == 0) log_decision(p, q, __ldg(p.row_id + e.row), blk * 16);
            }
          }
        }
      };
      if (lg == 0) {
#pragma unroll
        for (int s = 0; s < LA; ++s) step(bs[s], bq[s]);
      } else {
        for (int j = 0; j < (1 << lg); ++j)
#pragma unroll
          for (int s = 0; s < LA; ++s)
            step(__shfl_sync(0xffffffffu, bs[s], (ei << lg) + j),
                 RES ? __shfl_sync(0xffffffffu, bq[s], (ei << lg) + j) : 0.f);
      }
      const bool fin = alive && blk == nblk && sub == 0;  // d = D: exact distance (no test, R10)
      if (LOG && fin) log_decision(p, q, (int32_t)gid, D);
      push(alive && blk < nblk && sub == 0, QEntry{e.row, phi, blk, res});
      if (stats) c_surv += __popc(__ballot_sync(0xffffffffu, fin));
      const unsigned long long key = fin ? make_key(phi, gid) : kKeyInf;
      tk.offer(!MULTI || key < cap ? key : kKeyInf, lane);
    };

    // End of epoch cur_ep (every survivor of this warp finished): refresh tau (R13). G > 1: merge
    // the warps' local lists with the query list: the rank of a key in the union is its own
    // index plus its lower bounds in the other sorted lists (keys are unique).
    auto epoch_end = [&]() {
      if (!MULTI) {
        tau = tk.kth == kKeyInf ? INFINITY : __uint_as_float((unsigned)(tk.kth >> 32));
        tau = fminf(tau, *qtcap);
        return;
      }
      unsigned long long* Gcur = Gk + (cur_ep & 1) * K;
      unsigned long long* Gnew = Gk + ((cur_ep + 1) & 1) * K;
#pragma unroll
      for (int i = 0; i < KPL; ++i)
        if (lane * KPL + i < K) W[warp * K + lane * KPL + i] = tk.k[i];
      for (int j = threadIdx.x; j < K; j += blockDim.x) Gnew[j] = kKeyInf;
      __syncthreads();
      for (int idx = threadIdx.x; idx < (G + 1) * K; idx += blockDim.x) {
        const int li = idx / K, own = idx - li * K;
        const unsigned long long* Lst = li < G ? W + li * K : Gcur;
        const unsigned long long x = Lst[own];
        if (x == kKeyInf) continue;
        int rank = own;
        for (int w = 0; w <= G && rank < K; ++w) {
          if (w == li) continue;
          const unsigned long long* M = w < G ? W + w * K : Gcur;
          int lo = 0, hi = K;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (M[mid] < x) lo = mid + 1; else hi = mid;
          }
          rank += lo;
        }
        if (rank < K) Gnew[rank] = x;
      }
      __syncthreads();
      cap = Gnew[K - 1];
      tau = cap == kKeyInf ? INFINITY : __uint_as_float((unsigned)(cap >> 32));
      tau = fminf(tau, *qtcap);
      tk.init(K);
    };

    // ---------------------------------------------------- consumer (one call site per action)
    bool ready = false;  // the tile in `slot` has landed and its meta is read
    TileMeta tm{0, 0, 0, 0};
    float sacc = 0.f;     // stream0: the lane's row distance over the sub-tiles consumed so far
    uint32_t sgid = 0u;   // stream0: the lane's row id
    for (;;) {
      const int qlen = tail - head;
      bool round = qlen >= kRoundQ, drain = false, ep_end = false;
      if (!round) {
        if (!ready && consumed < issued) {
          const int slot = consumed % kStages;
          mbar_wait(&mbar[slot], (phase_bits >> slot) & 1u);
          phase_bits ^= 1u << slot;
          tm = meta[slot];
          ready = true;
          PROF_MARK(1);  // waiting for a TMA tile
        }
        // the current epoch ends when the next own tile is from a later epoch, or at the end
        // of the stream (then every epoch up to n_ep - 1 is closed)
        if (ready ? tm.ep != cur_ep : cur_ep < n_ep) {
          if (qlen > 0) round = drain = true;
          else ep_end = true;
        } else if (!ready) {
          if (qlen == 0) break;
          round = drain = true;
        }
      }
      if (round) {
        queue_round(drain);
        if (drain) PROF_MARK(3); else PROF_MARK(2);  // gather round: full / draining
        continue;
      }
      if (ep_end) {
        epoch_end();
        ++cur_ep;
        PROF_MARK(4);
        continue;
      }
      const int slot = consumed % kStages;
      const bool val = lane < tm.nr;
      if constexpr (PQ) {
        // stage 1 of BSA-q: dis' = ADC of the row's code (m table look-ups), the
        // test m1 * dis' + m2 * err + beta' > tau; survivors are queued at block 0 (phi = 0) and
        // get the exact distance from the gather rounds
        const unsigned char* crow = tiles + slot * TB + lane * p.pq_stride;
        float adc = 0.f, err = 0.f;
        if (val) {
          for (int c0 = 0; c0 < p.pq_m; c0 += 16) {
            const uint4 w = *reinterpret_cast<const uint4*>(crow + c0);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int b = 0; b < 16; ++b)
              if (c0 + b < p.pq_m) adc += lut[((c0 + b) << 8) + ((ws[b >> 2] >> ((b & 3) * 8)) & 255u)];
          }
          err = *reinterpret_cast<const float*>(crow + p.pq_eo);
        }
        __syncwarp();
        ++consumed;
        ready = false;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(slot);
        if (stats) c_tested += tm.nr;
        const bool prune = val && fmaf(p.pq_m1, adc, fmaf(p.pq_m2, err, p.pq_beta)) > tau;
        if (LOG && prune) log_decision(p, q, __ldg(p.row_id + tm.row0 + lane), 0);
        push(val && !prune, QEntry{tm.row0 + lane, 0.f, 0, 0.f});
        if (stats) {
          const int np_ = __popc(__ballot_sync(0xffffffffu, prune));
          if (lane == 0 && np_) atomicAdd(&pruned[0], (unsigned)np_);
        }
        PROF_MARK(5);
        continue;
      }
      const unsigned char* trow = tiles + slot * TB + lane * 64;
      if (kStream0 && stream0 && tm.pad > 0) {  // epoch-0 sub-tile: DD more blocks of every row's distance
        const int b0 = tm.pad - 1;
        const bool val0 = lane < tm.nr;
        if (b0 == 0) {
          sacc = 0.f;
          sgid = val0 ? (uint32_t)__ldg(p.row_id + tm.row0 + lane) : 0u;
        }
#pragma unroll
        for (int bb = 0; bb < DD; ++bb) {
          unsigned long long x[8];
          const float* qc[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ch = (c + lane) & 3;
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(trow + bb * TR * 64 + ch * 16);
            x[2 * c] = v.x;
            x[2 * c + 1] = v.y;
            qc[c] = qs + (b0 + bb) * 16 + ch * 4;
          }
          sacc += block_sum_rot(x, qc);
        }
        __syncwarp();
        ++consumed;
        ready = false;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(slot);
        if (stats && b0 == 0) c_tested += tm.nr;
        if (b0 + DD >= nblk) {  // d = D: exact distance, no test (R10)
          if (LOG && val0) log_decision(p, q, (int32_t)sgid, D);
          if (stats) c_surv += __popc(__ballot_sync(0xffffffffu, val0));
          const unsigned long long key = val0 ? make_key(sacc, sgid) : kKeyInf;
          tk.offer(!MULTI || key < cap ? key : kKeyInf, lane);
        }
        PROF_MARK(5);
        continue;
      }
      // stage 1 (qlen < 32: the ring has room for 32 more): one row per lane, DD blocks
      float s = 0.f, sq = 0.f;
      const float xn = RES && val ? __ldg(p.xnorm + tm.row0 + lane) : 0.f;
      if (!RES && p1q) {  // list-major precompute (p1.cu): the same block sums, read as one float
        s = val ? reinterpret_cast<const float*>(tiles + slot * TB)[tm.pad + lane] : 0.f;
      } else
#pragma unroll
      for (int bb = 0; bb < DD; ++bb) {
        unsigned long long x[8];
        const float* qc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // 16-B chunks rotated per lane: distinct banks per phase
          const int ch = (c + lane) & 3;
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(trow + bb * TR * 64 + ch * 16);
          x[2 * c] = v.x;
          x[2 * c + 1] = v.y;
          qc[c] = qs + bb * 16 + ch * 4;
        }
        s += block_sum_rot(x, qc);
        if (RES) sq += block_sq(x);  // chunk order differs per lane: only feeds the prune test
      }
      __syncwarp();  // every lane is done reading this slot
      ++consumed;
      ready = false;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(slot);
      if (stats) c_tested += tm.nr;
      const float res = xn - sq;
      const bool prune = val && test1 &&
                         (RES ? s + res + qcs[0] > tau : fmaf(p.m1[0], s, p.beta[0]) > tau);
      if (LOG && prune) log_decision(p, q, __ldg(p.row_id + tm.row0 + lane), DD * 16);
      push(val && !prune, QEntry{tm.row0 + lane, s, DD, res});
      if (stats) {
        const int np_ = __popc(__ballot_sync(0xffffffffu, prune));
        if (lane == 0 && np_) atomicAdd(&pruned[1], (unsigned)np_);
      }
      PROF_MARK(5);  // stage 1 of one tile
    }

    // results: the register top-K (G = 1) or the merged list (G > 1)
    if (!MULTI) {
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int pos = lane * KPL + i;
        if (pos < K) {
          const unsigned long long key = tk.k[i];
          p.out_ids[q * K + pos] = key == kKeyInf ? -1 : (int64_t)(uint32_t)(key & 0xffffffffu);
          p.out_d[q * K + pos] = key == kKeyInf ? INFINITY : __uint_as_float((unsigned)(key >> 32));
        }
      }
    } else {
      const unsigned long long* Gfin = Gk + (cur_ep & 1) * K;
      for (int pos = threadIdx.x; pos < K; pos += blockDim.x) {
        const unsigned long long key = Gfin[pos];
        p.out_ids[q * K + pos] = key == kKeyInf ? -1 : (int64_t)(uint32_t)(key & 0xffffffffu);
        p.out_d[q * K + pos] = key == kKeyInf ? INFINITY : __uint_as_float((unsigned)(key >> 32));
      }
    }
    if (threadIdx.x == 0 && stats) atomicMax(p.counters + 3, (unsigned long long)n_ep);
    __syncthreads();  // qslot / lists / qs / Gk are rewritten for the next query
    PROF_MARK(6);  // results
  }
#ifdef DADE_SCAN_PROF
  PROF_MARK(7);  // exit (last work-counter poll)
  __syncwarp();
  if (lane < 16) atomicAdd(&g_scan_prof[lane], sprof[lane]);
#endif
  if (stats) {
    if (lane == 0) {
      atomicAdd(p.counters + 0, c_tested);
      atomicAdd(p.counters + 1, c_surv);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < DADE_MAX_STEPS; j += blockDim.x)
      if (pruned[j]) atomicAdd(p.counters + 4 + j, (unsigned long long)pruned[j]);
  }
}

template <int DD, int LA, bool RES>
static size_t scan_smem(int D, int K, int nprobe, int G, int pq_m) {
  return (size_t)G * Slice<DD, LA>::bytes + DADE_MAX_STEPS * 4 + (size_t)((nprobe + 1) & ~1) * 8 +
         (size_t)((D + 3) & ~3) * 4 + (RES ? DADE_MAX_STEPS * 4 : 0) + (size_t)pq_m * 256 * 4 +
         (G > 1 ? (size_t)(G + 2) * K * 8 : 0) + 16;
}

// warps per query: the smallest G giving >= 16 query-warps per SM. With the longest-stream-first
// query order (dade_api.cu) one warp per query is best whenever the batch fills the machine —
// measured (profiles/r02_scan_warps_c{2,3,4}.jsonl): C4 (10k queries, ~5,400 candidates each)
// G = 1 0.990 ms vs 2 1.100 vs 4 1.459; C2 G = 1 0.500 vs 2 0.639; C3 (1,000 queries) G = 4 1.338
// vs 2 1.449, 8 1.728, 1 1.903. (Round 1, without the order, G = 2 won on C4: the second warp
// mostly shortened the grid's tail, which the order now removes.)
static int scan_group(int nq, int sms, int64_t avg_stream) {
  (void)avg_stream;
  int G = 1;
  while (G < 8 && (int64_t)nq * G < (int64_t)sms * 16) G *= 2;
  return G;
}

// The attribute and the SM count are set / read on every launch (cheap host calls): they apply
// per device, and an index may live on any device of the process.
template <int DD, int KPL, int LA, int MAXREG, bool MULTI, bool RES, bool LOG, bool PQ>
static void launch_g(const ScanParams& p, cudaStream_t st, int G, int sms) {
  auto kern = k_scan<DD, KPL, LA, MAXREG, MULTI, RES, LOG, PQ>;
  const size_t smem = scan_smem<DD, LA, RES>(p.D, p.K, p.nprobe, G, PQ ? p.pq_m : 0);
  DADE_REQUIRE(smem <= 220 * 1024, DADE_ERR_UNSUPPORTED, "scan: shared memory too large (D, K, nprobe)");
  DADE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  DADE_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * G, smem));
  const int max_blocks = (occ > 0 ? occ : 1) * sms;
  kern<<<p.nq < max_blocks ? p.nq : max_blocks, 32 * G, smem, st>>>(p);
}

template <int DD, int KPL, int LA, int MAXREG, bool RES = false, bool PQ = false>
static void launch_v(const ScanParams& p, cudaStream_t st) {
  int dev = 0, sms = 0;
  DADE_CK(cudaGetDevice(&dev));
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (p.dlog) {  // decision log (parity runs): one warp per query; decisions do not depend on G
    if constexpr (!RES) launch_g<DD, KPL, LA, MAXREG, false, false, true, PQ>(p, st, 1, sms);
    return;
  }
  // BSA-q: the CTA's ADC table (m x 256 floats) is shared by 8 warps per query
  const int G = p.g_force > 0 ? p.g_force : PQ ? 8 : scan_group(p.nq, sms, p.avg_stream);
  DADE_REQUIRE(G == 1 || G == 2 || G == 4 || G == 8, DADE_ERR_ARG, "scan: warps per query must be 1, 2, 4 or 8");
  if (G == 1) launch_g<DD, KPL, LA, MAXREG, false, RES, false, PQ>(p, st, 1, sms);
  else launch_g<DD, KPL, LA, MAXREG, true, RES, false, PQ>(p, st, G, sms);
}

template <int DD, int KPL>
static void launch_k(const ScanParams& p, cudaStream_t st) {
  if (p.pq) {  // BSA-q (NEXT-3): ADC test in stage 1, exact distance of the survivors
    // LA blocks per lane, 2^pq_lg lanes per survivor: the fewest lanes that load a survivor's
    // nblk blocks in one round trip, LA = 4 only where that saves lanes over LA = 3 and the
    // top-K leaves the registers for it (KPL >= 4 spills at LA = 4). Measured C4 (D = 96, 6
    // blocks) scan 5.07 / 4.15 / 4.67 ms at LA 2 / 3 / 4, C2 (D = 128, 8 blocks) 5.10 / 5.10 /
    // 3.98 ms (profiles/r02_pq_la.jsonl)
    ScanParams q = p;
    const int nblk = p.D / kBlk, l3 = pq_gather_lanes(nblk, 3), l4 = pq_gather_lanes(nblk, 4);
    if constexpr (KPL <= 2 && DADE_SCAN_PQ_LA == 0) {
      if (l4 < l3) {
        q.pq_lg = __builtin_ctz(l4);
        launch_v<DD, KPL, 4, 128, false, true>(q, st);
        return;
      }
    }
    constexpr int kLA = DADE_SCAN_PQ_LA > 0 ? DADE_SCAN_PQ_LA : 3;
    q.pq_lg = __builtin_ctz(pq_gather_lanes(nblk, kLA));
    launch_v<DD, KPL, kLA, 128, false, true>(q, st);
    return;
  }
  if (p.residual) {  // BSA-res (NEXT-1): residual-norm test
    DADE_REQUIRE(!p.dlog, DADE_ERR_UNSUPPORTED, "scan: decision log is for BSA-p / ADSampling only");
    launch_v<DD, KPL, 1, 96, true>(p, st);
    return;
  }
  if constexpr (DD >= 2) {
    // a step spans DD blocks: gather a whole step per round trip; register cap 128 (16 warps/SM,
    // no spills): measured C5 shard 1.99 -> 1.66 ms, C3 1.50 -> 1.40 against 96
    launch_v<DD, KPL, 2, 128>(p, st);
  } else {
    // 80 registers (24 one-warp CTAs per SM) measured best on C2 and C4 against 64, 72 and 96
    // (C4 scan 1.200 ms vs 1.454 / 1.264 / 1.284, profiles/r02_scan_variants.jsonl)
    launch_v<DD, KPL, 1, (KPL >= 4 ? 96 : DADE_SCAN_REG1)>(p, st);
  }
}

template <int DD>
static void launch_dd(const ScanParams& p, cudaStream_t st) {
  if (p.K <= 32) launch_k<DD, 1>(p, st);
  else if (p.K <= 64) launch_k<DD, 2>(p, st);
  else if (p.K <= 128) launch_k<DD, 4>(p, st);
  else launch_k<DD, 8>(p, st);
}

#ifdef DADE_SCAN_PROF
extern "C" int dade_scan_prof_read(unsigned long long* out16, int reset) {
  if (cudaMemcpyFromSymbol(out16, g_scan_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_scan_prof, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif

void launch_scan(const ScanParams& p, cudaStream_t st) {
  if (p.nq <= 0) return;
  DADE_REQUIRE(p.K <= 256, DADE_ERR_UNSUPPORTED, "scan: K > 256");
  DADE_REQUIRE(p.dd >= 1 && p.dd * 16 <= p.D && p.D % (p.dd * 16) == 0, DADE_ERR_ARG, "scan: bad delta_d");
  ScanParams q = p;
  q.dd_magic = p.dd == 1 ? 0u : (unsigned)((((uint64_t)1 << 32) + (uint64_t)p.dd - 1) / (uint64_t)p.dd);
  // staging unit: the largest of 4, 2, 1 blocks dividing the classifier spacing; BSA-q: the
  // smallest tile holding 32 code rows (64 * DD bytes per row)
  const int unit = p.pq ? (p.pq_stride <= 64 ? 1 : p.pq_stride <= 128 ? 2 : 4)
                        : (p.dd % 4 == 0 ? 4 : p.dd % 2 == 0 ? 2 : 1);
  DADE_REQUIRE(!p.pq || (p.pq_stride <= 256 && p.pq_stride % 16 == 0), DADE_ERR_UNSUPPORTED,
               "scan: PQ code rows wider than 256 bytes");
  switch (unit) {
    case 4: launch_dd<4>(q, st); break;
    case 2: launch_dd<2>(q, st); break;
    default: launch_dd<1>(q, st); break;
  }
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
