// a5 probe (and every exact k-nearest search with small k): the tensor-core distance filter FUSED
// with the candidate selection, so the m x n matrix of filter distances is never written.
//
// Definition (R20): the k nearest columns of every row under the EXACT fp64 sequential
// sum of squared differences, ordered by (dist, column). The filter d_hat and its rigorous error
// window are those of gemm_tf32.cu (centred 3-pass tf32 tcgen05 GEMM): every column whose exact
// distance can be among the k smallest satisfies d_hat <= thr(t), t = the k-th smallest d_hat,
// thr(v) = (v + slack)(1 + delta)/(1 - delta) + slack.
//
// k_probe_tc: CTA = 128 rows x a contiguous range of column tiles (grid.y splits the columns).
// Warp specialisation: warp 0 = TMA producer (bulk copies of pre-split operand chunks into a
// 2-stage ring), warp 1 = MMA issuer (one thread, tcgen05.mma kind::tf32 x3 per k-step into one
// of two 128-column TMEM accumulators), warps 2-5 = epilogue (tcgen05.ld, one thread per row).
// The epilogue keeps, per row, the k smallest d_hat seen so far (sorted, shared memory) and the
// list of every column with d_hat <= thr(current k-th); a column above the threshold costs one
// compare. Since t_split >= t (the split sees a subset), thr(t_split) >= thr(t): the union of
// the splits' lists contains every exact k-nearest column.
// k_probe_finish: warp per row, exact fp64 distances of the union (one candidate per lane, its row
// streamed with 16-B loads), bitonic sort by (dist, column), first k out.
// A row whose list overflowed is finished by an exact scan of all n columns (correct, slow).
#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "dade_internal.h"
#include "exact_batch.cuh"

// DADE_DEBUG_CHECKS builds (tools/build_variant.py; compute-sanitizer is closed on the GPU pool):
// device-side invariants — a violation traps and the next synchronising call reports it
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

namespace dade {

namespace {
constexpr int kTM = 128;
constexpr int kKC = 16;
constexpr int kSub = kTM * kKC;            // floats per (tile, chunk) block
constexpr int kSBO = (kKC / 4) * 128;
constexpr int kStageBytes = 4 * kSub * 4;  // A_hi, A_lo, B_hi, B_lo = 32 KB
constexpr int kStages = 2;
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
#ifndef DADE_MBAR_HINT
#define DADE_MBAR_HINT 0
#endif
// DADE_MBAR_HINT > 0: try_wait with a suspend-time hint (ns), so a waiting warp yields its issue slots
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  if (DADE_MBAR_HINT > 0) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra W%=;\n}" ::"r"(smem_u32(b)),
        "r"(ph), "r"((uint32_t)DADE_MBAR_HINT)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W%=;\n}" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}

#define TMEM_LD32(taddr, r)                                                                          \
  asm volatile(                                                                                      \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),        \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),    \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), \
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), \
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                         \
      : "r"(taddr))

constexpr unsigned kAll = 0x7fffffffu;  // window that accepts every value (signed compare)

// certified window of the filter (gemm_tf32.cu): bits of thr(v), rounded up
__device__ __forceinline__ unsigned win_bits(float v, float slack) {
  const double delta = 9.5367431640625e-07;  // 2^-20
  const double T = ((double)v + (double)slack) * (1.0 + delta) / (1.0 - delta) + (double)slack;
  const float tf = (float)T;
  if (!(tf >= 0.f)) return kAll;
  const unsigned b = __float_as_uint(tf);
  return b >= 0x7f800000u ? kAll : b + 2u;
}

__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// smem: stages | bars | per-row S[k][128] (floats) | Lv[C][128] | Lc[C][128]
__global__ void __launch_bounds__(kThreads, 1) k_probe_tc(
    const float* __restrict__ Ahi, const float* __restrict__ Alo, const float* __restrict__ an,
    const float* __restrict__ Bhi, const float* __restrict__ Blo, const float* __restrict__ bn, int nkc,
    int64_t m, int64_t n, int tiles_per_split, int k, int C, const float* __restrict__ slack,
    int32_t* __restrict__ cand, int32_t* __restrict__ ccount, int passes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* S = reinterpret_cast<float*>(sm + kStages * kStageBytes + 128);
  float* Lv = S + (size_t)k * kTM;
  int32_t* Lc = reinterpret_cast<int32_t*>(Lv + (size_t)C * kTM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tm = blockIdx.x;
  const int64_t ntiles = (n + kTM - 1) / kTM;
  const int64_t t0 = (int64_t)blockIdx.y * tiles_per_split;
  const int64_t rem = ntiles - t0;
  const int nt = rem <= 0 ? 0 : (int)(rem < tiles_per_split ? rem : tiles_per_split);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int it = 0;
      for (int t = 0; t < nt; ++t) {
        const int64_t tn = t0 + t;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % kStages;
          if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
          unsigned char* st = sm + s * kStageBytes;
          mbar_expect_tx(&full[s], passes == 1 ? kStageBytes / 2 : kStageBytes);
          const int64_t ao = (tm * nkc + kc) * kSub, bo = (tn * nkc + kc) * kSub;
          bulk_g2s(st, Ahi + ao, kSub * 4, &full[s]);
          bulk_g2s(st + 2 * kSub * 4, Bhi + bo, kSub * 4, &full[s]);
          if (passes != 1) {  // 3-pass split: the lo parts too
            bulk_g2s(st + kSub * 4, Alo + ao, kSub * 4, &full[s]);
            bulk_g2s(st + 3 * kSub * 4, Blo + bo, kSub * 4, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTM >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
      int it = 0;
      for (int t = 0; t < nt; ++t) {
        const int b = t & 1;
        if (t >= 2) mbar_wait(&tempty[b], ((t >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + b * kTM;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          unsigned char* st = sm + s * kStageBytes;
#pragma unroll
          for (int j = 0; j < kKC / 8; ++j) {
            const uint64_t ah = umma_desc(st + j * 256, 128, kSBO);
            const uint64_t al = umma_desc(st + kSub * 4 + j * 256, 128, kSBO);
            const uint64_t bh = umma_desc(st + 2 * kSub * 4 + j * 256, 128, kSBO);
            const uint64_t bl = umma_desc(st + 3 * kSub * 4 + j * 256, 128, kSBO);
            mma_tf32(acc, ah, bh, idesc, (kc | j) != 0);
            if (passes != 1) {
              mma_tf32(acc, ah, bl, idesc, 1);
              mma_tf32(acc, al, bh, idesc, 1);
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[b]);
      }
    }
  } else {  // ---------------- epilogue: one thread per row
    // Per row: the list L of every column whose d_hat was <= the window bits thr at the time it
    // was seen. L always contains the k smallest d_hat seen (thr >= thr(k-th) >= k-th), so
    // reduce() can recompute the exact k-th smallest from L alone, tighten thr and drop the
    // entries above it. Appends are branch-free (predicated, unrolled); reduce() runs only when
    // L fills up or thr is still open.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;
    const int64_t row = tm * kTM + r;
    const bool live = row < m;
    const float a2 = live ? an[row] : 0.f;
    const float sl = live ? slack[row] : 0.f;
    unsigned thr = kAll;
    int nl = 0;
    bool ovf = false;
    auto reduce = [&]() {
      int ns = 0;
      for (int i = 0; i < nl; ++i) {  // k smallest of L, ascending, into S
        const float v = Lv[i * kTM + r];
        if (ns < k || v < S[(k - 1) * kTM + r]) {
          int pos = ns < k ? ns++ : k - 1;
          while (pos > 0 && S[(pos - 1) * kTM + r] > v) {
            S[pos * kTM + r] = S[(pos - 1) * kTM + r];
            --pos;
          }
          S[pos * kTM + r] = v;
        }
      }
      if (ns < k) return;
      thr = win_bits(S[(k - 1) * kTM + r], sl);
      int j = 0;
      for (int i = 0; i < nl; ++i) {
        const float v = Lv[i * kTM + r];
        if (__float_as_uint(v) <= thr) {
          Lv[j * kTM + r] = v;
          Lc[j * kTM + r] = Lc[i * kTM + r];
          ++j;
        }
      }
      nl = j;
    };
    for (int t = 0; t < nt; ++t) {
      const int b = t & 1;
      mbar_wait(&tfull[b], (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t cb0 = (t0 + t) * kTM;
#pragma unroll 1
      for (int cb = 0; cb < kTM / 32; ++cb) {
        uint32_t v[32];
        TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + b * kTM + cb * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (cb == kTM / 32 - 1) {  // the accumulator may be overwritten from here on
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
        const int64_t c0 = cb0 + cb * 32;
        // d_hat = max(0, fma(-2, acc, a2 + bn)) in packed FP32x2 (same roundings as the scalar
        // form); the max(0, .) is applied on append only: as signed ints, negative d compare
        // below any window, like 0 does
        float d[32];
        unsigned mask = 0;
        const float2* bn2 = reinterpret_cast<const float2*>(bn + c0);  // bn is padded to 128
        const unsigned long long a2p = pk2(a2, a2), m2 = pk2(-2.f, -2.f);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float2 bb = __ldg(bn2 + jj);
          const unsigned long long x = fma2(m2, pk2(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1])),
                                            add2(a2p, pk2(bb.x, bb.y)));
          const float2 xf = *reinterpret_cast<const float2*>(&x);
          d[2 * jj] = xf.x;
          d[2 * jj + 1] = xf.y;
          mask |= (unsigned)((int)__float_as_uint(xf.x) <= (int)thr) << (2 * jj);
          mask |= (unsigned)((int)__float_as_uint(xf.y) <= (int)thr) << (2 * jj + 1);
        }
        {
          const int64_t valid = live ? n - c0 : 0;
          mask &= valid >= 32 ? 0xffffffffu : valid <= 0 ? 0u : ((1u << valid) - 1u);
        }
        // list maintenance is warp-synchronous (every lane reduces when any lane must), so the
        // warp never serialises per-lane slow paths
        if (__any_sync(0xffffffffu, nl + __popc(mask) > C)) {
          reduce();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if ((int)__float_as_uint(d[j]) > (int)thr) mask &= ~(1u << j);
          if (nl + __popc(mask) > C) { ovf = true; mask = 0; }  // k_probe_finish rescans the row
        }
        if (__any_sync(0xffffffffu, mask != 0)) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const bool on = (mask >> j) & 1u;
            if (on) {
              Lv[nl * kTM + r] = fmaxf(0.f, d[j]);
              Lc[nl * kTM + r] = (int32_t)(c0 + j);
            }
            nl += on;
          }
          if (__any_sync(0xffffffffu, nl >= k && (thr == kAll || 2 * nl > C))) reduce();
        }
      }
    }
    if (live) {
      if (nl >= k) reduce();
      const int64_t slot = row * gridDim.y + blockIdx.y;
      for (int i = 0; i < nl; ++i) {  // (column, d_hat bits) pairs
        cand[(slot * C + i) * 2] = Lc[i * kTM + r];
        cand[(slot * C + i) * 2 + 1] = (int32_t)__float_as_uint(Lv[i * kTM + r]);
      }
      ccount[slot] = ovf ? -1 : nl;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// d_hat writer (the filter of the group-minima select, exact.cu): the same warp-specialised
// pipeline as k_probe_tc — TMA warp, MMA warp, two TMEM accumulators, 4 epilogue warps, each CTA
// looping over a range of column tiles so MMA of tile t+1 overlaps the epilogue of tile t — with
// an epilogue that writes d_hat (each warp transposes its 32 x 32 chunk through shared memory
// for row-contiguous stores) and the per-row minima of 2^gshift-column groups. 1-pass: four
// 16 KB stages (hi parts), 3-pass: two 32 KB stages.
__global__ void __launch_bounds__(kThreads, 2) k_dhat_tc(
    const float* __restrict__ Ahi, const float* __restrict__ Alo, const float* __restrict__ an,
    const float* __restrict__ Bhi, const float* __restrict__ Blo, const float* __restrict__ bn, int nkc,
    int64_t m, int64_t n, int tiles_per_split, float* __restrict__ out, int64_t ldo, float* __restrict__ gmin,
    int64_t ldg, int gshift, int passes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int S = passes == 1 ? 4 : 2;
  const int SB = (kStages * kStageBytes) / S;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);
  uint64_t* empty = full + 4;
  uint64_t* tfull = empty + 4;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stg_all = reinterpret_cast<float*>(sm + kStages * kStageBytes + 128);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tm = blockIdx.x;
  const int64_t ntiles = (n + kTM - 1) / kTM;
  const int64_t t0 = (int64_t)blockIdx.y * tiles_per_split;
  const int64_t rem = ntiles - t0;
  const int nt = rem <= 0 ? 0 : (int)(rem < tiles_per_split ? rem : tiles_per_split);
  const int offB = passes == 1 ? kSub * 4 : 2 * kSub * 4;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int it = 0;
      for (int t = 0; t < nt; ++t) {
        const int64_t tn = t0 + t;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % S;
          if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
          unsigned char* st = sm + s * SB;
          mbar_expect_tx(&full[s], SB);
          const int64_t ao = (tm * nkc + kc) * kSub, bo = (tn * nkc + kc) * kSub;
          bulk_g2s(st, Ahi + ao, kSub * 4, &full[s]);
          bulk_g2s(st + offB, Bhi + bo, kSub * 4, &full[s]);
          if (passes != 1) {
            bulk_g2s(st + kSub * 4, Alo + ao, kSub * 4, &full[s]);
            bulk_g2s(st + 3 * kSub * 4, Blo + bo, kSub * 4, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTM >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
      int it = 0;
      for (int t = 0; t < nt; ++t) {
        const int b = t & 1;
        if (t >= 2) mbar_wait(&tempty[b], ((t >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + b * kTM;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          unsigned char* st = sm + s * SB;
#pragma unroll
          for (int j = 0; j < kKC / 8; ++j) {
            const uint64_t ah = umma_desc(st + j * 256, 128, kSBO);
            const uint64_t bh = umma_desc(st + offB + j * 256, 128, kSBO);
            mma_tf32(acc, ah, bh, idesc, (kc | j) != 0);
            if (passes != 1) {
              const uint64_t al = umma_desc(st + kSub * 4 + j * 256, 128, kSBO);
              const uint64_t bl = umma_desc(st + 3 * kSub * 4 + j * 256, 128, kSBO);
              mma_tf32(acc, ah, bl, idesc, 1);
              mma_tf32(acc, al, bh, idesc, 1);
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[b]);
      }
    }
  } else {  // ---------------- epilogue: one thread per row, warp-transposed stores
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int64_t row = tm * kTM + r;
    const float a2 = row < m ? an[row] : 0.f;
    float* stg = stg_all + (warp - 2) * 32 * 33;
    float gmn = INFINITY;
    for (int t = 0; t < nt; ++t) {
      const int b = t & 1;
      mbar_wait(&tfull[b], (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t cb0 = (t0 + t) * kTM;
#pragma unroll 1
      for (int cb = 0; cb < kTM / 32; ++cb) {
        uint32_t v[32];
        TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + b * kTM + cb * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (cb == kTM / 32 - 1) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
        const int64_t c0 = cb0 + cb * 32;
        const bool fullc = c0 + 32 <= n;
        float d[32];
        const float2* bn2 = reinterpret_cast<const float2*>(bn + c0);  // bn is padded to 128
        const unsigned long long a2p = pk2(a2, a2), m2 = pk2(-2.f, -2.f);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float2 bb = __ldg(bn2 + jj);
          const unsigned long long x = fma2(m2, pk2(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1])),
                                            add2(a2p, pk2(bb.x, bb.y)));
          const float2 xf = *reinterpret_cast<const float2*>(&x);
          d[2 * jj] = c0 + 2 * jj < n ? fmaxf(0.f, xf.x) : INFINITY;
          d[2 * jj + 1] = c0 + 2 * jj + 1 < n ? fmaxf(0.f, xf.y) : INFINITY;
        }
        if (gmin && row < m && c0 < n) {
          float mn = d[0];
#pragma unroll
          for (int j = 1; j < 32; ++j) mn = fminf(mn, d[j]);
          if (gshift == 6) {
            if ((cb & 1) == 0) gmn = mn;
            mn = fminf(mn, gmn);
          }
          if (gshift == 5 || (cb & 1) == 1 || c0 + 32 >= n) gmin[row * ldg + (c0 >> gshift)] = mn;
        }
        if (fullc && (ldo & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = d[j];
          __syncwarp();
#pragma unroll
          for (int itr = 0; itr < 8; ++itr) {
            const int ri = itr * 4 + (lane >> 3), cc = (lane & 7) * 4;
            const int64_t grow = tm * kTM + q * 32 + ri;
            if (grow < m) {
              const float* sp = stg + ri * 33 + cc;
              *reinterpret_cast<float4*>(out + grow * ldo + c0 + cc) = make_float4(sp[0], sp[1], sp[2], sp[3]);
            }
          }
          __syncwarp();
        } else if (row < m) {
          float* o = out + row * ldo + c0;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < n) o[j] = d[j];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// k_dhat_tc with the row tile's A operand RESIDENT in shared memory (1-pass, nkc * 8 KB <= 168 KB,
// i.e. D <= 336): the A chunks are fetched once per CTA instead of once per column tile, halving
// the L2 -> SM operand traffic that bounds the wide-row d_hat writer (C5 shard: 128 KB of A and
// 128 KB of B per 128 x 128 tile at D = 256). One CTA per SM (A + a four-stage B ring).
__global__ void __launch_bounds__(kThreads, 1) k_dhat_ares(
    const float* __restrict__ Ahi, const float* __restrict__ an, const float* __restrict__ Bhi,
    const float* __restrict__ bn, int nkc, int64_t m, int64_t n, int tiles_per_split, float* __restrict__ out,
    int64_t ldo, float* __restrict__ gmin, int64_t ldg, int gshift) {
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr int S = 4;
  constexpr int CB = kSub * 4;  // bytes of one (tile, chunk) operand block
  unsigned char* areg = sm;
  unsigned char* ring = sm + (size_t)nkc * CB;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * CB);
  uint64_t* empty = full + 4;
  uint64_t* tfull = empty + 4;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(afull + 1);
  float* stg_all = reinterpret_cast<float*>(ring + S * CB + 128);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tm = blockIdx.x;
  const int64_t ntiles = (n + kTM - 1) / kTM;
  const int64_t t0 = (int64_t)blockIdx.y * tiles_per_split;
  const int64_t rem = ntiles - t0;
  const int nt = rem <= 0 ? 0 : (int)(rem < tiles_per_split ? rem : tiles_per_split);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    mbar_init(afull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0 && nt > 0) {  // ---------------- TMA producer: A once, then the B chunks
      mbar_expect_tx(afull, (uint32_t)nkc * CB);
      for (int kc = 0; kc < nkc; ++kc) bulk_g2s(areg + (size_t)kc * CB, Ahi + (tm * nkc + kc) * kSub, CB, afull);
      int it = 0;
      for (int t = 0; t < nt; ++t) {
        const int64_t tn = t0 + t;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % S;
          if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
          mbar_expect_tx(&full[s], CB);
          bulk_g2s(ring + s * CB, Bhi + (tn * nkc + kc) * kSub, CB, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nt > 0) {  // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTM >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
      mbar_wait(afull, 0);
      int it = 0;
      for (int t = 0; t < nt; ++t) {
        const int b = t & 1;
        if (t >= 2) mbar_wait(&tempty[b], ((t >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + b * kTM;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int j = 0; j < kKC / 8; ++j) {
            const uint64_t ah = umma_desc(areg + (size_t)kc * CB + j * 256, 128, kSBO);
            const uint64_t bh = umma_desc(ring + s * CB + j * 256, 128, kSBO);
            mma_tf32(acc, ah, bh, idesc, (kc | j) != 0);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[b]);
      }
    }
  } else {  // ---------------- epilogue: one thread per row, warp-transposed stores
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int64_t row = tm * kTM + r;
    const float a2 = row < m ? an[row] : 0.f;
    float* stg = stg_all + (warp - 2) * 32 * 33;
    float gmn = INFINITY;
    for (int t = 0; t < nt; ++t) {
      const int b = t & 1;
      mbar_wait(&tfull[b], (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t cb0 = (t0 + t) * kTM;
#pragma unroll 1
      for (int cb = 0; cb < kTM / 32; ++cb) {
        uint32_t v[32];
        TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + b * kTM + cb * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (cb == kTM / 32 - 1) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
        const int64_t c0 = cb0 + cb * 32;
        const bool fullc = c0 + 32 <= n;
        float d[32];
        const float2* bn2 = reinterpret_cast<const float2*>(bn + c0);  // bn is padded to 128
        const unsigned long long a2p = pk2(a2, a2), m2 = pk2(-2.f, -2.f);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float2 bb = __ldg(bn2 + jj);
          const unsigned long long x = fma2(m2, pk2(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1])),
                                            add2(a2p, pk2(bb.x, bb.y)));
          const float2 xf = *reinterpret_cast<const float2*>(&x);
          d[2 * jj] = c0 + 2 * jj < n ? fmaxf(0.f, xf.x) : INFINITY;
          d[2 * jj + 1] = c0 + 2 * jj + 1 < n ? fmaxf(0.f, xf.y) : INFINITY;
        }
        if (gmin && row < m && c0 < n) {
          float mn = d[0];
#pragma unroll
          for (int j = 1; j < 32; ++j) mn = fminf(mn, d[j]);
          if (gshift == 6) {
            if ((cb & 1) == 0) gmn = mn;
            mn = fminf(mn, gmn);
          }
          if (gshift == 5 || (cb & 1) == 1 || c0 + 32 >= n) gmin[row * ldg + (c0 >> gshift)] = mn;
        }
        if (fullc && (ldo & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = d[j];
          __syncwarp();
#pragma unroll
          for (int itr = 0; itr < 8; ++itr) {
            const int ri = itr * 4 + (lane >> 3), cc = (lane & 7) * 4;
            const int64_t grow = tm * kTM + q * 32 + ri;
            if (grow < m) {
              const float* sp = stg + ri * 33 + cc;
              *reinterpret_cast<float4*>(out + grow * ldo + c0 + cc) = make_float4(sp[0], sp[1], sp[2], sp[3]);
            }
          }
          __syncwarp();
        } else if (row < m) {
          float* o = out + row * ldo + c0;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < n) o[j] = d[j];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

__device__ __forceinline__ bool cless(double d0, int32_t c0, double d1, int32_t c1) {
  return d0 < d1 || (d0 == d1 && c0 < c1);
}

constexpr int kFinWarps = 4;
constexpr int kFinCapMax = 512;  // candidates per row held at once (running top-k beyond that)
// per-warp shared memory for a capacity: cd | cc | sel | ucol | udh | hist[256]
__host__ __device__ constexpr size_t fin_warp_bytes(int cap) { return (size_t)cap * (8 + 4 * 4) + 256 * 4; }

// exact distance of one candidate column per lane (c < 0 = none), accumulated sequentially over
// j = 0..D-1 in fp64 (R20). Each lane streams its own candidate row with 16-B loads (the row is
// contiguous), so a lane keeps several loads in flight instead of a chain of dependent gathers.
__device__ __forceinline__ double exact_batch(const float* __restrict__ a, const float* __restrict__ B, int D,
                                              int32_t c, float* /*stage*/, int /*lane*/) {
  double acc = 0.0;
  if (c < 0) return acc;
  const float* b = B + (int64_t)c * D;
  if ((D & 3) == 0) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll 8
    for (int j = 0; j < D / 4; ++j) {
      const float4 y = __ldg(b4 + j), x = __ldg(a4 + j);
      double t = __dsub_rn((double)x.x, (double)y.x);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)x.y, (double)y.y);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)x.z, (double)y.z);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)x.w, (double)y.w);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  } else {
    for (int j = 0; j < D; ++j) {
      const double t = __dsub_rn((double)__ldg(a + j), (double)__ldg(b + j));
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  }
  return acc;
}

__global__ void __launch_bounds__(kFinWarps * 32) k_probe_finish(
    const int32_t* __restrict__ cand, const int32_t* __restrict__ ccount, int nsplit, int C, int64_t m,
    int64_t n, int k, const float* __restrict__ A, const float* __restrict__ B, int D,
    const float* __restrict__ slack, int32_t* __restrict__ out_idx, double* __restrict__ out_d, int kFinCap) {
  extern __shared__ __align__(16) unsigned char fs[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // per-warp region: cd | cc | sel | ucol | udh | hist[256]
  unsigned char* base = fs + (size_t)w * fin_warp_bytes(kFinCap);
  double* cd = reinterpret_cast<double*>(base);
  int32_t* cc = reinterpret_cast<int32_t*>(cd + kFinCap);
  int32_t* sel = cc + kFinCap;
  int32_t* ucol = sel + kFinCap;
  unsigned* udh = reinterpret_cast<unsigned*>(ucol + kFinCap);
  unsigned* hist = udh + kFinCap;
  float* stage = nullptr;  // (exact_batch reads candidate rows directly)
  const int64_t row = (int64_t)blockIdx.x * kFinWarps + w;
  if (row >= m) return;
  const float* a = A + row * (int64_t)D;
  // list counts: lane s holds list s's (nsplit <= 32: one load per lane, all in flight at once),
  // their exclusive prefix places each list in the union
  bool full_scan = false;
  int total = 0, my_c = 0, my_off = 0;
  if (nsplit <= 32) {
    my_c = lane < nsplit ? ccount[row * nsplit + lane] : 0;
    full_scan = __any_sync(0xffffffffu, my_c < 0);
    const int c = my_c < 0 ? 0 : my_c;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    my_off = inc - c;
    total = __shfl_sync(0xffffffffu, inc, 31);
  } else {
    for (int s = 0; s < nsplit; ++s) {
      const int c = ccount[row * nsplit + s];
      full_scan |= c < 0;
      total += c < 0 ? 0 : c;
    }
  }
  for (int i = lane; i < k; i += 32) { cd[i] = DBL_MAX; cc[i] = 0x7fffffff; }
  int cnt = k;
  auto compact = [&]() {
    int P = 1;
    while (P < cnt) P <<= 1;
    for (int i = cnt + lane; i < P; i += 32) { cd[i] = DBL_MAX; cc[i] = 0x7fffffff; }
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = lane; i < P / 2; i += 32) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const double x = cd[lo], y = cd[hi];
          const int32_t xc = cc[lo], yc = cc[hi];
          if (cless(y, yc, x, xc) == up) { cd[lo] = y; cd[hi] = x; cc[lo] = yc; cc[hi] = xc; }
        }
        __syncwarp();
      }
    cnt = k;
  };
  auto add32 = [&](int32_t c) {  // one candidate per lane (c < 0: none)
    if (cnt + 32 > kFinCap) compact();
    const double d = exact_batch(a, B, D, c, stage, lane);
    cd[cnt + lane] = c >= 0 ? d : DBL_MAX;
    cc[cnt + lane] = c >= 0 ? c : 0x7fffffff;
    cnt += 32;
    __syncwarp();
  };
  if (!full_scan && total >= k) {
    // stage the union (column, d_hat bits) in shared memory once; with the counts and offsets in
    // registers the lists' loads do not wait on one another
    if (total > kFinCap) {
      full_scan = true;
    } else if (nsplit <= 32) {
#pragma unroll 4
      for (int s = 0; s < nsplit; ++s) {
        const int nc = __shfl_sync(0xffffffffu, my_c, s), o = __shfl_sync(0xffffffffu, my_off, s);
        const int2* cl = reinterpret_cast<const int2*>(cand + (row * nsplit + s) * (int64_t)C * 2);
        for (int i = lane; i < nc; i += 32) {
          DADE_DCHECK(o + i < kFinCap && nc <= C);
          const int2 e = __ldg(cl + i);
          ucol[o + i] = e.x;
          udh[o + i] = (unsigned)e.y;
        }
      }
    } else {
      int nu = 0;
      for (int s = 0; s < nsplit; ++s) {
        const int nc = ccount[row * nsplit + s];
        const int32_t* cl = cand + (row * nsplit + s) * (int64_t)C * 2;
        for (int i = lane; i < nc; i += 32) {
          ucol[nu + i] = cl[2 * i];
          udh[nu + i] = (unsigned)cl[2 * i + 1];
        }
        nu += nc;
      }
    }
    __syncwarp();
  }
  if (full_scan || total < k) {
    for (int64_t c0 = 0; c0 < n; c0 += 32) add32(c0 + lane < n ? (int32_t)(c0 + lane) : -1);
  } else {
    const int nu = total;
    // E = k-th smallest d_hat of the union (it holds every split's k smallest): radix select
    unsigned prefix = 0;
    int krem = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = lane; i < 256; i += 32) hist[i] = 0;
      __syncwarp();
      for (int i = lane; i < nu; i += 32) {
        const unsigned v = udh[i];
        if (shift == 24 || ((v ^ prefix) >> (shift + 8)) == 0) atomicAdd(&hist[(v >> shift) & 255u], 1u);
      }
      __syncwarp();
      unsigned h[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { h[j] = hist[lane * 8 + j]; tot += h[j]; }
      unsigned inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      unsigned before = inc - tot;
      const bool mine = before < (unsigned)krem && (unsigned)krem <= inc;
      int bin = 0;
      unsigned below = 0;
      if (mine) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (before + h[j] >= (unsigned)krem) { bin = lane * 8 + j; below = before; break; }
          before += h[j];
        }
      }
      const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
      bin = __shfl_sync(0xffffffffu, bin, src);
      below = __shfl_sync(0xffffffffu, below, src);
      prefix |= (unsigned)bin << shift;
      krem -= (int)below;
      __syncwarp();
    }
    const unsigned tb = win_bits(__uint_as_float(prefix), slack[row]);
    // the union's columns inside the global window, ballot-compacted into a list, then exact
    // distances 32 at a time
    int np = 0;
    for (int i0 = 0; i0 < nu; i0 += 32) {
      const int i = i0 + lane;
      const bool in = i < nu && udh[i] <= tb;
      const unsigned bal = __ballot_sync(0xffffffffu, in);
      const int pos = np + __popc(bal & ((1u << lane) - 1));
      if (in) sel[pos] = ucol[i];
      np += __popc(bal);
    }
    __syncwarp();
    if (np > kFinCap) {  // cannot happen for nsplit * C <= kFinCap; stay exact anyway
      for (int64_t c0 = 0; c0 < n; c0 += 32) add32(c0 + lane < n ? (int32_t)(c0 + lane) : -1);
    } else {
      for (int i0 = 0; i0 < np; i0 += 32) add32(i0 + lane < np ? sel[i0 + lane] : -1);
    }
  }
  compact();
  for (int i = lane; i < k; i += 32) {
    const bool ok = cd[i] != DBL_MAX;
    out_idx[row * k + i] = ok ? cc[i] : -1;
    if (out_d) out_d[row * k + i] = ok ? cd[i] : DBL_MAX;
  }
}
}  // namespace

int probe_tc_cap(int k) { return k + 32; }

void launch_dhat_tc(const float* Ahi, const float* Alo, const float* an, int64_t m, const float* Bhi,
                    const float* Blo, const float* bn, int64_t n, int D, float* out, int64_t ldo, float* gmin,
                    int gshift, int passes, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  int dev = 0, sms = 0;  // per call: the index may live on any device
  DADE_CK(cudaGetDevice(&dev));
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = kStages * kStageBytes + 128 + 4 * 32 * 33 * 4;
  DADE_CK(cudaFuncSetAttribute(k_dhat_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  // per launch: per device
  const int64_t mt = (m + kTM - 1) / kTM, ntiles = (n + kTM - 1) / kTM;
  int64_t nsplit = 1;
  while (mt * nsplit < 2 * sms && nsplit * 4 <= ntiles) nsplit *= 2;  // >= 4 tiles per CTA
  const int tps = (int)((ntiles + nsplit - 1) / nsplit);
  dim3 grid((unsigned)mt, (unsigned)((ntiles + tps - 1) / tps));
  k_dhat_tc<<<grid, kThreads, smem, st>>>(Ahi, Alo, an, Bhi, Blo, bn, tc_nkc(D), m, n, tps, out, ldo, gmin,
                                         (n + (1 << gshift) - 1) >> gshift, gshift, passes);
  DADE_CK(cudaGetLastError());
}

// the A-resident writer applies to the 1-pass filter with nkc * 8 KB of A <= 168 KB (D <= 336).
// Off by default (DADE_OPT_DHAT_ARES = 1 enables it): measured on the C5 shard it is SLOWER
// (search 3.03 -> 3.76 ms) — the writer is bound by its epilogue, not by operand traffic, and one
// CTA per SM halves the epilogue warps.
static size_t dhat_ares_smem(int nkc) { return (size_t)nkc * kSub * 4 + 4 * kSub * 4 + 128 + 4 * 32 * 33 * 4; }
bool dhat_ares_ok(int D, int passes) { return passes == 1 && dhat_ares_smem(tc_nkc(D)) <= 220 * 1024; }

void launch_dhat_ares(const float* Ahi, const float* an, int64_t m, const float* Bhi, const float* bn, int64_t n,
                      int D, float* out, int64_t ldo, float* gmin, int gshift, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  int dev = 0, sms = 0;  // per call: the index may live on any device
  DADE_CK(cudaGetDevice(&dev));
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int nkc = tc_nkc(D);
  const size_t smem = dhat_ares_smem(nkc);
  DADE_CK(cudaFuncSetAttribute(k_dhat_ares, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  // per launch: per device
  const int64_t mt = (m + kTM - 1) / kTM, ntiles = (n + kTM - 1) / kTM;
  // one CTA per SM: about three waves of (row tile, column range) CTAs, >= 4 column tiles each
  int64_t nsplit = std::max<int64_t>(1, (3 * (int64_t)sms + mt - 1) / mt);
  nsplit = std::min<int64_t>(nsplit, std::max<int64_t>(1, ntiles / 4));
  const int tps = (int)((ntiles + nsplit - 1) / nsplit);
  dim3 grid((unsigned)mt, (unsigned)((ntiles + tps - 1) / tps));
  k_dhat_ares<<<grid, kThreads, smem, st>>>(Ahi, an, Bhi, bn, nkc, m, n, tps, out, ldo, gmin,
                                            (n + (1 << gshift) - 1) >> gshift, gshift);
  DADE_CK(cudaGetLastError());
}

int probe_tc_splits(int64_t m, int64_t n, int sms) {
  const int64_t mt = (m + kTM - 1) / kTM, nt = (n + kTM - 1) / kTM;
  int64_t s = 1;
  while (mt * s < 2 * sms && s * 2 <= nt / 2) s *= 2;  // >= 2 tiles per split
  return (int)s;
}

void launch_probe_tc(const float* Ahi, const float* Alo, const float* an, int64_t m, const float* Bhi,
                     const float* Blo, const float* bn, int64_t n, int D, int k, const float* slack,
                     const float* A, const float* B, int32_t* cand, int32_t* ccount, int nsplit,
                     int32_t* out_idx, double* out_d64, cudaStream_t st, int passes) {
  if (m <= 0) return;
  const int C = probe_tc_cap(k);
  const size_t smem = kStages * kStageBytes + 128 + (size_t)kTM * (k * 4 + C * 8);
  DADE_REQUIRE(smem <= 227 * 1024, DADE_ERR_UNSUPPORTED, "probe: k too large for the fused filter");
  DADE_CK(cudaFuncSetAttribute(k_probe_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  // per launch: per device
  const int64_t ntiles = (n + kTM - 1) / kTM;
  const int tps = (int)((ntiles + nsplit - 1) / nsplit);
  dim3 grid((unsigned)((m + kTM - 1) / kTM), (unsigned)nsplit);
  k_probe_tc<<<grid, kThreads, smem, st>>>(Ahi, Alo, an, Bhi, Blo, bn, tc_nkc(D), m, n, tps, k, C, slack, cand,
                                          ccount, passes);
  DADE_CK(cudaGetLastError());
  launch_probe_finish(cand, ccount, nsplit, C, m, n, k, A, B, D, slack, out_idx, out_d64, st);
}

void launch_probe_finish(const int32_t* cand, const int32_t* ccount, int nlists, int C, int64_t m, int64_t n, int k,
                         const float* A, const float* B, int D, const float* slack, int32_t* out_idx, double* out_d64,
                         cudaStream_t st) {
  // capacity: the union of the lists (nlists x C) rounded up, so small unions leave room for more
  // resident CTAs (C5 shard: 256 instead of 512 -> 7 CTAs per SM instead of 4 on the gathers)
  // (a power of two: the bitonic compaction sorts up to the next power of two of its count)
  int cap = 64;
  while (cap < kFinCapMax && cap < (int64_t)nlists * C + 32) cap <<= 1;
  const size_t fsm = (size_t)kFinWarps * fin_warp_bytes(cap);
  DADE_CK(cudaFuncSetAttribute(k_probe_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));  // per launch: per device
  k_probe_finish<<<(unsigned)((m + kFinWarps - 1) / kFinWarps), kFinWarps * 32, fsm, st>>>(
      cand, ccount, nlists, C, m, n, k, A, B, D, slack, out_idx, out_d64, cap);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
