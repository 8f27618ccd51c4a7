// a5 probe, round 3 design: the certified tensor-core filter FUSED with the candidate selection
// (no m x n d_hat matrix), built for throughput on sm_100a.
//
// Definition (R20): the k nearest columns of every row under the EXACT fp64 sequential
// sum of squared differences, ordered by (dist, column). As in probe_tc.cu, a filter value
// d_hat = max(0, fl(fl(||a'||^2 + ||b'||^2) - 2 <a', b'>~)) with a rigorous per-row error bound
// (slack) selects, per row, every column inside the certified window thr(t) of the k-th smallest
// d_hat t; k_probe_finish re-ranks that union in fp64.
//
// Operands (a' = fl(x - c), both centred on the B operand's mean c):
//  * KIND 1 (fp16, tcgen05.mma kind::f16): a' scaled by a power of two and rounded to fp16
//    (cvt.rn). The row scale s_a = 2^(14 - E) with ||a'||_inf < 2^E keeps |a' s_a| < 2^14 (no
//    overflow); B takes one matrix scale from its largest centred norm. fp16 keeps an 11-bit
//    significand like tf32 (relative rounding 2^-11 for normal values), so the 1-pass tf32 bound
//    applies, plus the absolute error of values that land in fp16's subnormal range,
//    |eta| <= 2^-25 / s per element (k_slack_h16). Twice the tensor rate of tf32 and half the
//    operand bytes.
//  * KIND 0 (tf32, kind::tf32): the hi parts of the tf32 split (gemm_tf32.cu), 1 pass.
// Both use the same 8 KB (128-row tile, 64-B K chunk) blocks in the UMMA K-major no-swizzle
// layout, so the pipeline is identical: chunk = 32 halves or 16 floats.
//
// k_probe_fz: CTA = one 128-row tile of A x a contiguous range of 128-column tiles of B.
//  warp 0    : TMA producer — the A tile once (resident in shared memory), then B chunks into an
//              S-stage ring (cp.async.bulk + mbarrier complete_tx);
//  warp 1    : MMA issuer (one thread) into 2G TMEM accumulators of 128 columns;
//  warps 2.. : G epilogue groups of 4 warps (one thread per row, the TMEM lane quarter of the
//              warp); group g takes the tiles t = g (mod G).
// Epilogue per 32-column chunk: u_j = fl(m2 acc_j + ||b_j||^2) (packed FFMA2) and its minimum
// (3-input FMNMX); if no lane's minimum can be inside its window (u_min > thr_u, a conservative
// image of the window on u, see win_u) the chunk costs ~45 instructions per thread. Otherwise
// the exact d_hat values go through the list logic of probe_tc.cu (per row: every column with
// d_hat <= the window of the k-th smallest seen so far; the window only tightens).
// Outputs per (row, split, group): the list (column, d_hat bits); k_probe_finish takes the union.
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <algorithm>

#include <cuda_fp16.h>
#include <cstdio>

#include "dade_internal.h"

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

#ifndef DADE_FZ_BN_TMA
#define DADE_FZ_BN_TMA 0
#endif

namespace dade {

namespace {
constexpr int kTM = 128;
constexpr int kChunkBytes = 8192;          // one (128-row tile, 64-B K chunk) operand block
constexpr int kKH = 32;                    // fp16 elements per chunk row
constexpr int kSBO = 512;                  // bytes between 8-row core-matrix groups
constexpr unsigned kAll = 0x7fffffffu;     // window accepting every value (signed compare)

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
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(smem_u32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ uint64_t umma_desc(const void* smem) {  // K-major, no swizzle
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFFu);
  d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;          // LBO: K-adjacent core matrices
  d |= (uint64_t)(((uint32_t)kSBO >> 4) & 0x3FFFu) << 32;  // SBO: 8-row groups
  d |= (uint64_t)1 << 46;
  return d;
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
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
#define FZ_TMEM_LD32(taddr, r)                                                                       \
  asm volatile(                                                                                      \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),        \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),    \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), \
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), \
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                         \
      : "r"(taddr))

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
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// certified window of the filter (gemm_tf32.cu, probe_tc.cu): bits of thr(v), rounded up
__device__ __forceinline__ unsigned win_bits(float v, float slack) {
  const double delta = 9.5367431640625e-07;  // 2^-20
  const double T = ((double)v + (double)slack) * (1.0 + delta) / (1.0 - delta) + (double)slack;
  const float tf = (float)T;
  if (!(tf >= 0.f)) return kAll;
  const unsigned b = __float_as_uint(tf);
  return b >= 0x7f800000u ? kAll : b + 2u;
}

// The window's image on u = fl(x + bn), x = m2 acc exact (m2 a power of two), for the skip test.
// d_hat = fl(x + s), s = fl(a2 + bn), a2, bn >= 0, |x| <= 2.02 (a2 + bmax) (Cauchy-Schwarz plus
// the filter error). If d_hat <= T (T >= 0; negative d_hat pass every window) then
//   x + s <= T (1 + 2^-23),  x + bn <= T (1 + 2^-23) - a2 + (a2 + bn) 2^-24,
//   u <= x + bn + |x + bn| 2^-24 <= T + T 2^-23 - a2 + (a2 + bmax) 2^-22,
// so u > T_u = T - a2 + (T + a2 + bmax) 2^-20 (rounded up) proves d_hat > T for every column.
__device__ __forceinline__ float win_u(unsigned thr, float a2, float bmax) {
  if (thr >= kAll) return INFINITY;
  const double T = (double)__uint_as_float(thr);
  const double tu = T - (double)a2 + (T + (double)a2 + (double)bmax) * 9.5367431640625e-07;
  return __double2float_ru(tu);
}

// Work split: the (row tile, column tile) pairs in row-major order are cut into gridDim.x equal
// contiguous ranges, one per persistent CTA (perfect balance to one tile). A CTA's range covers
// one or two (rarely more) row tiles: each stretch of one row tile is a SEGMENT — A is reloaded
// between segments, and the per-row lists persist over a segment and are written out at its end
// (both epilogue groups' lists merged first). Output list slot of (row, CTA c): row * maxL +
// (c - the first CTA of the row's tile); unused slots keep the count 0 the host set.
__device__ __forceinline__ int64_t fz_cta_of(int64_t i, int64_t I, int64_t P) { return ((i + 1) * P - 1) / I; }

// Two passes over the same MMA pipeline (identical operands and instruction sequence, so the
// filter values are bit-identical):
//  MODE 1 (seed): per row and segment, the k smallest 32-column group minima of d_hat (registers,
//    a branch-free insertion network of KS slots) -> seeds[(row, segment, group)][k].
//  MODE 2 (select): per row, U = the k-th smallest of the union of its seeds — at least k distinct
//    columns have d_hat <= U, so U >= the k-th smallest d_hat and every list may start with the
//    window thr(U) instead of an open window. The lists then see only the few columns inside the
//    window (no warm-up of a running threshold per list).
// smem: A region | B ring | barriers | Sk[G][128][k] | stage[4G][32 x 33]
template <int KIND, int MODE, int KS, int RP, int CS>
__global__ void __launch_bounds__(64 + 128 * (CS == 2 ? 4 : 2), 1) k_probe_fz(
    const unsigned char* __restrict__ Aop, const float* __restrict__ an, const float* __restrict__ ahs,
    const unsigned char* __restrict__ Bop, const float* __restrict__ bn, float bhs, float bmax, int nkc,
    int64_t m, int64_t n, int maxL, int k, int C, int G, int S, int cpc, const float* __restrict__ slack,
    float* __restrict__ seeds, int32_t* __restrict__ cand, int32_t* __restrict__ ccount, int cstride,
    int nlists_seed) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* areg = sm;
  unsigned char* ring = sm + (size_t)RP * nkc * kChunkBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * cpc * kChunkBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 4;
  uint64_t* afull = tempty + 4;
  uint64_t* afree = afull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(afree + 1);
  // ||b||^2 of the columns of tile T at bnbuf[T mod 2NB]: the slot is rewritten only for tile
  // T + 2NB, whose accumulator buffer the epilogue frees after finishing tile T + NB
  float* bnbuf = reinterpret_cast<float*>(ring + (size_t)S * cpc * kChunkBytes + 16 * S + 256);  // [8][128]
  float* lists = bnbuf + 8 * kTM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NB = 2 * G;
  // this launch's column tiles: every cstride-th of the row (MODE 1 may sample a subset: its
  // seeds stay valid upper bounds), ntiles of them per row tile
  // RP = 2: a row tile is a pair of 128-row A tiles (both resident) sharing every B chunk — two
  // MMAs per chunk into two accumulators, one epilogue group per half — so each B byte brought
  // into the SM feeds twice the tensor work (the B stream is the pipeline's bound)
  const int64_t mt = (m + kTM * RP - 1) / (kTM * RP), ntiles = ((n + kTM - 1) / kTM + cstride - 1) / cstride;
  const int64_t I = mt * ntiles, P = gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * I / P, i1 = ((int64_t)blockIdx.x + 1) * I / P;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    // tfull: the accumulator's commit + the MMA thread's expect_tx for the tile's column norms
    for (int b = 0; b < NB; ++b) { mbar_init(&tfull[b], DADE_FZ_BN_TMA ? 2 : 1); mbar_init(&tempty[b], 4 * RP * CS); }
    mbar_init(afull, 1);
    mbar_init(afree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    const uint32_t ncols = 128u * NB * RP;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: per segment the A tile, then B chunks
      int it = 0, seg = 0;
      for (int64_t i = i0; i < i1; ++seg) {
        const int64_t rt = i / ntiles, iend = min(i1, (rt + 1) * ntiles);
        if (seg > 0) mbar_wait(afree, (seg - 1) & 1);  // every MMA of the last segment completed
        mbar_expect_tx(afull, (uint32_t)(RP * nkc) * kChunkBytes);
        for (int kc = 0; kc < RP * nkc; ++kc)  // RP consecutive 128-row tiles (padded to RP * 128 rows)
          bulk_g2s(areg + (size_t)kc * kChunkBytes, Aop + (size_t)(rt * RP * nkc + kc) * kChunkBytes, kChunkBytes, afull);
        for (; i < iend; ++i) {
          const int64_t tn = (i - rt * ntiles) * cstride;
          for (int kc = 0; kc < nkc; kc += cpc, ++it) {  // one copy per stage of cpc chunks
            const int s = it % S;
            if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
            if (MODE == 3 && blockIdx.x == 0 && it < 512) reinterpret_cast<unsigned long long*>(seeds)[it] = clock64();
            mbar_expect_tx(&full[s], (uint32_t)cpc * kChunkBytes);
            bulk_g2s(ring + (size_t)s * cpc * kChunkBytes, Bop + (size_t)(tn * nkc + kc) * kChunkBytes,
                     (uint32_t)cpc * kChunkBytes, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      // kind::f16: a/b format F16 (0); kind::tf32: TF32 (2); F32 accumulate, K-major, M = N = 128
      const uint32_t fmt = KIND == 1 ? 0u : 2u;
      const uint32_t idesc =
          (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(kTM >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
      int it = 0, seg = 0;
      int64_t T = 0;  // tiles issued by this CTA (accumulator buffer = T % NB)
      unsigned long long* dbg = reinterpret_cast<unsigned long long*>(seeds);  // MODE 3 timeline (CTA 0)
      for (int64_t i = i0; i < i1; ++seg) {
        const int64_t rt = i / ntiles, iend = min(i1, (rt + 1) * ntiles);
        mbar_wait(afull, seg & 1);
        for (; i < iend; ++i, ++T) {
          const int b = (int)(T % NB);
          if (T >= NB) mbar_wait(&tempty[b], (uint32_t)((T / NB) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          // the tile's column norms into bnbuf[T mod 2NB] (last read for tile T - 2NB, finished before
          // the epilogue released tile T - NB's buffer), completing on tfull[b] with the accumulator
          if (DADE_FZ_BN_TMA) {
            mbar_expect_tx(&tfull[b], kTM * 4);
            bulk_g2s(bnbuf + (T % (2 * NB)) * kTM, bn + (i - rt * ntiles) * cstride * kTM, kTM * 4, &tfull[b]);
          }
          if (MODE == 3 && blockIdx.x == 0 && T < 256) dbg[1024 + T] = clock64();
          const uint32_t acc = tmem + b * RP * kTM;
          for (int kc = 0; kc < nkc; kc += cpc, ++it) {
            const int s = it % S;
            mbar_wait(&full[s], (it / S) & 1);
            if (MODE == 3 && blockIdx.x == 0 && it < 512) dbg[512 + it] = clock64();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int c = 0; c < cpc; ++c)
#pragma unroll
              for (int j = 0; j < 2; ++j)  // two MMAs of K = 32 B per row (16 halves / 8 floats)
#pragma unroll
                for (int h = 0; h < RP; ++h)  // one per resident A tile, the same B chunk
                  if (MODE != 3)  // (MODE 3: pipeline measurement without the MMAs)
                    mma<KIND>(acc + h * kTM, umma_desc(areg + (size_t)(h * nkc + kc + c) * kChunkBytes + j * 256),
                              umma_desc(ring + ((size_t)s * cpc + c) * kChunkBytes + j * 256), idesc,
                              ((kc + c) | j) != 0);
            mma_commit(&empty[s]);
          }
          mma_commit(&tfull[b]);
        }
        mma_commit(afree);  // arrives when every MMA of the segment (all readers of A) completed
      }
    }
  } else {  // ---------------- epilogue
    // epilogue group eg = (g RP + h) CS + cs: tile group g (tiles T = g mod G), A half h, column
    // share cs (CS = 2: two groups drain each accumulator, 64 columns each, with their own
    // per-row windows and lists — every list / seed set is a valid partial, the finish and the
    // select pass take their union over Gt = G CS slots per (row, segment))
    const int eg = (warp - 2) >> 2;
    const int cs = eg % CS, h = (eg / CS) % RP, g = eg / (CS * RP);
    const int Gt = G * CS, gt = g * CS + cs;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;
    float* Sk = lists + (size_t)eg * kTM * k;  // [128][k] sorted k smallest d_hat seen (MODE 2)
    float* stage = lists + (size_t)G * RP * CS * kTM * k + (size_t)(warp - 2) * 32 * 33;
    const unsigned lt = (1u << lane) - 1u;
    int64_t T = 0;
    for (int64_t i = i0; i < i1;) {
      const int64_t rt = i / ntiles, iend = min(i1, (rt + 1) * ntiles);
      const int64_t rbase = (rt * RP + h) * kTM;  // first row of this group's A tile
      const int64_t row = rbase + r;
      const bool live = row < m;
      const int jseg = (int)(blockIdx.x - fz_cta_of(rt * ntiles, I, P));
      const float a2 = live ? an[row] : 0.f;
      const float sl = live ? slack[row] : 0.f;
      const float m2 = KIND == 1 ? (live ? -2.f * ahs[row] * bhs : -2.f) : -2.f;  // powers of two: exact
      const unsigned long long m2p = pk2(m2, m2), a2p = pk2(a2, a2);
      float kb[KS];  // MODE 1: the k smallest group minima (ascending); MODE 2: seed union
#pragma unroll
      for (int j = 0; j < KS; ++j) kb[j] = INFINITY;
      bool ovf = !(sl <= FLT_MAX);  // an unbounded filter error: k_probe_finish scans the row exactly
      unsigned thr = kAll;
      float thr_u = INFINITY;
      int nl = 0;
      if (MODE == 2) {
        if (live && !ovf) {  // U = the k-th smallest of the union of the row's seeds
          for (int l = 0; l < nlists_seed; ++l)
            for (int e = 0; e < k; ++e) {
              float x = seeds[((size_t)row * nlists_seed + l) * k + e];
#pragma unroll
              for (int j = 0; j < KS; ++j) {
                const float lo = fminf(kb[j], x);
                x = fmaxf(kb[j], x);
                kb[j] = lo;
              }
            }
          float U = INFINITY;
#pragma unroll
          for (int j = 0; j < KS; ++j)
            if (j == k - 1) U = kb[j];
          thr = win_bits(U, sl);
          thr_u = win_u(thr, a2, bmax);
        }
        if (ovf) thr_u = -INFINITY;
        for (int e = lane; e < 32 * k; e += 32) Sk[(size_t)q * 32 * k + e] = INFINITY;
        __syncwarp();
      }
      for (; i < iend; ++i, ++T) {
        if ((int)(T % G) != g) continue;  // tile T belongs to group T mod G
        const int b = (int)(T % NB);
        mbar_wait(&tfull[b], (uint32_t)(T / NB) & 1);
        if (MODE == 3 && blockIdx.x == 0 && T < 256 && lane == 0 && q == 2) reinterpret_cast<unsigned long long*>(seeds)[1536 + T] = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int64_t cb0 = (i - rt * ntiles) * cstride * kTM;
        // this tile's column norms: read by the epilogue straight from global memory (L2/L1-resident,
        // broadcast loads). DADE_FZ_BN_TMA = 1 (measurement builds): staged by a TMA copy the MMA
        // thread issues when it starts the tile — its latency then sits on every tile's critical path
        const float* bns = DADE_FZ_BN_TMA ? bnbuf + (size_t)(T % (2 * NB)) * kTM : bn + cb0;
        // per 32-column chunk (v: the chunk's accumulators of this thread's row)
        auto chunk = [&](const uint32_t* v, int cb) {
          float4 bq[8];  // the chunk's column norms (broadcast shared-memory loads)
#pragma unroll
          for (int j = 0; j < 8; ++j) bq[j] = reinterpret_cast<const float4*>(bns + cb * 32)[j];
          const float bnl = bns[cb * 32 + lane];
          const int64_t c0 = cb0 + cb * 32;
          if (MODE == 1) {
            // d_hat = fl(m2 acc + fl(a2 + bn)) (packed), invalid columns excluded, group minimum
            float u[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 f = bq[j];
              const unsigned long long x0 = fma2(m2p, pk2(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1])),
                                                 add2(a2p, pk2(f.x, f.y)));
              const unsigned long long x1 = fma2(m2p, pk2(__uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])),
                                                 add2(a2p, pk2(f.z, f.w)));
              u[4 * j] = __uint_as_float((unsigned)x0);
              u[4 * j + 1] = __uint_as_float((unsigned)(x0 >> 32));
              u[4 * j + 2] = __uint_as_float((unsigned)x1);
              u[4 * j + 3] = __uint_as_float((unsigned)(x1 >> 32));
            }
            if (c0 + 32 > n) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j >= n) u[j] = INFINITY;
            }
            float w[12];
#pragma unroll
            for (int j = 0; j < 10; ++j) w[j] = fmin3(u[3 * j], u[3 * j + 1], u[3 * j + 2]);
            w[10] = u[30];
            w[11] = u[31];
            float x = fmaxf(0.f, fminf(fmin3(fmin3(w[0], w[1], w[2]), fmin3(w[3], w[4], w[5]), fmin3(w[6], w[7], w[8])),
                                       fmin3(w[9], w[10], w[11])));
#pragma unroll
            for (int j = 0; j < KS; ++j) {
              const float lo = fminf(kb[j], x);
              x = fmaxf(kb[j], x);
              kb[j] = lo;
            }
            return;
          }
          // ---- MODE 2: skip test on u = fl(m2 acc + bn), the window's image thr_u
          float u[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 f = bq[j];
            const unsigned long long x0 =
                fma2(m2p, pk2(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1])), pk2(f.x, f.y));
            const unsigned long long x1 =
                fma2(m2p, pk2(__uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])), pk2(f.z, f.w));
            u[4 * j] = __uint_as_float((unsigned)x0);
            u[4 * j + 1] = __uint_as_float((unsigned)(x0 >> 32));
            u[4 * j + 2] = __uint_as_float((unsigned)x1);
            u[4 * j + 3] = __uint_as_float((unsigned)(x1 >> 32));
          }
          float w[12];
#pragma unroll
          for (int j = 0; j < 10; ++j) w[j] = fmin3(u[3 * j], u[3 * j + 1], u[3 * j + 2]);
          w[10] = u[30];
          w[11] = u[31];
          const float umin = fminf(fmin3(fmin3(w[0], w[1], w[2]), fmin3(w[3], w[4], w[5]), fmin3(w[6], w[7], w[8])),
                                   fmin3(w[9], w[10], w[11]));
          unsigned nm = __ballot_sync(0xffffffffu, live && umin <= thr_u);
          if (!nm) return;
          // ---- slow path: stage the chunk (column j of row w at stage[j * 33 + w]); the rows that
          // may hold a window column, one at a time, one column per lane
#pragma unroll
          for (int j = 0; j < 32; ++j) stage[j * 33 + lane] = __uint_as_float(v[j]);
          __syncwarp();
          const bool colok = c0 + lane < n;
          while (nm) {
            const int rr = __ffs(nm) - 1;
            nm &= nm - 1;
            const float a2r = __shfl_sync(0xffffffffu, a2, rr);
            const float m2r = __shfl_sync(0xffffffffu, m2, rr);
            const unsigned thrr = __shfl_sync(0xffffffffu, thr, rr);
            // the filter value of (row rr, column lane): the same roundings as the packed form
            const float d = __fmaf_rn(m2r, stage[lane * 33 + rr], __fadd_rn(a2r, bnl));
            const bool hit = colok && (int)__float_as_uint(d) <= (int)thrr;
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (!hm) continue;
            const int R = q * 32 + rr;
            const float dc = fmaxf(0.f, d);
            // 1. hits below the row's k-th smallest seen join Sk (sorted; lane i holds Sk[i],
            //    Sk[32 + i]); the window tightens to thr(min(U, k-th))
            float s0 = lane < k ? Sk[(size_t)R * k + lane] : INFINITY;
            float s1 = lane + 32 < k ? Sk[(size_t)R * k + 32 + lane] : INFINITY;
            const float kth0 = __shfl_sync(0xffffffffu, k > 32 ? s1 : s0, (k - 1) & 31);
            unsigned thr2 = thrr;
            const unsigned im0 = __ballot_sync(0xffffffffu, hit && dc < kth0);
            if (im0) {
              for (unsigned hh = im0; hh; hh &= hh - 1) {
                const float h = __shfl_sync(0xffffffffu, dc, __ffs(hh) - 1);
                const int pos = __popc(__ballot_sync(0xffffffffu, s0 <= h)) +
                                (k > 32 ? __popc(__ballot_sync(0xffffffffu, s1 <= h)) : 0);
                const float up0 = __shfl_up_sync(0xffffffffu, s0, 1);
                const float up1 = __shfl_up_sync(0xffffffffu, s1, 1);
                const float top0 = __shfl_sync(0xffffffffu, s0, 31);
                if (pos < k) {
                  const float n0 = lane < pos ? s0 : (lane == pos ? h : up0);
                  const float n1 = lane + 32 < pos ? s1 : (lane + 32 == pos ? h : (lane == 0 ? top0 : up1));
                  s0 = lane < k ? n0 : INFINITY;  // slots beyond k stay empty (they take part in the ballots)
                  s1 = lane + 32 < k ? n1 : INFINITY;
                }
              }
              if (lane < k) Sk[(size_t)R * k + lane] = s0;
              if (lane + 32 < k) Sk[(size_t)R * k + 32 + lane] = s1;
              const float kth = __shfl_sync(0xffffffffu, k > 32 ? s1 : s0, (k - 1) & 31);
              thr2 = min(thrr, win_bits(kth, __shfl_sync(0xffffffffu, sl, rr)));
            }
            // 2. the hits inside the (tightened) window join the row's list in global memory,
            //    compacted to the window when full
            const bool in = hit && (int)__float_as_uint(d) <= (int)thr2;
            const unsigned im = __ballot_sync(0xffffffffu, in);
            const int ni = __popc(im);
            int2* L = reinterpret_cast<int2*>(cand) + (((rbase + R) * maxL + jseg) * Gt + gt) * C;
            int nlr = __shfl_sync(0xffffffffu, nl, rr);
            bool over = false;
            if (nlr + ni > C) {
              int nn = 0;
              for (int e0 = 0; e0 < nlr; e0 += 32) {
                const int e = e0 + lane;
                const int2 x = e < nlr ? L[e] : make_int2(0, 0);
                const bool keep = e < nlr && (unsigned)x.y <= thr2;
                const unsigned km = __ballot_sync(0xffffffffu, keep);
                if (keep) L[nn + __popc(km & lt)] = x;
                nn += __popc(km);
                __syncwarp();
              }
              nlr = nn;
              over = nlr + ni > C;  // > C near-ties inside the window: k_probe_finish rescans the row
            }
            if (!over) {
              DADE_DCHECK(nlr + ni <= C && jseg >= 0 && jseg < maxL && c0 + lane < ((n + kTM - 1) / kTM) * kTM);
              if (in) L[nlr + __popc(im & lt)] = make_int2((int32_t)(c0 + lane), (int32_t)__float_as_uint(dc));
              nlr += ni;
            }
            if (lane == rr) {
              nl = nlr;
              if (thr2 != thr) {
                thr = thr2;
                thr_u = win_u(thr2, a2, bmax);
              }
              if (over) { ovf = true; thr_u = -INFINITY; }
            }
          }
          __syncwarp();  // the stage is rewritten by the next chunk
        };
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (b * RP + h) * kTM;
        if (MODE == 0 || MODE == 3) {  // pipeline measurement: drain the accumulator only
          uint32_t v0[32];
          FZ_TMEM_LD32(tbase, v0);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
          if (v0[0] == 0x7fc00001u && v0[1] == 0x7fc00001u) nl = -1;  // keep the load
          continue;
        }
        // one chunk at a time (measured faster than batching the TMEM loads: fewer live registers);
        // the buffer is released after the last chunk's load, its column norms stay in bnbuf
#pragma unroll 1
        for (int cb = cs * (4 / CS); cb < (cs + 1) * (4 / CS); ++cb) {
          uint32_t v[32];
          FZ_TMEM_LD32(tbase + cb * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (cb == (cs + 1) * (4 / CS) - 1) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
          }
          chunk(v, cb);
        }
      }
      // ---- segment end
      const int64_t slot = ((int64_t)row * maxL + jseg) * Gt + gt;
      if (MODE == 1) {
        if (live) {
          DADE_DCHECK(jseg >= 0 && jseg < maxL);
#pragma unroll
          for (int j = 0; j < KS; ++j)
            if (j < k) seeds[slot * k + j] = kb[j];
        }
      } else {
        // compact every row's list to its final window (the finish takes the union of <= maxL G
        // lists per row), then publish the count
        for (int rr = 0; rr < 32; ++rr) {
          const int nlr = __shfl_sync(0xffffffffu, nl, rr);
          const unsigned thrr = __shfl_sync(0xffffffffu, thr, rr);
          const int64_t rowr = rbase + q * 32 + rr;
          if (rowr >= m || nlr == 0) continue;
          int2* L = reinterpret_cast<int2*>(cand) + ((rowr * maxL + jseg) * Gt + gt) * C;
          int nn = 0;
          for (int e0 = 0; e0 < nlr; e0 += 32) {
            const int e = e0 + lane;
            const int2 x = e < nlr ? L[e] : make_int2(0, 0);
            const bool keep = e < nlr && (unsigned)x.y <= thrr;
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            if (keep) L[nn + __popc(km & lt)] = x;
            nn += __popc(km);
            __syncwarp();
          }
          if (lane == rr) nl = nn;
        }
        if (live) ccount[slot] = ovf ? -1 : nl;
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (MODE == 3 && blockIdx.x == 0 && tid == 0) {  // timeline summary of CTA 0 (measurement build)
    const unsigned long long* dbg = reinterpret_cast<const unsigned long long*>(seeds);
    const int64_t nch64 = (i1 - i0) * (nkc / cpc), nti64 = i1 - i0;
    const int nch = (int)(nch64 < 512 ? nch64 : 512), nti = (int)(nti64 < 256 ? nti64 : 256);
    double lat = 0, gap = 0, reuse = 0;
    for (int it = S; it < nch; ++it) {
      lat += (double)(dbg[512 + it] - dbg[it]);
      gap += (double)(dbg[it] - dbg[it - 1]);
      reuse += (double)(dbg[it] - dbg[512 + it - S]);
    }
    double tl = 0, tg = 0;
    for (int t = 1; t < nti; ++t) {
      tl += (double)(dbg[1536 + t] - dbg[1024 + t]);
      tg += (double)(dbg[1536 + t] - dbg[1536 + t - 1]);
    }
    printf("fz-timeline cpc=%d S=%d nkc=%d chunks=%d: issue->full %.0f cyc, issue gap %.0f, slot full->reissue %.0f; "
           "tiles=%d: mma-start->epi-tfull %.0f, epi tile gap %.0f\n",
           cpc, S, nkc, nch, lat / (nch - S), gap / (nch - S), reuse / (nch - S), nti, tl / (nti - 1), tg / (nti - 1));
  }
  if (warp == 1) {
    const uint32_t ncols = 128u * NB * RP;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
  }
}

// fp16 operand rows: one warp per row. a' = fl(x - c) (the tf32 split's centring), scaled by a
// power of two and rounded to fp16 (cvt.rn) into the K-major no-swizzle layout (32 halves per
// row per chunk). gscale > 0: that matrix scale for every row; else the row scale
// s = 2^(14 - E), ||a'||_inf < 2^E, clamped to [2^-60, 2^60] (the row is marked unbounded,
// inv_scale = +inf, if the clamp would let |a' s| reach 2^15). norm (nullable): fp64 ||a'||^2
// rounded to fp32, as k_split_tf32 writes it. Padding rows / columns are zeros.
__global__ void k_split_h16(const float* __restrict__ X, int64_t rows, int D, int nkc, const float* __restrict__ center,
                            __half* __restrict__ h, float* __restrict__ norm, float* __restrict__ inv_scale,
                            int64_t rows_pad, float gscale) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows_pad) return;
  const int Dp = nkc * kKH;
  float mx = 0.f;
  double s2 = 0.0;
  if (r < rows)
    for (int j = lane; j < D; j += 32) {
      const float x = center ? X[r * D + j] - center[j] : X[r * D + j];
      mx = fmaxf(mx, fabsf(x));
      s2 += (double)x * (double)x;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  float sc = gscale;
  bool bad = false;
  if (!(gscale > 0.f)) {
    int e = 0;
    if (mx > 0.f) {
      int E;
      frexpf(mx, &E);  // mx = f 2^E, f in [0.5, 1): mx < 2^E
      e = 14 - E;
      if (e < -60) { e = -60; bad = mx * 0x1p-60f >= 32768.f; }
      if (e > 60) e = 60;
    }
    sc = ldexpf(1.f, e);
  }
  const int64_t tile = r / kTM;
  const int rr = (int)(r % kTM);
  for (int j = lane; j < Dp; j += 32) {
    const float x = (r < rows && j < D) ? (center ? X[r * D + j] - center[j] : X[r * D + j]) : 0.f;
    const int kc = j / kKH, kk = j % kKH;
    const int64_t t = (tile * nkc + kc) * (kChunkBytes / 2) + (rr >> 3) * (kSBO / 2) + (kk >> 3) * 64 + (rr & 7) * 8 + (kk & 7);
    h[t] = __float2half_rn(x * sc);  // x * sc: exact (power of two, no overflow / underflow for valid scales)
  }
  if (lane == 0) {
    if (norm) norm[r] = (float)s2;
    if (inv_scale) inv_scale[r] = bad ? INFINITY : 1.f / sc;
  }
}

// Slack of the fp16 filter: the 1-pass bound of gemm_tf32.cu (gamma (||a'||^2 + bmax) + the
// centring term) plus fp16's subnormal range: |eta| <= 2^-25 / s per element gives
// |<a,b>~ - <a,b>| += 2^-25 (||b||_1 / s_a + ||a||_1 / s_b) + Dp 2^-50 / (s_a s_b), with
// ||v||_1 <= sqrt(Dp) ||v||_2; x2 for d_hat and x2 margin.
__global__ void k_slack_h16(const float* __restrict__ an, const float* __restrict__ ainv, int64_t m, float bmax,
                            float binv, float gamma, int Dp, float* __restrict__ slack) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double u = 5.9604644775390625e-08, delta = 9.5367431640625e-07;  // 2^-24, 2^-20
  const double a2 = an[i], ia = ainv[i];
  const double eps = u * 1.0001 * (sqrt(a2) + sqrt((double)bmax));
  double s = (double)gamma * (a2 + (double)bmax) + eps * eps * (1.0 + 1.0 / delta);
  s += 1.1920928955078125e-07 * sqrt((double)Dp) * (sqrt((double)bmax) * 1.0001 * ia + sqrt(a2) * 1.0001 * (double)binv);
  s += 3.552713678800501e-15 * (double)Dp * ia * (double)binv;  // 2^-48
  slack[i] = (isinf(ia) || !(s < 3.0e38)) ? INFINITY : (float)(s * (1.0 + 1e-6));
}
}  // namespace

// list capacity per (row, segment, group) in global scratch: the window's columns (typically ~k
// + a few) plus room for hits between compactions
int fz_cap(int k) { return k + 48; }

int fz_nkc(int D, int kind) { return kind == 1 ? (D + kKH - 1) / kKH : tc_nkc(D); }

size_t fz_smem(int D, int kind, int k, int G, int S, int cpc, int RP, int CS) {
  return (size_t)RP * fz_nkc(D, kind) * kChunkBytes + (size_t)S * cpc * kChunkBytes + 16 * S + 256 + 8 * kTM * 4 +
         (size_t)G * RP * CS * kTM * k * 4 +
         (size_t)G * RP * CS * 4 * 32 * 33 * 4;
}

// fp16 operand rows are padded to 256 (a whole row-tile pair for RP = 2)
int64_t fz_rows_pad(int64_t rows) { return (rows + 2 * kTM - 1) / (2 * kTM) * (2 * kTM); }

// Launch shape: two persistent CTAs per SM with one epilogue group each (TMEM 2 x 256 columns,
// <= 113 KB of shared memory each, >= 3 ring stages) when they fit — the pipeline is latency-
// bound per CTA and two independent CTAs measured 1.5x faster on the C5 shard probe — else one
// CTA with two groups (>= 6 stages), else one group (>= 4). k <= 32 (the seed pass keeps the k
// smallest group minima in registers).
bool fz_config(int D, int kind, int k, int* G, int* S, int* cps, int* RP) {
  if (k > 32) return false;
  *RP = 1;
  for (int s = 8; s >= 3; --s)
    if (2 * fz_smem(D, kind, k, 1, s, 1, 1) <= 226 * 1024) { *G = 1; *S = s; *cps = 2; return true; }
  const size_t cap = 225 * 1024;
  for (int g = 2; g >= 1; --g) {
    int s = 12;
    while (s >= (g == 2 ? 6 : 4) && fz_smem(D, kind, k, g, s, 1, 1) > cap) --s;
    if (s >= (g == 2 ? 6 : 4)) { *G = g; *S = s; *cps = 1; return true; }
  }
  return false;
}

// lists per row of the persistent split: CTAs covering one row tile (host mirror of fz_cta_of)
int fz_lists_per_row(int64_t m, int64_t n, int P, int cstride, int RP) {
  const int64_t mt = (m + kTM * RP - 1) / (kTM * RP), ntiles = ((n + kTM - 1) / kTM + cstride - 1) / cstride, I = mt * ntiles;
  int mx = 1;
  for (int64_t rt = 0; rt < mt; ++rt) {
    const int64_t c0 = ((rt * ntiles + 1) * P - 1) / I, c1 = (((rt + 1) * ntiles) * P - 1) / I;
    mx = std::max<int>(mx, (int)(c1 - c0 + 1));
  }
  return mx;
}

void launch_split_h16(const float* X, int64_t rows, int D, const float* center, uint16_t* h, float* norm,
                      float* inv_scale, float gscale, cudaStream_t st) {
  const int64_t rp = fz_rows_pad(rows);
  if (rp == 0) return;
  k_split_h16<<<(unsigned)((rp + 7) / 8), 256, 0, st>>>(X, rows, D, fz_nkc(D, 1), center,
                                                        reinterpret_cast<__half*>(h), norm, inv_scale, rp, gscale);
  DADE_CK(cudaGetLastError());
}

void launch_slack_h16(const float* an, const float* ainv, int64_t m, float bmax, float binv, int D, float* slack,
                      cudaStream_t st) {
  if (m <= 0) return;
  k_slack_h16<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(an, ainv, m, bmax, binv, tc_gamma(D, 1),
                                                           fz_nkc(D, 1) * kKH, slack);
  DADE_CK(cudaGetLastError());
}

template <int KIND, int MODE, int KS, int RP, int CS>
static void fz_launch(int P, unsigned threads, size_t smem, cudaStream_t st, const void* Aop, const float* an,
                      const float* ainv, const void* Bop, const float* bn, float binv, float bmax, int nkc, int64_t m,
                      int64_t n, int maxL, int k, int C, int G, int S, int cpc, const float* slack, float* seeds,
                      int32_t* cand, int32_t* ccount, int cstride = 1, int nlists_seed = 0) {
  DADE_CK(cudaFuncSetAttribute(k_probe_fz<KIND, MODE, KS, RP, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_probe_fz<KIND, MODE, KS, RP, CS><<<P, threads, smem, st>>>(static_cast<const unsigned char*>(Aop), an, ainv,
                                                       static_cast<const unsigned char*>(Bop), bn, binv, bmax, nkc, m,
                                                       n, maxL, k, C, G, S, cpc, slack, seeds, cand, ccount, cstride,
                                                       nlists_seed);
  DADE_CK(cudaGetLastError());
}

int g_fz_debug = 0;  // measurement: 1 = pipeline without epilogue math, 2 = pipeline without MMAs

template <int KIND, int KS, int RP, int CS>
static void fz_two_pass(int P, unsigned threads, size_t smem, cudaStream_t st, const void* Aop, const float* an,
                        const float* ainv, const void* Bop, const float* bn, float binv, float bmax, int nkc,
                        int64_t m, int64_t n, int maxL, int k, int C, int G, int S, int cpc, const float* slack,
                        float* seeds, int32_t* cand, int32_t* ccount, int cstride, int maxL1, int P1) {
  if (g_fz_debug) {
    if (g_fz_debug == 1)
      fz_launch<KIND, 0, KS, RP, CS>(P, threads, smem, st, Aop, an, ainv, Bop, bn, binv, bmax, nkc, m, n, maxL, k, C, G, S,
                             cpc, slack, seeds, cand, ccount, 1, 0);
    else
      fz_launch<KIND, 3, KS, RP, CS>(P, threads, smem, st, Aop, an, ainv, Bop, bn, binv, bmax, nkc, m, n, maxL, k, C, G, S,
                             cpc, slack, seeds, cand, ccount, 1, 0);
  }
  // seed pass over every cstride-th column tile (its own persistent split: P1 CTAs, maxL1 lists
  // per row), then the select pass over all columns, reading maxL1 G seed lists per row
  fz_launch<KIND, 1, KS, RP, CS>(P1, threads, smem, st, Aop, an, ainv, Bop, bn, binv, bmax, nkc, m, n, maxL1, k, C, G, S, cpc,
                         slack, seeds, cand, ccount, cstride, 0);
  fz_launch<KIND, 2, KS, RP, CS>(P, threads, smem, st, Aop, an, ainv, Bop, bn, binv, bmax, nkc, m, n, maxL, k, C, G, S, cpc,
                         slack, seeds, cand, ccount, 1, maxL1 * G * CS);
}

// The seed pass samples every cstride-th column tile so that >= 64 k group minima remain (their
// k-th smallest is still an upper bound of the row's k-th smallest d_hat; the select pass then
// starts from a somewhat wider window): on the C5 shard (512 column tiles, k = 8) one tile in 4.
// Measured there (tools/exp_probe_fz.py): probe 1.207 / 1.006 / 1.154 / 1.353 ms at strides
// 1 / 4 / 8 / 16 — sparser seeds cost the select pass more than they save. Its persistent split
// has P1 CTAs and maxL1 seed lists per row.
void fz_seed_plan(int64_t m, int64_t n, int k, int P, int force, int* cstride, int* P1, int* maxL1, int RP) {
  const int64_t mt = (m + kTM * RP - 1) / (kTM * RP), ntiles = (n + kTM - 1) / kTM;
  int64_t cs = force > 0 ? force : std::max<int64_t>(1, std::min<int64_t>(16, ntiles / (16 * (int64_t)k)));
  *cstride = (int)cs;
  const int64_t nts = (ntiles + cs - 1) / cs;
  *P1 = (int)std::min<int64_t>(P, mt * nts);
  *maxL1 = fz_lists_per_row(m, n, *P1, (int)cs, RP);
}

void launch_probe_fz(int kind, const void* Aop, const float* an, const float* ainv, int64_t m, const void* Bop,
                     const float* bn, float binv, float bmax, int64_t n, int D, int k, const float* slack,
                     const float* A, const float* B, float* seeds, int32_t* cand, int32_t* ccount, int P, int maxL,
                     int G, int S, int cpc, int cstride, int P1, int maxL1, int32_t* out_idx, double* out_d64,
                     cudaStream_t st, int RP, int CS) {
  if (m <= 0) return;
  DADE_REQUIRE(k >= 1 && k <= 32, DADE_ERR_UNSUPPORTED, "probe: fused filter needs k <= 32");
  const int C = fz_cap(k);
  DADE_REQUIRE(RP == 1 || (RP == 2 && kind == 1 && G == 1), DADE_ERR_ARG, "fz: row-tile pairs need fp16 operands and one group");
  DADE_REQUIRE((CS == 1 || (CS == 2 && kind == 1)) && G * RP * CS <= 4, DADE_ERR_ARG, "fz: column shares need fp16 operands, <= 4 groups");
  const size_t smem = fz_smem(D, kind, k, G, S, cpc, RP, CS);
  DADE_REQUIRE(cpc >= 1 && fz_nkc(D, kind) % cpc == 0, DADE_ERR_ARG, "fz: chunks per copy must divide the chunks per tile");
  DADE_REQUIRE(smem <= 227 * 1024, DADE_ERR_UNSUPPORTED, "probe: operands too wide for the fused filter");
  // seeds of rows / segments a CTA never covers stay huge (0x7f7f7f7f = 3.4e38: never below U)
  DADE_CK(cudaMemsetAsync(seeds, 0x7f, sizeof(float) * (size_t)m * maxL1 * G * CS * k, st));
  DADE_CK(cudaMemsetAsync(ccount, 0, sizeof(int32_t) * (size_t)m * maxL * G * CS, st));
  const unsigned threads = 64 + 128 * G * RP * CS;
  const int nkc = fz_nkc(D, kind);
  const float bi = kind == 1 ? binv : 1.f;
#define FZ_ARGS P, threads, smem, st, Aop, an, ainv, Bop, bn, bi, bmax, nkc, m, n, maxL, k, C, G, S, cpc, slack, seeds, cand, ccount, \
                cstride, maxL1, P1
  if (kind == 1 && RP == 2 && CS == 2) {
    if (k <= 8) fz_two_pass<1, 8, 2, 2>(FZ_ARGS);
    else if (k <= 16) fz_two_pass<1, 16, 2, 2>(FZ_ARGS);
    else fz_two_pass<1, 32, 2, 2>(FZ_ARGS);
  } else if (kind == 1 && RP == 2) {
    if (k <= 8) fz_two_pass<1, 8, 2, 1>(FZ_ARGS);
    else if (k <= 16) fz_two_pass<1, 16, 2, 1>(FZ_ARGS);
    else fz_two_pass<1, 32, 2, 1>(FZ_ARGS);
  } else if (kind == 1 && CS == 2) {
    if (k <= 8) fz_two_pass<1, 8, 1, 2>(FZ_ARGS);
    else if (k <= 16) fz_two_pass<1, 16, 1, 2>(FZ_ARGS);
    else fz_two_pass<1, 32, 1, 2>(FZ_ARGS);
  } else if (kind == 1) {
    if (k <= 8) fz_two_pass<1, 8, 1, 1>(FZ_ARGS);
    else if (k <= 16) fz_two_pass<1, 16, 1, 1>(FZ_ARGS);
    else fz_two_pass<1, 32, 1, 1>(FZ_ARGS);
  } else {
    if (k <= 8) fz_two_pass<0, 8, 1, 1>(FZ_ARGS);
    else if (k <= 16) fz_two_pass<0, 16, 1, 1>(FZ_ARGS);
    else fz_two_pass<0, 32, 1, 1>(FZ_ARGS);
  }
#undef FZ_ARGS
  launch_probe_finish(cand, ccount, maxL * G * CS, C, m, n, k, A, B, D, slack, out_idx, out_d64, st);
}

}  // namespace dade
