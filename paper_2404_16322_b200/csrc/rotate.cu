// Rotation x~ = R(x - mu) (centring P:L305) on the 5th-generation tensor cores,
// stored fp32. Database rows are written straight into the dimension-blocked, list-major layout
// (a1): block b = dims [16b, 16b+16) is an n x 16 fp32 matrix, row p = list-major position p, so
// one Delta_d = 16 step of one IVF list is one contiguous, 64-B-per-row, 128-bit stream.
//
// The contraction (N x D by D x D) runs as tcgen05.mma kind::i8 in split precision, exact in its
// integer part (the Ozaki splitting): each row v of the left operand (v = x - mu, formed in fp64)
// and each row r_i of R is scaled by its own power of two 2^e (max |v| < 2^e) and cut into kS
// signed 7-bit slices, the base-128 digits of T = trunc(v 2^(7 kS - e)) (|T| < 2^(7 kS)):
//   v 2^-e = sum_{s=1..kS} A_s 2^(-7s) + w,   A_s in [-127, 127],   |w| < 2^(-7 kS).
// Then
//   <v, r_i> ~ 2^(e_v + e_i) sum_{L=2..kS+1} 2^(-7L) P_L,   P_L = sum_{s+t=L} A_s . B_t,
// where every P_L is an EXACT int32 sum on the tensor cores (|P_L| <= kS D 127^2 < 2^31 for
// D <= 16,384) in its own TMEM accumulator, and the kS levels are combined in fp64 in the
// epilogue. The dropped cross terms (s + t > kS + 1) and the remainders bound the error of each
// output by 9 D 2^(-7 kS) 2^(e_v + e_i) (kS = 6: ~2^-27 max|v| at D = 960 in the worst case; the
// typical error is ~sqrt(D) times smaller) — below the final fp32 rounding of x~, so the stored
// layout carries the same ~2^-24 relative error as an fp64 rotation (tests/test_gpu_rotate.py).
//
// Level accumulation with one MMA per A slice: R's slices of a 32-dim output tile are stacked
// as one 192-row B operand (row 32 (t-1) + j = slice t of dim j), and the MMA of A_s with the
// first 32 (kS + 1 - s) rows of it is issued at TMEM column offset 32 (s - 1): column block
// L - 2 then receives exactly the pairs s + t = L. kS MMAs per 32-wide K step (N = 192, 160, ...,
// 32) instead of kS (kS + 1) / 2 small ones.
//
// k_rot_slice: 8 rows x 4 16-dim groups per warp pass, so each slice is written as 512
// contiguous bytes of the UMMA canonical K-major layout (one block per (row tile, 64-B K chunk)).
// k_rot_i8: persistent, warp-specialised: warp 0 issues the TMA bulk copies (3 stages of 6 x 8 KB
// of A + 12 KB of B), warp 1 the MMAs, warps 2-9 drain a double-buffered accumulator (2 x 192
// TMEM columns; 16 columns x 6 levels per warp, one tcgen05.ld wait) while the MMAs fill the
// other buffer; int32 -> fp64 by the 2^52 + 2^31 bias and one DADD, scaling by one multiply.
#include <algorithm>
#include <cstdint>

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

namespace dade {

namespace {
constexpr int kS = kRotSlices;            // slices per operand
constexpr int kTM = 128;                  // rows per tile (UMMA M)
constexpr int kTN = 32;                   // output dims per tile
constexpr int kBN = kS * kTN;             // stacked B rows (192)
constexpr int kKB = 64;                   // K bytes (int8 elements) per chunk
constexpr int kABlk = kTM * kKB;          // 8 KB: one slice of one (row tile, chunk)
constexpr int kBBlk = kBN * kKB;          // 12 KB: all slices of one (dim tile, chunk)
constexpr int kStage = kS * kABlk + kBBlk;  // 60 KB
constexpr int kStages = 3;
constexpr int kAccCols = kS * kTN;        // 192 TMEM columns per accumulator buffer
constexpr int kRowChunk = 1 << 20;        // rows sliced per pass (bounds the slice scratch)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major no-swizzle offset of byte kb of row rr inside a (rows x 64 B) block:
// core matrix = 8 rows x 16 B (128 B contiguous), LBO (K direction) = 128 B, SBO (8-row groups) = 512 B
__device__ __forceinline__ int canon_off(int rr, int kb) { return (rr >> 3) * 512 + (kb >> 4) * 128 + (rr & 7) * 16; }

// Slices of rows [0, rows_pad) of one pass. A mode (B = false): row r is input row
// src_rows ? src_rows[p0 + r] : p0 + r of the fp32 X, centred by the fp64 mu; slice s goes to
// block ((r / 128) nkc + kc) kS + s, row r % 128. B mode: row r is R's row r (fp64); slice s goes
// to block (r / 32) nkc + kc, row 32 s + r % 32. Rows >= rows and dims >= D are 0.
// Lane = (row % 8) + 8 (16-dim group % 4): 8 rows x 64 dims per warp pass.
template <typename T, bool B>
__global__ void __launch_bounds__(256) k_rot_slice(const T* __restrict__ X, const int32_t* __restrict__ src_rows,
                                                   int64_t p0, int64_t rows, int64_t rows_pad, int D, int nkc,
                                                   const double* __restrict__ mu, int8_t* __restrict__ out,
                                                   int32_t* __restrict__ expo,
                                                   const unsigned long long* __restrict__ rmax = nullptr,
                                                   int kcpb = 1 << 30) {
  const int lane = threadIdx.x & 31, r8 = lane & 7, g4 = lane >> 3;
  const int64_t r = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 8 + r8;
  if (r - r8 >= rows_pad) return;  // whole warp out of range
  const bool live = r < rows;
  const int64_t src = live ? (src_rows ? (int64_t)src_rows[p0 + r] : p0 + r) : 0;
  const T* xr = X + src * D;
  auto load16 = [&](int k0, double* v) {  // dims [k0, k0 + 16) of the row, centred, 0 outside
    if (!live || k0 >= D) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.0;
      return;
    }
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 f = *reinterpret_cast<const float4*>(xr + k0 + 4 * c);
        v[4 * c] = f.x; v[4 * c + 1] = f.y; v[4 * c + 2] = f.z; v[4 * c + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 f = *reinterpret_cast<const double2*>(xr + k0 + 2 * c);
        v[2 * c] = f.x; v[2 * c + 1] = f.y;
      }
    }
    if (mu) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] -= __ldg(mu + k0 + j);
    }
  };
  // pass 1: max |v| over the row (the 4 lanes of a row split its groups), or the row maxima
  // given (rmax: bit patterns of non-negative doubles; then blockIdx.y picks chunks
  // [kcpb y, kcpb (y + 1)) of a long row, so many CTAs share one row)
  double mx = 0.0;
  if (rmax) {
    mx = live ? __longlong_as_double((long long)rmax[r]) : 0.0;
  } else {
    for (int kc = 0; kc < nkc; ++kc) {
      double v[16];
      load16(kc * kKB + g4 * 16, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) mx = fmax(mx, fabs(v[j]));
    }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  }
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): max |v| < 2^e
  if (blockIdx.y == 0 && g4 == 0 && r < rows_pad) expo[r] = live ? e : 0;
  const int kcb = (int)min((int64_t)blockIdx.y * kcpb, (int64_t)nkc), kce = (int)min((int64_t)kcb + kcpb, (int64_t)nkc);
  // pass 2: digits of T = trunc(v 2^(7 kS - e)), 16 B per (lane, slice)
  const int64_t tile = B ? r / kTN : r / kTM;
  const int rr = (int)(B ? r % kTN : r % kTM);
  for (int kc = kcb; kc < kce; ++kc) {
    double v[16];
    load16(kc * kKB + g4 * 16, v);
    uint32_t pk[kS][4];
#pragma unroll
    for (int s = 0; s < kS; ++s) pk[s][0] = pk[s][1] = pk[s][2] = pk[s][3] = 0u;
    // 2^(7 kS - e) as a bit pattern (|v| 2^(7 kS - e) < 2^(7 kS): the product is exact)
    const int se = min(max(7 * kS - e, -1022), 1023);
    const double sc = __longlong_as_double((long long)(se + 1023) << 52);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const long long t = __double2ll_rz(v[j] * sc);
      const unsigned long long m = (unsigned long long)(t < 0 ? -t : t);
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        int d = (int)((m >> (7 * (kS - 1 - s))) & 127u);
        if (t < 0) d = -d;
        pk[s][j >> 2] |= ((uint32_t)(uint8_t)(int8_t)d) << ((j & 3) * 8);
      }
    }
    if (r >= rows_pad) continue;
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      int8_t* dst = B ? out + (tile * nkc + kc) * (int64_t)kBBlk + canon_off(s * kTN + rr, g4 * 16)
                      : out + ((tile * nkc + kc) * kS + s) * (int64_t)kABlk + canon_off(rr, g4 * 16);
      *reinterpret_cast<uint4*>(dst) = make_uint4(pk[s][0], pk[s][1], pk[s][2], pk[s][3]);
    }
  }
}

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
__device__ __forceinline__ uint64_t umma_desc(const void* smem) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;  // LBO: next core matrix along K
  d |= (uint64_t)(512u >> 4) << 32;  // SBO: next 8-row group
  d |= (uint64_t)1 << 46;            // descriptor version (Blackwell); no swizzle
  return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}

#define ROT_TMEM_LD16(taddr, r)                                                                         \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15])                                                                                   \
               : "r"(taddr))

// Tiles t = m * ntn + n (rows [128 m, +128) of the pass x dims [32 n, +32)), CTA c takes
// t = c, c + grid, ... (consecutive CTAs share an A tile in L2).
__global__ void __launch_bounds__(320, 1) k_rot_i8(const int8_t* __restrict__ As, const int32_t* __restrict__ ea,
                                                   const int8_t* __restrict__ Bs, const int32_t* __restrict__ eb,
                                                   int nkc, int64_t rows, int64_t p0, int64_t n_out, int D,
                                                   float* __restrict__ rm_out, float* __restrict__ blk_out,
                                                   double* __restrict__ acc64, const double* __restrict__ an64 = nullptr,
                                                   const double* __restrict__ bn64 = nullptr,
                                                   float* __restrict__ dist_out = nullptr,
                                                   unsigned* __restrict__ gmin_out = nullptr, int64_t ldg = 0) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStage);
  uint64_t* empty = full + kStages;
  uint64_t* accf = empty + kStages;  // [2] accumulator buffer b ready (MMA commit)
  uint64_t* acce = accf + 2;         // [2] accumulator buffer b drained (256 epilogue threads)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acce + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntn = (D + kTN - 1) / kTN;
  const int64_t ntm = (rows + kTM - 1) / kTM, ntiles = ntm * ntn;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&accf[b], 1); mbar_init(&acce[b], 256); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // 2 x 192 accumulator columns -> 512
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // producer: TMA bulk copies of each tile's K chunks
      int it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t m = t / ntn, n = t % ntn;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % kStages, u = it / kStages;
          if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
          unsigned char* st = sm + s * kStage;
          mbar_expect_tx(&full[s], kStage);
          bulk_g2s(st, As + (m * nkc + kc) * (int64_t)(kS * kABlk), kS * kABlk, &full[s]);
          bulk_g2s(st + kS * kABlk, Bs + (n * nkc + kc) * (int64_t)kBBlk, kBBlk, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, tl = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        const int b = tl & 1, ub = tl >> 1;
        if (ub > 0) mbar_wait(&acce[b], (ub - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc0 = tmem + (uint32_t)(b * kAccCols);
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int s = it % kStages, u = it / kStages;
          mbar_wait(&full[s], u & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const unsigned char* st = sm + s * kStage;
#pragma unroll
          for (int j = 0; j < kKB / 32; ++j) {  // UMMA_K = 32 for 8-bit operands (32 B of K)
            const uint64_t bd = umma_desc(st + kS * kABlk + j * 256);
#pragma unroll
            for (int sa = 0; sa < kS; ++sa) {
              // A slice sa+1 against B slices 1 .. kS - sa (N = 32 (kS - sa)) at column 32 sa:
              // column block L - 2 accumulates the pairs of level L; the sa = 0 MMA of the first
              // K step covers every block and overwrites
              const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((kTN * (kS - sa)) >> 3) << 17) |
                                     ((uint32_t)(kTM >> 4) << 24);
              mma_i8(acc0 + (uint32_t)(sa * kTN), umma_desc(st + sa * kABlk + j * 256), bd, idesc,
                     (kc | j) != 0 || sa != 0);
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accf[b]);
      }
    }
  } else {  // epilogue: warps 2..9; TMEM lane quarter warp % 4, columns 16 h .. 16 h + 15
    const int q = warp & 3, h = (warp - 2) >> 2;
    int tl = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      const int b = tl & 1, ub = tl >> 1;
      const int64_t m = t / ntn;
      const int n = (int)(t % ntn);
      const int64_t r = m * kTM + q * 32 + lane;
      const int e_row = r < rows ? __ldg(ea + r) : 0;
      const int i0 = n * kTN + h * 16;
      const int e_col = i0 + (lane & 15) < D ? __ldg(eb + i0 + (lane & 15)) : 0;
      mbar_wait(&accf[b], ub & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t v[kS][16];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kAccCols + h * 16);
#pragma unroll
      for (int L = 0; L < kS; ++L) ROT_TMEM_LD16(ta + (uint32_t)(L * kTN), v[L]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acce[b]);  // the MMAs may refill this buffer
      float o[16];
      double o64[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // sum_L P_L 2^(-7 (L + 2)), smallest terms first; int32 -> double exactly as
        // (2^52 + 2^31 + P) - (2^52 + 2^31) (one integer op and one DADD)
        double acc = 0.0;
#pragma unroll
        for (int L = kS - 1; L >= 0; --L) {
          const double d = __hiloint2double(0x43300000, (int)(v[L][j] ^ 0x80000000u)) - 4503601774854144.0;
          acc = fma(d, 1.0 / (double)(1ull << (7 * (L + 2))), acc);
        }
        // times 2^(e_row + e_col): one multiply by the power of two (clamped to the normal
        // range: beyond it the fp32 result is 0 or inf either way)
        int E = e_row + __shfl_sync(0xffffffffu, e_col, j);
        E = E < -1022 ? -1022 : (E > 1023 ? 1023 : E);
        o64[j] = acc * __longlong_as_double((long long)(E + 1023) << 52);
        o[j] = (float)o64[j];
      }
      if (r < rows) {
        const int64_t p = p0 + r;
        if (i0 < D) {
          if (rm_out) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(rm_out + p * D + i0 + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
          }
          if (dist_out) {  // distance mode (exact_knn's int8 filter): an + bn - 2 <a, b> in fp64 -> fp32
            DADE_DCHECK(r < rows && (i0 & 15) == 0);
            const double a2 = an64[r];
            float mn = INFINITY;
            float dv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const double dd = a2 + bn64[i0 + j] - 2.0 * o64[j];
              dv[j] = i0 + j < D ? fmaxf(0.f, (float)dd) : INFINITY;
              mn = fminf(mn, dv[j]);
            }
            float* dst = dist_out + p * D + i0;
            if ((D & 3) == 0 && i0 + 16 <= D) {  // (the last tile of a ragged row: scalar stores)
#pragma unroll
              for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(dv[j], dv[j + 1], dv[j + 2], dv[j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (i0 + j < D) dst[j] = dv[j];
            }
            // 32-column group minimum (the other 16 columns are another warp's): values >= 0, so
            // the float bits order as unsigned
            atomicMin(gmin_out + p * ldg + (i0 >> 5), __float_as_uint(mn));
          }
          if (acc64) {  // Gram mode (pca.cu): fp64 sums over the K chunks of successive launches
            double* dst = acc64 + p * D + i0;
#pragma unroll
            for (int j = 0; j < 16; ++j) dst[j] += o64[j];
          }
          if (blk_out) {
            float* dst = blk_out + (((int64_t)(i0 >> 4) * n_out + p) << 4);
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int rot_nkc(int D) { return (D + kKB - 1) / kKB; }
}  // namespace

void rot_prepare(RotOp& op, const double* R, int D, cudaStream_t st) {
  DADE_REQUIRE(D % 16 == 0 && D >= 16 && D <= kRotMaxD, DADE_ERR_UNSUPPORTED,
               "rotation: D must be a multiple of 16, <= 16384");
  const int nkc = rot_nkc(D);
  const int64_t ntn = (D + kTN - 1) / kTN, rp = ntn * kTN;
  op.bs.reserve((size_t)ntn * nkc * kBBlk);
  op.be.reserve((size_t)rp);
  k_rot_slice<double, true><<<(unsigned)((rp + 63) / 64), 256, 0, st>>>(R, nullptr, 0, D, rp, D, nkc, nullptr, op.bs.p,
                                                                         op.be.p);
  DADE_CK(cudaGetLastError());
  op.D = D;
}

void launch_rotate(const RotOp& op, RotWs& ws, const float* X, const int32_t* src_rows, int64_t n_out,
                   const double* mu, float* rowmajor_out, float* blocked_out, cudaStream_t st) {
  if (n_out <= 0) return;
  const int D = op.D;
  DADE_REQUIRE(D > 0, DADE_ERR_STATE, "rotation operand not prepared");
  const int nkc = rot_nkc(D);
  const int64_t chunk = std::min<int64_t>(n_out, kRowChunk);
  const int64_t cpad = (chunk + kTM - 1) / kTM * kTM;
  ws.as.reserve((size_t)cpad * nkc * kKB * kS);
  ws.ae.reserve((size_t)cpad);
  const size_t smem = (size_t)kStages * kStage + 128;
  int dev = 0, sms = 0;
  DADE_CK(cudaGetDevice(&dev));
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // set on every launch: the attribute is per device
  DADE_CK(cudaFuncSetAttribute(k_rot_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntn = (D + kTN - 1) / kTN;
  for (int64_t p0 = 0; p0 < n_out; p0 += chunk) {
    const int64_t rows = std::min<int64_t>(chunk, n_out - p0);
    const int64_t rp = (rows + kTM - 1) / kTM * kTM;
    k_rot_slice<float, false><<<(unsigned)((rp + 63) / 64), 256, 0, st>>>(X, src_rows, p0, rows, rp, D, nkc, mu,
                                                                          ws.as.p, ws.ae.p);
    DADE_CK(cudaGetLastError());
    const int64_t ntiles = rp / kTM * ntn;
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, sms);
    k_rot_i8<<<grid, 320, smem, st>>>(ws.as.p, ws.ae.p, op.bs.p, op.be.p, nkc, rows, p0, n_out, D, rowmajor_out,
                                      blocked_out, nullptr);
    DADE_CK(cudaGetLastError());
  }
}

// fp64 squared norms of the centred rows, sum_j (x_j - mu_j)^2 (warp per row; rows >= n and the
// padding up to rows_pad are 0)
__global__ void k_cnorm64(const float* __restrict__ X, int64_t n, int64_t rows_pad, int D, const double* __restrict__ mu,
                          double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows_pad) return;
  double s = 0.0;
  if (r < n)
    for (int j = lane; j < D; j += 32) {
      const double v = (double)X[r * D + j] - mu[j];
      s += v * v;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

// the int8 filter's error bound per row (rounded up to fp32): |d_hat - d| <= slack + 2^-20 d with
// slack = 2 * 9 D 2^-42 2^(e_a + e_bmax) (the exact split, R36, doubled for -2 <a, b>) plus the
// fp64 arithmetic ((D + 16) 2^-51 (an + bmax): the D-term norm sums and the final combination);
// the fp32 rounding of d_hat is inside the 2^-20 d term
__global__ void k_slack_i8(const double* __restrict__ an, const int32_t* __restrict__ ea, int64_t m,
                           const int* __restrict__ e_bmax, const unsigned long long* __restrict__ bmax_bits, int D,
                           float* __restrict__ slack) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double bmax = __longlong_as_double((long long)*bmax_bits);
  // fp64 part: the sequential norm sums (D terms each) and the final an + bn - 2 o, generously
  const double s = 18.0 * D * ldexp(1.0, ea[i] + *e_bmax - 42) + (D + 16) * 4.440892098500626e-16 * (an[i] + bmax);
  slack[i] = __double2float_ru(s);
}

// the B operand's largest slice exponent and largest centred norm (for the slack), and the fp64
// centre from the fp32 one
__global__ void k_i8_bstats(const int32_t* __restrict__ be, const double* __restrict__ bn, int64_t n,
                            int* __restrict__ emax, unsigned long long* __restrict__ bmax_bits) {
  int e = -1 << 30;
  double b = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    e = max(e, be[i]);
    b = fmax(b, bn[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(emax, e);
    atomicMax(bmax_bits, (unsigned long long)__double_as_longlong(b));
  }
}
__global__ void k_f2d(const float* __restrict__ a, double* __restrict__ b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (double)a[i];
}

void launch_cnorm64(const float* X, int64_t n, int64_t rows_pad, int D, const double* mu, double* out,
                    cudaStream_t st) {
  if (rows_pad <= 0) return;
  k_cnorm64<<<(unsigned)((rows_pad + 7) / 8), 256, 0, st>>>(X, n, rows_pad, D, mu, out);
  DADE_CK(cudaGetLastError());
}

void launch_slack_i8(const double* an, const int32_t* ea, int64_t m, const int* e_bmax,
                     const unsigned long long* bmax_bits, int D, float* slack, cudaStream_t st) {
  if (m <= 0) return;
  k_slack_i8<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(an, ea, m, e_bmax, bmax_bits, D, slack);
  DADE_CK(cudaGetLastError());
}

void launch_i8_bprep(const float* B, int64_t n, int D, const float* center, double* mu64, RotOp& ob, double* bn64,
                     int* emax, unsigned long long* bmax_bits, cudaStream_t st) {
  k_f2d<<<(D + 255) / 256, 256, 0, st>>>(center, mu64, D);
  DADE_CK(cudaGetLastError());
  prepare_i8_b(B, n, D, mu64, ob, st);
  const int64_t rp = (n + kTN - 1) / kTN * kTN;
  launch_cnorm64(B, n, rp, D, mu64, bn64, st);
  DADE_CK(cudaMemsetAsync(emax, 0x80, sizeof(int), st));  // 0x80808080: a very negative int
  DADE_CK(cudaMemsetAsync(bmax_bits, 0, sizeof(unsigned long long), st));
  k_i8_bstats<<<(unsigned)std::min<int64_t>((n + 255) / 256, 592), 256, 0, st>>>(ob.be.p, bn64, n, emax, bmax_bits);
  DADE_CK(cudaGetLastError());
}

// Filter distances on the int8 tensor cores (exact_knn, wide rows): d[p][i] = fp32(an[p] + bn[i] -
// 2 <a_p, b_i>) for centred A (rows p, the queries) and B (rows i, the centroids), both sliced by
// k_rot_slice with the same fp64 centre; the dot product carries the exact-split error bound
// 9 D 2^-42 2^(e_a + e_b) (R36), the rest is fp64 arithmetic and one fp32 rounding, so the
// certified window of the selection is ~k wide. gmin[p][g] = the minimum of columns [32 g, 32 g +
// 32) (as float bits; the caller fills it with 0x7f7f7f7f first).
void prepare_i8_b(const float* B, int64_t n, int D, const double* mu, RotOp& ob, cudaStream_t st) {
  const int nkc = rot_nkc(D);
  const int64_t ntn = (n + kTN - 1) / kTN, rp = ntn * kTN;
  ob.bs.reserve((size_t)ntn * nkc * kBBlk);
  ob.be.reserve((size_t)rp);
  k_rot_slice<float, true><<<(unsigned)((rp + 63) / 64), 256, 0, st>>>(B, nullptr, 0, n, rp, D, nkc, mu, ob.bs.p,
                                                                        ob.be.p);
  DADE_CK(cudaGetLastError());
  ob.D = D;
}

void launch_dist_i8(const float* A, int64_t m, int D, const double* mu, const double* an64, RotWs& wa,
                    const RotOp& ob, const double* bn64, int64_t n, float* dist, unsigned* gmin, int64_t ldg,
                    cudaStream_t st) {
  if (m <= 0) return;
  const int nkc = rot_nkc(D);
  const int64_t rp = (m + kTM - 1) / kTM * kTM;
  wa.as.reserve((size_t)rp * nkc * kKB * kS);
  wa.ae.reserve((size_t)rp);
  k_rot_slice<float, false><<<(unsigned)((rp + 63) / 64), 256, 0, st>>>(A, nullptr, 0, m, rp, D, nkc, mu, wa.as.p,
                                                                         wa.ae.p);
  DADE_CK(cudaGetLastError());
  const size_t smem = (size_t)kStages * kStage + 128;
  int dev = 0, sms = 0;
  DADE_CK(cudaGetDevice(&dev));
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DADE_CK(cudaFuncSetAttribute(k_rot_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntn = (n + kTN - 1) / kTN, ntiles = rp / kTM * ntn;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, sms);
  // "D" of the kernel = output width (n columns); K = nkc chunks of the D dims
  k_rot_i8<<<grid, 320, smem, st>>>(wa.as.p, wa.ae.p, ob.bs.p, ob.be.p, nkc, m, 0, m, (int)n, nullptr, nullptr,
                                    nullptr, an64, bn64, dist, gmin, ldg);
  DADE_CK(cudaGetLastError());
}

// Gram matrix on the int8 tensor cores (the PCA covariance, pca.cu): acc[a][b] += sum_k Y[a][k]
// Y[b][k] for the rows x K fp64 matrix Y (K a multiple of 64, <= 16,384 so every level sum stays
// an exact int32; rmax[a] = bits of max_k |Y[a][k]|). Y's rows are both operands: the A slices (per-row scale, 128-row tiles) and the
// B slices (32-row tiles) of the same digits, so the result is exactly symmetric; the error of each
// entry is bounded like the rotation's (R36): 9 K 2^-42 2^(e_a + e_b) with max_k |Y[a][k]| < 2^e_a.
void launch_gram_i8(const double* Y, int rows, int64_t K, const unsigned long long* rmax, RotWs& wa, RotOp& wb,
                    double* acc, cudaStream_t st) {
  DADE_REQUIRE(K % kKB == 0 && K > 0 && K <= kRotMaxD && rows % 16 == 0, DADE_ERR_UNSUPPORTED,
               "gram: K must be a positive multiple of 64, <= 16384, rows a multiple of 16");
  const int nkc = (int)(K / kKB);
  const int64_t rpa = (rows + kTM - 1) / kTM * kTM, ntn = (rows + kTN - 1) / kTN, rpb = ntn * kTN;
  wa.as.reserve((size_t)rpa * nkc * kKB * kS);
  wa.ae.reserve((size_t)rpa);
  wb.bs.reserve((size_t)ntn * nkc * kBBlk);
  wb.be.reserve((size_t)rpb);
  // long rows, few of them: CTAs split each row into 8-chunk (512-K) pieces; the row maxima come
  // from the gather (rmax), so the A and B digits use the same exponents
  constexpr int kcpb = 8;
  const unsigned gy = (unsigned)((nkc + kcpb - 1) / kcpb);
  k_rot_slice<double, false><<<dim3((unsigned)((rpa + 63) / 64), gy), 256, 0, st>>>(
      Y, nullptr, 0, rows, rpa, (int)K, nkc, nullptr, wa.as.p, wa.ae.p, rmax, kcpb);
  DADE_CK(cudaGetLastError());
  k_rot_slice<double, true><<<dim3((unsigned)((rpb + 63) / 64), gy), 256, 0, st>>>(
      Y, nullptr, 0, rows, rpb, (int)K, nkc, nullptr, wb.bs.p, wb.be.p, rmax, kcpb);
  DADE_CK(cudaGetLastError());
  const size_t smem = (size_t)kStages * kStage + 128;
  int dev = 0, sms = 0;
  DADE_CK(cudaGetDevice(&dev));
  DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DADE_CK(cudaFuncSetAttribute(k_rot_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntiles = rpa / kTM * ntn;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, sms);
  k_rot_i8<<<grid, 320, smem, st>>>(wa.as.p, wa.ae.p, wb.bs.p, wb.be.p, nkc, rows, 0, rows, rows, nullptr, nullptr,
                                    acc);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
