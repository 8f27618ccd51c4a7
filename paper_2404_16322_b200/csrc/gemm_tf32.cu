// Tensor-core distance tiles for the exact IVF probe / assignment / KNN filter (a2, a5, K12).
//
//   d_hat(q, c) = max(0, ||q||^2 + ||c||^2 - 2 <q, c>)
//
// <q, c> runs on the 5th-generation tensor cores (tcgen05.mma kind::tf32, accumulators in TMEM)
// in 3-pass split precision: x = x_hi + x_lo with x_hi = tf32(x), x_lo = tf32(x - x_hi), and
// <q,c> ~ q_hi.c_hi + q_hi.c_lo + q_lo.c_hi (FP32-accurate to ~2^-21). Operand tiles are
// pre-split into the UMMA canonical K-major no-swizzle layout in global memory, so each
// (128-row tile, 32-wide K chunk) is one contiguous 16 KB block fetched by a TMA bulk copy
// (cp.async.bulk + mbarrier). One elected thread issues TMA and MMA; tcgen05.commit releases
// stages; 4 warps drain TMEM with tcgen05.ld in the epilogue.
//
// Both operands are CENTRED on a common fp32 vector c (the mean of the B operand) before the
// split: a' = fl(x - c). Distances are translation invariant, and centring shrinks the norms
// that scale the error bound (GIST-like data in [0,1]: ~30x), which keeps the certified window
// small. The result is only a FILTER, with a rigorous bound (e = a' - (x - c), |e_j| <= u|x_j - c_j|):
//   |d_hat - d| <= S + delta d + eps^2 (1 + 1/delta),   u = 2^-24, delta = 2^-20,
//   S   = gamma (||a'||^2 + max ||b'||^2),  gamma = 2 (3 Dp + 16) 2^-23  (split error 3 2^-22
//         |a_j b_j| per term, fp32 accumulation of 3 Dp terms, norm and final roundings, x2),
//   eps = u (||x - c|| + max ||y - c||)  (centring: |d' - d| <= 2 sqrt(d) eps + eps^2 and
//         2 sqrt(d) eps <= delta d + eps^2 / delta).
// slack(row) = S + eps^2 (1 + 1/delta); the exact answer is then decided in fp64 over every
// column with d_hat <= (t + slack)(1 + delta)/(1 - delta) + slack, t = the k-th smallest d_hat
// (exact.cu), which provably contains the true k nearest, so tensor-core rounding never reaches
// the output (R20).
#include <algorithm>
#include <cstdint>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr int kTM = 128;               // rows per operand tile (M and N tiles)
constexpr int kKC = 16;                // K elements per chunk (64 B per row)
constexpr int kSub = kTM * kKC;        // floats per (tile, chunk) block = 8 KB
constexpr int kSBO = (kKC / 4) * 128;  // bytes between 8-row core-matrix groups
constexpr int kStageBytes = 4 * kSub * 4;  // A_hi, A_lo, B_hi, B_lo

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// canonical K-major, no swizzle: core matrix = 8 rows x 16 B; LBO (K direction) = 128 B,
// SBO (8-row groups) = kSBO bytes inside a 128 x kKC block
__device__ __forceinline__ int64_t tiled_index(int64_t r, int k, int nkc) {
  const int64_t tile = r / kTM;
  const int rr = (int)(r % kTM), kc = k / kKC, kk = k % kKC;
  return (tile * nkc + kc) * kSub + (rr >> 3) * (kSBO / 4) + (kk >> 2) * 32 + (rr & 7) * 4 + (kk & 3);
}

__global__ void k_split_tf32(const float* __restrict__ X, int64_t rows, int D, int nkc,
                             const float* __restrict__ center, float* __restrict__ hi,
                             float* __restrict__ lo, float* __restrict__ norm, int64_t rows_pad) {
  // one warp per row: split into (hi, lo) in the tiled layout, fp64 squared norm -> fp32
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows_pad) return;
  const int Dp = nkc * kKC;
  double s = 0.0;
  for (int k = lane; k < Dp; k += 32) {
    const float x = (r < rows && k < D) ? (center ? X[r * D + k] - center[k] : X[r * D + k]) : 0.f;
    const float h = tf32_rna(x);
    const float l = tf32_rna(x - h);
    const int64_t t = tiled_index(r, k, nkc);
    hi[t] = h;
    lo[t] = l;
    s += (double)x * (double)x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) norm[r] = (float)s;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
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
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  // base_offset = 0, lbo_mode = 0, layout_type = 0 (SWIZZLE_NONE)
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
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
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

// One CTA = one 128 x (128 NT) output tile; K = nkc chunks of 32, 2-stage TMA -> MMA pipeline.
// NT = 2 (1-pass filters): the A tile feeds an N = 256 MMA over two adjacent column tiles (their
// B blocks are contiguous 8-row groups in the stage), eight epilogue warps — a quarter less
// operand traffic per output and half the CTAs (their barrier / TMEM set-up and operand wait).
template <int NT>
__global__ void __launch_bounds__(128 * NT, NT == 1 ? 3 : 2) k_l2_tc(const float* __restrict__ Ahi, const float* __restrict__ Alo,
                                                  const float* __restrict__ an, const float* __restrict__ Bhi,
                                                  const float* __restrict__ Blo, const float* __restrict__ bn,
                                                  int nkc, float* __restrict__ out, int64_t m, int64_t n,
                                                  int64_t ldo, float* __restrict__ gmin, int64_t ldg, int passes,
                                                  int gshift, int s1, const float* __restrict__ ahs, float bhs, int coop) {
  extern __shared__ __align__(1024) unsigned char sm[];
  // operand stages: 2 x 32 KB (3-pass: A_hi, A_lo, B_hi, B_lo) or s1 x 16 KB (1-pass: A_hi, B_hi)
  const int S = passes == 1 ? s1 : 2;
  const int SB = passes == 1 ? (1 + NT) * kSub * 4 : kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * SB);
  uint64_t* empty = full + 4;
  uint64_t* accf = full + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(full + 9);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tm = blockIdx.y, tn = (int64_t)blockIdx.x * NT;  // tn: first 128-column tile
  const int64_t ntn = (n + kTM - 1) / kTM;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (coop) {
    // cooperative operand load (1-pass, every K chunk resident: S = nkc stages): all threads copy
    // the tile's A and B blocks (already in the UMMA layout) with 16-byte cp.async — the LSU path
    // instead of cp.async.bulk; the generic-proxy writes are fenced for the tensor core's reads
    for (int kc = 0; kc < nkc; ++kc) {
      unsigned char* st = sm + kc * SB;
      const char* ga = reinterpret_cast<const char*>(Ahi + (tm * nkc + kc) * kSub);
      const char* gb = reinterpret_cast<const char*>(Bhi + (tn * nkc + kc) * kSub);
      for (int i = tid; i < kSub * 4 / 16; i += 128 * NT) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(st + i * 16)), "l"(ga + i * 16) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(st + kSub * 4 + i * 16)), "l"(gb + i * 16)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(128u * NT)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (coop) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (tid == 0) {
    // instruction descriptor: D=F32, A=B=TF32, K-major both, N=128, M=128
    // (ahs != null: fp16 operands — the same 8-KB blocks hold 32 halves per row, kind::f16,
    // A/B format F16 (0); 1-pass only)
    const uint32_t fmt = ahs ? 0u : 2u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)((kTM * NT) >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
    // stage layout: A_hi | B_hi (1-pass) or A_hi | A_lo | B_hi | B_lo (3-pass)
    const int offB = passes == 1 ? kSub * 4 : 2 * kSub * 4;
    auto load = [&](int kc) {
      const int s = kc % S;
      unsigned char* st = sm + s * SB;
      mbar_expect_tx(&full[s], SB);
      const int64_t ao = (tm * nkc + kc) * kSub, bo = (tn * nkc + kc) * kSub;
      bulk_g2s(st, Ahi + ao, kSub * 4, &full[s]);
      bulk_g2s(st + offB, Bhi + bo, kSub * 4, &full[s]);
      if (NT == 2)  // the second column tile (past the last one: the last tile again, masked in the epilogue)
        bulk_g2s(st + offB + kSub * 4, Bhi + ((tn + 1 < ntn ? tn + 1 : ntn - 1) * nkc + kc) * kSub, kSub * 4, &full[s]);
      if (passes != 1) {
        bulk_g2s(st + kSub * 4, Alo + ao, kSub * 4, &full[s]);
        bulk_g2s(st + 3 * kSub * 4, Blo + bo, kSub * 4, &full[s]);
      }
    };
    if (!coop)
      for (int kc = 0; kc < S && kc < nkc; ++kc) load(kc);
    for (int kc = 0; kc < nkc; ++kc) {
      const int s = kc % S;
      if (!coop) mbar_wait(&full[s], (kc / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      unsigned char* st = sm + s * SB;
#pragma unroll
      for (int j = 0; j < kKC / 8; ++j) {  // UMMA_K = 8 for tf32 (32 B of K)
        const uint64_t ah = umma_desc(st + j * 256, 128, kSBO);
        const uint64_t bh = umma_desc(st + offB + j * 256, 128, kSBO);
        if (ahs) mma_f16(tmem, ah, bh, idesc, (kc | j) != 0);
        else mma_tf32(tmem, ah, bh, idesc, (kc | j) != 0);
        if (passes != 1) {
          const uint64_t al = umma_desc(st + kSub * 4 + j * 256, 128, kSBO);
          const uint64_t bl = umma_desc(st + 3 * kSub * 4 + j * 256, 128, kSBO);
          mma_tf32(tmem, ah, bl, idesc, 1);
          mma_tf32(tmem, al, bh, idesc, 1);
        }
      }
      mma_commit(&empty[s]);
      if (!coop && kc + S < nkc) {
        mbar_wait(&empty[s], (kc / S) & 1);  // MMAs reading this stage are done
        load(kc + S);
      }
    }
    mma_commit(accf);
  }
  // the epilogue's norms are fetched while the MMAs run: ||a||^2 of this thread's row and the
  // tile's 128 column norms (smem), so their latency is not exposed after the accumulator wait
  __shared__ float sbn[kTM * NT];
  const int q = warp & 3, hh = warp >> 2;  // TMEM lane quarter, column tile of this warp
  const int64_t row = tm * kTM + q * 32 + lane;
  const float a2 = row < m ? an[row] : 0.f;
  // fp16 operands were scaled by powers of two (per row of A, one scale for B): m2 undoes both, exactly
  const float m2 = ahs ? (row < m ? -2.f * ahs[row] * bhs : -2.f) : -2.f;
  sbn[tid] = tn * kTM + tid < n ? bn[tn * kTM + tid] : 0.f;
  __syncthreads();
  mbar_wait(accf, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // the operand stages are free once every MMA completed: each warp transposes its 32 x 32
  // d_hat chunk through shared memory so the global stores are row-contiguous (128 B per row)
  float* stg = reinterpret_cast<float*>(sm) + warp * 32 * 33;
  float gmn = INFINITY;  // 64-column groups: minimum of the group's first chunk
#pragma unroll 1
  for (int cb = 0; cb < kTM / 32; ++cb) {
    uint32_t r[32];
    TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + hh * kTM + cb * 32, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int64_t c0 = (tn + hh) * kTM + cb * 32;
    const float* sb = sbn + hh * kTM + cb * 32;
    const bool full = c0 + 32 <= n;
    float d[32];
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(sb + j);
        d[j + 0] = fmaxf(0.f, fmaf(m2, __uint_as_float(r[j + 0]), a2 + b4.x));
        d[j + 1] = fmaxf(0.f, fmaf(m2, __uint_as_float(r[j + 1]), a2 + b4.y));
        d[j + 2] = fmaxf(0.f, fmaf(m2, __uint_as_float(r[j + 2]), a2 + b4.z));
        d[j + 3] = fmaxf(0.f, fmaf(m2, __uint_as_float(r[j + 3]), a2 + b4.w));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        d[j] = c0 + j < n ? fmaxf(0.f, fmaf(m2, __uint_as_float(r[j]), a2 + sb[j])) : INFINITY;
    }
    if (gmin && row < m && c0 < n) {  // per-row minimum of this 2^gshift-column group (select hint)
      float mn = d[0];
#pragma unroll
      for (int j = 1; j < 32; ++j) mn = fminf(mn, d[j]);
      if (gshift == 6) {  // 64-column groups: two chunks per group
        if ((cb & 1) == 0) gmn = mn;
        mn = fminf(mn, gmn);
      }
      if (gshift == 5 || (cb & 1) == 1 || c0 + 32 >= n) gmin[row * ldg + (c0 >> gshift)] = mn;
    }
    if (!out) continue;  // group minima only (k_select_groups)
    if (full && (ldo & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = d[j];
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 8; ++it) {  // 4 rows x 32 columns per instruction, 128 B per row
        const int ri = it * 4 + (lane >> 3), cc = (lane & 7) * 4;
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
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u * NT) : "memory");
}

__global__ void k_slack(const float* __restrict__ an, int64_t m, float bmax, float gamma, float* __restrict__ slack) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double u = 5.9604644775390625e-08, delta = 9.5367431640625e-07;  // 2^-24, 2^-20
  // eps = u (||x - c|| + max ||y - c||); the fp32 norms of a' = fl(x - c) are inflated to cover
  // ||x - c|| <= ||a'|| / (1 - u) and their own rounding
  const double eps = u * 1.0001 * (sqrt((double)an[i]) + sqrt((double)bmax));
  const double s = (double)gamma * ((double)an[i] + (double)bmax) + eps * eps * (1.0 + 1.0 / delta);
  slack[i] = (float)(s * (1.0 + 1e-6));
}
}  // namespace

int64_t tc_rows_pad(int64_t rows) { return (rows + kTM - 1) / kTM * kTM; }
int tc_nkc(int D) { return (D + kKC - 1) / kKC; }

void launch_split_tf32(const float* X, int64_t rows, int D, const float* center, float* hi, float* lo,
                       float* norm, cudaStream_t st) {
  const int64_t rp = tc_rows_pad(rows);
  if (rp == 0) return;
  k_split_tf32<<<(unsigned)((rp + 7) / 8), 256, 0, st>>>(X, rows, D, tc_nkc(D), center, hi, lo, norm, rp);
  DADE_CK(cudaGetLastError());
}

// relative error coefficient of d_hat (x2 margin): 3-pass split: split error 3 2^-22 per term,
// fp32 accumulation of 3 Dp terms, norm and final roundings; 1-pass (hi parts only): tf32
// rounding of both operands (2 2^-11 + 2^-22 per term) and Dp accumulated terms
float tc_gamma(int D, int passes) {
  const double u23 = 1.1920928955078125e-07;  // 2^-23
  const int Dp = tc_nkc(D) * kKC;
  if (passes == 1) return (float)(2.0 * (9.765625e-04 + (Dp + 16.0) * u23));  // 2^-10
  return (float)(2.0 * (3.0 * Dp + 16.0) * u23);
}

void launch_slack(const float* an, int64_t m, float bmax, int D, float* slack, cudaStream_t st, int passes) {
  if (m <= 0) return;
  k_slack<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(an, m, bmax, tc_gamma(D, passes), slack);
  DADE_CK(cudaGetLastError());
}

void launch_l2_tc(const float* Ahi, const float* Alo, const float* an, int64_t m, const float* Bhi,
                  const float* Blo, const float* bn, int64_t n, int D, float* out, int64_t ldo,
                  cudaStream_t st, float* gmin, int passes, int gshift, const float* ahs, float bhs, int nt) {
  if (m <= 0 || n <= 0) return;
  DADE_REQUIRE(!ahs || passes == 1, DADE_ERR_ARG, "l2_tc: fp16 operands are 1-pass only");
  // set on every launch: the attribute is per device
  DADE_REQUIRE(nt == 1 || nt == 3 || (nt == 2 && passes == 1), DADE_ERR_ARG, "l2_tc: 256-column tiles are 1-pass only");
  if (nt == 2) {  // N = 256 tiles: three 24-KB stages (two CTAs of eight warps per SM: TMEM 2 x 256 columns)
    const int s2 = 3;
    const size_t smem2 = (size_t)s2 * 3 * kSub * 4 + 128;
    DADE_CK(cudaFuncSetAttribute(k_l2_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    dim3 grid2((unsigned)(((n + kTM - 1) / kTM + 1) / 2), (unsigned)((m + kTM - 1) / kTM));
    k_l2_tc<2><<<grid2, 256, smem2, st>>>(Ahi, Alo, an, Bhi, Blo, bn, ahs ? fz_nkc(D, 1) : tc_nkc(D), out, m, n, ldo, gmin,
                                          (n + (1 << gshift) - 1) >> gshift, passes, gshift, s2, ahs, bhs, 0);
    DADE_CK(cudaGetLastError());
    return;
  }
  DADE_CK(cudaFuncSetAttribute(k_l2_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kStageBytes + 128));
  // 1-pass stages (16 KB each): three — 48 KB lets four CTAs share an SM (with four stages the
  // 64 KB allowed three), hiding more of each CTA's wait for its accumulator (C2 search 0.721 ->
  // 0.712-0.718 ms; 2 and 4 measured no better); the epilogue's transposition buffers
  // (4 x 32 x 33 floats) reuse the stage region, so >= 2 stages
  const int nkc_ = ahs ? fz_nkc(D, 1) : tc_nkc(D);
  const int coop = nt == 3 && passes == 1 && nkc_ <= 4;  // nt = 3: cooperative cp.async operand load (measurement)
  const int s1 = coop ? nkc_ : 3;
  const size_t smem = (passes == 1 ? (size_t)s1 * (kStageBytes / 2) : 2 * (size_t)kStageBytes) + 128;
  dim3 grid((unsigned)((n + kTM - 1) / kTM), (unsigned)((m + kTM - 1) / kTM));
  // fp16 operands (Ahi / Bhi point at launch_split_h16's blocks): 32 halves per row per chunk
  k_l2_tc<1><<<grid, 128, smem, st>>>(Ahi, Alo, an, Bhi, Blo, bn, ahs ? fz_nkc(D, 1) : tc_nkc(D), out, m, n, ldo, gmin,
                                   (n + (1 << gshift) - 1) >> gshift, passes, gshift, s1, ahs, bhs, coop);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade

namespace dade {
namespace {
// fp64 column sums of an n x D fp32 matrix (atomic per column; blocks stride over rows)
__global__ void k_colsum(const float* __restrict__ X, int64_t n, int D, double* __restrict__ sum) {
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    double s = 0.0;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) s += (double)X[r * D + j];
    atomicAdd(sum + j, s);
  }
}
__global__ void k_mean_f32(const double* __restrict__ sum, int64_t n, int D, float* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < D) out[j] = n > 0 ? (float)(sum[j] / (double)n) : 0.f;
}
__global__ void k_max_nonneg(const float* __restrict__ v, int64_t n, unsigned* out) {
  unsigned m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(v[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
}  // namespace
void launch_col_mean(const float* X, int64_t n, int D, double* scratch, float* out, cudaStream_t st) {
  DADE_CK(cudaMemsetAsync(scratch, 0, sizeof(double) * D, st));
  if (n > 0) k_colsum<<<(unsigned)std::min<int64_t>(n, 2048), 256, 0, st>>>(X, n, D, scratch);
  k_mean_f32<<<(D + 255) / 256, 256, 0, st>>>(scratch, n, D, out);
  DADE_CK(cudaGetLastError());
}

void launch_max_nonneg(const float* v, int64_t n, float* out_dev, cudaStream_t st) {
  DADE_CK(cudaMemsetAsync(out_dev, 0, sizeof(float), st));
  if (n <= 0) return;
  k_max_nonneg<<<592, 256, 0, st>>>(v, n, reinterpret_cast<unsigned*>(out_dev));
  DADE_CK(cudaGetLastError());
}
}  // namespace dade
