// Exact nearest-centroid / nearest-neighbour selection (IVF assignment P:L172-173, probe P:L174,
// brute-force KNN P:L132-137) that is BIT-EXACT with the fp64 sequential-sum definition (R20):
//   1. d_hat = fp32 direct-difference distances for a tile of rows (FMA accumulation),
//   2. relative error bound rho = gamma_{D+2}: d_hat in [d(1-rho), d(1+rho)],
//   3. candidates = columns with d_hat <= d_hat_(k) * (1+rho)/(1-rho)  (contains every column whose
//      exact distance is <= the exact k-th distance, ties included),
//   4. exact fp64 sequential sums (no FMA contraction) for the candidates, sort by (dist, column).
#include <algorithm>
#include <cfloat>
#include <cstdio>

#include "dade_internal.h"
#include "exact_batch.cuh"

namespace dade {

// ------------------------------------------------------------------ fp32 tile distances
// 64 x 64 output tile per CTA, 256 threads, 4 x 4 outputs per thread, D consumed 16 dims at a time.
__global__ void __launch_bounds__(256) k_l2_tile(const float* __restrict__ A, int64_t m,
                                                 const float* __restrict__ B, int64_t n, int D,
                                                 float* __restrict__ out) {
  __shared__ __align__(16) float As[16][64];
  __shared__ __align__(16) float Bs[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // loader mapping: 256 threads load 64 rows x 16 dims = 1024 floats each for A and B (4 per thread)
  const int lr = threadIdx.x >> 2, lc = (threadIdx.x & 3) * 4;
  for (int k0 = 0; k0 < D; k0 += 16) {
    float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
    if (r0 + lr < m) va = *reinterpret_cast<const float4*>(A + (r0 + lr) * D + k0 + lc);
    if (c0 + lr < n) vb = *reinterpret_cast<const float4*>(B + (c0 + lr) * D + k0 + lc);
    As[lc + 0][lr] = va.x; As[lc + 1][lr] = va.y; As[lc + 2][lr] = va.z; As[lc + 3][lr] = va.w;
    Bs[lc + 0][lr] = vb.x; Bs[lc + 1][lr] = vb.y; Bs[lc + 2][lr] = vb.z; Bs[lc + 3][lr] = vb.w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float t = av[i] - bv[j];
          acc[i][j] = fmaf(t, t, acc[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty * 4 + i;
    if (r >= m) continue;
    const int64_t c = c0 + tx * 4;
    float* o = out + r * n + c;
    if (c + 3 < n && (n & 3) == 0) {
      *reinterpret_cast<float4*>(o) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c + j < n) o[j] = acc[i][j];
    }
  }
}

void launch_l2_tile(const float* A, int64_t m, const float* B, int64_t n, int D, float* out,
                    cudaStream_t st) {
  dim3 grid((unsigned)((n + 63) / 64), (unsigned)((m + 63) / 64));
  k_l2_tile<<<grid, 256, 0, st>>>(A, m, B, n, D, out);
  DADE_CK(cudaGetLastError());
}

// ------------------------------------------------------------------ exact fp64 distance
// The definition (R20): sum_{j=0}^{D-1} (a_j - b_j)^2 in IEEE fp64, sequential, each operation
// rounded separately (explicit _rn intrinsics forbid FMA contraction).
__device__ __forceinline__ double exact_sqdist(const float* __restrict__ a,
                                               const float* __restrict__ b, int D) {
  double acc = 0.0;
  for (int j = 0; j < D; ++j) {
    const double t = __dsub_rn((double)a[j], (double)b[j]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc;
}

// threshold on d_hat bits: T = v * (1+rho)/(1-rho) rounded up, rho = 2 * gamma_{D+2}
__device__ __forceinline__ unsigned thr_bits(float v, int D) {
  const double u = 5.9604644775390625e-08;  // 2^-24
  const double g = (D + 2) * u / (1.0 - (D + 2) * u);
  const double rho = 2.0 * g;
  const double T = (double)v * (1.0 + rho) / (1.0 - rho);
  float tf = (float)T;
  unsigned b = __float_as_uint(tf);
  if (!(tf >= 0.f)) return 0xffffffffu;
  return b == 0x7f800000u ? b : b + 2u;  // two ulps of slack on top of the rounding of T
}

// window for the tensor-core filter (gemm_tf32.cu): |d_hat - d| <= slack + delta d, so every true
// k-nearest column has d_hat <= (v + slack)(1 + delta)/(1 - delta) + slack, v = k-th smallest
// d_hat; bits rounded up
__device__ __forceinline__ unsigned abs_thr_bits(float v, float slack) {
  const double delta = 9.5367431640625e-07;  // 2^-20
  const double T = ((double)v + (double)slack) * (1.0 + delta) / (1.0 - delta) + (double)slack;
  const float tf = (float)T;
  if (!(tf >= 0.f)) return 0xffffffffu;
  const unsigned b = __float_as_uint(tf);
  return b == 0x7f800000u ? b : b + 2u;
}

struct Cand {
  double d;
  int32_t c;
};
__device__ __forceinline__ bool cand_less(const Cand& x, const Cand& y) {
  return x.d < y.d || (x.d == y.d && x.c < y.c);
}

constexpr int kSelThreads = 512;
constexpr int kSortCap = 4096;

// One CTA per row: radix-select the k-th smallest d_hat, collect candidates, exact re-rank, sort.
__global__ void __launch_bounds__(kSelThreads) k_select_exact(
    const float* __restrict__ dh, int64_t n, int k, const float* __restrict__ A,
    const float* __restrict__ B, int D, int32_t* __restrict__ out_idx, double* __restrict__ out_d,
    int32_t* __restrict__ cand_buf, int cand_cap, int* flag, const float* __restrict__ slack) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cand* cs = reinterpret_cast<Cand*>(smem_raw);  // kSortCap entries
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix, s_krem, s_count;
  const int64_t row = blockIdx.x;
  const float* d = dh + row * n;
  const unsigned* du = reinterpret_cast<const unsigned*>(d);
  const int tid = threadIdx.x;
  if (tid == 0) { s_prefix = 0; s_krem = (unsigned)k; s_count = 0; }
  unsigned mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned prefix = s_prefix;
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const unsigned b = du[i];
      if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      unsigned kr = s_krem, cum = 0;
      int dig = 0;
      for (; dig < 256; ++dig) {
        if (cum + hist[dig] >= kr) break;
        cum += hist[dig];
      }
      s_krem = kr - cum;
      s_prefix = prefix | ((unsigned)dig << shift);
    }
    mask |= 255u << shift;
    __syncthreads();
  }
  const unsigned tb = slack ? abs_thr_bits(__uint_as_float(s_prefix), slack[row])
                           : thr_bits(__uint_as_float(s_prefix), D);
  int32_t* cb = cand_buf + row * (int64_t)cand_cap;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    if (du[i] <= tb) {
      const unsigned pos = atomicAdd(&s_count, 1u);
      if (pos < (unsigned)cand_cap) cb[pos] = (int32_t)i;
    }
  }
  __syncthreads();
  unsigned cnt = s_count;
  if (cnt > (unsigned)cand_cap || cnt > (unsigned)kSortCap) {
    if (tid == 0) atomicExch(flag, 1);
    cnt = min(cnt, (unsigned)min(cand_cap, kSortCap));
  }
  unsigned P = 1;
  while (P < cnt) P <<= 1;
  const float* a = A + row * (int64_t)D;
  for (unsigned i = tid; i < P; i += blockDim.x) {
    if (i < cnt) {
      const int32_t c = cb[i];
      cs[i].d = exact_sqdist(a, B + (int64_t)c * D, D);
      cs[i].c = c;
    } else {
      cs[i].d = DBL_MAX;
      cs[i].c = 0x7fffffff;
    }
  }
  __syncthreads();
  // bitonic sort of P entries by (d, c)
  for (unsigned size = 2; size <= P; size <<= 1) {
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      for (unsigned i = tid; i < P / 2; i += blockDim.x) {
        const unsigned lo = 2 * i - (i & (stride - 1));
        const unsigned hi = lo + stride;
        const bool up = ((lo & size) == 0);
        Cand x = cs[lo], y = cs[hi];
        if (cand_less(y, x) == up) { cs[lo] = y; cs[hi] = x; }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < k; i += blockDim.x) {
    const bool ok = (unsigned)i < cnt;
    out_idx[row * k + i] = ok ? cs[i].c : -1;
    if (out_d) out_d[row * k + i] = ok ? cs[i].d : DBL_MAX;
  }
}

// Fast path for short rows (probe: n = nlist <= 8192): the row lives in registers; a linear
// histogram over [min, max] (refined on the boundary bin until few candidates remain) yields a
// value E >= the k-th smallest d_hat with few elements below it. Every column with
// d_hat <= E * (1+rho)/(1-rho) is re-ranked exactly (a superset of the certified set).
constexpr int kSmallThreads = 256;
constexpr int kBins = 1024;
constexpr int kSmallCap = 1024;

__device__ __forceinline__ float block_reduce(float v, bool is_max, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, x) : fminf(v, x);
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = red[0];
  for (int i = 1; i < kSmallThreads / 32; ++i) v = is_max ? fmaxf(v, red[i]) : fminf(v, red[i]);
  return v;
}

template <int EPT>
__global__ void __launch_bounds__(kSmallThreads) k_select_small(
    const float* __restrict__ dh, int64_t n, int k, const float* __restrict__ A,
    const float* __restrict__ B, int D, int32_t* __restrict__ out_idx, double* __restrict__ out_d,
    int* flag, const float* __restrict__ slack, const int32_t* __restrict__ rows,
    const int* __restrict__ nrows) {
  __shared__ unsigned hist[kBins];
  __shared__ float red[kSmallThreads / 32];
  __shared__ Cand cs[kSmallCap];
  __shared__ unsigned s_cnt, s_bin, s_cum;
  const int tid = threadIdx.x;
  // fallback mode (rows != null): a small grid walks the listed rows
  const int64_t nr = rows ? (int64_t)*nrows : (int64_t)gridDim.x;
  for (int64_t ri = blockIdx.x; ri < nr; ri += rows ? gridDim.x : nr) {
  const int64_t row = rows ? rows[ri] : ri;
  float v[EPT];
  uint32_t inplay = 0;
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int64_t idx = (int64_t)j * kSmallThreads + tid;
    v[j] = idx < n ? dh[row * n + idx] : INFINITY;
    if (idx < n) inplay |= 1u << j;
  }
  unsigned below = 0;  // elements known to be below the in-play range
  float E = 0.f;
  for (int level = 0; level < 4; ++level) {
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if (inplay >> j & 1u) { lo = fminf(lo, v[j]); hi = fmaxf(hi, v[j]); }
    lo = block_reduce(lo, false, red);
    hi = block_reduce(hi, true, red);
    if (!(hi > lo)) { E = hi; break; }  // all in-play values equal
    const float scale = (float)kBins / (hi - lo);
    for (int i = tid; i < kBins; i += kSmallThreads) hist[i] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if (inplay >> j & 1u) atomicAdd(&hist[min(kBins - 1, (int)((v[j] - lo) * scale))], 1u);
    __syncthreads();
    if (tid < 32) {  // warp prefix over 1024 bins: 32 bins per lane
      constexpr int BPL = kBins / 32;
      unsigned own = 0;
#pragma unroll 8
      for (int i = 0; i < BPL; ++i) own += hist[tid * BPL + i];
      unsigned inc = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
        if (tid >= o) inc += t;
      }
      const unsigned excl = below + inc - own;
      const unsigned hit = __ballot_sync(0xffffffffu, excl + own >= (unsigned)k);
      const int L0 = hit ? __ffs(hit) - 1 : 31;
      if (tid == L0) {
        unsigned cum = excl;
        int b = tid * BPL;
        for (; b < tid * BPL + BPL - 1; ++b) {
          if (cum + hist[b] >= (unsigned)k) break;
          cum += hist[b];
        }
        s_bin = (unsigned)b;
        s_cum = cum;  // elements strictly below bin b
      }
    }
    __syncthreads();
    const int b = (int)s_bin;
    const unsigned cum = s_cum;
    const unsigned in_b = hist[b];
    if (cum + in_b <= kSmallCap / 2 || level == 3) {
      float e = -INFINITY;  // E = largest in-play value with bin <= b (>= the k-th smallest)
#pragma unroll
      for (int j = 0; j < EPT; ++j)
        if ((inplay >> j & 1u) && min(kBins - 1, (int)((v[j] - lo) * scale)) <= b) e = fmaxf(e, v[j]);
      E = block_reduce(e, true, red);
      break;
    }
    below = cum;  // refine inside bin b
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if ((inplay >> j & 1u) && min(kBins - 1, (int)((v[j] - lo) * scale)) != b) inplay &= ~(1u << j);
    __syncthreads();
  }
  const unsigned tb = slack ? abs_thr_bits(E, slack[row]) : thr_bits(E, D);
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  const float* a = A + row * (int64_t)D;
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int64_t idx = (int64_t)j * kSmallThreads + tid;
    if (idx < n && __float_as_uint(v[j]) <= tb) {
      const unsigned pos = atomicAdd(&s_cnt, 1u);
      if (pos < (unsigned)kSmallCap) { cs[pos].c = (int32_t)idx; cs[pos].d = 0.0; }
    }
  }
  __syncthreads();
  unsigned cnt = s_cnt;
  if (cnt > (unsigned)kSmallCap) {
    if (tid == 0) atomicExch(flag, 1);
    cnt = kSmallCap;
  }
  unsigned P = 1;
  while (P < cnt) P <<= 1;
  for (unsigned i = tid; i < P; i += kSmallThreads) {
    if (i < cnt) cs[i].d = exact_sqdist(a, B + (int64_t)cs[i].c * D, D);
    else { cs[i].d = DBL_MAX; cs[i].c = 0x7fffffff; }
  }
  __syncthreads();
  for (unsigned size = 2; size <= P; size <<= 1)
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      for (unsigned i = tid; i < P / 2; i += kSmallThreads) {
        const unsigned lo2 = 2 * i - (i & (stride - 1)), hi2 = lo2 + stride;
        const bool up = (lo2 & size) == 0;
        const Cand x = cs[lo2], y = cs[hi2];
        if (cand_less(y, x) == up) { cs[lo2] = y; cs[hi2] = x; }
      }
      __syncthreads();
    }
  for (int i = tid; i < k; i += kSmallThreads) {
    const bool ok = (unsigned)i < cnt;
    out_idx[row * k + i] = ok ? cs[i].c : -1;
    if (out_d) out_d[row * k + i] = ok ? cs[i].d : DBL_MAX;
  }
  __syncthreads();  // shared state is reused by the next listed row
  }
}

// Warp-per-row exact select for the tensor-core filter. E = the k-th smallest of the row's
// 32-column group minima is >= the k-th smallest d_hat (k groups each hold an element <= E), so
// every column with d_hat <= E + 2 slack is re-ranked exactly; the certified set is contained.
constexpr int kGmWarps = 4;
constexpr int kGmCap = 256;

__device__ __forceinline__ bool cand_less2(double d0, int32_t c0, double d1, int32_t c1) {
  return d0 < d1 || (d0 == d1 && c0 < c1);
}


// The columns inside the window: every such column lies in a group whose minimum is inside it,
// so only those groups' d_hat are read, as 32-column (128-B, coalesced) segments. The selected
// groups are listed first (glist, per-warp smem) and their segments are then loaded kSegBatch at
// a time, so a row with many candidate groups pays ~1/kSegBatch of the dependent round trips.
// Returns the candidate count (may exceed kGmCap: only the first kGmCap are stored in cc).
constexpr int kSegBatch = 4;
template <int GPL>
__device__ __forceinline__ int window_cands(const float (&gv)[GPL], unsigned tb, const float* __restrict__ d, int64_t n,
                                            int gshift, int lane, int* glist, int32_t* cc) {
  int ns = 0;
#pragma unroll
  for (int j = 0; j < GPL; ++j) {
    const bool in = __float_as_uint(gv[j]) <= tb;
    const unsigned b = __ballot_sync(0xffffffffu, in);
    if (in) glist[ns + __popc(b & ((1u << lane) - 1))] = lane + 32 * j;
    ns += __popc(b);
  }
  __syncwarp();
  const int sh = gshift - 5;  // log2 segments per group
  const int nseg = ns << sh;
  int cnt = 0;
#pragma unroll 1
  for (int s0 = 0; s0 < nseg; s0 += kSegBatch) {
    float v[kSegBatch];
    int64_t col[kSegBatch];
#pragma unroll
    for (int u = 0; u < kSegBatch; ++u) {
      const int s = s0 + u;
      col[u] = s < nseg ? ((int64_t)glist[s >> sh] << gshift) + ((s & ((1 << sh) - 1)) << 5) + lane : n;
      v[u] = col[u] < n ? __ldg(d + col[u]) : INFINITY;
    }
#pragma unroll
    for (int u = 0; u < kSegBatch; ++u) {
      const bool in = col[u] < n && __float_as_uint(v[u]) <= tb;
      const unsigned bal = __ballot_sync(0xffffffffu, in);
      if (in) {
        const int pos = cnt + __popc(bal & ((1u << lane) - 1));
        if (pos < kGmCap) cc[pos] = (int32_t)col[u];
      }
      cnt += __popc(bal);
    }
  }
  return cnt;
}

template <int GPL>  // group minima per lane: rows of up to 32 * GPL groups of 2^gshift columns
__global__ void __launch_bounds__(kGmWarps * 32) k_select_gmin(
    const float* __restrict__ dh, const float* __restrict__ gm, int gshift, int64_t m, int64_t n, int k,
    const float* __restrict__ A, const float* __restrict__ B, int D, int32_t* __restrict__ out_idx,
    double* __restrict__ out_d, int* ovf_n, int32_t* __restrict__ ovf_rows, const float* __restrict__ slack) {
  __shared__ float sg[kGmWarps][32 * GPL];
  __shared__ double cd[kGmWarps][kGmCap];
  __shared__ int32_t cc[kGmWarps][kGmCap];
  __shared__ __align__(16) float xstage[kGmWarps][kXbStage];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kGmWarps + w;
  if (row >= m) return;
  const int ng = (int)((n + (1 << gshift) - 1) >> gshift);
  // the k-th smallest group minimum E bounds the k-th smallest d_hat from above
  float gv[GPL];  // group lane + 32 j
#pragma unroll
  for (int j = 0; j < GPL; ++j) gv[j] = lane + 32 * j < ng ? gm[row * ng + lane + 32 * j] : INFINITY;
  float E;
  if (k <= 16) {  // k rounds of a warp-wide minimum (REDUX on the value bits: minima are >= 0 or
    // +inf, so unsigned order is float order); each round removes ONE occurrence of the minimum,
    // so E is the k-th smallest value of the multiset whichever tied group is removed
    unsigned rem[GPL];
#pragma unroll
    for (int j = 0; j < GPL; ++j) rem[j] = __float_as_uint(gv[j]);
    unsigned mn = 0;
    for (int r = 0; r < k; ++r) {
      unsigned lm = rem[0];
#pragma unroll
      for (int j = 1; j < GPL; ++j) lm = min(lm, rem[j]);
      mn = __reduce_min_sync(0xffffffffu, lm);
      const unsigned who = __ballot_sync(0xffffffffu, lm == mn);
      if (lane == __ffs(who) - 1) {
        bool done = false;
#pragma unroll
        for (int j = 0; j < GPL; ++j)
          if (!done && rem[j] == mn) {
            rem[j] = 0xffffffffu;  // removed: above every value, +inf included
            done = true;
          }
      }
    }
    E = __uint_as_float(mn);
  } else {  // bitonic sort of the group minima (GPL per lane)
    float* g = sg[w];
#pragma unroll
    for (int j = 0; j < GPL; ++j) g[lane + 32 * j] = gv[j];
    __syncwarp();
    for (int size = 2; size <= 32 * GPL; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = lane; i < 16 * GPL; i += 32) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const float x = g[lo], y = g[hi];
          if ((y < x) == up) { g[lo] = y; g[hi] = x; }
        }
        __syncwarp();
      }
    E = g[k - 1];
  }
  const unsigned tb = abs_thr_bits(E, slack[row]);
  __syncwarp();  // sg[w] (the k > 16 sort's buffer) now holds the selected group list
  const int cnt = window_cands<GPL>(gv, tb, dh + row * n, n, gshift, lane, reinterpret_cast<int*>(sg[w]), cc[w]);
  if (cnt > kGmCap) {  // too many near-ties: the histogram select redoes this row
    if (lane == 0) ovf_rows[atomicAdd(ovf_n, 1)] = (int32_t)row;
    return;
  }
  __syncwarp();
  const float* a = A + row * (int64_t)D;
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i0 = 0; i0 < P; i0 += 32) {  // exact fp64 distances, 32 candidates per staged batch
    const int i = i0 + lane;
    const int32_t c = (i < cnt) ? cc[w][i] : -1;
    const double d = i0 < cnt ? exact_batch32(a, B, D, c, xstage[w], lane, min(32, cnt - i0)) : 0.0;
    if (i < P) {
      if (i < cnt) cd[w][i] = d;
      else { cd[w][i] = DBL_MAX; cc[w][i] = 0x7fffffff; }
    }
  }
  __syncwarp();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < P / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double x = cd[w][lo], y = cd[w][hi];
        const int32_t xc = cc[w][lo], yc = cc[w][hi];
        if (cand_less2(y, yc, x, xc) == up) { cd[w][lo] = y; cd[w][hi] = x; cc[w][lo] = yc; cc[w][hi] = xc; }
      }
      __syncwarp();
    }
  for (int i = lane; i < k; i += 32) {
    const bool ok = i < cnt;
    out_idx[row * k + i] = ok ? cc[w][i] : -1;
    if (out_d) out_d[row * k + i] = ok ? cd[w][i] : DBL_MAX;
  }
}
// Same selection with ONE row per CTA (large k, e.g. nprobe 64 at D = 960): warp 0 finds the
// candidates, the four warps share the row's fp64 batches (each a long sequential chain), warp 0
// sorts. Used when k > 16.
template <int GPL>
__global__ void __launch_bounds__(kGmWarps * 32) k_select_gmin_wide(
    const float* __restrict__ dh, const float* __restrict__ gm, int gshift, int64_t m, int64_t n, int k,
    const float* __restrict__ A, const float* __restrict__ B, int D, int32_t* __restrict__ out_idx,
    double* __restrict__ out_d, int* ovf_n, int32_t* __restrict__ ovf_rows, const float* __restrict__ slack) {
  __shared__ float sg[1][32 * GPL];
  __shared__ double cd[1][kGmCap];
  __shared__ int32_t cc[1][kGmCap];
  __shared__ __align__(16) float xstage[kGmWarps][kXbStage];
  __shared__ int s_cnt;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, w = 0;
  const int64_t row = blockIdx.x;
  int cnt = 0;
  if (wid == 0) {
  const int ng = (int)((n + (1 << gshift) - 1) >> gshift);
  // the k-th smallest group minimum E bounds the k-th smallest d_hat from above
  float gv[GPL];  // group lane + 32 j
#pragma unroll
  for (int j = 0; j < GPL; ++j) gv[j] = lane + 32 * j < ng ? gm[row * ng + lane + 32 * j] : INFINITY;
  float E;
  if (k <= 16) {  // k rounds of a warp-wide minimum (REDUX on the value bits: minima are >= 0 or
    // +inf, so unsigned order is float order); each round removes ONE occurrence of the minimum,
    // so E is the k-th smallest value of the multiset whichever tied group is removed
    unsigned rem[GPL];
#pragma unroll
    for (int j = 0; j < GPL; ++j) rem[j] = __float_as_uint(gv[j]);
    unsigned mn = 0;
    for (int r = 0; r < k; ++r) {
      unsigned lm = rem[0];
#pragma unroll
      for (int j = 1; j < GPL; ++j) lm = min(lm, rem[j]);
      mn = __reduce_min_sync(0xffffffffu, lm);
      const unsigned who = __ballot_sync(0xffffffffu, lm == mn);
      if (lane == __ffs(who) - 1) {
        bool done = false;
#pragma unroll
        for (int j = 0; j < GPL; ++j)
          if (!done && rem[j] == mn) {
            rem[j] = 0xffffffffu;  // removed: above every value, +inf included
            done = true;
          }
      }
    }
    E = __uint_as_float(mn);
  } else {  // bitonic sort of the group minima (GPL per lane)
    float* g = sg[w];
#pragma unroll
    for (int j = 0; j < GPL; ++j) g[lane + 32 * j] = gv[j];
    __syncwarp();
    for (int size = 2; size <= 32 * GPL; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = lane; i < 16 * GPL; i += 32) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const float x = g[lo], y = g[hi];
          if ((y < x) == up) { g[lo] = y; g[hi] = x; }
        }
        __syncwarp();
      }
    E = g[k - 1];
  }
  const unsigned tb = abs_thr_bits(E, slack[row]);
  __syncwarp();  // sg[w] (the k > 16 sort's buffer) now holds the selected group list
  cnt = window_cands<GPL>(gv, tb, dh + row * n, n, gshift, lane, reinterpret_cast<int*>(sg[w]), cc[w]);
  if (cnt > kGmCap && lane == 0) ovf_rows[atomicAdd(ovf_n, 1)] = (int32_t)row;  // histogram select redoes it
  if (lane == 0) s_cnt = cnt;
  }
  __syncthreads();
  cnt = s_cnt;
  if (cnt > kGmCap) return;
  for (int i0 = wid * 32; i0 < cnt; i0 += kGmWarps * 32) {  // batches shared by the four warps
    const int i = i0 + lane;
    const int32_t c = i < cnt ? cc[0][i] : -1;
    const double d = exact_batch32(A + row * (int64_t)D, B, D, c, xstage[wid], lane, min(32, cnt - i0));
    if (i < cnt) cd[0][i] = d;
  }
  __syncthreads();
  if (wid != 0) return;
  const float* a = A + row * (int64_t)D;
  (void)a;
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + lane; i < P; i += 32) { cd[0][i] = DBL_MAX; cc[0][i] = 0x7fffffff; }
  __syncwarp();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < P / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double x = cd[w][lo], y = cd[w][hi];
        const int32_t xc = cc[w][lo], yc = cc[w][hi];
        if (cand_less2(y, yc, x, xc) == up) { cd[w][lo] = y; cd[w][hi] = x; cc[w][lo] = yc; cc[w][hi] = xc; }
      }
      __syncwarp();
    }
  for (int i = lane; i < k; i += 32) {
    const bool ok = i < cnt;
    out_idx[row * k + i] = ok ? cc[w][i] : -1;
    if (out_d) out_d[row * k + i] = ok ? cd[w][i] : DBL_MAX;
  }
}

// ------------------------------------------------------------------ group select (no d_hat)
// The filter GEMM wrote only the per-row minima of d_hat over 32-column groups (gm[row][g]). Every
// group minimum is some column's d_hat, so the k-th smallest group minimum E bounds the k-th
// smallest d_hat from above; every true k-nearest column therefore has d_hat <= thr(E) (window of
// abs_thr_bits) and lies in a group with gm <= thr(E). All columns of those groups get their
// exact fp64 distance (one lane per column) and the k smallest by (dist, column) are kept: a
// running top-k in shared memory (chunks of kGsCap - k new candidates, bitonic sort, truncate).
constexpr int kGsWarps = 4;
constexpr int kGsCap = 1024;

__global__ void __launch_bounds__(kGsWarps * 32) k_select_groups(
    const float* __restrict__ gm, int64_t m, int64_t n, int k, const float* __restrict__ A,
    const float* __restrict__ B, int D, int32_t* __restrict__ out_idx, double* __restrict__ out_d,
    const float* __restrict__ slack) {
  extern __shared__ __align__(16) unsigned char gs_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* cd = reinterpret_cast<double*>(gs_smem) + (size_t)w * kGsCap;
  int32_t* cc = reinterpret_cast<int32_t*>(reinterpret_cast<double*>(gs_smem) + (size_t)kGsWarps * kGsCap) +
                (size_t)w * kGsCap;
  unsigned* hist = reinterpret_cast<unsigned*>(reinterpret_cast<int32_t*>(
                       reinterpret_cast<double*>(gs_smem) + (size_t)kGsWarps * kGsCap) + (size_t)kGsWarps * kGsCap) +
                   w * 256;
  const int64_t row = (int64_t)blockIdx.x * kGsWarps + w;
  if (row >= m) return;
  const int ng = (int)((n + 31) / 32);
  const float* g = gm + row * ng;
  // 1. E = k-th smallest group minimum: radix select on the float bits (non-negative)
  unsigned prefix = 0;
  int krem = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    for (int i = lane; i < ng; i += 32) {
      const unsigned v = __float_as_uint(g[i]);
      if (shift == 24 || ((v ^ prefix) >> (shift + 8)) == 0) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncwarp();
    unsigned h[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { h[j] = hist[lane * 8 + j]; tot += h[j]; }
    unsigned inc = tot;  // inclusive scan over lanes
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
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    const int src = __ffs(bal) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    below = __shfl_sync(0xffffffffu, below, src);
    prefix |= (unsigned)bin << shift;
    krem -= (int)below;
    __syncwarp();
  }
  const unsigned tb = abs_thr_bits(__uint_as_float(prefix), slack[row]);
  // 2. exact distances of every column of every group inside the window; running top-k
  const float* a = A + row * (int64_t)D;
  for (int i = lane; i < k; i += 32) { cd[i] = DBL_MAX; cc[i] = 0x7fffffff; }
  int cnt = k;  // slots [0, k) hold the running top-k
  auto compact = [&]() {  // sort slots [0, cnt) (padded to a power of two) and keep the first k
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
          if (cand_less2(y, yc, x, xc) == up) { cd[lo] = y; cd[hi] = x; cc[lo] = yc; cc[hi] = xc; }
        }
        __syncwarp();
      }
    cnt = k;
  };
  for (int g0 = 0; g0 < ng; g0 += 32) {
    const int gi = g0 + lane;
    const bool in = gi < ng && __float_as_uint(g[gi]) <= tb;
    unsigned bal = __ballot_sync(0xffffffffu, in);
    while (bal) {
      const int grp = g0 + __ffs(bal) - 1;
      bal &= bal - 1;
      if (cnt + 32 > kGsCap) compact();
      const int64_t c = (int64_t)grp * 32 + lane;
      if (c < n) {
        cd[cnt + lane] = exact_sqdist(a, B + c * D, D);
        cc[cnt + lane] = (int32_t)c;
      } else {
        cd[cnt + lane] = DBL_MAX;
        cc[cnt + lane] = 0x7fffffff;
      }
      cnt += 32;
      __syncwarp();
    }
  }
  compact();
  for (int i = lane; i < k; i += 32) {
    const bool ok = cd[i] != DBL_MAX;
    out_idx[row * k + i] = ok ? cc[i] : -1;
    if (out_d) out_d[row * k + i] = ok ? cd[i] : DBL_MAX;
  }
}

void launch_select_groups(const float* gmin, int64_t m, int64_t n, int k, const float* A, const float* B,
                          int D, int32_t* out_idx, double* out_d64, const float* slack, cudaStream_t st) {
  if (m <= 0) return;
  DADE_REQUIRE(k >= 1 && k <= 512, DADE_ERR_UNSUPPORTED, "group select: k > 512");
  const size_t smem = (size_t)kGsWarps * kGsCap * 12 + (size_t)kGsWarps * 256 * 4;
  DADE_CK(cudaFuncSetAttribute(k_select_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  // per launch: per device
  k_select_groups<<<(unsigned)((m + kGsWarps - 1) / kGsWarps), kGsWarps * 32, smem, st>>>(
      gmin, m, n, k, A, B, D, out_idx, out_d64, slack);
  DADE_CK(cudaGetLastError());
}

void launch_select_gmin(const float* d_hat, const float* gmin, int gshift, int64_t m, int64_t n, int k,
                        const float* A, const float* B, int D, int32_t* out_idx, double* out_d64,
                        int* d_flag, const float* slack, int* ovf_n, int32_t* ovf_rows,
                        cudaStream_t st) {
  if (m <= 0) return;
  DADE_CK(cudaMemsetAsync(ovf_n, 0, sizeof(int), st));
  const int64_t ngr = (n + (1 << gshift) - 1) >> gshift;
  const unsigned gsz = (unsigned)((m + kGmWarps - 1) / kGmWarps);
  if (k > 16 && ngr <= 256)
    k_select_gmin_wide<8><<<(unsigned)m, kGmWarps * 32, 0, st>>>(d_hat, gmin, gshift, m, n, k, A, B, D, out_idx, out_d64, ovf_n, ovf_rows, slack);
  else if (k > 16 && ngr <= 512)
    k_select_gmin_wide<16><<<(unsigned)m, kGmWarps * 32, 0, st>>>(d_hat, gmin, gshift, m, n, k, A, B, D, out_idx, out_d64, ovf_n, ovf_rows, slack);
  else if (k > 16)
    k_select_gmin_wide<32><<<(unsigned)m, kGmWarps * 32, 0, st>>>(d_hat, gmin, gshift, m, n, k, A, B, D, out_idx, out_d64, ovf_n, ovf_rows, slack);
  else if (ngr <= 256)
    k_select_gmin<8><<<gsz, kGmWarps * 32, 0, st>>>(d_hat, gmin, gshift, m, n, k, A, B, D, out_idx, out_d64, ovf_n, ovf_rows, slack);
  else if (ngr <= 512)
    k_select_gmin<16><<<gsz, kGmWarps * 32, 0, st>>>(d_hat, gmin, gshift, m, n, k, A, B, D, out_idx, out_d64, ovf_n, ovf_rows, slack);
  else
    k_select_gmin<32><<<gsz, kGmWarps * 32, 0, st>>>(d_hat, gmin, gshift, m, n, k, A, B, D, out_idx, out_d64, ovf_n, ovf_rows, slack);
  DADE_CK(cudaGetLastError());
  // device-side fallback (no host round trip): a small grid walks the listed rows
  const unsigned fg = (unsigned)std::min<int64_t>(m, 296);
  if (n <= 16 * kSmallThreads)
    k_select_small<16><<<fg, kSmallThreads, 0, st>>>(d_hat, n, k, A, B, D, out_idx, out_d64, d_flag,
                                                      slack, ovf_rows, ovf_n);
  else
    k_select_small<32><<<fg, kSmallThreads, 0, st>>>(d_hat, n, k, A, B, D, out_idx, out_d64, d_flag,
                                                      slack, ovf_rows, ovf_n);
  DADE_CK(cudaGetLastError());
}

void launch_select_exact(const float* d_hat, int64_t m, int64_t n, int k, const float* A,
                         const float* B, int D, int32_t* out_idx, double* out_d64,
                         int32_t* cand_buf, int cand_cap, int* d_flag, cudaStream_t st,
                         const float* slack) {
  if (m <= 0) return;
  if (n <= 16 * kSmallThreads && k <= kSmallCap / 2) {
    k_select_small<16><<<(unsigned)m, kSmallThreads, 0, st>>>(d_hat, n, k, A, B, D, out_idx, out_d64, d_flag, slack,
                                                               nullptr, nullptr);
    DADE_CK(cudaGetLastError());
    return;
  }
  if (n <= 32 * kSmallThreads && k <= kSmallCap / 2) {
    k_select_small<32><<<(unsigned)m, kSmallThreads, 0, st>>>(d_hat, n, k, A, B, D, out_idx, out_d64, d_flag, slack,
                                                               nullptr, nullptr);
    DADE_CK(cudaGetLastError());
    return;
  }
  const size_t smem = kSortCap * sizeof(Cand);
  DADE_CK(cudaFuncSetAttribute(k_select_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));  // per launch: per device
  k_select_exact<<<(unsigned)m, kSelThreads, smem, st>>>(d_hat, n, k, A, B, D, out_idx, out_d64,
                                                         cand_buf, cand_cap, d_flag, slack);
  DADE_CK(cudaGetLastError());
}

// ------------------------------------------------------------------ argmin (k = 1), warp per row
__global__ void __launch_bounds__(256) k_argmin_exact(const float* __restrict__ dh, int64_t m,
                                                      int64_t n, const float* __restrict__ A,
                                                      const float* __restrict__ B, int D,
                                                      int32_t* __restrict__ out,
                                                      const float* __restrict__ slack) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= m) return;
  const float* d = dh + row * n;
  float mn = FLT_MAX;
  for (int64_t i = lane; i < n; i += 32) mn = fminf(mn, d[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  const unsigned tb = slack ? abs_thr_bits(mn, slack[row]) : thr_bits(mn, D);
  const float* a = A + row * (int64_t)D;
  double best = DBL_MAX;
  int32_t bc = 0x7fffffff;
  for (int64_t i0 = 0; i0 < n; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool c = i < n && __float_as_uint(d[i]) <= tb;
    if (c) {
      const double e = exact_sqdist(a, B + i * D, D);
      if (e < best || (e == best && (int32_t)i < bc)) { best = e; bc = (int32_t)i; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
    if (ob < best || (ob == best && oc < bc)) { best = ob; bc = oc; }
  }
  if (lane == 0) out[row] = bc;
}

void launch_argmin_exact(const float* d_hat, int64_t m, int64_t n, const float* A, const float* B,
                         int D, int32_t* out, int* d_flag, cudaStream_t st, const float* slack) {
  (void)d_flag;
  if (m <= 0) return;
  k_argmin_exact<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(d_hat, m, n, A, B, D, out, slack);
  DADE_CK(cudaGetLastError());
}

// ------------------------------------------------------------------ misc small kernels
__global__ void k_check_finite(const float* __restrict__ X, int64_t n, int* flag, int code) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(X[i])) { atomicExch(flag, code); return; }
}
void launch_check_finite(const float* X, int64_t n, int* flag, cudaStream_t st, int code) {
  if (n <= 0) return;
  k_check_finite<<<1184, 256, 0, st>>>(X, n, flag, code);
  DADE_CK(cudaGetLastError());
}

__global__ void k_gather_rows(const float* __restrict__ X, const int32_t* __restrict__ rows,
                              int64_t m, int D, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / D;
    out[i] = X[(int64_t)rows[r] * D + (i - r * D)];
  }
}
void launch_gather_rows(const float* X, const int32_t* rows, int64_t m, int D, float* out,
                        cudaStream_t st) {
  if (m <= 0) return;
  k_gather_rows<<<1184, 256, 0, st>>>(X, rows, m, D, out);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
