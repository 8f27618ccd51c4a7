// NEXT-2: the standalone approximation-accuracy scan of Exp-7 / Table III
// (P:L3862-3890): every base vector's distance to the query is ESTIMATED from its first d rotated
// dimensions only, and the K best by the estimate are returned (their recall@K against the exact
// K-NN is the table's metric). Estimators (R27):
//   partial  — P_d = ||x~_{:d} - q~_{:d}||^2 (the "PCA" column in the PCA basis; the "Rand" column
//              is the same estimate after installing a random orthogonal rotation);
//   residual — dis'_d = P_d + ||x~_r||^2 + ||q~_r||^2 (Eq. 2, P:L289-297 with the cross term
//              -2<q_r, x_r> dropped: the BSA-res estimate without its m*sigma margin, which is a
//              per-query constant and does not change the ranking).
//
// B200 mapping: one CTA per query sweeps the blocked layout's first d/16 blocks (contiguous
// 64-B rows, coalesced 16-B loads), fp32 block sums with the scan's fixed association (R21), and
// keeps a shared-memory candidate buffer of (estimate bits << 32 | global id) keys below the
// running threshold; when the buffer fills it is bitonic-sorted and cut to the best K, and the
// threshold becomes the K-th key. Concurrent CTAs sweep the same blocks, so most reads hit L2.
#include <cfloat>
#include <cstdint>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr int kEstThreads = 256;
constexpr int kEstCap = 2048;  // candidate buffer (keys); K <= 256 and a sweep chunk adds <= 1024
constexpr int kEstChunk = 4;   // rows per thread between buffer checks (1,024 per CTA)

__device__ __forceinline__ float est_block(const float* __restrict__ lay, int64_t n, int b, int64_t r,
                                           const float* q, float& sq) {
  const float4* v = reinterpret_cast<const float4*>(lay + (((int64_t)b * n + r) << 4));
  float a[4], s2[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 x = __ldg(v + c);
    const float d0 = x.x - q[4 * c], d1 = x.y - q[4 * c + 1], d2 = x.z - q[4 * c + 2], d3 = x.w - q[4 * c + 3];
    a[c] = fmaf(d3, d3, fmaf(d2, d2, fmaf(d1, d1, d0 * d0)));
    s2[c] = fmaf(x.w, x.w, fmaf(x.z, x.z, fmaf(x.y, x.y, x.x * x.x)));
  }
  sq += (s2[0] + s2[1]) + (s2[2] + s2[3]);
  return (a[0] + a[1]) + (a[2] + a[3]);
}

// ascending bitonic sort of buf[0, kEstCap) (pad with ~0ull)
__device__ void bitonic_sort(unsigned long long* buf) {
  for (int size = 2; size <= kEstCap; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < kEstCap / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long a = buf[lo], b = buf[hi];
        if ((a > b) == up) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kEstThreads) k_estimate_topk(const float* __restrict__ lay, const int32_t* __restrict__ row_id,
                                                               const float* __restrict__ xnorm, int64_t n, int D, int nblk_d,
                                                               const float* __restrict__ qrot, int K, float* __restrict__ out_est,
                                                               int64_t* __restrict__ out_ids) {
  __shared__ unsigned long long buf[kEstCap];
  __shared__ float qs[DADE_EST_MAX_D];
  __shared__ int cnt;
  __shared__ unsigned long long thr;
  __shared__ float qres;
  const int64_t q = blockIdx.x;
  const int d = nblk_d * 16;
  for (int j = threadIdx.x; j < d; j += blockDim.x) qs[j] = qrot[q * D + j];
  if (threadIdx.x == 0) {
    cnt = 0;
    thr = ~0ull;
    float r = 0.f;  // ||q~_r||^2, dims d..D-1, sequential fp32
    for (int j = d; j < D; ++j) r = fmaf(qrot[q * D + j], qrot[q * D + j], r);
    qres = r;
  }
  __syncthreads();
  const bool res = xnorm != nullptr;
  for (int64_t base = 0; base < n; base += (int64_t)kEstThreads * kEstChunk) {
#pragma unroll
    for (int c = 0; c < kEstChunk; ++c) {
      const int64_t r = base + (int64_t)c * kEstThreads + threadIdx.x;
      if (r < n) {
        float e = 0.f, sq = 0.f;
        for (int b = 0; b < nblk_d; ++b) e += est_block(lay, n, b, r, qs + b * 16, sq);
        if (res) e = fmaxf(e + (__ldg(xnorm + r) - sq) + qres, 0.f);
        const unsigned long long key = ((unsigned long long)__float_as_uint(e) << 32) | (uint32_t)__ldg(row_id + r);
        if (key < thr) buf[atomicAdd(&cnt, 1)] = key;
      }
    }
    __syncthreads();
    if (cnt > kEstCap - kEstThreads * kEstChunk) {  // the next chunk might not fit: keep the best K
      for (int i = cnt + threadIdx.x; i < kEstCap; i += blockDim.x) buf[i] = ~0ull;
      bitonic_sort(buf);
      if (threadIdx.x == 0) {
        cnt = K;
        thr = buf[K - 1];
      }
      __syncthreads();
    }
  }
  for (int i = cnt + threadIdx.x; i < kEstCap; i += blockDim.x) buf[i] = ~0ull;
  bitonic_sort(buf);
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const unsigned long long key = buf[i];
    out_ids[q * K + i] = key == ~0ull ? -1 : (int64_t)(uint32_t)(key & 0xffffffffu);
    out_est[q * K + i] = key == ~0ull ? INFINITY : __uint_as_float((unsigned)(key >> 32));
  }
}
}  // namespace

void launch_estimate_topk(const float* layout, const int32_t* row_id, const float* xnorm, int64_t n, int D, int d,
                          const float* qrot, int nq, int K, float* est, int64_t* ids, cudaStream_t st) {
  if (nq <= 0) return;
  k_estimate_topk<<<nq, kEstThreads, 0, st>>>(layout, row_id, xnorm, n, D, d / 16, qrot, K, est, ids);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
