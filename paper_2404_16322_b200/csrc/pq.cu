// NEXT-3 BSA-q (§V-B): product-quantization kernels — code assignment (OPQ training
// and the encoding of the rotated base), reconstruction errors, the calibration features (ADC
// distance, distance to the quantized centroid) and the fp64 cross-product of OPQ's Procrustes
// step. Codes: 256 codewords per subspace (nbits = 8), subspace j = dims [j*ds, (j+1)*ds).
// Exactness (R30): a code is the argmin of the fp64 SEQUENTIAL sum over the subspace's dims of
// (x_i - c_i)^2 (products and sums rounded separately, no FMA contraction), ties to the lower code.
#include <algorithm>

#include "dade_internal.h"

namespace dade {

namespace {
// x~ of row p, dim d: blocked layout (block d/16 is an n x 16 matrix) or row-major n x D
template <bool BLOCKED>
__device__ __forceinline__ float xval(const float* X, int64_t n, int D, int64_t p, int d) {
  return BLOCKED ? X[(((int64_t)(d >> 4) * n + p) << 4) + (d & 15)] : X[p * D + d];
}

// grid (row blocks, m): thread = row, block = one subspace whose codebook sits in shared memory
template <bool BLOCKED>
__global__ void __launch_bounds__(256) k_pq_assign(const float* __restrict__ X, int64_t n, int D, int ds,
                                                   const float* __restrict__ C, uint8_t* __restrict__ codes,
                                                   int stride) {
  extern __shared__ float cb[];  // 256 x ds
  const int j = blockIdx.y;
  for (int i = threadIdx.x; i < 256 * ds; i += blockDim.x) cb[i] = C[(int64_t)j * 256 * ds + i];
  __syncthreads();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double x[32];
#pragma unroll 4
  for (int i = 0; i < ds; ++i) x[i] = (double)xval<BLOCKED>(X, n, D, p, j * ds + i);
  double best = 0.0;
  int arg = 0;
  for (int c = 0; c < 256; ++c) {
    double acc = 0.0;
    for (int i = 0; i < ds; ++i) {
      const double t = __dsub_rn(x[i], (double)cb[c * ds + i]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    if (c == 0 || acc < best) {  // strict: the lower code wins ties
      best = acc;
      arg = c;
    }
  }
  codes[p * stride + j] = (uint8_t)arg;
}

// reconstruction error e = ||x - x^||^2 (fp64, subspaces in order), stored fp32 at byte offset `eo`
// of the code row
__global__ void k_pq_err(const float* __restrict__ layout, int64_t n, int D, int m, int ds,
                         const float* __restrict__ C, uint8_t* __restrict__ codes, int stride, int eo) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint8_t* row = codes + p * stride;
  double e = 0.0;
  for (int j = 0; j < m; ++j) {
    const float* c = C + ((int64_t)j * 256 + row[j]) * ds;
    for (int i = 0; i < ds; ++i) {
      const double t = __dsub_rn((double)xval<true>(layout, n, D, p, j * ds + i), (double)c[i]);
      e = __dadd_rn(e, __dmul_rn(t, t));
    }
  }
  *reinterpret_cast<float*>(row + eo) = (float)e;
}

// calibration features of pair i (query pq[i], list-major row pr[i]): the ADC distance
// sum_j ||q~_j - C_j[code_j]||^2 (fp64) and the stored reconstruction error
__global__ void k_pq_pair_feat(const uint8_t* __restrict__ codes, int stride, int eo, int m, int ds,
                               const float* __restrict__ C, const float* __restrict__ qrot, int D,
                               const int32_t* __restrict__ pq, const int32_t* __restrict__ pr, int npairs,
                               double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const uint8_t* row = codes + (int64_t)pr[i] * stride;
  const float* q = qrot + (int64_t)pq[i] * D;
  double a = 0.0;
  for (int j = 0; j < m; ++j) {
    const float* c = C + ((int64_t)j * 256 + row[j]) * ds;
    for (int t = 0; t < ds; ++t) {
      const double d = __dsub_rn((double)q[j * ds + t], (double)c[t]);
      a = __dadd_rn(a, __dmul_rn(d, d));
    }
  }
  out[2 * (int64_t)i] = a;
  out[2 * (int64_t)i + 1] = (double)*reinterpret_cast<const float*>(row + eo);
}

// M += sum over rows r of (x_r - mu)^T y_r (fp64; D x D), y_r = the reconstruction of code row r:
// OPQ's Procrustes cross-product. 32 x 32 output tiles, rows split over grid.z.
__global__ void __launch_bounds__(256) k_pq_cross(const float* __restrict__ X, const double* __restrict__ mu,
                                                  int64_t n, int D, int ds, const float* __restrict__ C,
                                                  const uint8_t* __restrict__ codes, int m,
                                                  double* __restrict__ M, int64_t rows_per) {
  __shared__ double xs[32][33];
  __shared__ double ys[32][33];
  const int a0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int64_t r0 = (int64_t)blockIdx.z * rows_per, r1 = min(n, r0 + rows_per);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps: each owns 4 output rows
  double acc[4] = {0, 0, 0, 0};
  for (int64_t rb = r0; rb < r1; rb += 32) {
    for (int k = ty; k < 32; k += 8) {
      const int64_t r = rb + k;
      const int a = a0 + tx, b = b0 + tx;
      xs[k][tx] = (r < r1 && a < D) ? (double)X[r * D + a] - mu[a] : 0.0;
      double y = 0.0;
      if (r < r1 && b < D) {
        const int j = b / ds;
        y = (double)C[((int64_t)j * 256 + codes[r * m + j]) * ds + (b - j * ds)];
      }
      ys[k][tx] = y;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      const double y = ys[k][tx];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += xs[k][ty * 4 + u] * y;
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int a = a0 + ty * 4 + u, b = b0 + tx;
    if (a < D && b < D) atomicAdd(&M[(int64_t)a * D + b], acc[u]);
  }
}
}  // namespace

void launch_pq_assign(const float* X, bool blocked, int64_t n, int D, int m, const float* C, uint8_t* codes,
                      int stride, cudaStream_t st) {
  if (n <= 0) return;
  const int ds = D / m;
  DADE_REQUIRE(ds <= 32, DADE_ERR_UNSUPPORTED, "pq: subspace wider than 32 dims");
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)m);
  const size_t smem = (size_t)256 * ds * 4;
  if (blocked) {
    DADE_CK(cudaFuncSetAttribute(k_pq_assign<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_pq_assign<true><<<grid, 256, smem, st>>>(X, n, D, ds, C, codes, stride);
  } else {
    DADE_CK(cudaFuncSetAttribute(k_pq_assign<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_pq_assign<false><<<grid, 256, smem, st>>>(X, n, D, ds, C, codes, stride);
  }
  DADE_CK(cudaGetLastError());
}

void launch_pq_err(const float* layout, int64_t n, int D, int m, const float* C, uint8_t* codes, int stride, int eo,
                   cudaStream_t st) {
  if (n <= 0) return;
  k_pq_err<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(layout, n, D, m, D / m, C, codes, stride, eo);
  DADE_CK(cudaGetLastError());
}

void launch_pq_pair_feat(const uint8_t* codes, int stride, int eo, int m, int D, const float* C, const float* qrot,
                         const int32_t* pq, const int32_t* pr, int npairs, double* out, cudaStream_t st) {
  if (npairs <= 0) return;
  k_pq_pair_feat<<<(npairs + 255) / 256, 256, 0, st>>>(codes, stride, eo, m, D / m, C, qrot, D, pq, pr, npairs, out);
  DADE_CK(cudaGetLastError());
}

void launch_pq_cross(const float* X, const double* mu, int64_t n, int D, int m, const float* C, const uint8_t* codes,
                     double* M, cudaStream_t st) {
  DADE_CK(cudaMemsetAsync(M, 0, sizeof(double) * D * D, st));
  if (n <= 0) return;
  const int t = (D + 31) / 32;
  const int64_t rows_per = std::max<int64_t>(256, (n + 63) / 64);
  dim3 grid((unsigned)t, (unsigned)t, (unsigned)((n + rows_per - 1) / rows_per));
  k_pq_cross<<<grid, 256, 0, st>>>(X, mu, n, D, D / m, C, codes, m, M, rows_per);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
