// a9 shard merge and calibration feature kernels.
#include <cfloat>

#include "dade_internal.h"

namespace dade {

// ------------------------------------------------------------------ a9: merge S local top-K lists
// each GPU returns its local top-K; after the all-gather every rank keeps the
// first K by (dist, id). Keys (dist bits << 32 | id) sort like (dist, id) for dist >= 0.
__global__ void __launch_bounds__(256) k_merge_topk(const int64_t* __restrict__ ids_in,
                                                    const float* __restrict__ d_in, int S, int nq,
                                                    int K, int64_t* __restrict__ ids_out,
                                                    float* __restrict__ d_out, int P) {
  extern __shared__ unsigned long long keys[];
  const int q = blockIdx.x;
  const int tot = S * K;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long k = ~0ull;
    if (i < tot) {
      const int s = i / K, j = i % K;
      const int64_t idx = ((int64_t)s * nq + q) * K + j;
      const int64_t id = ids_in[idx];
      if (id >= 0) k = ((unsigned long long)__float_as_uint(d_in[idx]) << 32) | (uint32_t)id;
    }
    keys[i] = k;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long x = keys[lo], y = keys[hi];
        if ((y < x) == up) { keys[lo] = y; keys[hi] = x; }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    const unsigned long long k = keys[i];
    ids_out[(int64_t)q * K + i] = k == ~0ull ? -1 : (int64_t)(uint32_t)(k & 0xffffffffu);
    d_out[(int64_t)q * K + i] = k == ~0ull ? INFINITY : __uint_as_float((unsigned)(k >> 32));
  }
}

void launch_merge_topk(const int64_t* ids_in, const float* d_in, int S, int nq, int K,
                       int64_t* ids_out, float* d_out, cudaStream_t st) {
  if (nq <= 0) return;
  int P = 1;
  while (P < S * K) P <<= 1;
  const size_t smem = (size_t)P * 8;
  DADE_REQUIRE(smem <= 200 * 1024, DADE_ERR_UNSUPPORTED, "merge: S*K too large");
  DADE_CK(cudaFuncSetAttribute(k_merge_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_merge_topk<<<nq, 256, smem, st>>>(ids_in, d_in, S, nq, K, ids_out, d_out, P);
  DADE_CK(cudaGetLastError());
}

// ------------------------------------------------------------------ a3: calibration features
// out[i * nblk + b] = sum_{j < 16(b+1)} (x~_j - q~_j)^2 in fp64 (sequential), for pair i =
// (query pair_q[i], list-major row pair_row[i]); the BSA-p feature dis'_d at every
// 16-dim prefix d.
__global__ void k_pair_prefix(const float* __restrict__ layout, int64_t n_rows, int D,
                              const float* __restrict__ qrot, const int32_t* __restrict__ pq,
                              const int32_t* __restrict__ pr, int npairs, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int nblk = D / kBlk;
  const float* qv = qrot + (int64_t)pq[i] * D;
  const int64_t row = pr[i];
  double acc = 0.0;
  for (int b = 0; b < nblk; ++b) {
    const float* x = layout + (((int64_t)b * n_rows + row) << 4);
    for (int j = 0; j < kBlk; ++j) {
      const double t = (double)x[j] - (double)qv[b * kBlk + j];
      acc += t * t;
    }
    out[(int64_t)i * nblk + b] = acc;
  }
}

void launch_pair_prefix(const float* layout, int64_t n_rows, int D, const float* qrot,
                        const int32_t* pair_q, const int32_t* pair_row, int npairs, double* out,
                        cudaStream_t st) {
  if (npairs <= 0) return;
  k_pair_prefix<<<(npairs + 127) / 128, 128, 0, st>>>(layout, n_rows, D, qrot, pair_q, pair_row,
                                                      npairs, out);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
