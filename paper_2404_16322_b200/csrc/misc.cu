// a9 shard merge and calibration feature kernels.
#include <algorithm>
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

// ------------------------------------------------------------------ scan query order
__global__ void k_order_hist(const int32_t* __restrict__ probes, int nq, int nprobe, int* __restrict__ cnt) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x)
    atomicAdd(&cnt[probes[(int64_t)q * nprobe]], 1);
}

// exclusive prefix sum of cnt[0, nlist) in place, one CTA of 1024 threads (contiguous chunks)
__global__ void __launch_bounds__(1024) k_order_offsets(int* __restrict__ cnt, int nlist) {
  __shared__ int part[1024];
  const int per = (nlist + 1023) / 1024;
  const int b = threadIdx.x * per, e = min(nlist, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += cnt[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan of the chunk sums
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int i = b; i < e; ++i) {
    const int c = cnt[i];
    cnt[i] = run;
    run += c;
  }
}

__global__ void k_order_scatter(const int32_t* __restrict__ probes, int nq, int nprobe, int* __restrict__ cur,
                                int32_t* __restrict__ order) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x)
    order[atomicAdd(&cur[probes[(int64_t)q * nprobe]], 1)] = q;
}

// longest candidate stream first (DADE_OPT_SCAN_ORDER = 2): bucket of query q = the length of its
// stream (sum of its probed lists' sizes) >> shift, buckets in DESCENDING order
constexpr int kLptBuckets = 1024;
__global__ void k_lpt_key(const int32_t* __restrict__ probes, int nq, int nprobe, const int32_t* __restrict__ off,
                          int shift, int* __restrict__ key, int* __restrict__ cnt) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    int64_t L = 0;
    for (int j = 0; j < nprobe; ++j) {
      const int l = probes[(int64_t)q * nprobe + j];
      L += off[l + 1] - off[l];
    }
    const int64_t bl = L >> shift;
    const int b = bl < kLptBuckets - 1 ? (int)bl : kLptBuckets - 1;
    const int k = kLptBuckets - 1 - b;
    key[q] = k;
    atomicAdd(&cnt[k], 1);
  }
}

__global__ void k_key_scatter(const int* __restrict__ key, int nq, int* __restrict__ cur, int32_t* __restrict__ order) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x)
    order[atomicAdd(&cur[key[q]], 1)] = q;
}

void launch_query_order_lpt(const int32_t* probes, int nq, int nprobe, const int32_t* off, int64_t avg_stream,
                            int* scratch, int32_t* order, cudaStream_t st) {
  if (nq <= 0) return;
  int shift = 0;
  while ((4 * std::max<int64_t>(avg_stream, 1) >> shift) >= kLptBuckets) ++shift;
  int* cnt = scratch;               // kLptBuckets
  int* key = scratch + kLptBuckets; // nq
  DADE_CK(cudaMemsetAsync(cnt, 0, sizeof(int) * kLptBuckets, st));
  const int g = std::min((nq + 255) / 256, 1184);
  k_lpt_key<<<g, 256, 0, st>>>(probes, nq, nprobe, off, shift, key, cnt);
  k_order_offsets<<<1, 1024, 0, st>>>(cnt, kLptBuckets);
  k_key_scatter<<<g, 256, 0, st>>>(key, nq, cnt, order);
  DADE_CK(cudaGetLastError());
}

void launch_query_order(const int32_t* probes, int nq, int nprobe, int nlist, int* cnt, int32_t* order,
                        cudaStream_t st) {
  if (nq <= 0) return;
  DADE_CK(cudaMemsetAsync(cnt, 0, sizeof(int) * nlist, st));
  const int g = std::min((nq + 255) / 256, 1184);
  k_order_hist<<<g, 256, 0, st>>>(probes, nq, nprobe, cnt);
  k_order_offsets<<<1, 1024, 0, st>>>(cnt, nlist);
  k_order_scatter<<<g, 256, 0, st>>>(probes, nq, nprobe, cnt, order);
  DADE_CK(cudaGetLastError());
}

// row-major n x D (list-major rows) -> the dimension-blocked layout: block b is an n x 16 matrix
__global__ void k_to_blocked(const float* __restrict__ X, int64_t n, int D, float* __restrict__ out) {
  const int nb = D / 16;
  const int64_t tot = n * nb * 4;  // 16-B chunks
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / (nb * 4);
    const int r = (int)(i - p * nb * 4), b = r >> 2, c = r & 3;
    const float4 v = reinterpret_cast<const float4*>(X + p * D + b * 16)[c];
    reinterpret_cast<float4*>(out + ((int64_t)b * n + p) * 16)[c] = v;
  }
}

void launch_to_blocked(const float* X, int64_t n, int D, float* out, cudaStream_t st) {
  if (n <= 0) return;
  k_to_blocked<<<1184, 256, 0, st>>>(X, n, D, out);
  DADE_CK(cudaGetLastError());
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

// ------------------------------------------------------------------ NEXT-1 BSA-res helpers
// ‖x~‖² per list-major row of the blocked layout (block b of row r at (b*n + r)*16): fp64 sum in
// block order, stored fp32 (the kernel subtracts fp32 block sums from it)
__global__ void k_row_norms(const float* __restrict__ lay, int64_t n, int nblk, float* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) {
      const float4* v = reinterpret_cast<const float4*>(lay + (((int64_t)b * n + r) << 4));
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 x = __ldg(v + c);
        s += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
      }
    }
    out[r] = (float)s;
  }
}

void launch_row_norms(const float* layout, int64_t n, int D, float* out, cudaStream_t st) {
  if (n <= 0) return;
  k_row_norms<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(layout, n, D / 16, out);
  DADE_CK(cudaGetLastError());
}

// c_s = sum_{i>=d} q_i^2 - m sqrt(4 sum_{i>=d} q_i^2 lam_i), d = s*delta_d, s = 1..D/delta_d-1
// (Alg. 2 / Eq. 3), one thread per (query, step), fp64
__global__ void k_res_consts(const float* __restrict__ qrot, int nq, int D, int delta_d, const double* __restrict__ lam,
                             double m, float* __restrict__ out) {
  const int ns = D / delta_d - 1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nq * ns) return;
  const int64_t q = t / ns;
  const int s = (int)(t % ns) + 1;
  double qr = 0.0, var = 0.0;
  for (int i = s * delta_d; i < D; ++i) {
    const double v = qrot[q * D + i];
    qr += v * v;
    var += v * v * lam[i];
  }
  out[t] = (float)(qr - m * sqrt(4.0 * var));
}

void launch_res_consts(const float* qrot, int nq, int D, int delta_d, const double* lam, double m, float* out,
                       cudaStream_t st) {
  const int64_t tot = (int64_t)nq * (D / delta_d - 1);
  if (tot <= 0) return;
  k_res_consts<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(qrot, nq, D, delta_d, lam, m, out);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
