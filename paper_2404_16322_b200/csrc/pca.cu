// fp64 moments of the strided PCA sample (Theorem 1; sample P:L3105 / R17;
// covariance divisor P:L4074). Deterministic: fixed-order partial sums, no atomics.
#include <algorithm>

#include "dade_internal.h"

namespace dade {

// sampled global ids g_k = floor(k * n_total / ns); rank owns [id_base, id_base + n)
static void owned_k_range(int64_t n, int64_t id_base, int64_t n_total, int64_t ns, int64_t* klo,
                          int64_t* khi) {
  auto ceil_div = [](__int128 a, __int128 b) { return (int64_t)((a + b - 1) / b); };
  *klo = ceil_div((__int128)id_base * ns, n_total);
  *khi = ceil_div((__int128)(id_base + n) * ns, n_total);
  if (*khi > ns) *khi = ns;
}

__device__ __forceinline__ int64_t sample_row(int64_t k, int64_t n_total, int64_t ns,
                                              int64_t id_base) {
  // floor(k n_total / ns): 64-bit when the product fits (k < ns <= 2^31-ish and n_total < 2^32
  // in every practical case), 128-bit otherwise (the 128-bit division is ~10x slower)
  if (k < ((int64_t)1 << 31) && n_total < ((int64_t)1 << 32))
    return (int64_t)((uint64_t)k * (uint64_t)n_total / (uint64_t)ns) - id_base;
  return (int64_t)(((__int128)k * n_total) / ns) - id_base;
}

constexpr int kSumRows = 256;  // sample rows per partial (a CTA each; partials added in chunk order)

// partial[c][j] = sum over sample chunk c (kSumRows consecutive k) of x_j, sequential in k
__global__ void k_pca_sum(const float* __restrict__ X, int64_t klo, int64_t khi, int64_t n_total,
                          int64_t ns, int64_t id_base, int D, double* __restrict__ partial) {
  const int64_t c = blockIdx.x;
  const int64_t k0 = klo + c * kSumRows, k1 = min(khi, k0 + kSumRows);
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    double s = 0.0;
    for (int64_t k = k0; k < k1; ++k) s += (double)X[sample_row(k, n_total, ns, id_base) * D + j];
    partial[c * D + j] = s;
  }
}

__global__ void k_reduce_partials(const double* __restrict__ partial, int64_t nchunks, int64_t len,
                                  double* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len;
       j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t c = 0; c < nchunks; ++c) s += partial[c * len + j];
    out[j] = s;
  }
}

void launch_pca_sum(const float* X, int64_t n, int64_t id_base, int64_t n_total, int64_t ns,
                    int D, double* sum_dev, int64_t* cnt_host, cudaStream_t st) {
  int64_t klo, khi;
  owned_k_range(n, id_base, n_total, ns, &klo, &khi);
  const int64_t cnt = khi > klo ? khi - klo : 0;
  *cnt_host = cnt;
  const int64_t nch = (cnt + kSumRows - 1) / kSumRows;
  if (nch == 0) {
    DADE_CK(cudaMemsetAsync(sum_dev, 0, sizeof(double) * D, st));
    return;
  }
  double* partial = nullptr;
  DADE_CK(cudaMallocAsync(&partial, sizeof(double) * nch * D, st));
  k_pca_sum<<<(unsigned)nch, 128, 0, st>>>(X, klo, khi, n_total, ns, id_base, D, partial);
  DADE_CK(cudaGetLastError());
  k_reduce_partials<<<(D + 127) / 128, 128, 0, st>>>(partial, nch, D, sum_dev);
  DADE_CK(cudaGetLastError());
  DADE_CK(cudaFreeAsync(partial, st));
}

constexpr int kCovRows = 8192;  // sample rows per split-K chunk
constexpr int kCovT = 32;       // output tile

// partial[c][a][b] (upper tiles only; mirrored later) = sum_k (x_a - mu_a)(x_b - mu_b), k in chunk c
__global__ void __launch_bounds__(256) k_pca_cov(const float* __restrict__ X, int64_t klo,
                                                 int64_t khi, int64_t n_total, int64_t ns,
                                                 int64_t id_base, int D,
                                                 const double* __restrict__ mu,
                                                 double* __restrict__ partial) {
  const int ta = blockIdx.y, tb = blockIdx.x;
  if (tb < ta) return;
  const int64_t c = blockIdx.z;
  __shared__ double Ya[32][kCovT + 1], Yb[32][kCovT + 1];
  const int tid = threadIdx.x;
  // each thread owns 4 outputs: (a = tid/8, b = (tid%8)*4 .. +4)
  const int oa = tid >> 3, ob = (tid & 7) * 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t k0 = klo + c * kCovRows, k1 = min(khi, k0 + kCovRows);
  for (int64_t kb = k0; kb < k1; kb += 32) {
    // load 32 sample rows x 32 cols for both column ranges
    for (int i = tid; i < 32 * kCovT; i += 256) {
      const int r = i / kCovT, col = i % kCovT;
      const int64_t k = kb + r;
      double va = 0.0, vb = 0.0;
      if (k < k1) {
        const int64_t row = sample_row(k, n_total, ns, id_base);
        const int ja = ta * kCovT + col, jb = tb * kCovT + col;
        if (ja < D) va = (double)X[row * D + ja] - mu[ja];
        if (jb < D) vb = (double)X[row * D + jb] - mu[jb];
      }
      Ya[r][col] = va;
      Yb[r][col] = vb;
    }
    __syncthreads();
    const int rmax = (int)min((int64_t)32, k1 - kb);
    for (int r = 0; r < rmax; ++r) {
      const double a = Ya[r][oa];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(a, Yb[r][ob + q], acc[q]);
    }
    __syncthreads();
  }
  const int ga = ta * kCovT + oa;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gb = tb * kCovT + ob + q;
    if (ga < D && gb < D) partial[(c * D + ga) * D + gb] = acc[q];
  }
}

__global__ void k_mirror(double* __restrict__ cov, int D) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)D * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(i / D), b = (int)(i % D);
    if ((a / kCovT) > (b / kCovT)) cov[i] = cov[(int64_t)b * D + a];
  }
}

int g_pca_tc = 1;  // covariance on the int8 tensor cores (Gram mode of rotate.cu); 0: fp64 CUDA cores
constexpr int64_t kGramK = 16384;  // sample rows per Gram launch (exact int32 levels up to 16,384)

static bool pca_tc(int D) { return g_pca_tc && D % 16 == 0 && D <= kRotMaxD; }

int64_t pca_cov_scratch_elems(int64_t n_owned, int D) {
  if (pca_tc(D)) return (int64_t)D * std::min<int64_t>(kGramK, (n_owned + 63) / 64 * 64);
  return ((n_owned + kCovRows - 1) / kCovRows) * (int64_t)D * D;
}

// Yt[a][kk] = x_a - mu_a (fp64) of sampled row kc0 + kk, kk < cnt; 0 for kk in [cnt, K):
// the transposed, centred sample chunk, 32 x 32 tiles through shared memory
__global__ void k_cov_gather_t(const float* __restrict__ X, int64_t kc0, int64_t cnt, int64_t K, int64_t n_total,
                               int64_t ns, int64_t id_base, int D, const double* __restrict__ mu,
                               double* __restrict__ Yt, unsigned long long* __restrict__ rmax) {
  __shared__ double t[32][33];
  const int64_t kb = (int64_t)blockIdx.x * 32;
  const int ab = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t kk = kb + i;
    const int a = ab + threadIdx.x;
    double v = 0.0;
    if (kk < cnt && a < D) v = (double)X[sample_row(kc0 + kk, n_total, ns, id_base) * D + a] - mu[a];
    t[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // one warp per dim: row maxima for the slices
    const int a = ab + i;
    const int64_t kk = kb + threadIdx.x;
    const double v = t[threadIdx.x][i];
    if (a < D && kk < K) Yt[(int64_t)a * K + kk] = v;
    double m = fabs(v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0 && a < D && m > 0.0) atomicMax(rmax + a, (unsigned long long)__double_as_longlong(m));
  }
}

// Sigma_sum = sum over the rank's sampled rows of (x - mu)(x - mu)^T in fp64. Tensor-core path:
// chunks of <= 16,384 sampled rows, each transposed and centred in fp64, then one Gram launch on
// the int8 tensor cores (rotate.cu, exact int32 levels, error bound of R36) accumulating into the
// fp64 result; the chunk sums are added in chunk order. CUDA-core path (g_pca_tc = 0): fp64 FMA
// tiles with split-K partials.
void launch_pca_cov(const float* X, int64_t n, int64_t id_base, int64_t n_total, int64_t ns, int D,
                    const double* mean_dev, double* cov_dev, double* scratch,
                    int64_t scratch_elems, cudaStream_t st) {
  if (pca_tc(D)) {
    int64_t klo, khi;
    owned_k_range(n, id_base, n_total, ns, &klo, &khi);
    const int64_t cnt = khi > klo ? khi - klo : 0;
    DADE_CK(cudaMemsetAsync(cov_dev, 0, sizeof(double) * D * D, st));
    if (cnt == 0) return;
    RotWs wa;
    RotOp wb;
    DBuf<unsigned long long> rmax;
    rmax.reserve((size_t)D);
    for (int64_t c0 = 0; c0 < cnt; c0 += kGramK) {
      const int64_t c = std::min(kGramK, cnt - c0), K = (c + 63) / 64 * 64;
      DADE_REQUIRE((int64_t)D * K <= scratch_elems, DADE_ERR_OOM, "pca scratch too small");
      DADE_CK(cudaMemsetAsync(rmax.p, 0, sizeof(unsigned long long) * D, st));
      dim3 grid((unsigned)(K / 32), (unsigned)((D + 31) / 32));
      k_cov_gather_t<<<grid, dim3(32, 8), 0, st>>>(X, klo + c0, c, K, n_total, ns, id_base, D, mean_dev, scratch,
                                                    rmax.p);
      DADE_CK(cudaGetLastError());
      launch_gram_i8(scratch, D, K, rmax.p, wa, wb, cov_dev, st);
    }
    DADE_CK(cudaStreamSynchronize(st));  // the slice scratch (wa, wb) is freed on return
    return;
  }
  int64_t klo, khi;
  owned_k_range(n, id_base, n_total, ns, &klo, &khi);
  const int64_t cnt = khi > klo ? khi - klo : 0;
  const int64_t nch = (cnt + kCovRows - 1) / kCovRows;
  if (nch == 0) {
    DADE_CK(cudaMemsetAsync(cov_dev, 0, sizeof(double) * D * D, st));
    return;
  }
  DADE_REQUIRE(nch * (int64_t)D * D <= scratch_elems, DADE_ERR_OOM, "pca scratch too small");
  DADE_CK(cudaMemsetAsync(scratch, 0, sizeof(double) * nch * D * D, st));
  const int nt = (D + kCovT - 1) / kCovT;
  dim3 grid(nt, nt, (unsigned)nch);
  k_pca_cov<<<grid, 256, 0, st>>>(X, klo, khi, n_total, ns, id_base, D, mean_dev, scratch);
  DADE_CK(cudaGetLastError());
  k_reduce_partials<<<256, 256, 0, st>>>(scratch, nch, (int64_t)D * D, cov_dev);
  DADE_CK(cudaGetLastError());
  k_mirror<<<256, 256, 0, st>>>(cov_dev, D);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
