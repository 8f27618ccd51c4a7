// Rotation x~ = R(x - mu) (centring P:L305) with fp64 accumulation, stored fp32.
// Database rows are written straight into the dimension-blocked, list-major layout (a1):
// block b = dims [16b, 16b+16) is an n x 16 fp32 matrix, row p = list-major position p, so one
// Delta_d = 16 step of one IVF list is one contiguous, 64-B-per-row, 128-bit-vectorisable stream.
#include "dade_internal.h"

namespace dade {

// 64 rows x 64 output dims per CTA, 256 threads, 4 x 4 fp64 accumulators per thread.
__global__ void __launch_bounds__(256) k_rotate(const float* __restrict__ X,
                                                const int32_t* __restrict__ src_rows,
                                                int64_t n_out, int D, const double* __restrict__ R,
                                                const double* __restrict__ mu,
                                                float* __restrict__ rm_out,
                                                float* __restrict__ blk_out) {
  __shared__ double Xs[16][64 + 1];
  __shared__ double Rs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * 64;
  const int i0 = blockIdx.y * 64;
  double acc[4][4] = {};
  const int lr = threadIdx.x >> 2, lc = (threadIdx.x & 3) * 4;  // 64 rows x 16 cols loader
  const int64_t p = p0 + lr;
  const int64_t src = (p < n_out) ? (src_rows ? (int64_t)src_rows[p] : p) : -1;
  for (int k0 = 0; k0 < D; k0 += 16) {
    if (src >= 0) {
      const float4 v = *reinterpret_cast<const float4*>(X + src * D + k0 + lc);
      Xs[lc + 0][lr] = (double)v.x - mu[k0 + lc + 0];
      Xs[lc + 1][lr] = (double)v.y - mu[k0 + lc + 1];
      Xs[lc + 2][lr] = (double)v.z - mu[k0 + lc + 2];
      Xs[lc + 3][lr] = (double)v.w - mu[k0 + lc + 3];
    } else {
      Xs[lc + 0][lr] = Xs[lc + 1][lr] = Xs[lc + 2][lr] = Xs[lc + 3][lr] = 0.0;
    }
    const int ri = i0 + lr;  // output dim (row of R)
#pragma unroll
    for (int c = 0; c < 4; ++c) Rs[lc + c][lr] = (ri < D) ? R[(int64_t)ri * D + k0 + lc + c] : 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double xv[4], rv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) { xv[a] = Xs[k][ty * 4 + a]; rv[a] = Rs[k][tx * 4 + a]; }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(xv[a], rv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t pp = p0 + ty * 4 + a;
    if (pp >= n_out) continue;
    const int i = i0 + tx * 4;
    if (i >= D) continue;
    const float4 v = make_float4((float)acc[a][0], (float)acc[a][1], (float)acc[a][2],
                                 (float)acc[a][3]);
    if (rm_out) *reinterpret_cast<float4*>(rm_out + pp * D + i) = v;
    if (blk_out)
      *reinterpret_cast<float4*>(blk_out + (((int64_t)(i >> 4) * n_out + pp) << 4) + (i & 15)) = v;
  }
}

// 128 rows x 64 output dims per CTA, 128 threads, 8 x 8 fp64 accumulators per thread: each k
// step reads 8 + 8 doubles with 128-bit shared loads for 64 DFMA (4x the FMA:load ratio of the
// 4 x 4 tile above). D is a multiple of 16, so output dims never straddle a 16-dim block.
__global__ void __launch_bounds__(128) k_rotate8(const float* __restrict__ X, const int32_t* __restrict__ src_rows,
                                                 int64_t n_out, int D, const double* __restrict__ R,
                                                 const double* __restrict__ mu, float* __restrict__ rm_out,
                                                 float* __restrict__ blk_out) {
  __shared__ __align__(16) double Xs[16][128];
  __shared__ __align__(16) double Rs[16][64];
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // 8 column groups x 16 row groups
  const int64_t p0 = (int64_t)blockIdx.x * 128;
  const int i0 = blockIdx.y * 64;
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < D; k0 += 16) {
    // X tile: 128 rows x 16 dims (one row per thread, four float4 loads), centred in fp64
    {
      const int64_t p = p0 + threadIdx.x;
      const int64_t src = (p < n_out) ? (src_rows ? (int64_t)src_rows[p] : p) : -1;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (src >= 0) v = *reinterpret_cast<const float4*>(X + src * D + k0 + c * 4);
        const int kk = c * 4;
        Xs[kk + 0][threadIdx.x] = src >= 0 ? (double)v.x - mu[k0 + kk + 0] : 0.0;
        Xs[kk + 1][threadIdx.x] = src >= 0 ? (double)v.y - mu[k0 + kk + 1] : 0.0;
        Xs[kk + 2][threadIdx.x] = src >= 0 ? (double)v.z - mu[k0 + kk + 2] : 0.0;
        Xs[kk + 3][threadIdx.x] = src >= 0 ? (double)v.w - mu[k0 + kk + 3] : 0.0;
      }
    }
    // R tile: 64 output dims x 16 input dims (8 doubles per thread)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = threadIdx.x * 8 + e;  // 0..1023
      const int r = idx >> 4, kk = idx & 15;
      Rs[kk][r] = (i0 + r < D) ? R[(int64_t)(i0 + r) * D + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double xv[8], rv[8];
#pragma unroll
      for (int a = 0; a < 8; a += 2) {
        const double2 t = *reinterpret_cast<const double2*>(&Xs[k][ty * 8 + a]);
        xv[a] = t.x; xv[a + 1] = t.y;
        const double2 u = *reinterpret_cast<const double2*>(&Rs[k][tx * 8 + a]);
        rv[a] = u.x; rv[a + 1] = u.y;
      }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fma(xv[a], rv[b], acc[a][b]);
    }
    __syncthreads();
  }
  const int i = i0 + tx * 8;
  if (i >= D) return;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int64_t pp = p0 + ty * 8 + a;
    if (pp >= n_out) continue;
    const float4 v0 = make_float4((float)acc[a][0], (float)acc[a][1], (float)acc[a][2], (float)acc[a][3]);
    const float4 v1 = make_float4((float)acc[a][4], (float)acc[a][5], (float)acc[a][6], (float)acc[a][7]);
    if (rm_out) {
      *reinterpret_cast<float4*>(rm_out + pp * D + i) = v0;
      *reinterpret_cast<float4*>(rm_out + pp * D + i + 4) = v1;
    }
    if (blk_out) {
      float* o = blk_out + (((int64_t)(i >> 4) * n_out + pp) << 4) + (i & 15);
      *reinterpret_cast<float4*>(o) = v0;
      *reinterpret_cast<float4*>(o + 4) = v1;
    }
  }
}

void launch_rotate(const float* X, const int32_t* src_rows, int64_t n_out, int D, const double* R,
                   const double* mu, float* rowmajor_out, float* blocked_out, cudaStream_t st) {
  if (n_out <= 0) return;
  if (n_out >= 65536) {  // database rotation: enough 128-row tiles to fill the machine
    dim3 grid((unsigned)((n_out + 127) / 128), (unsigned)((D + 63) / 64));
    k_rotate8<<<grid, 128, 0, st>>>(X, src_rows, n_out, D, R, mu, rowmajor_out, blocked_out);
  } else {  // query batches: smaller tiles, more CTAs (measured faster at 10k x 128)
    dim3 grid((unsigned)((n_out + 63) / 64), (unsigned)((D + 63) / 64));
    k_rotate<<<grid, 256, 0, st>>>(X, src_rows, n_out, D, R, mu, rowmajor_out, blocked_out);
  }
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
