// Exact fp64 distances of up to 32 candidate rows at once (one per lane), for the certification
// step of the exact selections (R20: sum_{j<D} (a_j - b_j)^2 in fp64, sequential, each operation
// rounded separately). Candidate rows are staged through shared memory in 32-dim slices so every
// global load is a coalesced 128-B row segment (lane-per-row loads would touch 32 lines per
// instruction); each lane then accumulates its own row in order j = 0..D-1.
#pragma once
#include <cstdint>

namespace dade {

constexpr int kXbDim = 32;  // dims staged per pass
// per-warp stage (floats, 8-byte aligned): 32 candidate rows x (kXbDim + 1), then the query's
// current slice as kXbDim doubles (read by every lane with one broadcast LDS.64 per dimension)
constexpr int kXbStage = 32 * (kXbDim + 1) + 2 * kXbDim;

// c: this lane's candidate row index (< 0: none); a: the query row (global, broadcast reads);
// nc (warp-uniform, <= 32): candidates are in lanes [0, nc) — only those rows are staged
__device__ __forceinline__ double exact_batch32(const float* __restrict__ a, const float* __restrict__ B, int D,
                                                int32_t c, float* stage, int lane, int nc = 32) {
  double acc = 0.0;
  double* qd = reinterpret_cast<double*>(stage + 32 * (kXbDim + 1));
  // the next slice's 32 loads are issued before the current slice is accumulated
  float v[32];
  auto load = [&](int j0) {
    const int w = min(kXbDim, D - j0);
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 8) {  // only the groups of 8 that hold candidates
      if (i0 < nc) {
#pragma unroll
        for (int i = i0; i < i0 + 8; ++i) {
          const int32_t ci = __shfl_sync(0xffffffffu, c, i);
          v[i] = (ci >= 0 && lane < w) ? __ldg(B + (int64_t)ci * D + j0 + lane) : 0.f;
        }
      }
    }
  };
  load(0);
  for (int j0 = 0; j0 < D; j0 += kXbDim) {
    const int w = min(kXbDim, D - j0);
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 8)
      if (i0 < nc) {
#pragma unroll
        for (int i = i0; i < i0 + 8; ++i) stage[i * (kXbDim + 1) + lane] = v[i];
      }
    qd[lane] = lane < w ? (double)__ldg(a + j0 + lane) : 0.0;
    __syncwarp();
    if (j0 + kXbDim < D) load(j0 + kXbDim);
    if (c >= 0) {
      const float* sr = stage + lane * (kXbDim + 1);
      for (int jj = 0; jj < w; ++jj) {
        const double t = __dsub_rn(qd[jj], (double)sr[jj]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
      }
    }
    __syncwarp();
  }
  return acc;
}

}  // namespace dade
