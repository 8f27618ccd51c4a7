// a7 stage 1, list-major: the first step's partial distances of every (query, candidate) pair,
// computed once per probed LIST for all queries that probe it, before the scan.
//
// Stage 1 of the progressive scan (Alg. 2's first iteration) reads the first step
// (Δd dims = 64 B per 16 dims) of EVERY candidate of a query's stream — the largest share of the
// scan's bytes (C4: ~3.1 of 5.1 GB). Queries that probe the same list read the same rows: with
// nq·nprobe / nlist ≈ 5 (C4) to 20 (C2) queries per list, reading each list's first-step rows
// once into shared memory and evaluating them against every query that probes it moves a
// fraction of the bytes; the scan then reads one fp32 partial distance per candidate (4 B)
// instead of the rows. The values are the same fp32 block sums the scan's gather rounds form
// (block_sum: fixed association, R21), added in block order, so every decision is a
// deterministic function of the inputs as before.
//
// Buffers: p1[base[q] + t] = P_{16 DD}(q, candidate t of q's stream), streams as in the scan
// (probed lists in probe order, rows in list order); base = exclusive prefix of the stream
// lengths.
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
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// the scan's block_sum (scan.cu): 4 packed accumulators, ((a0 + a1) + (a2 + a3)), then lo + hi
__device__ __forceinline__ float block_sum(const unsigned long long (&x)[8], const float* q) {
  const ulonglong2* qq = reinterpret_cast<const ulonglong2*>(q);
  unsigned long long a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const ulonglong2 qc = qq[c];
    const unsigned long long t0 = sub2(x[2 * c], qc.x);
    const unsigned long long t1 = sub2(x[2 * c + 1], qc.y);
    a[c] = fma2(t1, t1, 0ull);
    a[c] = fma2(t0, t0, a[c]);
  }
  unsigned long long s2 = add2(add2(a[0], a[1]), add2(a[2], a[3]));
  const float2 s = *reinterpret_cast<float2*>(&s2);
  return s.x + s.y;
}

// per query: its stream length; per list: how many queries probe it
__global__ void k_p1_count(const int32_t* __restrict__ probes, int nq, int nprobe, const int32_t* __restrict__ off,
                           int* __restrict__ qlen, int* __restrict__ lcnt) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    int L = 0;
    for (int j = 0; j < nprobe; ++j) {
      const int l = probes[(int64_t)q * nprobe + j];
      L += off[l + 1] - off[l];
      atomicAdd(&lcnt[l], 1);
    }
    qlen[q] = L;
  }
}

// exclusive prefix sum of v[0, len) in place (one CTA of 1024 threads, contiguous chunks)
__global__ void __launch_bounds__(1024) k_p1_excl(int* __restrict__ v, int len, long long* __restrict__ total) {
  __shared__ int part[1024];
  const int per = (len + 1023) / 1024;
  const int b = threadIdx.x * per, e = min(len, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int t = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int i = b; i < e; ++i) {
    const int c = v[i];
    v[i] = run;
    run += c;
  }
  if (total && threadIdx.x == 1023) *total = (long long)run;
}

// pairs grouped by list: pq[pos] = q, po[pos] = p1 offset of the list's first row in q's stream
__global__ void k_p1_pairs(const int32_t* __restrict__ probes, int nq, int nprobe, const int32_t* __restrict__ off,
                           const int* __restrict__ qbase, int* __restrict__ lcur, int32_t* __restrict__ pq,
                           int32_t* __restrict__ po) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    int o = qbase[q];
    for (int j = 0; j < nprobe; ++j) {
      const int l = probes[(int64_t)q * nprobe + j];
      const int pos = atomicAdd(&lcur[l], 1);
      pq[pos] = q;
      po[pos] = o;
      o += off[l + 1] - off[l];
    }
  }
}

constexpr int kP1Rows = 256;  // list rows per pass (one per thread)
constexpr int kP1Pairs = 64;  // (query, list) pairs staged per batch

// one CTA per list: its first-step rows (DD blocks) and a batch of the queries that probe it are
// staged in shared memory once; then every thread takes one row and walks the batch's queries
// (no barrier inside the walk), writing one fp32 partial distance per (query, row)
template <int DD>
__global__ void __launch_bounds__(kP1Rows) k_p1_fill(const float* __restrict__ layout, int64_t n,
                                                     const int32_t* __restrict__ off, const int* __restrict__ lstart,
                                                     const int32_t* __restrict__ pq, const int32_t* __restrict__ po,
                                                     const float* __restrict__ qrot, int D, float* __restrict__ p1,
                                                     const long long* __restrict__ total, long long cap) {
  constexpr int R = DD == 4 ? kP1Rows / 2 : kP1Rows;  // rows per pass (<= 32 KB of rows)
  constexpr int PB = DD == 4 ? kP1Pairs / 2 : kP1Pairs;  // pairs per batch (<= 8 KB of queries)
  __shared__ __align__(16) float xs[DD][R][16];
  __shared__ __align__(16) float qsh[PB][DD * 16];
  __shared__ int osh[PB];
  const int l = blockIdx.x;
  const int s0 = off[l], len = off[l + 1] - s0;
  const int pb = l ? lstart[l - 1] : 0, pe = lstart[l];  // (lstart holds each list's END after the scatter)
  if (len == 0 || pb == pe || *total > cap) return;  // (over capacity: the scan reads the rows)
  const int t = threadIdx.x;
  for (int b0 = pb; b0 < pe; b0 += PB) {
    const int nb = min(PB, pe - b0);
    __syncthreads();
    for (int i = t; i < nb * DD * 4; i += kP1Rows) {  // the batch's query blocks, 16 B each
      const int j = i / (DD * 4), c = i - j * (DD * 4);
      *reinterpret_cast<float4*>(&qsh[j][c * 4]) =
          __ldg(reinterpret_cast<const float4*>(qrot + (int64_t)pq[b0 + j] * D) + c);
    }
    for (int j = t; j < nb; j += kP1Rows) osh[j] = po[b0 + j];
    for (int r0 = 0; r0 < len; r0 += R) {
      const int nr = min(R, len - r0);
      __syncthreads();
      for (int i = t; i < DD * nr * 4; i += kP1Rows) {  // 16-B chunks, coalesced per block plane
        const int bb = i / (nr * 4), rem = i - bb * nr * 4, r = rem >> 2, c = rem & 3;
        *reinterpret_cast<float4*>(&xs[bb][r][c * 4]) =
            __ldg(reinterpret_cast<const float4*>(layout + (((int64_t)bb * n + s0 + r0 + r) << 4)) + c);
      }
      __syncthreads();
      if (t < nr) {
        unsigned long long x[DD][8];
#pragma unroll
        for (int bb = 0; bb < DD; ++bb) {
          const ulonglong2* xr = reinterpret_cast<const ulonglong2*>(&xs[bb][t][0]);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const ulonglong2 v = xr[c];
            x[bb][2 * c] = v.x;
            x[bb][2 * c + 1] = v.y;
          }
        }
        for (int j = 0; j < nb; ++j) {
          float s = 0.f;
#pragma unroll
          for (int bb = 0; bb < DD; ++bb) s += block_sum(x[bb], &qsh[j][bb * 16]);
          DADE_DCHECK((int64_t)osh[j] + r0 + t < *total);
          p1[(int64_t)osh[j] + r0 + t] = s;
        }
      }
    }
  }
}
}  // namespace

size_t p1_scratch_ints(int nq, int nprobe, int nlist) {
  return (size_t)nq + nlist + 2 * (size_t)nq * nprobe + 4;
}

// p1 holds p1_cap floats; the streams' total length lands in *total (device) and, when it
// exceeds p1_cap, nothing is written and the scan (which checks the same total) reads the rows
void p1_launch(const float* layout, int64_t n, const int32_t* off, int nlist, const int32_t* probes, int nq,
               int nprobe, const float* qrot, int D, int dd_unit, int* scratch, int* qbase_out, float* p1,
               int64_t p1_cap, long long* total, cudaStream_t st) {
  if (nq <= 0) return;
  int* lcnt = scratch;                       // nlist
  int32_t* pq = scratch + nlist;             // nq * nprobe
  int32_t* po = pq + (size_t)nq * nprobe;    // nq * nprobe
  int* qlen = qbase_out;                     // nq (becomes the exclusive prefix)
  DADE_CK(cudaMemsetAsync(lcnt, 0, sizeof(int) * nlist, st));
  const int g = std::min((nq + 255) / 256, 1184);
  k_p1_count<<<g, 256, 0, st>>>(probes, nq, nprobe, off, qlen, lcnt);
  k_p1_excl<<<1, 1024, 0, st>>>(qlen, nq, total);
  k_p1_excl<<<1, 1024, 0, st>>>(lcnt, nlist, nullptr);
  k_p1_pairs<<<g, 256, 0, st>>>(probes, nq, nprobe, off, qlen, lcnt, pq, po);
  DADE_CK(cudaGetLastError());
  switch (dd_unit) {
    case 4: k_p1_fill<4><<<nlist, kP1Rows, 0, st>>>(layout, n, off, lcnt, pq, po, qrot, D, p1, total, p1_cap); break;
    case 2: k_p1_fill<2><<<nlist, kP1Rows, 0, st>>>(layout, n, off, lcnt, pq, po, qrot, D, p1, total, p1_cap); break;
    default: k_p1_fill<1><<<nlist, kP1Rows, 0, st>>>(layout, n, off, lcnt, pq, po, qrot, D, p1, total, p1_cap); break;
  }
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
