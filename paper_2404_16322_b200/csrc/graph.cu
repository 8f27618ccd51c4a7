// NEXT-4: graph refinement with the DCO — HNSW's base-layer best-first search whose
// distance computations are the progressive, classifier-pruned ones of the scan (P:L535-541,
// P:L582-586). Readings R33-R35: a fixed-degree graph of M0 neighbours per node
// (HNSW's neighbour-selection heuristic over each node's nearest candidates), the entry point
// nearest to the base mean, a result queue W of size ef, and tau = max W frozen while one node is
// expanded.
//
// B200 mapping: one warp per query (CTA = 4 queries), persistent over an atomic query counter.
// An expansion hands the M0 <= 32 neighbours of the popped node to the 32 lanes: each lane tests
// its neighbour against a global per-warp-slot visited bitmap (atomicOr), then accumulates its
// squared distance block by block from the dimension-blocked layout (two 256-bit loads per 16
// dims, fp32 block sums added in block order — the scan's association, R21), testing the
// classifier at every step boundary and stopping at the first prune. W (ef keys) and the
// candidate queue C (keys + layout positions) are sorted arrays in shared memory; survivors are
// sorted by (dist, id) in registers (warp bitonic sort) and inserted in that order.
#include <cfloat>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr unsigned long long kInf = ~0ull;
constexpr int kGW = 4;  // warps (queries) per CTA

__device__ __forceinline__ unsigned long long gkey(float d, uint32_t id) {
  return ((unsigned long long)__float_as_uint(d) << 32) | id;
}
__device__ __forceinline__ float kdist(unsigned long long k) { return __uint_as_float((unsigned)(k >> 32)); }

__device__ __forceinline__ float block_sq_diff(const float* __restrict__ row, const float* q) {
  const float4* r4 = reinterpret_cast<const float4*>(row);
  float a[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 v = __ldg(r4 + c);
    const float t0 = v.x - q[4 * c], t1 = v.y - q[4 * c + 1], t2 = v.z - q[4 * c + 2], t3 = v.w - q[4 * c + 3];
    a[c] = fmaf(t1, t1, t0 * t0) + fmaf(t3, t3, t2 * t2);
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

// warp bitonic sort of one (key, val) per lane, ascending by key
__device__ __forceinline__ void warp_sort(unsigned long long& k, int& v, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k, stride);
      const int ov = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      const bool take = lower == up ? ok < k : ok > k;
      if (take) { k = ok; v = ov; }
    }
}
}  // namespace

__global__ void __launch_bounds__(kGW * 32) k_graph_search(const __grid_constant__ GraphParams p) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int D = p.D, ef = p.ef, capC = ef + 64;
  const size_t per = (size_t)D * 4 + (size_t)ef * 8 + (size_t)capC * 12 + 16;
  unsigned char* base = sm + w * ((per + 15) & ~(size_t)15);
  float* qs = reinterpret_cast<float*>(base);
  unsigned long long* W = reinterpret_cast<unsigned long long*>(qs + D);
  unsigned long long* Ck = W + ef;
  int* Cp = reinterpret_cast<int*>(Ck + capC);
  const int slot = blockIdx.x * kGW + w;
  const int nwords = (int)((p.n + 31) >> 5);
  unsigned* vis = p.visited + (size_t)slot * nwords;
  int32_t* vl = p.vlist + (size_t)slot * p.vcap;
  const int nblk = D >> 4;
  const bool stats = p.counters != nullptr;
  unsigned long long c_tested = 0, c_surv = 0, c_exp = 0;

  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(p.work, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= p.nq) break;
    const int64_t q = qi;
    for (int j = lane; j < D; j += 32) qs[j] = p.qrot[q * D + j];
    __syncwarp();
    int nvis = 1;  // visited positions recorded in vl (beyond vcap the whole bitmap is wiped)
    int wn = 1, ch = 0, cn = 1;  // W holds wn keys; C holds cn entries at [ch, ch + cn)
    if (lane == 0) {  // entry point: exact distance (dims = D)
      int e = p.entry;
      if (p.eprobes)
        for (int j = 0; j < p.eprobe; ++j) {
          const int l = p.eprobes[q * p.eprobe + j];
          const int o0 = __ldg(p.off + l), o1 = __ldg(p.off + l + 1);
          if (o1 > o0) { e = o0; break; }
        }
      float phi = 0.f;
      for (int b = 0; b < nblk; ++b) phi += block_sq_diff(p.layout + (((int64_t)b * p.n + e) << 4), qs + b * 16);
      const unsigned long long k = gkey(phi, (uint32_t)__ldg(p.row_id + e));
      W[0] = k;
      Ck[0] = k;
      Cp[0] = e;
      atomicOr(vis + (e >> 5), 1u << (e & 31));
      vl[0] = e;
      if (p.dlog) {
        const unsigned long long s = atomicAdd(p.dlog_n, 1ull);
        if ((int64_t)s < p.dlog_cap) {
          p.dlog[3 * s] = (int32_t)q; p.dlog[3 * s + 1] = (int32_t)(k & 0xffffffffu); p.dlog[3 * s + 2] = D;
        }
      }
    }
    c_tested += 1;
    c_surv += 1;
    __syncwarp();
    while (cn > 0) {
      const unsigned long long ck = Ck[ch];
      const int cpos = Cp[ch];
      ++ch;  // pop the nearest candidate
      --cn;
      if (wn >= ef && kdist(ck) > kdist(W[ef - 1])) break;
      ++c_exp;
      const float tau = wn >= ef ? kdist(W[ef - 1]) : INFINITY;  // frozen for this expansion (R34)
      // this lane's neighbour of the popped node
      int u = lane < p.M0 ? __ldg(p.adj + (int64_t)cpos * p.M0 + lane) : -1;
      if (u >= 0) {
        const unsigned bit = 1u << (u & 31);
        const unsigned old = atomicOr(vis + (u >> 5), bit);
        if (old & bit) u = -1;
      }
      const unsigned newm = __ballot_sync(0xffffffffu, u >= 0);
      if (newm == 0) continue;
      {  // record the newly visited positions (to clear the bitmap after the query)
        const int r = nvis + __popc(newm & ((1u << lane) - 1));
        if (u >= 0 && r < p.vcap) vl[r] = u;
        nvis += __popc(newm);
      }
      // progressive distance with the classifier at the step boundaries
      float phi = 0.f;
      int blk = 0;
      bool alive = u >= 0;
      int prune_step = 0;
      if (alive) {
        while (blk < nblk) {
          phi += block_sq_diff(p.layout + (((int64_t)blk * p.n + u) << 4), qs + blk * 16);
          ++blk;
          if (blk < nblk && blk % p.dd == 0) {
            const int ns = blk / p.dd;
            if (fmaf(p.m1[ns - 1], phi, p.beta[ns - 1]) > tau) {
              alive = false;
              prune_step = ns;
              break;
            }
          }
        }
      }
      const uint32_t gid = u >= 0 ? (uint32_t)__ldg(p.row_id + u) : 0u;
      if (stats && prune_step) atomicAdd(p.counters + 4 + prune_step, 1ull);
      if (p.dlog && u >= 0) {
        const unsigned long long s = atomicAdd(p.dlog_n, 1ull);
        if ((int64_t)s < p.dlog_cap) {
          p.dlog[3 * s] = (int32_t)q; p.dlog[3 * s + 1] = (int32_t)gid; p.dlog[3 * s + 2] = alive ? D : blk * 16;
        }
      }
      c_tested += __popc(newm);
      const unsigned smask = __ballot_sync(0xffffffffu, alive);
      c_surv += __popc(smask);
      if (smask == 0) continue;
      // survivors in (dist, id) order, inserted one by one (R34)
      unsigned long long key = alive ? gkey(phi, gid) : kInf;
      int kp = alive ? u : -1;
      warp_sort(key, kp, lane);
      const int nsv = __popc(smask);
      for (int j = 0; j < nsv; ++j) {
        const unsigned long long x = __shfl_sync(0xffffffffu, key, j);
        const int xp = __shfl_sync(0xffffffffu, kp, j);
        if (!(wn < ef || x < W[wn - 1])) continue;  // warp-uniform: W is in shared memory
        {  // W: insert x (sorted), the old maximum drops out when full
          int pos = 0;
          for (int i = lane; i < wn; i += 32) pos += W[i] < x;
          pos = __reduce_add_sync(0xffffffffu, pos);
          const int nw = wn < ef ? wn + 1 : ef;
          for (int i0 = nw - 1; i0 > pos; i0 -= 32) {
            const int i = i0 - lane;
            const bool act = i > pos;
            unsigned long long v = 0;
            if (act) v = W[i - 1];
            __syncwarp();
            if (act) W[i] = v;
            __syncwarp();
          }
          if (lane == 0) W[pos] = x;
          wn = nw;
          __syncwarp();
        }
        {  // C: insert (x, its layout position), compacting to the buffer start when needed
          if (ch + cn + 1 > capC && ch > 0) {
            for (int i0 = 0; i0 < cn; i0 += 32) {
              const int i = i0 + lane;
              unsigned long long v = 0;
              int vp = 0;
              if (i < cn) { v = Ck[ch + i]; vp = Cp[ch + i]; }
              __syncwarp();
              if (i < cn) { Ck[i] = v; Cp[i] = vp; }
              __syncwarp();
            }
            ch = 0;
          }
          int pos = 0;
          for (int i = lane; i < cn; i += 32) pos += Ck[ch + i] < x;
          pos = __reduce_add_sync(0xffffffffu, pos);
          if (ch + cn < capC) {
            for (int i0 = cn; i0 > pos; i0 -= 32) {
              const int i = i0 - lane;
              const bool act = i > pos;
              unsigned long long v = 0;
              int vp = 0;
              if (act) { v = Ck[ch + i - 1]; vp = Cp[ch + i - 1]; }
              __syncwarp();
              if (act) { Ck[ch + i] = v; Cp[ch + i] = vp; }
              __syncwarp();
            }
            if (lane == 0) { Ck[ch + pos] = x; Cp[ch + pos] = xp; }
            ++cn;
          }
          __syncwarp();
        }
      }
      // C entries farther than max W are never expanded: drop them (C is sorted)
      if (wn >= ef) {
        const float mx = kdist(W[ef - 1]);
        int keep = 0;
        for (int i = lane; i < cn; i += 32) keep += kdist(Ck[ch + i]) <= mx;
        cn = __reduce_add_sync(0xffffffffu, keep);
      }
    }
    // results: the first K of W
    for (int i = lane; i < p.K; i += 32) {
      const unsigned long long k = i < wn ? W[i] : kInf;
      p.out_ids[q * p.K + i] = k == kInf ? -1 : (int64_t)(uint32_t)(k & 0xffffffffu);
      p.out_d[q * p.K + i] = k == kInf ? INFINITY : kdist(k);
    }
    // clear this query's visited bits
    if (nvis <= p.vcap) {
      for (int i = lane; i < nvis; i += 32) {
        const int v = vl[i];
        vis[v >> 5] = 0u;
      }
    } else {
      for (int i = lane; i < nwords; i += 32) vis[i] = 0u;
    }
    __syncwarp();
  }
  if (stats && lane == 0) {
    atomicAdd(p.counters + 0, c_tested);
    atomicAdd(p.counters + 1, c_surv);
    atomicAdd(p.counters + 2, c_exp);
  }
}

// HNSW's neighbour-selection heuristic (R33), one warp per node: walk the candidate pool in
// (dist, id) order and keep e iff d(e, node) < d(e, r) for every kept r (lane r of the warp holds
// kept neighbour r's distance test); then fill up to M0 with the nearest dropped candidates. The
// kept rows' distances use fp32 block sums over the rotated layout (distances are rotation-invariant).
__global__ void __launch_bounds__(128) k_graph_prune(const float* __restrict__ layout, int64_t n, int D,
                                                     const int32_t* __restrict__ pool, const float* __restrict__ pool_d,
                                                     int P, int M0, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t node = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (node >= n) return;
  const int nblk = D >> 4;
  const int32_t* pl = pool + node * P;
  const float* pd = pool_d + node * P;
  int kept_r = -1;      // this lane's kept neighbour (lane < nkept)
  int nkept = 0;
  unsigned long long dropped_lo = 0, dropped_hi = 0;  // pool indices of dropped candidates (P <= 128)
  for (int c = 0; c < P; ++c) {
    const int e = pl[c];
    if (e < 0) continue;
    const float de = pd[c];
    bool closer = true;
    if (lane < nkept) {  // d(e, r) for this lane's kept r
      float acc = 0.f;
      for (int b = 0; b < nblk; ++b) {
        const float4* xe = reinterpret_cast<const float4*>(layout + (((int64_t)b * n + e) << 4));
        const float4* xr = reinterpret_cast<const float4*>(layout + (((int64_t)b * n + kept_r) << 4));
        float a = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float4 u = __ldg(xe + t), v = __ldg(xr + t);
          const float d0 = u.x - v.x, d1 = u.y - v.y, d2 = u.z - v.z, d3 = u.w - v.w;
          a += fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3);
        }
        acc += a;
      }
      closer = de < acc;
    }
    const bool keep = nkept < M0 && __all_sync(0xffffffffu, closer);
    if (keep) {
      if (lane == nkept) kept_r = e;
      if (lane == 0) out[node * M0 + nkept] = e;
      ++nkept;
    } else if (c < 64) {
      dropped_lo |= 1ull << c;
    } else {
      dropped_hi |= 1ull << (c - 64);
    }
  }
  // keepPrunedConnections: the nearest dropped candidates fill the list, then -1
  int k = nkept;
  for (int c = 0; c < P && k < M0; ++c) {
    const bool d = c < 64 ? (dropped_lo >> c) & 1 : (dropped_hi >> (c - 64)) & 1;
    if (d) {
      if (lane == 0) out[node * M0 + k] = pl[c];
      ++k;
    }
  }
  for (int j = k + lane; j < M0; j += 32) out[node * M0 + j] = -1;
}

void launch_graph_prune(const float* layout, int64_t n, int D, const int32_t* pool, const float* pool_d, int P,
                        int M0, int32_t* out, cudaStream_t st) {
  if (n <= 0) return;
  DADE_REQUIRE(P <= 128 && M0 <= 32, DADE_ERR_UNSUPPORTED, "graph: pool > 128 or M0 > 32");
  k_graph_prune<<<(unsigned)((n + 3) / 4), 128, 0, st>>>(layout, n, D, pool, pool_d, P, M0, out);
  DADE_CK(cudaGetLastError());
}

size_t graph_smem(int D, int ef) {
  const size_t per = (size_t)D * 4 + (size_t)ef * 8 + (size_t)(ef + 64) * 12 + 16;
  return kGW * ((per + 15) & ~(size_t)15);
}

int graph_slots(int sms) { return sms * 8 * kGW; }

void launch_graph_search(const GraphParams& p, int sms, cudaStream_t st) {
  if (p.nq <= 0) return;
  const size_t smem = graph_smem(p.D, p.ef);
  DADE_REQUIRE(smem <= 220 * 1024, DADE_ERR_UNSUPPORTED, "graph search: D / ef too large");
  DADE_CK(cudaFuncSetAttribute(k_graph_search, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::min(sms * 8, (p.nq + kGW - 1) / kGW);
  k_graph_search<<<grid, kGW * 32, smem, st>>>(p);
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
