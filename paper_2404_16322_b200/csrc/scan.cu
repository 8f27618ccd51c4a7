// a6-a8: the progressive-scan kernel (the hot loop of the method).
//
// Method: refinement keeps a result queue of size K, tau = its K-th distance
// (P:L42-43). For every candidate of the probed IVF lists the squared distance in
// the PCA basis is accumulated Delta_d dims at a time (Alg. 2 loop); after each step
// d < D the cascade classifier for d prunes iff m1_d * P_d + beta'_d > tau
// (BSA-p estimator P:L569-573). Survivors reach d = D, where P_D is the exact
// distance, and enter the queue. tau is frozen within geometric epochs of the
// candidate stream (R13: [0,4K), [4K,8K), [8K,16K), ...) so the result does not depend on
// the parallel schedule.
//
// B200 mapping: one CTA (4 warps) per query; the rotated query and the running top-K live in
// shared memory. The database layout is dimension-blocked and list-major (16 dims = one 64-B
// row per block), so the first step of a list segment is one contiguous stream: a warp loads
// 8 rows per 128-bit instruction (4 lanes per 64-B row, fully coalesced). Survivors of a step
// are compacted by warp ballot into a per-warp queue; each queue round gathers the next block
// of every queued survivor at once (one memory round trip for up to 32 survivors), so the chain
// of later steps is overlapped with the streaming of further tiles. Finished candidates are
// merged into the CTA's sorted top-K by a warp-cooperative merge (order-independent result).
#include <cfloat>
#include <cstdint>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kQCap = 64;  // per-warp survivor queue capacity
constexpr unsigned long long kKeyInf = ~0ull;

struct __align__(16) QEntry {
  int32_t row;
  float phi, plo;
  int32_t step;  // steps already accumulated
};

struct Shared {
  unsigned long long kth;  // key of the current K-th entry (valid when n == K)
  int n, sel, lock;
  float tau;
  unsigned pruned[DADE_MAX_STEPS];
};

__device__ __forceinline__ void two_sum(float a, float b, float& s, float& e) {
  s = a + b;
  const float bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

__device__ __forceinline__ unsigned long long make_key(float d, uint32_t id) {
  return ((unsigned long long)__float_as_uint(d) << 32) | id;
}

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// partial sum over the 4*DD dims this lane holds, then reduced over the 4 lanes of the row
template <int DD>
__device__ __forceinline__ float step_sum(const float4 (&v)[DD], const float* qs_step, int c) {
  float s = 0.f;
#pragma unroll
  for (int bb = 0; bb < DD; ++bb) {
    const float4 q = *reinterpret_cast<const float4*>(qs_step + bb * 16 + c * 4);
    float t = v[bb].x - q.x; s = fmaf(t, t, s);
    t = v[bb].y - q.y; s = fmaf(t, t, s);
    t = v[bb].z - q.z; s = fmaf(t, t, s);
    t = v[bb].w - q.w; s = fmaf(t, t, s);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  return s;
}

// Warp-cooperative merge of up to 32 keys (one per lane, kKeyInf = none) into the CTA top-K.
__device__ void topk_insert(unsigned long long key, Shared& sh, unsigned long long* topk, int K,
                            unsigned long long* sB, int lane) {
  if (key != kKeyInf) {  // racy read of the K-th key: stale values are only conservative
    const volatile Shared& vs = sh;
    if (vs.n == K && key >= vs.kth) key = kKeyInf;
  }
  if (__ballot_sync(0xffffffffu, key != kKeyInf) == 0) return;
  // bitonic sort of the 32 keys, ascending by lane
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, j);
      const bool lower = (lane & j) == 0;
      const bool up = (lane & k) == 0;
      const unsigned long long mn = key < o ? key : o, mx = key < o ? o : key;
      key = (lower == up) ? mn : mx;
    }
  }
  const int m = __popc(__ballot_sync(0xffffffffu, key != kKeyInf));
  if (lane == 0) {
    while (atomicCAS(&sh.lock, 0, 1) != 0) {
    }
  }
  __syncwarp();
  __threadfence_block();
  volatile Shared& vs = sh;
  const int sel = vs.sel, na = vs.n;
  const unsigned long long* A = topk + sel * DADE_MAX_K;
  unsigned long long* Bn = topk + (sel ^ 1) * DADE_MAX_K;
  sB[lane] = key;
  __syncwarp();
  if (lane < m) {  // rank of key among A (keys are distinct)
    int lo = 0, hi = na;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (A[mid] < key) lo = mid + 1; else hi = mid;
    }
    const int pos = lane + lo;
    if (pos < K) Bn[pos] = key;
  }
  for (int j = lane; j < na; j += 32) {
    const unsigned long long a = A[j];
    int lo = 0, hi = m;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sB[mid] < a) lo = mid + 1; else hi = mid;
    }
    const int pos = j + lo;
    if (pos < K) Bn[pos] = a;
  }
  __syncwarp();
  __threadfence_block();
  if (lane == 0) {
    const int nn = min(K, na + m);
    vs.n = nn;
    vs.sel = sel ^ 1;
    if (nn == K) vs.kth = Bn[K - 1];
    __threadfence_block();
    atomicExch(&sh.lock, 0);
  }
  __syncwarp();
}

}  // namespace

template <int DD>
__global__ void __launch_bounds__(kThreads, 4) k_scan(const __grid_constant__ ScanParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Shared sh;
  const int D = p.D, K = p.K;
  float* qs = reinterpret_cast<float*>(smem);                                  // D floats
  unsigned long long* topk = reinterpret_cast<unsigned long long*>(qs + D);    // 2 x MAX_K
  QEntry* queues = reinterpret_cast<QEntry*>(topk + 2 * DADE_MAX_K);          // kWarps x kQCap
  unsigned long long* sBall = reinterpret_cast<unsigned long long*>(queues + kWarps * kQCap);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  QEntry* queue = queues + warp * kQCap;
  unsigned long long* sB = sBall + warp * 32;
  const int64_t q = blockIdx.x;
  constexpr int TR = 64 / DD;  // rows per tile
  constexpr int NI = TR / 8;   // 8 rows per warp instruction
  const int nsteps = p.nsteps;
  const int64_t n = p.n;
  const float* lay = p.layout;

  for (int j = tid; j < D; j += kThreads) qs[j] = p.qrot[q * D + j];
  if (tid == 0) {
    sh.n = 0; sh.sel = 0; sh.lock = 0; sh.kth = kKeyInf; sh.tau = INFINITY;
  }
  for (int j = tid; j < DADE_MAX_STEPS; j += kThreads) sh.pruned[j] = 0;
  const int32_t* probes = p.probes + q * p.nprobe;
  int64_t L = 0;  // stream length, identical in every warp
  for (int j = lane; j < p.nprobe; j += 32) {
    const int l = probes[j];
    L += p.off[l + 1] - p.off[l];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  __syncthreads();

  unsigned long long c_tested = 0, c_surv = 0, c_dims = 0;
  int qcnt = 0;
  // stream cursor (warp-uniform, identical in all warps)
  int cj = 0;
  int64_t cpos = 0, cstart = 0, clen = 0;
  auto load_list = [&](int j) {
    if (j < p.nprobe) {
      const int l = probes[j];
      cstart = p.off[l];
      clen = p.off[l + 1] - cstart;
    } else {
      cstart = 0;
      clen = 0;
    }
  };
  load_list(0);

  // one queue round: advance every queued survivor by one step
  auto queue_round = [&](float tau) {
    const int nq_ = qcnt;
    int newc = 0;
    constexpr int NB = 4;  // 8-entry batches per sub-round
    for (int base = 0; base < nq_; base += 8 * NB) {
      QEntry e[NB];
      bool val[NB];
      float4 v[NB][DD];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int idx = base + i * 8 + g;
        val[i] = idx < nq_;
        e[i] = val[i] ? queue[idx] : QEntry{0, 0.f, 0.f, 0};
#pragma unroll
        for (int bb = 0; bb < DD; ++bb)
          v[i][bb] = val[i] ? ldg4(lay + (((int64_t)(e[i].step * DD + bb) * n + e[i].row) << 4) + c * 4)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int st = e[i].step;  // 0-based index of the step being added
        const float s = step_sum<DD>(v[i], qs + st * 16 * DD, c);
        float phi, plo, err;
        two_sum(e[i].phi, s, phi, err);
        plo = e[i].plo + err;
        const int ns = st + 1;
        const bool fin = val[i] && ns == nsteps;
        const float P = phi + plo;
        bool prune = false;
        if (val[i] && !fin) prune = fmaf(p.m1[ns - 1], P, p.beta[ns - 1]) > tau;
        const bool keep = val[i] && !fin && !prune;
        const unsigned km = __ballot_sync(0xffffffffu, keep && c == 0);
        if (keep && c == 0) {
          const int pos = newc + __popc(km & ((1u << lane) - 1));
          queue[pos] = QEntry{e[i].row, phi, plo, ns};
        }
        newc += __popc(km);
        if (c == 0) {
          if (prune) { c_dims += (unsigned long long)ns * DD * 16; atomicAdd(&sh.pruned[ns], 1u); }
          if (fin) { c_dims += D; ++c_surv; }
        }
        unsigned long long key = kKeyInf;
        if (fin && c == 0) key = make_key(P, (uint32_t)p.row_id[e[i].row]);
        topk_insert(key, sh, topk, K, sB, lane);
      }
      __syncwarp();
    }
    qcnt = newc;
  };

  int64_t e_lo = 0, e_hi_raw = p.c0;
  int n_epochs = 0;
  while (e_lo < L) {
    const int64_t e_hi = e_hi_raw < L ? e_hi_raw : L;
    ++n_epochs;
    const float tau = sh.tau;
    const bool full = !p.prune || !(tau < INFINITY);
    int t = 0;
    while (cj < p.nprobe) {
      const int64_t seg_lo = e_lo > cpos ? e_lo : cpos;
      const int64_t seg_hi = e_hi < cpos + clen ? e_hi : cpos + clen;
      for (int64_t r = seg_lo; r < seg_hi; r += TR, ++t) {
        if ((t % kWarps) != warp) continue;
        const int nr = (int)(seg_hi - r < TR ? seg_hi - r : TR);
        const int64_t row0 = cstart + (r - cpos);
        if (lane == 0) c_tested += nr;
        if (full) {
          float phi[NI], plo[NI];
#pragma unroll
          for (int i = 0; i < NI; ++i) { phi[i] = 0.f; plo[i] = 0.f; }
          for (int st = 0; st < nsteps; ++st) {
            float4 v[NI][DD];
#pragma unroll
            for (int i = 0; i < NI; ++i)
#pragma unroll
              for (int bb = 0; bb < DD; ++bb)
                v[i][bb] = (i * 8 + g < nr)
                               ? ldg4(lay + (((int64_t)(st * DD + bb) * n + row0 + i * 8 + g) << 4) + c * 4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const float s = step_sum<DD>(v[i], qs + st * 16 * DD, c);
              float err;
              if (st == 0) { phi[i] = s; plo[i] = 0.f; }
              else { two_sum(phi[i], s, phi[i], err); plo[i] += err; }
            }
          }
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const bool val = i * 8 + g < nr;
            unsigned long long key = kKeyInf;
            if (val && c == 0) {
              key = make_key(phi[i] + plo[i], (uint32_t)p.row_id[row0 + i * 8 + g]);
              c_dims += D;
              ++c_surv;
            }
            topk_insert(key, sh, topk, K, sB, lane);
          }
        } else {
          while (qcnt + TR > kQCap) queue_round(tau);
          float4 v[NI][DD];
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int bb = 0; bb < DD; ++bb)
              v[i][bb] = (i * 8 + g < nr)
                             ? ldg4(lay + (((int64_t)bb * n + row0 + i * 8 + g) << 4) + c * 4)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const bool val = i * 8 + g < nr;
            const float s = step_sum<DD>(v[i], qs, c);
            // nsteps >= 2 here (nsteps == 1 implies !prune, i.e. the full path)
            const bool prune = val && fmaf(p.m1[0], s, p.beta[0]) > tau;
            const bool keep = val && !prune;
            const unsigned km = __ballot_sync(0xffffffffu, keep && c == 0);
            if (keep && c == 0) {
              const int pos = qcnt + __popc(km & ((1u << lane) - 1));
              queue[pos] = QEntry{(int32_t)(row0 + i * 8 + g), s, 0.f, 1};
            }
            qcnt += __popc(km);
            if (prune && c == 0) { c_dims += DD * 16; atomicAdd(&sh.pruned[1], 1u); }
          }
          __syncwarp();
          if (qcnt > 0) queue_round(tau);
        }
      }
      if (cpos + clen <= e_hi) {
        cpos += clen;
        ++cj;
        load_list(cj);
      } else {
        break;
      }
    }
    while (qcnt > 0) queue_round(tau);
    __syncthreads();
    if (tid == 0) sh.tau = (sh.n == K) ? __uint_as_float((unsigned)(sh.kth >> 32)) : INFINITY;
    __syncthreads();
    e_lo = e_hi;
    e_hi_raw *= 2;
  }

  // output (ascending by (dist, id)); missing -> (-1, +inf)
  const unsigned long long* fin = topk + sh.sel * DADE_MAX_K;
  for (int i = tid; i < K; i += kThreads) {
    const unsigned long long key = i < sh.n ? fin[i] : kKeyInf;
    p.out_ids[q * K + i] = key == kKeyInf ? -1 : (int64_t)(uint32_t)(key & 0xffffffffu);
    p.out_d[q * K + i] = key == kKeyInf ? INFINITY : __uint_as_float((unsigned)(key >> 32));
  }
  // counters
  if (p.counters) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c_tested += __shfl_xor_sync(0xffffffffu, c_tested, o);
      c_surv += __shfl_xor_sync(0xffffffffu, c_surv, o);
      c_dims += __shfl_xor_sync(0xffffffffu, c_dims, o);
    }
    if (lane == 0) {
      atomicAdd(p.counters + 0, c_tested);
      atomicAdd(p.counters + 1, c_surv);
      atomicAdd(p.counters + 2, c_dims);
    }
    if (tid == 0) atomicMax(p.counters + 3, (unsigned long long)n_epochs);
    for (int j = tid; j < DADE_MAX_STEPS; j += kThreads)
      if (sh.pruned[j]) atomicAdd(p.counters + 4 + j, (unsigned long long)sh.pruned[j]);
  }
}

static size_t scan_smem(int D) {
  return (size_t)D * 4 + 2 * DADE_MAX_K * 8 + kWarps * kQCap * sizeof(QEntry) + kWarps * 32 * 8;
}

void launch_scan(const ScanParams& p, cudaStream_t st) {
  if (p.nq <= 0) return;
  const size_t smem = scan_smem(p.D);
  static bool attr[3] = {false, false, false};
  switch (p.dd) {
    case 1:
      if (!attr[0]) {
        DADE_CK(cudaFuncSetAttribute(k_scan<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
        attr[0] = true;
      }
      k_scan<1><<<p.nq, kThreads, smem, st>>>(p);
      break;
    case 2:
      if (!attr[1]) {
        DADE_CK(cudaFuncSetAttribute(k_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
        attr[1] = true;
      }
      k_scan<2><<<p.nq, kThreads, smem, st>>>(p);
      break;
    case 4:
      if (!attr[2]) {
        DADE_CK(cudaFuncSetAttribute(k_scan<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
        attr[2] = true;
      }
      k_scan<4><<<p.nq, kThreads, smem, st>>>(p);
      break;
    default:
      throw Error(DADE_ERR_UNSUPPORTED, "delta_d must be 16, 32 or 64");
  }
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
