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
constexpr int kQCap = 128;  // per-warp survivor ring capacity (power of two)
constexpr int kMinBlocks = 4;
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
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_scan(const __grid_constant__ ScanParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Shared sh;
  const int D = p.D, K = p.K;
  float* qs = reinterpret_cast<float*>(smem);                                  // D floats
  unsigned long long* topk = reinterpret_cast<unsigned long long*>(qs + D);    // 2 x MAX_K
  QEntry* queues = reinterpret_cast<QEntry*>(topk + 2 * DADE_MAX_K);          // kWarps x kQCap ring
  unsigned long long* sBall = reinterpret_cast<unsigned long long*>(queues + kWarps * kQCap);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  QEntry* ring = queues + warp * kQCap;
  unsigned long long* sB = sBall + warp * 32;
  const int64_t q = blockIdx.x;
  constexpr int TR = 64 / DD;  // rows per stage-1 tile (8 x 128-bit loads per lane)
  constexpr int NI = TR / 8;   // 8 rows per warp instruction
  constexpr int LA = 4;        // queue lookahead slots (blocks) per entry per round
  constexpr int NB = 2;        // queue batches (8 entries each) per round
  const int nsteps = p.nsteps;
  const int nblk = D >> 4;
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
  int head = 0, tail = 0;  // ring indices (monotonic), warp-uniform
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

  // finished candidate -> CTA top-K
  auto finish = [&](bool fin, float P, int32_t row) {
    unsigned long long key = kKeyInf;
    if (fin && c == 0) {
      key = make_key(P, (uint32_t)p.row_id[row]);
      c_dims += D;
      ++c_surv;
    }
    topk_insert(key, sh, topk, K, sB, lane);
  };

  // One memory round trip: stage 1 of an optional tile (rows row0..row0+nr) and up to
  // NB*8 queued survivors advanced by up to LA blocks (1 step for fresh survivors, LA blocks
  // for older ones or when draining), all loads issued before any arithmetic.
  auto round = [&](float tau, bool has_tile, int64_t row0, int nr, bool drain) {
    // ---- issue loads
    float4 tv[NI][DD];
    if (has_tile) {
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int bb = 0; bb < DD; ++bb)
          tv[i][bb] = (i * 8 + g < nr) ? ldg4(lay + (((int64_t)bb * n + row0 + i * 8 + g) << 4) + c * 4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int qn = min(tail - head, NB * 8);
    QEntry e[NB];
    int want[NB];
    float4 qv[NB][LA];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int idx = i * 8 + g;
      const bool val = idx < qn;
      e[i] = val ? ring[(head + idx) & (kQCap - 1)] : QEntry{0, 0.f, 0.f, nblk};
      const int rem = nblk - e[i].step;  // .step = blocks done
      want[i] = (drain || e[i].step > DD) ? LA : DD;
      want[i] = min(want[i], rem);
#pragma unroll
      for (int s = 0; s < LA; ++s)
        qv[i][s] = (s < want[i]) ? ldg4(lay + (((int64_t)(e[i].step + s) * n + e[i].row) << 4) + c * 4)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    head += qn;
    __syncwarp();
    // ---- stage 1 of the tile
    if (has_tile) {
      if (lane == 0) c_tested += nr;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const bool val = i * 8 + g < nr;
        const float s = step_sum<DD>(tv[i], qs, c);
        const int32_t row = (int32_t)(row0 + i * 8 + g);
        if (nsteps == 1) {
          finish(val, s, row);
          continue;
        }
        const bool prune = val && fmaf(p.m1[0], s, p.beta[0]) > tau;
        const bool keep = val && !prune;
        const unsigned km = __ballot_sync(0xffffffffu, keep && c == 0);
        if (keep && c == 0) ring[(tail + __popc(km & ((1u << lane) - 1))) & (kQCap - 1)] = QEntry{row, s, 0.f, DD};
        tail += __popc(km);
        if (prune && c == 0) { c_dims += DD * 16; atomicAdd(&sh.pruned[1], 1u); }
      }
    }
    // ---- queued survivors
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const bool val = i * 8 + g < qn;
      float phi = e[i].phi, plo = e[i].plo, acc = 0.f;
      int blk = e[i].step;
      bool alive = val, fin = false;
#pragma unroll
      for (int s = 0; s < LA; ++s) {
        const bool act = alive && s < want[i];
        // block sum (all lanes take part in the shuffles)
        const float4 qq = *reinterpret_cast<const float4*>(qs + min(blk, nblk - 1) * 16 + c * 4);
        float t = qv[i][s].x - qq.x, bs = t * t;
        t = qv[i][s].y - qq.y; bs = fmaf(t, t, bs);
        t = qv[i][s].z - qq.z; bs = fmaf(t, t, bs);
        t = qv[i][s].w - qq.w; bs = fmaf(t, t, bs);
        bs += __shfl_xor_sync(0xffffffffu, bs, 1);
        bs += __shfl_xor_sync(0xffffffffu, bs, 2);
        if (act) {
          acc += bs;
          ++blk;
          if (blk % DD == 0) {  // step boundary: compensated add, then the classifier
            float err;
            two_sum(phi, acc, phi, err);
            plo += err;
            acc = 0.f;
            const int ns = blk / DD;
            if (ns == nsteps) {
              fin = true;
              alive = false;
            } else if (fmaf(p.m1[ns - 1], phi + plo, p.beta[ns - 1]) > tau) {
              alive = false;
              if (c == 0) { c_dims += (unsigned long long)blk * 16; atomicAdd(&sh.pruned[ns], 1u); }
            }
          }
        }
      }
      // keep (step boundary reached with lookahead < remaining) -> back to the ring tail
      const unsigned km = __ballot_sync(0xffffffffu, alive && c == 0);
      if (alive && c == 0)
        ring[(tail + __popc(km & ((1u << lane) - 1))) & (kQCap - 1)] = QEntry{e[i].row, phi, plo, blk};
      tail += __popc(km);
      finish(fin, phi + plo, e[i].row);
    }
    __syncwarp();
  };

  int64_t e_lo = 0, e_hi_raw = p.c0;
  int n_epochs = 0;
  while (e_lo < L) {
    const int64_t e_hi = e_hi_raw < L ? e_hi_raw : L;
    ++n_epochs;
    const float tau = sh.tau;
    int t = 0;
    while (cj < p.nprobe) {
      const int64_t seg_lo = e_lo > cpos ? e_lo : cpos;
      const int64_t seg_hi = e_hi < cpos + clen ? e_hi : cpos + clen;
      for (int64_t r = seg_lo; r < seg_hi; r += TR, ++t) {
        if ((t % kWarps) != warp) continue;
        const int nr = (int)(seg_hi - r < TR ? seg_hi - r : TR);
        while (tail - head > kQCap - TR - NB * 8) round(tau, false, 0, 0, false);
        round(tau, true, cstart + (r - cpos), nr, false);
      }
      if (cpos + clen <= e_hi) {
        cpos += clen;
        ++cj;
        load_list(cj);
      } else {
        break;
      }
    }
    while (tail > head) round(tau, false, 0, 0, true);
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
