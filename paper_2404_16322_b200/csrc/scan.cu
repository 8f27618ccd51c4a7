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
// B200 mapping:
//  * persistent warps, ONE WARP PER QUERY (queries taken from an atomic counter): an epoch
//    boundary waits only for the warp's own survivors, never for a CTA barrier;
//  * the first step of every candidate is STREAMED with TMA bulk copies (cp.async.bulk, one
//    elected lane, mbarrier completion) into a per-warp shared-memory ring of tiles, issued
//    kStages tiles ahead of consumption (across list and epoch boundaries: the data does not
//    depend on tau). The dimension-blocked, list-major layout makes every tile one contiguous
//    block-row range (64 B per row per 16 dims);
//  * survivors of a step are ballot-compacted into a per-warp ring; their next blocks are
//    gathered with 128-bit loads, 4 lanes per 64-B row, several blocks of lookahead per round;
//  * finished candidates are merged into the warp's sorted top-K (order-independent result).
#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kQCap = 128;        // per-warp survivor ring capacity (power of two)
constexpr int kStages = 3;        // TMA tile ring depth per warp
constexpr unsigned long long kKeyInf = ~0ull;
constexpr int kMbarBytes = ((kStages * 8 + 15) / 16) * 16;  // keep the following arrays 16-B aligned

struct __align__(16) QEntry {
  int32_t row;
  float phi, plo;
  int32_t blk;  // 16-dim blocks already accumulated
};

struct TileMeta {
  int32_t row0, nr, ep, pad;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

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

// Warp-local top-K (owned by one warp): merge up to 32 keys (one per lane, kKeyInf = none).
struct TopK {
  unsigned long long* buf;  // 2 x K keys (double buffer)
  unsigned long long* sB;   // 32 keys scratch
  int K, n, sel;
  unsigned long long kth;   // K-th key when n == K

  __device__ __forceinline__ void insert(unsigned long long key, int lane) {
    if (n == K && key >= kth) key = kKeyInf;
    if (__ballot_sync(0xffffffffu, key != kKeyInf) == 0) return;
    merge(key, lane);
  }

  __device__ __noinline__ void merge(unsigned long long key, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, j);
        const bool lower = (lane & j) == 0, up = (lane & k) == 0;
        const unsigned long long mn = key < o ? key : o, mx = key < o ? o : key;
        key = (lower == up) ? mn : mx;
      }
    }
    const int m = __popc(__ballot_sync(0xffffffffu, key != kKeyInf));
    const unsigned long long* A = buf + sel * K;
    unsigned long long* Bn = buf + (sel ^ 1) * K;
    sB[lane] = key;
    __syncwarp();
    if (lane < m) {
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] < key) lo = mid + 1; else hi = mid;
      }
      if (lane + lo < K) Bn[lane + lo] = key;
    }
    for (int j = lane; j < n; j += 32) {
      const unsigned long long a = A[j];
      int lo = 0, hi = m;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sB[mid] < a) lo = mid + 1; else hi = mid;
      }
      if (j + lo < K) Bn[j + lo] = a;
    }
    __syncwarp();
    n = min(K, n + m);
    sel ^= 1;
    if (n == K) kth = Bn[K - 1];
  }
};

// Candidate-stream tile iterator (warp-uniform): tiles never cross a list or an epoch boundary.
struct TileIter {
  const int32_t* probes;
  const int32_t* off;
  int nprobe, cj;
  int cpos, cstart, clen, r, L, e_hi_raw, e_hi;  // stream positions (< 2^31)
  int ep;

  __device__ void load_list() {
    if (cj < nprobe) {
      const int l = probes[cj];
      cstart = off[l];
      clen = off[l + 1] - cstart;
    } else {
      cstart = 0;
      clen = 0;
    }
  }
  __device__ void init(const int32_t* pr, const int32_t* of, int np, int L_, int c0) {
    probes = pr; off = of; nprobe = np; cj = 0; cpos = 0; r = 0; L = L_;
    e_hi_raw = c0; e_hi = c0 < L ? c0 : L; ep = 0;
    load_list();
  }
  // next tile of at most TR rows; returns false at the end of the stream
  __device__ bool next(int TR, int32_t& row0, int& nr, int& epoch) {
    if (r >= L) return false;
    if (r >= e_hi) {  // epoch boundary (R13): [0,c0), [c0,2c0), [2c0,4c0), ...
      ++ep;
      e_hi_raw = e_hi_raw > (1 << 29) ? (1 << 30) : e_hi_raw * 2;
      e_hi = e_hi_raw < L ? e_hi_raw : L;
    }
    while (cj < nprobe && cpos + clen <= r) {  // skip exhausted (and empty) lists
      cpos += clen;
      ++cj;
      load_list();
    }
    if (cj >= nprobe) return false;
    const int hi = e_hi < cpos + clen ? e_hi : cpos + clen;
    nr = hi - r < TR ? hi - r : TR;
    row0 = cstart + (r - cpos);
    epoch = ep;
    r += nr;
    return true;
  }
};

}  // namespace

template <int DD, int LA, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_scan(const __grid_constant__ ScanParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int D = p.D, K = p.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int TR = 32;                 // rows per tile: one row per lane
  constexpr int TB = TR * 64 * DD;       // tile bytes (DD blocks of 32 rows)
  // per-warp smem slice: tiles | mbar | meta | ring | topk[2K] | sB | pruned | qs[D]
  const size_t slice = (size_t)kStages * TB + kMbarBytes + kStages * sizeof(TileMeta) +
                       kQCap * sizeof(QEntry) + (size_t)2 * K * 8 + 32 * 8 + DADE_MAX_STEPS * 4 + (size_t)D * 4;
  unsigned char* base = smem + warp * ((slice + 127) & ~(size_t)127);
  unsigned char* tiles = base;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + kStages * TB);
  TileMeta* meta = reinterpret_cast<TileMeta*>(base + kStages * TB + kMbarBytes);
  QEntry* ring = reinterpret_cast<QEntry*>(meta + kStages);
  unsigned long long* tkbuf = reinterpret_cast<unsigned long long*>(ring + kQCap);
  unsigned long long* sB = tkbuf + 2 * K;
  unsigned* pruned = reinterpret_cast<unsigned*>(sB + 32);
  float* qs = reinterpret_cast<float*>(pruned + DADE_MAX_STEPS);

  for (int j = lane; j < DADE_MAX_STEPS; j += 32) pruned[j] = 0;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  const int nsteps = p.nsteps;
  const int nblk = D >> 4;
  const int64_t n = p.n;
  const float* lay = p.layout;
  const bool stats = p.counters != nullptr;
  unsigned long long c_tested = 0, c_surv = 0, c_dims = 0;  // warp-uniform (lane 0 authoritative)
  uint32_t phase_bits = 0;
  const unsigned lt_mask = (1u << lane) - 1;

  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(p.work_counter, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= p.nq) break;
    const int64_t q = qi;
    for (int j = lane; j < D; j += 32) qs[j] = p.qrot[q * D + j];
    TopK tk{tkbuf, sB, K, 0, 0, kKeyInf};
    const int32_t* probes = p.probes + q * p.nprobe;
    int64_t L = 0;
    for (int j = lane; j < p.nprobe; j += 32) {
      const int l = probes[j];
      L += p.off[l + 1] - p.off[l];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    __syncwarp();

    // ------------------------------------------------------------ producer (TMA bulk copies)
    TileIter prod;
    prod.init(probes, p.off, p.nprobe, (int)L, p.c0);
    int issued = 0;
    auto issue = [&](int slot) {  // warp-uniform call; lane 0 issues
      int32_t row0;
      int nr, ep;
      if (!prod.next(TR, row0, nr, ep)) return false;
      if (lane == 0) {
        meta[slot] = TileMeta{row0, nr, ep, 0};
        const uint32_t bytes = (uint32_t)nr * 64u;
        mbar_expect_tx(&mbar[slot], bytes * DD);
#pragma unroll
        for (int bb = 0; bb < DD; ++bb)
          bulk_g2s(tiles + slot * TB + bb * TR * 64, lay + (((int64_t)bb * n + row0) << 4), bytes, &mbar[slot]);
      }
      ++issued;
      return true;
    };
    for (int s = 0; s < kStages; ++s)
      if (!issue(s)) break;

    int head = 0, tail = 0;  // survivor ring (monotonic indices), warp-uniform
    float tau = INFINITY;
    int cur_ep = 0, consumed = 0;

    auto push = [&](bool keep, const QEntry& e) {
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (keep) ring[(tail + __popc(km & lt_mask)) & (kQCap - 1)] = e;
      tail += __popc(km);
    };
    auto finish = [&](bool fin, float P, int32_t row) {
      unsigned long long key = kKeyInf;
      if (fin) key = make_key(P, (uint32_t)p.row_id[row]);
      if (stats) {
        const int nf = __popc(__ballot_sync(0xffffffffu, fin));
        c_surv += nf;
        c_dims += (unsigned long long)nf * D;
      }
      tk.insert(key, lane);
    };

    // one gather round: up to 32 queued survivors (one per lane) advanced by up to LA blocks
    auto queue_round = [&](bool drain) {
      const int qn = min(tail - head, 32);
      const bool val = lane < qn;
      QEntry e = val ? ring[(head + lane) & (kQCap - 1)] : QEntry{0, 0.f, 0.f, nblk};
      const int want = min((drain || e.blk > DD) ? LA : (DD < LA ? DD : LA), nblk - e.blk);
      float4 v[LA][4];
#pragma unroll
      for (int s = 0; s < LA; ++s)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[s][k] = (s < want) ? ldg4(lay + (((int64_t)(e.blk + s) * n + e.row) << 4) + k * 4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
      head += qn;
      __syncwarp();
      float phi = e.phi, plo = e.plo;
      int blk = e.blk;
      bool alive = val, fin = false;
#pragma unroll
      for (int s = 0; s < LA; ++s) {
        if (alive && s < want) {
          const float* qb = qs + blk * 16;
          float b4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 qq = *reinterpret_cast<const float4*>(qb + k * 4);
            float t = v[s][k].x - qq.x; b4[k] = t * t;
            t = v[s][k].y - qq.y; b4[k] = fmaf(t, t, b4[k]);
            t = v[s][k].z - qq.z; b4[k] = fmaf(t, t, b4[k]);
            t = v[s][k].w - qq.w; b4[k] = fmaf(t, t, b4[k]);
          }
          const float bs = (b4[0] + b4[1]) + (b4[2] + b4[3]);
          float err;  // compensated running sum over blocks (R21)
          two_sum(phi, bs, phi, err);
          plo += err;
          ++blk;
          if (blk % DD == 0) {  // step boundary: the classifier for d = blk*16
            const int ns = blk / DD;
            if (ns == nsteps) {
              fin = true;
              alive = false;
            } else if (fmaf(p.m1[ns - 1], phi + plo, p.beta[ns - 1]) > tau) {
              alive = false;
              if (stats) atomicAdd(&pruned[ns], 1u);
            }
          }
        }
      }
      if (stats) {
        // dims of candidates pruned in this round: blk*16 each (warp sum)
        unsigned long long dp = (val && !alive && !fin) ? (unsigned long long)blk * 16 : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
        c_dims += dp;
      }
      push(alive, QEntry{e.row, phi, plo, blk});
      finish(fin, phi + plo, e.row);
      __syncwarp();
    };

    // ------------------------------------------------------------ consumer
    while (consumed < issued) {
      const int slot = consumed % kStages;
      mbar_wait(&mbar[slot], (phase_bits >> slot) & 1u);
      phase_bits ^= 1u << slot;
      const TileMeta tm = meta[slot];
      if (tm.ep != cur_ep) {  // epoch boundary: finish every survivor, then refresh tau (R13)
        while (tail > head) queue_round(true);
        tau = (tk.n == K) ? __uint_as_float((unsigned)(tk.kth >> 32)) : INFINITY;
        cur_ep = tm.ep;
      }
      while (tail - head > kQCap - TR) queue_round(false);  // room for this tile's survivors
      const int nr = tm.nr;
      const bool val = lane < nr;
      // stage 1: one row per lane; the 16-B chunk order is rotated per lane so the 8 lanes of
      // each shared-memory phase hit distinct banks
      const unsigned char* trow = tiles + slot * TB + lane * 64;
      // 4 independent partial sums (one per 16-B chunk) keep the FMA pipes busy
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int bb = 0; bb < DD; ++bb) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int ch = (k + lane) & 3;
          const float4 x = *reinterpret_cast<const float4*>(trow + bb * TR * 64 + ch * 16);
          const float4 qq = *reinterpret_cast<const float4*>(qs + bb * 16 + ch * 4);
          float t = x.x - qq.x; s4[k] = fmaf(t, t, s4[k]);
          t = x.y - qq.y; s4[k] = fmaf(t, t, s4[k]);
          t = x.z - qq.z; s4[k] = fmaf(t, t, s4[k]);
          t = x.w - qq.w; s4[k] = fmaf(t, t, s4[k]);
        }
      }
      const float s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      __syncwarp();  // every lane is done reading this slot
      ++consumed;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(slot);
      const int32_t row = tm.row0 + lane;
      if (stats) c_tested += nr;
      if (nsteps == 1) {
        finish(val, s, row);
      } else {
        const bool prune = val && fmaf(p.m1[0], s, p.beta[0]) > tau;
        push(val && !prune, QEntry{row, s, 0.f, DD});
        if (stats) {
          const int np_ = __popc(__ballot_sync(0xffffffffu, prune));
          if (lane == 0 && np_) pruned[1] += np_;
          c_dims += (unsigned long long)np_ * DD * 16;
        }
      }
      if (tail - head >= 16) queue_round(false);
    }
    while (tail > head) queue_round(true);

    const unsigned long long* fin = tk.buf + tk.sel * K;
    for (int i = lane; i < K; i += 32) {
      const unsigned long long key = i < tk.n ? fin[i] : kKeyInf;
      p.out_ids[q * K + i] = key == kKeyInf ? -1 : (int64_t)(uint32_t)(key & 0xffffffffu);
      p.out_d[q * K + i] = key == kKeyInf ? INFINITY : __uint_as_float((unsigned)(key >> 32));
    }
    if (lane == 0 && stats) atomicMax(p.counters + 3, (unsigned long long)(L > 0 ? cur_ep + 1 : 0));
    __syncwarp();
  }
  if (stats) {
    if (lane == 0) {
      atomicAdd(p.counters + 0, c_tested);
      atomicAdd(p.counters + 1, c_surv);
      atomicAdd(p.counters + 2, c_dims);
    }
    __syncwarp();
    for (int j = lane; j < DADE_MAX_STEPS; j += 32)
      if (pruned[j]) atomicAdd(p.counters + 4 + j, (unsigned long long)pruned[j]);
  }
}

static size_t scan_smem(int D, int K, int DD) {
  const size_t slice = (size_t)kStages * 32 * 64 * DD + kMbarBytes + kStages * sizeof(TileMeta) +
                       kQCap * sizeof(QEntry) + (size_t)2 * K * 8 + 32 * 8 + DADE_MAX_STEPS * 4 + (size_t)D * 4;
  return kWarps * ((slice + 127) & ~(size_t)127);
}

template <int DD, int LA, int MINB>
static void launch_v(const ScanParams& p, cudaStream_t st) {
  const size_t smem = scan_smem(p.D, p.K, DD);
  static int sms = 0;
  if (!sms) {
    DADE_CK(cudaFuncSetAttribute(k_scan<DD, LA, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int dev;
    DADE_CK(cudaGetDevice(&dev));
    DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  DADE_REQUIRE(smem <= 200 * 1024, DADE_ERR_UNSUPPORTED, "scan: shared memory slice too large (D, K)");
  int occ = 0;
  DADE_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan<DD, LA, MINB>, kThreads, smem));
  const int max_blocks = (occ > 0 ? occ : 1) * sms;
  const int need = (p.nq + kWarps - 1) / kWarps;
  k_scan<DD, LA, MINB><<<need < max_blocks ? need : max_blocks, kThreads, smem, st>>>(p);
}

// variant (lookahead blocks, min CTAs/SM) selectable for tuning via DADE_SCAN_VARIANT
static int scan_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DADE_SCAN_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int DD>
static void launch_dd(const ScanParams& p, cudaStream_t st) {
  switch (scan_variant()) {
    case 1: launch_v<DD, 2, 4>(p, st); break;
    case 3: launch_v<DD, 4, 3>(p, st); break;
    default: launch_v<DD, 2, 6>(p, st); break;
  }
}

void launch_scan(const ScanParams& p, cudaStream_t st) {
  if (p.nq <= 0) return;
  switch (p.dd) {
    case 1: launch_dd<1>(p, st); break;
    case 2: launch_dd<2>(p, st); break;
    case 4: launch_dd<4>(p, st); break;
    default: throw Error(DADE_ERR_UNSUPPORTED, "delta_d must be 16, 32 or 64");
  }
  DADE_CK(cudaGetLastError());
}

}  // namespace dade
