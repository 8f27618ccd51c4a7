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
// B200 mapping: persistent warps, ONE WARP PER QUERY (queries fetched from an
// atomic counter), so an epoch boundary only waits for the warp's own survivors and never for a
// CTA barrier. The rotated query, the sorted top-K and a survivor ring live in the warp's slice
// of shared memory. The database layout is dimension-blocked and list-major (16 dims = one 64-B
// row per block): the first step of a tile is one contiguous stream, 4 lanes per row, 8 rows per
// 128-bit load (fully coalesced). Survivors are ballot-compacted into the ring; each round issues
// the tile's loads AND the next-block gathers of up to 16 queued survivors (with lookahead) before
// any arithmetic, so one memory round trip serves both. Finished candidates are merged into the
// warp's sorted top-K (order-independent result).
#include <cfloat>
#include <cstdint>

#include "dade_internal.h"

namespace dade {

namespace {
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kMinBlocks = 4;
constexpr int kQCap = 128;  // per-warp survivor ring capacity (power of two)
constexpr unsigned long long kKeyInf = ~0ull;

struct __align__(16) QEntry {
  int32_t row;
  float phi, plo;
  int32_t blk;  // 16-dim blocks already accumulated
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

// sum over the 4*DD dims this lane holds, reduced over the 4 lanes of the row
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

}  // namespace

template <int DD>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_scan(const __grid_constant__ ScanParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int D = p.D, K = p.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  // per-warp smem slice: qs[D] | topk[2K] | sB[32] | ring[kQCap] | pruned[64]
  const size_t slice = (size_t)D * 4 + (size_t)2 * K * 8 + 32 * 8 + kQCap * sizeof(QEntry) + DADE_MAX_STEPS * 4;
  unsigned char* base = smem + warp * ((slice + 15) & ~(size_t)15);
  float* qs = reinterpret_cast<float*>(base);
  unsigned long long* tkbuf = reinterpret_cast<unsigned long long*>(base + (size_t)D * 4);
  unsigned long long* sB = tkbuf + 2 * K;
  QEntry* ring = reinterpret_cast<QEntry*>(sB + 32);
  unsigned* pruned = reinterpret_cast<unsigned*>(ring + kQCap);
  for (int j = lane; j < DADE_MAX_STEPS; j += 32) pruned[j] = 0;

  constexpr int TR = 64 / DD;  // rows per stage-1 tile (8 x 128-bit loads per lane)
  constexpr int NI = TR / 8;   // 8 rows per warp instruction
  constexpr int LA = 4;        // lookahead slots (blocks) per queued survivor per round
  constexpr int NB = 2;        // queued-survivor batches (8 each) per round
  const int nsteps = p.nsteps;
  const int nblk = D >> 4;
  const int64_t n = p.n;
  const float* lay = p.layout;
  unsigned long long c_tested = 0, c_surv = 0, c_dims = 0, c_epochs = 0;

  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(p.work_counter, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= p.nq) break;
    const int64_t q = qi;
    __syncwarp();
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

    auto finish = [&](bool fin, float P, int32_t row) {
      unsigned long long key = kKeyInf;
      if (fin && c == 0) {
        key = make_key(P, (uint32_t)p.row_id[row]);
        c_dims += D;
        ++c_surv;
      }
      tk.insert(key, lane);
    };

    // One memory round trip: stage 1 of an optional tile and up to NB*8 queued survivors
    // advanced by up to LA blocks (one step for fresh survivors; LA blocks for older ones or
    // when draining), all loads issued before any arithmetic.
    auto round = [&](float tau, bool has_tile, int64_t row0, int nr, bool drain) {
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
        e[i] = idx < qn ? ring[(head + idx) & (kQCap - 1)] : QEntry{0, 0.f, 0.f, nblk};
        want[i] = min((drain || e[i].blk > DD) ? LA : (DD < LA ? DD : LA), nblk - e[i].blk);
#pragma unroll
        for (int s = 0; s < LA; ++s)
          qv[i][s] = (s < want[i]) ? ldg4(lay + (((int64_t)(e[i].blk + s) * n + e[i].row) << 4) + c * 4)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      head += qn;
      __syncwarp();
      if (has_tile) {
        if (lane == 0) c_tested += nr;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          if (i * 8 >= nr) break;  // warp-uniform: ragged tail of a list segment
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
          if (prune && c == 0) { c_dims += DD * 16; atomicAdd(&pruned[1], 1u); }
        }
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (i * 8 >= qn) break;  // warp-uniform: no queued entries left
        float phi = e[i].phi, plo = e[i].plo;
        int blk = e[i].blk;
        bool alive = i * 8 + g < qn, fin = false;
        const int wmax = __reduce_max_sync(0xffffffffu, alive ? want[i] : 0);
#pragma unroll
        for (int s = 0; s < LA; ++s) {
          if (s >= wmax) break;  // warp-uniform
          const bool act = alive && s < want[i];
          const float4 qq = *reinterpret_cast<const float4*>(qs + min(blk, nblk - 1) * 16 + c * 4);
          float t = qv[i][s].x - qq.x, bs = t * t;
          t = qv[i][s].y - qq.y; bs = fmaf(t, t, bs);
          t = qv[i][s].z - qq.z; bs = fmaf(t, t, bs);
          t = qv[i][s].w - qq.w; bs = fmaf(t, t, bs);
          bs += __shfl_xor_sync(0xffffffffu, bs, 1);
          bs += __shfl_xor_sync(0xffffffffu, bs, 2);
          if (act) {
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
                if (c == 0) { c_dims += (unsigned long long)blk * 16; atomicAdd(&pruned[ns], 1u); }
              }
            }
          }
        }
        const unsigned km = __ballot_sync(0xffffffffu, alive && c == 0);
        if (alive && c == 0)
          ring[(tail + __popc(km & ((1u << lane) - 1))) & (kQCap - 1)] = QEntry{e[i].row, phi, plo, blk};
        tail += __popc(km);
        finish(fin, phi + plo, e[i].row);
      }
      __syncwarp();
    };

    int64_t e_lo = 0, e_hi_raw = p.c0, e_hi = p.c0 < L ? p.c0 : L, r = 0;
    float tau = INFINITY;
    if (L > 0) ++c_epochs;
    while (e_lo < L) {
      // next action (warp-uniform): a stage-1 tile of the current epoch, a make-room round,
      // a drain round, or the epoch boundary
      bool has_tile = false;
      int64_t row0 = 0;
      int nr = 0;
      if (tail - head <= kQCap - TR - NB * 8) {
        while (cj < p.nprobe) {
          const int64_t lo = r > cpos ? r : cpos;
          const int64_t hi = e_hi < cpos + clen ? e_hi : cpos + clen;
          if (lo < hi) {
            nr = (int)(hi - lo < TR ? hi - lo : TR);
            row0 = cstart + (lo - cpos);
            r = lo + nr;
            has_tile = true;
            break;
          }
          if (cpos + clen <= e_hi) {
            cpos += clen;
            ++cj;
            load_list(cj);
          } else {
            break;
          }
        }
      }
      const bool epoch_done = !has_tile && (r >= e_hi || cj >= p.nprobe);
      if (!has_tile && epoch_done && tail == head) {  // epoch boundary: refresh tau (R13)
        tau = (tk.n == K) ? __uint_as_float((unsigned)(tk.kth >> 32)) : INFINITY;
        e_lo = e_hi;
        e_hi_raw *= 2;
        e_hi = e_hi_raw < L ? e_hi_raw : L;
        if (e_lo < L) ++c_epochs;
        continue;
      }
      round(tau, has_tile, row0, nr, epoch_done);
    }
    const unsigned long long* fin = tk.buf + tk.sel * K;
    for (int i = lane; i < K; i += 32) {
      const unsigned long long key = i < tk.n ? fin[i] : kKeyInf;
      p.out_ids[q * K + i] = key == kKeyInf ? -1 : (int64_t)(uint32_t)(key & 0xffffffffu);
      p.out_d[q * K + i] = key == kKeyInf ? INFINITY : __uint_as_float((unsigned)(key >> 32));
    }
    if (lane == 0 && p.counters) atomicMax(p.counters + 3, c_epochs);
    c_epochs = 0;
    __syncwarp();
  }
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
    __syncwarp();
    for (int j = lane; j < DADE_MAX_STEPS; j += 32)
      if (pruned[j]) atomicAdd(p.counters + 4 + j, (unsigned long long)pruned[j]);
  }
}

static size_t scan_smem(int D, int K) {
  const size_t slice = (size_t)D * 4 + (size_t)2 * K * 8 + 32 * 8 + kQCap * sizeof(QEntry) + DADE_MAX_STEPS * 4;
  return kWarps * ((slice + 15) & ~(size_t)15);
}

template <int DD>
static void launch_dd(const ScanParams& p, cudaStream_t st) {
  const size_t smem = scan_smem(p.D, p.K);
  static int sms = 0;
  if (!sms) {
    DADE_CK(cudaFuncSetAttribute(k_scan<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    int dev;
    DADE_CK(cudaGetDevice(&dev));
    DADE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  DADE_REQUIRE(smem <= 96 * 1024, DADE_ERR_UNSUPPORTED, "scan: shared memory slice too large (D, K)");
  int occ = 0;
  DADE_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan<DD>, kThreads, smem));
  const int max_blocks = (occ > 0 ? occ : 1) * sms;
  const int need = (p.nq + kWarps - 1) / kWarps;
  k_scan<DD><<<need < max_blocks ? need : max_blocks, kThreads, smem, st>>>(p);
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
