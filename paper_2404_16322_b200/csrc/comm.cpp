// Multi-rank plumbing owned by the library (SURVEY §8(b) dade_set_comm, §8(e)): one NCCL
// communicator per index, the collectives the sharded build and search need, and the host-side
// combination steps of the sharded build (pure host arithmetic, shared with the process-group
// driver in sharded.py).
//
// libnccl is resolved at run time with dlopen/dlsym (the process's already-loaded libnccl.so.2,
// e.g. the one torch ships, or the system one), so the library has no link-time NCCL dependency
// and single-GPU use never needs it. Types and enum values come from <nccl.h>.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "dade_internal.h"

namespace dade {

namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.GetErrorString;
  });
  DADE_REQUIRE(a.ok, DADE_ERR_NCCL, "libnccl.so.2 not found (dlopen) or incomplete");
  return a;
}

void nccl_ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(DADE_ERR_NCCL, std::string(what) + ": " + api().GetErrorString(r));
}
}  // namespace

struct Comm {
  ncclComm_t c = nullptr;
  int nranks = 1, rank = 0;
};

void comm_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId id;
  nccl_ck(api().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
}

Comm* comm_create(const void* id128, int nranks, int rank) {
  DADE_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, DADE_ERR_ARG, "comm: bad nranks / rank");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  auto* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = api().CommInitRank(&c->c, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_ck(r, "ncclCommInitRank");
  }
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->c) api().CommDestroy(c->c);
  delete c;
}

int comm_size(const Comm* c) { return c ? c->nranks : 1; }
int comm_rank(const Comm* c) { return c ? c->rank : 0; }

void comm_allreduce_sum(Comm* c, void* buf, size_t count, CommType t, cudaStream_t st) {
  if (!c || count == 0) return;
  const ncclDataType_t dt = t == CommType::F64 ? ncclFloat64 : ncclInt64;
  nccl_ck(api().AllReduce(buf, buf, count, dt, ncclSum, c->c, st), "ncclAllReduce");
}

void comm_allgather(Comm* c, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st) {
  if (!c) {
    if (send != recv) DADE_CK(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (bytes_per_rank == 0) return;
  nccl_ck(api().AllGather(send, recv, bytes_per_rank, ncclUint8, c->c, st), "ncclAllGather");
}

// ------------------------------------------------------------------ host combination steps
// k-means update (R19): centroid = fp64 sum / count rounded to fp32; an empty cluster keeps its
// centroid.
void kmeans_update(int nlist, int D, const double* sums, const int64_t* counts, float* cent) {
  for (int c = 0; c < nlist; ++c)
    if (counts[c] > 0)
      for (int j = 0; j < D; ++j)
        cent[(size_t)c * D + j] = (float)(sums[(size_t)c * D + j] / (double)counts[c]);
}

// the global K nearest of each query from S shards' K-NN lists (global ids, fp64 distances),
// ordered by (dist, id) (R12, R14); id < 0 entries are ignored, missing slots -> (-1, +inf)
void merge_knn(int S, int nq, int K, const int64_t* ids, const double* d, int64_t* out_ids, double* out_d) {
  std::vector<std::pair<double, int64_t>> c;
  for (int q = 0; q < nq; ++q) {
    c.clear();
    for (int s = 0; s < S; ++s)
      for (int j = 0; j < K; ++j) {
        const size_t i = ((size_t)s * nq + q) * K + j;
        if (ids[i] >= 0) c.emplace_back(d[i], ids[i]);
      }
    const size_t take = std::min<size_t>(K, c.size());
    std::partial_sort(c.begin(), c.begin() + take, c.end());
    for (int j = 0; j < K; ++j) {
      out_ids[(size_t)q * K + j] = (size_t)j < take ? c[j].second : -1;
      out_d[(size_t)q * K + j] = (size_t)j < take ? c[j].first : INFINITY;
    }
  }
}

// calibration pairs in dade_calibrate's order (R14-R16): per query its K nearest (Label 0, in
// (dist, id) order) then the n_neg smallest (hash, id) negatives over all shards' candidates
// (Label 1); tau = the query's K-th distance. keys / nids: S x nq x n_neg, cnt: S x nq.
// Outputs sized nq * (K + n_neg); returns the number of pairs.
int64_t calibration_pairs(int S, int nq, int K, int n_neg, const int64_t* knn_ids, const double* knn_d,
                          const uint64_t* keys, const int64_t* nids, const int32_t* cnt, int32_t* pq,
                          int64_t* pid, double* tau, double* y) {
  int64_t np = 0;
  std::vector<std::pair<uint64_t, int64_t>> c;
  for (int q = 0; q < nq; ++q) {
    const double t = knn_d[(size_t)q * K + K - 1];
    for (int j = 0; j < K; ++j) {
      pq[np] = q; pid[np] = knn_ids[(size_t)q * K + j]; tau[np] = t; y[np] = 0.0; ++np;
    }
    c.clear();
    for (int s = 0; s < S; ++s) {
      const int m = cnt[(size_t)s * nq + q];
      DADE_REQUIRE(m >= 0 && m <= n_neg, DADE_ERR_ARG, "calibration pairs: bad negative count");
      for (int j = 0; j < m; ++j) {
        const size_t i = ((size_t)s * nq + q) * n_neg + j;
        c.emplace_back(keys[i], nids[i]);
      }
    }
    const size_t take = std::min<size_t>(n_neg, c.size());
    std::partial_sort(c.begin(), c.begin() + take, c.end());
    for (size_t j = 0; j < take; ++j) {
      pq[np] = q; pid[np] = c[j].second; tau[np] = t; y[np] = 1.0; ++np;
    }
  }
  return np;
}

}  // namespace dade
