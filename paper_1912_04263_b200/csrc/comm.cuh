// comm.cuh — the collectives of the row-sharded path.
//
// A is cut into G contiguous, nnz-balanced row blocks ("shards").  A process
// owns L local shards on its device (L > 1 = "virtual shards", the single-GPU
// proof of the partition math) and R processes (one per GPU, torchrun ranks)
// are joined by one NCCL communicator, G = L * R.  The path needs only:
//   * allreduce(sum | max) of n-vectors (the A^T partials) and of a handful of
//     scalars (m-side norms, infeasibility support sums);
//   * a sequential chain across shards in row order (diag(A^T A) is a
//     sequential sum in the reference, sparse.hpp:401-408; chaining the
//     per-shard partial sums keeps it bit-exact);
//   * gathering the m-side results (z, y, the primal certificate).
// Local shards share one stream, so their combination is a plain ordered
// device kernel; across ranks NCCL (loaded with dlopen, so the engine loads on
// hosts without it and reuses the copy torch already mapped) does the rest.
#pragma once

#include <dlfcn.h>
#include <nccl.h>  // types and enums only: every symbol is resolved through dlopen

#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace qpcg_b200 {

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the soname torch (or the system) already mapped wins; fall back to the
    // unversioned development link
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (api.GetUniqueId && api.CommInitRank && api.AllReduce && api.Broadcast && api.Send &&
        api.Recv && api.GroupStart && api.GroupEnd && api.CommDestroy)
      api.h = h;
  });
  if (!api.h) throw NcclError("nccl: libnccl.so.2 not found or incomplete");
  return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* e = nccl_api().GetErrorString ? nccl_api().GetErrorString(r) : "?";
  throw NcclError(std::string("nccl: ") + what + " failed: " + e);
}

template <typename T>
inline ncclDataType_t nccl_type();
template <>
inline ncclDataType_t nccl_type<double>() { return ncclFloat64; }
template <>
inline ncclDataType_t nccl_type<float>() { return ncclFloat32; }
template <>
inline ncclDataType_t nccl_type<unsigned long long>() { return ncclUint64; }

// ------------------------------------------------------------------ kernels
constexpr int kMaxLocalShards = 16;
template <typename T>
struct ShardPtrs {
  T* p[kMaxLocalShards];
};

// b_l <- b_0 (+) b_1 (+) ... (+) b_{L-1} for every l: the local shards'
// partials combined in shard (= row) order, then replicated.
template <typename T, bool MAX>
__global__ void k_local_combine(ShardPtrs<T> b, int L, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T a = b.p[0][i];
    for (int l = 1; l < L; ++l) {
      const T v = b.p[l][i];
      a = MAX ? smax(a, v) : a + v;
    }
    for (int l = 0; l < L; ++l) b.p[l][i] = a;
  }
}

// ------------------------------------------------------------------ comm
struct ShardComm {
  int rank = 0, nranks = 1;  // NCCL process group (nranks == 1 and no comm: local only)
  int local = 1;             // shards on this device
  ncclComm_t comm = nullptr;
  cudaStream_t s = nullptr;

  int global_count() const { return local * nranks; }
  int global_index(int l) const { return rank * local + l; }

  // Communicators are cached per (unique id, rank, ranks, device) for the life
  // of the process: creating one costs a rendezvous of every rank (tens to
  // hundreds of ms), and a solve loop (bench steps, receding-horizon MPC)
  // sets up workspace after workspace on the same group.
  void init_nccl(const void* id, int r, int nr) {
    NcclApi& api = nccl_api();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    rank = r;
    nranks = nr;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::string key(reinterpret_cast<const char*>(&uid), sizeof(uid));
    key += ":" + std::to_string(r) + ":" + std::to_string(nr) + ":" + std::to_string(dev);
    static std::mutex mu;
    static std::map<std::string, ncclComm_t> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      comm = it->second;
      return;
    }
    nccl_check(api.CommInitRank(&comm, nr, uid, r), "ncclCommInitRank");
    cache.emplace(key, comm);
  }
  ~ShardComm() {}  // the cached communicator outlives the workspace

  // in-place allreduce of `count` elements held in one buffer per local shard
  template <typename T>
  void allreduce(const std::vector<T*>& bufs, size_t count, bool max) {
    if (count == 0) return;
    if (bufs.size() > 1) {
      ShardPtrs<T> p{};
      for (size_t l = 0; l < bufs.size(); ++l) p.p[l] = bufs[l];
      const uint32_t g = (uint32_t)std::min<size_t>((count + kThreads - 1) / kThreads, 4u * kNumSMs);
      if (max)
        k_local_combine<T, true><<<g, kThreads, 0, s>>>(p, (int)bufs.size(), count);
      else
        k_local_combine<T, false><<<g, kThreads, 0, s>>>(p, (int)bufs.size(), count);
      CK_LAUNCH();
    }
    if (comm) {
      nccl_check(nccl_api().AllReduce(bufs[0], bufs[0], count, nccl_type<T>(), max ? ncclMax : ncclSum,
                                      comm, s),
                 "ncclAllReduce");
      for (size_t l = 1; l < bufs.size(); ++l)
        CK(cudaMemcpyAsync(bufs[l], bufs[0], sizeof(T) * count, cudaMemcpyDeviceToDevice, s));
    }
  }

  // min over every rank of one device-resident uint64 (validation keys)
  void allreduce_min_u64(unsigned long long* dev) {
    if (comm)
      nccl_check(nccl_api().AllReduce(dev, dev, 1, ncclUint64, ncclMin, comm, s), "ncclAllReduce");
  }

  // Sequential chain across ranks in rank order: rank r receives the running
  // value from r-1, `body` continues it over its local shards, then it is
  // sent on to r+1 and the final value is broadcast from the last rank.
  template <typename T, typename F>
  void chain(T* acc, size_t count, F&& body) {
    NcclApi* api = comm ? &nccl_api() : nullptr;
    if (comm && rank > 0) nccl_check(api->Recv(acc, count, nccl_type<T>(), rank - 1, comm, s), "ncclRecv");
    body();
    if (comm && rank + 1 < nranks)
      nccl_check(api->Send(acc, count, nccl_type<T>(), rank + 1, comm, s), "ncclSend");
    if (comm && nranks > 1)
      nccl_check(api->Broadcast(acc, acc, count, nccl_type<T>(), nranks - 1, comm, s), "ncclBroadcast");
  }

  // Every rank contributes its contiguous block [off[r], off[r+1]) of `full`
  // (already in place locally); afterwards every rank holds all of it.
  template <typename T>
  void allgather_blocks(T* full, const std::vector<uint32_t>& off) {
    if (!comm || nranks == 1) return;
    NcclApi& api = nccl_api();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < nranks; ++r) {
      const size_t cnt = off[r + 1] - off[r];
      if (cnt == 0) continue;
      T* p = full + off[r];
      nccl_check(api.Broadcast(p, p, cnt, nccl_type<T>(), r, comm, s), "ncclBroadcast");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
};

// nnz-balanced contiguous row cuts (SURVEY.md §8(e) "Partitioning"): shard g
// owns rows [cuts[g], cuts[g+1]) with cuts[g] the first row whose row_ptr is
// >= g * nnz / G.  An invalid row_ptr (not starting at 0, not ending at nnz,
// or decreasing) puts every row on shard 0, so validation then reports the
// reference's error exactly as the unsharded engine does.  Returns false in
// that case.
inline bool shard_cuts(const uint32_t* rp, uint32_t rows, uint32_t nnz, uint32_t G, uint32_t* cuts) {
  bool ok = rp[0] == 0 && rp[rows] == nnz;
  for (uint32_t r = 0; ok && r < rows; ++r) ok = rp[r + 1] >= rp[r];
  cuts[0] = 0;
  for (uint32_t g = 1; g <= G; ++g) cuts[g] = rows;
  if (!ok) return false;
  for (uint32_t g = 1; g < G; ++g) {
    const uint64_t target = (uint64_t)nnz * g / G;
    uint32_t lo = cuts[g - 1], hi = rows;  // first r in [lo, rows] with rp[r] >= target
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if ((uint64_t)rp[mid] >= target) hi = mid;
      else lo = mid + 1;
    }
    cuts[g] = lo;
  }
  return true;
}

}  // namespace qpcg_b200
