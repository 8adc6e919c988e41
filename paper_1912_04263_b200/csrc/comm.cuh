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
#include <sys/stat.h>
#include <cstdlib>
#include <nccl.h>  // types and enums only: every symbol is resolved through dlopen

#include <chrono>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <thread>
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
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // 1. a copy already mapped into the process (torch's) wins;
    // 2. QPCG_NCCL_LIB (the Python layer points it at the pip NCCL that torch
    //    itself loads, so a later `import torch` finds the same library
    //    instead of clashing with an older system soname);
    // 3. the system soname, then the unversioned development link
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) {
      const char* lib = std::getenv("QPCG_NCCL_LIB");
      if (lib && lib[0]) h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
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
    sym(api.AllGather, "ncclAllGather");
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

// ------------------------------------------------------- peer transport
// The collectives over peer memory (NVLink P2P stores between the GPUs of one
// box; CUDA IPC mappings between processes).  Every rank owns one symmetric
// area (same layout everywhere), maps every peer's area, and:
//   * allreduce: each rank stores its blocks' partials into slot g (= global
//     block index) of EVERY rank's area, a device-side barrier (system-scope
//     arrival counters in every area), then each rank sums the G slots in
//     block order.  The combination is a flat sequential sum in block order on
//     every rank: bitwise identical across ranks AND to the single-process run
//     with the same G virtual blocks (k_local_combine).  The slot sets are
//     double-buffered, so no trailing barrier is needed;
//   * the diag(A^T A) chain and the block gather of the m-vectors use the
//     same stores and barriers.
// Bootstrap (exchanging the IPC handles) goes through NCCL when the caller
// gave an NCCL id, else through a rendezvous directory.
struct PeerPtrs {
  char* p[kMaxLocalShards];
};

// The barrier epoch (this rank's count of barriers, in its own area) is kept
// on the device, and the slot set of an allreduce is its parity before the
// barrier: no host state changes between collectives, so the whole loop can
// be captured into a CUDA graph (the set alternates every replay).
__device__ __forceinline__ unsigned long long p2p_epoch(const unsigned long long* e) {
  return *reinterpret_cast<const volatile unsigned long long*>(e);
}

// dst.p[r] = rank r's first slot set; set 1 starts set_bytes later
template <typename T>
__global__ void k_p2p_publish(ShardPtrs<T> src, int L, size_t count, PeerPtrs dst, int R,
                              size_t off_bytes, size_t slot_bytes, size_t set_bytes,
                              const unsigned long long* epoch) {
  const size_t set = (p2p_epoch(epoch) & 1ull) * set_bytes;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    for (int l = 0; l < L; ++l) {
      const T v = src.p[l][i];
      for (int r = 0; r < R; ++r)
        reinterpret_cast<T*>(dst.p[r] + set + off_bytes + l * slot_bytes)[i] = v;
    }
  }
}

// one thread: fence, arrive at every rank's counter (area offset 0), bump
// this rank's epoch (offset 8), wait until every rank arrived this epoch
static __global__ void k_p2p_barrier(PeerPtrs area, int R, int rank) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  __threadfence_system();
  for (int r = 0; r < R; ++r)
    atomicAdd_system(reinterpret_cast<unsigned long long*>(area.p[r]), 1ull);
  unsigned long long* ep = reinterpret_cast<unsigned long long*>(area.p[rank] + 8);
  const unsigned long long e = *ep + 1ull;
  *ep = e;
  const volatile unsigned long long* mine =
      reinterpret_cast<const volatile unsigned long long*>(area.p[rank]);
  // a rank that never arrives (crashed, or a peer mapping that does not
  // reach this GPU) must not hang the device: after 300 s the kernel traps,
  // which fails this process's context instead of spinning forever
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*mine < e * (unsigned long long)R) {
    __nanosleep(200);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 300ull * 1000000000ull) {
      printf("qpcg peer barrier: rank %d waited 300 s for %d ranks (epoch %llu): trap\n", rank,
             R, e);
      __trap();
    }
  }
  __threadfence_system();
}

// after the barrier: the set of the epoch just closed
template <typename T, bool MAX>
__global__ void k_p2p_reduce(const char* slots0, size_t slot_bytes, size_t set_bytes, int G,
                             size_t count, ShardPtrs<T> out, int L,
                             const unsigned long long* epoch) {
  const char* slots = slots0 + ((p2p_epoch(epoch) - 1ull) & 1ull) * set_bytes;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T a = __ldcv(reinterpret_cast<const T*>(slots) + i);
    for (int g = 1; g < G; ++g) {
      const T v = __ldcv(reinterpret_cast<const T*>(slots + g * slot_bytes) + i);
      a = MAX ? smax(a, v) : a + v;
    }
    for (int l = 0; l < L; ++l) out.p[l][i] = a;
  }
}

static __global__ void k_p2p_min_u64(const char* slots, size_t slot_bytes, int R,
                              unsigned long long* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long a = ~0ull;
  for (int r = 0; r < R; ++r) {
    const unsigned long long v = __ldcv(reinterpret_cast<const unsigned long long*>(slots + r * slot_bytes));
    a = v < a ? v : a;
  }
  *out = a;
}

struct P2PArea {
  int rank = 0, R = 1, G = 1, L = 1;
  char* mine = nullptr;
  size_t bytes = 0, vcap = 0, m = 0, n = 0;
  size_t off_vec = 0, off_u64 = 0, off_gbuf = 0, off_chain = 0;  // (flags at 0)
  std::vector<char*> peer;
  size_t vec_slot() const { return vcap * 8; }
  size_t vec_set() const { return vec_slot() * G; }
};

inline void p2p_exchange_file(const std::string& dir, int rank, int R, const void* mine, size_t bytes,
                              std::vector<std::string>& all) {
  // write my handle atomically, then poll for every rank's
  const std::string me = dir + "/rank" + std::to_string(rank) + ".ipc";
  {
    const std::string tmp = me + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) throw NcclError("p2p: cannot write the rendezvous file " + tmp);
    std::fwrite(mine, 1, bytes, f);
    std::fclose(f);
    std::rename(tmp.c_str(), me.c_str());
  }
  all.assign(R, std::string());
  const double t0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  for (int r = 0; r < R; ++r) {
    const std::string fn = dir + "/rank" + std::to_string(r) + ".ipc";
    for (;;) {
      FILE* f = std::fopen(fn.c_str(), "rb");
      if (f) {
        std::string buf(bytes, '\0');
        const size_t got = std::fread(&buf[0], 1, bytes, f);
        std::fclose(f);
        if (got == bytes) {
          all[r] = buf;
          break;
        }
      }
      const double t = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
      if (t - t0 > 120.0) throw NcclError("p2p: rendezvous timed out waiting for rank " + std::to_string(r));
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
}

// ------------------------------------------------------------------ comm
struct ShardComm {
  int rank = 0, nranks = 1;  // process group (nranks == 1 and no transport: local only)
  int local = 1;             // shards on this device
  ncclComm_t comm = nullptr;
  cudaStream_t s = nullptr;
  P2PArea* p2p = nullptr;    // the peer-memory transport (owned), else NCCL

  bool multi() const { return comm != nullptr || p2p != nullptr; }

  // Set up the peer transport for G = local * R blocks of an (n, m) problem.
  // The NCCL comm, when there is one, only carries the bootstrap.
  void init_p2p(int r, int R, const char* dir, size_t n, size_t m) {
    rank = r;
    nranks = R;
    auto* a = new P2PArea();
    p2p = a;
    a->rank = r;
    a->R = R;
    a->L = local;
    a->G = local * R;
    a->n = n;
    a->m = m;
    a->vcap = std::max<size_t>(2 * n, 16);
    size_t off = 64;
    a->off_vec = off;
    off += 2 * a->vec_set();
    a->off_u64 = off;
    off += 8 * size_t(R);
    a->off_gbuf = off;
    off += 8 * std::max<size_t>(m, 1);
    a->off_chain = off;
    off += 8 * std::max<size_t>(n, 1);
    a->bytes = off;
    CK(cudaMalloc(&a->mine, a->bytes));  // IPC needs a plain allocation
    CK(cudaMemset(a->mine, 0, a->bytes));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, a->mine));
    std::vector<std::string> all;
    if (comm) {  // bootstrap over NCCL
      char *dsend = nullptr, *drecv = nullptr;
      CK(cudaMalloc(&dsend, sizeof(h)));
      CK(cudaMalloc(&drecv, sizeof(h) * R));
      CK(cudaMemcpy(dsend, &h, sizeof(h), cudaMemcpyHostToDevice));
      nccl_check(nccl_api().AllGather(dsend, drecv, sizeof(h), ncclChar, comm, s), "ncclAllGather");
      std::string buf(sizeof(h) * R, '\0');
      CK(cudaMemcpyAsync(&buf[0], drecv, buf.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      cudaFree(dsend);
      cudaFree(drecv);
      all.assign(R, std::string());
      for (int i = 0; i < R; ++i) all[i] = buf.substr(i * sizeof(h), sizeof(h));
    } else {
      if (!dir) throw InvalidArgument("options: the peer transport needs an NCCL id or a rendezvous directory");
      // one fresh subdirectory per setup of the group (every rank sets up the
      // same sequence of workspaces, so the counters agree)
      static std::mutex gmu;
      static std::map<std::string, int> generation;
      int k = 0;
      {
        std::lock_guard<std::mutex> lock(gmu);
        k = generation[dir]++;
      }
      const std::string sub = std::string(dir) + "/g" + std::to_string(k);
      mkdir(sub.c_str(), 0700);  // EEXIST from the other ranks is fine
      p2p_exchange_file(sub, r, R, &h, sizeof(h), all);
    }
    a->peer.assign(R, nullptr);
    for (int i = 0; i < R; ++i) {
      if (i == r) {
        a->peer[i] = a->mine;
        continue;
      }
      cudaIpcMemHandle_t hi;
      std::memcpy(&hi, all[i].data(), sizeof(hi));
      void* q = nullptr;
      CK(cudaIpcOpenMemHandle(&q, hi, cudaIpcMemLazyEnablePeerAccess));
      a->peer[i] = static_cast<char*>(q);
    }
    barrier();  // every rank has mapped every area
    CK(cudaStreamSynchronize(s));
  }
  void free_p2p() {
    if (!p2p) return;
    cudaStreamSynchronize(s);
    barrier();  // nobody writes into an area after it is unmapped
    cudaStreamSynchronize(s);
    for (int i = 0; i < p2p->R; ++i)
      if (i != p2p->rank && p2p->peer[i]) cudaIpcCloseMemHandle(p2p->peer[i]);
    cudaFree(p2p->mine);
    delete p2p;
    p2p = nullptr;
  }
  PeerPtrs peers(size_t off) const {
    PeerPtrs pp{};
    for (int i = 0; i < p2p->R; ++i) pp.p[i] = p2p->peer[i] + off;
    return pp;
  }
  void barrier() {
    k_p2p_barrier<<<1, 32, 0, s>>>(peers(0), p2p->R, p2p->rank);
    CK_LAUNCH();
  }
  const unsigned long long* dev_epoch() const {
    return reinterpret_cast<const unsigned long long*>(p2p->mine + 8);
  }

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
  ~ShardComm() { free_p2p(); }  // (the cached NCCL communicator outlives the workspace)

  // in-place allreduce of `count` elements held in one buffer per local shard
  template <typename T>
  void allreduce(const std::vector<T*>& bufs, size_t count, bool max) {
    if (count == 0) return;
    if (p2p) {  // publish into every rank's slots, barrier, ordered sum of all G slots
      P2PArea& a = *p2p;
      if (count > a.vcap) throw InvalidArgument("p2p: allreduce larger than the slots");
      ShardPtrs<T> src{};
      for (size_t l = 0; l < bufs.size(); ++l) src.p[l] = bufs[l];
      const uint32_t g = (uint32_t)std::min<size_t>((count + kThreads - 1) / kThreads, 4u * kNumSMs);
      k_p2p_publish<T><<<g, kThreads, 0, s>>>(src, (int)bufs.size(), count, peers(a.off_vec), a.R,
                                               size_t(rank) * a.L * a.vec_slot(), a.vec_slot(),
                                               a.vec_set(), dev_epoch());
      CK_LAUNCH();
      p2p_reduce(bufs, count, max);
      return;
    }
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

  // The fused form (the A^T SpMV epilogue stores its rows straight into every
  // rank's slot): p2p_slot(l) is where local block l writes this time,
  // p2p_reduce() then barriers and sums the G slots into bufs.
  // block l's slot in set 0 of every rank's area (set 1: + vec_set(); the
  // epilogue picks the set from the device epoch)
  PeerPtrs p2p_slot(int l) const {
    return peers(p2p->off_vec + (size_t(rank) * p2p->L + l) * p2p->vec_slot());
  }
  template <typename T>
  void p2p_reduce(const std::vector<T*>& bufs, size_t count, bool max) {
    P2PArea& a = *p2p;
    ShardPtrs<T> out{};
    for (size_t l = 0; l < bufs.size(); ++l) out.p[l] = bufs[l];
    barrier();
    const uint32_t g = (uint32_t)std::min<size_t>((count + kThreads - 1) / kThreads, 4u * kNumSMs);
    if (max)
      k_p2p_reduce<T, true><<<g, kThreads, 0, s>>>(a.mine + a.off_vec, a.vec_slot(), a.vec_set(),
                                                   a.G, count, out, (int)bufs.size(), dev_epoch());
    else
      k_p2p_reduce<T, false><<<g, kThreads, 0, s>>>(a.mine + a.off_vec, a.vec_slot(), a.vec_set(),
                                                    a.G, count, out, (int)bufs.size(), dev_epoch());
    CK_LAUNCH();
  }

  // min over every rank of one device-resident uint64 (validation keys)
  void allreduce_min_u64(unsigned long long* dev) {
    if (p2p) {
      P2PArea& a = *p2p;
      for (int r = 0; r < a.R; ++r)
        CK(cudaMemcpyAsync(a.peer[r] + a.off_u64 + 8 * size_t(rank), dev, 8, cudaMemcpyDeviceToDevice, s));
      barrier();
      k_p2p_min_u64<<<1, 32, 0, s>>>(a.mine + a.off_u64, 8, a.R, dev);
      CK_LAUNCH();
      barrier();  // the u64 slots are single-buffered
      return;
    }
    if (comm)
      nccl_check(nccl_api().AllReduce(dev, dev, 1, ncclUint64, ncclMin, comm, s), "ncclAllReduce");
  }

  // Sequential chain across ranks in rank order: rank r receives the running
  // value from r-1, `body` continues it over its local shards, then it is
  // sent on to r+1 and the final value is broadcast from the last rank.
  template <typename T, typename F>
  void chain(T* acc, size_t count, F&& body) {
    if (p2p) {  // rank k continues the running value, hands it to k+1; the last one to all
      P2PArea& a = *p2p;
      T* mine = reinterpret_cast<T*>(a.mine + a.off_chain);
      for (int k = 0; k < a.R; ++k) {
        if (k == rank) {
          if (k > 0) CK(cudaMemcpyAsync(acc, mine, sizeof(T) * count, cudaMemcpyDeviceToDevice, s));
          body();
          for (int r = (k + 1 < a.R ? k + 1 : 0); r < (k + 1 < a.R ? k + 2 : a.R); ++r)
            if (r != rank)
              CK(cudaMemcpyAsync(a.peer[r] + a.off_chain, acc, sizeof(T) * count,
                                 cudaMemcpyDeviceToDevice, s));
        }
        barrier();
      }
      if (rank + 1 < a.R) CK(cudaMemcpyAsync(acc, mine, sizeof(T) * count, cudaMemcpyDeviceToDevice, s));
      barrier();  // the chain buffer is single-buffered
      return;
    }
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
    if (p2p) {
      P2PArea& a = *p2p;
      const size_t b = off[rank], cnt = off[rank + 1] - off[rank];
      if (cnt)
        for (int r = 0; r < a.R; ++r)
          if (r != rank)
            CK(cudaMemcpyAsync(a.peer[r] + a.off_gbuf + sizeof(T) * b, full + b, sizeof(T) * cnt,
                               cudaMemcpyDeviceToDevice, s));
      barrier();
      for (int r = 0; r < a.R; ++r) {
        const size_t rb = off[r], rc = off[r + 1] - off[r];
        if (r != rank && rc)
          CK(cudaMemcpyAsync(full + rb, a.mine + a.off_gbuf + sizeof(T) * rb, sizeof(T) * rc,
                             cudaMemcpyDeviceToDevice, s));
      }
      barrier();  // the gather buffer is single-buffered
      return;
    }
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
