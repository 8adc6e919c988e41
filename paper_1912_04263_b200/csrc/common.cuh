// common.cuh — shared device/host plumbing for the B200 ADMM/PCG engine.
//
// Build note: the whole engine is compiled with --fmad=false so that every
// `a * b + c` rounds twice, exactly like the reference built with
// -ffp-contract=off; setup kernels (Ruiz, symmetrize,
// transpose, diag caches) are therefore bit-exact with the reference and the
// iteration kernels differ only by summation order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <unordered_map>
#include <string>

namespace qpcg_b200 {

// ---------------------------------------------------------------- errors
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NotPositiveDefinite : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  std::string msg = std::string(what) + " failed: " + cudaGetErrorString(e) + " (" + file + ":" +
                    std::to_string(line) + ")";
  if (e == cudaErrorMemoryAllocation) throw OutOfMemory(msg);
  throw CudaError(msg);
}
#define CK(x) ::qpcg_b200::cuda_check((x), #x, __FILE__, __LINE__)
// every launch of one of our kernels goes through CK_LAUNCH, which also counts it
// (host-side launches; graph-executed kernels are counted from device counters)
inline thread_local uint64_t g_launches = 0;
#define CK_LAUNCH()                                                                   \
  do {                                                                                \
    ++::qpcg_b200::g_launches;                                                        \
    ::qpcg_b200::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
  } while (0)

// ------------------------------------------------------- device memory
// All engine allocations are stream-ordered from the engine's OWN memory pool
// per device (cudaMemPoolCreate; the device's default pool, which other
// cudaMallocAsync users of the process share, is left untouched) with an
// unbounded release threshold: a solve's ~9 GB (config 2) is recycled from the
// pool by the next workspace instead of being unmapped and re-mapped
// (cudaMalloc/cudaFree of multi-GB buffers costs ~100 ms per solve).
// qpcg_release_cached_memory() hands everything idle back to the driver.
inline thread_local cudaStream_t g_alloc_stream = nullptr;
constexpr int kMaxDevices = 64;
struct EnginePools {
  std::mutex mu;
  cudaMemPool_t pool[kMaxDevices] = {};
};
inline EnginePools& engine_pools() {
  static EnginePools p;
  return p;
}
inline cudaMemPool_t engine_pool(int device) {
  // QPCG_DEFAULT_POOL=1: allocate from the device's default pool instead
  static const bool use_default = [] {
    const char* e = std::getenv("QPCG_DEFAULT_POOL");
    return e && e[0] == '1';
  }();
  if (use_default || device < 0 || device >= kMaxDevices) return nullptr;
  EnginePools& P = engine_pools();
  std::lock_guard<std::mutex> g(P.mu);
  if (!P.pool[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    P.pool[device] = pool;
  }
  return P.pool[device];
}
inline void configure_pool(int device) { (void)engine_pool(device); }
inline cudaError_t pool_malloc(void** p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = engine_pool(dev);
  if (!pool) return cudaMallocAsync(p, bytes ? bytes : 1, g_alloc_stream);
  return cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, g_alloc_stream);
}
// A workspace's long-lived buffers (its matrices, scaled copies and vectors;
// ~9 GB at config 2) are recycled through a process-wide cache keyed by
// (device, size): the stream-ordered pool alone fragments across solves of the
// same problem (the next setup then grows the pool, i.e. maps new physical
// memory: 0.2-1.5 s).  A buffer enters the cache only after its owner has
// synchronised every stream that used it, so any stream may take it next.
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> idle;  // (device, bytes) -> block
  std::unordered_map<void*, std::pair<int, size_t>> owned;
  size_t idle_bytes = 0;
};
inline BlockCache& block_cache() {
  static BlockCache c;
  return c;
}
constexpr size_t kCacheMin = size_t(1) << 20;     // smaller buffers: the pool
// idle bytes kept at most: 32 GB, or QPCG_CACHE_MAX_GB (0 disables the cache)
inline size_t cache_max_bytes() {
  static const size_t v = [] {
    const char* e = std::getenv("QPCG_CACHE_MAX_GB");
    return e ? size_t(std::strtoull(e, nullptr, 10)) << 30 : size_t(32) << 30;
  }();
  return v;
}
inline void cache_flush_idle() {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> g(c.mu);
  for (auto& kv : c.idle) {
    c.owned.erase(kv.second);
    cudaFree(kv.second);
  }
  c.idle.clear();
  c.idle_bytes = 0;
}
inline cudaError_t cache_get(void** p, size_t bytes) {
  if (bytes < kCacheMin) return pool_malloc(p, bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  BlockCache& c = block_cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.idle.lower_bound({dev, bytes});
    if (it != c.idle.end() && it->first.first == dev && it->first.second <= bytes + bytes / 8) {
      *p = it->second;
      c.idle_bytes -= it->first.second;
      c.idle.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = pool_malloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {  // idle blocks first, then retry once
    cudaGetLastError();
    cache_flush_idle();
    e = pool_malloc(p, bytes);
  }
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(c.mu);
    c.owned[*p] = {dev, bytes};
  }
  return e;
}
// p's owner has synchronised the streams that used it
inline void cache_put(void* p) {
  if (!p) return;
  BlockCache& c = block_cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.owned.find(p);
    if (it != c.owned.end()) {
      if (c.idle_bytes + it->second.second <= cache_max_bytes()) {
        c.idle.emplace(it->second, p);
        c.idle_bytes += it->second.second;
        return;
      }
      c.owned.erase(it);
    }
  }
  cudaFreeAsync(p, g_alloc_stream);
}

inline bool cache_owned(void* p, size_t* bytes) {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.owned.find(p);
  if (it == c.owned.end()) return false;
  *bytes = it->second.second;
  return true;
}

// Can a cooperative launch be captured into a CUDA graph and replayed on this
// driver / device?  Probed once per process on a private stream.
static __global__ void coop_probe_kernel(int* out) {
  if (threadIdx.x == 0) atomicAdd(out, 1);
}
inline bool coop_capture_probe() {
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    cudaStream_t st = nullptr;
    int* d = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    int h = 0;
    bool good = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
                cudaMalloc(&d, sizeof(int)) == cudaSuccess &&
                cudaMemset(d, 0, sizeof(int)) == cudaSuccess &&
                cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (good) {
      void* args[] = {&d};
      const bool launched = cudaLaunchCooperativeKernel((const void*)coop_probe_kernel, dim3(2),
                                                        dim3(32), args, 0, st) == cudaSuccess;
      good = (cudaStreamEndCapture(st, &g) == cudaSuccess) && launched && g != nullptr;
    }
    good = good && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess &&
           cudaGraphLaunch(ge, st) == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess &&
           cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && h == 2;
    cudaGetLastError();  // a failed probe leaves no sticky error behind
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (d) cudaFree(d);
    if (st) cudaStreamDestroy(st);
    ok = good;
  });
  return ok;
}

// qpcg_release_cached_memory(): the idle cached blocks are freed, then every
// engine pool is trimmed to what live workspaces still hold.
inline void release_cached_memory() {
  cache_flush_idle();
  EnginePools& P = engine_pools();
  std::lock_guard<std::mutex> g(P.mu);
  int prev = 0;
  cudaGetDevice(&prev);
  for (int d = 0; d < kMaxDevices; ++d) {
    if (!P.pool[d]) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();  // frees enqueued on any stream have completed
    cudaMemPoolTrimTo(P.pool[d], 0);
  }
  cudaSetDevice(prev);
}

// A workspace's arena: every cached block it took, and the ones it already
// released again (stream-ordered on its stream, so reusable by its later
// allocations on that stream: the transient buffers of setup — sort keys,
// cub scratch, scan flags — cycle through here instead of the pool).  The
// owner returns all of them to the cache once its streams are idle.
struct Arena {
  std::multimap<size_t, void*> released;
  std::vector<void*> taken;
  void* get(size_t bytes) {
    auto it = released.lower_bound(bytes);
    if (it != released.end() && it->first <= bytes + bytes / 8) {
      void* p = it->second;
      released.erase(it);
      return p;
    }
    void* p = nullptr;
    if (cache_get(&p, bytes) != cudaSuccess) return nullptr;
    taken.push_back(p);
    return p;
  }
  void put(void* p, size_t bytes) { released.emplace(bytes, p); }
  void return_all() {  // owner's streams synchronised
    for (void* p : taken) cache_put(p);
    taken.clear();
    released.clear();
  }
};
inline thread_local Arena* g_arena = nullptr;

template <typename U>
inline cudaError_t dmalloc(U** p, size_t bytes) {
  if (g_arena && bytes >= kCacheMin) {
    void* q = g_arena->get(bytes);
    if (!q) return cudaErrorMemoryAllocation;
    *p = static_cast<U*>(q);
    return cudaSuccess;
  }
  return pool_malloc(reinterpret_cast<void**>(p), bytes);
}
inline cudaError_t dfree(void* p) {
  if (!p) return cudaSuccess;
  size_t bytes = 0;
  if (g_arena && cache_owned(p, &bytes)) {
    g_arena->put(p, bytes);
    return cudaSuccess;
  }
  return cudaFreeAsync(p, g_alloc_stream);
}

struct AllocScope {  // routes dmalloc/dfree of this thread to stream s (and arena a)
  cudaStream_t prev;
  Arena* prev_arena;
  explicit AllocScope(cudaStream_t s, Arena* a = nullptr)
      : prev(g_alloc_stream), prev_arena(g_arena) {
    g_alloc_stream = s;
    g_arena = a;
  }
  ~AllocScope() {
    g_alloc_stream = prev;
    g_arena = prev_arena;
  }
};

// ------------------------------------------------------------ constants
constexpr int kNumSMs = 148;           // B200
constexpr int kThreads = 256;          // default block size
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr uint32_t kShortRowMax = 8;   // rows with <= 8 nnz: one thread per row
// nnz per warp work item (long rows split): 2^plan_chunk_log2(nnz) per
// matrix (DESIGN.md §4 item-size sweep).  4096 for the 1e8-nnz class, where
// the passes are throughput-bound and every item pays a two-round-trip head;
// 2048 below 2^25 nnz, where a pass lasts a few item latencies and a few long
// rows cut into 4096-nnz items set its tail (portfolio at N = 1e6: 256 ms
// with 2048, 359 ms with 4096).  -DQPCG_CHUNK_LOG2=n forces a size.
inline uint32_t plan_chunk_log2(uint64_t nnz) {
#ifdef QPCG_CHUNK_LOG2
  (void)nnz;
  return QPCG_CHUNK_LOG2;
#else
  return nnz >= (uint64_t(1) << 25) ? 12u : 11u;
#endif
}
constexpr int kRedBlocks = 2 * kNumSMs;  // fixed grid of reduction kernels (deterministic)

__host__ __device__ inline uint32_t ceil_div(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------ CSR views
template <typename T>
struct DevCsr {
  uint32_t rows = 0, cols = 0, nnz = 0;
  T* val = nullptr;           // [nnz]
  uint32_t* rp = nullptr;     // [rows + 1]
  uint32_t* ci = nullptr;     // [nnz]
};

// ---------------------------------------------------------- warp helpers
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = v < w ? w : v;
  }
  return v;
}

// Deterministic block reductions (fixed tree); result valid in thread 0.
template <typename T, int NT>
__device__ __forceinline__ T block_sum(T v, T* sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  T r = T(0);
  if (w == 0) {
    r = (l < NT / 32) ? sm[l] : T(0);
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}
template <typename T, int NT>
__device__ __forceinline__ T block_max(T v, T* sm) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  T r = T(0);
  if (w == 0) {
    r = (l < NT / 32) ? sm[l] : T(0);
    r = warp_max(r);
  }
  __syncthreads();
  return r;
}

// std::max / std::min semantics (first argument wins ties / NaN ordering)
template <typename T>
__host__ __device__ __forceinline__ T smax(T a, T b) { return (a < b) ? b : a; }
template <typename T>
__host__ __device__ __forceinline__ T smin(T a, T b) { return (b < a) ? b : a; }

// streaming loads: bypass L1 allocation for the matrix streams
// (QPCG_LDMODE 1: + 256-byte L2 prefetch hint; 2: ld.global.cs)
#ifndef QPCG_LDMODE
#define QPCG_LDMODE 1
#endif
#if QPCG_LDMODE == 1
#define QPCG_LD_Q "ld.global.nc.L1::no_allocate.L2::256B"
#elif QPCG_LDMODE == 2
#define QPCG_LD_Q "ld.global.cs"
#else
#define QPCG_LD_Q "ld.global.nc.L1::no_allocate"
#endif
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile(QPCG_LD_Q ".f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm volatile(QPCG_LD_Q ".f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile(QPCG_LD_Q ".u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <typename T>
__device__ __forceinline__ T t_sqrt(T x);
template <>
__device__ __forceinline__ double t_sqrt<double>(double x) { return __dsqrt_rn(x); }
template <>
__device__ __forceinline__ float t_sqrt<float>(float x) { return __fsqrt_rn(x); }

template <typename T>
__device__ __forceinline__ T t_div(T a, T b);
template <>
__device__ __forceinline__ double t_div<double>(double a, double b) { return __ddiv_rn(a, b); }
template <>
__device__ __forceinline__ float t_div<float>(float a, float b) { return __fdiv_rn(a, b); }

// interleaved pair type for two-column gathers (one 16/8-byte load per nnz)
template <typename T>
struct Pair;
template <>
struct Pair<double> {
  using type = double2;
};
template <>
struct Pair<float> {
  using type = float2;
};
template <typename T>
using pair_t = typename Pair<T>::type;

}  // namespace qpcg_b200
