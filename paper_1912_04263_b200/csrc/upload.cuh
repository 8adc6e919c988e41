// upload.cuh — host -> device copies of the problem from PAGEABLE memory.
//
// The reference's callers hand over std::vector / numpy buffers, i.e.
// pageable memory.  cudaMemcpyAsync from pageable memory blocks the calling
// thread and moves ~10 GB/s through the driver's own staging buffer.  Here a
// large pageable source is copied by several host threads into a pinned
// staging ring (per device, process-wide) whose chunks the DMA engine drains
// while the next chunk is being filled; pinned sources go straight to
// cudaMemcpyAsync.  The copy of A's values can run on a background host
// thread (Workspace::load), so the structural setup on the GPU overlaps it.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace qpcg_b200 {

constexpr size_t kStageChunk = size_t(64) << 20;  // bytes per staging slot
constexpr int kStageSlots = 2;
constexpr size_t kStageMin = size_t(8) << 20;    // smaller copies: plain cudaMemcpyAsync

inline bool host_is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// memcpy split over up to `threads` host threads
inline void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
  const size_t min_part = size_t(4) << 20;
  const int t = int(std::max<size_t>(1, std::min<size_t>(size_t(threads), bytes / min_part)));
  if (t <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(t - 1);
  auto part = [&](int i) {
    const size_t lo = bytes * i / t, hi = bytes * (i + 1) / t;
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  };
  for (int i = 1; i < t; ++i) th.emplace_back(part, i);
  part(0);
  for (auto& x : th) x.join();
}

// One per device: a pinned ring of kStageSlots chunks; one copy at a time.
class Stager {
 public:
  explicit Stager(int device) : device_(device) {}
  // dst (device) <- src (pageable host), ordered on stream st; returns when
  // the last chunk is queued (the DMA may still be running on st)
  cudaError_t copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu_);
    cudaError_t e = ensure();
    if (e != cudaSuccess) return e;
    const int threads = std::max(1, std::min(8, int(std::thread::hardware_concurrency())));
    size_t off = 0;
    for (int i = 0; off < bytes; ++i, off += kStageChunk) {
      const int k = i % kStageSlots;
      const size_t n = std::min(kStageChunk, bytes - off);
      if ((e = cudaEventSynchronize(ev_[k])) != cudaSuccess) return e;  // slot drained
      parallel_memcpy(buf_[k], static_cast<const char*>(src) + off, n, threads);
      if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[k], n, cudaMemcpyHostToDevice,
                               st)) != cudaSuccess)
        return e;
      if ((e = cudaEventRecord(ev_[k], st)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  ~Stager() = default;  // process lifetime (freed with the context)

 private:
  cudaError_t ensure() {
    if (buf_[0]) return cudaSuccess;
    cudaError_t e;
    for (int k = 0; k < kStageSlots; ++k) {
      if ((e = cudaHostAlloc(&buf_[k], kStageChunk, cudaHostAllocPortable)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&ev_[k], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  int device_;
  std::mutex mu_;
  void* buf_[kStageSlots] = {};
  cudaEvent_t ev_[kStageSlots] = {};
};

inline Stager& stager_for(int device) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<Stager>> all;
  std::lock_guard<std::mutex> g(mu);
  if (device < 0) device = 0;
  if (all.size() <= size_t(device)) all.resize(size_t(device) + 1);
  if (!all[device]) all[device].reset(new Stager(device));
  return *all[device];
}

// H2D of `bytes` from host memory of either kind, ordered on st.
inline cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st, int device) {
  if (bytes == 0) return cudaSuccess;
  if (bytes < kStageMin || !host_is_pageable(src))
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  return stager_for(device).copy(dst, src, bytes, st);
}

}  // namespace qpcg_b200
