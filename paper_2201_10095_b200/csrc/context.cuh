// Execution context: one CUDA stream plus a growable device scratch arena.
// One context per stream; concurrent calls must use distinct contexts
// (SURVEY §8b threading contract).
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "scan_sort.cuh"

namespace rs {
// Cache of pinned host blocks.  Results handed to the caller (profile rows /
// CDFs) live in pinned memory so the D2H copies run at full PCIe speed;
// cudaHostAlloc costs milliseconds per 100 MB, so blocks are recycled.
// Shared by the context and the results that hold blocks, so either may go
// first.
struct PinnedPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;
  ~PinnedPool() {
    for (auto& kv : free_blocks) cudaFreeHost(kv.second);
  }
  // returns a block of at least `bytes` (its capacity in *cap)
  void* take(size_t bytes, size_t* cap) {
    bytes = std::max<size_t>((bytes + 4095) & ~size_t(4095), 4096);
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free_blocks.lower_bound(bytes);
      if (it != free_blocks.end() && it->first <= 2 * bytes + (64 << 20)) {
        void* p = it->second;
        *cap = it->first;
        free_blocks.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    RS_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
    *cap = bytes;
    return p;
  }
  void give(void* p, size_t cap) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu);
    free_blocks.emplace(cap, p);
  }
};
}  // namespace rs

struct rs_context {
  std::shared_ptr<rs::PinnedPool> host_pool = std::make_shared<rs::PinnedPool>();
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  char* arena = nullptr;
  size_t arena_cap = 0;
  char* pinned = nullptr;  // small pinned staging area for D2H scalars
  size_t pinned_cap = 0;

  // Returns a scratch view with at least `bytes` capacity.  Growing the arena
  // synchronises the stream first (the old arena may still be in use).
  rs::Scratch scratch(size_t bytes) {
    bytes = (bytes + (1 << 20)) & ~size_t((1 << 20) - 1);
    if (bytes > arena_cap) {
      RS_CUDA(cudaStreamSynchronize(stream));
      if (arena) RS_CUDA(cudaFree(arena));
      arena = nullptr;
      arena_cap = 0;
      RS_CUDA(cudaMalloc(&arena, bytes));
      arena_cap = bytes;
    }
    rs::Scratch s;
    s.base = arena;
    s.cap = arena_cap;
    return s;
  }

  template <class T>
  T* pinned_buf(size_t n) {
    size_t bytes = n * sizeof(T);
    if (bytes > pinned_cap) {
      RS_CUDA(cudaStreamSynchronize(stream));
      if (pinned) RS_CUDA(cudaFreeHost(pinned));
      pinned = nullptr;
      size_t cap = bytes < 4096 ? 4096 : bytes;
      RS_CUDA(cudaHostAlloc(&pinned, cap, cudaHostAllocDefault));
      pinned_cap = cap;
    }
    return reinterpret_cast<T*>(pinned);
  }

  void sync() { RS_CUDA(cudaStreamSynchronize(stream)); }

  // Releases the scratch arena (it holds no data between calls).  A profile
  // of a huge table set (RM3: ~2^31 counters per group) leaves an arena of
  // ~150 GB; an operator created on the same context next needs that HBM.
  void trim_scratch() {
    if (!arena) return;
    RS_CUDA(cudaStreamSynchronize(stream));
    RS_CUDA(cudaFree(arena));
    arena = nullptr;
    arena_cap = 0;
  }
};

namespace rs {

// True if `p` is device-accessible memory (device or managed allocation).
inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Copies a host or device array into scratch (device) memory.
template <class T>
T* stage(const T* src, size_t n, bool src_on_device, Scratch& scr, cudaStream_t st) {
  T* d = scr.take<T>(n ? n : 1);
  if (n)
    RS_CUDA(cudaMemcpyAsync(d, src, n * sizeof(T),
                            src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            st));
  return d;
}

}  // namespace rs
