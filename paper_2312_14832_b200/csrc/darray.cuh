// Owning device array over a per-device stream-ordered memory pool.
//
// Sessions are short-lived in the drop-in path (one per Solve call) and build
// ~100 arrays each; cudaMalloc / cudaFree map and unmap device memory and
// synchronise the whole device on every call. The pool keeps up to
// kPoolKeepBytes reserved across sessions, so after the first solve an
// allocation is a user-mode free-list hit. Frees stay as strict as cudaFree
// was: the stream that used the buffer (the session stream, published by an
// AllocScope) is synchronised first -- or the device, outside any scope.
#pragma once

#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace pdhg {

struct Arena {
  int64_t bytes = 0;
};

constexpr uint64_t kPoolKeepBytes = uint64_t(8) << 30;  // reserve kept at sync points

// The calling thread's session stream (AllocScope); nullptr outside sessions.
inline cudaStream_t& alloc_stream() {
  thread_local cudaStream_t s = nullptr;
  return s;
}

struct AllocScope {
  cudaStream_t prev;
  explicit AllocScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~AllocScope() { alloc_stream() = prev; }
  AllocScope(const AllocScope&) = delete;
  AllocScope& operator=(const AllocScope&) = delete;
};

// One pool + one never-destroyed allocation stream per device.
struct DevicePool {
  cudaMemPool_t pool = nullptr;
  cudaStream_t stream = nullptr;
};

inline DevicePool* device_pool(int dev) {
  static std::mutex mu;
  static std::vector<DevicePool> pools;
  std::lock_guard<std::mutex> lk(mu);
  if (pools.empty()) {
    int n = 0;
    PDHG_CUDA(cudaGetDeviceCount(&n));
    pools.resize(static_cast<size_t>(n));
  }
  DevicePool& p = pools.at(static_cast<size_t>(dev));
  if (!p.pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    PDHG_CUDA(cudaMemPoolCreate(&p.pool, &props));
    uint64_t keep = kPoolKeepBytes;
    PDHG_CUDA(cudaMemPoolSetAttribute(p.pool, cudaMemPoolAttrReleaseThreshold, &keep));
    PDHG_CUDA(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
  }
  return &p;
}

// Process-wide cache of pinned host blocks: cudaMallocHost page-locks and
// cudaFreeHost unlocks memory (milliseconds at staging sizes, and both
// serialise with the driver), so sessions return their blocks here.
constexpr size_t kPinnedKeepBytes = size_t(1) << 30;

struct PinnedCache {
  std::mutex mu;
  std::multimap<size_t, void*> free;
  size_t bytes = 0;
};

inline PinnedCache& pinned_cache() {
  static PinnedCache* c = new PinnedCache;  // never destroyed: blocks outlive static teardown
  return *c;
}

// A block of at least `bytes` (reused when no larger than 4x the request).
inline void* pinned_get(size_t bytes, size_t* got) {
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free.lower_bound(bytes);
    if (it != c.free.end() && it->first <= 4 * bytes + 4096) {
      void* p = it->second;
      *got = it->first;
      c.bytes -= it->first;
      c.free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  PDHG_CUDA(cudaMallocHost(&p, bytes));
  *got = bytes;
  return p;
}

inline void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.bytes + bytes <= kPinnedKeepBytes) {
      c.free.emplace(bytes, p);
      c.bytes += bytes;
      return;
    }
  }
  cudaFreeHost(p);
}

template <class T>
struct DArray {
  T* p = nullptr;
  size_t n = 0;
  Arena* arena = nullptr;
  int dev = 0;
  cudaStream_t user = nullptr;  // stream synchronised before the free

  DArray() = default;
  DArray(const DArray&) = delete;
  DArray& operator=(const DArray&) = delete;
  ~DArray() { release(); }

  void alloc(size_t count, Arena* a = nullptr) {
    release();
    arena = a;
    n = count;
    if (count) {
      PDHG_CUDA(cudaGetDevice(&dev));
      user = alloc_stream();
      DevicePool* dp = device_pool(dev);
      // 32 bytes of tail slack: TMA bulk copies widen ranges to 16 bytes
      // (the widened elements are staged but never consumed).
      PDHG_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), count * sizeof(T) + 32, dp->pool, dp->stream));
      PDHG_CUDA(cudaStreamSynchronize(dp->stream));  // usable from every stream
      if (arena) arena->bytes += static_cast<int64_t>(count * sizeof(T));
    }
  }
  void release() {
    if (p) {
      int cur = 0;
      cudaGetDevice(&cur);
      if (cur != dev) cudaSetDevice(dev);
      if (user) cudaStreamSynchronize(user);
      else cudaDeviceSynchronize();
      cudaFreeAsync(p, device_pool(dev)->stream);
      if (cur != dev) cudaSetDevice(cur);
      if (arena) arena->bytes -= static_cast<int64_t>(n * sizeof(T));
    }
    p = nullptr;
    n = 0;
    user = nullptr;
  }
  // Ownership transfer (e.g. a setup temporary becoming session storage).
  void take(DArray& o, Arena* a) {
    release();
    p = o.p;
    n = o.n;
    dev = o.dev;
    user = o.user;
    arena = a;
    if (o.arena) o.arena->bytes -= static_cast<int64_t>(o.n * sizeof(T));
    if (arena) arena->bytes += static_cast<int64_t>(n * sizeof(T));
    o.p = nullptr;
    o.n = 0;
    o.user = nullptr;
  }
  T* get() const { return p; }
  size_t size() const { return n; }
};

}  // namespace pdhg
