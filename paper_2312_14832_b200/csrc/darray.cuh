// Minimal owning device array.
#pragma once

#include "common.cuh"

namespace pdhg {

struct Arena {
  int64_t bytes = 0;
};

template <class T>
struct DArray {
  T* p = nullptr;
  size_t n = 0;
  Arena* arena = nullptr;

  DArray() = default;
  DArray(const DArray&) = delete;
  DArray& operator=(const DArray&) = delete;
  ~DArray() { release(); }

  void alloc(size_t count, Arena* a = nullptr) {
    release();
    arena = a;
    n = count;
    if (count) {
      // 32 bytes of tail slack: TMA bulk copies widen ranges to 16 bytes
      // (the widened elements are staged but never consumed).
      PDHG_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T) + 32));
      if (arena) arena->bytes += static_cast<int64_t>(count * sizeof(T));
    }
  }
  void release() {
    if (p) {
      cudaFree(p);
      if (arena) arena->bytes -= static_cast<int64_t>(n * sizeof(T));
    }
    p = nullptr;
    n = 0;
  }
  // Ownership transfer (e.g. a setup temporary becoming session storage).
  void take(DArray& o, Arena* a) {
    release();
    p = o.p;
    n = o.n;
    arena = a;
    if (o.arena) o.arena->bytes -= static_cast<int64_t>(o.n * sizeof(T));
    if (arena) arena->bytes += static_cast<int64_t>(n * sizeof(T));
    o.p = nullptr;
    o.n = 0;
  }
  T* get() const { return p; }
  size_t size() const { return n; }
};

}  // namespace pdhg
