// Shared definitions for the B200 restarted-PDHG library.
#pragma once

#include <algorithm>
#include <atomic>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace pdhg {

// NVTX range for the duration of a scope (session setup, scaling, the power
// iteration, the loop, every check, finish): names show up in Nsight
// Systems / Compute timelines (`ncu --nvtx --nvtx-include "pdhg.loop/"`).
// Without an attached tool each push / pop is a no-op call.
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

// Error carrying a C-ABI code (include/pdhg.h).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PDHG_CUDA(call)                                                     \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      throw ::pdhg::Error(3, std::string(#call) + ": " +                   \
                                 cudaGetErrorString(e_) + " (" __FILE__ ")"); \
  } while (0)

// Opt a kernel into more than 48 KB of dynamic shared memory, once per
// (kernel, device): the attribute belongs to the device the calling thread
// has current, so a process that drives several GPUs must set it on each.
// One static per kernel (non-type template parameter), a bit per device.
template <auto Kernel>
inline void smem_opt_in(int bytes) {
  static std::atomic<uint64_t> opted{0};
  int dev = 0;
  PDHG_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (opted.load(std::memory_order_acquire) & bit) return;
  PDHG_CUDA(cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  opted.fetch_or(bit, std::memory_order_release);
}

// Tile geometry of the segmented SpMV engine (see tile_spmv.cuh).
constexpr int kBlock = 256;        // threads per CTA
constexpr int kTile = 2048;        // nominal nonzeros per tile
constexpr int kSnap = 64;          // segments this short never straddle tiles
constexpr int kSeqMax = 32;        // segments up to this length: one thread, in order
constexpr int kWarpMax = 512;      // segments up to this length: one warp
constexpr int kCtaMax = 16384;     // segments up to this length: one CTA
constexpr int kTileCap = kTile + kSnap;
constexpr int kWarps = kBlock / 32;

// A compressed sparse matrix in either role: CSR (segments = rows, gathered
// vector indexed by columns) or CSC (segments = columns). Int32 indices,
// FP64 values; nnz < 2^31 is enforced at upload.
struct CMat {
  int32_t nseg = 0;  // rows (CSR) or columns (CSC)
  int32_t nvec = 0;  // length of the gathered vector
  int64_t nnz = 0;
  int32_t* ptr = nullptr;  // nseg + 1
  int32_t* idx = nullptr;  // nnz
  double* val = nullptr;   // nnz
  // Tile partition (computed once per matrix, tile_partition in kernels.cu).
  int32_t ntiles = 0;
  int32_t* tile_begin = nullptr;  // ntiles + 1 nonzero offsets
  int32_t* tile_seg = nullptr;    // ntiles + 1 first owned segment
  int32_t* head_first = nullptr;  // ntiles: first tile of the spanning head segment or -1
  int32_t* tail_owner = nullptr;  // ntiles: owner tile of the spanning tail segment or -1
  // Cross-tile scratch for segments longer than a tile.
  double* head_part = nullptr;  // ntiles * 2
  double* tail_part = nullptr;  // ntiles * 2
  unsigned* counter = nullptr;  // ntiles, zero between launches
  // Execution order (CTA b runs tile order[b]) or null (b runs tile b):
  // tiles sorted by the gathered index of their first nonzero, so the CTAs
  // resident at any moment gather from one narrow, L2-resident window of the
  // vector instead of every long segment's whole span (session.cu
  // PartitionLong). Every per-tile output is indexed by the tile, and the
  // cross-tile combination sums in tile order: results do not depend on it.
  const int32_t* order = nullptr;
};

// Device-resident solver scalars: the iteration kernels read these instead
// of taking per-iteration host arguments, so a 64-iteration block can be
// replayed as one CUDA graph.
// Elementwise kernels: grid-stride loops over at most 16 CTAs per SM.
constexpr int kEw = 256;  // elementwise block size

inline int ew_grid(int64_t n) {
  int64_t g = (n + kEw - 1) / kEw;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16)));
}

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

struct Scalars {
  double eta;
  double omega;
  double inner_base;  // RunningAverage weight at the start of the block
  double pw_norm;     // power iteration: norm of the current vector
  int32_t pw_zero;    // power iteration hit a zero vector
  int32_t halt;       // pipelined loop: skip queued blocks until the host clears it
  double adapt_iter;  // iterations_ at the start of the block (adaptive step)
  double lb, ub;      // the common scaled bound when every column shares it
  double step_p;      // eta / omega: the primal step (solver.cpp:285-290), set with eta / omega
  double step_d;      // eta * omega: the dual step (solver.cpp:292-298)
};

// The step sizes the step kernels read, derived once per change of eta or
// omega instead of once per thread (IEEE division on host and device alike).
__host__ __device__ inline void set_steps(Scalars& s) {
  s.step_p = s.eta / s.omega;
  s.step_d = s.eta * s.omega;
}

// Clamp with the reference's NaN behaviour: std::min(std::max(v, lo), hi)
// (solver.cpp:33-35) returns NaN for NaN input; fmin/fmax would mask it.
__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) {
  v = (v < lo) ? lo : v;        // std::max(v, lo) == (v < lo ? lo : v)
  return (hi < v) ? hi : v;     // std::min(v, hi) == (hi < v ? hi : v)
}
__device__ __forceinline__ double max0_ref(double v) { return (v < 0.0) ? 0.0 : v; }
__device__ __forceinline__ double min0_ref(double v) { return (0.0 < v) ? 0.0 : v; }

// ProjectReducedCost (kkt.cpp:29-41). cls: 0 free, 1 upper-only,
// 2 lower-only, 3 boxed (lp_problem.cpp:60-67).
__device__ __forceinline__ int bound_class(double lo, double hi) {
  const bool a = isfinite(lo), b = isfinite(hi);
  return (!a && !b) ? 0 : (!a ? 1 : (!b ? 2 : 3));
}
__device__ __forceinline__ double project_reduced(double v, int cls) {
  // std::min(v, 0.0) == (0.0 < v ? 0.0 : v); std::max(v, 0.0) == (v < 0.0 ? 0.0 : v)
  return cls == 0 ? 0.0 : (cls == 1 ? min0_ref(v) : (cls == 2 ? max0_ref(v) : v));
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace pdhg
