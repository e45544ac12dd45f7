// Persistent block kernel: `count` PDHG iterations in ONE cooperative launch.
//
// A transportation-size LP (BASELINE configs[1]: 2M nonzeros) keeps most of
// its 96 MB per-iteration working set in the 126 MB L2 across iterations:
// ncu over graph-launched 64-step blocks counts 17 MB of DRAM traffic per
// iteration (profiles/r02/), and L2 streams at ~21 TB/s on this B200
// (tools/dsmem_probe.cu, l2seq). The two step kernels then spend their time
// in launch, ramp and tail, not in moving bytes: 14.4 us per iteration
// against ~4.5 us of L2 traffic. Here every CTA stays resident for the whole
// block and walks the step passes' CTA-sized work items itself:
//   for j in block: primal items (K-CSC) -> grid barrier -> dual items
//   (K-CSR) -> grid barrier.
// The items are the standalone kernels' bodies (engine.cuh uniform_item,
// cta4_item) with an explicit block index, so every per-segment sum and
// epilogue is the same arithmetic in the same order: results are bitwise
// identical to the two-kernel path. The grid barrier is an arrival counter
// (zeroed before each launch) with release/acquire at gpu scope; its
// gpu-scope fence also invalidates the SM's L1 (CCTL.IVALL), so no CTA reads
// a line of the previous phase's vector from L1. The launch is cooperative:
// the driver guarantees every CTA is co-resident or refuses the launch.
//
// Scope: single-shard sessions whose CSC is one uniform-length class S
// (transport, assignment-type columns) and whose CSR is one class L of
// 4-row TMA-staged groups (Session::PersistOk); other layouts keep the
// two-kernel path.
//
// Measured on the B200 (transport 1000x1000, profiles/r02/block_kernel_r02u.txt):
// SLOWER, so opt-in (PDHG_PERSIST=1). 19.8 us per iteration against 14.3 us
// for the two PDL-chained kernels: the grid barrier alone costs 2.5 us (592
// CTAs arriving on one counter and polling it), the primal pass takes
// 9.2 us at 4 resident CTAs per SM (the merged kernel needs 64 registers;
// the standalone uniform kernel runs 8 at 32), the dual pass 5.8 us (8.2 us
// standalone: its stream is issued before the barrier). Beating the two
// kernels needs a sub-microsecond hierarchical barrier and a TMA-streamed
// primal phase. Tried and no better (r02v): cooperative_groups' grid sync or
// a release-add / relaxed-poll barrier (19.2 us), two primal blocks per CTA
// in flight (21.5-22.2 us).
#pragma once

#include "engine.cuh"

namespace pdhg {

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

template <class OpP, class OpD>
struct BlockArgs {
  // K-CSC: class S, uniform length (implicit offsets), modal prefix s_u
  const int32_t* p_idx;
  const double* p_val;
  const int32_t* p_ptr;
  int32_t p_send, p_su;
  int p_nb;
  // K-CSR: class L [d_s2, d_s3), 4 rows per item, stream staged by TMA
  const int32_t* d_ptr;
  const int32_t* d_idx;
  const double* d_val;
  int32_t d_s2, d_s3;
  int d_nb;
  OpP opp[2];  // by buffer parity
  OpD opd[2];
  int parity, count;
  unsigned* gbar;
};

template <class OpP, class OpD, int LP, bool kPrefixP>
__global__ void __launch_bounds__(kBlock, kCtaMinBlocks) pdhg_block_kernel(const BlockArgs<OpP, OpD> a) {
  extern __shared__ __align__(16) unsigned char stage[];
  __shared__ uint64_t bar;
  __shared__ double sh[kBlock / 32][4][1];
  const unsigned G = gridDim.x;
  unsigned target = 0;
  for (int j = 0; j < a.count; ++j) {
    const int q = (a.parity + j) & 1;
    OpP op = a.opp[q];
    op.j_in_block = j;
    for (int blk = blockIdx.x; blk < a.p_nb; blk += G)
      uniform_item<OpP, LP, kPrefixP>(blk, a.p_idx, a.p_val, a.p_send, op, nullptr, a.p_ptr, a.p_su);
    // This CTA's first dual group streams its matrix range while the grid
    // waits for the primal pass (the role PDL plays between the kernels).
    const bool first = static_cast<int>(blockIdx.x) < a.d_nb;
    if (first) {
      __syncthreads();  // the previous dual group's readers are done with the stage
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (threadIdx.x == 0) cta4_issue(blockIdx.x, a.d_ptr, a.d_idx, a.d_val, a.d_s2, a.d_s3, stage, &bar);
    }
    target += G;
    grid_barrier(a.gbar, target);
    OpD od = a.opd[q];
    od.j_in_block = j;
    if (first)
      cta4_item<OpD, true, true>(blockIdx.x, a.d_ptr, a.d_idx, a.d_val, a.d_s2, a.d_s3, od, nullptr, stage, &bar, sh);
    for (int blk = blockIdx.x + G; blk < a.d_nb; blk += G)
      cta4_item<OpD, true>(blk, a.d_ptr, a.d_idx, a.d_val, a.d_s2, a.d_s3, od, nullptr, stage, &bar, sh);
    target += G;
    grid_barrier(a.gbar, target);
  }
}

// Co-resident CTAs of one block kernel (cached per kernel and device).
inline int block_kernel_grid(const void* kernel, int smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  PDHG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find({kernel, dev});
  if (it != cache.end()) return it->second;
  int per = 0, sms = 0;
  PDHG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kBlock, smem));
  PDHG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int v = std::max(1, per) * sms;
  cache[{kernel, dev}] = v;
  return v;
}

template <class OpP, class OpD, int LP, bool kPrefixP>
inline void launch_block_kernel(const BlockArgs<OpP, OpD>& a, int smem, cudaStream_t st) {
  auto kern = pdhg_block_kernel<OpP, OpD, LP, kPrefixP>;
  if (smem > 48 * 1024) smem_opt_in<pdhg_block_kernel<OpP, OpD, LP, kPrefixP>>(smem);
  const int grid = std::min(block_kernel_grid(reinterpret_cast<const void*>(kern), smem), std::max(a.p_nb, a.d_nb));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PDHG_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
}

template <class OpP, class OpD>
inline void launch_block(const BlockArgs<OpP, OpD>& a, int lp, bool prefix, int smem, cudaStream_t st) {
#define PDHG_BLOCK(L)                                                               \
  case L:                                                                           \
    if (prefix) return launch_block_kernel<OpP, OpD, L, true>(a, smem, st);         \
    return launch_block_kernel<OpP, OpD, L, false>(a, smem, st);
  switch (lp) {
    PDHG_BLOCK(1)
    PDHG_BLOCK(2)
    PDHG_BLOCK(3)
    PDHG_BLOCK(4)
    PDHG_BLOCK(8)
    default: throw Error(3, "persistent block kernel: unsupported uniform length");
  }
#undef PDHG_BLOCK
}

}  // namespace pdhg
