// Deterministic tile-segmented SpMV engine (sm_100a, FP64, HBM-bound).
//
// Every matrix pass of the solver -- the fused PDHG step kernels, the check
// (KKT) passes, Ruiz/Pock-Chambolle norms and power sums, the power
// iteration -- is one instantiation of `tile_kernel<Op>` over a compressed
// matrix in CSR role (segments = rows of K, sparse_matrix.cpp:114-125) or CSC
// role (segments = columns, sparse_matrix.cpp:127-138).
//
// Work split (balanced by nonzeros AND by segments):
//  * Tile boundaries are the union of (a) every kBlock-th segment start and
//    (b) every kTile-th nonzero inside segment groups holding more than kTile
//    nonzeros, the latter snapped back to the start of any segment of at most
//    kSnap nonzeros. So a tile holds <= kTile + kSnap nonzeros, each thread owns
//    at most one (non-empty) segment, and short segments never straddle tiles.
//  * Kernel entry: one thread issues TMA bulk copies (cp.async.bulk, one
//    mbarrier) for everything contiguous the tile needs -- the (idx, val)
//    stream, the owned segments' offsets and each per-segment epilogue
//    operand array of the Op. Nothing is staged in registers, so CTAs stay
//    light and many are resident per SM. Threads then gather the dense
//    operand(s) and overwrite the values with the rounded products in place.
//  * Owned segments of <= kSeqMax nonzeros are summed by their thread in
//    storage order -- bit-identical to the reference's serial
//    `acc += v * x[j]` loop; up to kBlock by a warp (fixed butterfly); longer
//    by the whole CTA (fixed tree). The owning thread then runs the Op's fused
//    epilogue (`finish`) with its prefetched operands.
//  * Segments longer than a tile (PageRank's sum(x) row, hub rows,
//    transportation rows) publish per-tile partials; the last CTA to arrive
//    (atomic counter per segment) sums them in tile order and runs the
//    epilogue. No floating-point atomics: every pass is bitwise reproducible.
//  * Per-tile reduction partials (KKT sums, norms) use fixed trees; finalize
//    kernels sum tiles in a fixed order.
#pragma once

#include <type_traits>
#include <utility>

#include "common.cuh"
#include "tma.cuh"

namespace pdhg {

struct Nil {};

// Ops with `bool skip()` abandon the whole launch when it returns true (the
// pipelined loop's discarded blocks); evaluated before any barrier.
// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains. Each pass kernel runs its independent prologue (the
// static matrix stream, per-segment operands written two kernels back), then
// waits for the predecessor grid (griddepcontrol.wait) before touching the
// gathered operand or writing anything, then lets its own successor launch.
// Both instructions are no-ops for normally launched kernels.
__device__ __forceinline__ void pdl_wait_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class Kern, class... Args>
inline void launch_k(Kern kernel, int grid, int block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  if (!pdl) {
    kernel<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Ops that opt into programmatic dependent launch (the per-iteration steps).
template <class T, class = void>
struct PdlOk : std::false_type {};
template <class T>
struct PdlOk<T, std::void_t<decltype(T::kPdl)>> : std::integral_constant<bool, T::kPdl> {};

template <class T, class = void>
struct HasSkip : std::false_type {};
template <class T>
struct HasSkip<T, std::void_t<decltype(std::declval<T>().skip())>> : std::true_type {};
template <class Op>
__device__ __forceinline__ bool skip_launch(const Op& op) {
  if constexpr (HasSkip<Op>::value) return op.skip();
  else return false;
}


__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }

template <bool kMax>
__device__ __forceinline__ double combine(double a, double b) {
  if constexpr (kMax) {
    return (a < b) ? b : a;  // std::max(a, b) as in RowInfNorms (sparse_matrix.cpp:170)
  } else {
    return a + b;
  }
}

template <bool kMax>
__device__ __forceinline__ double warp_combine(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = combine<kMax>(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-shape CTA reduction of R values; result valid in thread 0.
template <int R, bool kMax, int kCols>
__device__ __forceinline__ void block_combine(double (&acc)[R], double (*sh)[kCols]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc[r] = warp_combine<kMax>(acc[r]);
    if (lane == 0) sh[warp][r] = acc[r];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double v = sh[0][r];
      for (int w = 1; w < kWarps; ++w) v = combine<kMax>(v, sh[w][r]);
      acc[r] = v;
    }
  }
  __syncthreads();
}

// Op contract:
//   static constexpr int kRhs;   // 1 or 2 gathered operands
//   static constexpr int kRed;   // reduction outputs per tile (0..32)
//   static constexpr bool kMax;  // combine with max instead of +
//   static constexpr int kOps;   // per-segment operand arrays staged by TMA
//   static constexpr int kOcc;   // target resident CTAs per SM (register cap)
//   using Pre = ...;             // per-segment epilogue operands
//   __device__ void map(int32_t idx, double val, double (&p)[kRhs]) const;
//   __device__ const double* operand(int k) const;                // k < kOps
//   __device__ Pre staged(int32_t seg, const double* st, int ld) const;  // st[k*ld]
//   __device__ Pre prefetch(int32_t seg) const;                   // from global
//   __device__ void finish(int32_t seg, const double (&s)[kRhs], const Pre&, double* red) const;

// Dynamic shared-memory layout of one tile (bytes, 16-aligned regions).
constexpr int kIdxCap = kTileCap + 8;   // widened int32 range
constexpr int kValCap = kTileCap + 4;   // widened f64 range (products in place)
constexpr int kPtrCap = kBlock + 1 + 8;
constexpr int kOpsLd = kBlock + 4;      // widened f64 range per operand array
__host__ __device__ constexpr int align16(int b) { return (b + 15) & ~15; }
__host__ __device__ constexpr int smem_off_idx() { return 16; }
__host__ __device__ constexpr int smem_off_val() { return smem_off_idx() + align16(kIdxCap * 4); }
__host__ __device__ constexpr int smem_off_p2() { return smem_off_val() + align16(kValCap * 8); }
__host__ __device__ constexpr int smem_off_ptr(int rhs) { return smem_off_p2() + (rhs == 2 ? align16(kTileCap * 8) : 0); }
__host__ __device__ constexpr int smem_off_ops(int rhs) { return smem_off_ptr(rhs) + align16(kPtrCap * 4); }
__host__ __device__ constexpr int smem_bytes(int rhs, int ops) { return smem_off_ops(rhs) + ops * kOpsLd * 8; }

template <class Op>
__global__ void __launch_bounds__(kBlock, Op::kOcc) tile_kernel(const CMat M, const Op op, double* __restrict__ tile_red,
                                                         double* __restrict__ span_red) {
  if (skip_launch(op)) return;
  using Pre = typename Op::Pre;
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  constexpr int NO = Op::kOps;
  constexpr int kPer = (kTileCap + kBlock - 1) / kBlock;
  constexpr int kShCols = R > NR ? R : NR;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int32_t* s_idx = reinterpret_cast<int32_t*>(smem + smem_off_idx());
  double* s_val = reinterpret_cast<double*>(smem + smem_off_val());
  double* s_p2 = reinterpret_cast<double*>(smem + smem_off_p2());
  int32_t* s_ptr = reinterpret_cast<int32_t*>(smem + smem_off_ptr(R));
  double* s_ops = reinterpret_cast<double*>(smem + smem_off_ops(R));
  __shared__ double bsum[kWarps][kShCols];
  constexpr int kMaxLong = kTileCap / (kBlock + 1) + 1;  // segments > kBlock per tile
  __shared__ int longs[kMaxLong], longb[kMaxLong], longe[kMaxLong];
  __shared__ int nlong;
  __shared__ int fin[2];

  const int t = M.order ? M.order[blockIdx.x] : static_cast<int>(blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31;
  const int kb = M.tile_begin[t];
  const int len = M.tile_begin[t + 1] - kb;
  const int sb = M.tile_seg[t], se = M.tile_seg[t + 1];
  const int hf = M.head_first[t];
  const int nown = (se - sb) < kBlock ? (se - sb) : kBlock;  // segments staged
  // Widened (16-byte) source ranges; every thread derives the same offsets.
  uint32_t b_idx, b_val, b_ptr, b_ops;
  const int64_t a_idx = widen16<int32_t>(kb, kb + len, &b_idx);
  const int64_t a_val = widen16<double>(kb, kb + len, &b_val);
  const int64_t a_ptr = widen16<int32_t>(sb, sb + nown + 1, &b_ptr);
  const int64_t a_ops = widen16<double>(sb, sb + nown, &b_ops);
  const int o_idx = static_cast<int>(kb - a_idx), o_val = static_cast<int>(kb - a_val);
  const int o_ptr = static_cast<int>(sb - a_ptr), o_ops = static_cast<int>(sb - a_ops);

  if (tid == 0) {
    nlong = 0;
    mbar_init(bar, 1);
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t total = (len ? b_idx + b_val : 0) + b_ptr + (nown ? NO * b_ops : 0);
    mbar_expect_tx(bar, total);
    if (len) {
      bulk_g2s(s_idx, M.idx + a_idx, b_idx, bar);
      bulk_g2s(s_val, M.val + a_val, b_val, bar);
    }
    bulk_g2s(s_ptr, M.ptr + a_ptr, b_ptr, bar);
    if (nown) {
#pragma unroll
      for (int k = 0; k < NO; ++k) bulk_g2s(s_ops + k * kOpsLd, op.operand(k) + a_ops, b_ops, bar);
    }
  }
  mbar_wait(bar, 0);
  pdl_wait_trigger();

  // ---- Gather + rounded products, in place over the staged values.
  {
    const int32_t* ix = s_idx + o_idx;
    double* pv = s_val + o_val;
    double g[kPer][R];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int q = tid + i * kBlock;
      if (q < len) op.map(ix[q], pv[q], g[i]);
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int q = tid + i * kBlock;
      if (q < len) {
        pv[q] = g[i][0];
        if constexpr (R == 2) s_p2[q] = g[i][1];
      }
    }
  }
  __syncthreads();
  const double* prod[2] = {s_val + o_val, s_p2};

  // Owned segment of this thread (round 0), operands from shared memory.
  const int s0 = sb + tid;
  const bool own0 = tid < nown;
  int b0 = 0, e0 = 0;
  Pre pre0{};
  if (own0) {
    const int p0 = s_ptr[o_ptr + tid];
    b0 = (p0 > kb ? p0 : kb) - kb;
    e0 = s_ptr[o_ptr + tid + 1] - kb;
    pre0 = op.staged(s0, s_ops + o_ops + tid, kOpsLd);
  }

  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;

  // Deliver a finished sum for owned segment s: head partial or epilogue.
  auto deliver = [&](int s, const double (&acc)[R], const Pre& pre) {
    if (s == sb && hf >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) M.head_part[2 * t + r] = acc[r];
      __threadfence();
    } else {
      op.finish(s, acc, pre, red);
    }
  };

  // ---- Owned segments (round 0 has its operands prefetched; further rounds
  // only occur when a tile owns more than kBlock empty segments).
  for (int base = sb; base < se; base += kBlock) {
    const int s = base + tid;
    const bool own = s < se;
    int b = b0, e = e0;
    Pre pre = pre0;
    if (base != sb && own) {
      const int p0 = M.ptr[s];
      b = (p0 > kb ? p0 : kb) - kb;
      e = M.ptr[s + 1] - kb;
      pre = op.prefetch(s);
    }
    const int n = e - b;
    if (own && n <= kSeqMax) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      for (int q = b; q < e; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], prod[r][q]);
      }
      deliver(s, acc, pre);
    }
    // 33..kBlock: one warp per segment (owner lane finishes).
    const bool mid = own && n > kSeqMax && n <= kBlock;
    unsigned mask = __ballot_sync(0xffffffffu, mid);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int b2 = __shfl_sync(0xffffffffu, b, src);
      const int e2 = __shfl_sync(0xffffffffu, e, src);
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      for (int q = b2 + lane; q < e2; q += 32) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], prod[r][q]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = warp_combine<MX>(acc[r]);
      if (lane == src) deliver(s, acc, pre);
    }
    // > kBlock: the whole CTA, one segment at a time.
    if (own && n > kBlock) {
      const int k = atomicAdd(&nlong, 1);
      longs[k] = tid;
      longb[k] = b;
      longe[k] = e;
    }
    __syncthreads();
    const int nl = nlong;
    for (int k = 0; k < nl; ++k) {
      const int owner = longs[k];
      const int s2 = base + owner;
      const int bb = longb[k], ee = longe[k];
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      for (int q = bb + tid; q < ee; q += kBlock) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], prod[r][q]);
      }
      block_combine<R, MX, kShCols>(acc, bsum);
      if (tid == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) bsum[0][r] = acc[r];
      }
      __syncthreads();
      if (tid == owner) {
        double tot[R];
#pragma unroll
        for (int r = 0; r < R; ++r) tot[r] = bsum[0][r];
        deliver(s2, tot, pre);
      }
      __syncthreads();
    }
    __syncthreads();
    if (tid == 0) nlong = 0;
    __syncthreads();
  }

  // ---- Tail: the segment that starts in (or passes through) this tile but
  // ends in a later one.
  const int to = M.tail_owner[t];
  if (to >= 0) {
    const int p0 = M.ptr[se];
    const int b = (p0 > kb ? p0 : kb) - kb;
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int q = b + tid; q < len; q += kBlock) {
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], prod[r][q]);
    }
    block_combine<R, MX, kShCols>(acc, bsum);
    if (tid == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) M.tail_part[2 * t + r] = acc[r];
      __threadfence();
    }
  }

  // ---- Per-tile reduction partials (fixed trees).
  if constexpr (Op::kRed > 0) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Op::kRed; ++i) {
      const double v = warp_combine<false>(red[i]);
      if (lane == 0) bsum[tid >> 5][i] = v;
    }
    __syncthreads();
    if (tid < Op::kRed) {
      double v = bsum[0][tid];
      for (int w = 1; w < kWarps; ++w) v += bsum[w][tid];
      tile_red[static_cast<int64_t>(t) * Op::kRed + tid] = v;
      if (hf < 0) span_red[static_cast<int64_t>(t) * Op::kRed + tid] = 0.0;
    }
  }

  // ---- Cross-tile segments, finished by the last arriving CTA.
  if (hf < 0 && to < 0) return;  // uniform across the CTA
  __syncthreads();
  if (tid == 0) {
    fin[0] = -1;
    fin[1] = -1;
    if (hf >= 0) {
      const unsigned old = atomicAdd(&M.counter[t], 1u);
      if (old == static_cast<unsigned>(t - hf)) fin[0] = t;
    }
    if (to >= 0) {
      const int hf2 = M.head_first[to];
      const unsigned old = atomicAdd(&M.counter[to], 1u);
      if (old == static_cast<unsigned>(to - hf2)) fin[1] = to;
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int w = 0; w < 2; ++w) {
    const int o = fin[w];
    if (o < 0) continue;
    __threadfence();
    const int f = M.head_first[o];
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int i = f + tid; i < o; i += kBlock) {
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], __ldcg(M.tail_part + 2 * i + r));
    }
    block_combine<R, MX, kShCols>(acc, bsum);
    if (tid == 0) {
      double s[R];
#pragma unroll
      for (int r = 0; r < R; ++r) s[r] = combine<MX>(acc[r], __ldcg(M.head_part + 2 * o + r));
      double red2[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) red2[i] = 0.0;
      const int seg = M.tile_seg[o];
      op.finish(seg, s, op.prefetch(seg), red2);
      if constexpr (Op::kRed > 0) {
        for (int i = 0; i < Op::kRed; ++i) span_red[static_cast<int64_t>(o) * Op::kRed + i] = red2[i];
      }
      M.counter[o] = 0u;
    }
    __syncthreads();
  }
}

template <class Op>
inline void launch_tiles(const CMat& M, const Op& op, double* tile_red, double* span_red, cudaStream_t st,
                         bool pdl = false) {
  constexpr int bytes = smem_bytes(Op::kRhs, Op::kOps);
  smem_opt_in<tile_kernel<Op>>(bytes);
  launch_k(tile_kernel<Op>, M.ntiles, kBlock, bytes, st, pdl, M, op, tile_red, span_red);
}

}  // namespace pdhg
