// Deterministic tile-segmented SpMV engine (sm_100a, FP64, HBM-bound).
//
// Every matrix pass of the solver -- the fused PDHG step kernels, the check
// (KKT) passes, Ruiz/Pock-Chambolle norms and power sums, the power
// iteration -- is one instantiation of `tile_kernel<Op>` over a compressed
// matrix in CSR role (segments = rows of K, sparse_matrix.cpp:114-125) or CSC
// role (segments = columns, sparse_matrix.cpp:127-138).
//
// Work split (merge-path style, balanced by nonzeros, not by segments):
//  * The nonzero stream is cut into tiles of ~kTile entries. A tile start is
//    snapped back to its segment's start when that segment is at most kSnap
//    long, so short segments never straddle tiles.
//  * Phase 1: the CTA streams its tile's (idx, val) pairs with coalesced,
//    evict-first loads, gathers the dense operand(s), and stages the rounded
//    products in shared memory.
//  * Phase 2: segments owned by the tile (those whose last nonzero lies in
//    it) are summed from shared memory: segments of <= kSeqMax nonzeros by
//    one thread in storage order -- bit-identical to the reference's serial
//    `acc += v * x[j]` loop -- and longer ones by a warp with a fixed
//    butterfly. The Op's epilogue (`finish`) then runs the fused per-row or
//    per-column update and accumulates reduction partials.
//  * Segments longer than a tile (the PageRank sum(x) row, hub rows,
//    transportation rows): each tile they cross publishes a partial; the
//    last CTA to arrive (atomic counter per segment) sums the partials in
//    tile order and runs the epilogue. No floating-point atomics anywhere, so
//    every pass is bitwise reproducible run to run.
//  * Phase 3: per-tile reduction partials are combined with fixed trees;
//    finalize kernels sum tiles in a fixed order.
#pragma once

#include "common.cuh"

namespace pdhg {

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

// Op contract:
//   static constexpr int kRhs;   // 1 or 2 gathered operands
//   static constexpr int kRed;   // reduction outputs per tile (0..32)
//   static constexpr bool kMax;  // combine with max instead of +
//   __device__ void map(int32_t idx, double val, double (&p)[kRhs]) const;
//   __device__ void finish(int32_t seg, const double (&s)[kRhs], double* red) const;
template <class Op>
__global__ void __launch_bounds__(kBlock) tile_kernel(const CMat M, const Op op, double* __restrict__ tile_red,
                                                      double* __restrict__ span_red) {
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  constexpr int kPer = (kTileCap + kBlock - 1) / kBlock;
  __shared__ double prod[R][kTileCap];
  __shared__ double bsum[kWarps][R > NR ? R : NR];
  __shared__ int fin[2];

  const int t = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = M.tile_begin[t];
  const int len = M.tile_begin[t + 1] - kb;

  // ---- Phase 1: stream the tile, gather, stage rounded products.
  {
    int32_t ix[kPer];
    double vv[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int q = tid + i * kBlock;
      if (q < len) {
        ix[i] = ld_stream(M.idx + kb + q);
        vv[i] = ld_stream(M.val + kb + q);
      }
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int q = tid + i * kBlock;
      if (q < len) {
        double p[R];
        op.map(ix[i], vv[i], p);
#pragma unroll
        for (int r = 0; r < R; ++r) prod[r][q] = p[r];
      }
    }
  }
  __syncthreads();

  const int sb = M.tile_seg[t], se = M.tile_seg[t + 1];
  const int hf = M.head_first[t];
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;

  // ---- Phase 2: owned segments.
  for (int base = sb; base < se; base += kBlock) {
    const int s = base + tid;
    const bool active = s < se;
    int b = 0, e = 0;
    if (active) {
      const int p0 = M.ptr[s];
      b = (p0 > kb ? p0 : kb) - kb;
      e = M.ptr[s + 1] - kb;
    }
    const bool longseg = active && (e - b > kSeqMax);
    if (active && !longseg) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      for (int q = b; q < e; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], prod[r][q]);
      }
      if (s == sb && hf >= 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) M.head_part[2 * t + r] = acc[r];
        __threadfence();
      } else {
        op.finish(s, acc, red);
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, longseg);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int b2 = __shfl_sync(0xffffffffu, b, src);
      const int e2 = __shfl_sync(0xffffffffu, e, src);
      const int s2 = base + warp * 32 + src;
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      for (int q = b2 + lane; q < e2; q += 32) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], prod[r][q]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = warp_combine<MX>(acc[r]);
      if (lane == 0) {
        if (s2 == sb && hf >= 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) M.head_part[2 * t + r] = acc[r];
          __threadfence();
        } else {
          op.finish(s2, acc, red);
        }
      }
    }
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
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = warp_combine<MX>(acc[r]);
      if (lane == 0) bsum[warp][r] = acc[r];
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double v = bsum[0][r];
        for (int w = 1; w < kWarps; ++w) v = combine<MX>(v, bsum[w][r]);
        M.tail_part[2 * t + r] = v;
      }
      __threadfence();
    }
  }

  // ---- Phase 3: per-tile reduction partials (fixed trees).
  if constexpr (Op::kRed > 0) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Op::kRed; ++i) {
      const double v = warp_combine<false>(red[i]);
      if (lane == 0) bsum[warp][i] = v;
    }
    __syncthreads();
    if (tid < Op::kRed) {
      double v = bsum[0][tid];
      for (int w = 1; w < kWarps; ++w) v += bsum[w][tid];
      tile_red[static_cast<int64_t>(t) * Op::kRed + tid] = v;
      if (hf < 0) span_red[static_cast<int64_t>(t) * Op::kRed + tid] = 0.0;
    }
  }

  // ---- Phase 4: cross-tile segments, finished by the last arriving CTA.
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
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = warp_combine<MX>(acc[r]);
      if (lane == 0) bsum[warp][r] = acc[r];
    }
    __syncthreads();
    if (tid == 0) {
      double s[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double v = bsum[0][r];
        for (int ww = 1; ww < kWarps; ++ww) v = combine<MX>(v, bsum[ww][r]);
        s[r] = combine<MX>(v, __ldcg(M.head_part + 2 * o + r));
      }
      double red2[NR];
#pragma unroll
      for (int i = 0; i < NR; ++i) red2[i] = 0.0;
      op.finish(M.tile_seg[o], s, red2);
      if constexpr (Op::kRed > 0) {
        for (int i = 0; i < Op::kRed; ++i) span_red[static_cast<int64_t>(o) * Op::kRed + i] = red2[i];
      }
      M.counter[o] = 0u;
    }
    __syncthreads();
  }
}

template <class Op>
inline void launch_tiles(const CMat& M, const Op& op, double* tile_red, double* span_red, cudaStream_t st) {
  tile_kernel<Op><<<M.ntiles, kBlock, 0, st>>>(M, op, tile_red, span_red);
}

}  // namespace pdhg
