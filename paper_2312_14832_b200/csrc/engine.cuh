// Length-class dispatch of every matrix pass.
//
// At setup the rows of K (CSR) and the columns (CSC) are permuted into four
// contiguous length classes, keeping the storage order inside each segment
// (so every segment sum is formed exactly as before):
//   S  (<= kThreadMax = 64 nonzeros, session.cu): one thread per segment, sum
//      in storage order -- bit-identical to the reference's `acc += v * x[j]`
//      loops. Kernels: direct loads, uniform length with implicit offsets,
//      or warp-staged chunks (with segment-order warps for shifted copies);
//   M  (65 .. kWarpMax = 512): one warp per segment, lane-strided loads,
//      fixed butterfly;
//   L  (513 .. kCtaMax = 16384): one CTA per segment (or per 4 adjacent
//      segments, interleaved lanes, stream staged by TMA), fixed tree;
//   XL (> kCtaMax): the TMA tile engine (tile_spmv.cuh), several CTAs per
//      segment with last-arriver combination.
// Each class writes its own reduction slots; the slot reductions sum them in
// a fixed order, so every pass stays bitwise reproducible.
#pragma once

#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "tile_spmv.cuh"

namespace pdhg {

constexpr int kUnroll = 4;
constexpr int kSChunkMax = 256;  // class-S staged chunk (entries per warp step), longest variant

// Equality rows after the class permutation: within each class the equality
// rows come first. [0,e0) eq S, [s1,e1) eq M, [s2,e2) eq L, [s3,e3) eq XL.
struct RowKind {
  int32_t e0, s1, e1, s2, e2, s3, e3;
  __device__ __forceinline__ bool eq(int32_t s) const {
    return s < e0 || (s >= s1 && s < e1) || (s >= s2 && s < e2) || (s >= s3 && s < e3);
  }
};

// One matrix layout split into classes.
struct Layout {
  int32_t nseg = 0, nvec = 0;
  int64_t nnz = 0;
  int32_t* ptr = nullptr;
  int32_t* idx = nullptr;
  double* val = nullptr;
  int32_t s1 = 0, s2 = 0, s3 = 0;  // class bounds S | M | L | XL
  bool s_staged = false;           // class S uses seg_thread_staged_kernel
  bool s_pipe = false;             // ... its cp.async-pipelined variant (one-operand Ops)
  int s_flow = 0;                  // ... its persistent variant (step Ops; 3 or 4 CTAs per SM)
  int s_chunk = kSChunkMax;        // ... its chunk of entries per warp step (128 or 256)
  const uint8_t* s_rm = nullptr;   // per-32-segment flags: segment-order gathers (staged kernel)
  int l_rpc = 1;                   // class L segments per CTA (1 or 4)
  int l_stage = 0;                 // > 0: RPC-4 stream staged by TMA, dynamic smem bytes
  int s_len = 0;                   // common class-S length (1,2,3,4,8) or 0
  int32_t s_u = 0;                 // s_len > 0: segments [0, s_u) have it (s_u = s1, or a kBlock multiple)
  CMat lng;                        // tile-engine view of [s3, nseg)
  // Gather-window split of class S (Session::BuildSplit; step passes only):
  // class S runs as two passes over copies of its entries -- those gathering
  // below split_w, then those at or above it -- the second continuing the
  // first's sums (`part`), so each pass gathers from half the vector, which
  // then stays L2-resident. Storage order is kept: every segment's low
  // entries precede its high ones (checked at setup), so the sums are
  // bit-identical to the one-pass kernel.
  struct Half {
    int32_t* ptr = nullptr;
    int32_t* idx = nullptr;
    double* val = nullptr;
    const uint8_t* rm = nullptr;
    int chunk = kSChunkMax;
  };
  int32_t split_w = 0;  // 0: no split
  Half lo, hi;
  double* part = nullptr;  // s1 partial sums of the low pass
  int nb_s() const { return ceil_div(s1, kBlock); }
  int nb_m() const { return ceil_div(static_cast<int64_t>(s2 - s1) * 32, kBlock); }
  int nb_l() const { return ceil_div(s3 - s2, l_rpc); }
  int nt_x() const { return nseg > s3 ? lng.ntiles : 0; }
  int parts() const { return nb_s() + nb_m() + nb_l() + 2 * nt_x(); }  // reduction slots
};

constexpr int pow2_ceil(int k) { return k <= 1 ? 1 : 2 * pow2_ceil((k + 1) / 2); }

// Warp sums of K <= 32 per-lane values by recursive halving: at each step a
// lane trades the half of its remaining values that its partner keeps, so a
// warp issues ~P = pow2_ceil(K) shuffles instead of 5K (the check passes
// carry 11 and 15 sums per thread and were shuffle-bound). After the halving
// steps the lanes of one group (equal above bit 32/P) share a value index;
// plain xor steps finish the sums inside the group. Every lane ends with the
// total of value index *idx; a fixed, deterministic tree.
template <int K>
__device__ __forceinline__ double warp_reduce_scatter(const double (&v)[K], int* idx) {
  constexpr int P = pow2_ceil(K);
  static_assert(P <= 32, "at most 32 values per lane");
  const int lane = threadIdx.x & 31;
  double w[P];
#pragma unroll
  for (int j = 0; j < P; ++j) w[j] = j < K ? v[j] : 0.0;
  int base = 0;
#pragma unroll
  for (int c = P, o = 16; c > 1; c >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int j = 0; j < c / 2; ++j) {
      const double send = up ? w[j] : w[j + c / 2];
      const double keep = up ? w[j + c / 2] : w[j];
      w[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    base += up ? c / 2 : 0;
  }
  double r = w[0];
#pragma unroll
  for (int o = 16 / P; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  *idx = base;
  return r;
}

template <class Op, int NW = kWarps>
__device__ __forceinline__ void block_reduce_out(double (&red)[Op::kRed > 0 ? Op::kRed : 1], double* out,
                                                 int slot = -1) {
  if constexpr (Op::kRed > 0) {
    __shared__ double sh[NW][Op::kRed];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (Op::kRed == 1) {
      const double v = warp_combine<false>(red[0]);
      if (lane == 0) sh[warp][0] = v;
    } else {
      int i;
      const double v = warp_reduce_scatter<Op::kRed>(red, &i);
      constexpr int G = 32 / pow2_ceil(Op::kRed);  // lanes per value index
      if ((lane & (G - 1)) == 0 && i < Op::kRed) sh[warp][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < Op::kRed) {
      double v = sh[0][threadIdx.x];
      for (int w = 1; w < NW; ++w) v += sh[w][threadIdx.x];
      out[static_cast<int64_t>(slot < 0 ? static_cast<int>(blockIdx.x) : slot) * Op::kRed + threadIdx.x] = v;
    }
  }
}

// Class S: one thread per segment, sum in storage order -- bit-identical to
// the reference's serial `acc += v * x[j]` loops. Two variants, chosen per
// layout from the class's mean segment length (Layout::s_staged):
//
// direct (very short segments, e.g. transport / MCF / PageRank columns of 2,
// 3, 8): each thread loads its own few entries; consecutive threads read
// adjacent ranges, so each warp load touches a couple of lines.
template <class Op>
__global__ void __launch_bounds__(kBlock) seg_thread_kernel(const int32_t* __restrict__ ptr,
                                                            const int32_t* __restrict__ idx,
                                                            const double* __restrict__ val, int32_t s_end,
                                                            const Op op, double* __restrict__ red_out) {
  if (skip_launch(op)) return;
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const int s = blockIdx.x * kBlock + threadIdx.x;
  int b = 0, e = 0;
  typename Op::Pre pre{};
  if (s < s_end) {
    b = ptr[s];
    e = ptr[s + 1];
    pre = op.prefetch(s);
  }
  pdl_wait_trigger();
  if (s < s_end) {
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int k = b;
    for (; k + kUnroll <= e; k += kUnroll) {
      int32_t j[kUnroll];
      double v[kUnroll], p[kUnroll][R];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        j[u] = ld_stream(idx + k + u);
        v[u] = ld_stream(val + k + u);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) op.map(j[u], v[u], p[u]);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[u][r]);  // storage order
    }
    for (; k < e; ++k) {
      double p[R];
      op.map(ld_stream(idx + k), ld_stream(val + k), p);
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[r]);
    }
    op.finish(s, acc, pre, red);
  }
  block_reduce_out<Op>(red, red_out);
}

// uniform (every class-S segment has the same length L in {1,2,3,4,8}, e.g.
// the columns of transportation / MCF / PageRank LPs): segment s occupies
// [s*L, (s+1)*L) of the layout (class S starts at nonzero 0), so the offsets
// array is never read and the L entries come in with vector loads. Only Ops
// that declare kUniform (the per-iteration step kernels) are instantiated.
template <class T, class = void>
struct UniformOk : std::false_type {};
template <class T>
struct UniformOk<T, std::void_t<decltype(T::kUniform)>> : std::integral_constant<bool, T::kUniform> {};

template <int L>
__device__ __forceinline__ void load_uniform(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                             int64_t b, int32_t (&j)[L], double (&v)[L]) {
  if constexpr (L == 2) {
    const int2 jj = __ldcs(reinterpret_cast<const int2*>(idx + b));
    const double2 vv = __ldcs(reinterpret_cast<const double2*>(val + b));
    j[0] = jj.x, j[1] = jj.y, v[0] = vv.x, v[1] = vv.y;
  } else if constexpr (L == 4 || L == 8) {
#pragma unroll
    for (int q = 0; q < L / 4; ++q) {
      const int4 jj = __ldcs(reinterpret_cast<const int4*>(idx + b) + q);
      const double2 v0 = __ldcs(reinterpret_cast<const double2*>(val + b) + 2 * q);
      const double2 v1 = __ldcs(reinterpret_cast<const double2*>(val + b) + 2 * q + 1);
      j[4 * q] = jj.x, j[4 * q + 1] = jj.y, j[4 * q + 2] = jj.z, j[4 * q + 3] = jj.w;
      v[4 * q] = v0.x, v[4 * q + 1] = v0.y, v[4 * q + 2] = v1.x, v[4 * q + 3] = v1.y;
    }
  } else {
#pragma unroll
    for (int u = 0; u < L; ++u) {
      j[u] = ld_stream(idx + b + u);
      v[u] = ld_stream(val + b + u);
    }
  }
}

//
// Modal prefix (Layout::s_u < s_end): only the first s_u segments -- a
// multiple of kBlock, permuted to the front of class S at setup because they
// have the class's modal length -- are uniform; the CTAs past s_u run the
// direct per-thread loop of seg_thread_kernel over the offsets (PageRank:
// 9,999,993 columns of 8 nonzeros, 7 of 3).
template <class Op>
__device__ __forceinline__ void seg_thread_direct(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                                  const double* __restrict__ val, int32_t s_end, const Op& op,
                                                  double (&red)[Op::kRed > 0 ? Op::kRed : 1], int blk) {
  constexpr int R = Op::kRhs;
  constexpr bool MX = Op::kMax;
  const int s = blk * kBlock + threadIdx.x;
  int b = 0, e = 0;
  typename Op::Pre pre{};
  if (s < s_end) {
    b = ptr[s];
    e = ptr[s + 1];
    pre = op.prefetch(s);
  }
  pdl_wait_trigger();
  if (s < s_end) {
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int k = b; k < e; ++k) {
      double p[R];
      op.map(ld_stream(idx + k), ld_stream(val + k), p);
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[r]);  // storage order
    }
    op.finish(s, acc, pre, red);
  }
}

// One CTA's worth (block `blk`: segments [blk * kBlock, +kBlock)) of the
// uniform kernel; the kernel runs it for blockIdx.x, the persistent block
// kernel (persist.cuh) for the blocks it is dealt.
template <class Op, int L, bool kPrefix>
__device__ __forceinline__ void uniform_item(int blk, const int32_t* __restrict__ idx, const double* __restrict__ val,
                                             int32_t s_end, const Op& op, double* __restrict__ red_out,
                                             const int32_t* __restrict__ ptr, int32_t s_u) {
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  if constexpr (kPrefix) {
    if (blk * kBlock >= s_u) {  // CTA-uniform: past the modal prefix
      if (skip_launch(op)) return;
      seg_thread_direct(ptr, idx, val, s_end, op, red, blk);
      block_reduce_out<Op>(red, red_out, blk);
      return;
    }
  }
  const int s = blk * kBlock + threadIdx.x;
  typename Op::Pre pre{};
  int32_t j[L];
  double v[L];
  if (s < s_end) {
    load_uniform<L>(idx, val, static_cast<int64_t>(s) * L, j, v);
    pre = op.prefetch(s);
  }
  // The halt flag (pipelined loop) is tested once the loads are in flight,
  // not before: it is one more dependent round trip ahead of every load.
  if (skip_launch(op)) return;
  pdl_wait_trigger();
  if (s < s_end) {
    double p[L][R];
#pragma unroll
    for (int u = 0; u < L; ++u) op.map(j[u], v[u], p[u]);
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
    for (int u = 0; u < L; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[u][r]);  // storage order
    op.finish(s, acc, pre, red);
  }
  block_reduce_out<Op>(red, red_out, blk);
}

// kPrefix: the modal-prefix variant (the plain one carries no direct path,
// which would cost the all-uniform transport primal 8 registers and a
// quarter of its occupancy: 10.3 -> 12.3 us).
template <class Op, int L, bool kPrefix>
__global__ void __launch_bounds__(kBlock) seg_thread_uniform_kernel(const int32_t* __restrict__ idx,
                                                                    const double* __restrict__ val, int32_t s_end,
                                                                    const Op op, double* __restrict__ red_out,
                                                                    const int32_t* __restrict__ ptr, int32_t s_u) {
  uniform_item<Op, L, kPrefix>(static_cast<int>(blockIdx.x), idx, val, s_end, op, red_out, ptr, s_u);
}

// Ops whose map() splits into gather(index) and prod(value, gathered, out).
template <class T, class = void>
struct HasGather : std::false_type {};
template <class T>
struct HasGather<T, std::void_t<decltype(std::declval<T>().gather(0))>> : std::true_type {};

template <class T, class = void>
struct HasInit : std::false_type {};
template <class T>
struct HasInit<T, std::void_t<decltype(std::declval<T>().init(0))>> : std::true_type {};

// Ops of the gather-window split (Layout::split_w): the low pass runs the
// step Op's products and stores each segment's partial sum; the high pass is
// the step Op itself, its sums starting from that partial.
template <class Op>
struct OpSplitLo {
  static constexpr int kRhs = 1, kRed = 0;
  static constexpr bool kMax = Op::kMax;
  struct Pre {};
  Op op;
  double* part;
  __device__ bool skip() const { return skip_launch(op); }
  __device__ void map(int32_t j, double v, double (&p)[1]) const { op.map(j, v, p); }
  __device__ Pre prefetch(int32_t) const { return {}; }
  __device__ void finish(int32_t s, const double (&a)[1], const Pre&, double*) const { part[s] = a[0]; }
};
template <class Op>
struct OpSplitHi : Op {
  static constexpr bool kUniform = false;
  const double* part;
  OpSplitHi(const Op& o, const double* p) : Op(o), part(p) {}
  __device__ double init(int32_t s) const { return part[s]; }
};
template <class T, class = void>
struct SplitOk : std::false_type {};
template <class T>
struct SplitOk<T, std::void_t<decltype(T::kSplit)>> : std::integral_constant<bool, T::kSplit> {};

// staged (longer short segments, e.g. 20-nonzero staircase rows): the 32
// segments of a warp are contiguous in the nonzero stream, so the warp
// streams that range in chunks of C entries (C = 128 or 256 by the class's
// mean length, Layout::s_chunk) with fully coalesced lane-strided loads, all
// gathers of a chunk in flight before the first product is staged in shared
// memory, and every lane then adds up the part of its own segment inside the
// chunk, chunk after chunk -- i.e. in storage order, exactly like the direct
// variant. The warp's range [wb, we) comes from the lanes' own offsets
// (shuffles) and the segment-order flag is loaded with them, before the
// programmatic wait: the group's dependent memory chain is offsets ->
// stream -> gathers.
constexpr int kSChunk = 256;

//
// Segment-order warps (kRM, per-warp flags `rm`): when a warp's 32 segments
// are shifted copies of each other -- segment s + 1 gathers index + 1 where s
// gathers index (one MCF node's conservation rows across commodities) -- the
// warp stages the raw (idx, val) chunk instead of the products and each lane
// then walks its own segment, so the 32 lanes gather 32 adjacent entries per
// step instead of one lane-strided entry each of 32 unrelated segments. The
// sums run in the same storage order either way.
template <class Op, bool kRM, int C>
__device__ __forceinline__ void staged_group(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                             const Op& op, int b, int e, int wb, int we, bool seg_order,
                                             double (*sp)[C], int32_t* si, double (&acc)[Op::kRhs]) {
  constexpr int R = Op::kRhs;
  constexpr bool MX = Op::kMax;
  constexpr int U = C / 32;
  const int lane = threadIdx.x & 31;  // acc holds the starting values (0, or a split pass's partial)
  for (int c0 = wb; c0 < we; c0 += C) {
    int32_t j[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = c0 + lane + 32 * u;
      j[u] = k < we ? ld_stream(idx + k) : 0;
      v[u] = k < we ? ld_stream(val + k) : 0.0;
    }
    const int lo = (b > c0 ? b : c0) - c0;
    const int hi = (e < c0 + C ? e : c0 + C) - c0;
    if (kRM && seg_order) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        si[lane + 32 * u] = j[u];
        sp[0][lane + 32 * u] = v[u];
      }
      __syncwarp();
      constexpr int Q = 4;
      int q = lo;
      for (; q + Q <= hi; q += Q) {
        double p[Q][R];
#pragma unroll
        for (int t = 0; t < Q; ++t) op.map(si[q + t], sp[0][q + t], p[t]);
#pragma unroll
        for (int t = 0; t < Q; ++t)
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[t][r]);  // storage order
      }
      for (; q < hi; ++q) {
        double p[R];
        op.map(si[q], sp[0][q], p);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[r]);
      }
    } else {
      constexpr int B = U <= 4 ? U : 1;  // C = 128: all gathers in flight; 256: scheduled by ptxas (64 registers)
#pragma unroll
      for (int u0 = 0; u0 < U; u0 += B) {
        double p[B][R];
#pragma unroll
        for (int u = 0; u < B; ++u) {  // the batch's gathers all in flight ...
          if (c0 + lane + 32 * (u0 + u) < we) op.map(j[u0 + u], v[u0 + u], p[u]);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {  // ... before its first product is staged
          if (c0 + lane + 32 * (u0 + u) < we) {
#pragma unroll
            for (int r = 0; r < R; ++r) sp[r][lane + 32 * (u0 + u)] = p[u][r];
          }
        }
      }
      __syncwarp();
      for (int q = lo; q < hi; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], sp[r][q]);  // storage order
      }
    }
    __syncwarp();
  }
}

template <class Op, bool kRM, int C>
__global__ void __launch_bounds__(kBlock, 4) seg_thread_staged_kernel(const int32_t* __restrict__ ptr,
                                                                      const int32_t* __restrict__ idx,
                                                                      const double* __restrict__ val,
                                                                      int32_t s_end, const Op op,
                                                                      double* __restrict__ red_out,
                                                                      const uint8_t* __restrict__ rm) {
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  __shared__ double sprod[kWarps][R][C];
  __shared__ int32_t sidx[kRM ? kWarps : 1][kRM ? C : 1];
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = blockIdx.x * kBlock + threadIdx.x;
  const int s0 = blockIdx.x * kBlock + warp * 32;
  const bool own = s < s_end;
  int b = 0, e = 0;
  bool seg_order = false;
  typename Op::Pre pre{};
  double acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  if (own) {
    b = ptr[s];
    e = ptr[s + 1];
    pre = op.prefetch(s);
    if constexpr (HasInit<Op>::value) acc[0] = op.init(s);  // split high pass: the low pass's partial
  }
  if (kRM && s0 < s_end) seg_order = rm[s0 >> 5];  // warp-uniform
  if (skip_launch(op)) return;  // halt flag (pipelined loop), once the loads are in flight
  pdl_wait_trigger();
  if (s0 < s_end) {  // warp-uniform
    const int wb = __shfl_sync(0xffffffffu, b, 0);
    const int we = __shfl_sync(0xffffffffu, e, min(31, s_end - 1 - s0));
    staged_group<Op, kRM, C>(idx, val, op, b, e, wb, we, seg_order, sprod[warp], kRM ? sidx[warp] : nullptr, acc);
    if (own) op.finish(s, acc, pre, red);
  }
  block_reduce_out<Op>(red, red_out);
}

// persistent (Layout::s_flow; the per-iteration step Ops, no reductions):
// the staged kernel's groups, but every warp walks a grid-strided sequence
// of 32-segment groups and loads the NEXT group's offsets, segment-order flag
// and epilogue operands while it streams and gathers the current one, so the
// offsets' round trip overlaps the previous group's chain. Same sums, same
// order: bit-identical with seg_thread_staged_kernel.
template <class Op, bool kRM, int C, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) seg_thread_flow_kernel(const int32_t* __restrict__ ptr,
                                                                       const int32_t* __restrict__ idx,
                                                                       const double* __restrict__ val,
                                                                       int32_t s_end, const Op op,
                                                                       const uint8_t* __restrict__ rm) {
  static_assert(Op::kRed == 0, "no per-CTA reduction slots in the persistent kernel");
  if (skip_launch(op)) return;
  constexpr int R = Op::kRhs;
  __shared__ double sprod[kWarps][R][C];
  __shared__ int32_t sidx[kRM ? kWarps : 1][kRM ? C : 1];
  double red[1] = {0.0};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ngroups = (s_end + 31) >> 5;
  const int stride = gridDim.x * kWarps;
  using Pre = typename Op::Pre;
  auto fetch = [&](int g, int& b, int& e, bool& so, Pre& pre) {
    const int s = (g << 5) + lane;
    if (g < ngroups && s < s_end) {
      b = ptr[s];
      e = ptr[s + 1];
      pre = op.prefetch(s);
    }
    if (kRM && g < ngroups) so = rm[g];
  };
  int g = blockIdx.x * kWarps + warp;
  int b = 0, e = 0;
  bool so = false;
  Pre pre{};
  fetch(g, b, e, so, pre);
  pdl_wait_trigger();
  for (; g < ngroups; g += stride) {  // warp-uniform
    int bn = 0, en = 0;
    bool son = false;
    Pre pren{};
    fetch(g + stride, bn, en, son, pren);  // in flight while this group streams
    const int s0 = g << 5, s = s0 + lane;
    const int wb = __shfl_sync(0xffffffffu, b, 0);
    const int we = __shfl_sync(0xffffffffu, e, min(31, s_end - 1 - s0));
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    staged_group<Op, kRM, C>(idx, val, op, b, e, wb, we, so, sprod[warp], kRM ? sidx[warp] : nullptr, acc);
    if (s < s_end) op.finish(s, acc, pre, red);
    b = bn;
    e = en;
    so = son;
    pre = pren;
  }
}

// Grid of a persistent kernel: resident CTAs per SM x SMs (occupancy query,
// cached per kernel and device), at most one CTA per kWarps groups.
inline int flow_grid(const void* kernel, int groups) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  PDHG_CUDA(cudaGetDevice(&dev));
  int v = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find({kernel, dev});
    if (it != cache.end()) v = it->second;
  }
  if (!v) {
    int per = 0, sms = 0;
    PDHG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kBlock, 0));
    PDHG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    v = std::max(1, per) * sms;
    std::lock_guard<std::mutex> g(mu);
    cache[{kernel, dev}] = v;
  }
  return std::max(1, std::min(v, (groups + kWarps - 1) / kWarps));
}

// pipelined (opt-in PDHG_S_PIPE=1; measured SLOWER than the register-staged
// kernel -- PageRank-10M dual 733 -> 898 us, MCF 285 -> 342 us, staircase
// 1073 -> 1188 us, profiles/r02/s_pipe_ab_r02i.txt -- kept for the record
// and bit-identity tested): the same
// warp-cooperative chunks and storage-order sums as the staged kernel, but
// the raw (idx, val) chunk is copied global -> shared by per-lane async
// copies (cp.async, LDGSTS) one chunk AHEAD, double-buffered per warp: while
// the lanes gather x for chunk c and sum it, chunk c + 1's stream is in
// flight, so a chunk costs one gather latency instead of a stream load
// followed by a gather. Products overwrite the staged values in place; chunk
// 0 is issued before the programmatic wait (the matrix does not depend on
// the predecessor). The profiled staged kernel was latency-bound (0.4
// eligible warps per cycle, DRAM 49 %, L2 36 % on the PageRank-10M dual).
// Shared memory: 2 x kSChunk x 12 bytes per warp (48 KB per CTA, 4 CTAs/SM).
constexpr int kPipeSmem = kWarps * 2 * kSChunk * 12;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <class Op, bool kRM = false>
__global__ void __launch_bounds__(kBlock, 4) seg_thread_pipe_kernel(const int32_t* __restrict__ ptr,
                                                                    const int32_t* __restrict__ idx,
                                                                    const double* __restrict__ val,
                                                                    int32_t s_end, const Op op,
                                                                    double* __restrict__ red_out,
                                                                    const uint8_t* __restrict__ rm = nullptr) {
  static_assert(Op::kRhs == 1, "products are staged in place of the values");
  if (skip_launch(op)) return;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  constexpr int C = kSChunk;
  constexpr int U = C / 32;
  extern __shared__ __align__(16) unsigned char pipe_smem[];
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sv = reinterpret_cast<double*>(pipe_smem) + warp * 2 * C;                   // [2][C] values
  int32_t* si = reinterpret_cast<int32_t*>(pipe_smem + kWarps * 2 * C * 8) + warp * 2 * C;  // [2][C] indices
  const int s = blockIdx.x * kBlock + threadIdx.x;
  const int s0 = blockIdx.x * kBlock + warp * 32;
  const bool own = s < s_end;
  const bool active = s0 < s_end;  // warp-uniform
  int b = 0, e = 0, wb = 0, we = 0;
  typename Op::Pre pre{};
  if (own) {
    b = ptr[s];
    e = ptr[s + 1];
    pre = op.prefetch(s);
  }
  auto issue = [&](int c0, int buf) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = lane + 32 * u;
      if (c0 + q < we) {
        cp_async4(si + buf * C + q, idx + c0 + q);
        cp_async8(sv + buf * C + q, val + c0 + q);
      }
    }
  };
  if (active) {
    wb = ptr[s0];
    we = ptr[s0 + 32 < s_end ? s0 + 32 : s_end];
    issue(wb, 0);
  }
  cp_async_commit();
  pdl_wait_trigger();
  if (active) {
    double acc = 0.0;
    const bool seg_order = kRM && rm[s0 >> 5];  // warp-uniform
    int buf = 0;
    for (int c0 = wb; c0 < we; c0 += C, buf ^= 1) {
      if (c0 + C < we) issue(c0 + C, buf ^ 1);
      cp_async_commit();
      cp_async_wait1();  // this lane's copies of chunk c0 have landed
      __syncwarp();      // ... and every other lane's
      const int32_t* ci = si + buf * C;
      double* cv = sv + buf * C;
      const int lo = (b > c0 ? b : c0) - c0;
      const int hi = (e < c0 + C ? e : c0 + C) - c0;
      if (kRM && seg_order) {
        int q = lo;
        for (; q + 4 <= hi; q += 4) {
          double p[4][1];
#pragma unroll
          for (int t = 0; t < 4; ++t) op.map(ci[q + t], cv[q + t], p[t]);
#pragma unroll
          for (int t = 0; t < 4; ++t) acc = combine<MX>(acc, p[t][0]);  // storage order
        }
        for (; q < hi; ++q) {
          double p[1];
          op.map(ci[q], cv[q], p);
          acc = combine<MX>(acc, p[0]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = lane + 32 * u;
          if (c0 + q < we) {
            double p[1];
            op.map(ci[q], cv[q], p);
            cv[q] = p[0];
          }
        }
        __syncwarp();
        for (int q = lo; q < hi; ++q) acc = combine<MX>(acc, cv[q]);  // storage order
      }
      __syncwarp();  // buffer `buf` is refilled two chunks on
    }
    if (own) {
      const double a[1] = {acc};
      op.finish(s, a, pre, red);
    }
  }
  block_reduce_out<Op>(red, red_out);
}

// Lane-strided partial sum of [b, e): batches of kStrideUnroll predicated
// loads per lane, so even the last partial batch keeps every load of the
// lane in flight at once (a sequential tail loop would serialise one
// idx -> gather latency chain per element). Masked-off slots contribute 0,
// the identity of both combines (sums, and max over |v| >= 0).
constexpr int kStrideUnroll = 8;
// kPdl: issue the first batch of stream loads, then wait for the predecessor
// grid (pdl_wait_trigger) before the first gather -- exactly once per thread.
template <class Op, int kStride, bool kPdl = false>
__device__ __forceinline__ void strided_sum(const Op& op, const int32_t* __restrict__ idx,
                                            const double* __restrict__ val, int b, int e, int t,
                                            double (&acc)[Op::kRhs]) {
  constexpr int R = Op::kRhs;
  constexpr bool MX = Op::kMax;
  constexpr int U = kStrideUnroll;
  bool waited = !kPdl;
  for (int k = b + t; k < e; k += kStride * U) {
    int32_t j[U];
    double v[U], p[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = k + kStride * u < e;
      j[u] = in ? ld_stream(idx + k + kStride * u) : 0;
      v[u] = in ? ld_stream(val + k + kStride * u) : 0.0;
    }
    if (!waited) {
      pdl_wait_trigger();
      waited = true;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k + kStride * u < e) {
        op.map(j[u], v[u], p[u]);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) p[u][r] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[u][r]);
  }
  if (!waited) pdl_wait_trigger();
}

// Class M: one warp per segment.
template <class Op>
__global__ void __launch_bounds__(kBlock) seg_warp_kernel(const int32_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ idx,
                                                          const double* __restrict__ val, int32_t s_begin,
                                                          int32_t s_end, const Op op, double* __restrict__ red_out) {
  if (skip_launch(op)) return;
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const int lane = threadIdx.x & 31;
  const int s = s_begin + blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (s >= s_end) pdl_wait_trigger();
  if (s < s_end) {  // warp-uniform
    const int b = ptr[s], e = ptr[s + 1];
    typename Op::Pre pre{};
    if (lane == 0) pre = op.prefetch(s);
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    strided_sum<Op, 32, true>(op, idx, val, b, e, lane, acc);
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = warp_combine<MX>(acc[r]);
    if (lane == 0) op.finish(s, acc, pre, red);
  }
  block_reduce_out<Op>(red, red_out);
}

// Class L: a CTA per RPC segments, kBlock / RPC threads per segment (fixed
// trees). RPC = 4 for moderately long segments whose neighbours gather
// neighbouring vector entries (transportation demand rows j..j+3 read
// x[i*T + j..j+3]): the lanes of a warp are interleaved across the 4
// segments (lane -> segment lane % 4, entry position warp * 8 + lane / 4), so
// one warp-wide gather reads 8 sectors of 4 adjacent entries instead of 32
// scattered sectors, and the stream loads stay 8-entry contiguous runs.
template <class Op, int RPC, int B = kBlock, int MINB = 1>
__global__ void __launch_bounds__(B, MINB) seg_cta_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                                    const double* __restrict__ val, int32_t s_begin, int32_t s_end,
                                                    const Op op, double* __restrict__ red_out) {
  if (skip_launch(op)) return;
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  constexpr bool IL = RPC > 1;  // interleaved lanes
  constexpr int T = B / RPC;    // threads per segment
  constexpr int W = T / 32;     // warps per segment (non-interleaved)
  constexpr int NW = B / 32;
  __shared__ double sh[NW][RPC][R];
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = IL ? lane % RPC : threadIdx.x / T;
  const int t = IL ? warp * (32 / RPC) + lane / RPC : threadIdx.x % T;
  const int s = s_begin + blockIdx.x * RPC + sub;
  const bool own = s < s_end;
  typename Op::Pre pre{};
  double acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  if (own) {
    if (t == 0) pre = op.prefetch(s);
    strided_sum<Op, T, true>(op, idx, val, ptr[s], ptr[s + 1], t, acc);
  } else {
    pdl_wait_trigger();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double v = acc[r];
    if constexpr (IL) {
#pragma unroll
      for (int o = 16; o >= RPC; o >>= 1) v = combine<MX>(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane < RPC) sh[warp][lane][r] = v;
    } else {
      v = warp_combine<MX>(v);
      if (lane == 0) sh[warp][0][r] = v;
    }
  }
  __syncthreads();
  if (own && t == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double v;
      if constexpr (IL) {
        v = sh[0][sub][r];
        for (int w = 1; w < NW; ++w) v = combine<MX>(v, sh[w][sub][r]);
      } else {
        v = sh[sub * W][0][r];
        for (int w = 1; w < W; ++w) v = combine<MX>(v, sh[sub * W + w][0][r]);
      }
      acc[r] = v;
    }
    op.finish(s, acc, pre, red);
  }
  block_reduce_out<Op, NW>(red, red_out);
}

template <class Op>
inline void launch_thread_class(const Layout& L, const Op& op, double* red, cudaStream_t st, bool pdl = false) {
  const int g = L.nb_s();
  if constexpr (UniformOk<Op>::value) {
    const int32_t* p = L.ptr;
    const bool pre = L.s_u < L.s1;
#define PDHG_UNIFORM(LEN)                                                                                   \
  case LEN:                                                                                                 \
    if (pre)                                                                                                \
      return launch_k(seg_thread_uniform_kernel<Op, LEN, true>, g, kBlock, 0, st, pdl, L.idx, L.val, L.s1, op, red, p, \
                      L.s_u);                                                                               \
    return launch_k(seg_thread_uniform_kernel<Op, LEN, false>, g, kBlock, 0, st, pdl, L.idx, L.val, L.s1, op, red, p,  \
                    L.s_u);
    switch (L.s_len) {
      PDHG_UNIFORM(1)
      PDHG_UNIFORM(2)
      PDHG_UNIFORM(3)
      PDHG_UNIFORM(4)
      PDHG_UNIFORM(8)
#undef PDHG_UNIFORM
      default: break;
    }
  }
  if constexpr (Op::kRhs == 1) {
    if (L.s_staged && L.s_pipe) {
      if (L.s_rm) {
        smem_opt_in<seg_thread_pipe_kernel<Op, true>>(kPipeSmem);
        launch_k(seg_thread_pipe_kernel<Op, true>, g, kBlock, kPipeSmem, st, pdl, L.ptr, L.idx, L.val, L.s1, op, red,
                 static_cast<const uint8_t*>(L.s_rm));
      } else {
        smem_opt_in<seg_thread_pipe_kernel<Op, false>>(kPipeSmem);
        launch_k(seg_thread_pipe_kernel<Op, false>, g, kBlock, kPipeSmem, st, pdl, L.ptr, L.idx, L.val, L.s1, op, red,
                 static_cast<const uint8_t*>(nullptr));
      }
      return;
    }
  }
  if (!L.s_staged) {
    launch_k(seg_thread_kernel<Op>, g, kBlock, 0, st, pdl, L.ptr, L.idx, L.val, L.s1, op, red);
    return;
  }
  const uint8_t* rm = L.s_rm;
  if constexpr (Op::kRed == 0) {
    if (L.s_flow) {
      const int groups = ceil_div(L.s1, 32);
      auto go = [&](auto k) {
        launch_k(k, flow_grid(reinterpret_cast<const void*>(k), groups), kBlock, 0, st, pdl, L.ptr, L.idx, L.val, L.s1,
                 op, rm);
      };
#define PDHG_FLOW(C, MINB)                                 \
  if (L.s_chunk == C && L.s_flow == MINB) {                \
    if (rm) go(seg_thread_flow_kernel<Op, true, C, MINB>); \
    else go(seg_thread_flow_kernel<Op, false, C, MINB>);   \
    return;                                                \
  }
      PDHG_FLOW(128, 3)
      PDHG_FLOW(128, 4)
      PDHG_FLOW(256, 3)
      PDHG_FLOW(256, 4)
#undef PDHG_FLOW
    }
  }
  auto go = [&](auto k) { launch_k(k, g, kBlock, 0, st, pdl, L.ptr, L.idx, L.val, L.s1, op, red, rm); };
  if (L.s_chunk == 128) {
    if (rm) go(seg_thread_staged_kernel<Op, true, 128>);
    else go(seg_thread_staged_kernel<Op, false, 128>);
  } else {
    if (rm) go(seg_thread_staged_kernel<Op, true, 256>);
    else go(seg_thread_staged_kernel<Op, false, 256>);
  }
}

// Residency: kBlock-thread CTAs capped at 64 registers (4 CTAs = 1024
// threads per SM). The 4-segments-per-CTA kernel runs one CTA per four rows
// of a short class-L (transportation: 500 CTAs); without the cap the compiler
// takes 66 registers, 3 CTAs fit per SM and the pass needs a second wave
// (transport dual 12.3 us vs 10.3 us).
constexpr int kCtaMinBlocks = 4;

// Dynamic shared memory cap of the TMA-staged variant: 4 CTAs per SM.
constexpr int kCtaStageMax = 50 * 1024;

// Class L, 4 segments per CTA (interleaved lanes as above), with the CTA's
// whole contiguous (idx, val) range -- the 4 segments are adjacent in the
// stream -- bulk-copied into shared memory by TMA BEFORE the programmatic
// wait: the stream then arrives while the predecessor kernel drains, and
// after the wait only the gathers, the sums and the epilogue remain. Same
// per-thread order (k = b + t, b + t + T, ...) and the same trees as
// seg_cta_kernel<Op, 4>, hence bit-identical results. Used when every
// 4-segment group fits kCtaStageMax (Layout::l_stage).
// One 4-segment group (block `blk`) of the staged kernel, with its shared
// memory passed in: the kernel runs it for blockIdx.x; the persistent block
// kernel (persist.cuh) for each group it is dealt, reusing the stage buffer
// and barrier (`reuse`: wait until every thread is done with the previous
// group's stage before the bulk copy overwrites it).
// Thread 0 of the group's CTA: initialise the barrier and start the bulk
// copies of group `blk`'s contiguous (val, idx) range into `stage`.
__device__ __forceinline__ void cta4_issue(int blk, const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                           const double* __restrict__ val, int32_t s_begin, int32_t s_end,
                                           unsigned char* stage, uint64_t* bar) {
  const int g0 = s_begin + blk * 4;
  const int g1 = min(g0 + 4, s_end);
  const int32_t lo = ptr[g0], hi = ptr[g1];
  uint32_t bv = 0, bi = 0;
  const int64_t av = widen16<double>(lo, hi, &bv);
  const int64_t ai = widen16<int32_t>(lo, hi, &bi);
  mbar_init(bar, 1);
  mbar_expect_tx(bar, hi > lo ? bv + bi : 0);
  if (hi > lo) {
    bulk_g2s(stage, val + av, bv, bar);
    bulk_g2s(stage + bv, idx + ai, bi, bar);
  }
}

// kIssued: the caller already ran cta4_issue for this group (the persistent
// block kernel starts a CTA's first group before the grid barrier: the
// matrix does not depend on the step it waits for).
template <class Op, bool kReuse = false, bool kIssued = false>
__device__ __forceinline__ void cta4_item(int blk, const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                          const double* __restrict__ val, int32_t s_begin, int32_t s_end, const Op& op,
                                          double* __restrict__ red_out, unsigned char* stage, uint64_t* bar,
                                          double (*sh)[4][Op::kRhs]) {
  const bool halted = skip_launch(op);  // tested after the offsets are loaded
  constexpr int RPC = 4;
  constexpr int R = Op::kRhs;
  constexpr int NR = Op::kRed > 0 ? Op::kRed : 1;
  constexpr bool MX = Op::kMax;
  constexpr int T = kBlock / RPC;
  constexpr int NW = kBlock / 32;
  constexpr int U = kStrideUnroll;
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane % RPC, t = warp * (32 / RPC) + lane / RPC;
  const int g0 = s_begin + blk * RPC;
  const int g1 = min(g0 + RPC, s_end);
  const int32_t lo = ptr[g0], hi = ptr[g1];
  if (halted) {  // before any bulk copy is issued: none may outlive the CTA
    if constexpr (kIssued) mbar_wait(bar, 0);
    return;
  }
  uint32_t bv = 0, bi = 0;
  const int64_t av = widen16<double>(lo, hi, &bv);
  const int64_t ai = widen16<int32_t>(lo, hi, &bi);
  double* sval = reinterpret_cast<double*>(stage);
  int32_t* sidx = reinterpret_cast<int32_t*>(stage + bv);
  if constexpr (kReuse && !kIssued) {
    __syncthreads();  // the previous group's readers are done with the stage
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (!kIssued && threadIdx.x == 0) cta4_issue(blk, ptr, idx, val, s_begin, s_end, stage, bar);
  const int s = g0 + sub;
  const bool own = s < s_end;
  typename Op::Pre pre{};
  int b = 0, e = 0;
  if (own) {
    b = ptr[s];
    e = ptr[s + 1];
    if (t == 0) pre = op.prefetch(s);
  }
  __syncthreads();  // barrier initialised
  pdl_wait_trigger();
  mbar_wait(bar, 0);
  double acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  if constexpr (HasGather<Op>::value) {
    // Gathers first (Op::gather / Op::prod): all of a thread's entries up to
    // 2U in flight at once -- one gather latency per group for rows of up to
    // 2U * T entries (transport's 1000) instead of one per U-batch -- then the
    // products in the same order. The zeros of masked slots are added exactly
    // where the U-batched loop adds them (up to the thread's entry count
    // rounded up to U), so the sums stay bitwise those of seg_cta_kernel.
    constexpr int G = 2 * U;
    const int n = e > b + t ? (e - (b + t) + T - 1) / T : 0;
    const int nz = (n + U - 1) / U * U;  // slots the U-batched loop combines
    int base = 0;
    for (int k = b + t; k < e; k += T * G) {
      double g[G];
#pragma unroll
      for (int u = 0; u < G; ++u) g[u] = (k + T * u < e) ? op.gather(sidx[k + T * u - ai]) : 0.0;
#pragma unroll
      for (int u = 0; u < G; ++u) {
        if (k + T * u < e) {
          double p[R];
          op.prod(sval[k + T * u - av], g[u], p);
          acc[0] = combine<MX>(acc[0], p[0]);
        } else if (base + u < nz) {
          acc[0] = combine<MX>(acc[0], 0.0);
        }
      }
      base += G;
    }
  } else {  // (braced: with `else for` + `#pragma unroll`, nvcc 12.9 dropped all code after the loop)
  for (int k = b + t; k < e; k += T * U) {
    int32_t j[U];
    double v[U], p[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = k + T * u < e;
      j[u] = in ? sidx[k + T * u - ai] : 0;
      v[u] = in ? sval[k + T * u - av] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k + T * u < e) {
        op.map(j[u], v[u], p[u]);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) p[u][r] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = combine<MX>(acc[r], p[u][r]);
  }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double v = acc[r];
#pragma unroll
    for (int o = 16; o >= RPC; o >>= 1) v = combine<MX>(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane < RPC) sh[warp][lane][r] = v;
  }
  __syncthreads();
  if (own && t == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double v = sh[0][sub][r];
      for (int w = 1; w < NW; ++w) v = combine<MX>(v, sh[w][sub][r]);
      acc[r] = v;
    }
    op.finish(s, acc, pre, red);
  }
  block_reduce_out<Op, NW>(red, red_out, blk);
}

template <class Op>
__global__ void __launch_bounds__(kBlock, kCtaMinBlocks)
    seg_cta4_staged_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                           const double* __restrict__ val, int32_t s_begin, int32_t s_end, const Op op,
                           double* __restrict__ red_out) {
  extern __shared__ __align__(16) unsigned char stage[];
  __shared__ uint64_t bar;
  __shared__ double sh[kBlock / 32][4][Op::kRhs];
  cta4_item<Op>(static_cast<int>(blockIdx.x), ptr, idx, val, s_begin, s_end, op, red_out, stage, &bar, sh);
}

// Class S of a pass, as one kernel or -- gather-window split, step Ops --
// as the low and high passes (Layout::split_w).
template <class Op>
inline void launch_class_s(const Layout& L, const Op& op, double* red, cudaStream_t st, bool pdl) {
  if constexpr (SplitOk<Op>::value) {
    if (L.split_w) {
      Layout h = L;
      h.s_len = 0;
      h.s_u = 0;
      h.s_flow = 0;
      h.s_pipe = false;
      h.s_staged = true;
      h.ptr = L.lo.ptr;
      h.idx = L.lo.idx;
      h.val = L.lo.val;
      h.s_rm = L.lo.rm;
      h.s_chunk = L.lo.chunk;
      launch_thread_class(h, OpSplitLo<Op>{op, L.part}, nullptr, st, pdl);
      h.ptr = L.hi.ptr;
      h.idx = L.hi.idx;
      h.val = L.hi.val;
      h.s_rm = L.hi.rm;
      h.s_chunk = L.hi.chunk;
      launch_thread_class(h, OpSplitHi<Op>(op, L.part), red, st, false);
      return;
    }
  }
  launch_thread_class(L, op, red, st, pdl);
}

template <class Op>
inline void launch_cta_class(const Layout& L, const Op& op, double* red, cudaStream_t st, bool pdl = false) {
  if (L.l_rpc == 4 && L.l_stage > 0) {
    smem_opt_in<seg_cta4_staged_kernel<Op>>(kCtaStageMax);  // > 48 KB, once per device
    launch_k(seg_cta4_staged_kernel<Op>, L.nb_l(), kBlock, static_cast<size_t>(L.l_stage), st, pdl, L.ptr, L.idx,
             L.val, L.s2, L.s3, op, red);
  } else if (L.l_rpc == 4) {
    launch_k(seg_cta_kernel<Op, 4, kBlock, kCtaMinBlocks>, L.nb_l(), kBlock, 0, st, pdl, L.ptr, L.idx, L.val, L.s2,
             L.s3, op, red);
  } else {
    launch_k(seg_cta_kernel<Op, 1, kBlock, kCtaMinBlocks>, L.nb_l(), kBlock, 0, st, pdl, L.ptr, L.idx, L.val, L.s2,
             L.s3, op, red);
  }
}

// Reduction slots of one pass: [S blocks | M blocks | L CTAs | XL tiles | XL spans].
struct RedSlots {
  double* base = nullptr;
  double* at(int64_t slot, int nr) const { return base ? base + slot * nr : nullptr; }
};

// Programmatic dependent launch for a pass that is one kernel of an opted-in
// Op (the per-iteration steps): its prologue overlaps the previous step's
// drain. PDHG_PDL=0 disables it.
inline bool& pdl_suspended() {  // per-kernel timing: launches must not overlap each other
  static thread_local bool v = false;
  return v;
}
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PDHG_PDL");
    return !(e && e[0] == '0');
  }();
  return on && !pdl_suspended();
}

template <class Op>
inline void run_pass(const Layout& L, const Op& op, const RedSlots& red, cudaStream_t st) {
  constexpr int nr = Op::kRed > 0 ? Op::kRed : 1;
  const int nclass = (L.s1 > 0) + (L.s2 > L.s1) + (L.s3 > L.s2) + (L.nseg > L.s3);
  const bool pdl = PdlOk<Op>::value && nclass == 1 && pdl_enabled();
  int64_t slot = 0;
  if (L.s1 > 0) launch_class_s(L, op, red.at(slot, nr), st, pdl);
  slot += L.nb_s();
  if (L.s2 > L.s1)
    launch_k(seg_warp_kernel<Op>, L.nb_m(), kBlock, 0, st, pdl, L.ptr, L.idx, L.val, L.s1, L.s2, op,
             red.at(slot, nr));
  slot += L.nb_m();
  if (L.s3 > L.s2) launch_cta_class(L, op, red.at(slot, nr), st, pdl);
  slot += L.nb_l();
  if (L.nseg > L.s3) launch_tiles(L.lng, op, red.at(slot, nr), red.at(slot + L.nt_x(), nr), st, pdl);
}

// A main stream plus side streams: the class kernels of one pass are
// independent (disjoint segments, disjoint reduction slots), so with more
// than one class present they run as parallel branches (fork/join events;
// inside a captured graph these become parallel graph nodes) instead of
// serialising their tails.
struct Fork {
  cudaStream_t main = nullptr;
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[3] = {nullptr, nullptr, nullptr};
};

template <class Op>
inline void run_pass(const Layout& L, const Op& op, const RedSlots& red, const Fork& f) {
  constexpr int nr = Op::kRed > 0 ? Op::kRed : 1;
  const bool has[4] = {L.s1 > 0, L.s2 > L.s1, L.s3 > L.s2, L.nseg > L.s3};
  const int nclass = has[0] + has[1] + has[2] + has[3];
  if (nclass <= 1 || !f.side[0]) {
    run_pass(L, op, red, f.main);
    return;
  }
  cudaEventRecord(f.fork, f.main);
  cudaStream_t on[4];
  int k = 0;
  for (int c = 0; c < 4; ++c) {
    if (!has[c]) continue;
    on[c] = k == 0 ? f.main : f.side[k - 1];
    if (k > 0) cudaStreamWaitEvent(on[c], f.fork, 0);
    ++k;
  }
  int64_t slot = 0;
  if (has[0]) launch_class_s(L, op, red.at(slot, nr), on[0], false);
  slot += L.nb_s();
  if (has[1])
    seg_warp_kernel<Op><<<L.nb_m(), kBlock, 0, on[1]>>>(L.ptr, L.idx, L.val, L.s1, L.s2, op, red.at(slot, nr));
  slot += L.nb_m();
  if (has[2]) launch_cta_class(L, op, red.at(slot, nr), on[2]);
  slot += L.nb_l();
  if (has[3]) launch_tiles(L.lng, op, red.at(slot, nr), red.at(slot + L.nt_x(), nr), on[3]);
  k = 0;
  for (int c = 0; c < 4; ++c) {
    if (!has[c]) continue;
    if (k > 0) {
      cudaEventRecord(f.join[k - 1], on[c]);
      cudaStreamWaitEvent(f.main, f.join[k - 1], 0);
    }
    ++k;
  }
}

// Number of kernels run_pass launches.
inline int pass_launches(const Layout& L) {
  return (L.s1 > 0) * (L.split_w ? 2 : 1) + (L.s2 > L.s1) + (L.s3 > L.s2) + (L.nseg > L.s3);
}

}  // namespace pdhg
