// Setup-time device kernels: upload narrowing, VStack, CSC build support,
// length-class permutation, scaling helpers, tile partitioning, reductions.
#pragma once

#include "common.cuh"
#include "tile_spmv.cuh"

namespace pdhg {


// ------------------------------------------------------------------ upload
__global__ void k_narrow(const int64_t* in, int32_t* out, int64_t count, int64_t limit, int* bad) {
  GRID_STRIDE(i, count) {
    const int64_t v = in[i];
    if (v < 0 || v >= limit) atomicOr(bad, 1);
    out[i] = static_cast<int32_t>(v);
  }
}

// K row_ptr = [A.row_ptr ; nnz(A) + G.row_ptr[1:]] (VStack, sparse_matrix.cpp:98-103).
__global__ void k_stack_ptr(const int64_t* ap, const int64_t* gp, int64_t m1, int64_t m2, int64_t nnz_a,
                            int32_t* out) {
  GRID_STRIDE(i, m1 + m2 + 1) { out[i] = static_cast<int32_t>(i <= m1 ? ap[i] : nnz_a + gp[i - m1]); }
}

__global__ void k_check_ptr(const int32_t* p, int64_t rows, int64_t nnz, int* bad) {
  GRID_STRIDE(i, rows) {
    if (p[i] > p[i + 1]) atomicOr(bad, 2);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (p[0] != 0 || p[rows] != nnz)) atomicOr(bad, 2);
}

// Segment id of every nonzero: count segment starts, then inclusive scan.
__global__ void k_seg_marks(const int32_t* p, int64_t nseg, int64_t nnz, int32_t* cnt) {
  GRID_STRIDE(r, nseg) {
    if (r >= 1 && p[r] < nnz) atomicAdd(cnt + p[r], 1);
  }
}

__global__ void k_iota(int32_t* v, int64_t n) {
  GRID_STRIDE(i, n) v[i] = static_cast<int32_t>(i);
}

// col_ptr[j] = first CSC slot with column >= j (sorted column keys).
__global__ void k_colptr(const int32_t* keys, int64_t nnz, int64_t n, int32_t* cp) {
  GRID_STRIDE(j, n + 1) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    cp[j] = static_cast<int32_t>(lo);
  }
}

__global__ void k_csc_gather(const int32_t* perm, const int32_t* row_of, const double* v, int32_t* ri, double* cv,
                             int64_t nnz) {
  GRID_STRIDE(q, nnz) {
    const int32_t k = perm[q];
    ri[q] = row_of[k];
    cv[q] = v[k];
  }
}

// ------------------------------------------------------- class permutation
// Block of original segment s (blocks contiguous in original order, P <= 64).
__device__ __forceinline__ int block_of(const int64_t* begin, int P, int64_t s) {
  int b = 0;
  while (b + 1 < P && begin[b + 1] <= s) ++b;
  return b;
}

// key = block * 8 + class(len) * 2 + (row is an inequality row); columns use
// eq_end = n. A stable sort by key puts every block's segments contiguously
// (in block order) and, inside a block, class by class with equality rows
// first, each run keeping the original order.
// modal > 0 (columns only, eq_end = nseg): inside class S the low bit
// separates the segments of the modal length (first) from the rest, so the
// uniform kernel takes a prefix of the class (Layout::s_u).
__global__ void k_class_keys(const int32_t* p, int64_t nseg, int64_t eq_end, const int64_t* begin, int P,
                             int thread_max, int warp_max, int cta_max, int32_t* key, int modal = 0) {
  GRID_STRIDE(s, nseg) {
    const int len = p[s + 1] - p[s];
    const int cls = len <= thread_max ? 0 : (len <= warp_max ? 1 : (len <= cta_max ? 2 : 3));
    const int lo = (modal > 0 && cls == 0) ? (len != modal) : (s >= eq_end ? 1 : 0);
    key[s] = block_of(begin, P, s) * 8 + cls * 2 + lo;
  }
}

// Number of segments of at most `le` nonzeros.
__global__ void k_count_le(const int32_t* p, int64_t nseg, int le, int* out) {
  int c = 0;
  GRID_STRIDE(s, nseg) c += (p[s + 1] - p[s]) <= le;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Histogram of segment lengths 0..8 (for the modal uniform prefix).
__global__ void k_len_hist9(const int32_t* p, int64_t nseg, int* hist) {
  __shared__ int h[9];
  if (threadIdx.x < 9) h[threadIdx.x] = 0;
  __syncthreads();
  GRID_STRIDE(s, nseg) {
    const int len = p[s + 1] - p[s];
    if (len <= 8) atomicAdd(&h[len], 1);
  }
  __syncthreads();
  if (threadIdx.x < 9 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// Padded index of original segment s: block b's segments occupy
// [b * slice, b * slice + size_b) in class order (inv = compact position).
__global__ void k_pad_index(const int32_t* inv, const int64_t* begin, int P, int64_t slice, int32_t* pad, int64_t n) {
  GRID_STRIDE(s, n) {
    const int b = block_of(begin, P, s);
    pad[s] = static_cast<int32_t>(b * slice + (inv[s] - begin[b]));
  }
}

// out[pad[i]] = in[i] (original -> padded order).
__global__ void k_scatter(const double* in, const int32_t* pad, double* out, int64_t n) {
  GRID_STRIDE(i, n) out[pad[i]] = in[i];
}

// Shard-local row_ptr: out[s] = ptr[s] - ptr[0] for s <= nseg.
__global__ void k_rebase(const int32_t* ptr, int64_t nseg, int32_t* out) {
  const int32_t base = ptr[0];
  GRID_STRIDE(s, nseg + 1) out[s] = ptr[s] - base;
}

// Sum of `count` reduction packs (fixed shard order) into pack 0.
__global__ void k_sum_packs(double* packs, int count, int stride, int n, const Scalars* guard) {
  if (guard && guard->halt) return;
  const int i = threadIdx.x;
  if (i >= n) return;
  double v = packs[i];
  for (int k = 1; k < count; ++k) v += packs[static_cast<int64_t>(k) * stride + i];
  packs[i] = v;
}

// Min / max segment length over [0, nseg) (out[0] = min, out[1] = max;
// initialise to INT32_MAX / 0).
__global__ void k_len_minmax(const int32_t* p, int64_t nseg, int* out) {
  int mn = INT32_MAX, mx = 0;
  GRID_STRIDE(s, nseg) {
    const int len = p[s + 1] - p[s];
    mn = len < mn ? len : mn;
    mx = len > mx ? len : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {  // one atomic pair per warp
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

// Neighbouring segments whose middle entries gather from the same 32-byte
// sector (|index difference| <= 3): the transportation pattern (demand rows
// j, j+1 read x[i*T + j], x[i*T + j + 1] at every position) that makes
// several segments per CTA share L1 sectors. Middle, not first, entries: the
// first in-neighbours of PageRank hub rows are the same few early nodes.
__global__ void k_adjacent_count(const int32_t* p, const int32_t* idx, int32_t lo, int32_t hi, int* out) {
  int c = 0;
  GRID_STRIDE(s, (int64_t)(hi - lo - 1)) {
    const int32_t a = lo + static_cast<int32_t>(s);
    const int32_t l0 = p[a + 1] - p[a], l1 = p[a + 2] - p[a + 1];
    if (l0 > 0 && l1 > 0) {
      const int d = idx[p[a + 1] + l1 / 2] - idx[p[a] + l0 / 2];
      c += (d >= -3 && d <= 3) ? 1 : 0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Segment-order flags of the staged class-S kernel: warp group g (segments
// [32g, 32g + 32) of [0, s1)) is flagged when at least half of its adjacent
// pairs have equal lengths and middle entries exactly one index apart (shifted
// copies). *any counts flagged groups.
__global__ void k_rowmajor_flags(const int32_t* p, const int32_t* idx, int32_t s1, uint8_t* flag, int* any) {
  const int64_t ng = (static_cast<int64_t>(s1) + 31) / 32;
  int c = 0;
  GRID_STRIDE(g, ng) {
    const int32_t a = static_cast<int32_t>(g * 32), z = a + 32 < s1 ? a + 32 : s1;
    int hit = 0, pairs = 0;
    for (int32_t s = a; s + 1 < z; ++s) {
      const int32_t l0 = p[s + 1] - p[s], l1 = p[s + 2] - p[s + 1];
      ++pairs;
      if (l0 > 0 && l0 == l1 && idx[p[s + 1] + l1 / 2] == idx[p[s] + l0 / 2] + 1) ++hit;
    }
    const uint8_t f = pairs > 0 && 2 * hit >= pairs;
    flag[g] = f;
    c += f;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(any, c);
}

// Ghost plans: mark every gathered index; count marked indices per block.
__global__ void k_mark(const int32_t* idx, int64_t n, uint8_t* mark) {
  GRID_STRIDE(k, n) mark[idx[k]] = 1;
}
__global__ void k_block_count(const int32_t* list, int64_t n, int64_t slice, int32_t* count) {
  GRID_STRIDE(i, n) atomicAdd(count + list[i] / slice, 1);
}

// Sort key putting longer segments first: INT32_MAX - length.
__global__ void k_len_desc_key(const int32_t* p, int64_t nseg, int32_t* key) {
  GRID_STRIDE(s, nseg) key[s] = INT32_MAX - (p[s + 1] - p[s]);
}

// Secondary order key: the segment's first index in the other dimension
// (INT32_MAX for an empty segment). Segments whose patterns are shifted
// copies of each other (e.g. one node's conservation rows across
// commodities) become neighbours, so thread-per-segment gathers coalesce.
__global__ void k_first_index_key(const int32_t* p, const int32_t* idx, int64_t nseg, int32_t* key) {
  GRID_STRIDE(s, nseg) key[s] = p[s + 1] > p[s] ? idx[p[s]] : INT32_MAX;
}

// Largest nonzero count of a group of `g` consecutive segments in [s0, s1)
// (groups aligned at s0), into *out (initialised to 0).
__global__ void k_group_max(const int32_t* ptr, int32_t s0, int32_t s1, int g, int* out) {
  const int64_t ng = (static_cast<int64_t>(s1) - s0 + g - 1) / g;
  int mx = 0;
  GRID_STRIDE(q, ng) {
    const int64_t a = s0 + q * g, b = a + g < s1 ? a + g : s1;
    const int n = ptr[b] - ptr[a];
    mx = n > mx ? n : mx;
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// RunningAverage weight base after a block of `count` steps (graph-resident
// update of Scalars::inner_base).
__global__ void k_inner_add(Scalars* sc, int count) { sc->inner_base += static_cast<double>(count); }

__global__ void k_gather_i32(const int32_t* in, const int32_t* perm, int32_t* out, int64_t n) {
  GRID_STRIDE(i, n) out[i] = in[perm[i]];
}

// Histogram of class keys (< nkeys <= 512): per-block shared-memory counts,
// one global atomic per non-empty bin and block (a global atomic per key
// serialised on the few hot bins: 0.3 ms for 1M columns).
__global__ void k_key_hist(const int32_t* key, int64_t n, int32_t* hist, int nkeys) {
  __shared__ int32_t sh[512];
  for (int i = threadIdx.x; i < nkeys; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  GRID_STRIDE(i, n) atomicAdd(sh + key[i], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < nkeys; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

__global__ void k_invert(const int32_t* perm, int32_t* inv, int64_t n) {
  GRID_STRIDE(i, n) inv[perm[i]] = static_cast<int32_t>(i);
}

__global__ void k_perm_len(const int32_t* p, const int32_t* perm, int64_t n, int32_t* len) {
  GRID_STRIDE(i, n) len[i] = p[perm[i] + 1] - p[perm[i]];
}

// Move every nonzero of segment s to the permuted layout, keeping its
// position inside the segment; remap the other dimension's index.
__global__ void k_perm_nnz(const int32_t* p0, const int32_t* seg_of, const int32_t* idx0, const double* val0,
                           const int32_t* inv_seg, const int32_t* inv_other, const int32_t* p1, int32_t* idx1,
                           double* val1, int64_t nnz) {
  GRID_STRIDE(k, nnz) {
    const int32_t s = seg_of[k];
    const int64_t dst = p1[inv_seg[s]] + (k - p0[s]);
    idx1[dst] = inv_other[idx0[k]];
    val1[dst] = val0[k];
  }
}

// out[i] = in[inv[i]] * (scale ? scale[inv[i]] : 1)  (padded -> original).
__global__ void k_unpermute(const double* in, const double* scale, const int32_t* inv, double* out, int64_t n) {
  GRID_STRIDE(i, n) {
    const int32_t j = inv[i];
    out[i] = scale ? in[j] * scale[j] : in[j];
  }
}

// ------------------------------------------------------------- vectors
// Scaled (sparse_matrix.cpp:213, :218): (row_scale * v) * col_scale.
// seg_of is shard-local; `soff` moves it into the padded vector space.
__global__ void k_scale_vals(const int32_t* seg_of, const int32_t* idx, const double* vin, double* vout,
                             const double* rs, const double* cs, int64_t nnz, int csr_role, int64_t soff) {
  GRID_STRIDE(k, nnz) {
    const int64_t r = csr_role ? soff + seg_of[k] : idx[k];
    const int64_t c = csr_role ? idx[k] : soff + seg_of[k];
    vout[k] = rs[r] * vin[k] * cs[c];
  }
}

// *diff = 1 unless v[pad[j]] is bitwise equal to v[pad[0]] for every j.
__global__ void k_uniform(const double* v, const int32_t* pad, int64_t n, int* diff) {
  const unsigned long long ref = __double_as_longlong(v[pad[0]]);
  GRID_STRIDE(j, n) {
    if (static_cast<unsigned long long>(__double_as_longlong(v[pad[j]])) != ref) *diff = 1;
  }
}

// Reads a buffer twice the L2 size (16-byte loads) so that afterwards L2
// holds only clean lines of that buffer: the next kernel starts cold, and
// write-backs of earlier dirty lines happen here, not inside it.
__global__ void k_l2_sweep(const double2* buf, int64_t n, double* sink) {
  double acc = 0.0;
  GRID_STRIDE(i, n) {
    const double2 v = buf[i];
    acc += v.x + v.y;
  }
  if (acc == 1.2345e300) *sink = acc;  // never true: keeps the loads live
}

__global__ void k_fill(double* v, double a, int64_t n) {
  GRID_STRIDE(i, n) v[i] = a;
}
__global__ void k_mul(const double* a, const double* b, double* out, int64_t n) {
  GRID_STRIDE(i, n) out[i] = a[i] * b[i];
}
__global__ void k_div(const double* a, const double* b, double* out, int64_t n) {
  GRID_STRIDE(i, n) out[i] = a[i] / b[i];
}
// x0 = Clamp(0, l, u) (solver.cpp:240-243).
__global__ void k_clamp0(const double* l, const double* u, double* x, int64_t n) {
  GRID_STRIDE(i, n) x[i] = clamp_ref(0.0, l[i], u[i]);
}
__global__ void k_reflect(const double* xn, const double* xo, double* ext, int64_t n) {
  GRID_STRIDE(i, n) ext[i] = 2.0 * xn[i] - xo[i];  // solver.cpp:141
}

// ------------------------------------------------------- tile partitioning
// For the long-segment class [lo, hi) of one layout; positions are absolute.
__device__ int64_t upper_bound_i32(const int32_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ int64_t seg_end_pos(const int32_t* p, int64_t s, int64_t nz1) {
  const int64_t b = p[s], e = p[s + 1];
  const int64_t pos = e > b ? e - 1 : b;
  return pos < nz1 - 1 ? pos : nz1 - 1;
}

// K_s values in the ORIGINAL CSR order (parity probe), one row block at a
// time: original row r of the block is local segment pad[r] - roff.
__global__ void k_values_orig(const int32_t* p0, int64_t m, int64_t k0, int64_t k1, const int32_t* pad_r,
                              int64_t roff, const int32_t* p1, const double* v1, double* out) {
  GRID_STRIDE(q, k1 - k0) {
    const int64_t k = k0 + q;
    const int64_t r = upper_bound_i32(p0, m + 1, k) - 1;
    out[k] = v1[p1[pad_r[r] - roff] + (k - p0[r])];
  }
}

// Tile-boundary candidates: every kBlock-th segment start and every kTile-th
// nonzero inside segment groups of more than kTile nonzeros (snapped back to
// the start of a segment of <= kSnap nonzeros). Dropped: INT32_MAX.
__global__ void k_part_cand(const int32_t* p, int32_t lo, int32_t hi, int64_t nz0, int64_t nz1, int32_t ngroups,
                            int32_t ncuts, int32_t* cand) {
  GRID_STRIDE(i, (int64_t)ngroups + ncuts) {
    int64_t v = INT32_MAX;
    if (i < ngroups) {
      const int64_t pos = p[lo + i * (int64_t)kBlock];
      if (pos < nz1) v = pos;
    } else {
      const int64_t pos = nz0 + (i - ngroups + 1) * (int64_t)kTile;
      if (pos < nz1) {
        const int64_t s = lo + upper_bound_i32(p + lo, hi - lo + 1, pos) - 1;
        const int64_t g0 = lo + ((s - lo) / kBlock) * kBlock;
        const int64_t g1 = g0 + kBlock < hi ? g0 + kBlock : hi;
        if (p[g1] - p[g0] > kTile) {
          const int64_t st = p[s], len = p[s + 1] - st;
          v = (st < pos && len <= kSnap) ? st : pos;
        }
      }
    }
    cand[i] = static_cast<int32_t>(v);
  }
}

// Gather-window split of class S (Session::BuildSplit): per segment, the
// number of entries gathering below w, and a flag when an entry at or above
// w precedes one below it (the split would reorder that segment's sum).
__global__ void k_split_count(const int32_t* p, const int32_t* idx, int32_t s1, int32_t w, int32_t* cnt, int* bad) {
  GRID_STRIDE(s, s1) {
    int c = 0;
    bool high = false, viol = false;
    for (int32_t k = p[s]; k < p[s + 1]; ++k) {
      if (idx[k] < w) {
        ++c;
        viol |= high;
      } else {
        high = true;
      }
    }
    cnt[s] = c;
    if (viol) atomicOr(bad, 1);
  }
}
// Copies each segment's low entries to [plo[s], plo[s + 1]) and its high
// entries to [p[s] - plo[s], ...) of the two halves, storage order kept.
__global__ void k_split_copy(const int32_t* p, const int32_t* idx, const double* val, int32_t s1,
                             const int32_t* plo, int32_t* ilo, double* vlo, int32_t* phi, int32_t* ihi, double* vhi) {
  GRID_STRIDE(s, (int64_t)s1 + 1) {
    const int32_t b = p[s], lo = plo[s];
    phi[s] = b - lo;
    if (s < s1) {
      const int32_t nlo = plo[s + 1] - lo;
      for (int32_t k = 0; k < p[s + 1] - b; ++k) {
        if (k < nlo) {
          ilo[lo + k] = idx[b + k];
          vlo[lo + k] = val[b + k];
        } else {
          ihi[b - lo + k - nlo] = idx[b + k];
          vhi[b - lo + k - nlo] = val[b + k];
        }
      }
    }
  }
}

// Sort key of the gather sweep: the gathered index of each tile's first
// nonzero (tiles are never empty).
__global__ void k_tile_first_index(const int32_t* tb, const int32_t* idx, int32_t ntiles, int32_t* key) {
  GRID_STRIDE(t, (int64_t)ntiles) key[t] = idx[tb[t]];
}

__global__ void k_part_seg(const int32_t* p, int32_t lo, int32_t hi, int64_t nz1, int32_t ntiles, const int32_t* tb,
                           int32_t* ts) {
  GRID_STRIDE(t, (int64_t)ntiles + 1) {
    int64_t v;
    if (t == 0) {
      v = lo;
    } else if (t == ntiles) {
      v = hi;
    } else {
      const int64_t key = tb[t];
      int64_t a = lo, b = hi;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (seg_end_pos(p, mid, nz1) < key) a = mid + 1;
        else b = mid;
      }
      v = a;
    }
    ts[t] = static_cast<int32_t>(v);
  }
}

__global__ void k_part_span(const int32_t* p, int32_t hi, int64_t nz1, int32_t ntiles, const int32_t* tb,
                            const int32_t* ts, int32_t* hf, int32_t* to) {
  GRID_STRIDE(t, (int64_t)ntiles) {
    const int64_t sb = ts[t], se = ts[t + 1], kb = tb[t], ke = tb[t + 1];
    int32_t h = -1, o = -1;
    if (sb < se && p[sb] < kb) h = static_cast<int32_t>(upper_bound_i32(tb, ntiles + 1, p[sb]) - 1);
    if (se < hi && p[se] < ke) o = static_cast<int32_t>(upper_bound_i32(tb, ntiles + 1, seg_end_pos(p, se, nz1)) - 1);
    hf[t] = h;
    to[t] = o;
  }
}

// --------------------------------------------------------------- reductions
// out[i] = sum over slots (fixed order); one CTA per output.
// Thread-strided sum of slot i over ntiles partials (t = tid, tid + B, ...),
// in that order; loads are issued 8 at a time so a thread's whole chain is
// not one dependent DRAM round trip per partial.
__device__ __forceinline__ double slot_sum(const double* tile, const double* span, int ntiles, int nred, int i) {
  constexpr int U = 8;
  const int B = blockDim.x;
  double acc = 0.0;
  int t = threadIdx.x;
  for (; t + (U - 1) * B < ntiles; t += U * B) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t o = (int64_t)(t + u * B) * nred + i;
      v[u] = tile[o] + (span ? span[o] : 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  for (; t < ntiles; t += B) acc += tile[(int64_t)t * nred + i] + (span ? span[(int64_t)t * nred + i] : 0.0);
  return acc;
}

__global__ void k_reduce_tiles(const double* tile, const double* span, int ntiles, int nred, double* out) {
  __shared__ double sh[kBlock / 32];
  const int i = blockIdx.x;
  double acc = slot_sum(tile, span, ntiles, nred, i);
  acc = warp_combine<false>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v += sh[w];
    out[i] = v;
  }
}

// Both check reductions in one launch: blocks [0, n0) reduce layout 0's
// slots (n0 sums), blocks [n0, n0 + n1) layout 1's; same fixed order as
// k_reduce_tiles.
__global__ void k_reduce_two(const double* t0, int nt0, int n0, const double* t1, int nt1, int n1, double* out) {
  __shared__ double sh[kBlock / 32];
  const bool second = static_cast<int>(blockIdx.x) >= n0;
  const int i = second ? blockIdx.x - n0 : blockIdx.x;
  const double* tile = second ? t1 : t0;
  const int ntiles = second ? nt1 : nt0, nred = second ? n1 : n0;
  double acc = slot_sum(tile, nullptr, ntiles, nred, i);
  acc = warp_combine<false>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v += sh[w];
    out[blockIdx.x] = v;
  }
}

__global__ void k_sumsq_partial(const double* v, int64_t n, double* part) {
  __shared__ double sh[kEw / 32];
  double acc = 0.0;
  GRID_STRIDE(i, n) acc += v[i] * v[i];
  acc = warp_combine<false>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = sh[0];
    for (int w = 1; w < kEw / 32; ++w) s += sh[w];
    part[blockIdx.x] = s;
  }
}

// Power-iteration normalisation (solver.cpp:103-105).
// k_reduce_tiles for one sum (ntiles slots of stride 1) followed by
// k_power_norm, in one single-block launch (one shard, no NCCL).
__global__ void k_reduce_power_norm(const double* tile, int ntiles, double* out, Scalars* sc) {
  __shared__ double sh[kBlock / 32];
  double acc = slot_sum(tile, nullptr, ntiles, 1, 0);
  acc = warp_combine<false>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v += sh[w];
    out[0] = v;
    const double nr = sqrt(v);
    if (nr == 0.0) {
      sc->pw_zero = 1;
      sc->pw_norm = 1.0;
    } else {
      sc->pw_norm = nr;
    }
  }
}

__global__ void k_power_norm(const double* sum, Scalars* sc) {
  const double nr = sqrt(sum[0]);
  if (nr == 0.0) {
    sc->pw_zero = 1;
    sc->pw_norm = 1.0;
  } else {
    sc->pw_norm = nr;
  }
}

// AdaptStepSize (solver.cpp:310-328) from the per-iteration partials:
// k_adapt_sum folds one shard's tile partials into (|dx|^2, |dy|^2, dy.K dx),
// k_adapt_apply updates eta from the (shard- and rank-summed) triple.
__global__ void k_adapt_sum(const double* cred, int cn, const double* rred, int rn, double* out, const Scalars* sc) {
  if (sc->halt) return;
  __shared__ double sh[3][kBlock / 32];
  double a[3] = {0.0, 0.0, 0.0};
  for (int t = threadIdx.x; t < cn; t += blockDim.x) a[0] += cred[t];
  for (int t = threadIdx.x; t < rn; t += blockDim.x) {
    a[1] += rred[2 * t];
    a[2] += rred[2 * t + 1];
  }
  for (int k = 0; k < 3; ++k) {
    a[k] = warp_combine<false>(a[k]);
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = a[k];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double dx = 0, dy = 0, it = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    dx += sh[0][w];
    dy += sh[1][w];
    it += sh[2][w];
  }
  out[0] = dx;
  out[1] = dy;
  out[2] = it;
}

__global__ void k_adapt_apply(const double* sum, Scalars* sc, int j) {
  if (sc->halt) return;
  const double dx = sum[0], dy = sum[1];
  const double it = fabs(sum[2]);
  if (it <= 0.0) return;
  const double om = sc->omega;
  const double lim = (om * dx + dy / om) / (2.0 * it);
  const double k = sc->adapt_iter + static_cast<double>(j) + 1.0;
  const double a1 = lim * (1.0 - pow(k, -0.3));
  const double a2 = sc->eta * (1.0 + pow(k, -0.6));
  sc->eta = (a2 < a1) ? a2 : a1;  // std::min(a1, a2)
  set_steps(*sc);
}

}  // namespace pdhg
