// Device-side problem assembly: SparseMatrix::FromTriplets
// (reference sparse_matrix.cpp:25-69) -- sort triplets by (row, col), sum
// duplicates, drop exact zeros, emit CSR -- as a radix sort plus three
// elementwise passes, for the 1e8-1e9-nonzero instances whose host
// O(nnz log nnz) sort dominates problem building.
//
// The sort is stable, so duplicates are summed sequentially in input order;
// the reference sums them in its std::sort order. Two duplicates give the
// same sum either way (a + b == b + a); three or more can differ in the last
// ulp. Everything else is exact: same entries, same order, same zero drops.
#pragma once

#include <cub/cub.cuh>

#include <stdexcept>
#include <string>

#include "../../include/pdhg.h"
#include "common.cuh"
#include "darray.cuh"

namespace pdhg {

// key = row * cols + col; bad |= 1 for an index out of range.
static __global__ void k_trip_keys(const pdhg_triplet* t, int64_t count, int64_t rows, int64_t cols, uint64_t* key,
                            double* val, int* bad) {
  GRID_STRIDE(i, count) {
    const int64_t r = t[i].row, c = t[i].col;
    if (r < 0 || r >= rows || c < 0 || c >= cols) {
      *bad = 1;
      key[i] = 0;
    } else {
      key[i] = static_cast<uint64_t>(r) * static_cast<uint64_t>(cols) + static_cast<uint64_t>(c);
    }
    val[i] = t[i].value;
  }
}

// Run heads of the sorted keys sum their run in order; keep[i] = 1 for a
// head whose sum is nonzero. A run of three or more duplicates whose values
// are not all bitwise equal sets bit 1 of *flags: its sum would depend on
// the order the reference's std::sort leaves them in (equal values -- the
// generators' repeated edges -- sum to the same bits in any order).
static __global__ void k_trip_runs(const uint64_t* key, const int32_t* perm, const double* val, int64_t count, double* sum,
                            int32_t* keep, int* flags) {
  GRID_STRIDE(i, count) {
    int32_t k = 0;
    if (i == 0 || key[i] != key[i - 1]) {
      double s = 0.0;
      int64_t j = i;
      const double v0 = val[perm[i]];
      bool mixed = false;
      for (; j < count && key[j] == key[i]; ++j) {
        const double v = val[perm[j]];
        mixed |= __double_as_longlong(v) != __double_as_longlong(v0);
        s += v;
      }
      if (j - i >= 3 && mixed) atomicOr(flags, 2);
      sum[i] = s;
      k = s != 0.0;
    }
    keep[i] = k;
  }
}

static __global__ void k_trip_emit(const uint64_t* key, const double* sum, const int32_t* keep, const int32_t* pos,
                            int64_t count, int64_t cols, int64_t* col_idx, double* values, int32_t* row_cnt) {
  GRID_STRIDE(i, count) {
    if (!keep[i]) continue;
    const int64_t o = pos[i];
    col_idx[o] = static_cast<int64_t>(key[i] % static_cast<uint64_t>(cols));
    values[o] = sum[i];
    atomicAdd(row_cnt + key[i] / static_cast<uint64_t>(cols), 1);
  }
}

static __global__ void k_i32_to_i64(const int32_t* in, int64_t* out, int64_t n) { GRID_STRIDE(i, n) out[i] = in[i]; }

static __global__ void k_trip_iota(int32_t* v, int64_t n) { GRID_STRIDE(i, n) v[i] = static_cast<int32_t>(i); }

// Scaled (sparse_matrix.cpp:206-222) for one compressed layout: entry k of
// segment s with index i becomes row_scale * v * col_scale, multiplied left
// to right as the reference does; `seg_is_row` says which side s is.
template <bool kSegIsRow>
static __global__ void k_scale_entries(const int64_t* ptr, const int64_t* idx, const double* val, int64_t nseg,
                                       const double* seg_scale, const double* idx_scale, double* out) {
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x)
    for (int64_t k = ptr[s] + threadIdx.x; k < ptr[s + 1]; k += blockDim.x) {
      if constexpr (kSegIsRow) out[k] = seg_scale[s] * val[k] * idx_scale[idx[k]];
      else out[k] = idx_scale[idx[k]] * val[k] * seg_scale[s];
    }
}

// Both layouts of D_r M D_c (values only; the pattern is unchanged).
inline void ScaleEntries(const pdhg_csr& csr, const int64_t* col_ptr, const int64_t* row_idx, const double* csc_val,
                         const double* row_scale, const double* col_scale, int device, double* csr_out,
                         double* csc_out) {
  PDHG_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  PDHG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{st};
  AllocScope scope(st);
  const int64_t m = csr.rows, n = csr.cols, nnz = m ? csr.row_ptr[m] : 0;
  if (nnz == 0) return;
  DArray<int64_t> rp, ci, cp, ri;
  DArray<double> v, cv, rs, cs, o1, o2;
  rp.alloc(m + 1);
  ci.alloc(nnz);
  cp.alloc(n + 1);
  ri.alloc(nnz);
  v.alloc(nnz);
  cv.alloc(nnz);
  rs.alloc(std::max<int64_t>(m, 1));
  cs.alloc(std::max<int64_t>(n, 1));
  o1.alloc(nnz);
  o2.alloc(nnz);
  auto up = [&](void* d, const void* h, size_t b) { PDHG_CUDA(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, st)); };
  up(rp.p, csr.row_ptr, (m + 1) * sizeof(int64_t));
  up(ci.p, csr.col_idx, nnz * sizeof(int64_t));
  up(v.p, csr.values, nnz * sizeof(double));
  up(cp.p, col_ptr, (n + 1) * sizeof(int64_t));
  up(ri.p, row_idx, nnz * sizeof(int64_t));
  up(cv.p, csc_val, nnz * sizeof(double));
  if (m) up(rs.p, row_scale, m * sizeof(double));
  if (n) up(cs.p, col_scale, n * sizeof(double));
  k_scale_entries<true><<<ew_grid(m), 128, 0, st>>>(rp.p, ci.p, v.p, m, rs.p, cs.p, o1.p);
  k_scale_entries<false><<<ew_grid(n), 128, 0, st>>>(cp.p, ri.p, cv.p, n, cs.p, rs.p, o2.p);
  PDHG_CUDA(cudaMemcpyAsync(csr_out, o1.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
  PDHG_CUDA(cudaMemcpyAsync(csc_out, o2.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
  PDHG_CUDA(cudaStreamSynchronize(st));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(PDHG_CUDA_ERROR, std::string("scaled: ") + cudaGetErrorString(e));
}

// Host entry: triplets in host memory -> CSR in host memory (outputs sized
// rows + 1 / count / count by the caller); returns the entries written.
inline int64_t CsrFromTriplets(int64_t rows, int64_t cols, int64_t count, const pdhg_triplet* trips, int device,
                               int64_t* row_ptr, int64_t* col_idx, double* values) {
  if (rows < 0 || cols < 0) throw Error(PDHG_INVALID_ARGUMENT, "negative matrix dimension");
  if (count < 0) throw Error(PDHG_INVALID_ARGUMENT, "negative triplet count");
  if (count >= (int64_t(1) << 31) - 1 || rows >= (int64_t(1) << 31) - 1 || cols >= (int64_t(1) << 31) - 1)
    throw Error(PDHG_INVALID_ARGUMENT, "too many triplets for device assembly (< 2^31)");
  if (count > 0 && (rows == 0 || cols == 0)) throw std::out_of_range("triplet index out of range");
  PDHG_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  PDHG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{st};
  int64_t nnz = 0;
  {
    AllocScope scope(st);
    DArray<int32_t> cnt, cnt_out;
    cnt.alloc(rows + 1);
    PDHG_CUDA(cudaMemsetAsync(cnt.p, 0, (rows + 1) * sizeof(int32_t), st));
    if (count > 0) {
      DArray<pdhg_triplet> t;
      DArray<uint64_t> key, key_out;
      DArray<double> val, sum;
      DArray<int32_t> iota, perm, keep, pos;
      DArray<int> bad;
      t.alloc(count);
      key.alloc(count);
      key_out.alloc(count);
      val.alloc(count);
      sum.alloc(count);
      iota.alloc(count);
      perm.alloc(count);
      keep.alloc(count + 1);
      pos.alloc(count + 1);
      bad.alloc(1);
      PDHG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
      PDHG_CUDA(cudaMemcpyAsync(t.p, trips, count * sizeof(pdhg_triplet), cudaMemcpyHostToDevice, st));
      k_trip_keys<<<ew_grid(count), kEw, 0, st>>>(t.p, count, rows, cols, key.p, val.p, bad.p);
      int hbad = 0;
      PDHG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      PDHG_CUDA(cudaStreamSynchronize(st));
      if (hbad) throw std::out_of_range("triplet index out of range");
      k_trip_iota<<<ew_grid(count), kEw, 0, st>>>(iota.p, count);
      int bits = 1;
      const uint64_t maxkey = static_cast<uint64_t>(rows) * static_cast<uint64_t>(cols);
      while (bits < 64 && (uint64_t(1) << bits) < maxkey) ++bits;
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_out.p, iota.p, perm.p, static_cast<int>(count), 0, bits,
                                      st);
      DArray<char> tmp;
      tmp.alloc(std::max<size_t>(tb, 1));
      PDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key_out.p, iota.p, perm.p, static_cast<int>(count),
                                                0, bits, st));
      k_trip_runs<<<ew_grid(count), kEw, 0, st>>>(key_out.p, perm.p, val.p, count, sum.p, keep.p, bad.p);
      PDHG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      PDHG_CUDA(cudaStreamSynchronize(st));
      if (hbad & 2)
        throw Error(PDHG_ORDER_DEPENDENT, "an entry has three or more duplicates: its sum depends on the reference's "
                                          "std::sort order; assemble on the host");
      PDHG_CUDA(cudaMemsetAsync(keep.p + count, 0, sizeof(int32_t), st));
      size_t ts = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, ts, keep.p, pos.p, static_cast<int>(count + 1), st);
      DArray<char> stmp;
      stmp.alloc(std::max<size_t>(ts, 1));
      PDHG_CUDA(cub::DeviceScan::ExclusiveSum(stmp.p, ts, keep.p, pos.p, static_cast<int>(count + 1), st));
      int32_t n32 = 0;
      PDHG_CUDA(cudaMemcpyAsync(&n32, pos.p + count, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      PDHG_CUDA(cudaStreamSynchronize(st));
      nnz = n32;
      DArray<int64_t> dci;
      DArray<double> dv;
      dci.alloc(std::max<int64_t>(nnz, 1));
      dv.alloc(std::max<int64_t>(nnz, 1));
      k_trip_emit<<<ew_grid(count), kEw, 0, st>>>(key_out.p, sum.p, keep.p, pos.p, count, cols, dci.p, dv.p,
                                                   cnt.p + 1);
      if (nnz) {
        PDHG_CUDA(cudaMemcpyAsync(col_idx, dci.p, nnz * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        PDHG_CUDA(cudaMemcpyAsync(values, dv.p, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
      }
    }
    // row_ptr: inclusive scan of the per-row counts (cnt[0] = 0).
    cnt_out.alloc(rows + 1);
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.p, cnt_out.p, static_cast<int>(rows + 1), st);
    DArray<char> tmp;
    tmp.alloc(std::max<size_t>(tb, 1));
    PDHG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, cnt.p, cnt_out.p, static_cast<int>(rows + 1), st));
    DArray<int64_t> rp;
    rp.alloc(rows + 1);
    k_i32_to_i64<<<ew_grid(rows + 1), kEw, 0, st>>>(cnt_out.p, rp.p, rows + 1);
    PDHG_CUDA(cudaMemcpyAsync(row_ptr, rp.p, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PDHG_CUDA(cudaStreamSynchronize(st));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(PDHG_CUDA_ERROR, std::string("csr from triplets: ") + cudaGetErrorString(e));
  }
  return nnz;
}

}  // namespace pdhg
