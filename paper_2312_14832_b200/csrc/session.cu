// B200 restarted-PDHG session: device setup + solve loop orchestration.
//
// Reference map (all under /root/reference/proj/core/src):
//   Solve               solver.cpp:521-543   -> pdhg_solve (abi.cu) = Session + Solve
//   StackK / VStack     lp_problem.cpp:78-83, sparse_matrix.cpp:90-112 -> Session::Upload
//   BuildCscFromCsr     sparse_matrix.cpp:71-88 -> Session::BuildCsc (stable radix sort)
//   ComputeScaling      scaling.cpp:49-91    -> Session::ComputeScaling (device)
//   ApplyScaling        scaling.cpp:93-116   -> Session::ComputeScaling (device)
//   EstimateOpNorm      solver.cpp:84-110    -> Session::OpNorm
//   SolveLoop::Run      solver.cpp:232-267   -> Session::Solve
//   Step                solver.cpp:284-306   -> OpPrimal + OpDual (ops.cuh), CUDA graph per block
//   Check / Restart     solver.cpp:390-446   -> LaunchCheck + host decision logic
#include "session.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>

#include "host_logic.h"
#include "ops.cuh"

namespace pdhg {

namespace {

constexpr int kEw = 256;  // elementwise block size

inline int ew_grid(int64_t n) {
  int64_t g = (n + kEw - 1) / kEw;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16)));
}

#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- setup
__global__ void k_narrow(const int64_t* in, int32_t* out, int64_t count, int64_t limit, int* bad) {
  GRID_STRIDE(i, count) {
    const int64_t v = in[i];
    if (v < 0 || v >= limit) atomicOr(bad, 1);
    out[i] = static_cast<int32_t>(v);
  }
}

// K row_ptr = [A.row_ptr ; nnz(A) + G.row_ptr[1:]] (VStack, sparse_matrix.cpp:98-103).
__global__ void k_stack_ptr(const int64_t* ap, const int64_t* gp, int64_t m1, int64_t m2, int64_t nnz_a, int32_t* out) {
  GRID_STRIDE(i, m1 + m2 + 1) {
    out[i] = static_cast<int32_t>(i <= m1 ? ap[i] : nnz_a + gp[i - m1]);
  }
}

__global__ void k_check_ptr(const int32_t* p, int64_t rows, int64_t nnz, int* bad) {
  GRID_STRIDE(i, rows) {
    if (p[i] > p[i + 1]) atomicOr(bad, 2);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (p[0] != 0 || p[rows] != nnz)) atomicOr(bad, 2);
}

// Row id of every CSR nonzero: count row starts, then inclusive scan.
__global__ void k_row_marks(const int32_t* p, int64_t rows, int64_t nnz, int32_t* cnt) {
  GRID_STRIDE(r, rows) {
    if (r >= 1 && p[r] < nnz) atomicAdd(cnt + p[r], 1);
  }
}

__global__ void k_iota(int32_t* v, int64_t n) {
  GRID_STRIDE(i, n) v[i] = static_cast<int32_t>(i);
}

__global__ void k_csc_gather(const int32_t* perm, const int32_t* row_of, const double* v, int32_t* ri, double* cv,
                             int64_t nnz) {
  GRID_STRIDE(q, nnz) {
    const int32_t k = perm[q];
    ri[q] = row_of[k];
    cv[q] = v[k];
  }
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

// Scaled (sparse_matrix.cpp:213, :218): (row_scale * v) * col_scale.
__global__ void k_scale_vals(const int32_t* seg_of, const int32_t* idx, const double* vin, double* vout,
                             const double* rs, const double* cs, int64_t nnz, int csr_role) {
  GRID_STRIDE(k, nnz) {
    const int32_t r = csr_role ? seg_of[k] : idx[k];
    const int32_t c = csr_role ? idx[k] : seg_of[k];
    vout[k] = rs[r] * vin[k] * cs[c];
  }
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

// ------------------------------------------------------- tile partitioning
__device__ int64_t upper_bound_i32(const int32_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Effective end position of a segment (its last nonzero; empty segments sit
// at their start), clamped into the last tile.
__device__ int64_t seg_end_pos(const int32_t* p, int64_t s, int64_t nnz) {
  const int64_t b = p[s], e = p[s + 1];
  const int64_t pos = e > b ? e - 1 : b;
  return pos < nnz - 1 ? pos : nnz - 1;
}

__global__ void k_part_begin(const int32_t* p, int32_t nseg, int64_t nnz, int32_t ntiles, int32_t* tb) {
  GRID_STRIDE(t, (int64_t)ntiles + 1) {
    int64_t v;
    if (t == ntiles) {
      v = nnz;
    } else if (t == 0) {
      v = 0;
    } else {
      const int64_t pos = t * (int64_t)kTile;
      const int64_t s = upper_bound_i32(p, nseg + 1, pos) - 1;
      const int64_t st = p[s], len = p[s + 1] - st;
      v = (st < pos && len <= kSnap) ? st : pos;
    }
    tb[t] = static_cast<int32_t>(v);
  }
}

__global__ void k_part_seg(const int32_t* p, int32_t nseg, int64_t nnz, int32_t ntiles, const int32_t* tb,
                           int32_t* ts) {
  GRID_STRIDE(t, (int64_t)ntiles + 1) {
    int64_t v;
    if (t == 0 || nnz == 0) {
      v = (t == 0) ? 0 : nseg;
    } else if (t == ntiles) {
      v = nseg;
    } else {
      const int64_t key = tb[t];
      int64_t lo = 0, hi = nseg;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (seg_end_pos(p, mid, nnz) < key) lo = mid + 1;
        else hi = mid;
      }
      v = lo;
    }
    ts[t] = static_cast<int32_t>(v);
  }
}

__global__ void k_part_span(const int32_t* p, int32_t nseg, int64_t nnz, int32_t ntiles, const int32_t* tb,
                            const int32_t* ts, int32_t* hf, int32_t* to) {
  GRID_STRIDE(t, (int64_t)ntiles) {
    const int64_t sb = ts[t], se = ts[t + 1], kb = tb[t], ke = tb[t + 1];
    int32_t h = -1, o = -1;
    if (nnz > 0) {
      if (sb < se && p[sb] < kb) h = static_cast<int32_t>(upper_bound_i32(tb, ntiles + 1, p[sb]) - 1);
      if (se < nseg && p[se] < ke)
        o = static_cast<int32_t>(upper_bound_i32(tb, ntiles + 1, seg_end_pos(p, se, nnz)) - 1);
    }
    hf[t] = h;
    to[t] = o;
  }
}

// --------------------------------------------------------------- reductions
// out[i] = sum_t (tile[t][i] + span[t][i]), fixed order; one CTA per output.
__global__ void k_reduce_tiles(const double* tile, const double* span, int ntiles, int nred, double* out) {
  __shared__ double sh[kBlock / 32];
  const int i = blockIdx.x;
  double acc = 0.0;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x)
    acc += tile[(int64_t)t * nred + i] + (span ? span[(int64_t)t * nred + i] : 0.0);
  acc = warp_combine<false>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v += sh[w];
    out[i] = v;
  }
}

// Deterministic sum of squares, two stages.
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

// Power-iteration normalisation (solver.cpp:103-105): norm = sqrt(sum);
// norm == 0 ends the estimate with 0 (flagged, host returns 0).
__global__ void k_power_norm(const double* sum, Scalars* sc) {
  const double nr = sqrt(sum[0]);
  if (nr == 0.0) {
    sc->pw_zero = 1;
    sc->pw_norm = 1.0;
  } else {
    sc->pw_norm = nr;
  }
}

// AdaptStepSize (solver.cpp:310-328) from the per-iteration partials.
__global__ void k_adapt(const double* ctile, const double* cspan, int cnt, const double* rtile, const double* rspan,
                        int rnt, Scalars* sc, int j) {
  __shared__ double sh[3][kBlock / 32];
  double a[3] = {0.0, 0.0, 0.0};
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) a[0] += ctile[t] + cspan[t];
  for (int t = threadIdx.x; t < rnt; t += blockDim.x) {
    a[1] += rtile[2 * t] + rspan[2 * t];
    a[2] += rtile[2 * t + 1] + rspan[2 * t + 1];
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
  it = fabs(it);
  if (it <= 0.0) return;
  const double om = sc->omega;
  const double lim = (om * dx + dy / om) / (2.0 * it);
  const double k = sc->adapt_iter + static_cast<double>(j) + 1.0;
  const double a1 = lim * (1.0 - pow(k, -0.3));
  const double a2 = sc->eta * (1.0 + pow(k, -0.6));
  sc->eta = (a2 < a1) ? a2 : a1;  // std::min(a1, a2)
}

template <class T>
void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(PDHG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// Host mirror of the check reductions (26 doubles).
struct CheckOut {
  double row[kRowRed];
  double col[kColRed];
};

// ============================================================== construction
Session::Session(const pdhg_lp& lp, const pdhg_params& prm, int device) : device_(device) {
  PDHG_CUDA(cudaSetDevice(device_));
  PDHG_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  PDHG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&host_red_), sizeof(CheckOut) + 64));
  m1_ = lp.a.rows;
  m2_ = lp.g.rows;
  m_ = m1_ + m2_;
  n_ = lp.n;
  offset_ = lp.objective_offset;
  const double t0 = now_s();
  Upload(lp);
  BuildCsc();
  Sync();
  Partition(csr_);
  Partition(csc_);
  Sync();
  upload_s_ = now_s() - t0;
  const double t1 = now_s();
  ComputeScaling(prm);
  Sync();
  scaling_s_ = now_s() - t1;
  // Iterate state.
  for (int p = 0; p < 2; ++p) {
    x_[p].alloc(n_, &arena_);
    y_[p].alloc(m_, &arena_);
    kx_[p].alloc(m_, &arena_);
  }
  xbar_.alloc(n_, &arena_);
  xstart_.alloc(n_, &arena_);
  xbest_.alloc(n_, &arena_);
  nvec_.alloc(n_, &arena_);
  ybar_.alloc(m_, &arena_);
  ystart_.alloc(m_, &arena_);
  ybest_.alloc(m_, &arena_);
  kxavg_.alloc(m_, &arena_);
  scal_.alloc(1, &arena_);
  for (int r = 0; r < 2; ++r) {
    const CMat& M = r == 0 ? csr_ : csc_;
    const int nred = std::max(kRowRed, kColRed);
    red_tile_[r].alloc((size_t)M.ntiles * nred, &arena_);
    red_span_[r].alloc((size_t)M.ntiles * nred, &arena_);
  }
  red_out_.alloc(64, &arena_);
  DeviceNorms();
  // Working set of one iteration vs L2 (126 MB on B200).
  const double iter_bytes = 24.0 * nnz_ + 68.0 * (m_ + n_);
  l2_resident_ = iter_bytes < 100e6;
  Sync();
}

Session::~Session() {
  cudaSetDevice(device_);
  for (cudaEvent_t e : ev_)
    if (e) cudaEventDestroy(e);
  for (Graph& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (host_red_) cudaFreeHost(host_red_);
  if (st_) cudaStreamDestroy(st_);
}

void Session::Sync() { PDHG_CUDA(cudaStreamSynchronize(st_)); }

void Session::Copy(double* dst, const double* src, size_t n) {
  if (n) PDHG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st_));
}

// H2D + int64 -> int32 narrowing + VStack of A and G straight into K's CSR.
void Session::Upload(const pdhg_lp& lp) {
  const int64_t nnz_a = lp.a.rows ? lp.a.row_ptr[lp.a.rows] : 0;
  const int64_t nnz_g = lp.g.rows ? lp.g.row_ptr[lp.g.rows] : 0;
  nnz_ = nnz_a + nnz_g;
  if (nnz_ >= (int64_t(1) << 31) - kTile || m_ >= (int64_t(1) << 31) - 1 || n_ >= (int64_t(1) << 31) - 1)
    throw Error(PDHG_INVALID_ARGUMENT, "problem too large for int32 device indices (nnz, rows, cols < 2^31)");
  csr_ptr_.alloc(m_ + 1, &arena_);
  csr_idx_.alloc(nnz_, &arena_);
  csr_val_.alloc(nnz_, &arena_);
  DArray<int64_t> stage;
  stage.alloc(std::max<int64_t>({nnz_a, nnz_g, m1_ + 1, m2_ + 1, 1}) * 2);
  DArray<int> bad;
  bad.alloc(1);
  PDHG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st_));
  // Row pointers.
  int64_t* ap = stage.p;
  int64_t* gp = stage.p + std::max<int64_t>(m1_ + 1, 1);
  PDHG_CUDA(cudaMemcpyAsync(ap, lp.a.row_ptr, (m1_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
  PDHG_CUDA(cudaMemcpyAsync(gp, lp.g.row_ptr, (m2_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
  k_stack_ptr<<<ew_grid(m_ + 1), kEw, 0, st_>>>(ap, gp, m1_, m2_, nnz_a, csr_ptr_.p);
  Sync();
  // Column indices and values.
  if (nnz_a) {
    PDHG_CUDA(cudaMemcpyAsync(stage.p, lp.a.col_idx, nnz_a * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    k_narrow<<<ew_grid(nnz_a), kEw, 0, st_>>>(stage.p, csr_idx_.p, nnz_a, n_, bad.p);
    PDHG_CUDA(cudaMemcpyAsync(csr_val_.p, lp.a.values, nnz_a * sizeof(double), cudaMemcpyHostToDevice, st_));
    Sync();
  }
  if (nnz_g) {
    PDHG_CUDA(cudaMemcpyAsync(stage.p, lp.g.col_idx, nnz_g * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    k_narrow<<<ew_grid(nnz_g), kEw, 0, st_>>>(stage.p, csr_idx_.p + nnz_a, nnz_g, n_, bad.p);
    PDHG_CUDA(cudaMemcpyAsync(csr_val_.p + nnz_a, lp.g.values, nnz_g * sizeof(double), cudaMemcpyHostToDevice, st_));
  }
  k_check_ptr<<<ew_grid(m_), kEw, 0, st_>>>(csr_ptr_.p, m_, nnz_, bad.p);
  // Vectors (original space).
  c_o_.alloc(n_, &arena_);
  l_o_.alloc(n_, &arena_);
  u_o_.alloc(n_, &arena_);
  q_o_.alloc(m_, &arena_);
  auto h2d = [&](double* d, const double* h, int64_t k) {
    if (k) PDHG_CUDA(cudaMemcpyAsync(d, h, k * sizeof(double), cudaMemcpyHostToDevice, st_));
  };
  h2d(c_o_.p, lp.c, n_);
  h2d(l_o_.p, lp.l, n_);
  h2d(u_o_.p, lp.u, n_);
  h2d(q_o_.p, lp.b, m1_);
  h2d(q_o_.p + m1_, lp.h, m2_);
  int hbad = 0;
  PDHG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
  Sync();
  if (hbad & 1) throw Error(PDHG_INVALID_ARGUMENT, "column index out of range");
  if (hbad & 2) throw Error(PDHG_INVALID_ARGUMENT, "row_ptr is not a valid CSR offset array");
  csr_.nseg = static_cast<int32_t>(m_);
  csr_.nvec = static_cast<int32_t>(n_);
  csr_.nnz = nnz_;
  csr_.ptr = csr_ptr_.p;
  csr_.idx = csr_idx_.p;
  csr_.val = csr_val_.p;
}

// CSC of K via a stable radix sort of (column, CSR position): rows stay in
// ascending order inside each column, as BuildCscFromCsr guarantees.
void Session::BuildCsc() {
  csc_ptr_.alloc(n_ + 1, &arena_);
  csc_idx_.alloc(nnz_, &arena_);
  csc_val_.alloc(nnz_, &arena_);
  csc_.nseg = static_cast<int32_t>(n_);
  csc_.nvec = static_cast<int32_t>(m_);
  csc_.nnz = nnz_;
  csc_.ptr = csc_ptr_.p;
  csc_.idx = csc_idx_.p;
  csc_.val = csc_val_.p;
  if (nnz_ == 0) {
    PDHG_CUDA(cudaMemsetAsync(csc_ptr_.p, 0, (n_ + 1) * sizeof(int32_t), st_));
    return;
  }
  DArray<int32_t> row_of, perm_in, perm_out, keys_out;
  row_of.alloc(nnz_);
  perm_in.alloc(nnz_);
  perm_out.alloc(nnz_);
  keys_out.alloc(nnz_);
  PDHG_CUDA(cudaMemsetAsync(row_of.p, 0, nnz_ * sizeof(int32_t), st_));
  k_row_marks<<<ew_grid(m_), kEw, 0, st_>>>(csr_ptr_.p, m_, nnz_, row_of.p);
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, row_of.p, row_of.p, (int)nnz_, st_);
  int end_bit = 1;
  while ((int64_t(1) << end_bit) <= n_) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp2, csr_idx_.p, keys_out.p, perm_in.p, perm_out.p, (int)nnz_, 0,
                                  end_bit, st_);
  DArray<char> tmp;
  tmp.alloc(std::max(tmp_bytes, tmp2));
  PDHG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, row_of.p, row_of.p, (int)nnz_, st_));
  k_iota<<<ew_grid(nnz_), kEw, 0, st_>>>(perm_in.p, nnz_);
  PDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp2, csr_idx_.p, keys_out.p, perm_in.p, perm_out.p, (int)nnz_, 0,
                                            end_bit, st_));
  k_csc_gather<<<ew_grid(nnz_), kEw, 0, st_>>>(perm_out.p, row_of.p, csr_val_.p, csc_idx_.p, csc_val_.p, nnz_);
  k_colptr<<<ew_grid(n_ + 1), kEw, 0, st_>>>(keys_out.p, nnz_, n_, csc_ptr_.p);
  Sync();
}

// Tile partition of one layout (see tile_spmv.cuh).
void Session::Partition(CMat& M) {
  const int r = (&M == &csr_) ? 0 : 1;
  M.ntiles = std::max(1, ceil_div(M.nnz, kTile));
  for (int k = 0; k < 4; ++k) part_[r][k].alloc(M.ntiles + 1, &arena_);
  head_[r].alloc(2 * (size_t)M.ntiles, &arena_);
  tail_[r].alloc(2 * (size_t)M.ntiles, &arena_);
  cnt_[r].alloc(M.ntiles, &arena_);
  PDHG_CUDA(cudaMemsetAsync(cnt_[r].p, 0, M.ntiles * sizeof(unsigned), st_));
  M.tile_begin = part_[r][0].p;
  M.tile_seg = part_[r][1].p;
  M.head_first = part_[r][2].p;
  M.tail_owner = part_[r][3].p;
  M.head_part = head_[r].p;
  M.tail_part = tail_[r].p;
  M.counter = cnt_[r].p;
  const int g = ew_grid(M.ntiles + 1);
  k_part_begin<<<g, kEw, 0, st_>>>(M.ptr, M.nseg, M.nnz, M.ntiles, M.tile_begin);
  k_part_seg<<<g, kEw, 0, st_>>>(M.ptr, M.nseg, M.nnz, M.ntiles, M.tile_begin, M.tile_seg);
  k_part_span<<<g, kEw, 0, st_>>>(M.ptr, M.nseg, M.nnz, M.ntiles, M.tile_begin, M.tile_seg, M.head_first,
                                  M.tail_owner);
  check_launch<int>("partition");
}

// Ruiz x10 + Pock-Chambolle on device (scaling.cpp:49-91), then
// ApplyScaling (scaling.cpp:93-116): K_s = (rs * K) * cs from the ORIGINAL
// values with the composed scales, c_s = c cs, l_s = l / cs, u_s = u / cs,
// q_s = q rs. Max is exact and 1/sqrt is IEEE on both sides, so the scales
// are bit-identical to the reference (power sums too for rows/cols of <= 32
// nonzeros, which are summed in storage order).
void Session::ComputeScaling(const pdhg_params& prm) {
  rs_.alloc(m_, &arena_);
  cs_.alloc(n_, &arena_);
  c_s_.alloc(n_, &arena_);
  l_s_.alloc(n_, &arena_);
  u_s_.alloc(n_, &arena_);
  q_s_.alloc(m_, &arena_);
  k_fill<<<ew_grid(m_), kEw, 0, st_>>>(rs_.p, 1.0, m_);
  k_fill<<<ew_grid(n_), kEw, 0, st_>>>(cs_.p, 1.0, n_);
  scaled_ = prm.scaling_enabled != 0;
  if (scaled_ && (prm.pc_alpha < 0.0 || prm.pc_alpha > 2.0))
    throw Error(PDHG_INVALID_ARGUMENT, "pock-chambolle alpha must lie in [0, 2]");
  if (scaled_ && nnz_ > 0) {
    DArray<int32_t> row_of, col_of;
    row_of.alloc(nnz_);
    col_of.alloc(nnz_);
    PDHG_CUDA(cudaMemsetAsync(row_of.p, 0, nnz_ * sizeof(int32_t), st_));
    k_row_marks<<<ew_grid(m_), kEw, 0, st_>>>(csr_ptr_.p, m_, nnz_, row_of.p);
    PDHG_CUDA(cudaMemsetAsync(col_of.p, 0, nnz_ * sizeof(int32_t), st_));
    k_row_marks<<<ew_grid(n_), kEw, 0, st_>>>(csc_ptr_.p, n_, nnz_, col_of.p);
    {
      size_t tb = 0;
      cub::DeviceScan::InclusiveSum(nullptr, tb, row_of.p, row_of.p, (int)nnz_, st_);
      DArray<char> tmp;
      tmp.alloc(tb);
      PDHG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, row_of.p, row_of.p, (int)nnz_, st_));
      PDHG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, col_of.p, col_of.p, (int)nnz_, st_));
    }
    DArray<double> orig_r, orig_c, dr, dc;
    orig_r.alloc(nnz_);
    orig_c.alloc(nnz_);
    dr.alloc(m_);
    dc.alloc(n_);
    Copy(orig_r.p, csr_val_.p, nnz_);
    Copy(orig_c.p, csc_val_.p, nnz_);
    for (int s = 0; s < prm.ruiz_iters; ++s) {
      launch_tiles(csr_, OpInfNormScale{dr.p, rs_.p}, nullptr, nullptr, st_);
      launch_tiles(csc_, OpInfNormScale{dc.p, cs_.p}, nullptr, nullptr, st_);
      k_scale_vals<<<ew_grid(nnz_), kEw, 0, st_>>>(row_of.p, csr_idx_.p, csr_val_.p, csr_val_.p, dr.p, dc.p, nnz_, 1);
      k_scale_vals<<<ew_grid(nnz_), kEw, 0, st_>>>(col_of.p, csc_idx_.p, csc_val_.p, csc_val_.p, dr.p, dc.p, nnz_, 0);
    }
    // PC on K.Scaled(ruiz) recomputed from the original values (scaling.cpp:89).
    k_scale_vals<<<ew_grid(nnz_), kEw, 0, st_>>>(row_of.p, csr_idx_.p, orig_r.p, csr_val_.p, rs_.p, cs_.p, nnz_, 1);
    k_scale_vals<<<ew_grid(nnz_), kEw, 0, st_>>>(col_of.p, csc_idx_.p, orig_c.p, csc_val_.p, rs_.p, cs_.p, nnz_, 0);
    auto mode_of = [](double p) { return p == 0.0 ? 0 : (p == 1.0 ? 1 : (p == 2.0 ? 2 : 3)); };
    const double pr = 2.0 - prm.pc_alpha, pc = prm.pc_alpha;
    launch_tiles(csr_, OpPowerSumScale{pr, mode_of(pr), rs_.p}, nullptr, nullptr, st_);
    launch_tiles(csc_, OpPowerSumScale{pc, mode_of(pc), cs_.p}, nullptr, nullptr, st_);
    // Final K_s from the original values (ApplyScaling, scaling.cpp:105-106).
    k_scale_vals<<<ew_grid(nnz_), kEw, 0, st_>>>(row_of.p, csr_idx_.p, orig_r.p, csr_val_.p, rs_.p, cs_.p, nnz_, 1);
    k_scale_vals<<<ew_grid(nnz_), kEw, 0, st_>>>(col_of.p, csc_idx_.p, orig_c.p, csc_val_.p, rs_.p, cs_.p, nnz_, 0);
    check_launch<int>("scaling");
    Sync();
  }
  // Vectors (scaling.cpp:107-115). With identity scales these are exact copies.
  k_mul<<<ew_grid(n_), kEw, 0, st_>>>(c_o_.p, cs_.p, c_s_.p, n_);
  k_div<<<ew_grid(n_), kEw, 0, st_>>>(l_o_.p, cs_.p, l_s_.p, n_);
  k_div<<<ew_grid(n_), kEw, 0, st_>>>(u_o_.p, cs_.p, u_s_.p, n_);
  k_mul<<<ew_grid(m_), kEw, 0, st_>>>(q_o_.p, rs_.p, q_s_.p, m_);
  check_launch<int>("apply scaling");
}

// ||c||, ||q|| in both spaces (kkt.cpp:45-56), deterministic device sums.
void Session::DeviceNorms() {
  const int g = 148;
  DArray<double> part, out;
  part.alloc(g * 4);
  out.alloc(4);
  const double* vecs[4] = {c_s_.p, q_s_.p, c_o_.p, q_o_.p};
  const int64_t lens[4] = {n_, m_, n_, m_};
  for (int k = 0; k < 4; ++k) {
    k_sumsq_partial<<<g, kEw, 0, st_>>>(vecs[k], lens[k], part.p + k * g);
    k_reduce_tiles<<<1, kBlock, 0, st_>>>(part.p + k * g, nullptr, g, 1, out.p + k);
  }
  double h[4];
  PDHG_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, st_));
  Sync();
  c_norm_s_ = std::sqrt(h[0]);
  q_norm_s_ = std::sqrt(h[1]);
  c_norm_o_ = std::sqrt(h[2]);
  q_norm_o_ = std::sqrt(h[3]);
}

// ================================================================== kernels
void Session::LaunchStep(int parity, int j, bool adapt) {
  const int a = parity, b = 1 - parity;
  launches_ += adapt ? 3 : 2;
  if (adapt) {
    launch_tiles(csc_, OpPrimal<true>{y_[a].p, x_[a].p, x_[b].p, xbar_.p, c_s_.p, l_s_.p, u_s_.p, scal_.p, j},
                 red_tile_[1].p, red_span_[1].p, st_);
    launch_tiles(csr_, OpDual<true>{x_[b].p, y_[a].p, y_[b].p, ybar_.p, kx_[a].p, kx_[b].p, q_s_.p, (int32_t)m1_, scal_.p, j},
                 red_tile_[0].p, red_span_[0].p, st_);
    k_adapt<<<1, kBlock, 0, st_>>>(red_tile_[1].p, red_span_[1].p, csc_.ntiles, red_tile_[0].p, red_span_[0].p,
                                   csr_.ntiles, scal_.p, j);
  } else {
    launch_tiles(csc_, OpPrimal<false>{y_[a].p, x_[a].p, x_[b].p, xbar_.p, c_s_.p, l_s_.p, u_s_.p, scal_.p, j},
                 nullptr, nullptr, st_);
    launch_tiles(csr_, OpDual<false>{x_[b].p, y_[a].p, y_[b].p, ybar_.p, kx_[a].p, kx_[b].p, q_s_.p, (int32_t)m1_, scal_.p, j},
                 nullptr, nullptr, st_);
  }
}

// `count` PDHG iterations starting from buffer `parity`. Full check blocks are
// replayed from a captured CUDA graph (one per parity/length/adapt combo).
void Session::RunSteps(int parity, int count, bool adapt) {
  Graph* g = nullptr;
  for (Graph& gg : graphs_)
    if (gg.steps == count && gg.parity == parity && gg.adapt == adapt) g = &gg;
  if (!g && count >= 4) {
    cudaGraph_t graph;
    PDHG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, adapt);
    PDHG_CUDA(cudaStreamEndCapture(st_, &graph));
    Graph ng;
    ng.steps = count;
    ng.parity = parity;
    ng.adapt = adapt;
    PDHG_CUDA(cudaGraphInstantiate(&ng.exec, graph, 0));
    cudaGraphDestroy(graph);
    graphs_.push_back(ng);
    g = &graphs_.back();
  }
  if (g) {
    launches_ += static_cast<int64_t>(count) * (adapt ? 3 : 2);
    PDHG_CUDA(cudaGraphLaunch(g->exec, st_));
  } else {
    for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, adapt);
  }
  check_launch<int>("pdhg steps");
}

void Session::LaunchCheck(const double* x, const double* y, const double* xb, const double* yb, const double* kx) {
  launches_ += 4;
  OpCheckRow row{xb, kxavg_.p, kx, y, yb, ystart_.p, q_s_.p, q_o_.p, rs_.p, (int32_t)m1_};
  launch_tiles(csr_, row, red_tile_[0].p, red_span_[0].p, st_);
  OpCheckCol col{y, yb, x, xb, xstart_.p, c_s_.p, l_s_.p, u_s_.p, c_o_.p, l_o_.p, u_o_.p, cs_.p};
  launch_tiles(csc_, col, red_tile_[1].p, red_span_[1].p, st_);
  k_reduce_tiles<<<kRowRed, kBlock, 0, st_>>>(red_tile_[0].p, red_span_[0].p, csr_.ntiles, kRowRed, red_out_.p);
  k_reduce_tiles<<<kColRed, kBlock, 0, st_>>>(red_tile_[1].p, red_span_[1].p, csc_.ntiles, kColRed,
                                              red_out_.p + kRowRed);
  check_launch<int>("check");
}

void Session::ReadCheck(CheckOut* out) {
  PDHG_CUDA(cudaMemcpyAsync(host_red_, red_out_.p, sizeof(CheckOut), cudaMemcpyDeviceToHost, st_));
  Sync();
  std::memcpy(out, host_red_, sizeof(CheckOut));
}

// ================================================================ solve loop
namespace {

}  // namespace

void Session::Solve(const pdhg_params& prm, pdhg_eval_cb cb, void* user, pdhg_result* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  if (!ev_[0]) {
    PDHG_CUDA(cudaEventCreate(&ev_[0]));
    PDHG_CUDA(cudaEventCreate(&ev_[1]));
  }
  launches_ = 0;
  PDHG_CUDA(cudaEventRecord(ev_[0], st_));
  const auto t0 = std::chrono::steady_clock::now();
  auto secs = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };

  // eta = 0.9 / ||K|| (solver.cpp:233-234), omega0 = ||c_s|| / ||q_s|| (:235-238).
  const double op = OpNorm(100, prm.seed);
  Scalars sc{};
  sc.eta = op > 0.0 ? 0.9 / op : 1.0;
  sc.omega = 1.0;
  if (c_norm_s_ > 1e-10 && q_norm_s_ > 1e-10) sc.omega = c_norm_s_ / q_norm_s_;
  sc.inner_base = 0.0;
  sc.pw_norm = 1.0;
  const bool adapt = prm.adaptive_step != 0;

  // x0 = proj(0), y0 = 0, kx = K x0 (solver.cpp:240-245).
  int par = 0;
  k_clamp0<<<ew_grid(n_), kEw, 0, st_>>>(l_s_.p, u_s_.p, x_[0].p, n_);
  if (m_) PDHG_CUDA(cudaMemsetAsync(y_[0].p, 0, m_ * sizeof(double), st_));
  launch_tiles(csr_, OpSpmv{x_[0].p, kx_[0].p}, nullptr, nullptr, st_);

  int64_t iters = 0, inner = 0, restarts = 0;
  double kkt_start = 0.0, kkt_prev = std::numeric_limits<double>::infinity();
  bool have_best = false;
  double best_k1 = 0.0;
  pdhg_report best_rep{}, last_rep{};
  int status = PDHG_ITER_LIMIT;
  int64_t last_log = -1;
  CheckOut ck{};

  auto reports = [&](int P, pdhg_report* scaled, pdhg_report* orig) {
    const double* r = ck.row + P * kRowPer;
    const double* c = ck.col + P * kColPer;
    *scaled = MakeReport(r[kPrS], c[kDuS], c[kBdS], c[kCxS], r[kQyS], offset_, q_norm_s_, c_norm_s_);
    *orig = MakeReport(r[kPrO], c[kDuO], c[kBdO], c[kCxO], r[kQyO], offset_, q_norm_o_, c_norm_o_);
  };
  auto copy_best = [&](int P) {
    Copy(xbest_.p, P == 0 ? x_[par].p : xbar_.p, n_);
    Copy(ybest_.p, P == 0 ? y_[par].p : ybar_.p, m_);
  };
  // RecordBest (solver.cpp:341-351).
  auto record_best = [&](int P, const pdhg_report& r) {
    const double k1 = Kkt1(r);
    if (!have_best || k1 < best_k1) {
      have_best = true;
      best_k1 = k1;
      copy_best(P);
      best_rep = r;
    }
  };
  // StartLoopAt (solver.cpp:275-281) with the candidate's scaled residuals.
  auto start_loop = [&](const pdhg_report& s) {
    Copy(xstart_.p, x_[par].p, n_);
    Copy(ystart_.p, y_[par].p, m_);
    kkt_start = KktError(s.primal_res, s.dual_res, s.gap_abs, sc.omega);
    kkt_prev = std::numeric_limits<double>::infinity();
    sc.inner_base = 0.0;
    inner = 0;
  };
  auto push_scalars = [&] {
    PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  };

  // Start point: scaled KKT for the loop start and the first termination test
  // (solver.cpp:246-249). The running average is not formed yet: evaluate
  // the current point as both operands.
  LaunchCheck(x_[0].p, y_[0].p, x_[0].p, y_[0].p, kx_[0].p);
  ReadCheck(&ck);
  pdhg_report s_cur, o_cur, s_avg, o_avg;
  reports(0, &s_cur, &o_cur);
  start_loop(s_cur);
  push_scalars();
  bool finished = false;
  if (Terminated(o_cur, prm.eps)) {
    status = PDHG_OPTIMAL;
    copy_best(0);
    best_rep = o_cur;
    have_best = true;
    finished = true;
  } else {
    record_best(0, o_cur);
    last_rep = o_cur;
  }

  while (!finished) {
    if (iters >= prm.iter_limit) {
      status = PDHG_ITER_LIMIT;
      break;
    }
    if (secs() >= prm.time_limit) {
      status = PDHG_TIME_LIMIT;
      break;
    }
    const int64_t to_check = prm.check_every - (iters % prm.check_every);
    const int64_t count = std::min<int64_t>(to_check, prm.iter_limit - iters);
    if (adapt) {
      sc.adapt_iter = static_cast<double>(iters);
      PDHG_CUDA(cudaMemcpyAsync(&scal_.p->adapt_iter, &sc.adapt_iter, sizeof(double), cudaMemcpyHostToDevice, st_));
    }
    RunSteps(par, static_cast<int>(count), adapt);
    par = static_cast<int>((par + count) & 1);
    iters += count;
    inner += count;
    sc.inner_base += static_cast<double>(count);
    PDHG_CUDA(cudaMemcpyAsync(&scal_.p->inner_base, &sc.inner_base, sizeof(double), cudaMemcpyHostToDevice, st_));
    if (iters % prm.check_every != 0) continue;

    // ---- Check (solver.cpp:390-428).
    LaunchCheck(x_[par].p, y_[par].p, xbar_.p, ybar_.p, kx_[par].p);
    if (adapt) PDHG_CUDA(cudaMemcpyAsync(&sc.eta, &scal_.p->eta, sizeof(double), cudaMemcpyDeviceToHost, st_));
    ReadCheck(&ck);
    if (ck.row[2 * kRowPer] > 0.0 || ck.col[2 * kColPer] > 0.0)
      throw Error(PDHG_NUMERICAL_FAILURE, "non-finite iterate at iteration " + std::to_string(iters));
    reports(0, &s_cur, &o_cur);
    reports(1, &s_avg, &o_avg);
    const double kkt_cur = KktError(s_cur.primal_res, s_cur.dual_res, s_cur.gap_abs, sc.omega);
    const double kkt_avg = KktError(s_avg.primal_res, s_avg.dual_res, s_avg.gap_abs, sc.omega);
    const bool take_cur = kkt_cur < kkt_avg;
    const double kkt_cand = take_cur ? kkt_cur : kkt_avg;

    // EvaluateAndMaybeFinish(cur, avg) (solver.cpp:355-387).
    if (Terminated(o_cur, prm.eps)) {
      status = PDHG_OPTIMAL;
      copy_best(0);
      best_rep = o_cur;
      have_best = true;
      break;
    }
    record_best(0, o_cur);
    last_rep = o_cur;
    if (Terminated(o_avg, prm.eps)) {
      status = PDHG_OPTIMAL;
      copy_best(1);
      best_rep = o_avg;
      have_best = true;
      break;
    }
    record_best(1, o_avg);
    if (Kkt1(o_avg) < Kkt1(o_cur)) last_rep = o_avg;

    pdhg_eval_info info{};
    info.iteration = iters;
    info.inner_iteration = inner;
    info.restarts = restarts;
    info.omega = sc.omega;
    info.eta = sc.eta;
    info.kkt_candidate = kkt_cand;
    info.kkt_loop_start = kkt_start;
    info.candidate_is_current = take_cur;
    info.original_report = last_rep;
    info.seconds = secs();

    if (prm.restart_enabled && ShouldRestart(prm, inner, iters, kkt_cand, kkt_start, kkt_prev)) {
      info.restarted = 1;
      // Restart (solver.cpp:430-446).
      const int P = take_cur ? 0 : 1;
      const double dx = std::sqrt(ck.col[P * kColPer + kDx2]);
      const double dy = std::sqrt(ck.row[P * kRowPer + kDy2]);
      sc.omega = UpdatePrimalWeight(sc.omega, dx, dy);
      if (!take_cur) {
        Copy(x_[par].p, xbar_.p, n_);
        Copy(y_[par].p, ybar_.p, m_);
        Copy(kx_[par].p, kxavg_.p, m_);  // ComputeKx(candidate): same pass, same sums
      }
      start_loop(take_cur ? s_cur : s_avg);
      ++restarts;
      push_scalars();
    } else {
      kkt_prev = kkt_cand;
    }

    if (prm.log_every > 0 && (info.iteration - last_log >= prm.log_every || info.iteration == 0)) {
      last_log = info.iteration;
      std::printf("iter=%lld time=%.3f rel_primal=%.3e rel_dual=%.3e rel_gap=%.3e omega=%.3e restarts=%lld\n",
                  (long long)info.iteration, info.seconds, info.original_report.rel_primal,
                  info.original_report.rel_dual, info.original_report.rel_gap, info.omega,
                  (long long)info.restarts);
    }
    if (cb && cb(&info, user) != 0) throw Error(PDHG_ABORTED, "aborted by observer");
  }

  if (!have_best) {  // UseBestSeen (solver.cpp:464-471)
    LaunchCheck(x_[par].p, y_[par].p, x_[par].p, y_[par].p, kx_[par].p);
    ReadCheck(&ck);
    reports(0, &s_cur, &o_cur);
    record_best(0, o_cur);
  }

  // Finish (solver.cpp:473-481): unscale best, lambda on the original problem.
  if (out->x) {
    k_mul<<<ew_grid(n_), kEw, 0, st_>>>(xbest_.p, cs_.p, nvec_.p, n_);
    PDHG_CUDA(cudaMemcpyAsync(out->x, nvec_.p, n_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
    Sync();
  }
  if (out->y) {
    k_mul<<<ew_grid(m_), kEw, 0, st_>>>(ybest_.p, rs_.p, kxavg_.p, m_);
    PDHG_CUDA(cudaMemcpyAsync(out->y, kxavg_.p, m_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
    Sync();
  }
  if (out->lambda) {
    launch_tiles(csc_, OpLambda{ybest_.p, c_o_.p, l_o_.p, u_o_.p, cs_.p, nvec_.p}, nullptr, nullptr, st_);
    PDHG_CUDA(cudaMemcpyAsync(out->lambda, nvec_.p, n_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
  }
  PDHG_CUDA(cudaEventRecord(ev_[1], st_));
  Sync();
  float ms = 0.f;
  PDHG_CUDA(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
  last_ms_ = ms;
  last_launches_ = launches_ + 4;  // + clamp0, kx0 SpMV, unscale/lambda kernels
  out->status = status;
  out->report = best_rep;
  out->iterations = iters;
  out->restarts = restarts;
  out->solve_seconds = secs();
  out->scaling_seconds = scaling_s_;
}

// EstimateOpNorm (solver.cpp:84-110) with the host start vector drawn from the
// same libstdc++ engines as the reference.
double Session::OpNorm(int iters, uint64_t seed) {
  PDHG_CUDA(cudaSetDevice(device_));
  if (nnz_ == 0) return 0.0;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> v(static_cast<size_t>(n_));
  for (double& e : v) e = gauss(rng);
  double acc = 0.0;
  for (double e : v) acc += e * e;
  double vnorm = std::sqrt(acc);
  if (vnorm == 0.0) {
    v[0] = 1.0;
    vnorm = 1.0;
  }
  DArray<double> u, kv;
  u.alloc(n_);
  kv.alloc(m_);
  PDHG_CUDA(cudaMemcpyAsync(u.p, v.data(), n_ * sizeof(double), cudaMemcpyHostToDevice, st_));
  Scalars sc{};
  sc.pw_norm = vnorm;
  PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  launches_ += 4 * static_cast<int64_t>(iters) + 2;
  for (int it = 0; it < iters; ++it) {
    launch_tiles(csr_, OpPowerStep<false>{u.p, scal_.p, 1, kv.p}, nullptr, nullptr, st_);
    launch_tiles(csc_, OpPowerStep<true>{kv.p, scal_.p, 0, u.p}, red_tile_[1].p, red_span_[1].p, st_);
    k_reduce_tiles<<<1, kBlock, 0, st_>>>(red_tile_[1].p, red_span_[1].p, csc_.ntiles, 1, red_out_.p);
    k_power_norm<<<1, 1, 0, st_>>>(red_out_.p, scal_.p);
  }
  launch_tiles(csr_, OpPowerStep<true>{u.p, scal_.p, 1, kv.p}, red_tile_[0].p, red_span_[0].p, st_);
  k_reduce_tiles<<<1, kBlock, 0, st_>>>(red_tile_[0].p, red_span_[0].p, csr_.ntiles, 1, red_out_.p);
  check_launch<int>("power iteration");
  double sum = 0.0;
  Scalars hs{};
  PDHG_CUDA(cudaMemcpyAsync(&sum, red_out_.p, sizeof(double), cudaMemcpyDeviceToHost, st_));
  PDHG_CUDA(cudaMemcpyAsync(&hs, scal_.p, sizeof(Scalars), cudaMemcpyDeviceToHost, st_));
  Sync();
  if (hs.pw_zero) return 0.0;
  return std::sqrt(sum);
}

// ============================================================ kernel probes
void Session::Scaling(double* rs, double* cs) {
  PDHG_CUDA(cudaSetDevice(device_));
  if (m_) PDHG_CUDA(cudaMemcpyAsync(rs, rs_.p, m_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
  if (n_) PDHG_CUDA(cudaMemcpyAsync(cs, cs_.p, n_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
  Sync();
}

void Session::ScaledProblem(double* kv, double* c, double* l, double* u, double* q) {
  PDHG_CUDA(cudaSetDevice(device_));
  auto d2h = [&](double* h, const double* d, int64_t k) {
    if (h && k) PDHG_CUDA(cudaMemcpyAsync(h, d, k * sizeof(double), cudaMemcpyDeviceToHost, st_));
  };
  d2h(kv, csr_val_.p, nnz_);
  d2h(c, c_s_.p, n_);
  d2h(l, l_s_.p, n_);
  d2h(u, u_s_.p, n_);
  d2h(q, q_s_.p, m_);
  Sync();
}

void Session::Spmv(int transpose, const double* in, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  const int64_t nin = transpose ? m_ : n_, nout = transpose ? n_ : m_;
  DArray<double> a, b;
  a.alloc(std::max<int64_t>(nin, 1));
  b.alloc(std::max<int64_t>(nout, 1));
  if (nin) PDHG_CUDA(cudaMemcpyAsync(a.p, in, nin * sizeof(double), cudaMemcpyHostToDevice, st_));
  launch_tiles(transpose ? csc_ : csr_, OpSpmv{a.p, b.p}, nullptr, nullptr, st_);
  check_launch<int>("spmv");
  if (nout) PDHG_CUDA(cudaMemcpyAsync(out, b.p, nout * sizeof(double), cudaMemcpyDeviceToHost, st_));
  Sync();
}

void Session::TimeKernels(int iters, double* ms_primal, double* ms_dual, double* ms_iter) {
  PDHG_CUDA(cudaSetDevice(device_));
  Scalars sc{};
  sc.eta = 1e-3;
  sc.omega = 1.0;
  PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  k_clamp0<<<ew_grid(n_), kEw, 0, st_>>>(l_s_.p, u_s_.p, x_[0].p, n_);
  if (m_) PDHG_CUDA(cudaMemsetAsync(y_[0].p, 0, m_ * sizeof(double), st_));
  launch_tiles(csr_, OpSpmv{x_[0].p, kx_[0].p}, nullptr, nullptr, st_);
  cudaEvent_t e0, e1, e2;
  PDHG_CUDA(cudaEventCreate(&e0));
  PDHG_CUDA(cudaEventCreate(&e1));
  PDHG_CUDA(cudaEventCreate(&e2));
  for (int w = 0; w < 3; ++w) LaunchStep(w & 1, w, false);
  Sync();
  // Each kernel alone, iters launches back to back, on the session stream.
  float t_p = 0, t_d = 0, t_i = 0;
  PDHG_CUDA(cudaEventRecord(e0, st_));
  for (int i = 0; i < iters; ++i)
    launch_tiles(csc_, OpPrimal<false>{y_[0].p, x_[0].p, x_[1].p, xbar_.p, c_s_.p, l_s_.p, u_s_.p, scal_.p, i + 1},
                 nullptr, nullptr, st_);
  PDHG_CUDA(cudaEventRecord(e1, st_));
  for (int i = 0; i < iters; ++i)
    launch_tiles(csr_, OpDual<false>{x_[1].p, y_[0].p, y_[1].p, ybar_.p, kx_[0].p, kx_[1].p, q_s_.p, (int32_t)m1_,
                                     scal_.p, i + 1},
                 nullptr, nullptr, st_);
  PDHG_CUDA(cudaEventRecord(e2, st_));
  PDHG_CUDA(cudaEventSynchronize(e2));
  PDHG_CUDA(cudaEventElapsedTime(&t_p, e0, e1));
  PDHG_CUDA(cudaEventElapsedTime(&t_d, e1, e2));
  // Whole iterations through the block graph.
  const int blk = 64;
  const int reps = std::max(1, iters / blk);
  RunSteps(0, blk, false);
  Sync();
  PDHG_CUDA(cudaEventRecord(e0, st_));
  for (int r = 0; r < reps; ++r) RunSteps(0, blk, false);
  PDHG_CUDA(cudaEventRecord(e1, st_));
  PDHG_CUDA(cudaEventSynchronize(e1));
  PDHG_CUDA(cudaEventElapsedTime(&t_i, e0, e1));
  *ms_primal = t_p / iters;
  *ms_dual = t_d / iters;
  *ms_iter = t_i / (reps * blk);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
}

__global__ void k_reflect(const double* xn, const double* xo, double* ext, int64_t n) {
  GRID_STRIDE(i, n) ext[i] = 2.0 * xn[i] - xo[i];  // solver.cpp:141
}

void Session::UnitPrimal(const double* x, const double* y, double eta, double omega, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  DArray<double> dx, dy, dout;
  dx.alloc(std::max<int64_t>(n_, 1));
  dy.alloc(std::max<int64_t>(m_, 1));
  dout.alloc(std::max<int64_t>(n_, 1));
  if (n_) PDHG_CUDA(cudaMemcpyAsync(dx.p, x, n_ * sizeof(double), cudaMemcpyHostToDevice, st_));
  if (m_) PDHG_CUDA(cudaMemcpyAsync(dy.p, y, m_ * sizeof(double), cudaMemcpyHostToDevice, st_));
  launch_tiles(csc_, OpUnitPrimal{dy.p, dx.p, c_s_.p, l_s_.p, u_s_.p, eta / omega, dout.p}, nullptr, nullptr, st_);
  check_launch<int>("primal step");
  if (n_) PDHG_CUDA(cudaMemcpyAsync(out, dout.p, n_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
  Sync();
}

void Session::UnitDual(const double* xn, const double* xo, const double* y, double eta, double omega, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  DArray<double> a, b, ext, dy, dout;
  a.alloc(std::max<int64_t>(n_, 1));
  b.alloc(std::max<int64_t>(n_, 1));
  ext.alloc(std::max<int64_t>(n_, 1));
  dy.alloc(std::max<int64_t>(m_, 1));
  dout.alloc(std::max<int64_t>(m_, 1));
  if (n_) {
    PDHG_CUDA(cudaMemcpyAsync(a.p, xn, n_ * sizeof(double), cudaMemcpyHostToDevice, st_));
    PDHG_CUDA(cudaMemcpyAsync(b.p, xo, n_ * sizeof(double), cudaMemcpyHostToDevice, st_));
  }
  if (m_) PDHG_CUDA(cudaMemcpyAsync(dy.p, y, m_ * sizeof(double), cudaMemcpyHostToDevice, st_));
  k_reflect<<<ew_grid(n_), kEw, 0, st_>>>(a.p, b.p, ext.p, n_);
  launch_tiles(csr_, OpUnitDual{ext.p, dy.p, q_s_.p, (int32_t)m1_, eta * omega, dout.p}, nullptr, nullptr, st_);
  check_launch<int>("dual step");
  if (m_) PDHG_CUDA(cudaMemcpyAsync(out, dout.p, m_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
  Sync();
}

// Evict the working set between benchmark steps: write 2x the L2 capacity.
void Session::FlushL2() {
  PDHG_CUDA(cudaSetDevice(device_));
  int l2 = 0;
  PDHG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device_));
  const size_t bytes = std::max<size_t>(2 * static_cast<size_t>(l2), 64u << 20);
  if (flush_.n < bytes) flush_.alloc(bytes);
  PDHG_CUDA(cudaMemsetAsync(flush_.p, 0x5a, bytes, st_));
  Sync();
}

void Session::Stats(pdhg_session_stats* s) const {
  s->m1 = m1_;
  s->m2 = m2_;
  s->n = n_;
  s->nnz = nnz_;
  s->csr_tiles = csr_.ntiles;
  s->csc_tiles = csc_.ntiles;
  s->device_bytes = arena_.bytes;
  s->upload_seconds = upload_s_;
  s->scaling_seconds = scaling_s_;
  s->device = device_;
  s->l2_resident = l2_resident_ ? 1 : 0;
}

}  // namespace pdhg
