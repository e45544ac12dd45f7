// B200 restarted-PDHG session: device setup + solve loop orchestration.
//
// Reference map (all under /root/reference/proj/core/src):
//   Solve               solver.cpp:521-543   -> pdhg_solve (abi.cu) = Session + Solve
//   StackK / VStack     lp_problem.cpp:78-83, sparse_matrix.cpp:90-112 -> Session::Upload
//   BuildCscFromCsr     sparse_matrix.cpp:71-88 -> Session::Permute (stable radix sort)
//   ComputeScaling      scaling.cpp:49-91    -> Session::ComputeScaling (device)
//   ApplyScaling        scaling.cpp:93-116   -> Session::ComputeScaling (device)
//   EstimateOpNorm      solver.cpp:84-110    -> Session::OpNorm
//   SolveLoop::Run      solver.cpp:232-267   -> Session::Solve
//   Step                solver.cpp:284-306   -> OpPrimal + OpDual (ops.cuh), CUDA graph per block
//   Check / Restart     solver.cpp:390-446   -> LaunchCheck + host decision logic
//
// Internally rows and columns live in length-class order (engine.cuh); the
// permutation is applied once at upload and undone at the boundary.
#include <optional>

#include "session.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cuda_profiler_api.h>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <random>

#include "host_logic.h"
#include "normal_rng.h"
#include "ops.cuh"
#include "setup_kernels.cuh"
#include "decide.cuh"

namespace pdhg {

namespace {

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(PDHG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class T>
void scan_exclusive(const T* in, T* out, int64_t n, cudaStream_t st) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, st);
  DArray<char> tmp;
  tmp.alloc(tb);
  PDHG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)n, st));
  PDHG_CUDA(cudaStreamSynchronize(st));
}

// seg_of[k] for every nonzero of a compressed layout.
void segment_ids(const int32_t* ptr, int64_t nseg, int64_t nnz, DArray<int32_t>& out, cudaStream_t st) {
  out.alloc(nnz);
  if (!nnz) return;
  PDHG_CUDA(cudaMemsetAsync(out.p, 0, nnz * sizeof(int32_t), st));
  k_seg_marks<<<ew_grid(nseg), kEw, 0, st>>>(ptr, nseg, nnz, out.p);
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, out.p, out.p, (int)nnz, st);
  DArray<char> tmp;
  tmp.alloc(tb);
  PDHG_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, out.p, out.p, (int)nnz, st));
  PDHG_CUDA(cudaStreamSynchronize(st));
}

// Stable sort of segment keys (values < 2^bits) -> permutation new -> old.
// Secondary order inside equal keys (`order`, with the segment offsets `ptr`
// and indices `idx`): kOrderLength -- longest first (a segment with L
// nonzeros is the target of L gathers in the other layout's pass, so hub rows
// / columns pack into few cache lines); kOrderFirst -- by first index in the
// other dimension (k_first_index_key). Ties keep the original order.
// Segment-internal nonzero order is untouched, so every segment sum is
// unchanged whatever the order.
enum SegOrder { kOrderNatural = 0, kOrderLength = 1, kOrderFirst = 2 };

void stable_order(const int32_t* keys, int64_t n, DArray<int32_t>& perm, int bits, cudaStream_t st,
                  SegOrder order = kOrderNatural, const int32_t* ptr = nullptr, const int32_t* idx = nullptr) {
  DArray<int32_t> iota, kout, first, k2;
  iota.alloc(std::max<int64_t>(n, 1));
  kout.alloc(std::max<int64_t>(n, 1));
  k_iota<<<ew_grid(n), kEw, 0, st>>>(iota.p, n);
  const int32_t* vals = iota.p;
  const int32_t* pkeys = keys;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, kout.p, iota.p, perm.p, (int)n, 0, 31, st);
  DArray<char> tmp;
  tmp.alloc(tb);
  if (order != kOrderNatural) {
    first.alloc(std::max<int64_t>(n, 1));
    k2.alloc(std::max<int64_t>(n, 1));
    if (order == kOrderLength) k_len_desc_key<<<ew_grid(n), kEw, 0, st>>>(ptr, n, k2.p);
    else k_first_index_key<<<ew_grid(n), kEw, 0, st>>>(ptr, idx, n, k2.p);
    PDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k2.p, kout.p, iota.p, first.p, (int)n, 0, 31, st));
    k_gather_i32<<<ew_grid(n), kEw, 0, st>>>(keys, first.p, k2.p, n);
    vals = first.p;
    pkeys = k2.p;
  }
  PDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, pkeys, kout.p, vals, perm.p, (int)n, 0, bits, st));
  PDHG_CUDA(cudaStreamSynchronize(st));
}

// Per-segment charge of the block balance (in nonzeros): the ~68 bytes of
// vector traffic per row / column against 12 bytes per nonzero.
constexpr int64_t kSegWeight = 6;

// Default secondary segment orders (stable_order). Rows by first column:
// MCF conservation rows of one node across commodities become neighbours
// (iteration 574 -> 500 us, primal at 95% of HBM); transport, PageRank,
// staircase and random LPs are unchanged (profiles/r01/order_r01z.md).
// Columns by first row split multicommodity arcs apart (MCF dual 311 ->
// 433 us), so they keep their natural order.
constexpr SegOrder kRowOrder = kOrderFirst;
constexpr SegOrder kColOrder = kOrderNatural;

// Mean class-S segment length from which the warp-staged S kernel is used.
constexpr double kStagedMin = 3.0;

// Mean class-S segment length under which the staged kernel steps 128
// entries per warp instead of 256.
constexpr double kChunkSmallMean = 4.0;

// Class S (one thread per segment, storage-order sums -- bit-exact with the
// reference) takes segments up to this length; past 32 they go through the
// warp-staged kernel, whose coalesced chunks beat a warp per 33..64 segment
// (MCF capacity rows of 50: dual 497 -> 337 us).
constexpr int kThreadMax = 64;

// Mean class-L segment length up to which a CTA takes 4 segments.
constexpr double kRpc4Max = 2048.0;

}  // namespace

// Host mirror of the check reductions (26 doubles).
struct CheckOut {
  double row[kRowRed];
  double col[kColRed];
};

// ============================================================== construction
Session::Session(const pdhg_lp& lp, const pdhg_params& prm, int device, const ShardSpec& spec, bool skip_pc)
    : device_(device), skip_pc_(skip_pc) {
  if (spec.world < 1 || spec.world > 64) throw Error(PDHG_INVALID_ARGUMENT, "shard world must lie in [1, 64]");
  if (spec.local != 1 && spec.local != spec.world)
    throw Error(PDHG_INVALID_ARGUMENT, "a session holds either one shard or all of them");
  if (spec.rank < 0 || spec.rank >= spec.world) throw Error(PDHG_INVALID_ARGUMENT, "shard rank out of range");
  world_ = spec.world;
  rank_ = spec.local == spec.world ? 0 : spec.rank;
  const char* tenv = std::getenv("PDHG_TRACE");
  const bool fine = tenv && tenv[0] == '2';  // per-phase construction trace
  double tp = now_s();
  auto phase = [&](const char* what) {
    if (!fine) return;
    Sync();
    const double t = now_s();
    std::fprintf(stderr, "[pdhg]   ctor %-28s %.4fs\n", what, t - tp);
    tp = t;
  };
  PDHG_CUDA(cudaSetDevice(device_));
  PDHG_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  streams_.st = st_;
  fork_.main = st_;
  PDHG_CUDA(cudaEventCreateWithFlags(&fork_.fork, cudaEventDisableTiming));
  streams_.fork.fork = fork_.fork;
  // PDHG_FORK=0: no side streams (class kernels of a pass and the check's
  // row / column passes serialise on the session stream) -- used by the
  // loopback tests, whose spinning rendezvous need a hardware queue per stream.
  const char* fenv = std::getenv("PDHG_FORK");
  const bool fork_on = !(fenv && fenv[0] == '0');
  for (int k = 0; k < 3; ++k) {
    if (fork_on) PDHG_CUDA(cudaStreamCreateWithFlags(&fork_.side[k], cudaStreamNonBlocking));
    PDHG_CUDA(cudaEventCreateWithFlags(&fork_.join[k], cudaEventDisableTiming));
    streams_.fork.side[k] = fork_.side[k];
    streams_.fork.join[k] = fork_.join[k];
  }
  AllocScope scope(st_);  // setup arrays are ordered on the session stream
  host_red_ = static_cast<double*>(pinned_get(kPack * sizeof(double) + 64, &host_red_bytes_));
  phase("streams+events+pinned");
  // NCCL whenever a one-shard-per-process id is given -- also for world = 1,
  // which runs the NCCL code path (collectives, graph capture, rank-0 clock,
  // abort all-reduce) on a single GPU.
  if (spec.local == 1 && (world_ > 1 || spec.nccl_id)) {
    if (!spec.nccl_id) throw Error(PDHG_INVALID_ARGUMENT, "a one-shard-per-process session needs an NCCL id");
    if (is_loopback_id(spec.nccl_id))  // in-process ranks on one device (tests)
      comm_ = std::make_unique<LoopbackComm>(loopback_key(spec.nccl_id), world_, rank_, device_);
    else
      comm_ = std::make_unique<NcclComm>(spec.nccl_id, world_, rank_);
  } else {
    comm_ = std::make_unique<LocalComm>();
  }
  n_ = lp.n;
  if (n_ > 0) start_ = std::thread([this, seed = prm.seed] { DrawStart(seed); });
  shards_ = std::vector<Shard>(spec.local);
  for (int k = 0; k < spec.local; ++k) shards_[k].block = spec.local == 1 ? rank_ : k;
  m1_ = lp.a.rows;
  m2_ = lp.g.rows;
  m_ = m1_ + m2_;
  offset_ = lp.objective_offset;
  try {
    NvtxScope nv("pdhg.session");
    const double t0 = now_s();
    {
      DArray<int32_t> ptr0, idx0;
      DArray<double> val0;
      Upload(lp, ptr0, idx0, val0);
      phase("upload");
      Permute(ptr0, idx0, val0);
      phase("csc+permute");
    }
    phase("free setup temporaries");
    for (Shard& h : shards_) {
      PartitionLong(h.csr, h.csr_st);
      PartitionLong(h.csc, h.csc_st);
    }
    phase("partition");
    // Original-space problem vectors into padded order.
    c_o_.alloc(np_, &arena_);
    l_o_.alloc(np_, &arena_);
    u_o_.alloc(np_, &arena_);
    q_o_.alloc(mp_, &arena_);
    ToInternal(lp.c, pad_c_, c_o_.p, n_, np_);
    ToInternal(lp.l, pad_c_, l_o_.p, n_, np_);
    ToInternal(lp.u, pad_c_, u_o_.p, n_, np_);
    {
      std::vector<double> q(static_cast<size_t>(m_));
      if (m1_) std::memcpy(q.data(), lp.b, m1_ * sizeof(double));
      if (m2_) std::memcpy(q.data() + m1_, lp.h, m2_ * sizeof(double));
      ToInternal(q.data(), pad_r_, q_o_.p, m_, mp_);
    }
    Sync();
    phase("problem vectors");
    upload_s_ = now_s() - t0;
    for (int p = 0; p < 2; ++p) {
      x_[p].alloc(np_, &arena_);
      y_[p].alloc(mp_, &arena_);
      kx_[p].alloc(mp_, &arena_);
    }
    xbar_.alloc(np_, &arena_);
    xstart_.alloc(np_, &arena_);
    xbest_.alloc(np_, &arena_);
    nvec_.alloc(np_, &arena_);
    ybar_.alloc(mp_, &arena_);
    ystart_.alloc(mp_, &arena_);
    ybest_.alloc(mp_, &arena_);
    kxavg_.alloc(mp_, &arena_);
    // Padding entries are never addressed by an index but travel with the
    // all-gathers: keep them zero.
    for (DArray<double>* v : {&x_[0], &x_[1], &xbar_, &xstart_, &xbest_, &nvec_, &y_[0], &y_[1], &ybar_, &ystart_,
                              &ybest_, &kx_[0], &kx_[1], &kxavg_})
      if (v->n) PDHG_CUDA(cudaMemsetAsync(v->p, 0, v->n * sizeof(double), st_));
    scal_.alloc(1, &arena_);
    const int nred = std::max(kRowRed, kColRed);
    for (Shard& h : shards_) {
      h.red[0].alloc(static_cast<size_t>(std::max(h.csr.parts(), 1)) * nred, &arena_);
      h.red[1].alloc(static_cast<size_t>(std::max(h.csc.parts(), 1)) * nred, &arena_);
    }
    red_out_.alloc(static_cast<size_t>(kPack) * shards_.size(), &arena_);
    phase("iterate vectors");
    const double t1 = now_s();
    ComputeScaling(prm);
    Sync();
    scaling_s_ = now_s() - t1;
    phase("scaling");
    DeviceNorms();
    UniformBounds();
    for (Shard& h : shards_) BuildSplit(h.csr, h.csr_st);
    persist_ = PersistOk();
    if (persist_) gbar_.alloc(1, &arena_);
    phase("norms+bounds+split");
    const double iter_bytes = (24.0 * nnz_ + 68.0 * (m_ + n_)) / world_;
    l2_resident_ = iter_bytes < 100e6;
    Sync();
    if (std::getenv("PDHG_TRACE"))
      std::fprintf(stderr, "[pdhg] session %.4fs: upload+csc+permute+partition %.4fs | scaling %.4fs | %.2f GB\n",
                   now_s() - t0, upload_s_, scaling_s_, arena_.bytes / 1e9);
  } catch (...) {
    if (start_.joinable()) start_.join();
    throw;
  }
}

Session::~Session() {
  const double t0 = now_s();
  if (start_.joinable()) start_.join();
  cudaSetDevice(device_);
  cudaStreamSynchronize(st_);
  const char* tenv = std::getenv("PDHG_TRACE");
  if (tenv && tenv[0] == '2') std::fprintf(stderr, "[pdhg]   dtor join+sync %.4fs\n", now_s() - t0);
  for (cudaEvent_t e : ev_)
    if (e) cudaEventDestroy(e);
  for (Graph& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (Graph& g : blocks_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (Graph& g : loops_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (power_graph_) cudaGraphExecDestroy(power_graph_);
  if (power_graph1_) cudaGraphExecDestroy(power_graph1_);
  pinned_put(host_red_, host_red_bytes_);
  pinned_put(hstage_, hstage_bytes_);
  pinned_put(hstate_, hstate_bytes_);
  pinned_put(start_host_, start_host_bytes_);
  for (cudaEvent_t e : pev_)
    if (e) cudaEventDestroy(e);
  comm_.reset();
  // Streams outlive the arrays (streams_ is destroyed last): each array's
  // release synchronises the stream that used it.
  if (tenv && tenv[0] == '2') std::fprintf(stderr, "[pdhg]   dtor body %.4fs\n", now_s() - t0);
}

bool Session::SameScaling(const pdhg_params& prm) const {
  if ((prm.scaling_enabled != 0) != scaled_) return false;
  return !scaled_ || (prm.ruiz_iters == ruiz_iters_ && prm.pc_alpha == pc_alpha_);
}

void Session::Sync() { PDHG_CUDA(cudaStreamSynchronize(st_)); }

void Session::Copy(double* dst, const double* src, size_t n) {
  if (n) PDHG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st_));
}

int Session::parts_csr() const {
  int k = 0;
  for (const Shard& h : shards_) k += h.csr.parts();
  return k;
}
int Session::parts_csc() const {
  int k = 0;
  for (const Shard& h : shards_) k += h.csc.parts();
  return k;
}
int Session::launches_csr() const {
  int k = 0;
  for (const Shard& h : shards_) k += pass_launches(h.csr);
  return k;
}
int Session::launches_csc() const {
  int k = 0;
  for (const Shard& h : shards_) k += pass_launches(h.csc);
  return k;
}

// H2D + int64 -> int32 narrowing + VStack of A and G straight into K's CSR.
void Session::Upload(const pdhg_lp& lp, DArray<int32_t>& ptr0, DArray<int32_t>& idx0, DArray<double>& val0) {
  const int64_t nnz_a = lp.a.rows ? lp.a.row_ptr[lp.a.rows] : 0;
  const int64_t nnz_g = lp.g.rows ? lp.g.row_ptr[lp.g.rows] : 0;
  nnz_ = nnz_a + nnz_g;
  if (nnz_ >= (int64_t(1) << 31) - kTile || m_ >= (int64_t(1) << 31) - 1 || n_ >= (int64_t(1) << 31) - 1)
    throw Error(PDHG_INVALID_ARGUMENT, "problem too large for int32 device indices (nnz, rows, cols < 2^31)");
  ptr0.alloc(m_ + 1);
  idx0.alloc(std::max<int64_t>(nnz_, 1));
  val0.alloc(std::max<int64_t>(nnz_, 1));
  DArray<int64_t> stage;
  stage.alloc(std::max<int64_t>({nnz_a, nnz_g, m1_ + 1, m2_ + 1, 1}) * 2);
  DArray<int> bad;
  bad.alloc(1);
  PDHG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st_));
  int64_t* ap = stage.p;
  int64_t* gp = stage.p + std::max<int64_t>(m1_ + 1, 1);
  // A block with no rows may pass row_ptr == NULL (ValidateLpHost accepts
  // it): its offset array is the single entry 0.
  if (m1_)
    PDHG_CUDA(cudaMemcpyAsync(ap, lp.a.row_ptr, (m1_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
  else
    PDHG_CUDA(cudaMemsetAsync(ap, 0, sizeof(int64_t), st_));
  if (m2_)
    PDHG_CUDA(cudaMemcpyAsync(gp, lp.g.row_ptr, (m2_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
  else
    PDHG_CUDA(cudaMemsetAsync(gp, 0, sizeof(int64_t), st_));
  k_stack_ptr<<<ew_grid(m_ + 1), kEw, 0, st_>>>(ap, gp, m1_, m2_, nnz_a, ptr0.p);
  Sync();
  if (nnz_a) {
    PDHG_CUDA(cudaMemcpyAsync(stage.p, lp.a.col_idx, nnz_a * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    k_narrow<<<ew_grid(nnz_a), kEw, 0, st_>>>(stage.p, idx0.p, nnz_a, n_, bad.p);
    PDHG_CUDA(cudaMemcpyAsync(val0.p, lp.a.values, nnz_a * sizeof(double), cudaMemcpyHostToDevice, st_));
    Sync();
  }
  if (nnz_g) {
    PDHG_CUDA(cudaMemcpyAsync(stage.p, lp.g.col_idx, nnz_g * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    k_narrow<<<ew_grid(nnz_g), kEw, 0, st_>>>(stage.p, idx0.p + nnz_a, nnz_g, n_, bad.p);
    PDHG_CUDA(cudaMemcpyAsync(val0.p + nnz_a, lp.g.values, nnz_g * sizeof(double), cudaMemcpyHostToDevice, st_));
  }
  k_check_ptr<<<ew_grid(m_), kEw, 0, st_>>>(ptr0.p, m_, nnz_, bad.p);
  int hbad = 0;
  PDHG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
  Sync();
  if (hbad & 1) throw Error(PDHG_INVALID_ARGUMENT, "column index out of range");
  if (hbad & 2) throw Error(PDHG_INVALID_ARGUMENT, "row_ptr is not a valid CSR offset array");
  check_launch("upload");
}

// Builds the CSC of K (stable radix sort of (column, CSR position): rows stay
// ascending inside each column, as BuildCscFromCsr guarantees), splits rows
// and columns into balanced blocks, and permutes each block into length
// classes (engine.cuh) for both layouts, keeping every segment's internal
// order. Indices are remapped into the padded vector spaces; each local shard
// receives its row block's CSR and its column block's CSC.
void Session::Permute(const DArray<int32_t>& ptr0, const DArray<int32_t>& idx0, const DArray<double>& val0) {
  // --- original-order CSC
  DArray<int32_t> cptr0, ridx0, row_of;
  DArray<double> cval0;
  cptr0.alloc(n_ + 1);
  ridx0.alloc(std::max<int64_t>(nnz_, 1));
  cval0.alloc(std::max<int64_t>(nnz_, 1));
  segment_ids(ptr0.p, m_, nnz_, row_of, st_);
  if (nnz_ > 0) {
    DArray<int32_t> perm_in, perm_out, keys_out;
    perm_in.alloc(nnz_);
    perm_out.alloc(nnz_);
    keys_out.alloc(nnz_);
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= n_) ++end_bit;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, idx0.p, keys_out.p, perm_in.p, perm_out.p, (int)nnz_, 0, end_bit,
                                    st_);
    DArray<char> tmp;
    tmp.alloc(tb);
    k_iota<<<ew_grid(nnz_), kEw, 0, st_>>>(perm_in.p, nnz_);
    PDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, idx0.p, keys_out.p, perm_in.p, perm_out.p, (int)nnz_, 0,
                                              end_bit, st_));
    k_csc_gather<<<ew_grid(nnz_), kEw, 0, st_>>>(perm_out.p, row_of.p, val0.p, ridx0.p, cval0.p, nnz_);
    k_colptr<<<ew_grid(n_ + 1), kEw, 0, st_>>>(keys_out.p, nnz_, n_, cptr0.p);
    Sync();
  } else {
    PDHG_CUDA(cudaMemsetAsync(cptr0.p, 0, (n_ + 1) * sizeof(int32_t), st_));
  }
  // --- balanced blocks (identical on every rank: same ptr arrays)
  row_begin_.assign(world_ + 1, 0);
  col_begin_.assign(world_ + 1, 0);
  if (world_ == 1) {
    row_begin_[1] = m_;
    col_begin_[1] = n_;
  } else {
    std::vector<int32_t> hp(std::max(m_, n_) + 1);
    PDHG_CUDA(cudaMemcpyAsync(hp.data(), ptr0.p, (m_ + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
    Sync();
    BalancedBlocks(hp.data(), m_, world_, kSegWeight, row_begin_.data());
    PDHG_CUDA(cudaMemcpyAsync(hp.data(), cptr0.p, (n_ + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
    Sync();
    BalancedBlocks(hp.data(), n_, world_, kSegWeight, col_begin_.data());
  }
  pm_ = pn_ = 0;
  gx_ = GhostPlan{};
  gy_ = GhostPlan{};
  for (int b = 0; b < world_; ++b) {
    pm_ = std::max(pm_, row_begin_[b + 1] - row_begin_[b]);
    pn_ = std::max(pn_, col_begin_[b + 1] - col_begin_[b]);
  }
  mp_ = pm_ * world_;
  np_ = pn_ * world_;
  gx_.slice = pn_;
  gy_.slice = pm_;
  if (mp_ >= (int64_t(1) << 31) - 1 || np_ >= (int64_t(1) << 31) - 1)
    throw Error(PDHG_INVALID_ARGUMENT, "padded vectors too large for int32 device indices");
  DArray<int64_t> rbeg, cbeg;
  rbeg.alloc(world_ + 1);
  cbeg.alloc(world_ + 1);
  PDHG_CUDA(cudaMemcpyAsync(rbeg.p, row_begin_.data(), (world_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
  PDHG_CUDA(cudaMemcpyAsync(cbeg.p, col_begin_.data(), (world_ + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st_));

  // --- length classes per block: key = block * 8 + class * 2 + inequality row
  DArray<int32_t> perm_r, perm_c, inv_r, inv_c;  // compact order <-> original
  perm_r.alloc(std::max<int64_t>(m_, 1));
  perm_c.alloc(std::max<int64_t>(n_, 1));
  inv_r.alloc(std::max<int64_t>(m_, 1));
  inv_c.alloc(std::max<int64_t>(n_, 1));
  const int nkeys = 8 * world_;
  std::vector<int> hr(nkeys, 0), hc(nkeys, 0);
  {
    DArray<int32_t> kr, kc, hist;
    kr.alloc(std::max<int64_t>(m_, 1));
    kc.alloc(std::max<int64_t>(n_, 1));
    hist.alloc(2 * nkeys);
    PDHG_CUDA(cudaMemsetAsync(hist.p, 0, 2 * nkeys * sizeof(int32_t), st_));
    // Class bounds: kThreadMax / kWarpMax / kCtaMax unless overridden
    // (PDHG_THREAD_MAX <= 64, PDHG_WARP_MAX, PDHG_CTA_MAX; tuning experiments).
    // Class S sums every segment in storage order (the reference's order);
    // the tile engine does so for segments <= 32.
    auto env_int = [](const char* k, int d) {
      const char* v = std::getenv(k);
      return v ? std::max(0, std::atoi(v)) : d;
    };
    const int thread_max = std::min(512, env_int("PDHG_THREAD_MAX", kThreadMax));
    const int warp_max = std::max(thread_max, env_int("PDHG_WARP_MAX", kWarpMax));
    const int cta_max = std::max(warp_max, env_int("PDHG_CTA_MAX", kCtaMax));
    k_class_keys<<<ew_grid(m_), kEw, 0, st_>>>(ptr0.p, m_, m1_, rbeg.p, world_, thread_max, warp_max, cta_max,
                                               kr.p);
    // Modal column length: when one length in {1,2,3,4,8} covers >= 90% (but
    // not all) of class S, those columns go first and the uniform kernel
    // (implicit offsets, vector loads) runs that prefix (Layout::s_u).
    modal_col_len_ = 0;
    const char* uenv0 = std::getenv("PDHG_UNIFORM_S");
    if (n_ >= kBlock && !(uenv0 && uenv0[0] == '0')) {
      DArray<int> lh;
      lh.alloc(9);
      PDHG_CUDA(cudaMemsetAsync(lh.p, 0, 9 * sizeof(int), st_));
      k_len_hist9<<<ew_grid(n_), kEw, 0, st_>>>(cptr0.p, n_, lh.p);
      DArray<int> cnt;
      cnt.alloc(1);
      PDHG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), st_));
      k_count_le<<<ew_grid(n_), kEw, 0, st_>>>(cptr0.p, n_, thread_max, cnt.p);
      int h9[9], ns = 0;
      PDHG_CUDA(cudaMemcpyAsync(h9, lh.p, sizeof(h9), cudaMemcpyDeviceToHost, st_));
      PDHG_CUDA(cudaMemcpyAsync(&ns, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
      Sync();
      int best = 0;
      for (int L : {1, 2, 3, 4, 8})
        if (L <= thread_max && h9[L] > (best ? h9[best] : 0)) best = L;
      if (best && h9[best] < ns && h9[best] >= kBlock && 10.0 * h9[best] >= 9.0 * ns) modal_col_len_ = best;
    }
    k_class_keys<<<ew_grid(n_), kEw, 0, st_>>>(cptr0.p, n_, n_, cbeg.p, world_, thread_max, warp_max, cta_max,
                                               kc.p, modal_col_len_);
    k_key_hist<<<ew_grid(m_), kEw, 0, st_>>>(kr.p, m_, hist.p, nkeys);
    k_key_hist<<<ew_grid(n_), kEw, 0, st_>>>(kc.p, n_, hist.p + nkeys, nkeys);
    int bits = 3;
    while ((1 << bits) < nkeys) ++bits;
    // Secondary segment order (tuning: PDHG_ROW_ORDER / PDHG_COL_ORDER =
    // natural | length | first; PDHG_DEGREE_ORDER=1 = length for both).
    auto seg_order = [](const char* var, SegOrder def) {
      const char* d = std::getenv("PDHG_DEGREE_ORDER");
      if (d && d[0] == '1') return kOrderLength;
      const char* v = std::getenv(var);
      if (!v) return def;
      const std::string s(v);
      return s == "length" ? kOrderLength : (s == "first" ? kOrderFirst : kOrderNatural);
    };
    const SegOrder ro = seg_order("PDHG_ROW_ORDER", kRowOrder), co = seg_order("PDHG_COL_ORDER", kColOrder);
    if (m_) stable_order(kr.p, m_, perm_r, bits, st_, ro, ptr0.p, idx0.p);
    if (n_) stable_order(kc.p, n_, perm_c, bits, st_, co, cptr0.p, ridx0.p);
    std::vector<int> h(2 * nkeys);
    PDHG_CUDA(cudaMemcpyAsync(h.data(), hist.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st_));
    Sync();
    std::copy(h.begin(), h.begin() + nkeys, hr.begin());
    std::copy(h.begin() + nkeys, h.end(), hc.begin());
  }
  k_invert<<<ew_grid(m_), kEw, 0, st_>>>(perm_r.p, inv_r.p, m_);
  k_invert<<<ew_grid(n_), kEw, 0, st_>>>(perm_c.p, inv_c.p, n_);
  pad_r_.alloc(std::max<int64_t>(m_, 1), &arena_);
  pad_c_.alloc(std::max<int64_t>(n_, 1), &arena_);
  k_pad_index<<<ew_grid(m_), kEw, 0, st_>>>(inv_r.p, rbeg.p, world_, pm_, pad_r_.p, m_);
  k_pad_index<<<ew_grid(n_), kEw, 0, st_>>>(inv_c.p, cbeg.p, world_, pn_, pad_c_.p, n_);

  // --- full compact layouts (every block, class order), indices padded
  auto build = [&](DArray<int32_t>& ptr, DArray<int32_t>& idx, DArray<double>& val, const DArray<int32_t>& p0,
                   const DArray<int32_t>& i0, const DArray<double>& v0, const DArray<int32_t>& seg_of, int64_t nseg,
                   const DArray<int32_t>& perm, const DArray<int32_t>& inv_seg, const DArray<int32_t>& pad_other) {
    ptr.alloc(nseg + 1);
    idx.alloc(std::max<int64_t>(nnz_, 1));
    val.alloc(std::max<int64_t>(nnz_, 1));
    DArray<int32_t> len;
    len.alloc(nseg + 1);
    PDHG_CUDA(cudaMemsetAsync(len.p, 0, (nseg + 1) * sizeof(int32_t), st_));
    k_perm_len<<<ew_grid(nseg), kEw, 0, st_>>>(p0.p, perm.p, nseg, len.p);
    scan_exclusive(len.p, ptr.p, nseg + 1, st_);
    if (nnz_)
      k_perm_nnz<<<ew_grid(nnz_), kEw, 0, st_>>>(p0.p, seg_of.p, i0.p, v0.p, inv_seg.p, pad_other.p, ptr.p, idx.p,
                                                  val.p, nnz_);
  };
  const char* uenv = std::getenv("PDHG_UNIFORM_S");
  const bool uniform_s = !(uenv && uenv[0] == '0');
  const char* rmax = std::getenv("PDHG_RPC4_MAX");
  const double rpc4_max = rmax ? std::atof(rmax) : kRpc4Max;
  const char* smin = std::getenv("PDHG_STAGED_MIN");
  const double staged_min = smin ? std::atof(smin) : kStagedMin;
  // One layout's block slice -> shard storage (ownership moves when the
  // session holds the whole matrix in one shard).
  auto slice = [&](Layout& L, Store& S, DArray<int32_t>& ptr, DArray<int32_t>& idx, DArray<double>& val, int64_t b0,
                   int64_t b1, const int* hist, int modal) {
    const int64_t nseg = b1 - b0;
    int32_t k0 = 0, k1 = 0;
    PDHG_CUDA(cudaMemcpyAsync(&k0, ptr.p + b0, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
    PDHG_CUDA(cudaMemcpyAsync(&k1, ptr.p + b1, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
    Sync();
    if (world_ == 1) {
      S.ptr.take(ptr, &arena_);
      S.idx.take(idx, &arena_);
      S.val.take(val, &arena_);
    } else {
      S.ptr.alloc(nseg + 1, &arena_);
      S.idx.alloc(std::max<int32_t>(k1 - k0, 1), &arena_);
      S.val.alloc(std::max<int32_t>(k1 - k0, 1), &arena_);
      k_rebase<<<ew_grid(nseg + 1), kEw, 0, st_>>>(ptr.p + b0, nseg, S.ptr.p);
      if (k1 > k0) {
        PDHG_CUDA(cudaMemcpyAsync(S.idx.p, idx.p + k0, (k1 - k0) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st_));
        PDHG_CUDA(cudaMemcpyAsync(S.val.p, val.p + k0, (k1 - k0) * sizeof(double), cudaMemcpyDeviceToDevice, st_));
      }
    }
    L.nseg = static_cast<int32_t>(nseg);
    L.nnz = k1 - k0;
    L.ptr = S.ptr.p;
    L.idx = S.idx.p;
    L.val = S.val.p;
    L.s1 = hist[0] + hist[1];
    L.s2 = L.s1 + hist[2] + hist[3];
    L.s3 = L.s2 + hist[4] + hist[5];
    // Class S kernel variant from the class's mean length (setup-time D2H
    // of one offset): warp-staged once segments average >= kStagedMin.
    int32_t se = 0;
    if (L.s1 > 0) {
      PDHG_CUDA(cudaMemcpyAsync(&se, L.ptr + L.s1, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
      Sync();
    }
    L.s_staged = L.s1 > 0 && static_cast<double>(se) >= staged_min * L.s1;
    const char* sp = std::getenv("PDHG_S_PIPE");  // "1": cp.async-pipelined variant (A/B, bit-identical; slower)
    L.s_pipe = L.s_staged && sp && sp[0] == '1';
    // PDHG_S_FLOW=3|4: persistent staged kernel for the step passes (3 or 4
    // CTAs per SM; 0 = off).
    // Staged chunk: 128 entries per warp step when the class's segments
    // average under kChunkSmallMean nonzeros (a 32-segment group then rarely
    // fills more: half the registers, every gather of a chunk in flight),
    // else 256. PDHG_S_CHUNK=128|256 overrides.
    const char* sc = std::getenv("PDHG_S_CHUNK");
    L.s_chunk = sc ? (std::atoi(sc) == 128 ? 128 : 256)
                   : (L.s1 > 0 && static_cast<double>(se) < kChunkSmallMean * L.s1 ? 128 : 256);
    const char* sf = std::getenv("PDHG_S_FLOW");
    L.s_flow = (L.s_staged && !L.s_pipe && sf && (sf[0] == '3' || sf[0] == '4')) ? sf[0] - '0' : 0;
    // Segment-order warps of the staged kernel (shifted-copy segment groups).
    L.s_rm = nullptr;
    const char* rmo = std::getenv("PDHG_SEG_ORDER_WARPS");  // "0": off (A/B)
    if (L.s_staged && !(rmo && rmo[0] == '0')) {
      const int64_t ng = (static_cast<int64_t>(L.s1) + 31) / 32;
      S.rm.alloc(ng, &arena_);
      DArray<int> any;
      any.alloc(1);
      PDHG_CUDA(cudaMemsetAsync(any.p, 0, sizeof(int), st_));
      k_rowmajor_flags<<<ew_grid(ng), kEw, 0, st_>>>(L.ptr, L.idx, L.s1, S.rm.p, any.p);
      int hany = 0;
      PDHG_CUDA(cudaMemcpyAsync(&hany, any.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
      Sync();
      if (hany) L.s_rm = S.rm.p;
      else S.rm.release();
    }
    // Class S of one common length (and starting at nonzero 0): offsets implicit.
    L.s_len = 0;
    L.s_u = 0;
    if (L.s1 > 0 && uniform_s) {
      DArray<int> mm;
      mm.alloc(2);
      const int init[2] = {INT32_MAX, 0};
      PDHG_CUDA(cudaMemcpyAsync(mm.p, init, sizeof(init), cudaMemcpyHostToDevice, st_));
      k_len_minmax<<<ew_grid(L.s1), kEw, 0, st_>>>(L.ptr, L.s1, mm.p);
      int h[2];
      int32_t p0 = 1;
      PDHG_CUDA(cudaMemcpyAsync(h, mm.p, sizeof(h), cudaMemcpyDeviceToHost, st_));
      PDHG_CUDA(cudaMemcpyAsync(&p0, L.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
      Sync();
      if (p0 == 0 && h[0] == h[1] && (h[0] == 1 || h[0] == 2 || h[0] == 3 || h[0] == 4 || h[0] == 8)) {
        L.s_len = h[0];
        L.s_u = L.s1;
      } else if (p0 == 0 && modal > 0 && hist[0] >= kBlock) {  // modal prefix (columns)
        L.s_len = modal;
        L.s_u = hist[0] / kBlock * kBlock;
      }
    }
    // Class L: 4 segments per CTA when they average <= kRpc4Max nonzeros and
    // most neighbours start gathering in the same sector (shared L1 lines).
    L.l_rpc = 1;
    if (L.s3 > L.s2) {
      int32_t lb = 0, le = 0;
      PDHG_CUDA(cudaMemcpyAsync(&lb, L.ptr + L.s2, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
      PDHG_CUDA(cudaMemcpyAsync(&le, L.ptr + L.s3, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
      Sync();
      int adj = 0;
      if (L.s3 - L.s2 > 1 && static_cast<double>(le - lb) <= rpc4_max * (L.s3 - L.s2)) {
        DArray<int> cnt;
        cnt.alloc(1);
        PDHG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), st_));
        k_adjacent_count<<<ew_grid(L.s3 - L.s2), kEw, 0, st_>>>(L.ptr, L.idx, L.s2, L.s3, cnt.p);
        PDHG_CUDA(cudaMemcpyAsync(&adj, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
        Sync();
      }
      if (4 * adj >= L.s3 - L.s2 - 1 && adj > 0) L.l_rpc = 4;  // >= 25% adjacent pairs
    }
    // RPC 4: stage each CTA's stream in shared memory when every group fits.
    L.l_stage = 0;
    const char* ts = std::getenv("PDHG_CTA_STAGE");
    if (L.l_rpc == 4 && !(ts && ts[0] == '0')) {
      DArray<int> mx;
      mx.alloc(1);
      PDHG_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), st_));
      k_group_max<<<ew_grid((L.s3 - L.s2 + 3) / 4), kEw, 0, st_>>>(L.ptr, L.s2, L.s3, 4, mx.p);
      int gmax = 0;
      PDHG_CUDA(cudaMemcpyAsync(&gmax, mx.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
      Sync();
      const int64_t bytes = 12 * static_cast<int64_t>(gmax) + 64;  // + 16-byte widening of both ranges
      if (bytes <= kCtaStageMax) L.l_stage = static_cast<int>(bytes);
    }
  };
  {
    DArray<int32_t> fptr, fidx;
    DArray<double> fval;
    build(fptr, fidx, fval, ptr0, idx0, val0, row_of, m_, perm_r, inv_r, pad_c_);
    if (world_ > 1) BuildGhostPlan(fptr.p, fidx.p, row_begin_, np_, pn_, gx_, gxs_, ghost_counts_x_);
    for (Shard& h : shards_) {
      const int b = h.block;
      const int* hb = hr.data() + 8 * b;
      h.roff = b * pm_;
      h.rows = row_begin_[b + 1] - row_begin_[b];
      slice(h.csr, h.csr_st, fptr, fidx, fval, row_begin_[b], row_begin_[b + 1], hb, 0);
      h.csr.nvec = static_cast<int32_t>(np_);
      h.rk.e0 = hb[0];
      h.rk.s1 = hb[0] + hb[1];
      h.rk.e1 = h.rk.s1 + hb[2];
      h.rk.s2 = h.rk.s1 + hb[2] + hb[3];
      h.rk.e2 = h.rk.s2 + hb[4];
      h.rk.s3 = h.rk.s2 + hb[4] + hb[5];
      h.rk.e3 = h.rk.s3 + hb[6];
    }
    Sync();
  }
  {
    DArray<int32_t> col_of, fptr, fidx;
    DArray<double> fval;
    segment_ids(cptr0.p, n_, nnz_, col_of, st_);
    build(fptr, fidx, fval, cptr0, ridx0, cval0, col_of, n_, perm_c, inv_c, pad_r_);
    if (world_ > 1) BuildGhostPlan(fptr.p, fidx.p, col_begin_, mp_, pm_, gy_, gys_, ghost_counts_y_);
    for (Shard& h : shards_) {
      const int b = h.block;
      h.coff = b * pn_;
      h.cols = col_begin_[b + 1] - col_begin_[b];
      slice(h.csc, h.csc_st, fptr, fidx, fval, col_begin_[b], col_begin_[b + 1], hc.data() + 8 * b, modal_col_len_);
      h.csc.nvec = static_cast<int32_t>(mp_);
    }
    Sync();
  }
  ptr0_.alloc(m_ + 1, &arena_);
  PDHG_CUDA(cudaMemcpyAsync(ptr0_.p, ptr0.p, (m_ + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st_));
  Sync();
  check_launch("permute");
}

// Ghost plan of one gather pattern, from the full compact layout (every
// block's segments, indices already padded) that every rank builds: for each
// reader block r, the distinct padded indices its segments read outside its
// own slice (sorted, hence grouped by source block). This rank receives its
// own list and sends, to each peer r, the part of r's list inside its slice.
// All ranks see the same counts, so they agree on ghost vs all-gather: ghosts
// when the largest per-rank ghost volume is at most half an all-gather.
void Session::BuildGhostPlan(const int32_t* ptr, const int32_t* idx, const std::vector<int64_t>& seg_begin,
                             int64_t nvec, int64_t slice, GhostPlan& plan, GhostStore& store,
                             std::vector<int64_t>& counts) {
  const int P = world_;
  counts.assign(static_cast<size_t>(P) * P, 0);
  DArray<uint8_t> mark;
  DArray<int32_t> list, nsel, bcount;
  mark.alloc(std::max<int64_t>(nvec, 1));
  list.alloc(std::max<int64_t>(nvec, 1));
  nsel.alloc(1);
  bcount.alloc(P);
  std::vector<int32_t> hptr(static_cast<size_t>(P) + 1);
  for (int r = 0; r <= P; ++r) {
    PDHG_CUDA(cudaMemcpyAsync(&hptr[r], ptr + seg_begin[r], sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
  }
  Sync();
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, static_cast<const int32_t*>(nullptr), static_cast<const uint8_t*>(nullptr),
                             list.p, nsel.p, static_cast<int>(nvec), st_);
  DArray<char> tmp;
  DArray<int32_t> iota;
  tmp.alloc(std::max<size_t>(tb, 1));
  iota.alloc(std::max<int64_t>(nvec, 1));
  k_iota<<<ew_grid(nvec), kEw, 0, st_>>>(iota.p, nvec);
  std::vector<int32_t> send_host;  // this rank's send lists, peer by peer
  std::vector<int64_t> send_off(P + 1, 0), recv_off(P + 1, 0);
  for (int r = 0; r < P; ++r) {
    PDHG_CUDA(cudaMemsetAsync(mark.p, 0, nvec, st_));
    const int64_t k0 = hptr[r], k1 = hptr[r + 1];
    if (k1 > k0) k_mark<<<ew_grid(k1 - k0), kEw, 0, st_>>>(idx + k0, k1 - k0, mark.p);
    PDHG_CUDA(cudaMemsetAsync(mark.p + r * slice, 0, slice, st_));  // own slice: local
    PDHG_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, iota.p, mark.p, list.p, nsel.p, static_cast<int>(nvec), st_));
    PDHG_CUDA(cudaMemsetAsync(bcount.p, 0, P * sizeof(int32_t), st_));
    int nl = 0;
    PDHG_CUDA(cudaMemcpyAsync(&nl, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
    Sync();
    if (nl) k_block_count<<<ew_grid(nl), kEw, 0, st_>>>(list.p, nl, slice, bcount.p);
    std::vector<int32_t> bc(P);
    PDHG_CUDA(cudaMemcpyAsync(bc.data(), bcount.p, P * sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
    Sync();
    int64_t before = 0;
    for (int b = 0; b < P; ++b) {
      counts[static_cast<size_t>(r) * P + b] = bc[b];
      if (b < rank_) before += bc[b];
    }
    if (r == rank_) {  // receive list: where the ghosts land
      for (int b = 0; b < P; ++b) recv_off[b + 1] = recv_off[b] + bc[b];
      store.recv_idx.alloc(std::max(nl, 1), &arena_);
      if (nl) PDHG_CUDA(cudaMemcpyAsync(store.recv_idx.p, list.p, nl * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                        st_));
    } else {  // what r reads from this rank's slice
      const int64_t c = bc[rank_];
      std::vector<int32_t> part(static_cast<size_t>(c));
      if (c) PDHG_CUDA(cudaMemcpyAsync(part.data(), list.p + before, c * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                       st_));
      Sync();
      send_host.insert(send_host.end(), part.begin(), part.end());
    }
    send_off[r + 1] = static_cast<int64_t>(send_host.size());
  }
  int64_t worst = 0;
  for (int r = 0; r < P; ++r) {
    int64_t g = 0;
    for (int b = 0; b < P; ++b)
      if (b != r) g += counts[static_cast<size_t>(r) * P + b];
    worst = std::max(worst, g);
  }
  const char* genv = std::getenv("PDHG_GHOST");
  const bool allow = !(genv && genv[0] == '0');
  plan.use = allow && !comm_->local() && 2 * worst <= static_cast<int64_t>(P - 1) * slice;
  plan.slice = slice;
  plan.send_off = send_off;
  plan.recv_off = recv_off;
  if (plan.use) {
    const int64_t ns = send_off[P], nr = recv_off[P];
    store.send_idx.alloc(std::max<int64_t>(ns, 1), &arena_);
    if (ns) PDHG_CUDA(cudaMemcpyAsync(store.send_idx.p, send_host.data(), ns * sizeof(int32_t),
                                      cudaMemcpyHostToDevice, st_));
    store.send_buf.alloc(std::max<int64_t>(ns, 1), &arena_);
    store.recv_buf.alloc(std::max<int64_t>(nr, 1), &arena_);
    plan.send_idx = store.send_idx.p;
    plan.recv_idx = store.recv_idx.p;
    plan.send_buf = store.send_buf.p;
    plan.recv_buf = store.recv_buf.p;
    Sync();
  } else {
    store.recv_idx.release();
  }
  check_launch("ghost plan");
}

void Session::GhostCounts(int64_t* x_counts, int64_t* y_counts, int32_t* use) const {
  std::copy(ghost_counts_x_.begin(), ghost_counts_x_.end(), x_counts);
  std::copy(ghost_counts_y_.begin(), ghost_counts_y_.end(), y_counts);
  use[0] = gx_.use;
  use[1] = gy_.use;
}

// Gather-window split of class S (Layout::split_w; PDHG_S_SPLIT=1 on, 0 off,
// default: off). Built from the SCALED values, for one-shard sessions whose
// staged class S gathers from a vector larger than the ~64 MB that random
// gathers keep L2-resident (tools/gather_probe.cu: 190 G gathers/s up to
// 59 MB, 140 G/s at 84 MB). Skipped when any segment's entries would be
// reordered by the split.
void Session::BuildSplit(Layout& L, Store& S) {
  L.split_w = 0;
  const char* e = std::getenv("PDHG_S_SPLIT");
  const bool on = e && e[0] == '1';
  const char* mb = std::getenv("PDHG_S_SPLIT_MIN_MB");  // vector-size threshold (tests: 0)
  const int64_t min_bytes = (mb ? std::atoll(mb) : 64) << 20;
  if (!on || world_ != 1 || !L.s_staged || L.s1 < kBlock || static_cast<int64_t>(L.nvec) * 8 <= min_bytes) return;
  const int32_t w = (L.nvec / 2 + 31) / 32 * 32;
  DArray<int32_t> cnt;
  DArray<int> bad;
  cnt.alloc(L.s1 + 1);
  bad.alloc(1);
  PDHG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st_));
  PDHG_CUDA(cudaMemsetAsync(cnt.p + L.s1, 0, sizeof(int32_t), st_));
  k_split_count<<<ew_grid(L.s1), kEw, 0, st_>>>(L.ptr, L.idx, L.s1, w, cnt.p, bad.p);
  int hbad = 0;
  PDHG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
  Sync();
  if (hbad) return;
  S.lo_ptr.alloc(L.s1 + 1, &arena_);
  S.hi_ptr.alloc(L.s1 + 1, &arena_);
  scan_exclusive(cnt.p, S.lo_ptr.p, L.s1 + 1, st_);
  int32_t nlo = 0, ns = 0;
  PDHG_CUDA(cudaMemcpyAsync(&nlo, S.lo_ptr.p + L.s1, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
  PDHG_CUDA(cudaMemcpyAsync(&ns, L.ptr + L.s1, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
  Sync();
  S.lo_idx.alloc(std::max(nlo, 1), &arena_);
  S.lo_val.alloc(std::max(nlo, 1), &arena_);
  S.hi_idx.alloc(std::max(ns - nlo, 1), &arena_);
  S.hi_val.alloc(std::max(ns - nlo, 1), &arena_);
  S.split_part.alloc(L.s1, &arena_);
  k_split_copy<<<ew_grid(L.s1 + 1), kEw, 0, st_>>>(L.ptr, L.idx, L.val, L.s1, S.lo_ptr.p, S.lo_idx.p, S.lo_val.p,
                                                   S.hi_ptr.p, S.hi_idx.p, S.hi_val.p);
  auto half = [&](Layout::Half& hf, DArray<int32_t>& ptr, DArray<int32_t>& idx, DArray<double>& val,
                  DArray<uint8_t>& rm, int64_t nnz) {
    hf.ptr = ptr.p;
    hf.idx = idx.p;
    hf.val = val.p;
    hf.chunk = static_cast<double>(nnz) < kChunkSmallMean * L.s1 ? 128 : 256;
    hf.rm = nullptr;
    if (L.s_rm) {  // segment-order warps, judged on this half's entries
      const int64_t ng = (static_cast<int64_t>(L.s1) + 31) / 32;
      rm.alloc(ng, &arena_);
      DArray<int> any;
      any.alloc(1);
      PDHG_CUDA(cudaMemsetAsync(any.p, 0, sizeof(int), st_));
      k_rowmajor_flags<<<ew_grid(ng), kEw, 0, st_>>>(ptr.p, idx.p, L.s1, rm.p, any.p);
      int hany = 0;
      PDHG_CUDA(cudaMemcpyAsync(&hany, any.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
      Sync();
      if (hany) hf.rm = rm.p;
    }
  };
  half(L.lo, S.lo_ptr, S.lo_idx, S.lo_val, S.lo_rm, nlo);
  half(L.hi, S.hi_ptr, S.hi_idx, S.hi_val, S.hi_rm, ns - nlo);
  L.part = S.split_part.p;
  L.split_w = w;
  Sync();
  check_launch("class-S split");
}

// Tile partition of the extra-long class [s3, nseg) of one layout (tile_spmv.cuh):
// sorted unique boundary candidates, owned-segment ranges, cross-tile links.
void Session::PartitionLong(Layout& L, Store& S) {
  CMat& M = L.lng;
  M.nseg = L.nseg;
  M.nvec = L.nvec;
  M.nnz = L.nnz;
  M.ptr = L.ptr;
  M.idx = L.idx;
  M.val = L.val;
  M.ntiles = 0;
  if (L.nseg <= L.s3) return;
  const int32_t lo = L.s3, hi = L.nseg;
  int32_t nz0 = 0;
  PDHG_CUDA(cudaMemcpyAsync(&nz0, L.ptr + lo, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
  Sync();
  const int64_t nz1 = L.nnz;
  const int ngroups = ceil_div(hi - lo, kBlock);
  const int ncuts = std::max(0, ceil_div(nz1 - nz0, kTile) - 1);
  const int nc = ngroups + ncuts;
  DArray<int32_t> cand, sorted, uniq, nsel;
  cand.alloc(nc);
  sorted.alloc(nc);
  uniq.alloc(nc + 1);
  nsel.alloc(1);
  k_part_cand<<<ew_grid(nc), kEw, 0, st_>>>(L.ptr, lo, hi, nz0, nz1, ngroups, ncuts, cand.p);
  size_t t1 = 0, t2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t1, cand.p, sorted.p, nc, 0, 32, st_);
  cub::DeviceSelect::Unique(nullptr, t2, sorted.p, uniq.p, nsel.p, nc, st_);
  DArray<char> tmp;
  tmp.alloc(std::max(t1, t2));
  PDHG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t1, cand.p, sorted.p, nc, 0, 32, st_));
  PDHG_CUDA(cub::DeviceSelect::Unique(tmp.p, t2, sorted.p, uniq.p, nsel.p, nc, st_));
  int nu = 0, last = 0;
  PDHG_CUDA(cudaMemcpyAsync(&nu, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st_));
  Sync();
  PDHG_CUDA(cudaMemcpyAsync(&last, uniq.p + nu - 1, sizeof(int), cudaMemcpyDeviceToHost, st_));
  Sync();
  const int ntiles = (last == INT32_MAX) ? nu - 1 : nu;
  M.ntiles = ntiles;
  for (int k = 0; k < 4; ++k) S.part[k].alloc(ntiles + 1, &arena_);
  S.head.alloc(2 * (size_t)ntiles, &arena_);
  S.tail.alloc(2 * (size_t)ntiles, &arena_);
  S.cnt.alloc(ntiles, &arena_);
  PDHG_CUDA(cudaMemsetAsync(S.cnt.p, 0, ntiles * sizeof(unsigned), st_));
  M.tile_begin = S.part[0].p;
  M.tile_seg = S.part[1].p;
  M.head_first = S.part[2].p;
  M.tail_owner = S.part[3].p;
  M.head_part = S.head.p;
  M.tail_part = S.tail.p;
  M.counter = S.cnt.p;
  const int32_t end = static_cast<int32_t>(nz1);
  PDHG_CUDA(cudaMemcpyAsync(M.tile_begin, uniq.p, ntiles * sizeof(int32_t), cudaMemcpyDeviceToDevice, st_));
  PDHG_CUDA(cudaMemcpyAsync(M.tile_begin + ntiles, &end, sizeof(int32_t), cudaMemcpyHostToDevice, st_));
  const int g = ew_grid(ntiles + 1);
  k_part_seg<<<g, kEw, 0, st_>>>(L.ptr, lo, hi, nz1, ntiles, M.tile_begin, M.tile_seg);
  k_part_span<<<g, kEw, 0, st_>>>(L.ptr, hi, nz1, ntiles, M.tile_begin, M.tile_seg, M.head_first, M.tail_owner);
  // Gather sweep (PDHG_TILE_SWEEP=0: off): tiles execute in the order of
  // their first gathered index, stable (CMat::order).
  const char* sw = std::getenv("PDHG_TILE_SWEEP");
  if (ntiles > 1 && !(sw && sw[0] == '0')) {
    DArray<int32_t> key, key2, iota;
    key.alloc(ntiles);
    key2.alloc(ntiles);
    iota.alloc(ntiles);
    S.order.alloc(ntiles, &arena_);
    k_tile_first_index<<<ew_grid(ntiles), kEw, 0, st_>>>(M.tile_begin, L.idx, ntiles, key.p);
    k_iota<<<ew_grid(ntiles), kEw, 0, st_>>>(iota.p, ntiles);
    const int bits = 31;  // padded (sharded) indices can exceed nvec
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, iota.p, S.order.p, ntiles, 0, bits, st_);
    DArray<char> tmp2;
    tmp2.alloc(tb);
    PDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp2.p, tb, key.p, key2.p, iota.p, S.order.p, ntiles, 0, bits, st_));
    M.order = S.order.p;
  }
  Sync();
  check_launch("partition");
}

// Ruiz x10 + Pock-Chambolle on device (scaling.cpp:49-91), then
// ApplyScaling (scaling.cpp:93-116): K_s = (rs * K) * cs from the ORIGINAL
// values with the composed scales, c_s = c cs, l_s = l / cs, u_s = u / cs,
// q_s = q rs. Max is exact and 1/sqrt is IEEE on both sides, so the scales
// are bit-identical to the reference (power sums too for rows/cols of <= 32
// nonzeros, which are summed in storage order) -- for any shard count: each
// shard owns whole rows (CSR) and whole columns (CSC), and the per-sweep
// factors are all-gathered before the values are rescaled.
void Session::ComputeScaling(const pdhg_params& prm) {
  NvtxScope nv("pdhg.scaling");
  rs_.alloc(mp_, &arena_);
  cs_.alloc(np_, &arena_);
  c_s_.alloc(np_, &arena_);
  l_s_.alloc(np_, &arena_);
  u_s_.alloc(np_, &arena_);
  q_s_.alloc(mp_, &arena_);
  k_fill<<<ew_grid(mp_), kEw, 0, st_>>>(rs_.p, 1.0, mp_);
  k_fill<<<ew_grid(np_), kEw, 0, st_>>>(cs_.p, 1.0, np_);
  scaled_ = prm.scaling_enabled != 0;
  ruiz_iters_ = prm.ruiz_iters;
  pc_alpha_ = prm.pc_alpha;
  if (scaled_ && (prm.pc_alpha < 0.0 || prm.pc_alpha > 2.0))
    throw Error(PDHG_INVALID_ARGUMENT, "pock-chambolle alpha must lie in [0, 2]");
  if (scaled_ && nnz_ > 0) {
    const size_t ns = shards_.size();
    std::vector<DArray<int32_t>> row_of(ns), col_of(ns);
    std::vector<DArray<double>> orig_r(ns), orig_c(ns);
    DArray<double> dr, dc;
    dr.alloc(mp_);
    dc.alloc(np_);
    PDHG_CUDA(cudaMemsetAsync(dr.p, 0, mp_ * sizeof(double), st_));
    PDHG_CUDA(cudaMemsetAsync(dc.p, 0, np_ * sizeof(double), st_));
    for (size_t k = 0; k < ns; ++k) {
      const Shard& h = shards_[k];
      segment_ids(h.csr.ptr, h.csr.nseg, h.csr.nnz, row_of[k], st_);
      segment_ids(h.csc.ptr, h.csc.nseg, h.csc.nnz, col_of[k], st_);
      orig_r[k].alloc(std::max<int64_t>(h.csr.nnz, 1));
      orig_c[k].alloc(std::max<int64_t>(h.csc.nnz, 1));
      Copy(orig_r[k].p, h.csr.val, h.csr.nnz);
      Copy(orig_c[k].p, h.csc.val, h.csc.nnz);
    }
    // Rescale every local layout: src values -> dst = (r * v) * c.
    auto rescale = [&](bool from_orig, const double* r, const double* c) {
      for (size_t k = 0; k < ns; ++k) {
        Shard& h = shards_[k];
        if (h.csr.nnz)
          k_scale_vals<<<ew_grid(h.csr.nnz), kEw, 0, st_>>>(row_of[k].p, h.csr.idx,
                                                           from_orig ? orig_r[k].p : h.csr.val, h.csr.val, r, c,
                                                           h.csr.nnz, 1, h.roff);
        if (h.csc.nnz)
          k_scale_vals<<<ew_grid(h.csc.nnz), kEw, 0, st_>>>(col_of[k].p, h.csc.idx,
                                                           from_orig ? orig_c[k].p : h.csc.val, h.csc.val, r, c,
                                                           h.csc.nnz, 0, h.coff);
      }
    };
    const RedSlots none{};
    for (int s = 0; s < prm.ruiz_iters; ++s) {
      for (Shard& h : shards_) {
        run_pass(h.csr, OpInfNormScale{dr.p + h.roff, rs_.p + h.roff}, none, st_);
        run_pass(h.csc, OpInfNormScale{dc.p + h.coff, cs_.p + h.coff}, none, st_);
      }
      GatherY(dr.p);
      GatherX(dc.p);
      rescale(false, dr.p, dc.p);
    }
    GatherYFull(rs_.p);
    GatherXFull(cs_.p);
    // PC on K.Scaled(ruiz) recomputed from the original values (scaling.cpp:89).
    rescale(true, rs_.p, cs_.p);
    auto mode_of = [](double p) { return p == 0.0 ? 0 : (p == 1.0 ? 1 : (p == 2.0 ? 2 : 3)); };
    const double pr = 2.0 - prm.pc_alpha, pc = prm.pc_alpha;
    for (Shard& h : shards_) {
      if (skip_pc_) break;  // RuizEquilibrate alone (pdhg_compute_scaling)
      run_pass(h.csr, OpPowerSumScale{pr, mode_of(pr), rs_.p + h.roff}, none, st_);
      run_pass(h.csc, OpPowerSumScale{pc, mode_of(pc), cs_.p + h.coff}, none, st_);
    }
    GatherYFull(rs_.p);
    GatherXFull(cs_.p);
    // Final K_s from the original values (ApplyScaling, scaling.cpp:105-106).
    rescale(true, rs_.p, cs_.p);
    check_launch("scaling");
    Sync();
  }
  k_mul<<<ew_grid(np_), kEw, 0, st_>>>(c_o_.p, cs_.p, c_s_.p, np_);
  k_div<<<ew_grid(np_), kEw, 0, st_>>>(l_o_.p, cs_.p, l_s_.p, np_);
  k_div<<<ew_grid(np_), kEw, 0, st_>>>(u_o_.p, cs_.p, u_s_.p, np_);
  k_mul<<<ew_grid(mp_), kEw, 0, st_>>>(q_o_.p, rs_.p, q_s_.p, mp_);
  check_launch("apply scaling");
}

// Common scaled bounds: bit 0 when every l_s is bitwise one value, bit 1 for
// u_s (the primal kernels then skip those streams). PDHG_UNIFORM_BOUNDS=0
// disables it (A/B timing).
void Session::UniformBounds() {
  bnd_ = 0;
  lb_ = ub_ = 0.0;
  const char* env = std::getenv("PDHG_UNIFORM_BOUNDS");
  if (n_ == 0 || (env && env[0] == '0')) return;
  DArray<int> diff;
  diff.alloc(2);
  PDHG_CUDA(cudaMemsetAsync(diff.p, 0, 2 * sizeof(int), st_));
  k_uniform<<<ew_grid(n_), kEw, 0, st_>>>(l_s_.p, pad_c_.p, n_, diff.p);
  k_uniform<<<ew_grid(n_), kEw, 0, st_>>>(u_s_.p, pad_c_.p, n_, diff.p + 1);
  int h[2];
  int32_t p0 = 0;
  PDHG_CUDA(cudaMemcpyAsync(h, diff.p, sizeof(h), cudaMemcpyDeviceToHost, st_));
  PDHG_CUDA(cudaMemcpyAsync(&p0, pad_c_.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
  Sync();
  PDHG_CUDA(cudaMemcpyAsync(&lb_, l_s_.p + p0, sizeof(double), cudaMemcpyDeviceToHost, st_));
  PDHG_CUDA(cudaMemcpyAsync(&ub_, u_s_.p + p0, sizeof(double), cudaMemcpyDeviceToHost, st_));
  Sync();
  bnd_ = (h[0] ? 0 : 1) | (h[1] ? 0 : 2);
  // The check may drop all four bound arrays when the original bounds are
  // the same common values as the scaled ones (l in {0, -inf}, u in {0, +inf}).
  bnd_all_ = false;
  if (bnd_ == 3) {
    PDHG_CUDA(cudaMemsetAsync(diff.p, 0, 2 * sizeof(int), st_));
    k_uniform<<<ew_grid(n_), kEw, 0, st_>>>(l_o_.p, pad_c_.p, n_, diff.p);
    k_uniform<<<ew_grid(n_), kEw, 0, st_>>>(u_o_.p, pad_c_.p, n_, diff.p + 1);
    double lo = 0.0, uo = 0.0;
    PDHG_CUDA(cudaMemcpyAsync(h, diff.p, sizeof(h), cudaMemcpyDeviceToHost, st_));
    PDHG_CUDA(cudaMemcpyAsync(&lo, l_o_.p + p0, sizeof(double), cudaMemcpyDeviceToHost, st_));
    PDHG_CUDA(cudaMemcpyAsync(&uo, u_o_.p + p0, sizeof(double), cudaMemcpyDeviceToHost, st_));
    Sync();
    bnd_all_ = !h[0] && !h[1] && std::memcmp(&lo, &lb_, sizeof(double)) == 0 &&
               std::memcmp(&uo, &ub_, sizeof(double)) == 0;
  }
}

// ||c||, ||q|| in both spaces (kkt.cpp:45-56), deterministic device sums over
// the full (padded, zero-filled) vectors every rank holds.
void Session::DeviceNorms() {
  const int g = 148;
  DArray<double> part, out;
  part.alloc(g * 4);
  out.alloc(4);
  const double* vecs[4] = {c_s_.p, q_s_.p, c_o_.p, q_o_.p};
  const int64_t lens[4] = {np_, mp_, np_, mp_};
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

// Session-lifetime staging: one device vector and one pinned host vector of
// max(m, n) doubles, so no solve-path call allocates (cudaMalloc / cudaFree
// synchronise the device and were the largest non-kernel cost of a solve).
double* Session::DevStage() {
  const size_t need = static_cast<size_t>(std::max<int64_t>(std::max(m_, n_), 1));
  if (dstage_.n < need) dstage_.alloc(need, &arena_);
  return dstage_.p;
}

double* Session::HostStage(size_t at_least) {
  const size_t need = std::max(at_least, static_cast<size_t>(std::max<int64_t>(std::max(m_, n_), 1)));
  if (hstage_n_ < need) {
    pinned_put(hstage_, hstage_bytes_);
    hstage_ = nullptr;
    hstage_ = static_cast<double*>(pinned_get(need * sizeof(double), &hstage_bytes_));
    hstage_n_ = hstage_bytes_ / sizeof(double);
  }
  return hstage_;
}

// Host vector (original order) -> device (padded order); padding zeroed.
// `host` may already be the pinned stage.
void Session::ToInternal(const double* host, const DArray<int32_t>& pad, double* dev, int64_t n, int64_t padded) {
  if (padded) PDHG_CUDA(cudaMemsetAsync(dev, 0, padded * sizeof(double), st_));
  if (!n) return;
  double* d = DevStage();
  PDHG_CUDA(cudaMemcpyAsync(d, host, n * sizeof(double), cudaMemcpyHostToDevice, st_));
  k_scatter<<<ew_grid(n), kEw, 0, st_>>>(d, pad.p, dev, n);
  Sync();
}

// Host copy of a staged result. Destinations are usually fresh pageable
// buffers (numpy / std::vector): the copy is dominated by first-touch page
// faults, which the kernel serves in parallel -- so large copies are split
// over up to 8 threads.
static void CopyOut(double* dst, const double* src, int64_t n) {
  constexpr int64_t kChunk = int64_t(1) << 18;  // doubles per thread, at least
  const int hw = static_cast<int>(std::thread::hardware_concurrency());
  const int threads = static_cast<int>(std::min<int64_t>(std::min(std::max(hw, 1), 8), n / kChunk));
  if (threads <= 1) {
    std::memcpy(dst, src, n * sizeof(double));
    return;
  }
  std::vector<std::thread> pool;
  const int64_t per = (n + threads - 1) / threads;
  for (int t = 1; t < threads; ++t) {
    const int64_t b = std::min(n, t * per), e = std::min(n, b + per);
    pool.emplace_back([=] { std::memcpy(dst + b, src + b, (e - b) * sizeof(double)); });
  }
  std::memcpy(dst, src, std::min(n, per) * sizeof(double));
  for (auto& th : pool) th.join();
}

void Session::ToHost(const double* dev, const double* scale, const DArray<int32_t>& pad, double* host, int64_t n) {
  if (!n || !host) return;
  double* d = DevStage();
  double* h = HostStage();
  k_unpermute<<<ew_grid(n), kEw, 0, st_>>>(dev, scale, pad.p, d, n);
  PDHG_CUDA(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st_));
  Sync();
  CopyOut(host, h, n);
}

// ================================================================== kernels
// One PDHG iteration (solver.cpp:284-306): every local shard's K-CSC primal
// pass writes its slice of x+, one all-gather rebuilds x+ everywhere, then the
// K-CSR dual passes and the all-gather of y+.
template <bool kAdapt, int kBnd>
void Session::PrimalPass(Shard& h, int a, int b, int j) {
  const int64_t o = h.coff;
  OpPrimal<kAdapt, kBnd> op{y_[a].p, x_[a].p + o, x_[b].p + o, xbar_.p + o, c_s_.p + o, l_s_.p + o, u_s_.p + o,
                            scal_.p, j};
  op.halt = halt_ptr_;
  run_pass(h.csc, op, RedSlots{kAdapt ? h.red[1].p : nullptr}, fork_);
}

void Session::LaunchPrimal(Shard& h, int a, int b, int j, bool adapt) {
  switch (bnd_ + 4 * adapt) {
    case 0: PrimalPass<false, 0>(h, a, b, j); break;
    case 1: PrimalPass<false, 1>(h, a, b, j); break;
    case 2: PrimalPass<false, 2>(h, a, b, j); break;
    case 3: PrimalPass<false, 3>(h, a, b, j); break;
    case 4: PrimalPass<true, 0>(h, a, b, j); break;
    case 5: PrimalPass<true, 1>(h, a, b, j); break;
    case 6: PrimalPass<true, 2>(h, a, b, j); break;
    default: PrimalPass<true, 3>(h, a, b, j); break;
  }
}

void Session::LaunchStep(int parity, int j, bool adapt) {
  const int a = parity, b = 1 - parity;
  launches_ += launches_csc() + launches_csr();
  for (Shard& h : shards_) LaunchPrimal(h, a, b, j, adapt);
  GatherX(x_[b].p);
  for (Shard& h : shards_) {
    const int64_t o = h.roff;
    if (adapt) {
      OpDual<true> op{x_[b].p, y_[a].p + o, y_[b].p + o, ybar_.p + o, kx_[a].p + o, kx_[b].p + o, q_s_.p + o,
                      h.rk, scal_.p, j};
      op.halt = halt_ptr_;
      run_pass(h.csr, op, RedSlots{h.red[0].p}, fork_);
    } else {
      OpDual<false> op{x_[b].p, y_[a].p + o, y_[b].p + o, ybar_.p + o, kx_[a].p + o, kx_[b].p + o, q_s_.p + o,
                       h.rk, scal_.p, j};
      op.halt = halt_ptr_;
      run_pass(h.csr, op, RedSlots{}, fork_);
    }
  }
  GatherY(y_[b].p);
  if (adapt) {
    for (size_t k = 0; k < shards_.size(); ++k) {
      Shard& h = shards_[k];
      k_adapt_sum<<<1, kBlock, 0, st_>>>(h.red[1].p, h.csc.parts(), h.red[0].p, h.csr.parts(), red_out_.p + k * kPack,
                                         scal_.p);
    }
    SumPacks(3, scal_.p);
    k_adapt_apply<<<1, 1, 0, st_>>>(red_out_.p, scal_.p, j);
    launches_ += static_cast<int64_t>(shards_.size()) + 1 + (shards_.size() > 1);
  }
}

// Shard packs -> pack 0 (fixed shard order), then the sum over ranks.
void Session::SumPacks(int n, const Scalars* guard) {
  if (shards_.size() > 1)
    k_sum_packs<<<1, kPack, 0, st_>>>(red_out_.p, static_cast<int>(shards_.size()), kPack, n, guard);
  comm_->AllReduceSum(red_out_.p, n, st_);
}

// Persistent block kernel eligibility (persist.cuh; opt-in PDHG_PERSIST=1,
// measured slower): one shard, one device, the K-CSC entirely one
// uniform-length class S, the K-CSR entirely one class L of 4-row
// TMA-staged groups (transportation / assignment shapes), no class-S
// variants that change the pass structure.
bool Session::PersistOk() const {
  const char* e = std::getenv("PDHG_PERSIST");
  if (!(e && e[0] == '1') || world_ != 1 || shards_.size() != 1 || !comm_->local()) return false;
  const Layout& c = shards_[0].csc;
  const Layout& r = shards_[0].csr;
  const bool csc_ok = c.nseg > 0 && c.s1 == c.nseg && c.s_len > 0 && c.split_w == 0;
  const bool csr_ok = r.nseg > 0 && r.s1 == 0 && r.s2 == 0 && r.s3 == r.nseg && r.l_rpc == 4 && r.l_stage > 0;
  return csc_ok && csr_ok;
}

template <int kBnd>
void Session::LaunchBlockT(int parity, int count) {
  Shard& h = shards_[0];
  BlockArgs<OpPrimal<false, kBnd>, OpDual<false>> a{};
  a.p_idx = h.csc.idx;
  a.p_val = h.csc.val;
  a.p_ptr = h.csc.ptr;
  a.p_send = h.csc.s1;
  a.p_su = h.csc.s_u;
  a.p_nb = h.csc.nb_s();
  a.d_ptr = h.csr.ptr;
  a.d_idx = h.csr.idx;
  a.d_val = h.csr.val;
  a.d_s2 = h.csr.s2;
  a.d_s3 = h.csr.s3;
  a.d_nb = h.csr.nb_l();
  for (int q = 0; q < 2; ++q) {
    const int x0 = q, x1 = 1 - q;
    a.opp[q] = OpPrimal<false, kBnd>{y_[x0].p, x_[x0].p + h.coff, x_[x1].p + h.coff, xbar_.p + h.coff,
                                     c_s_.p + h.coff, l_s_.p + h.coff, u_s_.p + h.coff, scal_.p, 0};
    a.opd[q] = OpDual<false>{x_[x1].p, y_[x0].p + h.roff, y_[x1].p + h.roff, ybar_.p + h.roff, kx_[x0].p + h.roff,
                             kx_[x1].p + h.roff, q_s_.p + h.roff, h.rk, scal_.p, 0};
  }
  a.parity = parity;
  a.count = count;
  a.gbar = gbar_.p;
  PDHG_CUDA(cudaMemsetAsync(gbar_.p, 0, sizeof(unsigned), st_));
  launch_block(a, h.csc.s_len, h.csc.s_u < h.csc.s1, h.csr.l_stage, st_);
}

void Session::LaunchBlock(int parity, int count) {
  switch (bnd_) {
    case 0: return LaunchBlockT<0>(parity, count);
    case 1: return LaunchBlockT<1>(parity, count);
    case 2: return LaunchBlockT<2>(parity, count);
    default: return LaunchBlockT<3>(parity, count);
  }
}

// `count` PDHG iterations starting from buffer `parity`. Blocks are replayed
// from captured CUDA graphs (one per parity/length/adapt combination).
void Session::RunSteps(int parity, int count, bool adapt) {
  Graph* g = nullptr;
  for (Graph& gg : graphs_)
    if (gg.steps == count && gg.parity == parity && gg.adapt == adapt) g = &gg;
  const bool block = persist_ && !adapt;
  if (!g && count >= 4 && comm_->graphs()) {
    cudaGraph_t graph;
    const int64_t before = launches_;
    PDHG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    if (block) LaunchBlock(parity, count);
    else
      for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, adapt);
    PDHG_CUDA(cudaStreamEndCapture(st_, &graph));
    launches_ = before;
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
    const int64_t per = launches_csc() + launches_csr() +
                        (adapt ? static_cast<int64_t>(shards_.size()) + 1 + (shards_.size() > 1) : 0);
    launches_ += block ? 1 : static_cast<int64_t>(count) * per;
    trace_graph("steps", count);
    PDHG_CUDA(cudaGraphLaunch(g->exec, st_));
  } else if (block) {
    LaunchBlock(parity, count);
  } else {
    for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, adapt);
  }
  check_launch("pdhg steps");
}

// Synchronous loop, block ending at a check: ONE captured graph holds the
// block's steps, the inner_base advance, the check passes and the D2H of the
// reduced pack into pinned host memory, so a check costs one graph launch and
// one stream synchronisation instead of eager launches and a separate copy.
void Session::RunChecked(int parity, int count, bool adapt) {
  static const bool check_branches = [] {  // PDHG_CHECK_BRANCHES=0: serial check passes (A/B)
    const char* e = std::getenv("PDHG_CHECK_BRANCHES");
    return !(e && e[0] == '0');
  }();
  const int key = parity + 8;  // graphs_ key space: plain blocks use 0 / 1
  Graph* g = nullptr;
  for (Graph& gg : graphs_)
    if (gg.steps == count && gg.parity == key && gg.adapt == adapt) g = &gg;
  const int pa = (parity + count) & 1;
  if (!g) {
    cudaGraph_t graph;
    const int64_t before = launches_;
    PDHG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    if (persist_ && !adapt) LaunchBlock(parity, count);
    else
      for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, adapt);
    k_inner_add<<<1, 1, 0, st_>>>(scal_.p, count);
    LaunchCheck(x_[pa].p, y_[pa].p, xbar_.p, ybar_.p, kx_[pa].p, nullptr, check_branches);
    PDHG_CUDA(cudaMemcpyAsync(host_red_, red_out_.p, sizeof(CheckOut), cudaMemcpyDeviceToHost, st_));
    if (adapt)  // the block's adapted step size, for EvalInfo and later pushes (slot kPack - 2)
      PDHG_CUDA(cudaMemcpyAsync(host_red_ + kPack - 2, &scal_.p->eta, sizeof(double), cudaMemcpyDeviceToHost, st_));
    PDHG_CUDA(cudaStreamEndCapture(st_, &graph));
    launches_ = before;
    Graph ng;
    ng.steps = count;
    ng.parity = key;
    ng.adapt = adapt;
    PDHG_CUDA(cudaGraphInstantiate(&ng.exec, graph, 0));
    cudaGraphDestroy(graph);
    graphs_.push_back(ng);
    g = &graphs_.back();
  }
  const int64_t per = launches_csc() + launches_csr() +
                      (adapt ? static_cast<int64_t>(shards_.size()) + 1 + (shards_.size() > 1) : 0);
  launches_ += (persist_ && !adapt ? 1 : static_cast<int64_t>(count) * per) + 1 + launches_csr() + launches_csc() +
               static_cast<int64_t>(shards_.size()) + (shards_.size() > 1);
  PDHG_CUDA(cudaGraphLaunch(g->exec, st_));
  check_launch("pdhg block + check");
}

// Device-resident loop: ONE graph launch runs blocks of `count` steps, each
// followed by the check, the device decision (decide.cuh) and the best copy,
// inside a conditional WHILE node whose condition k_decide_loop sets on the
// device -- the host is needed again only for a restart (glibc exp/log),
// termination, a limit or a non-finite iterate. `count` is even, so every
// block starts at the same parity and one body serves all blocks.
void Session::RunDeviceLoop(int parity, int count) {
  Graph* g = nullptr;
  for (Graph& gg : loops_)
    if (gg.steps == count && gg.parity == parity) g = &gg;
  if (!g) {
    cudaGraph_t parent;
    PDHG_CUDA(cudaGraphCreate(&parent, 0));
    // k_loop_start, then the WHILE node depending on it.
    PDHG_CUDA(cudaStreamBeginCaptureToGraph(st_, parent, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_loop_start<<<1, 1, 0, st_>>>(dstate_.p);
    cudaGraph_t captured;
    PDHG_CUDA(cudaStreamEndCapture(st_, &captured));
    size_t nn = 0;
    PDHG_CUDA(cudaGraphGetNodes(parent, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    PDHG_CUDA(cudaGraphGetNodes(parent, nodes.data(), &nn));
    cudaGraphConditionalHandle cond;
    PDHG_CUDA(cudaGraphConditionalHandleCreate(&cond, parent, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    PDHG_CUDA(cudaGraphAddNode(&wnode, parent, nodes.data(), nn, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const int64_t before = launches_;
    PDHG_CUDA(cudaStreamBeginCaptureToGraph(st_, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, false);
    const int pa = (parity + count) & 1;
    LaunchCheck(x_[pa].p, y_[pa].p, xbar_.p, ybar_.p, kx_[pa].p, scal_.p, true);
    k_decide_loop<<<1, 1, 0, st_>>>(red_out_.p, scal_.p, dstate_.p, count, cond);
    k_copy_best<<<ew_grid(np_ + mp_), kEw, 0, st_>>>(scal_.p, dstate_.p, x_[pa].p, xbar_.p, xbest_.p, np_, y_[pa].p,
                                                      ybar_.p, ybest_.p, mp_);
    PDHG_CUDA(cudaStreamEndCapture(st_, &captured));
    launches_ = before;
    Graph ng;
    ng.steps = count;
    ng.parity = parity;
    ng.adapt = false;
    PDHG_CUDA(cudaGraphInstantiate(&ng.exec, parent, 0));
    cudaGraphDestroy(parent);
    loops_.push_back(ng);
    g = &loops_.back();
  }
  PDHG_CUDA(cudaGraphLaunch(g->exec, st_));
  check_launch("device loop");
}

// Pipelined loop: one captured graph per (length, parity, adapt, check,
// slot) holding the block's steps, the counter advance and -- at check
// iterations -- the check passes, k_decide, the best copy, the halt settle
// and the D2H of the decision state into pinned slot `slot`.
void Session::RunBlock(int parity, int count, bool adapt, bool check, int slot) {
  const int key_par = parity + 2 * (check ? 1 + slot : 0);
  Graph* g = nullptr;
  for (Graph& gg : blocks_)
    if (gg.steps == count && gg.parity == key_par && gg.adapt == adapt) g = &gg;
  const int pa = (parity + count) & 1;
  auto body = [&] {
    halt_ptr_ = &scal_.p->halt;  // queued blocks must stop after a halting check
    for (int j = 0; j < count; ++j) LaunchStep((parity + j) & 1, j, adapt);
    halt_ptr_ = nullptr;
    k_advance<<<1, 1, 0, st_>>>(scal_.p, dstate_.p, count);
    if (check) {
      LaunchCheck(x_[pa].p, y_[pa].p, xbar_.p, ybar_.p, kx_[pa].p, scal_.p);
      k_decide<<<1, 1, 0, st_>>>(red_out_.p, scal_.p, dstate_.p);
      k_copy_best<<<ew_grid(np_ + mp_), kEw, 0, st_>>>(scal_.p, dstate_.p, x_[pa].p, xbar_.p, xbest_.p, np_,
                                                        y_[pa].p, ybar_.p, ybest_.p, mp_);
      k_settle<<<1, 1, 0, st_>>>(scal_.p);
      PDHG_CUDA(cudaMemcpyAsync(hstate_ + slot, dstate_.p, sizeof(DecideState), cudaMemcpyDeviceToHost, st_));
    }
  };
  const int64_t before = launches_;
  if (!g) {
    cudaGraph_t graph;
    PDHG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    body();
    PDHG_CUDA(cudaStreamEndCapture(st_, &graph));
    Graph ng;
    ng.steps = count;
    ng.parity = key_par;
    ng.adapt = adapt;
    PDHG_CUDA(cudaGraphInstantiate(&ng.exec, graph, 0));
    cudaGraphDestroy(graph);
    blocks_.push_back(ng);
    g = &blocks_.back();
  }
  launches_ = before;
  const int64_t per = launches_csc() + launches_csr() +
                      (adapt ? static_cast<int64_t>(shards_.size()) + 1 + (shards_.size() > 1) : 0);
  launches_ += static_cast<int64_t>(count) * per + 1;
  if (check)
    launches_ += launches_csr() + launches_csc() + static_cast<int64_t>(shards_.size()) + (shards_.size() > 1) + 3;
  PDHG_CUDA(cudaGraphLaunch(g->exec, st_));
  check_launch("pdhg block");
}

// The check (solver.cpp:390-428) as two matrix passes per shard: the row
// side gathers x_bar (K x_bar), the column side gathers [y, y_bar]. Both
// gathered operands are all-gathered first; the 26 sums are reduced per
// shard, over local shards and over ranks.
void Session::LaunchCheck(const double* x, const double* y, const double* xb, const double* yb, const double* kx,
                          const Scalars* guard, bool branches) {
  if (xb != x) GatherX(const_cast<double*>(xb));
  if (yb != y) GatherY(const_cast<double*>(yb));
  launches_ += launches_csr() + launches_csc() + static_cast<int64_t>(shards_.size()) + (shards_.size() > 1);
  for (size_t k = 0; k < shards_.size(); ++k) {
    Shard& h = shards_[k];
    const int64_t r = h.roff, c = h.coff;
    OpCheckRow row{xb, kxavg_.p + r, kx + r, y + r, yb + r, ystart_.p + r, q_s_.p + r, q_o_.p + r, rs_.p + r, h.rk,
                   guard};
    // Inside a captured graph (`branches`) the independent row and column
    // passes become parallel branches when the row pass is one kernel.
    cudaStream_t side = fork_.side[2];
    const bool beside = branches && side && pass_launches(h.csr) == 1;
    if (beside) {
      PDHG_CUDA(cudaEventRecord(fork_.fork, st_));
      PDHG_CUDA(cudaStreamWaitEvent(side, fork_.fork, 0));
      run_pass(h.csr, row, RedSlots{h.red[0].p}, side);
    } else {
      run_pass(h.csr, row, RedSlots{h.red[0].p}, fork_);
    }
    if (bnd_all_) {
      OpCheckCol<true> col{y, yb, x + c, xb + c, xstart_.p + c, c_s_.p + c, l_s_.p + c, u_s_.p + c, c_o_.p + c,
                           l_o_.p + c, u_o_.p + c, cs_.p + c, guard, lb_, ub_};
      run_pass(h.csc, col, RedSlots{h.red[1].p}, fork_);
    } else {
      OpCheckCol<false> col{y, yb, x + c, xb + c, xstart_.p + c, c_s_.p + c, l_s_.p + c, u_s_.p + c, c_o_.p + c,
                            l_o_.p + c, u_o_.p + c, cs_.p + c, guard};
      run_pass(h.csc, col, RedSlots{h.red[1].p}, fork_);
    }
    if (beside) {  // join (a 4-class column pass may re-record join[2] on the same stream: still after)
      PDHG_CUDA(cudaEventRecord(fork_.join[2], side));
      PDHG_CUDA(cudaStreamWaitEvent(st_, fork_.join[2], 0));
    }
    double* pk = red_out_.p + k * kPack;
    if (guard)
      k_reduce_two_guarded<<<kRowRed + kColRed, kBlock, 0, st_>>>(guard, h.red[0].p, h.csr.parts(), kRowRed,
                                                                  h.red[1].p, h.csc.parts(), kColRed, pk);
    else
      k_reduce_two<<<kRowRed + kColRed, kBlock, 0, st_>>>(h.red[0].p, h.csr.parts(), kRowRed, h.red[1].p,
                                                          h.csc.parts(), kColRed, pk);
  }
  SumPacks(kRowRed + kColRed, guard);
  check_launch("check");
}

void Session::ReadCheck(CheckOut* out) {
  PDHG_CUDA(cudaMemcpyAsync(host_red_, red_out_.p, sizeof(CheckOut), cudaMemcpyDeviceToHost, st_));
  Sync();
  std::memcpy(out, host_red_, sizeof(CheckOut));
}

// ================================================================ solve loop
void Session::Solve(const pdhg_params& prm, pdhg_eval_cb cb, void* user, pdhg_result* out) {
  NvtxScope nv("pdhg.solve");
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  if (!ev_[0]) {
    PDHG_CUDA(cudaEventCreate(&ev_[0]));
    PDHG_CUDA(cudaEventCreate(&ev_[1]));
  }
  launches_ = 0;
  PDHG_CUDA(cudaEventRecord(ev_[0], st_));
  const auto t0 = std::chrono::steady_clock::now();
  auto secs = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };

  // eta = 0.9 / ||K|| (solver.cpp:233-234), omega0 = ||c_s|| / ||q_s|| (:235-238).
  std::optional<NvtxScope> nv_phase;
  nv_phase.emplace("pdhg.opnorm");
  const double op = OpNorm(100, prm.seed);
  nv_phase.reset();
  const double t_opnorm = secs();
  double t_checks = 0.0;
  int64_t nchecks = 0;
  Scalars sc{};
  sc.eta = op > 0.0 ? 0.9 / op : 1.0;
  sc.omega = 1.0;
  if (c_norm_s_ > 1e-10 && q_norm_s_ > 1e-10) sc.omega = c_norm_s_ / q_norm_s_;
  sc.inner_base = 0.0;
  sc.pw_norm = 1.0;
  sc.lb = lb_;
  sc.ub = ub_;
  const bool adapt = prm.adaptive_step != 0;

  // x0 = proj(0), y0 = 0, kx = K x0 (solver.cpp:240-245).
  int par = 0;
  k_clamp0<<<ew_grid(np_), kEw, 0, st_>>>(l_s_.p, u_s_.p, x_[0].p, np_);
  if (mp_) PDHG_CUDA(cudaMemsetAsync(y_[0].p, 0, mp_ * sizeof(double), st_));
  for (Shard& h : shards_) run_pass(h.csr, OpSpmv{x_[0].p, kx_[0].p + h.roff}, RedSlots{}, st_);
  launches_ += 1 + launches_csr();

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
    Copy(xbest_.p, P == 0 ? x_[par].p : xbar_.p, np_);
    Copy(ybest_.p, P == 0 ? y_[par].p : ybar_.p, mp_);
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
    Copy(xstart_.p, x_[par].p, np_);
    Copy(ystart_.p, y_[par].p, mp_);
    kkt_start = KktError(s.primal_res, s.dual_res, s.gap_abs, sc.omega);
    kkt_prev = std::numeric_limits<double>::infinity();
    sc.inner_base = 0.0;
    inner = 0;
  };
  auto push_scalars = [&] {
    set_steps(sc);
    PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  };

  // Start point: scaled KKT for the loop start and the first termination test
  // (solver.cpp:246-249); the current point stands in for the average.
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

  // ---- Pipelined loop (one process, no NCCL): the next block is queued
  // before the host looks at the previous check; decisions run on the
  // device (decide.cuh), the host only steps in for restarts, termination,
  // limits and the observer. Identical trajectory to the synchronous loop.
  // Opt-in (PDHG_PIPELINE=1): measured on B200 it does not beat the
  // synchronous loop -- a check costs ~80 us of GPU work either way, and a
  // block queued behind a restarting check must still be launched (empty).
  const char* penv = std::getenv("PDHG_PIPELINE");
  const bool pipelined = !finished && !nccl() && (penv && penv[0] == '1');
  if (pipelined) {
    DecideState ds{};
    ds.eps = prm.eps;
    ds.suff = prm.sufficient_decay;
    ds.nec = prm.necessary_decay;
    ds.frac = prm.long_loop_frac;
    ds.offset = offset_;
    ds.qn_s = q_norm_s_;
    ds.cn_s = c_norm_s_;
    ds.qn_o = q_norm_o_;
    ds.cn_o = c_norm_o_;
    ds.restart_enabled = prm.restart_enabled;
    ds.kkt_start = kkt_start;
    ds.kkt_prev = kkt_prev;
    ds.best_k1 = best_k1;
    ds.have_best = have_best;
    ds.checks = 0;
    ds.best_from = -1;
    ds.best_rep = best_rep;
    ds.last_rep = last_rep;
    if (!dstate_.p) dstate_.alloc(1, &arena_);
    if (!hstate_) hstate_ = static_cast<DecideState*>(pinned_get(2 * sizeof(DecideState), &hstate_bytes_));
    if (!pev_[0])
      for (cudaEvent_t& e : pev_) PDHG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sc.halt = 0;
    push_scalars();
    PDHG_CUDA(cudaMemcpyAsync(dstate_.p, &ds, sizeof(DecideState), cudaMemcpyHostToDevice, st_));
    struct Pend {
      int64_t count, iters_after;
      int par_after, slot, id;
      bool check;
    };
    std::deque<Pend> q;
    int64_t it_enq = 0;
    int par_enq = par, next_id = 0, checks_base = 0;
    bool stop_enq = false;
    int limit_status = PDHG_ITER_LIMIT;
    int hslot = 0;
    while (true) {
      while (!stop_enq && q.size() < 2) {
        if (it_enq >= prm.iter_limit) {
          stop_enq = true;
          limit_status = PDHG_ITER_LIMIT;
          break;
        }
        if (secs() >= prm.time_limit) {
          stop_enq = true;
          limit_status = PDHG_TIME_LIMIT;
          break;
        }
        const int64_t count = std::min<int64_t>(prm.check_every - (it_enq % prm.check_every), prm.iter_limit - it_enq);
        if (adapt) {
          sc.adapt_iter = static_cast<double>(it_enq);
          PDHG_CUDA(cudaMemcpyAsync(&scal_.p->adapt_iter, &sc.adapt_iter, sizeof(double), cudaMemcpyHostToDevice,
                                    st_));
        }
        Pend pd{count, it_enq + count, static_cast<int>((par_enq + count) & 1), hslot, -1, false};
        pd.check = pd.iters_after % prm.check_every == 0;
        if (pd.check) pd.id = next_id++;
        RunBlock(par_enq, static_cast<int>(count), adapt, pd.check, hslot);
        PDHG_CUDA(cudaEventRecord(pev_[hslot], st_));
        hslot ^= 1;
        q.push_back(pd);
        it_enq = pd.iters_after;
        par_enq = pd.par_after;
      }
      if (q.empty()) {
        status = limit_status;
        break;
      }
      const Pend pd = q.front();
      q.pop_front();
      const double tc0 = secs();
      PDHG_CUDA(cudaEventSynchronize(pev_[pd.slot]));
      iters = pd.iters_after;
      inner += pd.count;
      par = pd.par_after;
      sc.inner_base += static_cast<double>(pd.count);
      if (!pd.check) continue;
      ++nchecks;
      t_checks += secs() - tc0;
      const DecideState& h = hstate_[pd.slot];
      if (h.checks != pd.id + 1 + checks_base)
        throw Error(PDHG_CUDA_ERROR, "pipelined loop: check skipped unexpectedly");
      have_best = h.have_best != 0;
      best_k1 = h.best_k1;
      best_rep = h.best_rep;
      last_rep = h.last_rep;
      if (adapt) sc.eta = h.eta;
      if (h.action == kNonFinite)
        throw Error(PDHG_NUMERICAL_FAILURE, "non-finite iterate at iteration " + std::to_string(iters));
      if (h.action == kOptimalCur || h.action == kOptimalAvg) {
        status = PDHG_OPTIMAL;  // best copied on the device; queued block skipped
        break;
      }
      pdhg_eval_info info{};
      info.iteration = iters;
      info.inner_iteration = inner;
      info.restarts = restarts;
      info.omega = sc.omega;
      info.eta = sc.eta;
      info.kkt_candidate = h.kkt_cand;
      info.kkt_loop_start = kkt_start;
      info.candidate_is_current = h.take_cur;
      info.original_report = last_rep;
      info.seconds = secs();
      if (h.action == kRestart) {
        // Queued blocks were skipped: requeue from here after the restart.
        for (const Pend& dropped : q)
          if (dropped.check) --checks_base;  // ids handed out to skipped checks
        q.clear();
        it_enq = iters;
        par_enq = par;
        stop_enq = false;
        info.restarted = 1;
        // Restart (solver.cpp:430-446), as in the synchronous loop.
        const bool take_cur = h.take_cur != 0;
        const pdhg_report& ps = take_cur ? h.s_cur : h.s_avg;
        // dx, dy from the check pack (still in red_out_: nothing ran after it).
        double pack[kRowRed + kColRed];
        PDHG_CUDA(cudaMemcpyAsync(pack, red_out_.p, sizeof(pack), cudaMemcpyDeviceToHost, st_));
        Sync();
        const int P = take_cur ? 0 : 1;
        const double dx = std::sqrt(pack[kRowRed + P * kColPer + kDx2]);
        const double dy = std::sqrt(pack[P * kRowPer + kDy2]);
        sc.omega = UpdatePrimalWeight(sc.omega, dx, dy);
        if (!take_cur) {
          Copy(x_[par].p, xbar_.p, np_);
          Copy(y_[par].p, ybar_.p, mp_);
          Copy(kx_[par].p, kxavg_.p, mp_);
        }
        start_loop(ps);
        ++restarts;
        sc.halt = 0;
        push_scalars();
        DecideState reset = h;
        reset.kkt_start = kkt_start;
        reset.kkt_prev = kkt_prev;
        reset.inner = 0;
        reset.iters = iters;
        PDHG_CUDA(cudaMemcpyAsync(dstate_.p, &reset, sizeof(DecideState), cudaMemcpyHostToDevice, st_));
      } else {
        kkt_prev = h.kkt_cand;
      }
      if (prm.log_every > 0 && (info.iteration - last_log >= prm.log_every || info.iteration == 0)) {
        last_log = info.iteration;
        std::printf("iter=%lld time=%.3f rel_primal=%.3e rel_dual=%.3e rel_gap=%.3e omega=%.3e restarts=%lld\n",
                    (long long)info.iteration, info.seconds, info.original_report.rel_primal,
                    info.original_report.rel_dual, info.original_report.rel_gap, info.omega,
                    (long long)info.restarts);
      }
      if (cb && cb(&info, user) != 0) {
        Sync();
        throw Error(PDHG_ABORTED, "aborted by observer");
      }
    }
    Sync();  // queued (skipped) blocks drain
    sc.halt = 0;
    push_scalars();
    finished = true;
  }

  // Time limit: one clock decides for every rank (rank 0's, shipped in the
  // check pack), so all ranks leave the loop after the same block.
  bool time_up = !(prm.time_limit > 0.0);
  static const bool fused_check = [] {  // PDHG_FUSED_CHECK=0: eager checks (A/B)
    const char* e = std::getenv("PDHG_FUSED_CHECK");
    return !(e && e[0] == '0');
  }();
  // PDHG_DEVICE_LOOP=1: device-resident loop (read per solve: A/B, tests).
  // Opt-in: 0.3 % faster on transport, but kernels inside conditional-graph
  // bodies are invisible to kernel-replay profilers (ncu), so the default
  // keeps every launch observable.
  const bool device_loop_on = [] {
    const char* e = std::getenv("PDHG_DEVICE_LOOP");
    return e && e[0] == '1';
  }();
  // The device-resident loop needs the host only for restarts, termination,
  // limits: not with an observer or a progress log (called at every check),
  // adaptive steps (host-pushed iteration counter) or NCCL (rank-0 clock).
  const bool device_loop = device_loop_on && fused_check && !cb && prm.log_every <= 0 && !adapt && !nccl() &&
                           prm.check_every >= 4 && prm.check_every % 2 == 0;
  const double t_loop0 = secs();
  nv_phase.emplace("pdhg.loop");
  while (!finished) {
    if (iters >= prm.iter_limit) {
      status = PDHG_ITER_LIMIT;
      break;
    }
    if (!nccl()) time_up = secs() >= prm.time_limit;
    if (time_up) {
      status = PDHG_TIME_LIMIT;
      break;
    }
    if (device_loop && iters % prm.check_every == 0 && prm.iter_limit - iters >= prm.check_every) {
      DecideState ds{};
      ds.eps = prm.eps;
      ds.suff = prm.sufficient_decay;
      ds.nec = prm.necessary_decay;
      ds.frac = prm.long_loop_frac;
      ds.offset = offset_;
      ds.qn_s = q_norm_s_;
      ds.cn_s = c_norm_s_;
      ds.qn_o = q_norm_o_;
      ds.cn_o = c_norm_o_;
      ds.restart_enabled = prm.restart_enabled;
      ds.kkt_start = kkt_start;
      ds.kkt_prev = kkt_prev;
      ds.best_k1 = best_k1;
      ds.have_best = have_best;
      ds.checks = 0;
      ds.iters = iters;
      ds.inner = inner;
      ds.block = prm.check_every;
      ds.iter_limit = prm.iter_limit;
      const double left = prm.time_limit - secs();
      ds.remaining_ns = left >= 1.8e10 ? ~uint64_t(0) >> 1 : static_cast<uint64_t>(std::max(left, 0.0) * 1e9);
      ds.deadline_ns = 0;
      ds.best_from = -1;
      ds.best_rep = best_rep;
      ds.last_rep = last_rep;
      if (!dstate_.p) dstate_.alloc(1, &arena_);
      if (!hstate_) hstate_ = static_cast<DecideState*>(pinned_get(2 * sizeof(DecideState), &hstate_bytes_));
      sc.halt = 0;
      push_scalars();
      PDHG_CUDA(cudaMemcpyAsync(dstate_.p, &ds, sizeof(DecideState), cudaMemcpyHostToDevice, st_));
      const double tc0 = secs();
      RunDeviceLoop(par, static_cast<int>(prm.check_every));
      PDHG_CUDA(cudaMemcpyAsync(hstate_, dstate_.p, sizeof(DecideState), cudaMemcpyDeviceToHost, st_));
      Sync();
      t_checks += secs() - tc0;
      const DecideState h = hstate_[0];
      const int64_t ran = h.iters - iters;
      if (ran <= 0 || ran % prm.check_every != 0 || h.checks != ran / prm.check_every)
        throw Error(PDHG_CUDA_ERROR, "device loop: inconsistent block count");
      // per block: steps, the check passes and their reduction, k_decide_loop,
      // k_copy_best; per launch: k_loop_start
      launches_ += 1 + (ran / prm.check_every) *
                           (prm.check_every * (launches_csr() + launches_csc()) + launches_csr() + launches_csc() + 3);
      iters = h.iters;
      inner = h.inner;
      sc.inner_base += static_cast<double>(ran);
      nchecks += h.checks;
      have_best = h.have_best != 0;
      best_k1 = h.best_k1;
      best_rep = h.best_rep;
      last_rep = h.last_rep;
      kkt_prev = h.kkt_prev;
      if (h.action == kNonFinite)
        throw Error(PDHG_NUMERICAL_FAILURE, "non-finite iterate at iteration " + std::to_string(iters));
      if (h.action == kOptimalCur || h.action == kOptimalAvg) {
        status = PDHG_OPTIMAL;  // best iterate copied on the device
        sc.halt = 0;
        push_scalars();
        break;
      }
      if (h.action == kRestart) {  // Restart (solver.cpp:430-446), as in the loops below
        const bool take_cur = h.take_cur != 0;
        double pack[kRowRed + kColRed];
        PDHG_CUDA(cudaMemcpyAsync(pack, red_out_.p, sizeof(pack), cudaMemcpyDeviceToHost, st_));
        Sync();
        const int P = take_cur ? 0 : 1;
        const double dx = std::sqrt(pack[kRowRed + P * kColPer + kDx2]);
        const double dy = std::sqrt(pack[P * kRowPer + kDy2]);
        sc.omega = UpdatePrimalWeight(sc.omega, dx, dy);
        if (!take_cur) {
          Copy(x_[par].p, xbar_.p, np_);
          Copy(y_[par].p, ybar_.p, mp_);
          Copy(kx_[par].p, kxavg_.p, mp_);
        }
        start_loop(take_cur ? h.s_cur : h.s_avg);
        ++restarts;
      }
      sc.halt = 0;
      push_scalars();
      continue;
    }
    const int64_t to_check = prm.check_every - (iters % prm.check_every);
    int64_t count = std::min<int64_t>(to_check, prm.iter_limit - iters);
    // The reference tests the clock before every iteration (solver.cpp:256).
    // A block is therefore cut to the iterations the remaining budget holds
    // at the measured per-iteration rate, and the block after a cut one is
    // synchronised so the next clock test sees the device's progress. (NCCL
    // sessions decide on rank 0's clock at checks only.)
    bool capped = false;
    if (!nccl() && std::isfinite(prm.time_limit) && iters > 0) {
      const double now = secs();
      const double per = (now - t_loop0) / static_cast<double>(iters);
      const double left = prm.time_limit - now;
      if (per > 0.0 && static_cast<double>(count) * per > left) {
        count = std::max<int64_t>(1, static_cast<int64_t>(left / per));
        capped = true;
      }
    }
    // A block ending at a check runs as one graph with the check (RunChecked;
    // with adaptive steps the graph also copies the adapted step size out);
    // NCCL sessions keep the eager check.
    const bool fused = fused_check && !nccl() && count == to_check && count >= 4;
    if (adapt) {
      sc.adapt_iter = static_cast<double>(iters);
      PDHG_CUDA(cudaMemcpyAsync(&scal_.p->adapt_iter, &sc.adapt_iter, sizeof(double), cudaMemcpyHostToDevice, st_));
    }
    if (fused) RunChecked(par, static_cast<int>(count), adapt);
    else RunSteps(par, static_cast<int>(count), adapt);
    par = static_cast<int>((par + count) & 1);
    iters += count;
    inner += count;
    sc.inner_base += static_cast<double>(count);
    if (!fused)
      PDHG_CUDA(cudaMemcpyAsync(&scal_.p->inner_base, &sc.inner_base, sizeof(double), cudaMemcpyHostToDevice, st_));
    if (capped) Sync();
    if (iters % prm.check_every != 0) continue;

    // ---- Check (solver.cpp:390-428).
    NvtxScope nv_check("pdhg.check");
    const double tc0 = secs();
    ++nchecks;
    if (fused) {
      Sync();
      std::memcpy(&ck, host_red_, sizeof(CheckOut));
      if (adapt) sc.eta = host_red_[kPack - 2];
    } else {
      LaunchCheck(x_[par].p, y_[par].p, xbar_.p, ybar_.p, kx_[par].p);
    }
    if (!fused && nccl()) {  // rank 0's clock, summed into slot kPack - 1 of every rank
      host_red_[kPack - 1] = (rank_ == 0 && secs() >= prm.time_limit) ? 1.0 : 0.0;
      PDHG_CUDA(cudaMemcpyAsync(red_out_.p + kPack - 1, host_red_ + kPack - 1, sizeof(double), cudaMemcpyHostToDevice,
                                st_));
      comm_->AllReduceMax(red_out_.p + kPack - 1, 1, st_);
      PDHG_CUDA(cudaMemcpyAsync(host_red_ + kPack - 1, red_out_.p + kPack - 1, sizeof(double), cudaMemcpyDeviceToHost,
                                st_));
    }
    if (!fused) {
      if (adapt) PDHG_CUDA(cudaMemcpyAsync(&sc.eta, &scal_.p->eta, sizeof(double), cudaMemcpyDeviceToHost, st_));
      ReadCheck(&ck);
    }
    t_checks += secs() - tc0;  // includes the wait for the block before it
    if (nccl()) time_up = host_red_[kPack - 1] > 0.0;
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
        Copy(x_[par].p, xbar_.p, np_);
        Copy(y_[par].p, ybar_.p, mp_);
        Copy(kx_[par].p, kxavg_.p, mp_);  // ComputeKx(candidate): same pass, same sums
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
    int stop = (cb && cb(&info, user) != 0) ? 1 : 0;
    // An abort on any rank stops every rank. Every rank joins this
    // all-reduce whether or not it has an observer (under torchrun often only
    // rank 0 does), so the collectives stay paired.
    if (nccl()) {
      host_red_[kPack - 1] = stop;
      PDHG_CUDA(cudaMemcpyAsync(red_out_.p + kPack - 1, host_red_ + kPack - 1, sizeof(double), cudaMemcpyHostToDevice,
                                st_));
      comm_->AllReduceMax(red_out_.p + kPack - 1, 1, st_);
      PDHG_CUDA(cudaMemcpyAsync(host_red_ + kPack - 1, red_out_.p + kPack - 1, sizeof(double), cudaMemcpyDeviceToHost,
                                st_));
      Sync();
      stop = host_red_[kPack - 1] > 0.0;
    }
    if (stop) throw Error(PDHG_ABORTED, "aborted by observer");
  }

  if (!have_best) {  // UseBestSeen (solver.cpp:464-471)
    LaunchCheck(x_[par].p, y_[par].p, x_[par].p, y_[par].p, kx_[par].p);
    ReadCheck(&ck);
    reports(0, &s_cur, &o_cur);
    record_best(0, o_cur);
  }

  // Finish (solver.cpp:473-481): unscale best, lambda on the original problem.
  nv_phase.emplace("pdhg.finish");
  const double t_loop = secs();
  if (gx_.use) GatherXFull(xbest_.p);  // ghost exchange left only the read entries valid
  if (gy_.use) GatherYFull(ybest_.p);
  // x | y | lambda staged back-to-back in one pinned buffer with a single
  // synchronisation; the stage-to-caller copies then run side by side.
  {
    double* hs = HostStage(static_cast<size_t>(2 * n_ + m_));
    double* ds = DevStage();
    auto stage = [&](const double* dev, const double* scale, const DArray<int32_t>& pad, double* h, int64_t k) {
      if (!k) return;
      k_unpermute<<<ew_grid(k), kEw, 0, st_>>>(dev, scale, pad.p, ds, k);
      PDHG_CUDA(cudaMemcpyAsync(h, ds, k * sizeof(double), cudaMemcpyDeviceToHost, st_));
    };
    if (out->x) stage(xbest_.p, cs_.p, pad_c_, hs, n_);
    if (out->y) stage(ybest_.p, rs_.p, pad_r_, hs + n_, m_);
    if (out->lambda) {
      for (Shard& h : shards_) {
        const int64_t c = h.coff;
        run_pass(h.csc, OpLambda{ybest_.p, c_o_.p + c, l_o_.p + c, u_o_.p + c, cs_.p + c, nvec_.p + c}, RedSlots{},
                 st_);
      }
      GatherXFull(nvec_.p);
      stage(nvec_.p, nullptr, pad_c_, hs + n_ + m_, n_);
    }
    Sync();
    std::thread ty;
    if (out->y && m_) ty = std::thread([&] { CopyOut(out->y, hs + n_, m_); });
    std::thread tl;
    if (out->lambda && n_) tl = std::thread([&] { CopyOut(out->lambda, hs + n_ + m_, n_); });
    if (out->x && n_) CopyOut(out->x, hs, n_);
    if (ty.joinable()) ty.join();
    if (tl.joinable()) tl.join();
  }
  PDHG_CUDA(cudaEventRecord(ev_[1], st_));  // after the copy-out, as before: the solve's whole time
  Sync();
  float ms = 0.f;
  PDHG_CUDA(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
  last_ms_ = ms;
  last_launches_ = launches_ + 3 + launches_csc();
  out->status = status;
  out->report = best_rep;
  out->iterations = iters;
  out->restarts = restarts;
  out->solve_seconds = secs();
  out->scaling_seconds = scaling_s_;
  if (std::getenv("PDHG_TRACE"))
    std::fprintf(stderr,
                 "[pdhg] solve %.4fs: opnorm %.4fs | loop %.4fs (%lld its, %lld checks, host-side check wait %.4fs) "
                 "| finish %.4fs | device %.4fs | graphs %zu\n",
                 out->solve_seconds, t_opnorm, t_loop - t_opnorm, (long long)iters, (long long)nchecks, t_checks,
                 out->solve_seconds - t_loop, ms * 1e-3, graphs_.size() + loops_.size());
}

// EstimateOpNorm (solver.cpp:84-110) with the host start vector drawn from the
// same libstdc++ engines as the reference (original column order). Per step:
// K-CSR passes (gather u) -> all-gather kv -> K-CSC passes with sum(u^2)
// partials -> normalisation from the shard/rank sum -> all-gather u.
double Session::OpNorm(int iters, uint64_t seed) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  if (nnz_ == 0) return 0.0;
  // Scratch: x_[1] and kx_[1] are free until the loop starts.
  double* u = x_[1].p;
  double* kv = kx_[1].p;
  const int64_t ns = static_cast<int64_t>(shards_.size());
  const bool single = shards_.size() == 1 && !nccl();
  launches_ += static_cast<int64_t>(iters) * (launches_csr() + launches_csc() + (single ? 1 : ns + (ns > 1) + 1)) +
               launches_csr() + ns + (ns > 1);
  // Power steps run as captured graphs per session (a 100-step graph costs
  // more to instantiate than it saves for a one-shot solve; kPowerSteps-step
  // graphs do not); the final K u pass is launched directly.
  auto step = [&] {
    for (Shard& h : shards_) run_pass(h.csr, OpPowerStep<false>{u, scal_.p, 1, kv + h.roff}, RedSlots{}, fork_);
    GatherY(kv);
    for (size_t k = 0; k < shards_.size(); ++k) {
      Shard& h = shards_[k];
      run_pass(h.csc, OpPowerStep<true>{kv, scal_.p, 0, u + h.coff}, RedSlots{h.red[1].p}, fork_);
      if (single)  // the reduction and the normalisation in one launch
        k_reduce_power_norm<<<1, kBlock, 0, st_>>>(h.red[1].p, h.csc.parts(), red_out_.p, scal_.p);
      else
        k_reduce_tiles<<<1, kBlock, 0, st_>>>(h.red[1].p, nullptr, h.csc.parts(), 1, red_out_.p + k * kPack);
    }
    if (!single) {
      SumPacks(1);
      k_power_norm<<<1, 1, 0, st_>>>(red_out_.p, scal_.p);
    }
    GatherX(u);
  };
  // kPowerSteps steps per graph (PDHG_POWER_GRAPH_STEPS; 4 measured equal to
  // 1 on transport, so 1), single-step graph for the remainder.
  auto capture = [&](int steps, cudaGraphExec_t* exec) {
    cudaGraph_t graph;
    PDHG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    for (int s = 0; s < steps; ++s) step();
    PDHG_CUDA(cudaStreamEndCapture(st_, &graph));
    PDHG_CUDA(cudaGraphInstantiate(exec, graph, 0));
    cudaGraphDestroy(graph);
  };
  static const int kPowerSteps = [] {
    const char* e = std::getenv("PDHG_POWER_GRAPH_STEPS");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  const bool graphs = comm_->graphs();  // loopback transport: eager steps
  const int many = graphs ? iters / kPowerSteps : 0, rest = graphs ? iters % kPowerSteps : 0;
  if (many && !power_graph_) capture(kPowerSteps, &power_graph_);
  if (rest && !power_graph1_) capture(1, &power_graph1_);
  // The graphs never read the start vector's values, so they are captured
  // first, while the host thread may still be drawing it.
  // Start vector (solver.cpp:88-97): drawn on a host thread while the
  // session was being built (upload, CSC, scaling) for the seed the session
  // was created with; another seed is drawn here.
  const char* tenv = std::getenv("PDHG_TRACE");
  const bool fine = tenv && tenv[0] == '2';
  const double tj0 = fine ? now_s() : 0.0;
  if (fine) Sync();
  const double tj1 = fine ? now_s() : 0.0;
  if (start_.joinable()) start_.join();
  if (start_seed_ != seed || !start_host_) DrawStart(seed);
  if (fine)
    std::fprintf(stderr, "[pdhg]   opnorm graphs captured %.4fs, start-vector wait %.4fs\n", tj1 - tj0,
                 now_s() - tj1);
  double* v = start_host_;  // pinned: ToInternal copies it straight to the device
  double vnorm = start_norm_;
  if (vnorm == 0.0) {
    v[0] = 1.0;
    vnorm = 1.0;
  }
  PDHG_CUDA(cudaMemsetAsync(kv, 0, mp_ * sizeof(double), st_));
  ToInternal(v, pad_c_, u, n_, np_);
  Scalars sc{};
  sc.pw_norm = vnorm;
  set_steps(sc);
    PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  trace_graph("power", many);
  for (int it = 0; it < many; ++it) PDHG_CUDA(cudaGraphLaunch(power_graph_, st_));
  for (int it = 0; it < rest; ++it) PDHG_CUDA(cudaGraphLaunch(power_graph1_, st_));
  if (!graphs)
    for (int it = 0; it < iters; ++it) step();
  for (size_t k = 0; k < shards_.size(); ++k) {
    Shard& h = shards_[k];
    run_pass(h.csr, OpPowerStep<true>{u, scal_.p, 1, kv + h.roff}, RedSlots{h.red[0].p}, fork_);
    k_reduce_tiles<<<1, kBlock, 0, st_>>>(h.red[0].p, nullptr, h.csr.parts(), 1, red_out_.p + k * kPack);
  }
  SumPacks(1);
  check_launch("power iteration");
  double sum = 0.0;
  Scalars hs{};
  PDHG_CUDA(cudaMemcpyAsync(&sum, red_out_.p, sizeof(double), cudaMemcpyDeviceToHost, st_));
  PDHG_CUDA(cudaMemcpyAsync(&hs, scal_.p, sizeof(Scalars), cudaMemcpyDeviceToHost, st_));
  Sync();
  if (hs.pw_zero) return 0.0;
  return std::sqrt(sum);
}

// n draws of std::normal_distribution(0,1) over std::mt19937_64(seed) and
// the sequential sum of squares (solver.cpp:88-97), on a host thread that
// overlaps session setup; the draw itself is the pipelined bit-identical
// replica of normal_rng.h (engine on this thread, transforms on workers).
void Session::DrawStart(uint64_t seed) {
  if (!start_host_) start_host_ = static_cast<double*>(pinned_get(n_ * sizeof(double), &start_host_bytes_));
  // Bit-identical to the sequential draw; engine on this thread, transforms
  // on workers (normal_rng.h).
  const int hw = static_cast<int>(std::thread::hardware_concurrency());
  NormalVector(seed, n_, start_host_, n_ >= (int64_t(1) << 17) ? std::min(std::max(hw, 1), 16) : 1);
  double acc = 0.0;
  for (int64_t j = 0; j < n_; ++j) acc += start_host_[j] * start_host_[j];
  start_norm_ = std::sqrt(acc);
  start_seed_ = seed;
}

// ============================================================ kernel probes
void Session::Scaling(double* rs, double* cs) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  ToHost(rs_.p, nullptr, pad_r_, rs, m_);
  ToHost(cs_.p, nullptr, pad_c_, cs, n_);
}

void Session::ScaledProblem(double* kv, double* c, double* l, double* u, double* q) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  if (kv && nnz_) {
    if (nccl()) throw Error(PDHG_INVALID_ARGUMENT, "scaled values are only available when all shards are local");
    std::vector<int32_t> hp(static_cast<size_t>(m_) + 1);
    PDHG_CUDA(cudaMemcpyAsync(hp.data(), ptr0_.p, (m_ + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st_));
    Sync();
    DArray<double> tmp;
    tmp.alloc(nnz_);
    for (Shard& h : shards_) {
      const int64_t k0 = hp[row_begin_[h.block]], k1 = hp[row_begin_[h.block + 1]];
      if (k1 > k0)
        k_values_orig<<<ew_grid(k1 - k0), kEw, 0, st_>>>(ptr0_.p, m_, k0, k1, pad_r_.p, h.roff, h.csr.ptr,
                                                          h.csr.val, tmp.p);
    }
    PDHG_CUDA(cudaMemcpyAsync(kv, tmp.p, nnz_ * sizeof(double), cudaMemcpyDeviceToHost, st_));
    Sync();
  }
  ToHost(c_s_.p, nullptr, pad_c_, c, n_);
  ToHost(l_s_.p, nullptr, pad_c_, l, n_);
  ToHost(u_s_.p, nullptr, pad_c_, u, n_);
  ToHost(q_s_.p, nullptr, pad_r_, q, m_);
}

void Session::Spmv(int transpose, const double* in, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  const int64_t nin = transpose ? m_ : n_, nout = transpose ? n_ : m_;
  const int64_t pin = transpose ? mp_ : np_, pout = transpose ? np_ : mp_;
  DArray<double> a, b;
  a.alloc(std::max<int64_t>(pin, 1));
  b.alloc(std::max<int64_t>(pout, 1));
  PDHG_CUDA(cudaMemsetAsync(b.p, 0, std::max<int64_t>(pout, 1) * sizeof(double), st_));
  ToInternal(in, transpose ? pad_r_ : pad_c_, a.p, nin, pin);
  for (Shard& h : shards_) run_pass(transpose ? h.csc : h.csr, OpSpmv{a.p, b.p + (transpose ? h.coff : h.roff)},
                                    RedSlots{}, st_);
  if (transpose) GatherXFull(b.p);
  else GatherYFull(b.p);
  check_launch("spmv");
  ToHost(b.p, nullptr, transpose ? pad_c_ : pad_r_, out, nout);
}

// RowInfNorms / ColInfNorms / RowPowerSums / ColPowerSums
// (sparse_matrix.cpp:166-204) of this session's K_s, original order.
void Session::SegmentNorms(int columns, int power, double p, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  const int64_t nout = columns ? n_ : m_, pout = columns ? np_ : mp_;
  DArray<double> b;
  b.alloc(std::max<int64_t>(pout, 1));
  PDHG_CUDA(cudaMemsetAsync(b.p, 0, std::max<int64_t>(pout, 1) * sizeof(double), st_));
  const int mode = p == 0.0 ? 0 : (p == 1.0 ? 1 : (p == 2.0 ? 2 : 3));
  for (Shard& h : shards_) {
    const Layout& L = columns ? h.csc : h.csr;
    double* o = b.p + (columns ? h.coff : h.roff);
    if (power) run_pass(L, OpRawNorm<false>{p, mode, o}, RedSlots{}, st_);
    else run_pass(L, OpRawNorm<true>{p, mode, o}, RedSlots{}, st_);
  }
  if (columns) GatherXFull(b.p);
  else GatherYFull(b.p);
  check_launch("segment norms");
  ToHost(b.p, nullptr, columns ? pad_c_ : pad_r_, out, nout);
}

// Mean device time of the two fused step kernels (all local shards, gathers
// included) and of a graph-launched 64-iteration block, on the solver stream.
void Session::TimeKernels(int iters, double* ms_primal, double* ms_dual, double* ms_iter) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  Scalars sc{};
  sc.eta = 1e-3;
  sc.omega = 1.0;
  sc.inner_base = 1.0;
  sc.lb = lb_;
  sc.ub = ub_;
  set_steps(sc);
    PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  k_clamp0<<<ew_grid(np_), kEw, 0, st_>>>(l_s_.p, u_s_.p, x_[0].p, np_);
  if (mp_) PDHG_CUDA(cudaMemsetAsync(y_[0].p, 0, mp_ * sizeof(double), st_));
  for (Shard& h : shards_) run_pass(h.csr, OpSpmv{x_[0].p, kx_[0].p + h.roff}, RedSlots{}, fork_);
  cudaEvent_t e0, e1, e2;
  PDHG_CUDA(cudaEventCreate(&e0));
  PDHG_CUDA(cudaEventCreate(&e1));
  PDHG_CUDA(cudaEventCreate(&e2));
  for (int w = 0; w < 3; ++w) LaunchStep(w & 1, w, false);
  Sync();
  float t_p = 0, t_d = 0, t_i = 0;
  // Per-kernel times: back-to-back launches of ONE kernel, without
  // programmatic overlap between them (that overlap belongs to the
  // primal -> dual chain, measured by the graph-launched block below).
  pdl_suspended() = true;
  PDHG_CUDA(cudaEventRecord(e0, st_));
  for (int i = 0; i < iters; ++i) {
    for (Shard& h : shards_) LaunchPrimal(h, 0, 1, i + 1, false);
    GatherX(x_[1].p);
  }
  PDHG_CUDA(cudaEventRecord(e1, st_));
  for (int i = 0; i < iters; ++i) {
    for (Shard& h : shards_) {
      const int64_t o = h.roff;
      run_pass(h.csr,
               OpDual<false>{x_[1].p, y_[0].p + o, y_[1].p + o, ybar_.p + o, kx_[0].p + o, kx_[1].p + o, q_s_.p + o,
                             h.rk, scal_.p, i + 1},
               RedSlots{}, fork_);
    }
    GatherY(y_[1].p);
  }
  PDHG_CUDA(cudaEventRecord(e2, st_));
  pdl_suspended() = false;
  PDHG_CUDA(cudaEventSynchronize(e2));
  PDHG_CUDA(cudaEventElapsedTime(&t_p, e0, e1));
  PDHG_CUDA(cudaEventElapsedTime(&t_d, e1, e2));
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

// Cold-cache kernel times without launch overhead: three captured graphs of
// `reps` repetitions -- (L2 sweep, primal), (L2 sweep, dual), (L2 sweep,
// primal, dual) -- and one of the sweep alone; each kernel's time is its
// graph's time minus the sweep graph's, per repetition. Inside a graph the
// launches are back to back as in the solve loop, but every kernel starts
// with L2 holding none of its data (and the write-back of the previous
// kernel's dirty lines is charged to the sweep). Events on the session
// stream bracket each graph launch; the median of 5 launches is kept.
void Session::TimeKernelsCold(int iters, double* ms_primal, double* ms_dual, double* ms_iter) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  Scalars sc{};
  sc.eta = 1e-3;
  sc.omega = 1.0;
  sc.inner_base = 1.0;
  sc.lb = lb_;
  sc.ub = ub_;
  set_steps(sc);
    PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  k_clamp0<<<ew_grid(np_), kEw, 0, st_>>>(l_s_.p, u_s_.p, x_[0].p, np_);
  if (mp_) PDHG_CUDA(cudaMemsetAsync(y_[0].p, 0, mp_ * sizeof(double), st_));
  for (Shard& h : shards_) run_pass(h.csr, OpSpmv{x_[0].p, kx_[0].p + h.roff}, RedSlots{}, fork_);
  for (int w = 0; w < 3; ++w) LaunchStep(w & 1, w, false);
  SweepL2();  // allocates the sweep buffer outside any capture
  Sync();
  const int reps = std::max(1, std::min(iters, 64));
  auto primal = [&](int i) {
    for (Shard& h : shards_) LaunchPrimal(h, 0, 1, i + 1, false);
    GatherX(x_[1].p);
  };
  auto dual = [&](int i) {
    for (Shard& h : shards_) {
      const int64_t o = h.roff;
      run_pass(h.csr,
               OpDual<false>{x_[1].p, y_[0].p + o, y_[1].p + o, ybar_.p + o, kx_[0].p + o, kx_[1].p + o, q_s_.p + o,
                             h.rk, scal_.p, i + 1},
               RedSlots{}, fork_);
    }
    GatherY(y_[1].p);
  };
  cudaEvent_t e0, e1;
  PDHG_CUDA(cudaEventCreate(&e0));
  PDHG_CUDA(cudaEventCreate(&e1));
  auto graph_ms = [&](auto&& body) {
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    PDHG_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < reps; ++i) {
      SweepL2();
      body(i);
    }
    PDHG_CUDA(cudaStreamEndCapture(st_, &graph));
    PDHG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    PDHG_CUDA(cudaGraphLaunch(exec, st_));  // warm-up launch
    std::vector<double> t;
    for (int k = 0; k < 5; ++k) {
      PDHG_CUDA(cudaEventRecord(e0, st_));
      PDHG_CUDA(cudaGraphLaunch(exec, st_));
      PDHG_CUDA(cudaEventRecord(e1, st_));
      PDHG_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      PDHG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      t.push_back(ms);
    }
    cudaGraphExecDestroy(exec);
    std::sort(t.begin(), t.end());
    return t[2] / reps;
  };
  const double t_sweep = graph_ms([](int) {});
  const double t_p = graph_ms(primal);
  const double t_d = graph_ms(dual);
  const double t_i = graph_ms([&](int i) {
    primal(i);
    dual(i);
  });
  *ms_primal = std::max(t_p - t_sweep, 0.0);
  *ms_dual = std::max(t_d - t_sweep, 0.0);
  *ms_iter = std::max(t_i - t_sweep, 0.0);
  launches_ = 0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void Session::RunBlock(int iters, bool profiler_range) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  Scalars sc{};
  sc.eta = 1e-3;
  sc.omega = 1.0;
  sc.inner_base = 1.0;
  sc.lb = lb_;
  sc.ub = ub_;
  set_steps(sc);
    PDHG_CUDA(cudaMemcpyAsync(scal_.p, &sc, sizeof(Scalars), cudaMemcpyHostToDevice, st_));
  k_clamp0<<<ew_grid(np_), kEw, 0, st_>>>(l_s_.p, u_s_.p, x_[0].p, np_);
  if (mp_) PDHG_CUDA(cudaMemsetAsync(y_[0].p, 0, mp_ * sizeof(double), st_));
  for (Shard& h : shards_) run_pass(h.csr, OpSpmv{x_[0].p, kx_[0].p + h.roff}, RedSlots{}, fork_);
  const int blk = 64;
  RunSteps(0, blk, false);  // instantiate the block graph outside the range
  Sync();
  if (profiler_range) PDHG_CUDA(cudaProfilerStart());
  for (int done = 0; done < iters; done += blk) RunSteps(0, std::min(blk, iters - done), false);
  Sync();
  if (profiler_range) PDHG_CUDA(cudaProfilerStop());
}

void Session::SweepL2() {
  int l2 = 0;
  PDHG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device_));
  const size_t bytes = std::max<size_t>(2 * static_cast<size_t>(l2), 64u << 20);
  if (sweep_.n < bytes) {
    sweep_.alloc(bytes + 64);
    PDHG_CUDA(cudaMemsetAsync(sweep_.p, 0, bytes + 64, st_));
  }
  int sms = 0;
  PDHG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
  k_l2_sweep<<<4 * sms, 512, 0, st_>>>(reinterpret_cast<const double2*>(sweep_.p), bytes / 16,
                                       reinterpret_cast<double*>(sweep_.p + bytes));
  check_launch("l2 sweep");
}

// Check cost probe: distinct current / average iterates so both halves of
// every check pass are live, as in the loop.
void Session::TimeCheck(int iters, double* ms_device, double* ms_wall) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  for (int w = 0; w < 2; ++w) LaunchCheck(x_[0].p, y_[0].p, x_[1].p, y_[1].p, kx_[0].p);
  Sync();
  cudaEvent_t e0, e1;
  PDHG_CUDA(cudaEventCreate(&e0));
  PDHG_CUDA(cudaEventCreate(&e1));
  PDHG_CUDA(cudaEventRecord(e0, st_));
  for (int i = 0; i < iters; ++i) LaunchCheck(x_[0].p, y_[0].p, x_[1].p, y_[1].p, kx_[0].p);
  PDHG_CUDA(cudaEventRecord(e1, st_));
  PDHG_CUDA(cudaEventSynchronize(e1));
  float t = 0.f;
  PDHG_CUDA(cudaEventElapsedTime(&t, e0, e1));
  *ms_device = t / iters;
  CheckOut ck;
  const double w0 = now_s();
  for (int i = 0; i < iters; ++i) {
    LaunchCheck(x_[0].p, y_[0].p, x_[1].p, y_[1].p, kx_[0].p);
    ReadCheck(&ck);
  }
  *ms_wall = (now_s() - w0) * 1e3 / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void Session::UnitPrimal(const double* x, const double* y, double eta, double omega, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  DArray<double> dx, dy, dout;
  dx.alloc(std::max<int64_t>(np_, 1));
  dy.alloc(std::max<int64_t>(mp_, 1));
  dout.alloc(std::max<int64_t>(np_, 1));
  ToInternal(x, pad_c_, dx.p, n_, np_);
  ToInternal(y, pad_r_, dy.p, m_, mp_);
  for (Shard& h : shards_) {
    const int64_t o = h.coff;
    run_pass(h.csc, OpUnitPrimal{dy.p, dx.p + o, c_s_.p + o, l_s_.p + o, u_s_.p + o, eta / omega, dout.p + o},
             RedSlots{}, st_);
  }
  GatherXFull(dout.p);
  check_launch("primal step");
  ToHost(dout.p, nullptr, pad_c_, out, n_);
}

// ComputeResiduals (kkt.cpp:143-145) of (x, y) on this session's problem in
// its ORIGINAL space: one check pass with the point standing in for the
// average, the "original" half of the pack.
void Session::Residuals(const double* x, const double* y, pdhg_report* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  ToInternal(x, pad_c_, x_[0].p, n_, np_);
  ToInternal(y, pad_r_, y_[0].p, m_, mp_);
  // The check works in the scaled space: map the original point into it.
  k_div<<<ew_grid(np_), kEw, 0, st_>>>(x_[0].p, cs_.p, x_[0].p, np_);
  k_div<<<ew_grid(mp_), kEw, 0, st_>>>(y_[0].p, rs_.p, y_[0].p, mp_);
  GatherXFull(x_[0].p);
  GatherYFull(y_[0].p);
  for (Shard& h : shards_) run_pass(h.csr, OpSpmv{x_[0].p, kx_[0].p + h.roff}, RedSlots{}, st_);
  Copy(xstart_.p, x_[0].p, np_);
  Copy(ystart_.p, y_[0].p, mp_);
  LaunchCheck(x_[0].p, y_[0].p, x_[0].p, y_[0].p, kx_[0].p);
  CheckOut ck;
  ReadCheck(&ck);
  *out = MakeReport(ck.row[kPrO], ck.col[kDuO], ck.col[kBdO], ck.col[kCxO], ck.row[kQyO], offset_, q_norm_o_,
                    c_norm_o_);
}

// DeriveLambda (kkt.cpp:127-141) for an original-space y.
void Session::Lambda(const double* y, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  ToInternal(y, pad_r_, y_[0].p, m_, mp_);
  k_div<<<ew_grid(mp_), kEw, 0, st_>>>(y_[0].p, rs_.p, y_[0].p, mp_);
  GatherYFull(y_[0].p);
  for (Shard& h : shards_) {
    const int64_t c = h.coff;
    run_pass(h.csc, OpLambda{y_[0].p, c_o_.p + c, l_o_.p + c, u_o_.p + c, cs_.p + c, nvec_.p + c}, RedSlots{}, st_);
  }
  GatherXFull(nvec_.p);
  check_launch("lambda");
  ToHost(nvec_.p, nullptr, pad_c_, out, n_);
}

void Session::UnitDual(const double* xn, const double* xo, const double* y, double eta, double omega, double* out) {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
  DArray<double> a, b, ext, dy, dout;
  a.alloc(std::max<int64_t>(np_, 1));
  b.alloc(std::max<int64_t>(np_, 1));
  ext.alloc(std::max<int64_t>(np_, 1));
  dy.alloc(std::max<int64_t>(mp_, 1));
  dout.alloc(std::max<int64_t>(mp_, 1));
  ToInternal(xn, pad_c_, a.p, n_, np_);
  ToInternal(xo, pad_c_, b.p, n_, np_);
  ToInternal(y, pad_r_, dy.p, m_, mp_);
  k_reflect<<<ew_grid(np_), kEw, 0, st_>>>(a.p, b.p, ext.p, np_);
  for (Shard& h : shards_) {
    const int64_t o = h.roff;
    run_pass(h.csr, OpUnitDual{ext.p, dy.p + o, q_s_.p + o, h.rk, eta * omega, dout.p + o}, RedSlots{}, st_);
  }
  GatherYFull(dout.p);
  check_launch("dual step");
  ToHost(dout.p, nullptr, pad_r_, out, m_);
}

// Evict the working set between benchmark steps: write 2x the L2 capacity.
void Session::FlushL2() {
  PDHG_CUDA(cudaSetDevice(device_));
  AllocScope scope(st_);
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
  s->csr_tiles = parts_csr();
  s->csc_tiles = parts_csc();
  s->device_bytes = arena_.bytes;
  s->upload_seconds = upload_s_;
  s->scaling_seconds = scaling_s_;
  s->device = device_;
  s->l2_resident = l2_resident_ ? 1 : 0;
  s->world = world_;
  s->local_shards = static_cast<int32_t>(shards_.size());
  s->rank = rank_;
  s->uniform_bounds = bnd_;
  // Uniform only if every local shard's whole layout is one uniform class S.
  auto all_uniform = [&](bool csr) {
    int len = -1;
    for (const Shard& h : shards_) {
      const Layout& L = csr ? h.csr : h.csc;
      if (L.nseg == 0) continue;
      if (L.s1 != L.nseg || L.s_len == 0 || L.s_u != L.s1 || (len >= 0 && L.s_len != len)) return 0;
      len = L.s_len;
    }
    return len > 0 ? len : 0;
  };
  s->csr_uniform_len = all_uniform(true);
  s->csc_uniform_len = all_uniform(false);
  s->csr_split = shards_.size() == 1 ? shards_[0].csr.split_w : 0;
  s->block_kernel = persist_ ? 1 : 0;
}

void Session::Blocks(int64_t* row_begin, int64_t* col_begin) const {
  std::copy(row_begin_.begin(), row_begin_.end(), row_begin);
  std::copy(col_begin_.begin(), col_begin_.end(), col_begin);
}

}  // namespace pdhg
