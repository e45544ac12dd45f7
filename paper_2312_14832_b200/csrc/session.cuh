// Resident solve session: the scaled stacked problem in HBM plus all PDHG
// state. Host orchestration mirrors SolveLoop (reference solver.cpp:203-517).
//
// Sharding: K is split into `world` contiguous row blocks (the
// CSR side, K x) and column blocks (the CSC side, K^T y), balanced by
// nonzeros. A Shard owns one row block and one column block; a session holds
// either every shard (world = 1, or the in-process multi-shard mode) or the
// one shard of its rank (one process per GPU, NCCL exchanges). Vectors live in
// the padded index space of comm.cuh; full copies of x and y are rebuilt by
// one all-gather after each half-step.
#pragma once

#include <chrono>
#include <functional>
#include <memory>
#include <thread>
#include <vector>

#include "../../include/pdhg.h"
#include "comm.cuh"
#include "darray.cuh"
#include "engine.cuh"
#include "persist.cuh"

namespace pdhg {

struct CheckOut;     // host mirror of the check reductions
struct DecideState;  // device-side check decisions (decide.cuh)

// How K is distributed (pdhg_shard_spec in include/pdhg.h).
struct ShardSpec {
  int world = 1;                  // number of shards
  int rank = 0;                   // this process's shard (NCCL mode)
  int local = 1;                  // shards held by this session: 1 or world
  const void* nccl_id = nullptr;  // 128-byte ncclUniqueId (NCCL mode)
};

class Session {
 public:
  Session(const pdhg_lp& lp, const pdhg_params& prm, int device, const ShardSpec& spec = ShardSpec{},
          bool skip_pc = false);
  ~Session();

  void Solve(const pdhg_params& prm, pdhg_eval_cb cb, void* user, pdhg_result* out);
  void Scaling(double* rs, double* cs);
  void ScaledProblem(double* kv, double* c, double* l, double* u, double* q);
  void Spmv(int transpose, const double* in, double* out);
  void SegmentNorms(int columns, int power, double p, double* out);
  double OpNorm(int iters, uint64_t seed);
  // True when `prm` asks for the scaling this session applied at creation
  // (solve params cannot rescale a resident problem).
  bool SameScaling(const pdhg_params& prm) const;
  void TimeKernels(int iters, double* ms_primal, double* ms_dual, double* ms_iter);
  // Cold-cache per-launch times: L2 swept clean before every launch, CUDA
  // events bracketing each launch (primal, dual, and one whole iteration).
  void TimeKernelsCold(int iters, double* ms_primal, double* ms_dual, double* ms_iter);
  // `iters` plain PDHG steps as graph-launched blocks (check_every-step
  // graphs), optionally inside cudaProfilerStart/Stop: an ncu range-replay
  // target whose DRAM counters include the write-backs of each iteration.
  void RunBlock(int iters, bool profiler_range);
  void TimeCheck(int iters, double* ms_device, double* ms_wall);
  void Stats(pdhg_session_stats* s) const;
  void Blocks(int64_t* row_begin, int64_t* col_begin) const;
  void GhostCounts(int64_t* x_counts, int64_t* y_counts, int32_t* use) const;
  void UnitPrimal(const double* x, const double* y, double eta, double omega, double* out);
  void Residuals(const double* x, const double* y, pdhg_report* out);
  void Lambda(const double* y, double* out);
  void UnitDual(const double* xn, const double* xo, const double* y, double eta, double omega, double* out);
  int device() const { return device_; }
  void FlushL2();
  void SweepL2();  // read a 2x L2 buffer: L2 left clean and cold
  double last_device_ms() const { return last_ms_; }
  int64_t last_launches() const { return last_launches_; }

 private:
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int steps = 0;
    int parity = 0;
    bool adapt = false;
  };
  // Storage of one permuted layout (CSR of a row block or CSC of a column block).
  struct Store {
    DArray<int32_t> ptr, idx;
    DArray<double> val;
    DArray<int32_t> part[4];  // tile_begin, tile_seg, head_first, tail_owner (long class)
    DArray<double> head, tail;
    DArray<unsigned> cnt;
    DArray<uint8_t> rm;  // staged class-S segment-order warp flags
    DArray<int32_t> order;  // tile execution order (long class, gather sweep)
    DArray<int32_t> lo_ptr, lo_idx, hi_ptr, hi_idx;  // gather-window split of class S
    DArray<double> lo_val, hi_val, split_part;
    DArray<uint8_t> lo_rm, hi_rm;
  };
  struct Shard {
    int block = 0;
    int64_t roff = 0, coff = 0;  // padded offsets of the block's rows / columns
    int64_t rows = 0, cols = 0;  // block sizes
    Layout csr, csc;             // segment s of the block <-> vector index off + s
    Store csr_st, csc_st;
    RowKind rk{};                // equality rows of the block (local order)
    DArray<double> red[2];       // reduction slots: [0] CSR passes, [1] CSC passes
  };
  static constexpr int kPack = 32;  // doubles per reduction pack (>= kRowRed + kColRed)

  void Upload(const pdhg_lp& lp, DArray<int32_t>& ptr0, DArray<int32_t>& idx0, DArray<double>& val0);
  void Permute(const DArray<int32_t>& ptr0, const DArray<int32_t>& idx0, const DArray<double>& val0);
  void ComputeScaling(const pdhg_params& prm);
  void PartitionLong(Layout& L, Store& S);
  void DeviceNorms();
  void Sync();
  void LaunchStep(int parity, int j, bool adapt);
  template <bool kAdapt, int kBnd>
  void PrimalPass(Shard& h, int a, int b, int j);
  void LaunchPrimal(Shard& h, int a, int b, int j, bool adapt);
  void UniformBounds();
  void BuildSplit(Layout& L, Store& S);
  void DrawStart(uint64_t seed);
  void RunSteps(int parity, int count, bool adapt);
  void RunBlock(int parity, int count, bool adapt, bool check, int slot);
  void RunChecked(int parity, int count, bool adapt = false);
  // Persistent block kernel (persist.cuh): `count` iterations in one launch.
  bool PersistOk() const;
  void LaunchBlock(int parity, int count);
  template <int kBnd>
  void LaunchBlockT(int parity, int count);
  void RunDeviceLoop(int parity, int count);
  void LaunchCheck(const double* x, const double* y, const double* xb, const double* yb, const double* kx,
                   const Scalars* guard = nullptr, bool branches = false);
  void ReadCheck(CheckOut* out);
  void SumPacks(int n, const Scalars* guard = nullptr);  // shard packs -> red_out_[0..n), all ranks
  void Copy(double* dst, const double* src, size_t n);
  void ToInternal(const double* host, const DArray<int32_t>& pad, double* dev, int64_t n, int64_t padded);
  void ToHost(const double* dev, const double* scale, const DArray<int32_t>& pad, double* host, int64_t n);
  double* DevStage();
  double* HostStage(size_t at_least = 0);
  // Gathers for the next matrix pass (ghost entries only when the plan says
  // so) and full gathers for values leaving the session.
  // PDHG_LOOP_TRACE=1: graph replays of a multi-rank session (collectives
  // inside graphs run once per replay without a host call).
  void trace_graph(const char* what, int64_t n) const {
    static const bool on = [] {
      const char* e = std::getenv("PDHG_LOOP_TRACE");
      return e && e[0] == '1';
    }();
    if (on && world_ > 1) std::fprintf(stderr, "[loop] rank %d graph %s x%lld\n", rank_, what, (long long)n);
  }
  void GatherX(double* v) { comm_->Exchange(v, gx_, st_); }
  void GatherY(double* v) { comm_->Exchange(v, gy_, st_); }
  void GatherXFull(double* v) { comm_->AllGather(v, pn_, st_); }
  void GatherYFull(double* v) { comm_->AllGather(v, pm_, st_); }
  struct GhostStore {
    DArray<int32_t> send_idx, recv_idx;
    DArray<double> send_buf, recv_buf;
  };
  void BuildGhostPlan(const int32_t* ptr, const int32_t* idx, const std::vector<int64_t>& seg_begin, int64_t nvec,
                      int64_t slice, GhostPlan& plan, GhostStore& store, std::vector<int64_t>& counts);
  bool nccl() const { return !comm_->local(); }
  int parts_csr() const;
  int parts_csc() const;
  int launches_csr() const;
  int launches_csc() const;

  // Owns the session stream and the fork streams / events. Declared first so
  // it is destroyed last, after every DArray member has been released on it.
  struct StreamOwner {
    cudaStream_t st = nullptr;
    Fork fork;
    StreamOwner() = default;
    StreamOwner(const StreamOwner&) = delete;
    StreamOwner& operator=(const StreamOwner&) = delete;
    ~StreamOwner() {
      if (fork.fork) cudaEventDestroy(fork.fork);
      for (int k = 0; k < 3; ++k) {
        if (fork.side[k]) cudaStreamDestroy(fork.side[k]);
        if (fork.join[k]) cudaEventDestroy(fork.join[k]);
      }
      if (st) cudaStreamDestroy(st);
    }
  };
  StreamOwner streams_;
  int device_ = 0;
  bool skip_pc_ = false;  // scaling = Ruiz sweeps only (pdhg_compute_scaling)
  cudaStream_t st_ = nullptr;
  Fork fork_;  // st_ + side streams for parallel class kernels
  Arena arena_;
  int64_t m1_ = 0, m2_ = 0, m_ = 0, n_ = 0, nnz_ = 0;
  double offset_ = 0.0;
  double upload_s_ = 0.0, scaling_s_ = 0.0;
  bool scaled_ = false;
  int ruiz_iters_ = 0;   // scaling config the session was built with
  double pc_alpha_ = 0.0;
  bool l2_resident_ = false;

  // Distribution: blocks in original order, padded slice sizes.
  int world_ = 1, rank_ = 0;
  std::vector<int64_t> row_begin_, col_begin_;
  int64_t pm_ = 0, pn_ = 0;      // padded slice (rows / columns per block)
  int64_t mp_ = 0, np_ = 0;      // padded vector lengths world * pm_, world * pn_
  std::unique_ptr<Comm> comm_;
  std::vector<Shard> shards_;
  DArray<int32_t> pad_r_, pad_c_;  // original row / column -> padded index
  GhostPlan gx_, gy_;               // x pattern (CSR reads), y pattern (CSC reads)
  GhostStore gxs_, gys_;
  std::vector<int64_t> ghost_counts_x_, ghost_counts_y_;  // [reader block][source block] entries
  DArray<int32_t> ptr0_;           // original CSR row_ptr (probe only)

  // Problem vectors (padded order): scaled (loop) and original (termination).
  DArray<double> c_s_, l_s_, u_s_, c_o_, l_o_, u_o_, cs_;  // np_
  DArray<double> q_s_, q_o_, rs_;                          // mp_
  double c_norm_s_ = 0, q_norm_s_ = 0, c_norm_o_ = 0, q_norm_o_ = 0;
  int bnd_ = 0;               // uniform-bound bits (UniformBounds)
  bool persist_ = false;      // step blocks as one persistent launch (PersistOk, PDHG_PERSIST)
  const int32_t* halt_ptr_ = nullptr;  // step Ops' halt flag while the pipelined loop queues blocks
  DArray<unsigned> gbar_;     // its grid-barrier counter
  int modal_col_len_ = 0;     // columns: modal class-S length placed first (Layout::s_u), or 0
  bool bnd_all_ = false;      // original bounds equal the common scaled ones too
  double lb_ = 0.0, ub_ = 0.0;

  // Iterates (ping-pong x/y/kx), averages, loop start, best, scratch.
  DArray<double> x_[2], xbar_, xstart_, xbest_, nvec_;            // np_
  DArray<double> y_[2], ybar_, ystart_, ybest_, kx_[2], kxavg_;  // mp_
  DArray<Scalars> scal_;
  DArray<double> red_out_;  // per-shard packs; pack 0 holds the reduced result
  double* host_red_ = nullptr;  // pinned (darray.cuh pinned cache)
  size_t host_red_bytes_ = 0;
  DArray<double> dstage_;       // max(m, n) device staging
  double* hstage_ = nullptr;    // max(m, n) pinned host staging
  size_t hstage_n_ = 0, hstage_bytes_ = 0;

  // Power-iteration start vector, drawn on a host thread during setup.
  std::thread start_;
  double* start_host_ = nullptr;  // pinned, n doubles
  size_t start_host_bytes_ = 0;
  uint64_t start_seed_ = ~uint64_t(0);
  double start_norm_ = 0.0;

  // Pipelined loop: device decision state, its pinned host mirrors, events.
  DArray<DecideState> dstate_;
  DecideState* hstate_ = nullptr;
  size_t hstate_bytes_ = 0;
  cudaEvent_t pev_[2] = {nullptr, nullptr};

  std::vector<Graph> graphs_;
  std::vector<Graph> blocks_;  // pipelined-loop block graphs
  std::vector<Graph> loops_;   // device-resident loop graphs (conditional WHILE)
  cudaGraphExec_t power_graph_ = nullptr;   // kPowerSteps EstimateOpNorm steps (OpNorm)
  cudaGraphExec_t power_graph1_ = nullptr;  // one step (remainder)
  DArray<char> flush_;
  DArray<char> sweep_;
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  double last_ms_ = 0.0;
  int64_t launches_ = 0, last_launches_ = 0;
};

}  // namespace pdhg
