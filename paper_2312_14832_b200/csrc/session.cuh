// Resident solve session: the scaled stacked problem in HBM plus all PDHG
// state. Host orchestration mirrors SolveLoop (reference solver.cpp:203-517).
#pragma once

#include <chrono>
#include <functional>
#include <vector>

#include "../../include/pdhg.h"
#include "darray.cuh"
#include "engine.cuh"

namespace pdhg {

struct CheckOut;  // host mirror of the check reductions

class Session {
 public:
  Session(const pdhg_lp& lp, const pdhg_params& prm, int device);
  ~Session();

  void Solve(const pdhg_params& prm, pdhg_eval_cb cb, void* user, pdhg_result* out);
  void Scaling(double* rs, double* cs);
  void ScaledProblem(double* kv, double* c, double* l, double* u, double* q);
  void Spmv(int transpose, const double* in, double* out);
  double OpNorm(int iters, uint64_t seed);
  void TimeKernels(int iters, double* ms_primal, double* ms_dual, double* ms_iter);
  void Stats(pdhg_session_stats* s) const;
  void UnitPrimal(const double* x, const double* y, double eta, double omega, double* out);
  void UnitDual(const double* xn, const double* xo, const double* y, double eta, double omega, double* out);
  int device() const { return device_; }
  void FlushL2();
  double last_device_ms() const { return last_ms_; }
  int64_t last_launches() const { return last_launches_; }

 private:
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int steps = 0;
    int parity = 0;
    bool adapt = false;
  };
  // Storage of one permuted layout (CSR of K or CSC of K).
  struct Store {
    DArray<int32_t> ptr, idx;
    DArray<double> val;
    DArray<int32_t> part[4];  // tile_begin, tile_seg, head_first, tail_owner (long class)
    DArray<double> head, tail;
    DArray<unsigned> cnt;
  };

  void Upload(const pdhg_lp& lp, DArray<int32_t>& ptr0, DArray<int32_t>& idx0, DArray<double>& val0);
  void Permute(const DArray<int32_t>& ptr0, const DArray<int32_t>& idx0, const DArray<double>& val0);
  void ComputeScaling(const pdhg_params& prm);
  void PartitionLong(Layout& L, Store& S);
  void DeviceNorms();
  void Sync();
  void LaunchStep(int parity, int j, bool adapt);
  void RunSteps(int parity, int count, bool adapt);
  void LaunchCheck(const double* x, const double* y, const double* xb, const double* yb, const double* kx);
  void ReadCheck(CheckOut* out);
  void Copy(double* dst, const double* src, size_t n);
  void ToInternal(const double* host, const DArray<int32_t>& perm, double* dev, int64_t n);
  void ToHost(const double* dev, const double* scale, const DArray<int32_t>& inv, double* host, int64_t n);

  int device_ = 0;
  cudaStream_t st_ = nullptr;
  Arena arena_;
  int64_t m1_ = 0, m2_ = 0, m_ = 0, n_ = 0, nnz_ = 0;
  double offset_ = 0.0;
  double upload_s_ = 0.0, scaling_s_ = 0.0;
  bool scaled_ = false;
  bool l2_resident_ = false;

  // K_s in both layouts, rows / columns permuted into length classes.
  Layout csr_, csc_;
  Store csr_st_, csc_st_;
  RowKind rk_{};
  DArray<int32_t> perm_r_, inv_r_, perm_c_, inv_c_;  // new->old, old->new
  DArray<int32_t> ptr0_;                             // original CSR row_ptr (probe only)

  // Problem vectors (permuted order): scaled (loop) and original (termination).
  DArray<double> c_s_, l_s_, u_s_, c_o_, l_o_, u_o_, cs_;  // n
  DArray<double> q_s_, q_o_, rs_;                          // m
  double c_norm_s_ = 0, q_norm_s_ = 0, c_norm_o_ = 0, q_norm_o_ = 0;

  // Iterates (ping-pong x/y/kx), averages, loop start, best, scratch.
  DArray<double> x_[2], xbar_, xstart_, xbest_, nvec_;            // n
  DArray<double> y_[2], ybar_, ystart_, ybest_, kx_[2], kxavg_;  // m
  DArray<Scalars> scal_;
  DArray<double> red_[2], red_out_;
  double* host_red_ = nullptr;  // pinned

  std::vector<Graph> graphs_;
  DArray<char> flush_;
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  double last_ms_ = 0.0;
  int64_t launches_ = 0, last_launches_ = 0;
};

}  // namespace pdhg
