// Device-side check decisions for the pipelined solve loop.
//
// The reference decides at every check on the host thread (solver.cpp:390-428):
// reports -> candidate -> EvaluateAndMaybeFinish (termination, best-by-KKT1)
// -> restart test. Evaluated on the host, every check is a device->host->
// device round trip during which the GPU idles. Here one thread evaluates the
// same decision functions (host_logic.h, compiled for both sides: sqrt /
// fabs / compares only, no FMA -> bit-identical) right after the check
// reductions, copies a new best iterate on the device, and -- for the common
// outcome "keep iterating" -- lets the next, already queued block run
// without any host involvement. Only outcomes that need the host (a restart:
// the primal-weight update uses glibc exp/log, which the device cannot match
// bit for bit; termination; a non-finite iterate) set Scalars::halt, which
// makes every queued kernel return at entry until the host has acted.
// halt: 0 running; 2 set by the check that just ran (its best-iterate copy
// still happens); 1 settled -- everything queued after it is skipped. A
// whole block (steps + check + decision + copy + the D2H of the state) is one
// captured graph, so a check costs no host round trip and no launch gaps.
#pragma once

#include "host_logic.h"
#include "ops.cuh"

namespace pdhg {

enum DecideAction : int32_t {
  kContinue = 0,
  kOptimalCur = 1,
  kOptimalAvg = 2,
  kRestart = 3,
  kNonFinite = 4,
};

struct DecideState {
  // constants of the solve
  double eps, suff, nec, frac;
  double offset, qn_s, cn_s, qn_o, cn_o;
  int32_t restart_enabled;
  int32_t pad0;
  // loop state (device-owned between host interventions)
  double kkt_start, kkt_prev, best_k1;
  int32_t have_best;
  int32_t checks;      // checks evaluated so far (the host verifies its count)
  int64_t iters, inner;
  // device-resident loop (Session::RunDeviceLoop): block length, iteration
  // limit, time budget and the globaltimer deadline derived from it
  int64_t block, iter_limit;
  uint64_t remaining_ns, deadline_ns;
  // outputs of the latest check
  int32_t action, take_cur, best_from, restart_flag;
  double kkt_cand, eta;
  pdhg_report s_cur, o_cur, s_avg, o_avg, last_rep, best_rep;
};

// The block's iterations happened (not skipped): advance the counters the
// host used to push after every block.
__global__ void k_advance(Scalars* sc, DecideState* ds, int count) {
  if (sc->halt) return;
  sc->inner_base += static_cast<double>(count);
  ds->iters += count;
  ds->inner += count;
}

// Check reductions for the pipelined loop (skipped after a halt).
__global__ void k_reduce_two_guarded(const Scalars* sc, const double* t0, int nt0, int n0, const double* t1, int nt1,
                                     int n1, double* out) {
  if (sc->halt) return;
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

// One check's decisions from the reduced pack (row sums then column sums,
// ops.cuh CheckRow / CheckCol layout). Mirrors Session::Solve's host path.
__device__ __forceinline__ void decide(const double* pack, Scalars* sc, DecideState* ds) {
  DecideState& d = *ds;
  const double* row = pack;
  const double* col = pack + kRowRed;
  ++d.checks;
  d.best_from = -1;
  d.restart_flag = 0;
  d.eta = sc->eta;
  if (row[2 * kRowPer] > 0.0 || col[2 * kColPer] > 0.0) {
    d.action = kNonFinite;
    sc->halt = 2;
    return;
  }
  auto reports = [&](int P, pdhg_report* s, pdhg_report* o) {
    const double* r = row + P * kRowPer;
    const double* c = col + P * kColPer;
    *s = MakeReport(r[kPrS], c[kDuS], c[kBdS], c[kCxS], r[kQyS], d.offset, d.qn_s, d.cn_s);
    *o = MakeReport(r[kPrO], c[kDuO], c[kBdO], c[kCxO], r[kQyO], d.offset, d.qn_o, d.cn_o);
  };
  reports(0, &d.s_cur, &d.o_cur);
  reports(1, &d.s_avg, &d.o_avg);
  const double w = sc->omega;
  const double kkt_cur = KktError(d.s_cur.primal_res, d.s_cur.dual_res, d.s_cur.gap_abs, w);
  const double kkt_avg = KktError(d.s_avg.primal_res, d.s_avg.dual_res, d.s_avg.gap_abs, w);
  d.take_cur = kkt_cur < kkt_avg;
  d.kkt_cand = d.take_cur ? kkt_cur : kkt_avg;
  // EvaluateAndMaybeFinish(cur, avg) (solver.cpp:355-387).
  if (Terminated(d.o_cur, d.eps)) {
    d.best_from = 0;
    d.best_rep = d.o_cur;
    d.have_best = 1;
    d.action = kOptimalCur;
    sc->halt = 2;
    return;
  }
  auto record = [&](int P, const pdhg_report& r) {  // RecordBest (solver.cpp:341-351)
    const double k1 = Kkt1(r);
    if (!d.have_best || k1 < d.best_k1) {
      d.have_best = 1;
      d.best_k1 = k1;
      d.best_from = P;
      d.best_rep = r;
    }
  };
  record(0, d.o_cur);
  d.last_rep = d.o_cur;
  if (Terminated(d.o_avg, d.eps)) {
    d.best_from = 1;
    d.best_rep = d.o_avg;
    d.have_best = 1;
    d.action = kOptimalAvg;
    sc->halt = 2;
    return;
  }
  record(1, d.o_avg);
  if (Kkt1(d.o_avg) < Kkt1(d.o_cur)) d.last_rep = d.o_avg;
  if (d.restart_enabled && ShouldRestartV(d.suff, d.nec, d.frac, d.inner, d.iters, d.kkt_cand, d.kkt_start, d.kkt_prev)) {
    d.action = kRestart;  // the host applies it (UpdatePrimalWeight needs glibc exp/log)
    d.restart_flag = 1;
    sc->halt = 2;
    return;
  }
  d.kkt_prev = d.kkt_cand;
  d.action = kContinue;
}

__global__ void k_decide(const double* pack, Scalars* sc, DecideState* ds) {
  if (sc->halt) return;
  decide(pack, sc, ds);
}

// Best-iterate copy decided by the check that just ran (halt 0 or 2); a
// skipped check (halt 1) copies nothing.
__global__ void k_copy_best(const Scalars* sc, const DecideState* ds, const double* xc, const double* xa, double* xb,
                            int64_t n, const double* yc, const double* ya, double* yb, int64_t m) {
  if (sc->halt == 1 || ds->best_from < 0) return;
  const double* xs = ds->best_from == 0 ? xc : xa;
  const double* ys = ds->best_from == 0 ? yc : ya;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + m; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) xb[i] = xs[i];
    else yb[i - n] = ys[i - n];
  }
}

__global__ void k_settle(Scalars* sc) {
  if (sc->halt == 2) sc->halt = 1;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t globaltimer_ns();

// Device-resident loop, end of a block (one thread): advance the counters
// (k_advance), take the check's decisions (k_decide), then keep looping only
// while the decision is "continue" (halt 0), a whole block still fits the
// iteration limit and the time budget is not spent -- the tests the host loop
// makes before queueing a block (solver.cpp:252-259). The best-iterate copy
// after it still runs in this body iteration.
__global__ void k_decide_loop(const double* pack, Scalars* sc, DecideState* ds, int count,
                              cudaGraphConditionalHandle h) {
  sc->inner_base += static_cast<double>(count);
  ds->iters += count;
  ds->inner += count;
  decide(pack, sc, ds);
  const bool go = sc->halt == 0 && ds->iters + ds->block <= ds->iter_limit && globaltimer_ns() < ds->deadline_ns;
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

// Device-resident loop: the deadline from the host's remaining time budget,
// on the GPU's own clock, once per launch.
__global__ void k_loop_start(DecideState* ds) {
  const uint64_t r = ds->remaining_ns;
  const uint64_t now = globaltimer_ns();
  ds->deadline_ns = r > ~uint64_t(0) - now ? ~uint64_t(0) : now + r;
}


}  // namespace pdhg
