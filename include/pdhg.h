/*
 * pdhg.h — C-ABI of the B200 restarted-PDHG LP solver (libpdhg_b200.so).
 *
 * This is the drop-in boundary for the reference's solve path
 * `rpdlp::Solve(const LpProblem&, const SolverParams&, const EvalObserver&)`
 * (reference proj/core/include/rpdlp/solver.hpp:145-146). Everything is plain
 * C: borrowed pointers + sizes in, caller-allocated buffers out, an integer
 * return code plus a message buffer instead of exceptions. The C++ shim in
 * include/rpdlp/ maps the codes back onto the reference's exception types
 * (std::invalid_argument, rpdlp::NumericalFailure).
 *
 * Layout contract: matrices are passed exactly as the reference stores them
 * (CSR with int64 row_ptr / col_idx and double values,
 * sparse_matrix.hpp:94-98), A (equality rows) and G (>= rows) separately
 * (lp_problem.hpp:33-45). The library narrows indices to int32 on the device
 * and builds K = [A; G] in CSR and CSC there. No host pointer is retained
 * after a call returns (SURVEY §8b ownership rule).
 */
#ifndef PDHG_H_
#define PDHG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDHG_ABI_VERSION 1

/* Return codes (SURVEY §8b "Errors"). */
enum {
  PDHG_OK = 0,
  PDHG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  PDHG_NUMERICAL_FAILURE = 2, /* rpdlp::NumericalFailure (solver.cpp:391-394) */
  PDHG_CUDA_ERROR = 3,
  PDHG_NCCL_ERROR = 4,
  PDHG_ABORTED = 5, /* the eval callback asked to stop */
  PDHG_PARSE_ERROR = 6, /* rpdlp::MpsParseError (mps.hpp:26-36); line in err_line */
  PDHG_IO_ERROR = 7,    /* std::runtime_error from file access (mps_reader.cpp:453-468) */
  PDHG_ORDER_DEPENDENT = 8 /* device triplet assembly: an entry has >= 3 duplicates, whose sum depends on
                              the reference's std::sort order (sparse_matrix.cpp:35); nothing written */
};

/* rpdlp::SolveStatus (solver.hpp:57). */
enum { PDHG_OPTIMAL = 0, PDHG_ITER_LIMIT = 1, PDHG_TIME_LIMIT = 2 };

/* One CSR block, reference layout (sparse_matrix.hpp:83-101). */
typedef struct {
  int64_t rows;
  int64_t cols;
  const int64_t* row_ptr; /* rows + 1 */
  const int64_t* col_idx; /* nnz, strictly increasing per row */
  const double* values;   /* nnz, no explicit zeros */
} pdhg_csr;

/* rpdlp::LpProblem (lp_problem.hpp:33-45):
 *   min c'x  s.t.  A x = b,  G x >= h,  l <= x <= u. */
typedef struct {
  pdhg_csr a; /* m1 x n */
  pdhg_csr g; /* m2 x n */
  int64_t n;  /* length of c, l, u */
  const double* c;
  const double* b; /* m1 */
  const double* h; /* m2 */
  const double* l; /* -inf allowed */
  const double* u; /* +inf allowed */
  double objective_offset;
  int32_t negated_objective;
} pdhg_lp;

/* rpdlp::SolverParams (solver.hpp:32-55) with ScalingConfig
 * (scaling.hpp:40-44) flattened, field for field, same defaults. */
typedef struct {
  double eps;
  double time_limit;
  int64_t iter_limit;
  double sufficient_decay;
  double necessary_decay;
  double long_loop_frac;
  int32_t restart_enabled;
  int64_t check_every;
  int32_t scaling_enabled;
  int32_t ruiz_iters;
  double pc_alpha;
  uint64_t seed;
  int32_t adaptive_step;
  int64_t log_every;
} pdhg_params;

/* rpdlp::ResidualReport (kkt.hpp:32-41). */
typedef struct {
  double primal_res;
  double dual_res;
  double gap_abs;
  double primal_obj;
  double dual_obj;
  double rel_primal;
  double rel_dual;
  double rel_gap;
} pdhg_report;

/* rpdlp::EvalInfo (solver.hpp:127-140). */
typedef struct {
  int64_t iteration;
  int64_t inner_iteration;
  int64_t restarts;
  double omega;
  double eta;
  double kkt_candidate;
  double kkt_loop_start;
  int32_t candidate_is_current;
  int32_t restarted;
  pdhg_report original_report;
  double seconds;
} pdhg_eval_info;

/* rpdlp::EvalObserver (solver.hpp:142). Called synchronously on the calling
 * thread at every non-terminal check. A nonzero return aborts the solve with
 * PDHG_ABORTED (used by the C++ shim to rethrow observer exceptions). */
typedef int (*pdhg_eval_cb)(const pdhg_eval_info* info, void* user);

/* rpdlp::SolveResult (solver.hpp:59-70). x (n), y (m1+m2) and lambda (n)
 * are caller-allocated; any of them may be NULL to skip the copy-out. */
typedef struct {
  int32_t status;
  double* x;
  double* y;
  double* lambda;
  pdhg_report report;
  int64_t iterations;
  int64_t restarts;
  double solve_seconds;
  double scaling_seconds;
} pdhg_result;

/* Statistics of a resident session (sizes, partitions, timings). */
typedef struct {
  int64_t m1, m2, n, nnz;
  int64_t csr_tiles, csc_tiles;
  int64_t device_bytes;
  double upload_seconds;  /* H2D + int32 narrowing + stacking + CSC build */
  double scaling_seconds; /* Ruiz + Pock-Chambolle + ApplyScaling on device */
  int32_t device;
  int32_t l2_resident; /* 1 if the per-iteration working set fits in L2 */
  int32_t world;        /* shards K is split into */
  int32_t local_shards; /* shards held by this session (1 or world) */
  int32_t rank;         /* this session's shard when local_shards == 1 */
  int32_t uniform_bounds; /* bit 0: all scaled l equal, bit 1: all u equal
                             (those streams are skipped by the primal step) */
  int32_t csr_uniform_len; /* every short row has this many nonzeros (offsets
                              implicit, never read), else 0 */
  int32_t csc_uniform_len; /* same for short columns */
  int32_t csr_split;       /* > 0: the short rows' step pass runs as two
                              gather-window passes split at this column
                              (PDHG_S_SPLIT), else 0 */
  int32_t block_kernel;    /* 1: step blocks run as one persistent launch
                              (transport-shaped layouts; PDHG_PERSIST=0 off) */
} pdhg_session_stats;

/* Distribution of K over shards: `world` balanced row blocks
 * (K x, CSR) and column blocks (K^T y, CSC).
 *   world = 1                      one GPU, no exchange (the default path);
 *   local_shards = world           every shard in this session on one device,
 *                                  exchanges are in-place no-ops (exercises
 *                                  the sharded path on a single GPU);
 *   local_shards = 1, nccl_id set  one process per GPU: this session holds
 *                                  shard `rank`; x+ / y+ slices are
 *                                  all-gathered with NCCL every half-step,
 *                                  the check sums all-reduced every
 *                                  check_every iterations. Every rank passes
 *                                  the same problem and params and receives
 *                                  the same result. */
typedef struct {
  int32_t world;
  int32_t rank;
  int32_t local_shards;
  const void* nccl_id; /* 128-byte ncclUniqueId from pdhg_nccl_unique_id */
} pdhg_shard_spec;

typedef struct pdhg_session pdhg_session;

/* Defaults of rpdlp::SolverParams{} (solver.hpp:33-54). */
void pdhg_params_default(pdhg_params* p);

/* Library / ABI identification. */
int pdhg_abi_version(void);
const char* pdhg_build_info(void);
int pdhg_device_count(void);

/* ---- the drop-in entry point: rpdlp::Solve (solver.cpp:521-543) ----------
 * Validates problem and params (lp_problem.cpp:22-58, solver.cpp:59-70),
 * uploads, scales on device, runs the restarted PDHG loop on `device`,
 * copies the best iterate out. */
int pdhg_solve(const pdhg_lp* lp, const pdhg_params* params, pdhg_eval_cb cb,
               void* user, pdhg_result* out, char* err, size_t errlen);
int pdhg_solve_on(const pdhg_lp* lp, const pdhg_params* params, int device,
                  pdhg_eval_cb cb, void* user, pdhg_result* out, char* err,
                  size_t errlen);

/* ---- resident sessions (problem kept in HBM between solves) --------------
 * create = validate + upload + StackK + CSC build + ComputeScaling +
 * ApplyScaling (solver.cpp:523-537) on `device`. `params` supplies only the
 * scaling configuration. */
int pdhg_session_create(const pdhg_lp* lp, const pdhg_params* params,
                        int device, pdhg_session** out, char* err,
                        size_t errlen);
/* Same as pdhg_session_create with K distributed by `spec`. */
int pdhg_session_create_sharded(const pdhg_lp* lp, const pdhg_params* params,
                                int device, const pdhg_shard_spec* spec,
                                pdhg_session** out, char* err, size_t errlen);
/* One-shot sharded solve (rpdlp::Solve semantics on every rank). */
int pdhg_solve_sharded(const pdhg_lp* lp, const pdhg_params* params,
                       int device, const pdhg_shard_spec* spec,
                       pdhg_eval_cb cb, void* user, pdhg_result* out,
                       char* err, size_t errlen);
/* ncclGetUniqueId (rank 0 creates it and broadcasts the 128 bytes). */
int pdhg_nccl_unique_id(void* out128, char* err, size_t errlen);
/* An in-process LOOPBACK id (tests on one GPU): `world` one-shard sessions
 * created in one process on one device with this id in pdhg_shard_spec and
 * ranks 0..world-1 -- each constructed and solved on its own host thread --
 * run the multi-rank code path above with device-memory copies and
 * rendezvous kernels in place of NCCL (csrc/comm.cuh LoopbackComm). */
int pdhg_loopback_id(void* out128, char* err, size_t errlen);
/* Block boundaries in original row / column order (world + 1 each). */
int pdhg_session_blocks(pdhg_session* s, int64_t* row_begin,
                        int64_t* col_begin);
/* Ghost-exchange plan of a sharded session: x_counts[r * world + b] = number
 * of distinct x entries (columns) of block b that row block r reads (b != r;
 * the diagonal is 0), y_counts likewise for the column blocks' row reads;
 * use[0] / use[1] = whether the x / y exchange sends only those entries
 * (NCCL mode, ghost volume <= half an all-gather) instead of all-gathering. */
int pdhg_session_ghost_counts(pdhg_session* s, int64_t* x_counts,
                              int64_t* y_counts, int32_t* use);
/* The balanced split every rank computes: `parts` contiguous blocks of the
 * `nseg` segments of a CSR/CSC offset array (`begin`: parts + 1 entries). */
int pdhg_partition_blocks(const int64_t* ptr, int64_t nseg, int parts,
                          int64_t seg_weight, int64_t* begin);
void pdhg_session_destroy(pdhg_session* s);
/* SparseMatrix::FromTriplets (sparse_matrix.cpp:25-69) on the device: sort
 * by (row, col), sum duplicates, drop exact zeros, emit CSR (SURVEY §8f
 * rank 1: device-side problem assembly). `trips` is the reference's Triplet
 * layout {int64 row, int64 col, double value}. The sort is stable, so
 * duplicates are summed in input order; the reference sums them in its
 * std::sort order, which is the same sum for up to two duplicates of one
 * entry (a + b == b + a) or for any number of bitwise-equal values, but not
 * for three or more differing values. Such an input returns
 * PDHG_ORDER_DEPENDENT without output, and the C++ drop-in then assembles
 * on the host with the reference's std::sort. Outputs are caller-allocated:
 * row_ptr[rows + 1], col_idx[count], values[count]; *nnz receives the
 * entries written. An index out of range returns PDHG_INVALID_ARGUMENT
 * ("triplet index out of range"). count < 2^31. */
typedef struct pdhg_triplet {
  int64_t row, col;
  double value;
} pdhg_triplet;
int pdhg_csr_from_triplets(int64_t rows, int64_t cols, int64_t count, const pdhg_triplet* trips, int device,
                           int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* nnz,
                           char* err, size_t errlen);
/* SparseMatrix::FromTriplets exactly as the C++ drop-in runs it
 * (include/rpdlp/sparse_matrix.hpp): pdhg_csr_from_triplets from 2^20
 * triplets when a GPU is visible, the reference's std::sort assembly on the
 * host otherwise and for PDHG_ORDER_DEPENDENT inputs. Same outputs and
 * errors as pdhg_csr_from_triplets (other device failures: PDHG_CUDA_ERROR). */
int pdhg_from_triplets(int64_t rows, int64_t cols, int64_t count, const pdhg_triplet* trips,
                       int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* nnz,
                       char* err, size_t errlen);
/* The power-iteration start vector of EstimateOpNorm (solver.cpp:88-97):
 * n draws of std::normal_distribution<double>(0,1) over
 * std::mt19937_64(seed). threads < 0: the sequential libstdc++ draw;
 * otherwise the bit-identical multi-threaded replica the solver uses
 * (0 = all host threads). */
int pdhg_normal_vector(uint64_t seed, int64_t n, int threads, double* out);
int pdhg_session_stats_get(pdhg_session* s, pdhg_session_stats* out);
/* SolveLoop(...).Run() (solver.cpp:232-267) on the resident scaled problem.
 * out->scaling_seconds reports the session's device scaling time. The
 * problem was scaled once at session creation: params whose scaling config
 * (scaling_enabled, ruiz_iters, pc_alpha) differs from the creation params
 * are rejected with PDHG_INVALID_ARGUMENT. */
int pdhg_session_solve(pdhg_session* s, const pdhg_params* params,
                       pdhg_eval_cb cb, void* user, pdhg_result* out,
                       char* err, size_t errlen);

/* ---- kernel-level entry points (parity tests, benchmarks) ----------------
 * All vectors are host buffers. */
/* Composed Ruiz x PC scales (scaling.cpp:86-91): row_scale m, col_scale n. */
int pdhg_session_scaling(pdhg_session* s, double* row_scale,
                         double* col_scale, char* err, size_t errlen);
/* The scaled problem as the loop sees it: K_s values in CSR order (nnz),
 * c_s, l_s, u_s (n), q_s (m). Any pointer may be NULL. */
int pdhg_session_scaled(pdhg_session* s, double* k_values, double* c,
                        double* l, double* u, double* q, char* err,
                        size_t errlen);
/* SpMV with the scaled stacked K: transpose=0 -> out(m) = K_s in(n)
 * (sparse_matrix.cpp:114-125); transpose=1 -> out(n) = K_s^T in(m)
 * (sparse_matrix.cpp:127-138). */
int pdhg_session_spmv(pdhg_session* s, int transpose, const double* in,
                      double* out, char* err, size_t errlen);
/* EstimateOpNorm(K_s, iters, seed) (solver.cpp:84-110). */
int pdhg_session_opnorm(pdhg_session* s, int iters, uint64_t seed,
                        double* out, char* err, size_t errlen);
/* Times the two fused step kernels of one PDHG iteration (K-CSC primal and
 * K-CSR dual) launched `iters` times each back to back on the session
 * stream, bracketed by CUDA events on that stream; returns mean milliseconds
 * per launch and the whole-iteration mean from a graph-launched block. L2 is
 * NOT flushed between launches: where the working set fits the 126 MB L2
 * these figures are L2-assisted (warm). */
int pdhg_session_time_kernels(pdhg_session* s, int iters, double* ms_primal,
                              double* ms_dual, double* ms_iteration,
                              char* err, size_t errlen);
/* The same kernels timed cold: before every launch a read sweep over a
 * buffer twice the L2 size leaves L2 clean and holding none of the solver's
 * data; CUDA events on the session stream bracket each launch (primal, dual,
 * and one whole iteration with its programmatic overlap); means over
 * `iters` launches. These are the roofline figures. */
int pdhg_session_time_kernels_cold(pdhg_session* s, int iters, double* ms_primal,
                                   double* ms_dual, double* ms_iteration,
                                   char* err, size_t errlen);
/* Runs `iters` plain PDHG steps as the solver's graph-launched blocks on the
 * resident problem; with profiler_range != 0 bracketed by
 * cudaProfilerStart/Stop (an `ncu --replay-mode app-range` target: DRAM
 * counters over whole iterations, write-backs included). */
int pdhg_session_run_block(pdhg_session* s, int iters, int profiler_range,
                           char* err, size_t errlen);

/* Times the termination / restart check (SolveLoop::Check, solver.cpp:390-428:
 * residual passes over K for the current and average iterates plus their
 * reductions): mean device milliseconds per check from `iters` back-to-back
 * checks bracketed by CUDA events, and mean wall milliseconds per check
 * including the device -> host read the host loop waits on. */
int pdhg_session_time_check(pdhg_session* s, int iters, double* ms_device,
                            double* ms_wall, char* err, size_t errlen);

/* SparseMatrix::Multiply / MultiplyTranspose / MultiplyAdd /
 * MultiplyTransposeAdd (sparse_matrix.cpp:114-164) on the device:
 * t = M x (transpose: M^T x) -- every row / column of <= 64 nonzeros summed in
 * storage order, bit-identical with the reference -- then y = t
 * (accumulate = 0) or y += alpha * t (accumulate = 1: the sum is completed
 * first, then added, as the reference does). */
int pdhg_csr_spmv(const pdhg_csr* m, int transpose, int accumulate, double alpha,
                  const double* x, double* y, char* err, size_t errlen);

/* RowInfNorms / ColInfNorms (power = 0) and RowPowerSums / ColPowerSums
 * (power = 1, exponent p) (sparse_matrix.cpp:166-204) on the device; out has
 * rows (columns = 0) or cols (columns = 1) entries. Sums run in storage order
 * (bit-identical for <= 64 nonzeros per segment; p outside {0, 1, 2} uses the
 * device pow). */
int pdhg_csr_norms(const pdhg_csr* m, int columns, int power, double p, double* out,
                   char* err, size_t errlen);
/* SparseMatrix::Scaled (sparse_matrix.cpp:206-222): the values of both
 * layouts of D_r M D_c (row_scale * v * col_scale, left to right). The CSC
 * arrays are the matrix's own (col_ptr, row_idx, csc values). */
int pdhg_csr_scaled(const pdhg_csr* m, const int64_t* col_ptr, const int64_t* row_idx,
                    const double* csc_values, const double* row_scale,
                    const double* col_scale, double* csr_out, double* csc_out,
                    char* err, size_t errlen);

/* ---- unit-level exports (solver.hpp:81-125), device-backed ---------------
 * PrimalStep (solver.cpp:112-129): out(n) = proj_[l,u](x - eta/omega (c - K'y))
 * DualStep (solver.cpp:131-154): out(m) = proj_Y(y + eta*omega (q - K(2x_new - x_old)))
 * These run on the unscaled problem's K. */
int pdhg_primal_step(const pdhg_lp* lp, const double* x, const double* y,
                     double eta, double omega, double* out, char* err,
                     size_t errlen);
int pdhg_dual_step(const pdhg_lp* lp, const double* x_new,
                   const double* x_old, const double* y, double eta,
                   double omega, double* out, char* err, size_t errlen);

/* ---- scaling and residual utilities (scaling.hpp:49-59, kkt.hpp:45-60) ----
 * Device-backed; the device is $PDHG_DEVICE (default 0).
 * pdhg_compute_scaling: stages 1 = RuizEquilibrate(k, ruiz_iters)
 * (scaling.cpp:49-68), 2 = PockChambolleScale(k, pc_alpha) (:70-84),
 * 3 = ComputeScaling (:86-91; Ruiz then PC on the Ruiz-scaled matrix,
 * composed). row_scale has k->rows entries, col_scale k->cols. */
int pdhg_compute_scaling(const pdhg_csr* k, int ruiz_iters, double pc_alpha,
                         int stages, double* row_scale, double* col_scale,
                         char* err, size_t errlen);
/* ComputeResiduals(problem, {x, y}) (kkt.cpp:143-145) on the original
 * problem. */
int pdhg_residuals(const pdhg_lp* lp, const double* x, const double* y,
                   pdhg_report* out, char* err, size_t errlen);
/* DeriveLambda(problem, y) (kkt.cpp:127-141): lambda (n). */
int pdhg_derive_lambda(const pdhg_lp* lp, const double* y, double* lambda,
                       char* err, size_t errlen);

/* ---- bench instrumentation ------------------------------------------------
 * flush_l2 writes a buffer of twice the L2 size on the session stream.
 * last_solve reports the device time of the most recent pdhg_session_solve
 * (CUDA events on the session stream bracketing the whole solve, power
 * iteration included) and how many kernels it launched (graph nodes
 * counted individually). */
int pdhg_session_flush_l2(pdhg_session* s, char* err, size_t errlen);
int pdhg_session_last_solve(pdhg_session* s, double* device_ms,
                            int64_t* kernel_launches);

/* ---- host decision logic (pure host code, no device) -----------------------
 * ShouldRestart (solver.cpp:178-189), UpdatePrimalWeight (solver.cpp:191-196),
 * KktError (kkt.cpp:153-157), CheckTermination (kkt.cpp:147-151): the exact
 * functions the solve loop uses, exported for unit tests and API parity. */
int pdhg_should_restart(const pdhg_params* p, int64_t t, int64_t k,
                        double kkt_candidate, double kkt_loop_start,
                        double kkt_prev_candidate);
double pdhg_update_primal_weight(double omega, double dx_norm, double dy_norm);
double pdhg_kkt_error(double primal_res, double dual_res, double gap,
                      double omega);
int pdhg_check_termination(const pdhg_report* r, double eps);

/* ---- instance generators (instance_gen.hpp:39-59 + SURVEY §8d shapes) ----
 * Host-side input builders; they own their arrays until freed. */
typedef struct pdhg_instance pdhg_instance;
/* GenRandomLp (instance_gen.cpp:143-188), bit-identical per seed. */
int pdhg_gen_random_lp(int64_t m, int64_t n, double density, uint64_t seed,
                       pdhg_instance** out, char* err, size_t errlen);
/* GenPagerank (instance_gen.cpp:27-64, 90-141), bit-identical per seed. */
int pdhg_gen_pagerank(int64_t n_nodes, double damping, int64_t attachment,
                      uint64_t seed, pdhg_instance** out, char* err,
                      size_t errlen);
/* GenPagerankGraph (instance_gen.cpp:27-64): `edges` receives count pairs
 * (src, dst) as 2*count int64s; capacity (in pairs) must be at least
 * pdhg_pagerank_graph_edges(n_nodes, attachment). */
int64_t pdhg_pagerank_graph_edges(int64_t n_nodes, int64_t attachment);
int pdhg_gen_pagerank_graph(int64_t n_nodes, double damping, int64_t attachment,
                            uint64_t seed, int64_t* edges, int64_t capacity,
                            int64_t* count, char* err, size_t errlen);
/* BuildPagerankLp (instance_gen.cpp:90-137) over `count` (src, dst) pairs. */
int pdhg_build_pagerank_lp(const int64_t* edges, int64_t count, int64_t n_nodes,
                           double damping, pdhg_instance** out, char* err,
                           size_t errlen);
/* Transportation LP, `sources` x `sinks`: demand rows
 * sum_i x_ij = d_j in A, supply rows -sum_j x_ij >= -s_i in G, x >= 0. */
int pdhg_gen_transport(int64_t sources, int64_t sinks, uint64_t seed,
                       pdhg_instance** out, char* err, size_t errlen);
/* Multicommodity network flow: power-law digraph of
 * `nodes` nodes and `arcs` arcs, `commodities` commodities; conservation rows
 * (=, heavy-tailed lengths) in A, arc capacity rows (>= after negation) in G,
 * x >= 0. Feasible by construction (witness flow available). */
int pdhg_gen_mcf(int64_t nodes, int64_t arcs, int64_t commodities,
                 uint64_t seed, pdhg_instance** out, char* err, size_t errlen);
/* Block-angular staircase: `stages` stages of
 * `rows_per_stage` x `cols_per_stage`, `nnz_per_row` nonzeros per row of which
 * `linking_per_row` reach into the previous stage; the first
 * `eq_rows_per_stage` rows of each stage are equalities. Generated by
 * `threads` host threads (0 = all), bit-identical for any thread count. */
int pdhg_gen_staircase(int64_t stages, int64_t rows_per_stage,
                       int64_t cols_per_stage, int64_t nnz_per_row,
                       int64_t linking_per_row, int64_t eq_rows_per_stage,
                       uint64_t seed, int threads, pdhg_instance** out,
                       char* err, size_t errlen);
/* Moves the first `m1` rows of G into A with b = G_rows * witness
 * (SURVEY §8d config 1 post-pass). Requires a witness (GenRandomLp). */
int pdhg_instance_make_equalities(pdhg_instance* inst, int64_t m1, char* err,
                                  size_t errlen);
int pdhg_instance_view(const pdhg_instance* inst, pdhg_lp* out);
/* Witness x_hat (GenRandomLp, MCF, staircase; length n) or NULL. */
const double* pdhg_instance_witness(const pdhg_instance* inst);
void pdhg_instance_free(pdhg_instance* inst);
/* NAME of an instance read from MPS ("" otherwise). */
const char* pdhg_instance_name(const pdhg_instance* inst);

/* ---- MPS ingestion (mps.hpp:50-56; reader mps_reader.cpp, writer
 * mps_writer.cpp): same normalisations, errors and messages as the
 * reference's ParseMps / WriteMps. Read results are instances (view them with
 * pdhg_instance_view, free with pdhg_instance_free). Parse failures return
 * PDHG_PARSE_ERROR with "mps parse error at line N: ..." in err and N in
 * *err_line; unreadable files PDHG_IO_ERROR; an invalid LP (e.g. an infinite
 * cost) PDHG_INVALID_ARGUMENT. Paths ending in .gz are read through zlib. */
int pdhg_mps_read_file(const char* path, int fixed_format, pdhg_instance** out,
                       char* err, size_t errlen, int* err_line);
int pdhg_mps_read_string(const char* text, size_t len, int fixed_format,
                         pdhg_instance** out, char* err, size_t errlen,
                         int* err_line);
/* WriteMps / WriteMpsFile: free format, %.17g numbers. The string variant
 * returns a malloc'ed buffer released with pdhg_free_string. */
int pdhg_mps_write_file(const pdhg_lp* lp, const char* name, const char* path,
                        char* err, size_t errlen);
int pdhg_mps_write_string(const pdhg_lp* lp, const char* name, char** out,
                          size_t* out_len, char* err, size_t errlen);
void pdhg_free_string(char* s);

#ifdef __cplusplus
}
#endif

#endif /* PDHG_H_ */
