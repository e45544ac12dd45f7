"""Python mirror of the reference's solve-path interface (rpdlp, C++).

Names, fields, defaults and error behaviour follow
/root/reference/proj/core/include/rpdlp/{lp_problem,solver,kkt,scaling}.hpp:

    LpProblem        lp_problem.hpp:33-57   (A eq rows, G >= rows, c, b, h, l, u)
    SolverParams     solver.hpp:32-55       (+ ScalingConfig, scaling.hpp:40-44)
    SolveResult      solver.hpp:59-70
    EvalInfo         solver.hpp:127-140     (observer snapshot)
    ResidualReport   kkt.hpp:32-41
    Solve            solver.hpp:145-146     -> pdhg_solve (C-ABI) on a B200
    NumericalFailure solver.hpp:73-75       (ValueError plays std::invalid_argument)

Everything computes in libpdhg_b200.so; this module only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import abi

INT64_MAX = (1 << 63) - 1
kInf = float("inf")


class NumericalFailure(RuntimeError):
    """Non-finite iterate (solver.cpp:391-394)."""


class MpsParseError(RuntimeError):
    """rpdlp::MpsParseError (mps.hpp:26-36): message carries the line."""

    def __init__(self, message: str, line: int):
        super().__init__(message)
        self.line = line


class CudaError(RuntimeError):
    pass


class OrderDependent(RuntimeError):
    """Device triplet assembly refused an entry duplicated three or more
    times (PDHG_ORDER_DEPENDENT): only the reference's std::sort order gives
    the reference's sum; CsrMatrix.from_triplets assembles those on the host."""


class SolveStatus(enum.IntEnum):
    kOptimal = abi.PDHG_OPTIMAL
    kIterLimit = abi.PDHG_ITER_LIMIT
    kTimeLimit = abi.PDHG_TIME_LIMIT


def ToString(status: SolveStatus) -> str:  # solver.cpp:72-82
    return {0: "Optimal", 1: "IterLimit", 2: "TimeLimit"}.get(int(status), "Unknown")


@dataclass
class ScalingConfig:
    enabled: bool = True
    ruiz_iters: int = 10
    pc_alpha: float = 1.0


@dataclass
class SolverParams:
    eps: float = 1e-4
    time_limit: float = 3600.0
    iter_limit: int = INT64_MAX
    sufficient_decay: float = 0.2
    necessary_decay: float = 0.8
    long_loop_frac: float = 0.36
    restart_enabled: bool = True
    check_every: int = 64
    scaling: ScalingConfig = field(default_factory=ScalingConfig)
    seed: int = 0
    adaptive_step: bool = False
    log_every: int = 0

    def to_c(self) -> abi.Params:
        return abi.Params(self.eps, self.time_limit, int(self.iter_limit), self.sufficient_decay,
                          self.necessary_decay, self.long_loop_frac, int(bool(self.restart_enabled)),
                          int(self.check_every), int(bool(self.scaling.enabled)), int(self.scaling.ruiz_iters),
                          self.scaling.pc_alpha, int(self.seed) & ((1 << 64) - 1), int(bool(self.adaptive_step)),
                          int(self.log_every))


@dataclass
class CsrMatrix:
    """CSR block with the reference's int64 index layout (sparse_matrix.hpp:94-98)."""
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @staticmethod
    def empty(rows: int, cols: int) -> "CsrMatrix":
        return CsrMatrix(rows, cols, np.zeros(rows + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))

    @staticmethod
    def from_triplets(rows: int, cols: int, trips) -> "CsrMatrix":
        """SparseMatrix::FromTriplets (sparse_matrix.cpp:25-69) with the C++
        drop-in's semantics (pdhg_from_triplets): duplicates summed in the
        reference's std::sort order, exact zeros dropped; an index out of
        range raises IndexError."""
        t = list(trips)
        arr = np.empty(len(t), dtype=[("row", "<i8"), ("col", "<i8"), ("value", "<f8")])
        for i, (r, c, v) in enumerate(t):
            arr[i] = (int(r), int(c), float(v))
        return CsrMatrix._assemble(rows, cols, arr, None)

    @staticmethod
    def from_arrays(rows: int, cols: int, row, col, value) -> "CsrMatrix":
        """from_triplets on index / value arrays (the drop-in's FromTriplets:
        device assembly from 2^20 triplets where that reproduces the
        reference, the reference's host std::sort otherwise)."""
        row, col, value = np.asarray(row), np.asarray(col), np.asarray(value, np.float64)
        trips = np.empty(row.size, dtype=[("row", "<i8"), ("col", "<i8"), ("value", "<f8")])
        trips["row"], trips["col"], trips["value"] = row, col, value
        return CsrMatrix._assemble(rows, cols, trips, None)

    @staticmethod
    def _assemble(rows: int, cols: int, trips: np.ndarray, device: Optional[int]) -> "CsrMatrix":
        n = int(trips.size)
        ptr = np.zeros(rows + 1, np.int64)
        idx, val = np.empty(max(n, 1), np.int64), np.empty(max(n, 1), np.float64)
        nnz = C.c_int64(0)
        err = C.create_string_buffer(abi.ERRLEN)
        lib = abi.load()
        if device is None:
            code = lib.pdhg_from_triplets(rows, cols, n, trips.ctypes.data, _i64p(ptr), _i64p(idx), _dp(val),
                                          C.byref(nnz), err, abi.ERRLEN)
        else:
            code = lib.pdhg_csr_from_triplets(rows, cols, n, trips.ctypes.data, device, _i64p(ptr), _i64p(idx),
                                              _dp(val), C.byref(nnz), err, abi.ERRLEN)
        if code == abi.PDHG_INVALID_ARGUMENT and b"out of range" in err.value:
            raise IndexError(err.value.decode())
        if code == abi.PDHG_ORDER_DEPENDENT:
            raise OrderDependent(err.value.decode())
        raise_for(code, err)
        k = nnz.value
        return CsrMatrix(rows, cols, ptr, idx[:k].copy(), val[:k].copy())

    @staticmethod
    def from_triplets_device(rows: int, cols: int, row, col, value, device: int = 0) -> "CsrMatrix":
        """FromTriplets on the device (pdhg_csr_from_triplets, SURVEY §8f
        rank 1): stable radix sort, duplicates summed in input order, exact
        zeros dropped. Arrays of row / column indices and values."""
        row, col, value = np.asarray(row), np.asarray(col), np.asarray(value, np.float64)
        n = int(row.size)
        if not (col.size == n and value.size == n):
            raise ValueError("row / col / value lengths differ")
        trips = np.empty(n, dtype=[("row", "<i8"), ("col", "<i8"), ("value", "<f8")])
        trips["row"], trips["col"], trips["value"] = row, col, value
        return CsrMatrix._assemble(rows, cols, trips, device)

    def multiply(self, x, transpose: bool = False) -> np.ndarray:
        """SparseMatrix::Multiply / MultiplyTranspose (sparse_matrix.cpp:114-138)
        on the device (pdhg_csr_spmv; storage-order sums)."""
        x = _f64(x)
        out = np.zeros(self.cols if transpose else self.rows)
        c = self.to_c()
        err = C.create_string_buffer(abi.ERRLEN)
        raise_for(abi.load().pdhg_csr_spmv(C.byref(c), int(transpose), 0, 1.0, _dp(x), _dp(out), err, abi.ERRLEN),
                  err)
        return out

    def norms(self, columns: bool = False, power: float = None) -> np.ndarray:
        """Row/ColInfNorms (power None) or Row/ColPowerSums(power)
        (sparse_matrix.cpp:166-204) on the device."""
        out = np.zeros(self.cols if columns else self.rows)
        c = self.to_c()
        err = C.create_string_buffer(abi.ERRLEN)
        raise_for(abi.load().pdhg_csr_norms(C.byref(c), int(columns), int(power is not None),
                                            float(power or 0.0), _dp(out), err, abi.ERRLEN), err)
        return out

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.rows else 0

    def to_c(self) -> abi.Csr:
        return abi.Csr(self.rows, self.cols, _i64p(self.row_ptr), _i64p(self.col_idx), _dp(self.values))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols))
        for r in range(self.rows):
            for k in range(self.row_ptr[r], self.row_ptr[r + 1]):
                d[r, self.col_idx[k]] += self.values[k]
        return d


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(abi.dptr)


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(abi.i64ptr)


@dataclass
class LpProblem:
    """min c'x  s.t.  A x = b,  G x >= h,  l <= x <= u (lp_problem.hpp:33-45)."""
    a: CsrMatrix
    g: CsrMatrix
    c: np.ndarray
    b: np.ndarray
    h: np.ndarray
    l: np.ndarray
    u: np.ndarray
    objective_offset: float = 0.0
    negated_objective: bool = False
    name: str = ""

    def __post_init__(self):
        for m in (self.a, self.g):
            m.row_ptr, m.col_idx, m.values = _i64(m.row_ptr), _i64(m.col_idx), _f64(m.values)
        self.c, self.b, self.h, self.l, self.u = map(_f64, (self.c, self.b, self.h, self.l, self.u))

    def num_vars(self) -> int:
        return len(self.c)

    def num_eq_rows(self) -> int:
        return self.a.rows

    def num_ineq_rows(self) -> int:
        return self.g.rows

    def num_rows(self) -> int:
        return self.a.rows + self.g.rows

    def to_c(self) -> abi.Lp:
        return abi.Lp(self.a.to_c(), self.g.to_c(), len(self.c), _dp(self.c), _dp(self.b), _dp(self.h),
                      _dp(self.l), _dp(self.u), float(self.objective_offset), int(bool(self.negated_objective)))

    def nnz(self) -> int:
        return self.a.nnz + self.g.nnz


@dataclass
class ResidualReport:
    primal_res: float = 0.0
    dual_res: float = 0.0
    gap_abs: float = 0.0
    primal_obj: float = 0.0
    dual_obj: float = 0.0
    rel_primal: float = 0.0
    rel_dual: float = 0.0
    rel_gap: float = 0.0

    @staticmethod
    def from_c(r: abi.Report) -> "ResidualReport":
        return ResidualReport(*(getattr(r, k) for k, _ in abi.Report._fields_))


@dataclass
class EvalInfo:
    iteration: int
    inner_iteration: int
    restarts: int
    omega: float
    eta: float
    kkt_candidate: float
    kkt_loop_start: float
    candidate_is_current: bool
    restarted: bool
    original_report: ResidualReport
    seconds: float

    @staticmethod
    def from_c(e: abi.EvalInfo) -> "EvalInfo":
        return EvalInfo(e.iteration, e.inner_iteration, e.restarts, e.omega, e.eta, e.kkt_candidate,
                        e.kkt_loop_start, bool(e.candidate_is_current), bool(e.restarted),
                        ResidualReport.from_c(e.original_report), e.seconds)


@dataclass
class SolveResult:
    status: SolveStatus
    x: np.ndarray
    y: np.ndarray
    lambda_: np.ndarray
    report: ResidualReport
    iterations: int
    restarts: int
    solve_seconds: float
    scaling_seconds: float


EvalObserver = Callable[[EvalInfo], None]


def raise_for(code: int, err: bytes, pending: Optional[BaseException] = None) -> None:
    if code == abi.PDHG_OK:
        return
    if pending is not None:
        raise pending
    msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
    if code == abi.PDHG_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == abi.PDHG_NUMERICAL_FAILURE:
        raise NumericalFailure(msg)
    raise CudaError(f"code {code}: {msg}")


class _Observer:
    """Trampoline: Python observer -> C callback; exceptions abort the solve
    and are re-raised after the device state is released."""

    def __init__(self, fn: Optional[EvalObserver], factory=EvalInfo.from_c):
        self.fn, self.error, self.factory = fn, None, factory

        def cb(info_p, _user):
            try:
                self.fn(self.factory(info_p.contents))
                return 0
            except BaseException as e:  # noqa: BLE001 - rethrown by raise_for
                self.error = e
                return 1

        self.c = abi.EVAL_CB(cb) if fn is not None else abi.EVAL_CB()


def _result(problem: LpProblem):
    n, m = problem.num_vars(), problem.num_rows()
    x, y, lam = np.empty(n), np.empty(m), np.empty(n)
    res = abi.Result()
    res.x, res.y, res.lambda_ = _dp(x), _dp(y), _dp(lam)
    return res, x, y, lam


def _pack(res, x, y, lam) -> SolveResult:
    return SolveResult(SolveStatus(res.status), x, y, lam, ResidualReport.from_c(res.report), res.iterations,
                       res.restarts, res.solve_seconds, res.scaling_seconds)


@dataclass
class Shards:
    """How K is distributed (pdhg_shard_spec).

    Shards(world=P, local=True): all P shards in this process on one device
    (exchanges are in-place no-ops) -- the sharded path on a single GPU.
    Shards.from_process_group(): one shard per torch.distributed rank (one
    process per GPU); rank 0 creates the NCCL id and broadcasts it over the
    group, the solver then all-gathers x / y slices with NCCL itself."""
    world: int = 1
    rank: int = 0
    local: bool = True
    nccl_id: Optional[bytes] = None

    @staticmethod
    def nccl_single() -> "Shards":
        """One rank, one GPU, through the NCCL exchange path (tests)."""
        buf = C.create_string_buffer(128)
        err = C.create_string_buffer(abi.ERRLEN)
        raise_for(abi.load().pdhg_nccl_unique_id(buf, err, abi.ERRLEN), err)
        return Shards(1, 0, False, bytes(buf.raw))

    @staticmethod
    def loopback(world: int) -> "list[Shards]":
        """`world` rank specs for in-process loopback ranks on one device
        (pdhg_loopback_id): construct and solve one Session per spec, each on
        its own thread -- the multi-rank code path without NCCL (tests)."""
        buf = C.create_string_buffer(128)
        err = C.create_string_buffer(abi.ERRLEN)
        raise_for(abi.load().pdhg_loopback_id(buf, err, abi.ERRLEN), err)
        return [Shards(world, r, False, bytes(buf.raw)) for r in range(world)]

    @staticmethod
    def from_process_group(group=None) -> "Shards":
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if world == 1:
            return Shards()
        uid = bytearray(128)
        if rank == 0:
            buf = C.create_string_buffer(128)
            err = C.create_string_buffer(abi.ERRLEN)
            raise_for(abi.load().pdhg_nccl_unique_id(buf, err, abi.ERRLEN), err)
            uid = bytearray(buf.raw)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        return Shards(world, rank, False, bytes(t.cpu().tolist()))

    def to_c(self):
        spec = abi.ShardSpec(self.world, self.rank, self.world if self.local else 1, None)
        keep = None
        if not self.local:
            if self.nccl_id is None or len(self.nccl_id) != 128:
                raise ValueError("one-shard-per-process mode needs a 128-byte NCCL id")
            keep = C.create_string_buffer(self.nccl_id, 128)
            spec.nccl_id = C.cast(keep, C.c_void_p)
        return spec, keep


def Solve(problem: LpProblem, params: Optional[SolverParams] = None, observer: Optional[EvalObserver] = None,
          device: int = 0, shards: Optional[Shards] = None) -> SolveResult:
    """rpdlp::Solve (solver.cpp:521-543) on a B200 through pdhg_solve_on, or
    pdhg_solve_sharded when `shards` distributes K."""
    lib = abi.load()
    params = params or SolverParams()
    lp, prm = problem.to_c(), params.to_c()
    res, x, y, lam = _result(problem)
    obs = _Observer(observer)
    err = C.create_string_buffer(abi.ERRLEN)
    if shards is None or (shards.world == 1 and shards.local):
        code = lib.pdhg_solve_on(C.byref(lp), C.byref(prm), device, obs.c, None, C.byref(res), err, abi.ERRLEN)
    else:
        spec, _keep = shards.to_c()
        code = lib.pdhg_solve_sharded(C.byref(lp), C.byref(prm), device, C.byref(spec), obs.c, None, C.byref(res),
                                      err, abi.ERRLEN)
    raise_for(code, err, obs.error)
    return _pack(res, x, y, lam)


class Session:
    """Problem resident in HBM (upload + CSC build + device scaling once)."""

    def __init__(self, problem: LpProblem, params: Optional[SolverParams] = None, device: int = 0,
                 shards: Optional[Shards] = None):
        self.lib = abi.load()
        self.problem = problem
        self.params = params or SolverParams()
        self.shards = shards or Shards()
        lp, prm = problem.to_c(), self.params.to_c()
        self.h = C.c_void_p()
        err = C.create_string_buffer(abi.ERRLEN)
        if self.shards.world == 1 and self.shards.local:
            code = self.lib.pdhg_session_create(C.byref(lp), C.byref(prm), device, C.byref(self.h), err, abi.ERRLEN)
        else:
            spec, _keep = self.shards.to_c()
            code = self.lib.pdhg_session_create_sharded(C.byref(lp), C.byref(prm), device, C.byref(spec),
                                                        C.byref(self.h), err, abi.ERRLEN)
        raise_for(code, err)

    def close(self):
        if self.h:
            self.lib.pdhg_session_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def _err(self):
        return C.create_string_buffer(abi.ERRLEN)

    def solve(self, params: Optional[SolverParams] = None, observer: Optional[EvalObserver] = None) -> SolveResult:
        prm = (params or self.params).to_c()
        res, x, y, lam = _result(self.problem)
        obs = _Observer(observer)
        err = self._err()
        code = self.lib.pdhg_session_solve(self.h, C.byref(prm), obs.c, None, C.byref(res), err, abi.ERRLEN)
        raise_for(code, err, obs.error)
        return _pack(res, x, y, lam)

    def flush_l2(self) -> None:
        err = self._err()
        raise_for(self.lib.pdhg_session_flush_l2(self.h, err, abi.ERRLEN), err)

    def last_solve(self):
        """(device milliseconds, kernel launches) of the latest solve."""
        ms, n = C.c_double(), C.c_int64()
        self.lib.pdhg_session_last_solve(self.h, C.byref(ms), C.byref(n))
        return ms.value, n.value

    def stats(self) -> abi.SessionStats:
        s = abi.SessionStats()
        self.lib.pdhg_session_stats_get(self.h, C.byref(s))
        return s

    def blocks(self):
        """(row_begin, col_begin): the balanced blocks in original order."""
        w = self.shards.world
        rb, cb = np.empty(w + 1, np.int64), np.empty(w + 1, np.int64)
        raise_for(self.lib.pdhg_session_blocks(self.h, _i64p(rb), _i64p(cb)), b"")
        return rb, cb

    def ghost_counts(self):
        """(x_counts, y_counts, (use_x, use_y)): world x world matrices of the
        ghost entries each block reads from each other block."""
        w = self.shards.world
        xc, yc = np.zeros((w, w), np.int64), np.zeros((w, w), np.int64)
        use = (C.c_int32 * 2)()
        if w > 1:
            raise_for(self.lib.pdhg_session_ghost_counts(self.h, _i64p(xc), _i64p(yc), use), b"")
        return xc, yc, (bool(use[0]), bool(use[1]))

    def scaling(self):
        rs, cs = np.empty(self.problem.num_rows()), np.empty(self.problem.num_vars())
        err = self._err()
        raise_for(self.lib.pdhg_session_scaling(self.h, _dp(rs), _dp(cs), err, abi.ERRLEN), err)
        return rs, cs

    def scaled(self):
        p = self.problem
        kv, c, l, u, q = (np.empty(p.nnz()), np.empty(p.num_vars()), np.empty(p.num_vars()),
                          np.empty(p.num_vars()), np.empty(p.num_rows()))
        err = self._err()
        raise_for(self.lib.pdhg_session_scaled(self.h, _dp(kv), _dp(c), _dp(l), _dp(u), _dp(q), err, abi.ERRLEN),
                  err)
        return kv, c, l, u, q

    def spmv(self, vec, transpose: bool = False) -> np.ndarray:
        v = _f64(vec)
        out = np.empty(self.problem.num_vars() if transpose else self.problem.num_rows())
        err = self._err()
        raise_for(self.lib.pdhg_session_spmv(self.h, int(transpose), _dp(v), _dp(out), err, abi.ERRLEN), err)
        return out

    def opnorm(self, iters: int = 100, seed: int = 0) -> float:
        o = C.c_double()
        err = self._err()
        raise_for(self.lib.pdhg_session_opnorm(self.h, iters, seed, C.byref(o), err, abi.ERRLEN), err)
        return o.value

    def time_kernels(self, iters: int = 200):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        err = self._err()
        raise_for(self.lib.pdhg_session_time_kernels(self.h, iters, C.byref(a), C.byref(b), C.byref(c), err,
                                                     abi.ERRLEN), err)
        return a.value, b.value, c.value

    def time_kernels_cold(self, iters: int = 64):
        """(primal, dual, iteration) mean ms per launch with L2 swept clean
        before every launch (pdhg_session_time_kernels_cold)."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        err = self._err()
        raise_for(self.lib.pdhg_session_time_kernels_cold(self.h, iters, C.byref(a), C.byref(b), C.byref(c), err,
                                                          abi.ERRLEN), err)
        return a.value, b.value, c.value

    def run_block(self, iters: int = 64, profiler_range: bool = False) -> None:
        err = self._err()
        raise_for(self.lib.pdhg_session_run_block(self.h, iters, int(profiler_range), err, abi.ERRLEN), err)

    def time_check(self, iters: int = 50):
        """(device ms, wall ms) per termination/restart check (solver.cpp:390-428)."""
        a, b = C.c_double(), C.c_double()
        err = self._err()
        raise_for(self.lib.pdhg_session_time_check(self.h, iters, C.byref(a), C.byref(b), err, abi.ERRLEN), err)
        return a.value, b.value


def PrimalStep(problem: LpProblem, x, y, eta: float, omega: float) -> np.ndarray:
    """solver.cpp:112-129 on the unscaled problem (device)."""
    lib = abi.load()
    lp = problem.to_c()
    xa, ya, out = _f64(x), _f64(y), np.empty(problem.num_vars())
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(lib.pdhg_primal_step(C.byref(lp), _dp(xa), _dp(ya), eta, omega, _dp(out), err, abi.ERRLEN), err)
    return out


def DualStep(problem: LpProblem, x_new, x_old, y, eta: float, omega: float) -> np.ndarray:
    """solver.cpp:131-154 on the unscaled problem (device)."""
    lib = abi.load()
    lp = problem.to_c()
    a, b, ya, out = _f64(x_new), _f64(x_old), _f64(y), np.empty(problem.num_rows())
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(lib.pdhg_dual_step(C.byref(lp), _dp(a), _dp(b), _dp(ya), eta, omega, _dp(out), err, abi.ERRLEN), err)
    return out


# ------------------------------------------- host decision logic (no device)
def ShouldRestart(params: SolverParams, t: int, k: int, kkt_candidate: float, kkt_loop_start: float,
                  kkt_prev_candidate: float) -> bool:
    """solver.cpp:178-189."""
    prm = params.to_c()
    return bool(abi.load().pdhg_should_restart(C.byref(prm), t, k, kkt_candidate, kkt_loop_start,
                                               kkt_prev_candidate))


def UpdatePrimalWeight(omega: float, dx_norm: float, dy_norm: float) -> float:
    """solver.cpp:191-196."""
    return abi.load().pdhg_update_primal_weight(omega, dx_norm, dy_norm)


def KktError(primal_res: float, dual_res: float, gap: float, omega: float) -> float:
    """kkt.cpp:153-157."""
    return abi.load().pdhg_kkt_error(primal_res, dual_res, gap, omega)


def CheckTermination(report: ResidualReport, eps: float) -> bool:
    """kkt.cpp:147-151."""
    r = abi.Report(*(getattr(report, k) for k, _ in abi.Report._fields_))
    return bool(abi.load().pdhg_check_termination(C.byref(r), eps))


# --------------------------------------- scaling / residual utilities
@dataclass
class ScalingInfo:
    """scaling.hpp:30-38: positive diagonal scales of K = [A; G]."""
    row_scale: np.ndarray
    col_scale: np.ndarray

    @staticmethod
    def Identity(n_rows: int, n_cols: int) -> "ScalingInfo":
        return ScalingInfo(np.ones(n_rows), np.ones(n_cols))

    def Composed(self, other: "ScalingInfo") -> "ScalingInfo":
        return ScalingInfo(self.row_scale * other.row_scale, self.col_scale * other.col_scale)

    def UnscaleIterate(self, x: np.ndarray, y: np.ndarray) -> None:
        x *= self.col_scale
        y *= self.row_scale


def _scaling(k: CsrMatrix, iters: int, alpha: float, stages: int) -> ScalingInfo:
    rs, cs = np.empty(k.rows), np.empty(k.cols)
    csr = k.to_c()
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(abi.load().pdhg_compute_scaling(C.byref(csr), iters, alpha, stages, _dp(rs), _dp(cs), err,
                                              abi.ERRLEN), err)
    return ScalingInfo(rs, cs)


def RuizEquilibrate(k: CsrMatrix, iters: int) -> ScalingInfo:
    """scaling.cpp:49-68 (device)."""
    return _scaling(k, iters, 1.0, 1)


def PockChambolleScale(k: CsrMatrix, alpha: float) -> ScalingInfo:
    """scaling.cpp:70-84 (device)."""
    return _scaling(k, 0, alpha, 2)


def ComputeScaling(k: CsrMatrix, config: Optional[ScalingConfig] = None) -> ScalingInfo:
    """scaling.cpp:86-91: Ruiz sweeps, then PC on the Ruiz-scaled matrix, composed."""
    config = config or ScalingConfig()
    if not config.enabled:
        return ScalingInfo.Identity(k.rows, k.cols)
    return _scaling(k, config.ruiz_iters, config.pc_alpha, 3)


def ApplyScaling(problem: LpProblem, info: ScalingInfo) -> LpProblem:
    """scaling.cpp:93-116 (host; same operations and rounding order)."""
    m1, m2 = problem.num_eq_rows(), problem.num_ineq_rows()
    if len(info.row_scale) != m1 + m2 or len(info.col_scale) != problem.num_vars():
        raise ValueError("scaling dimensions do not match problem")
    er, ir = info.row_scale[:m1], info.row_scale[m1:]

    def scaled(m: CsrMatrix, rs) -> CsrMatrix:  # Scaled: (rs * v) * cs (sparse_matrix.cpp:213)
        rows = np.repeat(np.arange(m.rows), np.diff(m.row_ptr))
        return CsrMatrix(m.rows, m.cols, m.row_ptr.copy(), m.col_idx.copy(),
                         (rs[rows] * m.values) * info.col_scale[m.col_idx])

    return LpProblem(scaled(problem.a, er), scaled(problem.g, ir), problem.c * info.col_scale, problem.b * er,
                     problem.h * ir, problem.l / info.col_scale, problem.u / info.col_scale, problem.objective_offset,
                     problem.negated_objective, problem.name)


def ComputeResiduals(problem: LpProblem, x, y) -> ResidualReport:
    """kkt.cpp:143-145 on the original problem (device)."""
    lp = problem.to_c()
    rep = abi.Report()
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(abi.load().pdhg_residuals(C.byref(lp), _dp(_f64(x)), _dp(_f64(y)), C.byref(rep), err, abi.ERRLEN),
              err)
    return ResidualReport.from_c(rep)


def KktOmega(problem: LpProblem, x, y, omega: float) -> float:
    """kkt.cpp:159-161."""
    r = ComputeResiduals(problem, x, y)
    return KktError(r.primal_res, r.dual_res, r.gap_abs, omega)


def ChooseRestartCandidate(problem: LpProblem, z_cur, z_avg, omega: float):
    """solver.cpp:170-176: (x, y) of the current iterate when its KKT_omega
    error is strictly smaller, else the average (ties -> average)."""
    cur = KktOmega(problem, z_cur[0], z_cur[1], omega)
    avg = KktOmega(problem, z_avg[0], z_avg[1], omega)
    return z_cur if cur < avg else z_avg


def DeriveLambda(problem: LpProblem, y) -> np.ndarray:
    """kkt.cpp:127-141 (device)."""
    lp = problem.to_c()
    out = np.empty(problem.num_vars())
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(abi.load().pdhg_derive_lambda(C.byref(lp), _dp(_f64(y)), _dp(out), err, abi.ERRLEN), err)
    return out


def PartitionBlocks(ptr, parts: int, seg_weight: int = 6) -> np.ndarray:
    """The balanced contiguous split every rank computes (host_logic.h)."""
    p = _i64(ptr)
    out = np.empty(parts + 1, np.int64)
    code = abi.load().pdhg_partition_blocks(_i64p(p), len(p) - 1, parts, seg_weight, _i64p(out))
    raise_for(code, b"invalid partition arguments")
    return out


# ---------------------------------------------- host-owned instances
class _InstanceOwner:
    """Frees a generated pdhg_instance once no array view into it is alive."""

    def __init__(self, h: C.c_void_p):
        self.h = h

    def __del__(self):
        if self.h:
            abi.load().pdhg_instance_free(self.h)
            self.h = None


def _from_instance(h: C.c_void_p, name: str) -> LpProblem:
    """Zero-copy view of a generated instance: every array's buffer keeps the
    owner alive, so multi-GB instances are never duplicated on the host."""
    lib = abi.load()
    owner = _InstanceOwner(h)
    v = abi.Lp()
    lib.pdhg_instance_view(h, C.byref(v))

    def arr(p, n, ct, dt):
        if not n:
            return np.zeros(0, dt)
        buf = (ct * n).from_address(C.cast(p, C.c_void_p).value)
        buf._owner = owner
        return np.frombuffer(buf, dtype=dt)

    def csr(m: abi.Csr) -> CsrMatrix:
        ptr = arr(m.row_ptr, m.rows + 1, C.c_int64, np.int64)
        nz = int(ptr[-1])
        return CsrMatrix(m.rows, m.cols, ptr, arr(m.col_idx, nz, C.c_int64, np.int64),
                         arr(m.values, nz, C.c_double, np.float64))

    d = lambda p, n: arr(p, n, C.c_double, np.float64)  # noqa: E731
    a, g = csr(v.a), csr(v.g)
    own_name = (lib.pdhg_instance_name(h) or b"").decode()
    p = LpProblem(a, g, d(v.c, v.n), d(v.b, a.rows), d(v.h, g.rows), d(v.l, v.n), d(v.u, v.n),
                  v.objective_offset, bool(v.negated_objective), own_name or name)
    w = lib.pdhg_instance_witness(h)
    p.witness = d(w, v.n) if w else None
    return p


def _gen(fn, *args, name=""):
    lib = abi.load()
    h = C.c_void_p()
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(getattr(lib, fn)(*args, C.byref(h), err, abi.ERRLEN), err)
    return h


# ------------------------------------------------------------------ MPS
def _mps_result(code, h, err, line):
    if code == abi.PDHG_PARSE_ERROR:
        raise MpsParseError(err.value.decode(errors="replace"), line.value)
    if code == abi.PDHG_IO_ERROR:
        raise OSError(err.value.decode(errors="replace"))
    raise_for(code, err)
    return _from_instance(h, "")


def ParseMpsString(text, fixed_format: bool = False) -> LpProblem:
    """ParseMpsString (mps.hpp:53, mps_reader.cpp) -- same normalisations and
    errors; MpsParseError carries the line number."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h, err, line = C.c_void_p(), C.create_string_buffer(abi.ERRLEN), C.c_int(0)
    code = abi.load().pdhg_mps_read_string(data, len(data), int(fixed_format), C.byref(h), err, abi.ERRLEN,
                                           C.byref(line))
    return _mps_result(code, h, err, line)


def ParseMpsFile(path, fixed_format: bool = False) -> LpProblem:
    """ParseMpsFile (mps.hpp:55): plain or .gz (zlib)."""
    h, err, line = C.c_void_p(), C.create_string_buffer(abi.ERRLEN), C.c_int(0)
    code = abi.load().pdhg_mps_read_file(str(path).encode(), int(fixed_format), C.byref(h), err, abi.ERRLEN,
                                         C.byref(line))
    return _mps_result(code, h, err, line)


def WriteMps(problem: LpProblem) -> str:
    """WriteMps (mps_writer.cpp:37-107): free format, %.17g."""
    lib = abi.load()
    lp = problem.to_c()
    out, n, err = C.c_void_p(), C.c_size_t(0), C.create_string_buffer(abi.ERRLEN)
    raise_for(lib.pdhg_mps_write_string(C.byref(lp), (problem.name or "").encode(), C.byref(out), C.byref(n), err,
                                        abi.ERRLEN), err)
    try:
        return C.string_at(out, n.value).decode()
    finally:
        lib.pdhg_free_string(out)


def WriteMpsFile(problem: LpProblem, path) -> None:
    lp = problem.to_c()
    err = C.create_string_buffer(abi.ERRLEN)
    code = abi.load().pdhg_mps_write_file(C.byref(lp), (problem.name or "").encode(), str(path).encode(), err,
                                          abi.ERRLEN)
    if code == abi.PDHG_IO_ERROR:
        raise OSError(err.value.decode(errors="replace"))
    raise_for(code, err)


# ------------------------------------------------------------ generators
def GenRandomLp(m: int, n: int, density: float, seed: int, equality_rows: int = 0) -> LpProblem:
    """instance_gen.cpp:143-188; `equality_rows` moves the first rows of G into
    A with b = A x_hat."""
    lib = abi.load()
    h = _gen("pdhg_gen_random_lp", m, n, density, seed)
    if equality_rows:
        err = C.create_string_buffer(abi.ERRLEN)
        code = lib.pdhg_instance_make_equalities(h, equality_rows, err, abi.ERRLEN)
        if code:
            lib.pdhg_instance_free(h)
            raise_for(code, err)
    return _from_instance(h, f"rand_{m}x{n}_s{seed}")


def GenPagerank(n_nodes: int, damping: float = 0.85, attachment: int = 3, seed: int = 0) -> LpProblem:
    """instance_gen.cpp:27-64, 90-141."""
    return _from_instance(_gen("pdhg_gen_pagerank", n_nodes, damping, attachment, seed), "pagerank")


def GenPagerankGraph(n_nodes: int, damping: float = 0.85, attachment: int = 3, seed: int = 0) -> np.ndarray:
    """instance_gen.cpp:27-64: (count, 2) int64 array of src -> dst edges."""
    lib = abi.load()
    cap = max(int(lib.pdhg_pagerank_graph_edges(n_nodes, attachment)), 1)
    e = np.empty((cap, 2), np.int64)
    cnt = C.c_int64(0)
    err = C.create_string_buffer(abi.ERRLEN)
    raise_for(lib.pdhg_gen_pagerank_graph(n_nodes, damping, attachment, seed, _i64p(e), cap, C.byref(cnt), err,
                                          abi.ERRLEN), err)
    return e[:cnt.value].copy()


def BuildPagerankLp(edges, n_nodes: int, damping: float = 0.85) -> LpProblem:
    """instance_gen.cpp:90-137 over a (count, 2) src -> dst edge array."""
    e = np.ascontiguousarray(np.asarray(edges, np.int64).reshape(-1, 2))
    return _from_instance(_gen("pdhg_build_pagerank_lp", _i64p(e), e.shape[0], n_nodes, damping), "pagerank")


def ReadEdgeList(path):
    """instance_gen.cpp:66-88: "src dst" per line, '#' comment lines; ids
    compacted to 0..n-1 in order of first appearance. Returns (edges, n)."""
    ids, edges = {}, []
    with open(path) as f:
        for line in f:
            s = line.lstrip(" \t\r")
            if not s.strip() or s.startswith("#"):
                continue
            parts = line.split()
            try:
                a, b = int(parts[0]), int(parts[1])
            except (IndexError, ValueError):
                raise RuntimeError("malformed edge line: " + line.rstrip("\n")) from None
            ia = ids.setdefault(a, len(ids))
            ib = ids.setdefault(b, len(ids))
            edges.append((ia, ib))
    return np.asarray(edges, np.int64).reshape(-1, 2), len(ids)


def GenTransport(sources: int, sinks: int, seed: int = 1) -> LpProblem:
    """Transportation LP of SURVEY §8d config 2."""
    return _from_instance(_gen("pdhg_gen_transport", sources, sinks, seed), f"transport_{sources}x{sinks}_s{seed}")


def GenMcf(nodes: int, arcs: int, commodities: int, seed: int = 1) -> LpProblem:
    """Multicommodity network flow LP of SURVEY §8d config 3 (heavy-tailed
    conservation rows, capacity rows of length `commodities`, columns of 3)."""
    return _from_instance(_gen("pdhg_gen_mcf", nodes, arcs, commodities, seed),
                          f"mcf_{nodes}v_{arcs}a_{commodities}k_s{seed}")


def GenStaircase(stages: int, rows_per_stage: int, cols_per_stage: int, nnz_per_row: int = 20,
                 linking_per_row: int = 5, eq_rows_per_stage: Optional[int] = None, seed: int = 1,
                 threads: int = 0) -> LpProblem:
    """Block-angular staircase LP of SURVEY §8d config 5; bit-identical per
    seed for any `threads` (0 = all host cores)."""
    req = rows_per_stage // 2 if eq_rows_per_stage is None else eq_rows_per_stage
    return _from_instance(_gen("pdhg_gen_staircase", stages, rows_per_stage, cols_per_stage, nnz_per_row,
                               linking_per_row, req, seed, threads),
                          f"staircase_{stages}x{rows_per_stage}x{cols_per_stage}_d{nnz_per_row}_s{seed}")
