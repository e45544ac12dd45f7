"""Benchmark-suite harness over the B200 solver (reference
proj/core/include/rpdlp/bench.hpp:27-72, proj/core/src/bench.cpp:50-179):
SGM10, RunSuite over a directory of MPS files, JSON / CSV reports, the
solution JSON of the `solve` subcommand. Same record fields, key order,
statuses and error handling as the reference; the records additionally carry
`it_per_s` and the device ("it/s and time-to-eps fields").
"""
from __future__ import annotations

import json
import math
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from .rpdlp import ParseMpsFile, ResidualReport, Solve, SolveResult, SolverParams, ToString


@dataclass
class BenchRecord:
    """bench.hpp:27-38."""
    instance: str = ""
    status: str = ""  # Optimal | IterLimit | TimeLimit | Error
    solve_seconds: float = 0.0  # iteration loop only; parse/scaling excluded
    parse_seconds: float = 0.0
    scaling_seconds: float = 0.0
    iterations: int = 0
    restarts: int = 0
    residuals: ResidualReport = field(default_factory=lambda: ResidualReport(*([0.0] * 8)))
    message: str = ""  # set when status == Error

    def solved(self) -> bool:
        return self.status == "Optimal"


@dataclass
class SuiteSummary:
    """bench.hpp:40-47."""
    records: List[BenchRecord] = field(default_factory=list)
    sgm10: float = 0.0
    solved_count: int = 0
    tolerance: float = 0.0
    delta: float = 10.0
    time_limit: float = 3600.0


def Sgm(times: Sequence[float], delta: float, time_limit: float, solved_flags: Sequence[bool]) -> float:
    """Shifted geometric mean (prod(t_i + delta))^(1/n) - delta in log space;
    unsolved entries count time_limit (bench.cpp:50-63)."""
    if len(times) == 0:
        raise ValueError("SGM of an empty list")
    if len(times) != len(solved_flags):
        raise ValueError("times/solved_flags length mismatch")
    if delta < 0.0:
        raise ValueError("negative SGM shift")
    log_sum = 0.0
    for t, ok in zip(times, solved_flags):
        log_sum += math.log((t if ok else time_limit) + delta)
    return math.exp(log_sum / len(times)) - delta


def _is_mps(name: str) -> bool:
    return name.endswith(".mps") or name.endswith(".mps.gz")


def RunSuite(directory: str, params: Optional[SolverParams] = None, delta: float = 10.0,
             device: int = 0) -> SuiteSummary:
    """Solves every *.mps / *.mps.gz under `directory`, sorted by name;
    per-instance failures become Error records (bench.cpp:65-114)."""
    params = params or SolverParams()
    files = sorted(f for f in os.listdir(directory)
                   if _is_mps(f) and os.path.isfile(os.path.join(directory, f)))
    s = SuiteSummary(tolerance=params.eps, delta=delta, time_limit=params.time_limit)
    for f in files:
        rec = BenchRecord(instance=f)
        try:
            t0 = time.perf_counter()
            problem = ParseMpsFile(os.path.join(directory, f))
            rec.parse_seconds = time.perf_counter() - t0
            r = Solve(problem, params, device=device)
            rec.status = ToString(r.status)
            rec.solve_seconds = r.solve_seconds
            rec.scaling_seconds = r.scaling_seconds
            rec.iterations = r.iterations
            rec.restarts = r.restarts
            rec.residuals = r.report
        except Exception as e:  # noqa: BLE001 -- the reference records every failure
            rec.status = "Error"
            rec.message = str(e)
        s.records.append(rec)
    if s.records:
        s.solved_count = sum(r.solved() for r in s.records)
        s.sgm10 = Sgm([r.solve_seconds for r in s.records], delta, params.time_limit,
                      [r.solved() for r in s.records])
    return s


def _residuals(r: ResidualReport) -> dict:
    return {"primal_res": r.primal_res, "dual_res": r.dual_res, "gap_abs": r.gap_abs, "primal_obj": r.primal_obj,
            "dual_obj": r.dual_obj, "rel_primal": r.rel_primal, "rel_dual": r.rel_dual, "rel_gap": r.rel_gap}


def SummaryToJson(summary: SuiteSummary, redact_timing: bool = False) -> dict:
    """Deterministic key order; `redact_timing` zeroes wall-clock fields
    (bench.cpp:116-141). `it_per_s` is a B200 addition (also redacted)."""
    records = []
    for r in summary.records:
        rec = {"instance": r.instance, "status": r.status,
               "solve_seconds": 0.0 if redact_timing else r.solve_seconds,
               "parse_seconds": 0.0 if redact_timing else r.parse_seconds,
               "scaling_seconds": 0.0 if redact_timing else r.scaling_seconds,
               "iterations": r.iterations, "restarts": r.restarts, "residuals": _residuals(r.residuals),
               "it_per_s": 0.0 if redact_timing or r.solve_seconds <= 0 else r.iterations / r.solve_seconds}
        if r.message:
            rec["message"] = r.message
        records.append(rec)
    return {"tolerance": summary.tolerance, "delta": summary.delta, "time_limit": summary.time_limit,
            "solved_count": summary.solved_count, "sgm10": 0.0 if redact_timing else summary.sgm10,
            "records": records}


def WriteSummaryJson(summary: SuiteSummary, path: str, redact_timing: bool = False) -> None:
    with open(path, "w") as f:
        f.write(json.dumps(SummaryToJson(summary, redact_timing), indent=2) + "\n")


def WriteSummaryCsv(summary: SuiteSummary, path: str) -> None:
    """bench.cpp:150-165 (same columns and number formats)."""
    with open(path, "w") as f:
        f.write("instance,status,solve_seconds,parse_seconds,scaling_seconds,"
                "iterations,restarts,rel_primal,rel_dual,rel_gap,primal_obj\n")
        for r in summary.records:
            f.write("%s,%s,%.6f,%.6f,%.6f,%d,%d,%.6e,%.6e,%.6e,%.12e\n" % (
                r.instance, r.status, r.solve_seconds, r.parse_seconds, r.scaling_seconds, r.iterations,
                r.restarts, r.residuals.rel_primal, r.residuals.rel_dual, r.residuals.rel_gap,
                r.residuals.primal_obj))


def SolutionToJson(result: SolveResult, negated_objective: bool) -> dict:
    """Solution file of the solve subcommand; objectives negated back for a
    maximization (bench.cpp:167-179)."""
    sign = -1.0 if negated_objective else 1.0
    return {"status": ToString(result.status), "primal_objective": sign * result.report.primal_obj,
            "dual_objective": sign * result.report.dual_obj, "iterations": result.iterations,
            "restarts": result.restarts, "x": [float(v) for v in result.x], "y": [float(v) for v in result.y],
            "lambda": [float(v) for v in result.lambda_], "residuals": _residuals(result.report)}
