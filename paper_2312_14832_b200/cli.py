"""Command line front-end (reference proj/tools/rpdlp_main.cpp:126-220):

    python -m paper_2312_14832_b200.cli solve FILE [--eps E] [--time-limit S] [--iter-limit N]
        [--log-every N] [--check-every N] [--seed S] [--ruiz-iters N] [--pc-alpha A]
        [--out SOLUTION.json] [--no-scaling] [--no-restarts] [--adaptive-step] [--strict-mps] [--device D]
    python -m paper_2312_14832_b200.cli bench DIR [--eps E] [--time-limit S] [--iter-limit N] [--seed S]
        [--delta D] [--report R.json] [--csv R.csv] [--no-scaling] [--redact-timing] [--device D]
    python -m paper_2312_14832_b200.cli gen pagerank --nodes N [--damping D] [--attachment A] [--seed S] --out F
    python -m paper_2312_14832_b200.cli gen random --rows M --cols N [--density D] [--seed S] --out F
    python -m paper_2312_14832_b200.cli gen transport|mcf|staircase ... --out F      (SURVEY §8d shapes)

Exit codes as the reference: 0 ok, 2 limit reached, 3 input error,
4 numerical failure.
"""
from __future__ import annotations

import argparse
import json
import sys

from . import rpdlp, suite

EXIT_OK, EXIT_LIMIT, EXIT_INPUT, EXIT_NUMERICAL = 0, 2, 3, 4


def _params(a) -> rpdlp.SolverParams:
    p = rpdlp.SolverParams()
    for k in ("eps", "time_limit", "iter_limit", "seed", "log_every", "check_every"):
        v = getattr(a, k, None)
        if v is not None:
            setattr(p, k, v)
    if getattr(a, "ruiz_iters", None) is not None:
        p.scaling.ruiz_iters = a.ruiz_iters
    if getattr(a, "pc_alpha", None) is not None:
        p.scaling.pc_alpha = a.pc_alpha
    p.scaling.enabled = not a.no_scaling
    if getattr(a, "no_restarts", False):
        p.restart_enabled = False
    if getattr(a, "adaptive_step", False):
        p.adaptive_step = True
    return p


def run_solve(a) -> int:
    try:
        problem = rpdlp.ParseMpsFile(a.file, fixed_format=a.strict_mps)
    except Exception as e:  # noqa: BLE001 -- parse and I/O errors alike
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    params = _params(a)
    try:
        r = rpdlp.Solve(problem, params, device=a.device)
    except rpdlp.NumericalFailure as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    sign = -1.0 if problem.negated_objective else 1.0
    print("status=%s objective=%.12e iterations=%d restarts=%d solve_seconds=%.3f"
          % (rpdlp.ToString(r.status), sign * r.report.primal_obj, r.iterations, r.restarts, r.solve_seconds))
    if a.out:
        try:
            with open(a.out, "w") as f:
                f.write(json.dumps(suite.SolutionToJson(r, problem.negated_objective), indent=2) + "\n")
        except OSError:
            print(f"error: cannot write {a.out}", file=sys.stderr)
            return EXIT_INPUT
    return EXIT_OK if r.status == rpdlp.SolveStatus.kOptimal else EXIT_LIMIT


def run_bench(a) -> int:
    try:
        s = suite.RunSuite(a.dir, _params(a), a.delta, device=a.device)
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    for r in s.records:
        print("instance=%s status=%s solve_seconds=%.3f iterations=%d" % (r.instance, r.status, r.solve_seconds,
                                                                          r.iterations))
    print("solved=%d/%d sgm10=%.4f" % (s.solved_count, len(s.records), s.sgm10))
    try:
        if a.report:
            suite.WriteSummaryJson(s, a.report, a.redact_timing)
        if a.csv:
            suite.WriteSummaryCsv(s, a.csv)
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    return EXIT_OK


def run_gen(a) -> int:
    if a.kind == "pagerank":
        p = rpdlp.GenPagerank(a.nodes, a.damping, a.attachment, a.seed)
    elif a.kind == "random":
        p = rpdlp.GenRandomLp(a.rows, a.cols, a.density, a.seed)
    elif a.kind == "transport":
        p = rpdlp.GenTransport(a.sources, a.sinks, a.seed)
    elif a.kind == "mcf":
        p = rpdlp.GenMcf(a.nodes, a.arcs, a.commodities, a.seed)
    else:
        p = rpdlp.GenStaircase(a.stages, a.rows_per_stage, a.cols_per_stage, a.nnz_per_row, a.linking_per_row,
                               seed=a.seed)
    rpdlp.WriteMpsFile(p, a.out)
    return EXIT_OK


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="rpdlp-b200", description="Restarted primal-dual hybrid gradient LP solver "
                                 "(B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="Solve a single MPS file")
    s.add_argument("file")
    s.add_argument("--eps", type=float)
    s.add_argument("--time-limit", type=float)
    s.add_argument("--iter-limit", type=int)
    s.add_argument("--log-every", type=int)
    s.add_argument("--check-every", type=int)
    s.add_argument("--seed", type=int)
    s.add_argument("--ruiz-iters", type=int)
    s.add_argument("--pc-alpha", type=float)
    s.add_argument("--out", default="")
    s.add_argument("--no-scaling", action="store_true")
    s.add_argument("--no-restarts", action="store_true")
    s.add_argument("--adaptive-step", action="store_true")
    s.add_argument("--strict-mps", action="store_true")
    s.add_argument("--device", type=int, default=0)
    b = sub.add_parser("bench", help="Solve a directory of MPS files")
    b.add_argument("dir")
    b.add_argument("--eps", type=float)
    b.add_argument("--time-limit", type=float)
    b.add_argument("--iter-limit", type=int)
    b.add_argument("--seed", type=int)
    b.add_argument("--delta", type=float, default=10.0)
    b.add_argument("--report", default="")
    b.add_argument("--csv", default="")
    b.add_argument("--no-scaling", action="store_true")
    b.add_argument("--redact-timing", action="store_true")
    b.add_argument("--device", type=int, default=0)
    g = sub.add_parser("gen", help="Generate synthetic instances")
    gs = g.add_subparsers(dest="kind", required=True)
    pr = gs.add_parser("pagerank")
    pr.add_argument("--nodes", type=int, required=True)
    pr.add_argument("--damping", type=float, default=0.85)
    pr.add_argument("--attachment", type=int, default=3)
    pr.add_argument("--seed", type=int, default=0)
    pr.add_argument("--out", required=True)
    rd = gs.add_parser("random")
    rd.add_argument("--rows", type=int, required=True)
    rd.add_argument("--cols", type=int, required=True)
    rd.add_argument("--density", type=float, default=0.5)
    rd.add_argument("--seed", type=int, default=0)
    rd.add_argument("--out", required=True)
    tr = gs.add_parser("transport")
    tr.add_argument("--sources", type=int, required=True)
    tr.add_argument("--sinks", type=int, required=True)
    tr.add_argument("--seed", type=int, default=1)
    tr.add_argument("--out", required=True)
    mc = gs.add_parser("mcf")
    mc.add_argument("--nodes", type=int, required=True)
    mc.add_argument("--arcs", type=int, required=True)
    mc.add_argument("--commodities", type=int, required=True)
    mc.add_argument("--seed", type=int, default=1)
    mc.add_argument("--out", required=True)
    st = gs.add_parser("staircase")
    st.add_argument("--stages", type=int, required=True)
    st.add_argument("--rows-per-stage", type=int, required=True)
    st.add_argument("--cols-per-stage", type=int, required=True)
    st.add_argument("--nnz-per-row", type=int, default=20)
    st.add_argument("--linking-per-row", type=int, default=5)
    st.add_argument("--seed", type=int, default=1)
    st.add_argument("--out", required=True)
    return ap


def main(argv=None) -> int:
    a = parser().parse_args(argv)
    if a.cmd != "solve":
        a.no_restarts = getattr(a, "no_restarts", False)
    try:
        if a.cmd == "solve":
            return run_solve(a)
        if a.cmd == "bench":
            return run_bench(a)
        return run_gen(a)
    except Exception as e:  # noqa: BLE001 -- rpdlp_main.cpp:212-215
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
