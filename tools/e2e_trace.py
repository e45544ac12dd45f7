"""End-to-end (pdhg_solve_on, pinned host buffers) phase trace of the bench
workload: `PDHG_TRACE=2 python tools/e2e_trace.py [--solves N] [--config C]`.
Prints the wall time per solve and the session's per-phase construction /
teardown times (stderr)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2312_14832_b200 import rpdlp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="transport")
    ap.add_argument("--solves", type=int, default=4)
    ap.add_argument("--eps", type=float, default=1e-4)
    a = ap.parse_args()
    args = argparse.Namespace(config=a.config, eps=a.eps, transport=1000, pagerank_n=1_000_000,
                              mcf=(50_000, 330_000, 50), staircase=(5, 10_000_000, 20))
    problem, workload = bench.make_problem(a.config, args)
    pinned = bench.pinned_copy(problem)
    prm = rpdlp.SolverParams(eps=a.eps)
    for k in range(a.solves):
        t = time.perf_counter()
        r = rpdlp.Solve(pinned, prm)
        dt = time.perf_counter() - t
        print(f"solve {k}: {dt:.4f}s status={int(r.status)} it={r.iterations} -> {r.iterations / dt:.0f} it/s",
              flush=True)


if __name__ == "__main__":
    main()
