"""Full-scale golden traces for BASELINE configs 2-4, from the REFERENCE build.

    make -C oracle ref
    python tests/golden/make_fullscale.py transport        # ~4 min, eps 1e-4 full solve
    python tests/golden/make_fullscale.py transport_tight  # ~25 min, eps 1e-8 full solve
    python tests/golden/make_fullscale.py mcf              # ~6 min, iter_limit 192
    python tests/golden/make_fullscale.py pagerank         # ~10 min, iter_limit 128

Writes tests/golden/fullscale_<name>.json: the instance digest (sha256 over
every array, so the GPU test proves it rebuilt the same LP), the reference
solve's status / counts / report, and its EvalObserver decision trace
(solver.cpp:390-428: one record per check). Every number comes from the
unmodified reference rpdlp (oracle/_ref/librpdlp_ref.so, compiled from
/root/reference by oracle/Makefile); the GPU box has no /root/reference, so
tests/test_gpu_fullscale.py reads these fixtures.

Instances: transport = the reference-side generator in oracle/ref_shim.cpp
(pinned to the product's GenTransport by tests/test_oracle.py); pagerank =
the reference's own GenPagerank; mcf = the product's GenMcf (the reference has
no MCF generator) -- the generator is not what these fixtures pin.
Configs 3 and 4 cannot be solved to eps on a CPU in reasonable time (SURVEY
§8d: ~1.6 and 0.46 it/s), so their fixtures are iteration-limited runs whose
first checks the GPU trace must reproduce.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402
from paper_2312_14832_b200.rpdlp import SolverParams  # noqa: E402

TRACE_FIELDS = ("iteration", "inner_iteration", "restarts", "omega", "eta", "kkt_candidate", "kkt_loop_start",
                "candidate_is_current", "restarted")
REPORT_FIELDS = ("primal_res", "dual_res", "gap_abs", "primal_obj", "dual_obj", "rel_primal", "rel_dual", "rel_gap")

CASES = {
    # name: (instance builder spec, params)
    "transport": ({"kind": "transport", "sources": 1000, "sinks": 1000, "seed": 1}, {"eps": 1e-4}),
    "transport_tight": ({"kind": "transport", "sources": 1000, "sinks": 1000, "seed": 1}, {"eps": 1e-8}),
    "mcf": ({"kind": "mcf", "nodes": 50_000, "arcs": 330_000, "commodities": 50, "seed": 1},
            {"eps": 1e-4, "iter_limit": 192}),
    "pagerank": ({"kind": "pagerank", "nodes": 10_000_000, "damping": 0.85, "attachment": 6, "seed": 1},
                 {"eps": 1e-4, "iter_limit": 128}),
}


def digest(p) -> str:
    h = hashlib.sha256()
    for a in (p.a.row_ptr, p.a.col_idx, p.a.values, p.g.row_ptr, p.g.col_idx, p.g.values, p.c, p.b, p.h, p.l, p.u):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def build(spec, ref):
    k = spec["kind"]
    if k == "transport":
        return ref.gen_transport(spec["sources"], spec["sinks"], spec["seed"])
    if k == "pagerank":
        return ref.gen_pagerank(spec["nodes"], spec["damping"], spec["attachment"], spec["seed"])
    if k == "mcf":
        from paper_2312_14832_b200 import rpdlp
        return rpdlp.GenMcf(spec["nodes"], spec["arcs"], spec["commodities"], spec["seed"])
    raise ValueError(k)


def main(name: str) -> None:
    ref = oracle.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/librpdlp_ref.so not built (make -C oracle ref)")
    spec, prm = CASES[name]
    t0 = time.time()
    p = build(spec, ref)
    dg = digest(p)
    print(f"[{name}] built m={p.num_rows()} n={p.num_vars()} nnz={p.nnz()} in {time.time() - t0:.1f}s", flush=True)
    trace = []

    def obs(e):
        rec = {f: (bool(getattr(e, f)) if f in ("candidate_is_current", "restarted") else getattr(e, f))
               for f in TRACE_FIELDS}
        rec["report"] = {f: getattr(e.original_report, f) for f in REPORT_FIELDS}
        trace.append(rec)
        print(f"[{name}] check it={e.iteration} restarted={e.restarted} kkt={e.kkt_candidate:.6e}", flush=True)

    t1 = time.time()
    r = ref.solve(p, SolverParams(**prm), obs)
    out = {
        "case": name, "instance": spec, "params": prm, "digest": dg,
        "m": p.num_rows(), "n": p.num_vars(), "nnz": p.nnz(),
        "status": int(r.status), "iterations": r.iterations, "restarts": r.restarts,
        "report": {f: getattr(r.report, f) for f in REPORT_FIELDS},
        "solve_seconds": r.solve_seconds, "scaling_seconds": r.scaling_seconds,
        "restart_iterations": [t["iteration"] for t in trace if t["restarted"]],
        "trace": trace,
        "generator": "reference build (oracle/_ref/librpdlp_ref.so), tests/golden/make_fullscale.py",
    }
    (HERE / f"fullscale_{name}.json").write_text(json.dumps(out, indent=1) + "\n")
    print(f"[{name}] status={int(r.status)} it={r.iterations} restarts={r.restarts} "
          f"pobj={r.report.primal_obj!r} in {time.time() - t1:.1f}s", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        main(a)
