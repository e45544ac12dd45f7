"""Regenerate tests/golden/golden.npz from the REFERENCE build.

    make -C oracle ref && python tests/golden/make_golden.py

Every value here comes from the unmodified reference rpdlp library
(oracle/_ref/librpdlp_ref.so, compiled from /root/reference by
oracle/Makefile): instance checksums of its generators, full solve outputs
(status, iteration/restart counts, reports, x/y/lambda, decision traces),
scaling vectors and operator-norm estimates. The fixtures let the CPU tests
pin the oracle restatement and the product's generators on machines where the
reference is absent (the GPU box).
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import oracle  # noqa: E402
from paper_2312_14832_b200.rpdlp import SolverParams  # noqa: E402

import problems  # noqa: E402

TRACE_FIELDS = ("iteration", "inner_iteration", "restarts", "omega", "eta", "kkt_candidate", "kkt_loop_start",
                "candidate_is_current", "restarted")

GEN_RANDOM = [(6, 8, 0.5, 9), (4, 4, 0.8, 301), (4, 4, 0.8, 304), (40, 30, 0.3, 60), (1000, 2000, 0.005, 1),
              (1000, 2000, 0.005, 2), (1000, 2000, 0.005, 3)]
GEN_PAGERANK = [(200, 0.85, 3, 4), (2000, 0.85, 3, 1), (3000, 0.85, 6, 2), (10000, 0.85, 3, 2026)]


def digest(p) -> str:
    h = hashlib.sha256()
    for a in (p.a.row_ptr, p.a.col_idx, p.a.values, p.g.row_ptr, p.g.col_idx, p.g.values, p.c, p.b, p.h, p.l, p.u):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def solve_cases():
    d = dict(problems.small_cases())
    d["config1"] = problems.config1(1)
    d["ref_config1"] = problems.ref_config1(1)
    return d


def main():
    ref = oracle.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/librpdlp_ref.so not built (make -C oracle ref)")
    out = {}
    for (m, n, dens, s) in GEN_RANDOM:
        out[f"gen/random/{m}/{n}/{dens}/{s}"] = np.array(digest(ref.gen_random_lp(m, n, dens, s)))
    for (nn, dmp, att, s) in GEN_PAGERANK:
        out[f"gen/pagerank/{nn}/{dmp}/{att}/{s}"] = np.array(digest(ref.gen_pagerank(nn, dmp, att, s)))
    for name, p in solve_cases().items():
        out[f"instance/{name}"] = np.array(digest(p))
        for eps in (1e-4, 1e-8):
            tr = []
            r = ref.solve(p, SolverParams(eps=eps), observer=tr.append)
            k = f"solve/{name}/{eps:g}"
            out[k + "/meta"] = np.array([int(r.status), r.iterations, r.restarts], np.int64)
            out[k + "/report"] = np.array([getattr(r.report, f) for f in
                                           ("primal_res", "dual_res", "gap_abs", "primal_obj", "dual_obj",
                                            "rel_primal", "rel_dual", "rel_gap")])
            out[k + "/x"], out[k + "/y"], out[k + "/lambda"] = r.x, r.y, r.lambda_
            out[k + "/trace"] = np.array([[float(getattr(e, f)) for f in TRACE_FIELDS] for e in tr]).reshape(-1, 9)
        rs, cs = ref.scaling(p)
        out[f"scaling/{name}/row"], out[f"scaling/{name}/col"] = rs, cs
        out[f"opnorm/{name}"] = np.array([ref.opnorm(p, 100, 0), ref.opnorm(p, 40, 7)])
    np.savez_compressed(HERE / "golden.npz", **out)
    print(f"wrote {len(out)} arrays to {HERE / 'golden.npz'} ({(HERE / 'golden.npz').stat().st_size / 1e3:.0f} kB)")


if __name__ == "__main__":
    main()
