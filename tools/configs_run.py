"""Every BASELINE.json config on one B200: setup, kernel rooflines, solve to
eps = 1e-4 (and 1e-8 where it finishes), the CPU reference beside it.

    python tools/configs_run.py [names...] [--time-limit S] [--json out.jsonl]

names: random transport mcf pagerank10m staircase (default: all). One JSON
object per config on stdout; a markdown table on stderr at the end.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import algorithmic_bytes  # noqa: E402
from paper_2312_14832_b200 import rpdlp  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0

CONFIGS = {
    # BASELINE configs[0]: random LP with equality + inequality rows (CPU-runnable oracle case)
    "random": dict(make=lambda: rpdlp.GenRandomLp(1000, 2000, 0.005, 1, equality_rows=300),
                   tight=True, cpu=lambda p: p),
    # configs[1]: transportation 1000 x 1000 (1M vars, 2M nnz)
    "transport": dict(make=lambda: rpdlp.GenTransport(1000, 1000, 1), tight=True, cpu=lambda p: p),
    # configs[2]: multicommodity flow, skewed rows, ~50M nnz (CPU sample on 1/10 of the arcs)
    "mcf": dict(make=lambda: rpdlp.GenMcf(50_000, 330_000, 50, 1), tight=False,
                cpu=lambda p: rpdlp.GenMcf(50_000, 33_000, 50, 1), cpu_note="CPU sample on E=33k (1/10 of the arcs)"),
    # configs[3]: PageRank n = 10M, ~80M nnz (CPU sample at n = 1M: the reference needs ~7 min of setup at 10M)
    "pagerank10m": dict(make=lambda: rpdlp.GenPagerank(10_000_000, 0.85, 6, 1), tight=False,
                        cpu=lambda p: rpdlp.GenPagerank(1_000_000, 0.85, 6, 1), cpu_note="CPU sample at n=1M"),
    # configs[4]: block-angular staircase, 1e9 nnz (the 1-GPU baseline of the 8-GPU config)
    "staircase": dict(make=lambda: rpdlp.GenStaircase(500, 100_000, 100_000, 20, 5, seed=1), tight=False,
                      cpu=None, cpu_note="not runnable on the host: the reference keeps ~4 matrix copies"),
}


def cpu_rate(p, budget=20.0):
    from oracle import oracle
    ref = oracle.cpu_baseline()
    r0 = ref.solve(p, rpdlp.SolverParams(eps=1e-4, iter_limit=0))
    r1 = ref.solve(p, rpdlp.SolverParams(eps=1e-4, iter_limit=64))
    per = max((r1.solve_seconds - r0.solve_seconds) / max(r1.iterations, 1), 1e-7)
    k = int(max(64, min(100000, budget / per)) // 64 * 64)
    r2 = ref.solve(p, rpdlp.SolverParams(eps=1e-4, iter_limit=k))
    it_s = r2.iterations / max(r2.solve_seconds - r0.solve_seconds, 1e-9)
    return {"it_per_s": it_s, "iterations": r2.iterations, "setup_s": r0.solve_seconds,
            "scaling_s": r2.scaling_seconds, "kind": "reference" if ref is oracle.reference() else "port",
            "threads": 1}


def run(name, time_limit, no_cpu):
    cfg = CONFIGS[name]
    t = time.time()
    p = cfg["make"]()
    gen_s = time.time() - t
    m, n, nnz = p.num_rows(), p.num_vars(), p.nnz()
    out = {"config": name, "m": m, "n": n, "nnz": nnz, "gen_s": gen_s}
    t = time.time()
    with rpdlp.Session(p) as s:
        out["session_s"] = time.time() - t
        st = s.stats()
        out["device_gb"] = st.device_bytes / 1e9
        ms_p, ms_d, ms_it = s.time_kernels(64 if nnz > 1e8 else 256)
        bp, bd, bi = algorithmic_bytes(m, n, nnz, st.uniform_bounds, st.csr_uniform_len, st.csc_uniform_len)
        out["kernels"] = {"primal_us": ms_p * 1e3, "primal_gbs": bp / ms_p / 1e6, "dual_us": ms_d * 1e3,
                          "dual_gbs": bd / ms_d / 1e6, "iter_us": ms_it * 1e3, "iter_gbs": bi / ms_it / 1e6,
                          "iter_frac_of_hbm": bi / ms_it / 1e6 / PEAK, "steady_it_per_s": 1e3 / ms_it}
        for eps in ([1e-4, 1e-8] if cfg["tight"] else [1e-4]):
            s.flush_l2()
            r = s.solve(rpdlp.SolverParams(eps=eps, time_limit=time_limit))
            dev_ms, _ = s.last_solve()
            out[f"eps_{eps:g}"] = {"status": rpdlp.ToString(r.status), "iterations": r.iterations,
                                   "restarts": r.restarts, "device_s": dev_ms / 1e3,
                                   "it_per_s": r.iterations / (dev_ms / 1e3),
                                   "rel_primal": r.report.rel_primal, "rel_dual": r.report.rel_dual,
                                   "rel_gap": r.report.rel_gap, "primal_obj": r.report.primal_obj}
            print(f"  {name} eps={eps:g}: {out[f'eps_{eps:g}']}", file=sys.stderr, flush=True)
    if not no_cpu and cfg["cpu"] is not None:
        q = cfg["cpu"](p)
        out["cpu"] = cpu_rate(q)
        out["cpu"]["instance"] = cfg.get("cpu_note", "same instance")
    elif cfg["cpu"] is None:
        out["cpu"] = {"note": cfg.get("cpu_note")}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=list(CONFIGS))
    ap.add_argument("--time-limit", type=float, default=240.0)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    rows = []
    for name in a.names:
        r = run(name, a.time_limit, a.no_cpu)
        rows.append(r)
        print(json.dumps(r), flush=True)
    print("| config | nnz | steady it/s | iter GB/s (frac) | eps 1e-4: status, its, s | CPU it/s |", file=sys.stderr)
    print("|---|---|---|---|---|---|", file=sys.stderr)
    for r in rows:
        e = r["eps_0.0001"]
        k = r["kernels"]
        cpu = r.get("cpu", {}).get("it_per_s")
        print(f"| {r['config']} | {r['nnz']:.3g} | {k['steady_it_per_s']:.0f} | {k['iter_gbs']:.0f} "
              f"({k['iter_frac_of_hbm']:.2f}) | {e['status']}, {e['iterations']}, {e['device_s']:.2f} | "
              f"{cpu if cpu is None else round(cpu, 2)} |", file=sys.stderr)


if __name__ == "__main__":
    main()
