"""A/B of session env switches on the step kernels: one instance, one session
per setting (env read at session creation), warm in-loop iteration time and
the per-kernel times.

    python tools/ab_kernels.py VAR "v1,v2,..." case [case ...]
    python tools/ab_kernels.py - "A=1+B=2,A=3+B=4" case ...   (combined settings, applied cumulatively)

Only switches the session reads when it is created take effect between
settings; process-wide ones (read once into a static: PDHG_PDL,
PDHG_FUSED_CHECK, PDHG_CHECK_BRANCHES, ...) need one process per setting
(tools/profile_step.py under `VAR=value`, or tools/ab_solve.py).
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_14832_b200 import rpdlp  # noqa: E402
from bench import algorithmic_bytes  # noqa: E402

cases = {
    "transport": lambda: rpdlp.GenTransport(1000, 1000, 1),
    "pagerank10m": lambda: rpdlp.GenPagerank(10_000_000, 0.85, 6, 1),
    "pagerank1m": lambda: rpdlp.GenPagerank(1_000_000, 0.85, 6, 1),
    "mcf": lambda: rpdlp.GenMcf(50_000, 330_000, 50, 1),
    "staircase": lambda: rpdlp.GenStaircase(100, 100_000, 100_000, 20, 5, seed=1),
    "staircase1b": lambda: rpdlp.GenStaircase(500, 100_000, 100_000, 20, 5, seed=1),
}
var, vals = sys.argv[1], sys.argv[2].split(",")
for name in sys.argv[3:]:
    p = cases[name]()
    big = p.nnz() > 2e8
    for v in vals:
        # "VAR val,val" or, with VAR "-", settings "A=1+B=2"
        if var == "-":
            for kv in v.split("+"):
                if "=" in kv:
                    k, x = kv.split("=", 1)
                    os.environ[k] = x
        else:
            os.environ[var] = v
        with rpdlp.Session(p) as s:
            st = s.stats()
            bp, bd, bi = algorithmic_bytes(p.num_rows(), p.num_vars(), p.nnz(), st.uniform_bounds,
                                           st.csr_uniform_len, st.csc_uniform_len)
            ms_p, ms_d, ms_it = s.time_kernels(32 if big else 128)
            cp, cd, ci = s.time_kernels_cold(8 if big else 32)
            print(f"{name} {var}={v}: warm primal {ms_p*1e3:.1f} dual {ms_d*1e3:.1f} iter {ms_it*1e3:.1f} us "
                  f"({bi/ms_it/1e6:.0f} GB/s) | cold primal {cp*1e3:.1f} ({bp/cp/1e6:.0f}) dual {cd*1e3:.1f} "
                  f"({bd/cd/1e6:.0f}) iter {ci*1e3:.1f}", flush=True)
    del p
