"""Quick per-kernel timing probe across workloads (no ncu)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_14832_b200 import rpdlp  # noqa: E402
from bench import algorithmic_bytes  # noqa: E402

cases = {
    "transport": lambda: rpdlp.GenTransport(1000, 1000, 1),
    "pagerank1m": lambda: rpdlp.GenPagerank(1_000_000, 0.85, 6, 1),
    "random": lambda: rpdlp.GenRandomLp(1000, 2000, 0.005, 1, equality_rows=300),
}
which = sys.argv[1:] or list(cases)
for name in which:
    t = time.time()
    p = cases[name]()
    tg = time.time() - t
    with rpdlp.Session(p) as s:
        st = s.stats()
        ms_p, ms_d, ms_it = s.time_kernels(256)
        bp, bd, bi = algorithmic_bytes(p.num_rows(), p.num_vars(), p.nnz())
        print(f"{name}: gen {tg:.1f}s upload {st.upload_seconds:.3f}s scaling {st.scaling_seconds:.3f}s tiles "
              f"{st.csr_tiles}/{st.csc_tiles} | primal {ms_p*1e3:.1f}us {bp/ms_p/1e6:.0f} GB/s | dual {ms_d*1e3:.1f}us "
              f"{bd/ms_d/1e6:.0f} GB/s | iter {ms_it*1e3:.1f}us {bi/ms_it/1e6:.0f} GB/s", flush=True)
        if name != "pagerank1m":
            r = s.solve(rpdlp.SolverParams(eps=1e-4))
            ms, nl = s.last_solve()
            print(f"   solve: status {int(r.status)} it {r.iterations} restarts {r.restarts} device {ms:.1f} ms "
                  f"-> {r.iterations / ms * 1e3:.0f} it/s", flush=True)
        else:
            r = s.solve(rpdlp.SolverParams(eps=1e-4, iter_limit=640))
            ms, nl = s.last_solve()
            print(f"   640 its: device {ms:.1f} ms -> {r.iterations / ms * 1e3:.0f} it/s", flush=True)
