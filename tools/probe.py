"""Quick per-kernel timing probe across workloads (no ncu).

    python tools/probe.py [transport|pagerank1m|pagerank10m|random|mcf|staircase ...] [--shards P]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_14832_b200 import rpdlp  # noqa: E402
from bench import algorithmic_bytes  # noqa: E402

cases = {
    "transport": lambda: rpdlp.GenTransport(1000, 1000, 1),
    "pagerank1m": lambda: rpdlp.GenPagerank(1_000_000, 0.85, 6, 1),
    "pagerank10m": lambda: rpdlp.GenPagerank(10_000_000, 0.85, 6, 1),
    "random": lambda: rpdlp.GenRandomLp(1000, 2000, 0.005, 1, equality_rows=300),
    "mcf": lambda: rpdlp.GenMcf(50_000, 330_000, 50, 1),
    "staircase": lambda: rpdlp.GenStaircase(100, 100_000, 100_000, 20, 5, seed=1),
}
args = sys.argv[1:]
shards = 1
if "--shards" in args:
    i = args.index("--shards")
    shards = int(args[i + 1])
    del args[i:i + 2]
which = args or ["transport", "pagerank1m", "random", "mcf"]
full_solve = {"transport", "random"}
short = {"pagerank10m", "staircase", "mcf"}
for name in which:
    t = time.time()
    p = cases[name]()
    tg = time.time() - t
    sp = rpdlp.Shards(world=shards) if shards > 1 else None
    with rpdlp.Session(p, shards=sp) as s:
        st = s.stats()
        ms_p, ms_d, ms_it = s.time_kernels(64 if p.nnz() > 2e7 else 256)
        bp, bd, bi = algorithmic_bytes(p.num_rows(), p.num_vars(), p.nnz(), st.uniform_bounds, st.csr_uniform_len,
                                       st.csc_uniform_len)
        print(f"{name}: m={p.num_rows()} n={p.num_vars()} nnz={p.nnz()} gen {tg:.1f}s upload {st.upload_seconds:.3f}s "
              f"scaling {st.scaling_seconds:.3f}s bnd {st.uniform_bounds} ulen {st.csr_uniform_len}/{st.csc_uniform_len} tiles {st.csr_tiles}/{st.csc_tiles} dev {st.device_bytes / 1e9:.2f} GB"
              f"\n   primal {ms_p*1e3:.1f}us {bp/ms_p/1e6:.0f} GB/s | dual {ms_d*1e3:.1f}us "
              f"{bd/ms_d/1e6:.0f} GB/s | iter {ms_it*1e3:.1f}us {bi/ms_it/1e6:.0f} GB/s -> {1e3 / ms_it:.0f} it/s",
              flush=True)
        cd, cw = s.time_check(20 if p.nnz() > 2e7 else 100)
        print(f"   check: device {cd*1e3:.1f}us, with host read {cw*1e3:.1f}us (= {cd / ms_it:.1f} / {cw / ms_it:.1f} "
              f"iterations)", flush=True)
        if name in full_solve:
            r = s.solve(rpdlp.SolverParams(eps=1e-4))
            ms, nl = s.last_solve()
            print(f"   solve: status {int(r.status)} it {r.iterations} restarts {r.restarts} device {ms:.1f} ms "
                  f"-> {r.iterations / ms * 1e3:.0f} it/s", flush=True)
        else:
            r = s.solve(rpdlp.SolverParams(eps=1e-4, iter_limit=128 if name in short else 640))
            ms, nl = s.last_solve()
            print(f"   {r.iterations} its: device {ms:.1f} ms -> {r.iterations / ms * 1e3:.0f} it/s", flush=True)
    del p
