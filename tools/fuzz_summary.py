"""Randomised class-mix LPs (tests/test_gpu_fuzz.py): GPU vs the CPU oracle
restatement, status / iterations / restarts per seed.
    python tools/fuzz_summary.py [seeds=12]"""
import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_fuzz import _random_lp
from paper_2312_14832_b200 import rpdlp
from oracle import oracle
R = oracle.restatement()
n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 12
same = 0
for s in range(n_seeds):
    p = _random_lp(1000 + s)
    prm = rpdlp.SolverParams(eps=1e-6, iter_limit=60000)
    g = rpdlp.Solve(p, prm); o = R.solve(p, prm)
    lens = p.g.row_ptr[1:] - p.g.row_ptr[:-1]
    print(s, p.num_rows(), p.num_vars(), p.g.nnz + p.a.nnz, int(lens.max(initial=0)), int(g.status), int(o.status), g.iterations, o.iterations, g.restarts, o.restarts, flush=True)
    same += (int(g.status), g.iterations, g.restarts) == (int(o.status), o.iterations, o.restarts)
print(f"# identical status / iterations / restarts: {same} of {n_seeds}")
