import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_fuzz import _random_lp
from paper_2312_14832_b200 import rpdlp
from oracle import oracle
R = oracle.restatement()
for s in range(12):
    p = _random_lp(1000 + s)
    prm = rpdlp.SolverParams(eps=1e-6, iter_limit=60000)
    g = rpdlp.Solve(p, prm); o = R.solve(p, prm)
    lens = p.g.row_ptr[1:] - p.g.row_ptr[:-1]
    print(s, p.num_rows(), p.num_vars(), p.g.nnz + p.a.nnz, int(lens.max(initial=0)), int(g.status), int(o.status), g.iterations, o.iterations, g.restarts, o.restarts)
