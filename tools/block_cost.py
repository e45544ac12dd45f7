import sys; sys.path.insert(0, ".")
from paper_2312_14832_b200 import rpdlp
p = rpdlp.GenTransport(1000, 1000, 1)
with rpdlp.Session(p) as s:
    ms_p, ms_d, ms_it = s.time_kernels(256)
    cd, cw = s.time_check(100)
    for lim in (64 * 50, 64 * 150):
        for _ in range(2):
            s.solve(rpdlp.SolverParams(eps=1e-15, iter_limit=lim, restart_enabled=False))
        r = s.solve(rpdlp.SolverParams(eps=1e-15, iter_limit=lim, restart_enabled=False))
        ms, _ = s.last_solve()
        print(f"iters {lim}: {ms:.2f} ms -> {ms * 1e3 / lim:.2f} us/it (iteration alone {ms_it * 1e3:.2f} us, check {cd * 1e3:.1f} us)")
