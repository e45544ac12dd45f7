"""Drive the fused PDHG step kernels for an ncu capture (one GPU).

    ncu --set full -k regex:"OpPrimal|OpDual" -s 4 -c 2 python tools/profile_step.py transport
    ncu --set full -k regex:"OpCheck|k_reduce_two" -s 6 -c 3 python tools/profile_step.py transport - 2 --check
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2312_14832_b200 import rpdlp  # noqa: E402


def problem(name):
    if name == "transport":
        return rpdlp.GenTransport(1000, 1000, 1)
    if name == "pagerank":
        return rpdlp.GenPagerank(int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000, 0.85, 6, 1)
    if name == "mcf":
        return rpdlp.GenMcf(50_000, 330_000, 50, 1)
    if name == "staircase":
        return rpdlp.GenStaircase(100, 100_000, 100_000, 20, 5, seed=1)
    if name == "random":
        return rpdlp.GenRandomLp(1000, 2000, 0.005, 1, equality_rows=300)
    raise SystemExit(name)


if __name__ == "__main__":
    p = problem(sys.argv[1] if len(sys.argv) > 1 else "transport")
    with rpdlp.Session(p) as s:
        iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
        if "--check" in sys.argv:  # drive the check kernels instead (OpCheckRow|OpCheckCol|k_reduce_two)
            cd, cw = s.time_check(iters)
            print(f"check {cd * 1e3:.1f} us device, {cw * 1e3:.1f} us with the host read")
        else:
            ms_p, ms_d, ms_it = s.time_kernels(iters)
            print(f"primal {ms_p * 1e3:.1f} us  dual {ms_d * 1e3:.1f} us  iteration {ms_it * 1e3:.1f} us")
