"""Small solves through every kernel family, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
(TMA-staged class L, segment-order warps, uniform / staged / direct class S,
warp and CTA classes, the tile engine in gather-sweep order, the check, power
iteration, device triplet assembly, matrix norms, the opt-in device-resident
loop; SANITIZE_VARIANTS=1 adds the opt-in round-2 variants: persistent class
S, gather-window split, the persistent block kernel, the adaptive fused
check)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2312_14832_b200 import rpdlp  # noqa: E402

prm = rpdlp.SolverParams(eps=1e-5, iter_limit=640)
cases = {
    "transport": rpdlp.GenTransport(40, 700, 1),           # RPC-4 rows, TMA-staged
    "mcf": rpdlp.GenMcf(300, 2000, 8, 1),                    # segment-order warps
    "pagerank": rpdlp.GenPagerank(20000, 0.85, 3, 1),        # XL sum row (tile engine)
    "random": rpdlp.GenRandomLp(200, 300, 0.05, 2, equality_rows=40),
    "staircase": rpdlp.GenStaircase(3, 300, 300, 20, 5, seed=1),
}
for name, p in cases.items():
    loops = ("0",) if os.environ.get("SANITIZE_HOST_LOOP_ONLY") else ("0", "1")
    for loop in loops:
        os.environ["PDHG_DEVICE_LOOP"] = loop
        r = rpdlp.Solve(p, prm)
        print(name, "device_loop" if loop == "1" else "host_loop", int(r.status), r.iterations, flush=True)
if os.environ.get("SANITIZE_VARIANTS"):
    os.environ["PDHG_DEVICE_LOOP"] = "0"
    big_t = rpdlp.GenTransport(40, 900, 2)  # rows of 900: the block kernel's layout
    for env, names in ((("PDHG_S_FLOW", "3"), ("mcf", "staircase", "pagerank")),
                       (("PDHG_S_SPLIT", "1"), ("mcf", "pagerank")),
                       (("PDHG_PERSIST", "1"), ("big_t",))):
        os.environ[env[0]] = env[1]
        os.environ["PDHG_S_SPLIT_MIN_MB"] = "0"
        for name in names:
            p = big_t if name == "big_t" else cases[name]
            r = rpdlp.Solve(p, prm)
            print(name, "=".join(env), int(r.status), r.iterations, flush=True)
        del os.environ[env[0]]
    r = rpdlp.Solve(cases["random"], rpdlp.SolverParams(eps=1e-5, iter_limit=640, adaptive_step=True))
    print("random adaptive", int(r.status), r.iterations, flush=True)
k = cases["random"].g
d = rpdlp.CsrMatrix.from_triplets_device(k.rows, k.cols, np.repeat(np.arange(k.rows), np.diff(k.row_ptr)),
                                         k.col_idx, k.values)
assert np.array_equal(d.values, k.values)
print("norms", float(k.norms().sum()), float(k.multiply(np.ones(k.cols)).sum()))
print("sanitize smoke done")
