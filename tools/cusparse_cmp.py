"""cuSPARSE comparator: one PDHG iteration as
cusparseSpMV (CSR FP64, ALG2 / ALG1 / transpose-op) plus separate elementwise
kernels, against the fused K-CSC primal + K-CSR dual step kernels, on the
same matrices (BASELINE configs 2-5). Measurement tool only.

    python tools/cusparse_cmp.py [transport mcf pagerank10m staircase] [--json out.jsonl]
"""
import ctypes as C
import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import algorithmic_bytes  # noqa: E402
from paper_2312_14832_b200 import rpdlp  # noqa: E402

LIB = ROOT / "tools" / "_build" / "libcusparse_cmp.so"
CASES = {
    "transport": lambda: rpdlp.GenTransport(1000, 1000, 1),
    "mcf": lambda: rpdlp.GenMcf(50_000, 330_000, 50, 1),
    "pagerank10m": lambda: rpdlp.GenPagerank(10_000_000, 0.85, 6, 1),
    "staircase": lambda: rpdlp.GenStaircase(100, 100_000, 100_000, 20, 5, seed=1),
}
NAMES = ["KTy_alg2", "Kx_alg2", "KTy_alg1", "Kx_alg1", "KTy_transpose_op", "primal_elementwise", "dual_elementwise",
         "unfused_iteration"]


def build():
    src = ROOT / "tools" / "cusparse_cmp.cu"
    if LIB.exists() and LIB.stat().st_mtime >= src.stat().st_mtime:
        return
    LIB.parent.mkdir(exist_ok=True)
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(LIB), str(src), "-lcusparse"], check=True)


def stacked(p):
    """K = [A; G] as int32 CSR, and its transpose (K's CSC) as int32 CSR."""
    a, g = p.a, p.g
    rp = np.concatenate([a.row_ptr, g.row_ptr[1:] + a.row_ptr[-1]]).astype(np.int32)
    ci = np.concatenate([a.col_idx, g.col_idx]).astype(np.int32)
    rv = np.concatenate([a.values, g.values])
    m, n = a.rows + g.rows, p.num_vars()
    nnz = rv.size
    cnt = np.bincount(ci, minlength=n)
    cp = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    order = np.argsort(ci, kind="stable")  # rows ascending inside each column
    rows = np.repeat(np.arange(m, dtype=np.int32), np.diff(rp))
    return m, a.rows, n, nnz, rp, ci, rv, cp.astype(np.int32), rows[order], rv[order]


def main(argv):
    out = None
    if "--json" in argv:
        i = argv.index("--json")
        out = open(argv[i + 1], "w")
        del argv[i:i + 2]
    build()
    lib = C.CDLL(str(LIB))
    lib.cmp_iteration.restype = C.c_int
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    for name in argv or list(CASES):
        t = time.time()
        p = CASES[name]()
        m, m1, n, nnz, rp, ci, rv, cp, ri, cv = stacked(p)
        prep = time.time() - t
        times = np.zeros(16)
        P = lambda a, ty: a.ctypes.data_as(C.POINTER(ty))  # noqa: E731
        reps = 20 if nnz > 2e8 else 100
        rc = lib.cmp_iteration(C.c_int64(m), C.c_int64(m1), C.c_int64(n), C.c_int64(nnz), P(rp, C.c_int32),
                               P(ci, C.c_int32), P(rv, C.c_double), P(cp, C.c_int32), P(ri, C.c_int32),
                               P(cv, C.c_double), reps, P(times, C.c_double))
        if rc:
            raise SystemExit(f"cmp_iteration failed: {rc}")
        del rp, ci, rv, cp, ri, cv
        with rpdlp.Session(p) as s:
            st = s.stats()
            wp, wd, wi = s.time_kernels(32 if nnz > 2e8 else 128)
            cpm, cdm, cim = s.time_kernels_cold(8 if nnz > 2e8 else 32)
        bp, bd, bi = algorithmic_bytes(m, n, nnz, st.uniform_bounds, st.csr_uniform_len, st.csc_uniform_len)
        rec = {"config": name, "m": m, "n": n, "nnz": nnz, "prep_s": prep, "hbm_peak_gbs": peak,
               "cusparse_warm_ms": dict(zip(NAMES, times[:8].tolist())),
               "cusparse_cold_ms": dict(zip(NAMES, times[8:].tolist())),
               "fused_warm_ms": {"primal_csc": wp, "dual_csr": wd, "iteration": wi},
               "fused_cold_ms": {"primal_csc": cpm, "dual_csr": cdm, "iteration": cim},
               "algorithmic_bytes": {"primal": bp, "dual": bd, "iteration": bi}}
        unf_w, unf_c = times[7], times[15]
        rec["speedup_iteration_warm"] = unf_w / wi
        rec["speedup_iteration_cold"] = unf_c / cim
        print(f"{name}: m={m} n={n} nnz={nnz}\n"
              f"  cuSPARSE ALG2  K^T y {times[0] * 1e3:8.1f} us  K x {times[1] * 1e3:8.1f} us | ALG1 {times[2] * 1e3:8.1f} / "
              f"{times[3] * 1e3:8.1f} us | transpose-op K^T y {times[4] * 1e3:8.1f} us\n"
              f"  elementwise    primal {times[5] * 1e3:8.1f} us  dual {times[6] * 1e3:8.1f} us\n"
              f"  unfused iteration (ALG2 + elementwise): warm {unf_w * 1e3:8.1f} us  cold {unf_c * 1e3:8.1f} us\n"
              f"  fused (ours): primal {wp * 1e3:8.1f} dual {wd * 1e3:8.1f} iteration {wi * 1e3:8.1f} us warm; "
              f"iteration {cim * 1e3:8.1f} us cold -> {unf_w / wi:.2f}x warm, {unf_c / cim:.2f}x cold "
              f"(algorithmic {bi / wi / 1e6:.0f} GB/s = {bi / wi / 1e6 / peak:.2f} of peak)", flush=True)
        if out:
            out.write(json.dumps(rec) + "\n")
            out.flush()
        del p


if __name__ == "__main__":
    main(sys.argv[1:])
