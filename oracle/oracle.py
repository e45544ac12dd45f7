"""ORACLE — TEST INFRASTRUCTURE ONLY.

Python access to the CPU checkers:
  * liboracle.so           — serial restatement of the reference solve path
                             (rpdlp_oracle.cpp), always available once built;
  * _ref/librpdlp_ref.so   — the reference itself, compiled from
                             /root/reference by oracle/Makefile (present when it
                             was built in the dev container; the file travels to
                             the GPU box, the sources do not).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Optional

import numpy as np

from paper_2312_14832_b200 import abi
from paper_2312_14832_b200.rpdlp import (CsrMatrix, EvalInfo, LpProblem, ResidualReport, SolverParams, _dp,
                                         _f64, _Observer, _pack, _result, raise_for)

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "librpdlp_ref.so"

_ERR = abi.ERRLEN
_LP = C.POINTER(abi.Lp)
_PRM = C.POINTER(abi.Params)


def _sigs(prefix: str):
    d = abi.dptr
    return {
        f"{prefix}_solve": (C.c_int, [_LP, _PRM, abi.EVAL_CB, C.c_void_p, C.POINTER(abi.Result), C.c_char_p,
                                      C.c_size_t]),
        f"{prefix}_scaling": (C.c_int, [_LP, _PRM, d, d, C.c_char_p, C.c_size_t]),
        f"{prefix}_scaled": (C.c_int, [_LP, _PRM, d, d, d, d, d, C.c_char_p, C.c_size_t]),
        f"{prefix}_spmv": (C.c_int, [_LP, _PRM, C.c_int, d, d, C.c_char_p, C.c_size_t]),
        f"{prefix}_opnorm": (C.c_int, [_LP, _PRM, C.c_int, C.c_uint64, d, C.c_char_p, C.c_size_t]),
        f"{prefix}_residuals": (C.c_int, [_LP, d, d, C.POINTER(abi.Report), C.c_char_p, C.c_size_t]),
        f"{prefix}_primal_step": (C.c_int, [_LP, d, d, C.c_double, C.c_double, d, C.c_char_p, C.c_size_t]),
        f"{prefix}_dual_step": (C.c_int, [_LP, d, d, d, C.c_double, C.c_double, d, C.c_char_p, C.c_size_t]),
    }


class Checker:
    """One CPU implementation (restatement or reference) behind one API."""

    def __init__(self, path: Path, prefix: str):
        self.path, self.prefix = path, prefix
        self.lib = abi.bind(C.CDLL(str(path)), _sigs(prefix))
        if prefix == "oracle":
            abi.bind(self.lib, {"oracle_residuals_view": (C.c_int, [_LP, abi.dptr, abi.dptr, C.POINTER(abi.Report),
                                                                    C.c_char_p, C.c_size_t])})
        if prefix == "ref":
            vp = C.c_void_p
            abi.bind(self.lib, {
                "ref_gen_random_lp": (vp, [C.c_int64, C.c_int64, C.c_double, C.c_uint64]),
                "ref_gen_pagerank": (vp, [C.c_int64, C.c_double, C.c_int64, C.c_uint64]),
                "ref_instance_view": (None, [vp, _LP]),
                "ref_instance_witness": (abi.dptr, [vp]),
                "ref_instance_free": (None, [vp]),
                "ref_gen_transport": (vp, [C.c_int64, C.c_int64, C.c_uint64]),
                "ref_from_triplets": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.POINTER(C.c_int64),
                                                C.POINTER(C.c_int64), abi.dptr, C.POINTER(C.c_int64), C.c_char_p,
                                                C.c_size_t]),
                "ref_solve_instance": (C.c_int, [vp, _PRM, C.POINTER(abi.Result), C.c_char_p, C.c_size_t]),
            })

    def _f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def solve(self, p: LpProblem, params: Optional[SolverParams] = None, observer=None):
        params = params or SolverParams()
        lp, prm = p.to_c(), params.to_c()
        res, x, y, lam = _result(p)
        obs = _Observer(observer)
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("solve")(C.byref(lp), C.byref(prm), obs.c, None, C.byref(res), err, _ERR), err, obs.error)
        return _pack(res, x, y, lam)

    def scaling(self, p: LpProblem, params: Optional[SolverParams] = None):
        prm = (params or SolverParams()).to_c()
        lp = p.to_c()
        rs, cs = np.empty(p.num_rows()), np.empty(p.num_vars())
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("scaling")(C.byref(lp), C.byref(prm), _dp(rs), _dp(cs), err, _ERR), err)
        return rs, cs

    def scaled(self, p: LpProblem, params: Optional[SolverParams] = None):
        prm = (params or SolverParams()).to_c()
        lp = p.to_c()
        kv, c, l, u, q = (np.empty(p.nnz()), np.empty(p.num_vars()), np.empty(p.num_vars()),
                          np.empty(p.num_vars()), np.empty(p.num_rows()))
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("scaled")(C.byref(lp), C.byref(prm), _dp(kv), _dp(c), _dp(l), _dp(u), _dp(q), err, _ERR),
                  err)
        return kv, c, l, u, q

    def spmv(self, p: LpProblem, vec, transpose=False, params: Optional[SolverParams] = None):
        prm = (params or SolverParams()).to_c()
        lp = p.to_c()
        v = _f64(vec)
        out = np.empty(p.num_vars() if transpose else p.num_rows())
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("spmv")(C.byref(lp), C.byref(prm), int(transpose), _dp(v), _dp(out), err, _ERR), err)
        return out

    def opnorm(self, p: LpProblem, iters=100, seed=0, params: Optional[SolverParams] = None) -> float:
        prm = (params or SolverParams()).to_c()
        lp = p.to_c()
        o = C.c_double()
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("opnorm")(C.byref(lp), C.byref(prm), iters, seed, C.byref(o), err, _ERR), err)
        return o.value

    def residuals(self, p: LpProblem, x, y) -> ResidualReport:
        lp = p.to_c()
        xa, ya = _f64(x), _f64(y)
        r = abi.Report()
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("residuals")(C.byref(lp), _dp(xa), _dp(ya), C.byref(r), err, _ERR), err)
        return ResidualReport.from_c(r)

    def residuals_view(self, p: LpProblem, x, y) -> ResidualReport:
        """ComputeResiduals on the CSR view without host matrix copies
        (restatement only: oracle_residuals_view; bit-identical to the
        reference's, pinned in tests/test_oracle.py)."""
        if self.prefix != "oracle":
            return self.residuals(p, x, y)
        lp = p.to_c()
        rep = abi.Report()
        err = C.create_string_buffer(_ERR)
        raise_for(self.lib.oracle_residuals_view(C.byref(lp), _dp(_f64(x)), _dp(_f64(y)), C.byref(rep), err, _ERR),
                  err)
        return ResidualReport.from_c(rep)

    def primal_step(self, p, x, y, eta, omega):
        lp = p.to_c()
        xa, ya, out = _f64(x), _f64(y), np.empty(p.num_vars())
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("primal_step")(C.byref(lp), _dp(xa), _dp(ya), eta, omega, _dp(out), err, _ERR), err)
        return out

    def dual_step(self, p, xn, xo, y, eta, omega):
        lp = p.to_c()
        a, b, ya, out = _f64(xn), _f64(xo), _f64(y), np.empty(p.num_rows())
        err = C.create_string_buffer(_ERR)
        raise_for(self._f("dual_step")(C.byref(lp), _dp(a), _dp(b), _dp(ya), eta, omega, _dp(out), err, _ERR),
                  err)
        return out

    # Reference generators (ref only).
    def _instance(self, h, name) -> LpProblem:
        v = abi.Lp()
        self.lib.ref_instance_view(h, C.byref(v))

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True) if n else np.zeros(0, dt)

        def csr(m):
            rp = arr(m.row_ptr, m.rows + 1, np.int64)
            nz = int(rp[-1])
            return CsrMatrix(m.rows, m.cols, rp, arr(m.col_idx, nz, np.int64), arr(m.values, nz, np.float64))

        a, g = csr(v.a), csr(v.g)
        p = LpProblem(a, g, arr(v.c, v.n, np.float64), arr(v.b, a.rows, np.float64), arr(v.h, g.rows, np.float64),
                      arr(v.l, v.n, np.float64), arr(v.u, v.n, np.float64), v.objective_offset, False, name)
        w = self.lib.ref_instance_witness(h)
        p.witness = arr(w, v.n, np.float64) if w else None
        self.lib.ref_instance_free(h)
        return p

    def gen_random_lp(self, m, n, density, seed) -> LpProblem:
        return self._instance(self.lib.ref_gen_random_lp(m, n, density, seed), f"rand_{m}x{n}_s{seed}")

    def gen_pagerank(self, n, damping=0.85, attachment=3, seed=0) -> LpProblem:
        return self._instance(self.lib.ref_gen_pagerank(n, damping, attachment, seed), "pagerank")

    def gen_transport(self, sources, sinks, seed=1) -> LpProblem:
        return self._instance(self.lib.ref_gen_transport(sources, sinks, seed), "transport")

    def from_triplets(self, rows, cols, r, c, v) -> CsrMatrix:
        """The reference's SparseMatrix::FromTriplets on arrays (ref only)."""
        r, c, v = np.asarray(r), np.asarray(c), np.asarray(v, np.float64)
        t = np.empty(r.size, dtype=[("row", "<i8"), ("col", "<i8"), ("value", "<f8")])
        t["row"], t["col"], t["value"] = r, c, v
        ptr = np.zeros(rows + 1, np.int64)
        idx, val = np.empty(max(r.size, 1), np.int64), np.empty(max(r.size, 1), np.float64)
        nnz = C.c_int64(0)
        err = C.create_string_buffer(_ERR)
        P = C.POINTER(C.c_int64)
        if self.lib.ref_from_triplets(rows, cols, r.size, t.ctypes.data, ptr.ctypes.data_as(P),
                                      idx.ctypes.data_as(P), _dp(val), C.byref(nnz), err, _ERR) != 0:
            raise IndexError(err.value.decode())
        k = nnz.value
        return CsrMatrix(rows, cols, ptr, idx[:k].copy(), val[:k].copy())

    def transport_instance(self, sources, sinks, seed=1) -> "RefInstance":
        """A reference-owned transportation LP (built by the reference's own
        FromTriplets): the reference arm of bench.py solves it in place, so
        that arm never loads the product library."""
        return RefInstance(self, self.lib.ref_gen_transport(sources, sinks, seed))


class RefInstance:
    """Handle to an LpProblem owned by the reference build (ref only)."""

    def __init__(self, chk: Checker, h):
        self.chk, self.h = chk, h
        v = abi.Lp()
        chk.lib.ref_instance_view(h, C.byref(v))
        self.m, self.n = v.a.rows + v.g.rows, v.n
        self.nnz = int(v.a.row_ptr[v.a.rows]) + int(v.g.row_ptr[v.g.rows])

    def solve(self, params: Optional[SolverParams] = None):
        """Reference Solve on the resident instance; x, y, lambda not copied."""
        prm = (params or SolverParams()).to_c()
        res = abi.Result()
        err = C.create_string_buffer(_ERR)
        raise_for(self.chk.lib.ref_solve_instance(self.h, C.byref(prm), C.byref(res), err, _ERR), err)
        return res

    def __del__(self):
        if getattr(self, "h", None):
            self.chk.lib.ref_instance_free(self.h)
            self.h = None


_cache = {}


def restatement() -> Checker:
    """The C++ restatement (always present once `make -C oracle` ran)."""
    if "o" not in _cache:
        if not ORACLE_LIB.exists():
            raise RuntimeError(f"{ORACLE_LIB} missing: run python -m paper_2312_14832_b200.build")
        _cache["o"] = Checker(ORACLE_LIB, "oracle")
    return _cache["o"]


def reference() -> Optional[Checker]:
    """The reference build, or None where it was not compiled."""
    if "r" not in _cache:
        _cache["r"] = Checker(REF_LIB, "ref") if REF_LIB.exists() else None
    return _cache["r"]


def cpu_baseline() -> Checker:
    """The reference when built, else the restatement (bench cpu_baseline)."""
    return reference() or restatement()
