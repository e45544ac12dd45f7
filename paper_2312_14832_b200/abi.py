"""ctypes mirror of include/pdhg.h and the loader for libpdhg_b200.so.

The product path is the CUDA library; there is no Python or CPU fallback.
`load()` raises if the built library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libpdhg_b200.so"

PDHG_OK = 0
PDHG_INVALID_ARGUMENT = 1
PDHG_NUMERICAL_FAILURE = 2
PDHG_CUDA_ERROR = 3
PDHG_NCCL_ERROR = 4
PDHG_ABORTED = 5
PDHG_PARSE_ERROR = 6
PDHG_IO_ERROR = 7
PDHG_ORDER_DEPENDENT = 8

PDHG_OPTIMAL = 0
PDHG_ITER_LIMIT = 1
PDHG_TIME_LIMIT = 2

dptr = C.POINTER(C.c_double)
i64ptr = C.POINTER(C.c_int64)


class Csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("row_ptr", i64ptr), ("col_idx", i64ptr),
                ("values", dptr)]


class Lp(C.Structure):
    _fields_ = [("a", Csr), ("g", Csr), ("n", C.c_int64), ("c", dptr), ("b", dptr), ("h", dptr), ("l", dptr),
                ("u", dptr), ("objective_offset", C.c_double), ("negated_objective", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("eps", C.c_double), ("time_limit", C.c_double), ("iter_limit", C.c_int64),
                ("sufficient_decay", C.c_double), ("necessary_decay", C.c_double),
                ("long_loop_frac", C.c_double), ("restart_enabled", C.c_int32), ("check_every", C.c_int64),
                ("scaling_enabled", C.c_int32), ("ruiz_iters", C.c_int32), ("pc_alpha", C.c_double),
                ("seed", C.c_uint64), ("adaptive_step", C.c_int32), ("log_every", C.c_int64)]


class Report(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("primal_res", "dual_res", "gap_abs", "primal_obj", "dual_obj",
                                          "rel_primal", "rel_dual", "rel_gap")]


class EvalInfo(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("inner_iteration", C.c_int64), ("restarts", C.c_int64),
                ("omega", C.c_double), ("eta", C.c_double), ("kkt_candidate", C.c_double),
                ("kkt_loop_start", C.c_double), ("candidate_is_current", C.c_int32), ("restarted", C.c_int32),
                ("original_report", Report), ("seconds", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("x", dptr), ("y", dptr), ("lambda_", dptr), ("report", Report),
                ("iterations", C.c_int64), ("restarts", C.c_int64), ("solve_seconds", C.c_double),
                ("scaling_seconds", C.c_double)]


class SessionStats(C.Structure):
    _fields_ = [("m1", C.c_int64), ("m2", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64),
                ("csr_tiles", C.c_int64), ("csc_tiles", C.c_int64), ("device_bytes", C.c_int64),
                ("upload_seconds", C.c_double), ("scaling_seconds", C.c_double), ("device", C.c_int32),
                ("l2_resident", C.c_int32), ("world", C.c_int32), ("local_shards", C.c_int32),
                ("rank", C.c_int32), ("uniform_bounds", C.c_int32),
                ("csr_uniform_len", C.c_int32), ("csc_uniform_len", C.c_int32), ("csr_split", C.c_int32),
                ("block_kernel", C.c_int32)]


class ShardSpec(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("local_shards", C.c_int32), ("nccl_id", C.c_void_p)]


EVAL_CB = C.CFUNCTYPE(C.c_int, C.POINTER(EvalInfo), C.c_void_p)
ERRLEN = 512

# name -> (restype, argtypes); every symbol include/pdhg.h declares.
SIGNATURES = {
    "pdhg_params_default": (None, [C.POINTER(Params)]),
    "pdhg_abi_version": (C.c_int, []),
    "pdhg_build_info": (C.c_char_p, []),
    "pdhg_device_count": (C.c_int, []),
    "pdhg_solve": (C.c_int, [C.POINTER(Lp), C.POINTER(Params), EVAL_CB, C.c_void_p, C.POINTER(Result), C.c_char_p,
                             C.c_size_t]),
    "pdhg_solve_on": (C.c_int, [C.POINTER(Lp), C.POINTER(Params), C.c_int, EVAL_CB, C.c_void_p, C.POINTER(Result),
                                C.c_char_p, C.c_size_t]),
    "pdhg_session_create": (C.c_int, [C.POINTER(Lp), C.POINTER(Params), C.c_int, C.POINTER(C.c_void_p), C.c_char_p,
                                      C.c_size_t]),
    "pdhg_session_create_sharded": (C.c_int, [C.POINTER(Lp), C.POINTER(Params), C.c_int, C.POINTER(ShardSpec),
                                              C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "pdhg_solve_sharded": (C.c_int, [C.POINTER(Lp), C.POINTER(Params), C.c_int, C.POINTER(ShardSpec), EVAL_CB,
                                     C.c_void_p, C.POINTER(Result), C.c_char_p, C.c_size_t]),
    "pdhg_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "pdhg_loopback_id": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "pdhg_session_blocks": (C.c_int, [C.c_void_p, i64ptr, i64ptr]),
    "pdhg_compute_scaling": (C.c_int, [C.POINTER(Csr), C.c_int, C.c_double, C.c_int, dptr, dptr, C.c_char_p,
                                       C.c_size_t]),
    "pdhg_residuals": (C.c_int, [C.POINTER(Lp), dptr, dptr, C.POINTER(Report), C.c_char_p, C.c_size_t]),
    "pdhg_derive_lambda": (C.c_int, [C.POINTER(Lp), dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_ghost_counts": (C.c_int, [C.c_void_p, i64ptr, i64ptr, C.POINTER(C.c_int32)]),
    "pdhg_partition_blocks": (C.c_int, [i64ptr, C.c_int64, C.c_int, C.c_int64, i64ptr]),
    "pdhg_normal_vector": (C.c_int, [C.c_uint64, C.c_int64, C.c_int, dptr]),
    "pdhg_session_destroy": (None, [C.c_void_p]),
    "pdhg_session_stats_get": (C.c_int, [C.c_void_p, C.POINTER(SessionStats)]),
    "pdhg_session_solve": (C.c_int, [C.c_void_p, C.POINTER(Params), EVAL_CB, C.c_void_p, C.POINTER(Result),
                                     C.c_char_p, C.c_size_t]),
    "pdhg_session_scaling": (C.c_int, [C.c_void_p, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_scaled": (C.c_int, [C.c_void_p, dptr, dptr, dptr, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_spmv": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_opnorm": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_time_kernels": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_time_kernels_cold": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_session_run_block": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "pdhg_session_time_check": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_csr_spmv": (C.c_int, [C.POINTER(Csr), C.c_int, C.c_int, C.c_double, dptr, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_csr_norms": (C.c_int, [C.POINTER(Csr), C.c_int, C.c_int, C.c_double, dptr, C.c_char_p, C.c_size_t]),
    "pdhg_csr_scaled": (C.c_int, [C.POINTER(Csr), i64ptr, i64ptr, dptr, dptr, dptr, dptr, dptr, C.c_char_p,
                                  C.c_size_t]),
    "pdhg_csr_from_triplets": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int, i64ptr, i64ptr, dptr,
                                         C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]),
    "pdhg_from_triplets": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, i64ptr, i64ptr, dptr,
                                     C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]),
    "pdhg_session_flush_l2": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "pdhg_session_last_solve": (C.c_int, [C.c_void_p, dptr, i64ptr]),
    "pdhg_should_restart": (C.c_int, [C.POINTER(Params), C.c_int64, C.c_int64, C.c_double, C.c_double,
                                      C.c_double]),
    "pdhg_update_primal_weight": (C.c_double, [C.c_double, C.c_double, C.c_double]),
    "pdhg_kkt_error": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_double]),
    "pdhg_check_termination": (C.c_int, [C.POINTER(Report), C.c_double]),
    "pdhg_primal_step": (C.c_int, [C.POINTER(Lp), dptr, dptr, C.c_double, C.c_double, dptr, C.c_char_p,
                                   C.c_size_t]),
    "pdhg_dual_step": (C.c_int, [C.POINTER(Lp), dptr, dptr, dptr, C.c_double, C.c_double, dptr, C.c_char_p,
                                 C.c_size_t]),
    "pdhg_gen_random_lp": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.POINTER(C.c_void_p),
                                     C.c_char_p, C.c_size_t]),
    "pdhg_gen_pagerank": (C.c_int, [C.c_int64, C.c_double, C.c_int64, C.c_uint64, C.POINTER(C.c_void_p),
                                    C.c_char_p, C.c_size_t]),
    "pdhg_pagerank_graph_edges": (C.c_int64, [C.c_int64, C.c_int64]),
    "pdhg_gen_pagerank_graph": (C.c_int, [C.c_int64, C.c_double, C.c_int64, C.c_uint64, i64ptr, C.c_int64, i64ptr,
                                          C.c_char_p, C.c_size_t]),
    "pdhg_build_pagerank_lp": (C.c_int, [i64ptr, C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_void_p),
                                         C.c_char_p, C.c_size_t]),
    "pdhg_gen_transport": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_void_p), C.c_char_p,
                                     C.c_size_t]),
    "pdhg_gen_mcf": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_void_p), C.c_char_p,
                               C.c_size_t]),
    "pdhg_gen_staircase": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                     C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "pdhg_instance_make_equalities": (C.c_int, [C.c_void_p, C.c_int64, C.c_char_p, C.c_size_t]),
    "pdhg_instance_view": (C.c_int, [C.c_void_p, C.POINTER(Lp)]),
    "pdhg_instance_witness": (dptr, [C.c_void_p]),
    "pdhg_instance_free": (None, [C.c_void_p]),
    "pdhg_instance_name": (C.c_char_p, [C.c_void_p]),
    "pdhg_mps_read_file": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t,
                                     C.POINTER(C.c_int)]),
    "pdhg_mps_read_string": (C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p), C.c_char_p,
                                       C.c_size_t, C.POINTER(C.c_int)]),
    "pdhg_mps_write_file": (C.c_int, [C.POINTER(Lp), C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t]),
    "pdhg_mps_write_string": (C.c_int, [C.POINTER(Lp), C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                        C.c_char_p, C.c_size_t]),
    "pdhg_free_string": (None, [C.c_void_p]),
}

_lib = None


def bind(lib, signatures):
    for name, (res, args) in signatures.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def load():
    """Load the in-tree CUDA library; fail loudly if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2312_14832_b200.build` "
                               "(there is no CPU fallback)")
        _point_at_torch_nccl()
        _lib = bind(C.CDLL(str(LIB_PATH)), SIGNATURES)
    return _lib


def _point_at_torch_nccl():
    """The sharded path dlopens NCCL on first use. If that were the system
    libnccl.so.2 while PyTorch bundles a newer one, a later `import torch` in
    the same process would bind to the older library (same soname) and fail
    on missing symbols; so name PyTorch's copy (without importing torch)."""
    if os.environ.get("PDHG_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["PDHG_NCCL_LIB"] = cand
            return


def default_params() -> Params:
    p = Params()
    load().pdhg_params_default(C.byref(p))
    return p
