"""Regenerate tests/golden/mps_golden.json from the REFERENCE MPS reader and
writer (oracle/_ref/librpdlp_ref.so, built from /root/reference by
oracle/Makefile). Values are stored as float.hex strings (bit-exact).

    python tests/golden/make_mps_golden.py
"""
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2312_14832_b200 import abi  # noqa: E402
from paper_2312_14832_b200.rpdlp import GenRandomLp  # noqa: E402

import mps_corpus  # noqa: E402


def ref_lib():
    ref = oracle.reference()
    if ref is None:
        raise SystemExit("reference build missing (make -C oracle ref)")
    lib = ref.lib
    vp = C.c_void_p
    lib.ref_parse_mps.restype = C.c_int
    lib.ref_parse_mps.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t,
                                  C.POINTER(C.c_int)]
    lib.ref_instance_name.restype = C.c_char_p
    lib.ref_instance_name.argtypes = [vp]
    lib.ref_write_mps.restype = C.c_int
    lib.ref_write_mps.argtypes = [C.POINTER(abi.Lp), C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    return lib


def hexs(a):
    return [float(v).hex() for v in a]


def ref_parse(lib, text, fixed):
    data = text.encode()
    h, err, line = C.c_void_p(), C.create_string_buffer(512), C.c_int(0)
    code = lib.ref_parse_mps(data, len(data), int(fixed), C.byref(h), err, 512, C.byref(line))
    if code != 0:
        return {"code": code, "error": err.value.decode(), "line": line.value}
    v = abi.Lp()
    lib.ref_instance_view(h, C.byref(v))

    def arr(p, n, dt):
        return np.ctypeslib.as_array(p, shape=(n,)).astype(dt).tolist() if n else []

    def csr(m):
        rp = arr(m.row_ptr, m.rows + 1, np.int64)
        nz = rp[-1] if rp else 0
        return {"rows": m.rows, "row_ptr": rp, "col_idx": arr(m.col_idx, nz, np.int64),
                "values": hexs(arr(m.values, nz, np.float64))}

    out = {"code": 0, "name": lib.ref_instance_name(h).decode(), "n": v.n, "a": csr(v.a), "g": csr(v.g),
           "c": hexs(arr(v.c, v.n, np.float64)), "b": hexs(arr(v.b, v.a.rows, np.float64)),
           "h": hexs(arr(v.h, v.g.rows, np.float64)), "l": hexs(arr(v.l, v.n, np.float64)),
           "u": hexs(arr(v.u, v.n, np.float64)), "offset": float(v.objective_offset).hex(),
           "negated": int(v.negated_objective)}
    lib.ref_instance_free(h)
    return out


def ref_write(lib, p):
    lp = p.to_c()
    n = C.c_size_t(0)
    assert lib.ref_write_mps(C.byref(lp), (p.name or "").encode(), None, 0, C.byref(n)) == 0
    buf = C.create_string_buffer(n.value)
    assert lib.ref_write_mps(C.byref(lp), (p.name or "").encode(), buf, n.value, C.byref(n)) == 0
    return buf.raw[:n.value].decode()


def writer_cases():
    p = GenRandomLp(12, 9, 0.4, 3, equality_rows=4)
    p.l[0], p.u[0] = -np.inf, np.inf
    p.l[1], p.u[1] = -np.inf, 2.5
    p.l[2], p.u[2] = 1.25, 1.25
    p.l[3], p.u[3] = -3.0, np.inf
    p.objective_offset = 0.75
    p.name = "RANDW"
    return {"random_mixed": p}


def main():
    lib = ref_lib()
    out = {"good": {}, "fixed": {}, "bad": {}, "writer": {}}
    for k, t in mps_corpus.GOOD.items():
        out["good"][k] = ref_parse(lib, t, False)
    for k, t in mps_corpus.FIXED.items():
        out["fixed"][k] = ref_parse(lib, t, True)
    for k, t in mps_corpus.BAD.items():
        out["bad"][k] = ref_parse(lib, t, False)
    for k, p in writer_cases().items():
        out["writer"][k] = ref_write(lib, p)
    dst = Path(__file__).resolve().parent / "mps_golden.json"
    dst.write_text(json.dumps(out, indent=0, sort_keys=True))
    print(f"wrote {dst}")


if __name__ == "__main__":
    main()
