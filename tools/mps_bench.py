"""MPS ingestion: the product reader (mps.cpp, COLUMNS
tokenised on worker threads) against the unmodified reference parser
(oracle/_ref, mps_reader.cpp), same text in memory, parse only.

    python tools/mps_bench.py [pagerank1m transport mcf_small] [--json out.json]
"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2312_14832_b200 import abi, rpdlp  # noqa: E402

CASES = {
    "pagerank1m": lambda: rpdlp.GenPagerank(1_000_000, 0.85, 6, 1),
    "transport": lambda: rpdlp.GenTransport(1000, 1000, 1),
    "mcf_small": lambda: rpdlp.GenMcf(5_000, 33_000, 50, 1),
}


def main(argv):
    out = None
    if "--json" in argv:
        i = argv.index("--json")
        out = argv[i + 1]
        del argv[i:i + 2]
    from golden.make_mps_golden import ref_lib
    ref = ref_lib()
    lib = abi.load()
    recs = []
    for name in argv or list(CASES):
        p = CASES[name]()
        text = rpdlp.WriteMps(p).encode()
        del p
        best = {}
        for who in ("reference", "b200"):
            ts = []
            for _ in range(3):
                h = C.c_void_p()
                err = C.create_string_buffer(512)
                line = C.c_int(0)
                t = time.perf_counter()
                if who == "reference":
                    code = ref.ref_parse_mps(text, len(text), 0, C.byref(h), err, 512, C.byref(line))
                else:
                    code = lib.pdhg_mps_read_string(text, len(text), 0, C.byref(h), err, 512, C.byref(line))
                ts.append(time.perf_counter() - t)
                assert code == 0, err.value
                (ref.ref_instance_free if who == "reference" else lib.pdhg_instance_free)(h)
            best[who] = min(ts)
        rec = {"instance": name, "mb": len(text) / 1e6, "reference_s": best["reference"], "b200_s": best["b200"],
               "speedup": best["reference"] / best["b200"], "host_threads": os.cpu_count(),
               "reference_mb_s": len(text) / 1e6 / best["reference"], "b200_mb_s": len(text) / 1e6 / best["b200"]}
        recs.append(rec)
        print(f"{name}: {rec['mb']:.0f} MB  reference {rec['reference_s']:.3f}s ({rec['reference_mb_s']:.0f} MB/s)  "
              f"b200 reader {rec['b200_s']:.3f}s ({rec['b200_mb_s']:.0f} MB/s)  -> {rec['speedup']:.1f}x "
              f"({os.cpu_count()} host threads)", flush=True)
    if out:
        Path(out).write_text(json.dumps(recs, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
