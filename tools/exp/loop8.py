"""Debug: 8 loopback ranks on the staircase ghost case (run with
CUDA_DEVICE_MAX_CONNECTIONS=32 PDHG_LOOP_TRACE=1)."""
import faulthandler
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
faulthandler.dump_traceback_later(170, exit=True)
from paper_2312_14832_b200 import rpdlp  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = rpdlp.GenStaircase(16, 60, 60, 8, 2, seed=5)
params = rpdlp.SolverParams(eps=1e-6, iter_limit=20000)
specs = rpdlp.Shards.loopback(W)
out = [None] * W


def rank(r):
    try:
        with rpdlp.Session(p, params, shards=specs[r]) as s:
            print(f"rank {r} constructed ghost={s.ghost_counts()[2]}", flush=True)
            out[r] = s.solve(params)
            print(f"rank {r} solved {out[r].iterations}", flush=True)
    except BaseException as e:  # noqa: BLE001
        out[r] = e
        print(f"rank {r} error {e!r}", flush=True)


th = [threading.Thread(target=rank, args=(r,)) for r in range(W)]
for t in th:
    t.start()
for t in th:
    t.join()
print([getattr(o, "iterations", o) for o in out])
