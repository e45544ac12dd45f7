import os, subprocess, sys, numpy as np
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2312_14832_b200 import rpdlp
out = {}
for name, p in [("t1000", rpdlp.GenTransport(1000, 1000, 1)), ("t600", rpdlp.GenTransport(600, 40, 3)), ("t64", rpdlp.GenTransport(64, 900, 2))]:
    r = rpdlp.Solve(p, rpdlp.SolverParams(eps=1e-6, iter_limit=3000))
    out[name] = (r.iterations, r.x, r.y)
np.savez(sys.argv[1], **{k + "_x": v[1] for k, v in out.items()}, **{k + "_y": v[2] for k, v in out.items()}, **{k + "_it": v[0] for k, v in out.items()})
'''
for flag in ("0", "1"):
    env = dict(os.environ, PDHG_CTA_STAGE=flag)
    subprocess.run([sys.executable, "-c", code, f"/tmp/st{flag}.npz"], env=env, check=True)
a, b = np.load("/tmp/st0.npz"), np.load("/tmp/st1.npz")
for k in a.files:
    print(k, "identical" if np.array_equal(a[k], b[k]) else "DIFFERENT")
