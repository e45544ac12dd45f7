#!/bin/bash
# Segment-order warps of the staged class-S kernel: A/B and bit-identity.
O=gpurun_out/rm; mkdir -p $O
for f in 0 1 0 1; do
  PDHG_SEG_ORDER_WARPS=$f timeout 300 python tools/probe.py mcf pagerank1m staircase > $O/probe_$f.log 2>&1
  echo "flag $f: $(grep -E 'iter ' $O/probe_$f.log | tr '\n' ' ')" >> $O/summary.txt
done
timeout 600 python - >> $O/summary.txt 2>&1 <<'PY'
import os, subprocess, sys
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2312_14832_b200 import rpdlp
p = rpdlp.GenMcf(3000, 20000, 20, 2)
r = rpdlp.Solve(p, rpdlp.SolverParams(eps=1e-6, iter_limit=2000))
np.savez(sys.argv[1], x=r.x, y=r.y, it=r.iterations)
'''
for f in ("0", "1"):
    subprocess.run([sys.executable, "-c", code, f"/tmp/rm{f}.npz"], env=dict(os.environ, PDHG_SEG_ORDER_WARPS=f), check=True)
import numpy as np
a, b = np.load("/tmp/rm0.npz"), np.load("/tmp/rm1.npz")
print("bit-identical:", all(np.array_equal(a[k], b[k]) for k in a.files))
PY
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
