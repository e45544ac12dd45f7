"""A/B of an env toggle on resident solves (AB_PROBLEM=transport | random |
pagerank | mcf), alternating in fresh processes on one box:
python tools/ab_solve.py VAR A B [rounds]."""
import json
import os
import subprocess
import sys

code = r'''
import sys, json
sys.path.insert(0, ".")
from paper_2312_14832_b200 import rpdlp
import os
which = os.environ.get("AB_PROBLEM", "transport")
p = {"transport": lambda: rpdlp.GenTransport(1000, 1000, 1),
     "random": lambda: rpdlp.GenRandomLp(1000, 2000, 0.005, 1, equality_rows=300),
     "pagerank": lambda: rpdlp.GenPagerank(100_000, 0.85, 6, 1),
     "mcf": lambda: rpdlp.GenMcf(50_000, 330_000, 50, 1)}[which]()
prm = rpdlp.SolverParams(eps=1e-4)
with rpdlp.Session(p) as s:
    for _ in range(2):
        s.solve(prm)
    ms = []
    for _ in range(5):
        s.flush_l2()
        r = s.solve(prm)
        ms.append(s.last_solve()[0])
print(json.dumps(ms))
'''
var, a, b = sys.argv[1:4]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
res = {a: [], b: []}
for _ in range(rounds):
    for v in (a, b):
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **{var: v}), capture_output=True,
                             text=True, check=True).stdout
        res[v] += json.loads(out.strip().splitlines()[-1])
for v in (a, b):
    xs = sorted(res[v])
    print(f"{var}={v}: median {xs[len(xs) // 2]:.2f} ms, min {xs[0]:.2f} ms over {len(xs)} solves")
