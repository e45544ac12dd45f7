import time, numpy as np, ctypes as C, sys
sys.path.insert(0, ".")
from paper_2312_14832_b200 import abi
L = abi.load()
P=C.POINTER(C.c_double)
n=1_000_000
for th in (1, 4, 8, 16):
    out = np.empty(n); ts=[]
    for _ in range(7):
        t=time.perf_counter(); L.pdhg_normal_vector(7, n, th, out.ctypes.data_as(P)); ts.append(time.perf_counter()-t)
    print(th, round(min(ts)*1e3,2), "ms median", round(sorted(ts)[3]*1e3,2))
