#!/usr/bin/env bash
# modal-prefix primal: parity subset, timing, ncu of PageRank-10M and staircase step kernels
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_fullscale.py > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python tools/exp/pol_probe.py PDHG_UNIFORM_S 1,0 pagerank10m > $O/probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 10 -o $O/ncu_pr10m python tools/profile_step.py pagerank 10000000 2 > $O/ncu_pr10m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 4 -o $O/ncu_stair python tools/profile_step.py staircase - 2 > $O/ncu_stair.log 2>&1
echo done
