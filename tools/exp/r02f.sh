#!/usr/bin/env bash
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -p no:cacheprovider -x > $O/pytest_loop.log 2>&1; echo "exit $?" >> $O/pytest_loop.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 10 -o $O/ncu_pr10m python tools/profile_step.py pagerank 10000000 2 > $O/ncu_pr10m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 4 -o $O/ncu_stair python tools/profile_step.py staircase - 2 > $O/ncu_stair.log 2>&1
echo done
