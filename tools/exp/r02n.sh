#!/usr/bin/env bash
# Event-barrier loopback suite; persistent / 128-chunk class-S kernels:
# bit-identity tests and per-kernel A/B on configs 2-5.
O=gpurun_out/r02n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider > $O/loop.log 2>&1; echo "exit $?" >> $O/loop.log
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > $O/pytest_solve.log 2>&1; echo "exit $?" >> $O/pytest_solve.log
timeout 300 python tools/profile_step.py transport - 512 > $O/transport.txt 2>&1
timeout 1500 python tools/exp/pol_probe.py - "PDHG_S_CHUNK=256,PDHG_S_CHUNK=128,PDHG_S_FLOW=3+PDHG_S_CHUNK=128,PDHG_S_FLOW=4+PDHG_S_CHUNK=128" pagerank10m > $O/ab_pr.txt 2> $O/ab_pr.err
timeout 1500 python tools/exp/pol_probe.py - "PDHG_S_FLOW=0+PDHG_S_CHUNK=256,PDHG_S_FLOW=3,PDHG_S_FLOW=4" mcf staircase > $O/ab_mcf_stair.txt 2> $O/ab_mcf_stair.err
echo done
