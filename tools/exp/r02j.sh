#!/usr/bin/env bash
O=gpurun_out/r02k; mkdir -p $O
CUDA_DEVICE_MAX_CONNECTIONS=32 PDHG_FORK=0 PDHG_LOOP_TRACE=1 timeout 200 python tools/exp/loop8.py 8 > $O/loop8.out 2> $O/loop8.err
tail -c 100000 $O/loop8.err > $O/loop8_tail.err; rm $O/loop8.err
timeout 1500 python -m pytest tests/test_gpu_loopback.py -m gpu -q -p no:cacheprovider > $O/pytest_loop.log 2>&1; echo "exit $?" >> $O/pytest_loop.log
echo done
timeout 900 python tools/exp/pol_probe.py - "PDHG_THREAD_MAX=64,PDHG_CTA_MAX=512,PDHG_WARP_MAX=64+PDHG_CTA_MAX=64,PDHG_WARP_MAX=512+PDHG_CTA_MAX=16384+PDHG_STAGED_MIN=100,PDHG_STAGED_MIN=3+PDHG_ROW_ORDER=natural" pagerank10m > gpurun_out/r02k/route_probe.log 2>&1
