#!/usr/bin/env bash
O=gpurun_out/r02i; mkdir -p $O
CUDA_DEVICE_MAX_CONNECTIONS=32 PDHG_LOOP_TRACE=1 timeout 200 python tools/exp/loop8.py 8 > $O/loop8.out 2> $O/loop8.err
tail -c 300000 $O/loop8.err > $O/loop8_tail.err; rm $O/loop8.err
timeout 900 python -m pytest tests/test_gpu_solve.py -q -p no:cacheprovider -k "pipelined_class_s or kernel_variant or staged_cta" > $O/pytest_pipe.log 2>&1
timeout 900 python tools/exp/pol_probe.py PDHG_S_PIPE 1,0 pagerank10m mcf staircase > $O/pipe_probe.log 2>&1
echo done
