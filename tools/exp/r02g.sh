#!/usr/bin/env bash
O=gpurun_out/r02g; mkdir -p $O
PDHG_LOOP_TRACE=1 timeout 300 python -m pytest tests/test_gpu_loopback.py -q -p no:cacheprovider -x -k "eight or observer or limits" > $O/pytest_loop.log 2> $O/loop_trace.err; echo "exit $?" >> $O/pytest_loop.log
tail -c 200000 $O/loop_trace.err > $O/loop_trace_tail.err; rm -f $O/loop_trace.err
timeout 1200 python tools/cusparse_cmp.py transport mcf pagerank10m staircase --json $O/cusparse.jsonl > $O/cusparse.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 4 -o $O/ncu_transport python tools/profile_step.py transport > $O/ncu_transport.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 4 -o $O/ncu_mcf python tools/profile_step.py mcf > $O/ncu_mcf.log 2>&1
echo done
