#!/usr/bin/env bash
# Session-3 diagnostics: loopback rendezvous trace, HEAD vs round-1 A/B on
# transport, gather-roofline calibration, GPU suite (minus loopback), fresh
# per-kernel times on configs 2-5, ncu of the PageRank-10M dual class-S kernel.
O=gpurun_out/r02m; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 PDHG_FORK=0 PDHG_LOOP_TRACE=1 timeout 240 python -m pytest tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider -k "config1-2 or config1-3" > $O/loop.log 2> $O/loop.err; echo "exit $?" >> $O/loop.log
tail -c 300000 $O/loop.err > $O/loop_tail.err; rm -f $O/loop.err
for t in . _old; do (cd $t && timeout 300 python tools/profile_step.py transport - 512) >> $O/ab_transport.txt 2>&1; done
for t in . _old; do (cd $t && timeout 300 python tools/profile_step.py transport - 512) >> $O/ab_transport.txt 2>&1; done
(cd _old && timeout 600 python bench.py --extra "" --steps 5 --warmup 3 > ../$O/bench_old.json 2> ../$O/bench_old.err)
timeout 600 python bench.py --extra "" --steps 5 --warmup 3 > $O/bench_new.json 2> $O/bench_new.err
timeout 300 tools/_build/gather_probe 80 > $O/gather_probe_80m.jsonl 2> $O/gather_probe.err
timeout 300 tools/_build/gather_probe 200 > $O/gather_probe_200m.jsonl 2>> $O/gather_probe.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_loopback.py::test_loopback_suite > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"seg_thread_staged_kernel<pdhg::OpDual" -c 1 -o $O/ncu_pr10m_dualS python tools/profile_step.py pagerank 10000000 2 > $O/ncu_pr10m.log 2>&1
timeout 1200 python tools/exp/pol_probe.py PDHG_NOP 0 transport mcf pagerank10m staircase > $O/kernels.txt 2> $O/kernels.err
echo done
