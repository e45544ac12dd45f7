#!/usr/bin/env bash
set -u
O=gpurun_out/r01f
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m mcf staircase random > "$O/probe.log" 2>&1
PDHG_WARP_MAX=1024 timeout 300 python tools/probe.py transport > "$O/probe_warp1024.log" 2>&1
unset PDHG_TRACE
timeout 900 python bench.py > "$O/bench.json" 2> "$O/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/launches.csv" \
    python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --kernel-iters 8 --eps-tight 0 > "$O/ncu_bench.log" 2>&1
echo done
