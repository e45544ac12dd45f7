#!/usr/bin/env bash
set -u
O=gpurun_out/r01e
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m mcf staircase random > "$O/probe.log" 2>&1
PDHG_STAGED_MIN=4 timeout 600 python tools/probe.py pagerank1m mcf > "$O/probe_st4.log" 2>&1
timeout 900 python bench.py --no-cpu --eps-tight 0 > "$O/bench.json" 2> "$O/bench.err"
echo done
