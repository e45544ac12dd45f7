#!/usr/bin/env bash
set -u
O=gpurun_out/r01j
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m random > "$O/probe.log" 2>&1
PDHG_PIPELINE=0 timeout 600 python tools/probe.py transport random > "$O/probe_sync.log" 2>&1
unset PDHG_TRACE
timeout 900 python bench.py --no-cpu > "$O/bench.json" 2> "$O/bench.err"
echo done
