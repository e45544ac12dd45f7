#!/usr/bin/env bash
set -u
O=gpurun_out/r01r
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
PDHG_TRACE=1 timeout 900 python bench.py --no-cpu --eps-tight 0 > "$O/bench.json" 2> "$O/bench.err"
echo done
