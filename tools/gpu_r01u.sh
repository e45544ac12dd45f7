#!/usr/bin/env bash
set -u
O=gpurun_out/r01u
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
timeout 900 python tools/probe.py transport random mcf pagerank1m staircase > "$O/probe.log" 2>&1
echo done
