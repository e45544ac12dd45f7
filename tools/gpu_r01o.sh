#!/usr/bin/env bash
set -u
O=gpurun_out/r01o
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
timeout 600 python tools/probe.py transport staircase --shards 4 > "$O/probe_shards4.log" 2>&1
echo done
