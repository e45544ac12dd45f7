#!/usr/bin/env bash
set -u
O=gpurun_out/r01p
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport random pagerank1m > "$O/probe.log" 2>&1
PDHG_PDL=0 timeout 600 python tools/probe.py transport random pagerank1m > "$O/probe_nopdl.log" 2>&1
echo done
