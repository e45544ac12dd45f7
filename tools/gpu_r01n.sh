#!/usr/bin/env bash
set -u
O=gpurun_out/r01n
mkdir -p "$O"
timeout 600 python tools/probe.py transport > "$O/probe.log" 2>&1
PDHG_L_WIDE=0 timeout 600 python tools/probe.py transport > "$O/probe_narrow.log" 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py -m gpu -x -q > "$O/pytest.log" 2>&1; echo "exit $?" >> "$O/pytest.log"
echo done
