#!/usr/bin/env bash
set -u
O=gpurun_out/r01g
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m mcf staircase random > "$O/probe.log" 2>&1
PDHG_RPC4_MAX=0 PDHG_UNIFORM_S=0 timeout 300 python tools/probe.py transport pagerank1m mcf > "$O/probe_off.log" 2>&1
unset PDHG_TRACE
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k regex:"OpDual|OpPrimal" -s 6 -c 4 -o "$O/prof_transport" python tools/profile_step.py transport > "$O/ncu_transport.log" 2>&1
echo done
