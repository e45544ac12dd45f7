#!/usr/bin/env bash
# Round-1 pass d: warp-staged thread kernel, uniform bounds, no solve-path allocations.
set -u
O=gpurun_out/r01d
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m mcf staircase random > "$O/probe.log" 2>&1
PDHG_THREAD_MAX=4 PDHG_WARP_MAX=4 PDHG_CTA_MAX=4 timeout 600 python tools/probe.py pagerank1m mcf staircase > "$O/probe_tile4.log" 2>&1
PDHG_UNIFORM_BOUNDS=0 timeout 300 python tools/probe.py transport > "$O/probe_nobnd.log" 2>&1
unset PDHG_TRACE
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k regex:"OpDual|OpPrimal" -s 6 -c 4 -o "$O/prof_transport" python tools/profile_step.py transport 40 > "$O/ncu_transport.log" 2>&1
timeout 600 $NCU -k regex:"OpDual|OpPrimal" -s 12 -c 8 -o "$O/prof_pagerank" python tools/profile_step.py pagerank 1000000 > "$O/ncu_pagerank.log" 2>&1
timeout 900 python bench.py > "$O/bench.json" 2> "$O/bench.err"
echo done
