#!/usr/bin/env bash
# Round-1 pass c: parity suite, engine variants (predicated batches, fork/join
# classes, degree order, tile-engine routing), ncu of the transport step kernels.
set -u
O=gpurun_out/r01c
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m mcf staircase > "$O/probe.log" 2>&1
PDHG_DEGREE_ORDER=0 timeout 600 python tools/probe.py pagerank1m mcf staircase > "$O/probe_nodeg.log" 2>&1
PDHG_THREAD_MAX=4 PDHG_WARP_MAX=4 PDHG_CTA_MAX=4 timeout 600 python tools/probe.py transport pagerank1m mcf staircase > "$O/probe_tile4.log" 2>&1
PDHG_THREAD_MAX=8 PDHG_WARP_MAX=8 PDHG_CTA_MAX=8 timeout 600 python tools/probe.py pagerank1m mcf staircase > "$O/probe_tile8.log" 2>&1
PDHG_THREAD_MAX=2 PDHG_WARP_MAX=2 PDHG_CTA_MAX=2 timeout 600 python tools/probe.py pagerank1m mcf staircase > "$O/probe_tile2.log" 2>&1
unset PDHG_TRACE
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"OpDual" -s 3 -c 2 \
    -o "$O/prof_transport_dual" python tools/profile_step.py transport > "$O/ncu_transport_dual.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"OpPrimal" -s 3 -c 2 \
    -o "$O/prof_transport_primal" python tools/profile_step.py transport > "$O/ncu_transport_primal.log" 2>&1
echo done
