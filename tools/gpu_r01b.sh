#!/usr/bin/env bash
# Round-1 pass b: sharded-path parity, class-threshold sweep, ncu of the step kernels.
set -u
O=gpurun_out/r01b
mkdir -p "$O"
free -g > "$O/free.txt"; nproc >> "$O/free.txt"
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
timeout 900 python tools/probe.py transport pagerank1m mcf staircase > "$O/probe.log" 2>&1
for t in 256 768; do PDHG_CTA_MAX=$t timeout 300 python tools/probe.py transport pagerank1m mcf > "$O/probe_cta$t.log" 2>&1; done
PDHG_WARP_MAX=128 timeout 300 python tools/probe.py transport pagerank1m mcf > "$O/probe_warp128.log" 2>&1
timeout 600 python tools/probe.py transport mcf staircase --shards 4 > "$O/probe_shards4.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"OpPrimal|OpDual" -s 6 -c 4 \
    -o "$O/prof_transport" python tools/profile_step.py transport > "$O/ncu_transport.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"OpPrimal|OpDual" -s 12 -c 8 \
    -o "$O/prof_pagerank" python tools/profile_step.py pagerank > "$O/ncu_pagerank.log" 2>&1
echo done
