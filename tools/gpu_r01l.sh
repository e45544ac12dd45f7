#!/usr/bin/env bash
set -u
O=gpurun_out/r01l
mkdir -p "$O"
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
# warm-up steps: 3 x (primal + dual classes); then profile the next ~8 launches
timeout 1200 $NCU -k regex:"OpDual|OpPrimal" -s 12 -c 10 -o "$O/prof_pagerank10m" python tools/profile_step.py pagerank 10000000 > "$O/ncu_pr.log" 2>&1
timeout 600 $NCU -k regex:"OpDual|OpPrimal" -s 6 -c 6 -o "$O/prof_mcf" python tools/profile_step.py mcf > "$O/ncu_mcf.log" 2>&1
echo done
