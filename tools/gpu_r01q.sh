#!/usr/bin/env bash
set -u
O=gpurun_out/r01q
mkdir -p "$O"
timeout 900 python bench.py > "$O/bench.json" 2> "$O/bench.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/launches.csv" \
    python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --kernel-iters 8 --eps-tight 0 > "$O/ncu_bench.log" 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k regex:"OpDual|OpPrimal" -s 6 -c 4 -o "$O/prof_transport" python tools/profile_step.py transport > "$O/ncu_transport.log" 2>&1
echo done
