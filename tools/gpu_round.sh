#!/usr/bin/env bash
# One GPU-box pass: parity suite, smoke, per-kernel probe, bench line, ncu
# launch list and one full ncu capture of the step kernels.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$O/nvidia_smi.txt" 2>&1
nproc > "$O/nproc.txt"
timeout 900 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; echo "smoke exit $?" >> "$O/smoke.log"
timeout 600 python tools/probe.py > "$O/probe.log" 2>&1
timeout 900 python bench.py > "$O/bench.json" 2> "$O/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$O/bench_ref.json" 2> "$O/bench_ref.err"
# launch list of one bench solve (cold-cache, serialised: shares only). ncu
# does not profile kernels inside conditional-graph bodies: keep the default
# host-driven loop here (PDHG_DEVICE_LOOP unset).
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/launches.csv" \
    python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --kernel-iters 8 > "$O/ncu_bench.log" 2>&1
# full capture of the fused step kernels on the transport workload
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"OpPrimal|OpDual" -s 4 -c 4 \
    -o "$O/prof_transport" python tools/profile_step.py transport > "$O/ncu_full.log" 2>&1
echo done
