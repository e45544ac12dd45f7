#!/usr/bin/env bash
# One GPU-box pass: parity suite, smoke, bench line (+ configs 3-5 extras),
# reference arm. Profiling passes live in tools/gpu_ncu.sh.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh <tag>'
set -u
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$O/nvidia_smi.txt" 2>&1
{ nproc; free -g; } > "$O/host.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; echo "smoke exit $?" >> "$O/smoke.log"
timeout 1200 python bench.py ${BENCH_ARGS:-} > "$O/bench.json" 2> "$O/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$O/bench_ref.json" 2> "$O/bench_ref.err"
echo done
