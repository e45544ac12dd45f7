#!/usr/bin/env bash
set -u
O=gpurun_out/r01h
mkdir -p "$O"
timeout 1500 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$O/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; echo "smoke exit $?" >> "$O/smoke.log"
export PDHG_TRACE=1
timeout 600 python tools/probe.py transport pagerank1m mcf > "$O/probe.log" 2>&1
unset PDHG_TRACE
timeout 900 python bench.py > "$O/bench.json" 2> "$O/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$O/bench_ref.json" 2> "$O/bench_ref.err"
echo done
