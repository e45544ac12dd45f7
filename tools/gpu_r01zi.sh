#!/usr/bin/env bash
set -u
O=gpurun_out/r01zi
mkdir -p "$O"
timeout 3000 python tools/configs_run.py random transport mcf pagerank10m staircase --time-limit 200 > "$O/configs.jsonl" 2> "$O/configs.err"
echo done
