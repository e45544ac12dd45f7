#!/usr/bin/env bash
set -u
O=gpurun_out/r01t
mkdir -p "$O"
timeout 900 python tools/probe.py mcf pagerank1m staircase > "$O/probe.log" 2>&1
PDHG_THREAD_MAX=64 timeout 900 python tools/probe.py mcf pagerank1m staircase > "$O/probe_t64.log" 2>&1
PDHG_THREAD_MAX=64 PDHG_STAGED_MIN=3 timeout 900 python tools/probe.py mcf pagerank1m > "$O/probe_t64s3.log" 2>&1
echo done
