#!/usr/bin/env bash
set -u
O=gpurun_out/r01v
mkdir -p "$O"
for t in 128 256; do PDHG_THREAD_MAX=$t timeout 900 python tools/probe.py mcf pagerank1m staircase random > "$O/probe_t$t.log" 2>&1; done
echo done
