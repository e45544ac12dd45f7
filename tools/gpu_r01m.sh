#!/usr/bin/env bash
set -u
O=gpurun_out/r01m
mkdir -p "$O"
timeout 900 python tools/probe.py pagerank10m mcf transport > "$O/probe.log" 2>&1
PDHG_L2_PERSIST=0 timeout 900 python tools/probe.py pagerank10m mcf > "$O/probe_nopersist.log" 2>&1
echo done
