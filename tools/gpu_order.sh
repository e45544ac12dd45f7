#!/bin/bash
# Secondary segment order experiment (PDHG_ROW_ORDER / PDHG_COL_ORDER).
O=gpurun_out/order; mkdir -p $O
for ro in natural first; do
  for co in natural first; do
    PDHG_ROW_ORDER=$ro PDHG_COL_ORDER=$co timeout 900 python tools/probe.py mcf pagerank1m pagerank10m staircase transport random > $O/probe_${ro}_${co}.log 2>&1
  done
done
