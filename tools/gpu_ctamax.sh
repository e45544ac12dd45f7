#!/bin/bash
# Class-L / XL boundary (PDHG_CTA_MAX) on the power-law instances.
O=gpurun_out/ctamax; mkdir -p $O
for c in 16384 4096 2048 16384 4096 2048; do
  PDHG_CTA_MAX=$c timeout 300 python tools/probe.py pagerank1m pagerank10m mcf > $O/probe_$c.log 2>&1
  echo "cta_max $c: $(grep -E 'iter ' $O/probe_$c.log | sed 's/ -> .*//' | tr '\n' ' ')" >> $O/summary.txt
done
