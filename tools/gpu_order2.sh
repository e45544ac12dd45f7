#!/bin/bash
# MCF kernel-variant experiment under first-column row order.
O=gpurun_out/order2; mkdir -p $O
export PDHG_ROW_ORDER=first
timeout 300 python tools/probe.py mcf > $O/base.log 2>&1
PDHG_STAGED_MIN=1000 timeout 300 python tools/probe.py mcf > $O/direct.log 2>&1
PDHG_THREAD_MAX=32 timeout 300 python tools/probe.py mcf > $O/t32.log 2>&1
PDHG_THREAD_MAX=32 PDHG_STAGED_MIN=1000 timeout 300 python tools/probe.py mcf > $O/t32_direct.log 2>&1
PDHG_THREAD_MAX=16 PDHG_STAGED_MIN=1000 timeout 300 python tools/probe.py mcf > $O/t16_direct.log 2>&1
