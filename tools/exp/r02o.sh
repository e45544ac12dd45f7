#!/usr/bin/env bash
# Tile gather sweep (default on) + routing of long PageRank rows; effective
# L2 capacity for random gathers; GPU suite.
O=gpurun_out/r02o; mkdir -p $O
timeout 300 tools/_build/gather_probe 80 > $O/gather_probe_80m.jsonl 2> $O/gather_probe.err
timeout 1500 python tools/exp/pol_probe.py - "PDHG_TILE_SWEEP=0,PDHG_TILE_SWEEP=1,PDHG_CTA_MAX=512,PDHG_WARP_MAX=64+PDHG_CTA_MAX=64,PDHG_TILE_SWEEP=0" pagerank10m > $O/ab_sweep.txt 2> $O/ab_sweep.err
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
echo done
