#!/usr/bin/env bash
# Gather-window split of class S: bit-identity tests, per-kernel A/B.
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider -k "split or persistent or staged" > $O/pytest_split.log 2>&1; echo "exit $?" >> $O/pytest_split.log
timeout 1500 python tools/exp/pol_probe.py PDHG_S_SPLIT "0,1" pagerank10m mcf > $O/ab_split.txt 2> $O/ab_split.err
echo done
