set -e
timeout 600 python tools/ab_solve.py PDHG_POWER_GRAPH_STEPS 1 4 3 > gpurun_out/ab_power.log 2>&1
for s in 1 4 1 4; do echo "steps=$s"; PDHG_POWER_GRAPH_STEPS=$s PDHG_TRACE=1 timeout 300 python tools/e2e_trace.py --solves 4 2>&1 | grep -E "^solve|\] solve" | tail -4; done >> gpurun_out/ab_power.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/power_pytest.log 2>&1
