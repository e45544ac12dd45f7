#!/usr/bin/env bash
O=gpurun_out/r02h; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_solve.py tests/test_suite_cli.py tests/test_gpu_reference_tests.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
echo done
