#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_checked.py -x -q -rA > gpurun_out/pytest_checked.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_checked.log
RADULS_GPU_LIB=checked RADULS_GPU_CHECK_JITTER=1 timeout 900 python scripts/sanitize_driver.py > gpurun_out/checked_driver_jitter.log 2>&1
echo "rc=$?" >> gpurun_out/checked_driver_jitter.log
