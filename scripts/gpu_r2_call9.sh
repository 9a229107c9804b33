#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest -x -q -m gpu tests/test_gpu_kernels.py tests/test_gpu_distributed.py tests/test_gpu_multi.py tests/test_gpu_checked.py > gpurun_out/r2_p9_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2_p9_pytest.log
