#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_local_edges.py tests/test_gpu_digit_array.py tests/test_gpu_progressive.py tests/test_gpu_lsd.py tests/test_gpu_checked.py > gpurun_out/r2_p8_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2_p8_pytest.log
timeout 1200 python scripts/ab_interleave.py c1 c3 c4 c5 c2 --reps 5 --kt > gpurun_out/r2_ab_list.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ab_list.log
