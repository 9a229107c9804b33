#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest3.log
( time timeout 600 python bench.py --steps 3 --warmup 3 --no-per-config --no-cpu-baseline ) > gpurun_out/bench3.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench3.log
