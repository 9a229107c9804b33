#!/bin/bash
# round 2, call 2: new distributed tests, bench (N=1, per_config, full C5 CPU baseline), reference arm
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
timeout 1200 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_dist.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_dist.log
( time timeout 900 python bench.py --steps 5 --warmup 3 ) > gpurun_out/bench2.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench2.log
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/bench_ref.log
