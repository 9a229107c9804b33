#!/bin/bash
# round 2, call 1: box facts, scatter-ranking A/B, GPU tests
mkdir -p gpurun_out
{ nvidia-smi; nproc; free -g; lscpu | head -30; cat /proc/meminfo | head -5; } > gpurun_out/box.txt 2>&1
timeout 900 python scripts/ab_interleave.py c1 c2 c5 c4 --reps 5 --kt > gpurun_out/ab_rank.log 2>&1
echo "ab rc=$?" >> gpurun_out/ab_rank.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
