#!/bin/bash
# round 2: GPU suite + rank mode + default bench
mkdir -p gpurun_out
{ nvidia-smi; nproc; free -g; lscpu | head -20; } > gpurun_out/box.txt 2>&1
python -c "import paper_1612_02557_b200 as rg; print('rank_mode', rg.rank_mode())" > gpurun_out/rank_mode.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
