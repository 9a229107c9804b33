#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import paper_1612_02557_b200 as rg; print('rank_mode', rg.rank_mode())" >> gpurun_out/pytest_gpu.log 2>&1
bash scripts/sanitize.sh memcheck synccheck racecheck > gpurun_out/sanitize_summary.log 2>&1
