#!/bin/bash
# One gpurun call: box probe, GPU tests, perf probe. Output under gpurun_out/.
mkdir -p gpurun_out
{ nvidia-smi; nproc; free -g; lscpu | head -20; } > gpurun_out/box.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/perf_probe.py ${PROBE_CONFIGS:-c1 c2 c3 c4} > gpurun_out/perf.log 2>&1
echo "perf rc=$?" >> gpurun_out/perf.log
