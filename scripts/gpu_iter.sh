#!/bin/bash
# iteration call: GPU tests, perf probe, launch list of one config
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/perf_probe.py ${PROBE_CONFIGS:-c1 c2 c3 c4} > gpurun_out/perf.log 2>&1
echo "perf rc=$?" >> gpurun_out/perf.log
if [ -n "$PROF_CFG" ]; then bash scripts/gpu_prof.sh $PROF_CFG; fi
