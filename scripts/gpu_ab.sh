#!/bin/bash
# A/B call: new tests first, the GPU suite, then the perf probe with and without a knob (env AB_ENV).
mkdir -p gpurun_out
timeout 600 python -m pytest ${FIRST_TESTS:-tests/test_gpu_digit_array.py} -x -q > gpurun_out/pytest_first.log 2>&1
echo "first rc=$?" >> gpurun_out/pytest_first.log
timeout 300 python scripts/perf_probe.py ${PROBE_CONFIGS:-c1 c2 c3 c4 c5} > gpurun_out/perf_a.log 2>&1
echo "perf rc=$?" >> gpurun_out/perf_a.log
if [ -n "$AB_ENV" ]; then
  env $AB_ENV timeout 300 python scripts/perf_probe.py ${PROBE_CONFIGS:-c1 c2 c3 c4 c5} > gpurun_out/perf_b.log 2>&1
  echo "perf rc=$?" >> gpurun_out/perf_b.log
fi
if [ -z "$SKIP_SUITE" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
