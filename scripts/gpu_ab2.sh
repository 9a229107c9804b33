#!/bin/bash
# A/B of var/lib_*.so (ROUNDS passes, KT_CONFIGS), then the GPU suite on the in-tree library.
mkdir -p gpurun_out
cp paper_1612_02557_b200/libraduls_gpu.so /tmp/intree.so
for r in $(seq ${ROUNDS:-2}); do bash scripts/gpu_variants.sh; done > gpurun_out/ab.log 2>&1
cp /tmp/intree.so paper_1612_02557_b200/libraduls_gpu.so
if [ -z "$SKIP_SUITE" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
