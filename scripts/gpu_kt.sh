#!/bin/bash
# per-kernel times of the bench workloads (no e2e / cpu baseline)
mkdir -p gpurun_out
for c in ${KT_CONFIGS:-c5}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/kt_$c.json 2> gpurun_out/kt_$c.err
done
