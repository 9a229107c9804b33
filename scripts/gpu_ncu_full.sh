#!/bin/bash
# full ncu capture of selected kernels of one config (after a plain run)
mkdir -p gpurun_out
CFG=${1:-c1}
TAG=${2:-r1}
shift 2
KERNELS=${@:-k_local_sort k_scatter}
timeout 300 python scripts/prof_one.py $CFG 1 > gpurun_out/full_plain_$CFG.log 2>&1 || { echo "plain failed" >> gpurun_out/full_plain_$CFG.log; exit 1; }
for K in $KERNELS; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 0 -c 1 \
     -o gpurun_out/full_${CFG}_${K}_${TAG} -f python scripts/prof_one.py $CFG 1 > gpurun_out/full_ncu_${CFG}_${K}.log 2>&1
  echo "rc=$?" >> gpurun_out/full_ncu_${CFG}_${K}.log
done
