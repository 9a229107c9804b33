#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_driver.py), both
# scatter ranking modes. Logs to gpurun_out/sanitize_<tool>[_ballot].log.
#   bash scripts/sanitize.sh [memcheck racecheck synccheck initcheck]
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
tools=${@:-memcheck racecheck synccheck}
for tool in $tools; do
  for mode in atomic ballot; do
    log=gpurun_out/sanitize_${tool}_${mode}.log
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    [ "$mode" = ballot ] && export RADULS_GPU_STABLE_RANK=ballot || unset RADULS_GPU_STABLE_RANK
    q=""; [ "$tool" = racecheck ] && q="--quick"
    timeout 1500 $CS --tool $tool $extra --print-limit 50 python scripts/sanitize_driver.py $q > $log 2>&1
    echo "rc=$?" >> $log
    tail -3 $log
  done
done
