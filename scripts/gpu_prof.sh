#!/bin/bash
# launch list of one config under ncu (after a plain run)
mkdir -p gpurun_out
CFG=${1:-c1}
timeout 300 python scripts/prof_one.py $CFG 2 > gpurun_out/prof_plain_$CFG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python scripts/prof_one.py $CFG 2 > gpurun_out/ncu_$CFG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$CFG.log
