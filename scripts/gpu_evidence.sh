#!/bin/bash
# round 2 evidence: driver-shaped bench line, launch list of the bench command, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2_box.txt 2>&1
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
echo "bench rc=$?" >> gpurun_out/r2_bench_c5.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/r2_launches_bench_c5.csv $CMD > gpurun_out/r2_ncu_bench.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/r2_ncu_bench.log
