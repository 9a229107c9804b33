#!/bin/bash
# round profile artifacts: launch list of the bench command + full captures of the scatter and the local sort (C1)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/launches_bench_c5.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_bench.log
timeout 300 python scripts/prof_one.py c1 1 > gpurun_out/full_plain_c1.log 2>&1 && \
for K in k_scatter k_local; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 0 -c 1 \
     -o gpurun_out/full_c1_${K}_final -f python scripts/prof_one.py c1 1 > gpurun_out/full_ncu_$K.log 2>&1
  echo "full $K rc=$?" >> gpurun_out/full_ncu_$K.log
done
