#!/bin/bash
# the round's evidence run: driver-shaped bench line, reference arm, ncu launch
# list of the bench command, full captures of the local sort and the scatter (C1)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/ev_box.txt 2>&1
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_bench_c5.json 2> gpurun_out/ev_bench_c5.err
echo "bench rc=$?" >> gpurun_out/ev_bench_c5.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
echo "ref rc=$?" >> gpurun_out/ev_bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/ev_launches_bench_c5.csv $CMD > gpurun_out/ev_ncu_bench.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ev_ncu_bench.log
cap() {  # name regex skip config
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$2" -s $3 -c 1 \
     -o gpurun_out/ev_full_$1 -f python scripts/prof_one.py $4 2 > gpurun_out/ev_ncu_full_$1.log 2>&1
  ncu -i gpurun_out/ev_full_$1.ncu-rep --page raw --csv > gpurun_out/ev_full_$1_raw.csv 2>&1
  ncu -i gpurun_out/ev_full_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ev_full_$1_sass.csv 2>&1
}
cap local_c1 '^k_local_bm$' 1 c1
cap scatter_c1 'k_scatter' 2 c1
cap local_c2 '^k_local_bm8$' 1 c2
cap local_c4 '^k_local_bm$' 1 c4
rm -f gpurun_out/*.ncu-rep
python scripts/traffic_from_launches.py gpurun_out/ev_launches_bench_c5.csv > gpurun_out/ev_ncu_traffic_c5.json 2>&1
