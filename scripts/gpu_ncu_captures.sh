#!/bin/bash
# checked suite log; ncu source-level captures of k_local (C1, C2) and k_scatter (C1); bench launch list
mkdir -p gpurun_out
RADULS_GPU_LIB=checked timeout 1500 python -m pytest -q -rA -m gpu -k "not full_size and not c5_full and not concurrent and not frees_its and not allocation_failure" \
  tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_lsd.py tests/test_gpu_local_edges.py tests/test_gpu_digit_array.py tests/test_gpu_progressive.py \
  > gpurun_out/checked_parity_suite.log 2>&1
echo "rc=$?" >> gpurun_out/checked_parity_suite.log
for CFG in c1 c2; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_local -s 1 -c 1 \
     -o gpurun_out/loc_$CFG -f python scripts/prof_one.py $CFG 2 > gpurun_out/loc_ncu_$CFG.log 2>&1
  ncu -i gpurun_out/loc_$CFG.ncu-rep --page source --csv --print-source sass > gpurun_out/loc_${CFG}_sass.csv 2>&1
  ncu -i gpurun_out/loc_$CFG.ncu-rep --page raw --csv > gpurun_out/loc_${CFG}_raw.csv 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scatter -s 2 -c 1 \
   -o gpurun_out/sc_c1 -f python scripts/prof_one.py c1 2 > gpurun_out/sc_ncu_c1.log 2>&1
ncu -i gpurun_out/sc_c1.ncu-rep --page source --csv --print-source sass > gpurun_out/sc_c1_sass.csv 2>&1
ncu -i gpurun_out/sc_c1.ncu-rep --page raw --csv > gpurun_out/sc_c1_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
