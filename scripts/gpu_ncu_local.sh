mkdir -p gpurun_out
for CFG in ${CFGS:-c1 c2}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:${KERN:-k_local} -s ${SKIP:-0} -c 1 \
     -o gpurun_out/${TAG:-loc}_$CFG -f python scripts/prof_one.py $CFG 1 > gpurun_out/${TAG:-loc}_ncu_$CFG.log 2>&1
  ncu -i gpurun_out/${TAG:-loc}_$CFG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG:-loc}_${CFG}_sass.csv 2>&1
done
