#!/bin/bash
# per-kernel times of each var/lib_<tag>.so on the configs in KT_CONFIGS
mkdir -p gpurun_out
for lib in var/lib_*.so; do
  tag=$(basename $lib .so); tag=${tag#lib_}
  cp $lib paper_1612_02557_b200/libraduls_gpu.so
  for c in ${KT_CONFIGS:-c5}; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_${tag}_$c.json 2> gpurun_out/var_${tag}_$c.err
    python -c "import json;d=json.load(open('gpurun_out/var_${tag}_$c.json'));k=d['kernels'];print('$tag','$c',round(d['ms_per_step'],3),{n:(v['ms'],v['GBps']) for n,v in k.items() if v['ms']>1})"
  done
done
