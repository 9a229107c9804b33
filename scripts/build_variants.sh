#!/bin/bash
# build libraduls_gpu.so variants into var/lib_<tag>.so: build_variants.sh tag "-DX=1 -DY=2" ...
cd "$(dirname "$0")/.."
mkdir -p var
while [ $# -ge 2 ]; do
  tag=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
    -shared -cudart static -I include $defs -o var/lib_$tag.so paper_1612_02557_b200/csrc/raduls_gpu.cu &
done
wait
ls -la var/
