#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_lsd.py tests/test_records_harness.py -k "host or out_of_core or frees or dropin or harness or lsd" > gpurun_out/r2_p12_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2_p12_pytest.log
RADULS_GPU_HOST_TIMING=1 timeout 600 python -c "
import time, torch, numpy as np, paper_1612_02557_b200 as rg
n=1<<32; lay=rg.RecordLayout(16,8)
host=torch.empty(n*16,dtype=torch.uint8,pin_memory=True)
for c in range(0,n,1<<28):
    host[c*16:(c+(1<<28))*16].copy_(rg.generate(1<<28,lay,seed=0x5EED0005,index_base=c,device='cuda'))
torch.cuda.synchronize(); torch.cuda.empty_cache()
for cache in (False, False, False, True, True):
    rg.set_host_cache(cache)
    t=time.perf_counter(); rg.sort(host.numpy(), n, lay); print('cache',cache, time.perf_counter()-t, flush=True)
" > gpurun_out/r2_probe_host_timing_vmm.txt 2>&1
