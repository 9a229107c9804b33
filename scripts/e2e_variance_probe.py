import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
import paper_1612_02557_b200 as rg
from scripts.perf_probe import CONFIGS
n, rs, ks, dist, seed = CONFIGS["c5"]
lay = rg.RecordLayout(rs, ks)
host = torch.empty(n * rs, dtype=torch.uint8, pin_memory=True)
chunk = (4 << 30) // rs
L = rg._lib.load()
for cached in (0, 1, 0):
    L.raduls_gpu_set_host_cache(cached)
    ts = []
    for rep in range(5):
        for c0 in range(0, n, chunk):
            cn = min(chunk, n - c0)
            g = rg.generate(cn, lay, dist=dist, seed=seed, index_base=c0)
            host[c0 * rs:(c0 + cn) * rs].copy_(g); del g
        torch.cuda.synchronize(); torch.cuda.empty_cache()
        t0 = time.perf_counter()
        rg.sort(host.numpy(), n, lay)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"cached": cached, "s": [round(t, 4) for t in ts]}), flush=True)
L.raduls_gpu_set_host_cache(0)
