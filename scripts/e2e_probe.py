import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1612_02557_b200 as rg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
from scripts.perf_probe import CONFIGS
n, rs, ks, dist, seed = CONFIGS[cfg]
lay = rg.RecordLayout(rs, ks)
host = torch.empty(n * rs, dtype=torch.uint8, pin_memory=True)
chunk = (4 << 30) // rs
out = {}
for mode in ("prog", "noprog", "prog"):
    os.environ["RADULS_GPU_PROGRESSIVE_BYTES"] = "0" if mode == "prog" else str(1 << 62)
    ts = []
    for rep in range(3):
        for c0 in range(0, n, chunk):
            cn = min(chunk, n - c0)
            g = rg.generate(cn, lay, dist=dist, seed=seed, index_base=c0)
            host[c0 * rs:(c0 + cn) * rs].copy_(g); del g
        torch.cuda.synchronize(); torch.cuda.empty_cache()
        t0 = time.perf_counter()
        rg.sort(host.numpy(), n, lay)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"cfg": cfg, "mode": mode, "s": [round(t, 4) for t in ts], "stats": rg.last_stats()}), flush=True)
