"""Host drop-in timing: raduls_gpu_sort_host on pageable vs pinned buffers,
plus raw H2D/D2H copy bandwidth (torch), to size the host-path pipeline."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_02557_b200 as rg

out = {}
for log2n in [int(x) for x in (sys.argv[1:] or ["26", "29"])]:
    n, rs, ks = 1 << log2n, 16, 8
    lay = rg.RecordLayout(rs, ks)
    src = rg.generate(n, lay, seed=0x5EED0001).cpu().numpy()
    pageable = np.empty_like(src)
    pinned_t = torch.empty(src.size, dtype=torch.uint8, pin_memory=True)
    pinned = pinned_t.numpy()
    res = {}
    for name, buf in [("pageable", pageable), ("pinned", pinned)]:
        ts = []
        for _ in range(3):
            buf[:] = src
            t0 = time.perf_counter()
            rg.sort(buf, n, lay)
            ts.append(time.perf_counter() - t0)
        res[f"sort_host_{name}_s"] = min(ts)
        res[f"sort_host_{name}_Grec_s"] = n / min(ts) / 1e9
    dev = torch.empty(src.size, dtype=torch.uint8, device="cuda")
    for name, t in [("pageable", torch.from_numpy(pageable)), ("pinned", pinned_t)]:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(t)
        torch.cuda.synchronize()
        h2d = time.perf_counter() - t0
        t0 = time.perf_counter()
        t.copy_(dev)
        torch.cuda.synchronize()
        d2h = time.perf_counter() - t0
        res[f"h2d_{name}_GBs"] = src.size / h2d / 1e9
        res[f"d2h_{name}_GBs"] = src.size / d2h / 1e9
    out[f"2^{log2n}x16"] = res
print(json.dumps(out, indent=1))
