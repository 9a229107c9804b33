"""Time raduls_gpu_sort_host vs raduls_gpu_lsd_sort_host on the same buffer
(pageable and pinned), to locate host-path overheads."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_02557_b200 as rg
from paper_1612_02557_b200 import _lib
L = _lib.load()
n, rs, ks = 1 << 26, 16, 8
src = rg.generate(n, rg.RecordLayout(rs, ks), seed=0x5EED0001).cpu().numpy()
page = np.empty_like(src)
pin = torch.empty(src.size, dtype=torch.uint8, pin_memory=True).numpy()
for name, buf in [("pageable", page), ("pinned", pin)]:
    for fn in ("raduls_gpu_sort_host", "raduls_gpu_lsd_sort_host"):
        ts = []
        for _ in range(4):
            buf[:] = src
            t0 = time.perf_counter()
            rc = getattr(L, fn)(buf.ctypes.data, None, n, rs, ks)
            ts.append(time.perf_counter() - t0)
            assert rc == 0
        print(f"{name:9s} {fn:26s} " + " ".join(f"{1e3*t:7.1f}" for t in ts) + " ms")
