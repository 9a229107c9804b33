"""Distribution of raduls_gpu_sort_host times (pageable), with and without
the device-budget query (RADULS_GPU_DEVICE_BUDGET set)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1612_02557_b200 as rg
from paper_1612_02557_b200 import _lib
L = _lib.load()
n, rs, ks = 1 << 26, 16, 8
src = rg.generate(n, rg.RecordLayout(rs, ks), seed=0x5EED0001).cpu().numpy()
page = np.empty_like(src)
for label in ("budget query", "budget env"):
    if label == "budget env":
        os.environ["RADULS_GPU_DEVICE_BUDGET"] = str(170 << 30)
    for fn in ("raduls_gpu_sort_host", "raduls_gpu_lsd_sort_host"):
        ts = []
        for _ in range(10):
            page[:] = src
            t0 = time.perf_counter()
            assert getattr(L, fn)(page.ctypes.data, None, n, rs, ks) == 0
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{label:12s} {fn:26s} " + " ".join(f"{t:6.1f}" for t in ts))
