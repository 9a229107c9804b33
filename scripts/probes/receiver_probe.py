"""Probe: the multi-GPU receiver's local sort at N ranks, emulated on one GPU.
A rank of an N-GPU C5 sort receives 2^32/N records from 1/N of the key space
(here: key byte 0 reduced to 256/N values). (A) raduls_gpu_sort of the range
(the receiver before this round); (B) the range already split by key byte 0
(what the digit-major exchange delivers) sorted with raduls_gpu_sort_segments
from byte 1. CUDA events, median of 5 after 2 warm-ups; both verified.

    python scripts/probes/receiver_probe.py [N ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_02557_b200 as rg  # noqa: E402
from paper_1612_02557_b200.distributed import DeviceOps  # noqa: E402

lay = rg.RecordLayout(16, 8)
ops = DeviceOps()
for N in [int(x) for x in sys.argv[1:]] or [8, 4, 2]:
    n = (1 << 32) // N
    src = torch.empty(n * 16, dtype=torch.uint8, device="cuda")
    rg.generate(n, lay, seed=0x5EED0005, out=src)
    v = src.view(n, 16)
    v[:, 0] = v[:, 0] // N  # this rank's share of key byte 0
    part = torch.empty_like(src)
    counts = rg.split(src, part, n, 16, 0)
    data = torch.empty_like(src)
    tmp = torch.empty_like(src)
    st = torch.cuda.current_stream()
    res = {}
    for mode in ("whole", "segments"):
        ts = []
        for it in range(7):
            data.copy_(src if mode == "whole" else part)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if mode == "whole":
                rg.sort(data, n, lay, tmp=tmp, stream=st)
            else:
                ops.sort_segments(data, n, lay, [int(c) for c in counts], [1] * 256, tmp)
            e1.record(st)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        assert rg.check_sorted(data, n, lay)[0] == 0
        res[mode] = (sorted(ts)[len(ts) // 2], rg.last_stats()["scatter_records"] / n)
    print(f"N={N}: n={n} whole {res['whole'][0]:.2f} ms ({res['whole'][1]:.2f} scatter passes), "
          f"pre-split segments {res['segments'][0]:.2f} ms ({res['segments'][1]:.2f} scatter passes)", flush=True)
    del src, part, data, tmp
    torch.cuda.empty_cache()
