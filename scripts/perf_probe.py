"""Developer probe: time the device sort on the BASELINE configs (no parity).

    python scripts/perf_probe.py [c1 c2 c3 c4 c5] [--reps 3]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1612_02557_b200 as rg  # noqa: E402

CONFIGS = {
    "c1": (1 << 26, 16, 8, 0, 0x5EED0001),
    "c2": (1 << 30, 8, 8, 0, 0x5EED0002),
    "c3": (1 << 29, 16, 8, 1, 0x5EED0003),
    "c4": (1 << 28, 32, 24, 0, 0x5EED0004),
    "c5": (1 << 32, 16, 8, 0, 0x5EED0005),
    # not a BASELINE config: 24-B records (a reference layout) for shape A/Bs
    "x24": (1 << 28, 24, 16, 0, 0x5EED0024),
    "x32": (1 << 26, 32, 24, 0, 0x5EED0032),
}


def main():
    names = [a for a in sys.argv[1:] if a in CONFIGS] or ["c1", "c2", "c3", "c4"]
    reps = 3
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    for name in names:
        n, rs, ks, dist, seed = CONFIGS[name]
        lay = rg.RecordLayout(rs, ks)
        data = torch.empty(n * rs, dtype=torch.uint8, device="cuda")
        tmp = torch.empty_like(data)
        times = []
        for r in range(reps + 1):
            rg.generate(n, lay, dist=dist, seed=seed, out=data)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            rg.sort(data, n, lay, tmp=tmp)
            e1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            if r:
                times.append((e0.elapsed_time(e1), wall * 1e3))
        st = rg.last_stats()
        v, _ = rg.check_sorted(data, n, lay)
        ms = sorted(t[0] for t in times)[len(times) // 2]
        print(json.dumps({"config": name, "n": n, "rs": rs, "ks": ks, "ms_event_median": ms,
                          "ms_wall": [round(t[1], 3) for t in times],
                          "Grec_s": n / ms / 1e6, "violations": v, "stats": st}), flush=True)
        del data, tmp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
