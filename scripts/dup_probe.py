"""Developer probe: cost of the bitmap local sort's hand-over on duplicate-heavy
keys (every group goes bitmap sort -> bucket sort): the default chain vs
RADULS_GPU_LOCAL=bucket on 2^26 16-B records whose keys are drawn from
`universe` distinct values.

    python scripts/dup_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_02557_b200 as rg  # noqa: E402


def main():
    n, rs, ks = 1 << 26, 16, 8
    lay = rg.RecordLayout(rs, ks)
    rg.set_profiling(True)
    for universe in (0, 1 << 26, 1 << 24, 1 << 22, 1 << 20):
        base = rg.generate(n, lay, seed=0xD0B)
        if universe:
            # keys <- keys of a random record among the first `universe`
            g = torch.Generator(device="cuda").manual_seed(1)
            idx = torch.randint(0, universe, (n,), device="cuda", generator=g)
            recs = base.view(n, rs)
            recs[:, :ks] = recs[idx, :ks]
            del idx
        out = {"universe": universe}
        for mode in ("bitmap", "bucket"):
            if mode == "bucket":
                os.environ["RADULS_GPU_LOCAL"] = "bucket"
            else:
                os.environ.pop("RADULS_GPU_LOCAL", None)
            ts, loc = [], []
            for r in range(4):
                d = base.clone()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rg.sort(d, n, lay)
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
                    loc.append(rg.last_kernel_times().get("local_sort", (0, 0.0))[1])
            st = rg.last_stats()
            v, _ = rg.check_sorted(d, n, lay)
            out[mode] = {"ms": round(sorted(ts)[1], 3), "local_ms": round(sorted(loc)[1], 3),
                         "bitmap_spill_groups": st["bitmap_spill_groups"],
                         "fallback_groups": st["fallback_groups"], "violations": v}
        os.environ.pop("RADULS_GPU_LOCAL", None)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
