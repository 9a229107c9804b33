"""Per-kernel GB/s of the sort vs input size (16-B records, uniform keys)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_02557_b200 as rg
rs, ks = 16, 8
lay = rg.RecordLayout(rs, ks)
for lg in [int(x) for x in (sys.argv[1:] or ["26", "28", "30", "31", "32"])]:
    n = 1 << lg
    data = torch.empty(n * rs, dtype=torch.uint8, device="cuda")
    tmp = torch.empty_like(data)
    for rep in range(2):
        rg.generate(n, lay, seed=7, out=data)
        torch.cuda.synchronize()
        rg.set_profiling(rep == 1)
        rg.sort(data, n, lay, tmp=tmp)
        torch.cuda.synchronize()
    kt = rg.last_kernel_times()
    st = rg.last_stats()
    rg.set_profiling(False)
    out = {"log2n": lg}
    for k, (l, ms) in kt.items():
        b = {"scatter": 2 * rs * st["scatter_records"], "local_sort": 2 * rs * st["local_records"],
             "tile_hist": rs * st["hist_records"]}.get(k)
        out[k] = (l, round(ms, 3), round(b / ms / 1e6, 0) if b else None)
    print(json.dumps(out), flush=True)
    del data, tmp
    torch.cuda.empty_cache()
