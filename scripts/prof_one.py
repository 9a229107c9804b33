"""Run warmup sorts then one sort of a config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_02557_b200 as rg
from scripts.perf_probe import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, rs, ks, dist, seed = CONFIGS[name]
lay = rg.RecordLayout(rs, ks)
data = torch.empty(n * rs, dtype=torch.uint8, device="cuda")
tmp = torch.empty_like(data)
for r in range(reps):
    rg.generate(n, lay, dist=dist, seed=seed, out=data)
    rg.sort(data, n, lay, tmp=tmp)
torch.cuda.synchronize()
print(rg.last_stats())
