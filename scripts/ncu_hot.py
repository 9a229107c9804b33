"""Summarise an ncu --page source --print-source=sass CSV: stall totals and hottest instructions.
    ncu -i rep --page source --csv --print-source=sass > x.csv; python scripts/ncu_hot.py x.csv [N]
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0 for h in stall_cols}
samples = []
for r in data:
    if len(r) != len(hdr):
        continue
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    for h in stall_cols:
        tot[h] += int(r[idx[h]] or 0)
    samples.append((s, r[idx["Address"]], r[idx["Source"]], {h: int(r[idx[h]] or 0) for h in stall_cols}))
T = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{h[6:]}={v*100/T:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
samples_sorted = sorted(samples, key=lambda x: -x[0])
for s, a, src, st in samples_sorted[:top]:
    main = ",".join(f"{h[6:]}:{v}" for h, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{s:6d} {a:>6} {src[:70]:70s} {main}")
