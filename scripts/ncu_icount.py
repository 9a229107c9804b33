"""Top SASS instructions by executed count from an ncu source CSV (sass view)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
ie = idx["Instructions Executed"]
tot = sum(int(r[ie] or 0) for r in data)
print("total warp-instructions executed:", tot)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
# group consecutive addresses into blocks of similar counts
for r in sorted(data, key=lambda r: -int(r[ie] or 0))[:top]:
    print(f"{int(r[ie] or 0):10d} {r[idx['Address']]:>8} {r[idx['Source']][:90]}")
