"""Basic-block summary of an ncu sass CSV: instruction share and stall-sample share per block."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
blocks = []
for r in data:
    c = int(r[idx['Instructions Executed']] or 0); a = r[idx['Address']]; src = r[idx['Source']]
    smp = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    op = src.split()[0] if src else ''
    if op.startswith('@'):
        op = src.split()[1] if len(src.split()) > 1 else op
    if blocks and blocks[-1][0] == c:
        blocks[-1][1] += 1; blocks[-1][3].append(op); blocks[-1][4] += smp
    else:
        blocks.append([c, 1, a, [op], smp])
tot = sum(b[0] * b[1] for b in blocks); stot = sum(b[4] for b in blocks) or 1
print(f"total warp instr {tot}  per unit {tot/div:.0f}")
big = sorted(blocks, key=lambda b: -(b[4] + b[0] * b[1] * stot / tot))[:top]
for b in sorted(big, key=lambda b: int(b[2], 16)):
    print(f"{b[2][-5:]} cnt={b[0]/div:9.1f} len={b[1]:>3} instr={b[0]*b[1]/tot*100:5.1f}% stall={b[4]/stot*100:5.1f}%  {' '.join(b[3][:14])}")
