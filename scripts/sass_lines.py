"""SASS instructions per source line for one kernel of the built library
(nvdisasm -g line info). Static count by default; with an ncu source CSV
(`ncu -i X --page source --csv --print-source sass`) of the same build, the
executed warp-instructions and sampled stalls per line instead.

Usage: sass_lines.py <kernel-substring> [top] [ncu_sass.csv]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ncu_csv = sys.argv[3] if len(sys.argv) > 3 else None
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all",
                    os.path.join(ROOT, "paper_1612_02557_b200", "libraduls_gpu.so")],
                   cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], check=True,
                         capture_output=True, text=True).stdout
line_of = {}  # offset -> (file, line)
inside = False
cur = None
for line in txt.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        if inside:
            break
        inside = pat in m.group(1)
        if inside:
            print("function", m.group(1))
        continue
    if not inside:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if m:
        line_of[int(m.group(1), 16)] = cur

cnt = collections.Counter()
stall = collections.Counter()
if ncu_csv:
    rows = list(csv.reader(open(ncu_csv)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    base = min(int(r[ix["Address"]], 16) for r in data)
    sc = ix.get("Warp Stall Sampling (All Samples)")
    if len(data) != len(line_of):
        print(f"warning: {len(data)} ncu rows vs {len(line_of)} disassembled instructions")
    for r in data:
        k = line_of.get(int(r[ix["Address"]], 16) - base)
        cnt[k] += int(r[ix["Instructions Executed"]] or 0)
        if sc is not None:
            stall[k] += int(r[sc] or 0)
else:
    for k in line_of.values():
        cnt[k] += 1
tot = sum(cnt.values()) or 1
stot = sum(stall.values()) or 1
print("total", tot, "stall samples", sum(stall.values()))
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:12d} {100 * v / tot:5.1f}%  stall {100 * stall[k] / stot:5.1f}%  {k[0]}:{k[1]}"
          if k else f"{v:12d} ?")
