"""Per-kernel SASS census of the built library (cuobjdump -sass): how many
instructions of each class every kernel holds — the static evidence of the
B200 features used (UBLKCP = cp.async.bulk TMA copies, UBLKPF = bulk L2
prefetch, SYNCS = mbarrier ops, REDUX = warp reductions, ATOMS = shared-memory
atomics, MATCH, LDGSTS = cp.async) and that no tensor-core instructions exist
(no dense contraction on this path).

    python scripts/sass_census.py [lib] > profiles/r2_sass_census.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1612_02557_b200", "libraduls_gpu.so")
CLASSES = ["UBLKCP", "UBLKPF", "SYNCS", "REDUX", "ATOMS", "ATOMG", "RED", "MATCH", "LDGSTS", "LDS", "STS",
           "LDG", "STG", "BAR", "VOTE", "SHFL", "PRMT", "UTCHMMA", "UTCMMA", "LDTM", "STTM", "UTMALDG"]
txt = subprocess.run(["cuobjdump", "-sass", lib], check=True, capture_output=True, text=True).stdout
kern = None
counts = collections.OrderedDict()
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and kern:
        op = m.group(1)
        counts[kern]["total"] += 1
        for c in CLASSES:
            if op == c or (c in ("LDS", "STS", "LDG", "STG", "BAR", "SHFL") and op == c):
                counts[kern][c] += 1


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


names = list(counts)
pretty = demangle(names)
print(f"# SASS census of {os.path.relpath(lib, ROOT)} (sm_100a), instructions per kernel")
print("# columns: total " + " ".join(CLASSES))
tot = collections.Counter()
for raw, nm in sorted(zip(names, pretty), key=lambda x: x[1]):
    c = counts[raw]
    tot.update(c)
    short = re.sub(r"\(.*", "", nm.replace("(anonymous namespace)::", ""))
    print(f"{short:60s} {c['total']:6d} " + " ".join(f"{c[k]:5d}" for k in CLASSES))
print(f"{'ALL':60s} {tot['total']:6d} " + " ".join(f"{tot[k]:5d}" for k in CLASSES))
