"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes) for the last sort."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
k = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0][:40]), {})[d["Metric Name"]] = d["Metric Value"].replace(",", "")
items = list(k.items())[-last:]
tot = 0.0
for (i, name), m in items:
    t = float(m.get("gpu__time_duration.sum", 0)) / 1e3
    rd = float(m.get("dram__bytes_read.sum", 0)); wr = float(m.get("dram__bytes_write.sum", 0))
    unit_t = "us"
    tot += t
    print(f"{i:4d} {name:40s} {t:9.1f} us  R {rd/1e9:7.3f} GB  W {wr/1e9:7.3f} GB  {((rd+wr)/1e3/t if t else 0):7.0f} GB/s")
print(f"total {tot:.1f} us")
