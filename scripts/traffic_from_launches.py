"""DRAM bytes per launch of each bench kernel class, from an ncu launch list
of the bench command (gpu__time_duration + dram__bytes_read/write), for
bench.py's roofline.traffic:

    python scripts/traffic_from_launches.py profiles/r2_launches_bench_c5.csv > profiles/ncu_traffic_c5.json

The whole list (warm-up and timed sorts) is averaged per kernel class."""
import collections
import csv
import json
import sys

CLASS = {"k_scatter": "scatter", "k_local": "local_sort", "k_local_bm": "local_sort", "k_local_bm8": "local_sort",
         "k_local_bm_med": "local_sort_handover", "k_local_list": "local_sort_handover",
         "k_tile_hist": "tile_hist",
         "k_tile_hist_nd": "tile_hist", "k_tile_hist_reg": "tile_hist", "k_tile_scan": "tile_scan",
         "k_plan": "plan", "k_copy_back": "copy_back"}
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].replace("<unnamed>::", "").split("(")[0].split("<")[0].replace("void ", "")
        name = name.split("::")[-1]
        per.setdefault(int(d["ID"]), {"name": name})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for v in per.values():
    c = CLASS.get(v["name"])
    if c:
        tot[c] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        cnt[c] += 1
out = {c: tot[c] / cnt[c] for c in tot}
out["_source"] = f"{sys.argv[1]}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum per launch, averaged per class"
print(json.dumps(out, indent=1))
