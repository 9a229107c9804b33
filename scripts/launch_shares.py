"""Per-kernel shares of the last sort in an ncu launch-list CSV of bench.py
(gpu__time_duration + dram bytes): python scripts/launch_shares.py launches.csv src_name > shares.json

The last sort = the launches from the last k_sample_andor up to the check
kernels (k_check_sorted / k_digest), which bench.py runs after the timed steps."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
src = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
hdr = None
k = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k.setdefault((int(d["ID"]), d["Kernel Name"].replace("<unnamed>::", "").split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]), {})[
            d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
items = list(k.items())
start = max(i for i, ((_, n), _) in enumerate(items) if n == "k_sample_andor")
end = next((i for i in range(start, len(items)) if items[i][0][1] in ("k_check_sorted", "k_digest")), len(items))
ms = collections.OrderedDict()
traffic = collections.defaultdict(float)
launches = collections.Counter()
for (_, name), m in items[start:end]:
    ms[name] = ms.get(name, 0.0) + m.get("gpu__time_duration.sum", 0) / 1e6
    traffic[name] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    launches[name] += 1
tot = sum(ms.values())
print(json.dumps({
    "sort_ms_ncu": round(tot, 3),
    "share": {n: round(v / tot, 4) for n, v in ms.items()},
    "ms": {n: round(v, 3) for n, v in ms.items()},
    "launches": dict(launches),
    "traffic_bytes_per_launch": {n: traffic[n] / launches[n] for n in ms},
    "source": f"{src}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              "--clock-control none, bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "
              "(last timed sort; cold-cache serialised launches)",
}, indent=1))
