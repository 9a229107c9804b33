"""Summarise perf_probe logs: python scripts/perf_show.py gpurun_out/perf_a.log [...]"""
import json
import sys

for path in sys.argv[1:]:
    print("==", path)
    for line in open(path):
        if line.startswith("{"):
            d = json.loads(line)
            st = d["stats"]
            print(f"  {d['config']}: {d['ms_event_median']:.2f} ms  {d['Grec_s']:.2f} G rec/s  viol={d['violations']}"
                  f"  levels={st['levels']} hist={st['hist_records']} digit={st.get('hist_digit_records')}")
        elif line.strip():
            print("  " + line.strip()[:200])
