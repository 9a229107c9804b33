"""Turn the files scripts/gpu_evidence.sh leaves in gpurun_out/ (ev_*) into the
tracked evidence files under profiles/ (the `_v2` set of round 2):

    python scripts/process_evidence.py
"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def run(*cmd):
    return subprocess.run([sys.executable, *cmd], cwd=ROOT, capture_output=True, text=True, check=True).stdout


def main():
    shutil.copy(os.path.join(G, "ev_bench_c5.json"), os.path.join(P, "r2_bench_c5_v2.json"))
    shutil.copy(os.path.join(G, "ev_bench_ref.json"), os.path.join(P, "r2_bench_ref_c5_v2.json"))
    shutil.copy(os.path.join(G, "ev_launches_bench_c5.csv"), os.path.join(P, "r2_launches_bench_c5_v2.csv"))
    if os.path.exists(os.path.join(G, "ev_sass_census.txt")):
        shutil.copy(os.path.join(G, "ev_sass_census.txt"), os.path.join(P, "r2_sass_census_v2.txt"))
    rel = "profiles/r2_launches_bench_c5_v2.csv"
    open(os.path.join(P, "r2_launch_shares_c5_v2.json"), "w").write(run("scripts/launch_shares.py", rel, rel))
    open(os.path.join(P, "ncu_traffic_c5.json"), "w").write(run("scripts/traffic_from_launches.py", rel))
    caps = [("local_c1", "k_local_bm<16> on C1 (2^26 x 16 B; 65536 groups of ~1024 records), second sort of scripts/prof_one.py c1 2"),
            ("scatter_c1", "k_scatter<16> on C1, second launch of the second sort"),
            ("local_c2", "k_local_bm8 on C2 (2^30 x 8 B; 65536 groups of ~16384 records)"),
            ("local_c4", "k_local_bm<32> on C4 (2^28 x 32 B; 65536 groups of ~4096 records)")]
    out = {}
    for name, desc in caps:
        f = os.path.join(G, f"ev_full_{name}_raw.csv")
        if os.path.exists(f):
            out[name] = json.loads(run("scripts/ncu_metrics.py", f, desc))
    json.dump(out, open(os.path.join(P, "r2_ncu_full_metrics_v2.json"), "w"), indent=1)
    # local-sort phases from the per-line counts (scripts/sass_lines.py output of the same build)
    lines_f = os.path.join(G, "ev_local_c1_lines.txt")
    if os.path.exists(lines_f):
        src = open(os.path.join(ROOT, "paper_1612_02557_b200", "csrc", "k_local_bm.cuh")).read().splitlines()
        def find(pat, start=0):
            return next(i + 1 for i, l in enumerate(src) if i >= start and pat in l)
        f0 = find("void local_group_bm(")
        marks = [("load+init", f0), ("windows+cells", find("---- 2./3. windows", f0)),
                 ("scan call", find("---- 4. scan", f0)), ("rank (clean words)", find("---- 5. clean words", f0)),
                 ("dirty-word pass", find("---- 6. dirty words", f0)),
                 ("kernel wrappers, 8-B kernel", find("// Bitmap local sort launch", f0))]
        scan0, scan1 = find("void bm_scan("), find("// Whether groups larger")
        agg, st, tot = {}, {}, 0
        for l in open(lines_f):
            m = re.match(r"\s*(\d+)\s+([\d.]+)%\s+stall\s+([\d.]+)%\s+(\S+):(\d+)", l)
            if not m:
                continue
            c, s, f, ln = int(m.group(1)), float(m.group(3)), m.group(4), int(m.group(5))
            tot += c
            if f == "k_local_bm.cuh":
                if scan0 <= ln < scan1:
                    k = "bm_scan"
                elif ln < f0:
                    k = "other k_local_bm.cuh"
                else:
                    k = [n for n, a in marks if a <= ln][-1]
            else:
                k = f
            agg[k] = agg.get(k, 0) + c
            st[k] = st.get(k, 0) + s
        n = 1 << 26
        rows = ["## k_local_bm<16> on C1 (final code): executed warp-instructions per record by phase",
                "## (ncu source counters of profiles/r2_ncu_full_metrics_v2.json local_c1 mapped to source lines by",
                "##  scripts/sass_lines.py; header files are the inlined record loads/stores, window permutes,",
                "##  atomics and warp reductions)"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1]):
            rows.append(f"{k:30s} {100 * v / tot:5.1f}% instr {st[k]:5.1f}% stall  {v / n:6.2f} warp-instr/rec")
        rows.append(f"total warp-instr/rec {tot / n:.2f} (bucket sort k_local<16>: 8.2)")
        open(os.path.join(P, "r2_local_sort_phases_v2.txt"), "w").write("\n".join(rows) + "\n")
    d = json.load(open(os.path.join(P, "r2_bench_c5_v2.json")))
    print("C5", round(d["ms_per_step"], 2), "ms", round(d["value"] / 1e9, 2), "G rec/s; scatter frac",
          d["roofline"]["frac"], "sort frac", d["roofline_sort"]["frac"], "e2e", round(d["e2e"]["value"] / 1e9, 3))
    print({k: round(x["ms"] / d["steps"], 2) for k, x in d["kernels"].items()})
    for c, v in d["per_config"].items():
        print(c, round(v["ms_per_step"], 3), round(v["value"] / 1e9, 2), v["roofline"]["kernel"], v["roofline"]["frac"],
              v["roofline_sort"]["frac"],
              {k: round(x["ms"] / v["steps"], 3) for k, x in v["kernels"].items() if x["ms"] > 0.05})
    r = json.load(open(os.path.join(P, "r2_bench_ref_c5_v2.json")))
    print("reference", round(r["value"] / 1e9, 4), "G rec/s", round(r["ms_per_step"]), "ms")
    for k, v in out.items():
        print(k, v.get("gpu__time_duration.sum"), "inst", v.get("smsp__inst_executed.sum"), "issue",
              v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"), "regs",
              v.get("launch__registers_per_thread"))


if __name__ == "__main__":
    main()
