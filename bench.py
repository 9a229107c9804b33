#!/usr/bin/env python
"""bench.py — sorted records/sec of the B200 MSD record sort (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
    python bench.py --impl reference ...      # the reference CPU sorter arm

A "step" is one complete sort of one batch: at N=1 the whole workload
(default C5: 2^32 records of 16 B, the paper's headline scale, BASELINE.json
configs[4]) through libraduls_gpu.so; at N>1 (torchrun, one rank per GPU) the
same total partitioned across ranks by key range (strong scaling) and
exchanged once (paper_1612_02557_b200/distributed.py), timed with both
exchanges — the partition kernel storing straight into peer windows over
NVLink ("p2p") and a local partition plus an NCCL all-to-all ("nccl") — the
faster one headlined, both reported with their NVLink fraction.

Timing: inputs are regenerated on the device before every step (untimed:
the sort is in place); the timed region is the sort call only, bracketed
by a barrier and torch.cuda.synchronize(), CUDA events on the sort's stream,
max over ranks. Inputs (1-64 GiB) exceed the 126 MB L2, so no flush is
needed. Per-kernel CUDA-event times of the timed steps give the live
roofline of the dominant kernel; `e2e` repeats the measurement through the
host-memory drop-in (pinned host buffer, H2D + sort + D2H inside the timed
region); `cpu_baseline` times the reference CPU sorter (oracle/_ref, the
unmodified reference library compiled here) on a bounded sample on the
box's host cores (the whole config when host RAM holds it); per_config
adds C1-C4 measured in the same run.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = 1 << 30
# name -> (n_records, rec_size, key_size, dist, seed, description); SURVEY.md §8(d)
CONFIGS = {
    "c1": (1 << 26, 16, 8, 0, 0x5EED0001, "C1: 2^26 x 16 B, 8-B uniform key + 8-B payload index"),
    "c2": (1 << 30, 8, 8, 0, 0x5EED0002, "C2: 2^30 x 8 B, key-only uniform"),
    "c3": (1 << 29, 16, 8, 1, 0x5EED0003,
           "C3: 2^29 x 16 B, top 24 bits zero, Zipf(1.2) byte, 32 uniform bits"),
    "c4": (1 << 28, 32, 24, 0, 0x5EED0004, "C4: 2^28 x 32 B, 24-B uniform key + 8-B payload"),
    "c5": (1 << 32, 16, 8, 0, 0x5EED0005, "C5: 2^32 x 16 B, 8-B uniform key + 8-B payload index"),
}
METRIC = "sorted records/sec"
UNIT = "records/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, window: tuple[float, float] | None = None) -> dict | None:
        """Summarise the samples taken inside `window` (time.time() bounds of
        the timed region; the sampler is started earlier so nvidia-smi's
        start-up does not eat the region). All samples if none fall inside."""
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        inside = [r for r in rows if window and window[0] <= r[0] <= window[1]]
        sel = inside or rows
        if not sel:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = {nm for r in sel for nm, v in zip(names, r[3]) if v.lower() == "active"}
        return {"sm_mhz": statistics.median(r[1] for r in sel), "sm_max_mhz": max(r[2] for r in sel),
                "reasons": sorted(reasons), "samples": len(sel),
                "in_timed_region": bool(inside)}


# ------------------------------------------------------------------ CPU baseline / reference arm

def mem_available() -> int:
    """MemAvailable of this host in bytes (0 if unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def _host_chunks(n: int, threads: int):
    step = max(1, -(-n // max(1, threads)))
    return [(a, min(n, a + step)) for a in range(0, n, step)]


def host_generate(out, n: int, rs: int, ks: int, dist: int, seed: int, threads: int) -> None:
    """The §8(d) generator (oracle/liboracle.so, bit-identical to the device
    k_gen) into the numpy buffer `out`, chunked over host threads (ctypes
    releases the GIL). Input preparation only: never timed."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    L = oracle.lib()
    base = out.ctypes.data

    def one(ab):
        a, b = ab
        rc = L.orc_generate(C.cast(base + a * rs, oracle._u8p), b - a, rs, ks, dist, seed, a)
        if rc:
            raise ValueError(f"orc_generate rejected layout ({rs},{ks})")

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, _host_chunks(n, threads)))


def host_sorted(a, n: int, rs: int, ks: int, threads: int) -> bool:
    """Key order of n records, chunked over threads plus the chunk seams."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    L = oracle.lib()
    base = a.ctypes.data
    ch = _host_chunks(n, threads)

    def one(ab):
        x, y = ab
        v = C.c_uint64(0)
        return bool(L.orc_check_sorted(C.cast(base + x * rs, oracle._u8p), y - x, rs, ks, C.byref(v)))

    with ThreadPoolExecutor(threads) as ex:
        ok = all(ex.map(one, ch))
    for (_, y), (x2, _) in zip(ch, ch[1:]):  # seams
        if bytes(a[(y - 1) * rs:(y - 1) * rs + ks]) > bytes(a[x2 * rs:x2 * rs + ks]):
            ok = False
    return ok


def run_cpu_reference(cfg_name: str, n_cap: int, steps: int, warmup: int,
                      threads: int | None = None) -> dict:
    """The reference CPU sorter (oracle/_ref: the unmodified reference library
    compiled here; else the plain-C port at T=1) on the first min(n, n_cap)
    records of a config, `threads` host threads (default: the physical cores,
    counted as P/tests/acceptance.cpp:52-66 does). Input regenerated before
    every run (untimed), as P/src/bench.cpp:121-125 re-copies it."""
    import numpy as np

    import oracle
    n, rs, ks, dist, seed, _ = CONFIGS[cfg_name]
    n_s = min(n, n_cap)
    cores = oracle.host_cores()
    threads = threads or cores
    kind = "reference" if oracle.ref_available() else "port"
    proxy = ""
    rks = ks
    if kind == "reference" and ks not in (8, 16):
        rks = 16  # the reference rejects ks=24: (32,16) proxy, exact on these inputs
        proxy = f" (run as layout ({rs},16): the reference rejects key_size={ks})"
    work = np.empty(n_s * rs, dtype=np.uint8)
    times = []
    for i in range(warmup + steps):
        host_generate(work, n_s, rs, ks, dist, seed, cores)
        t0 = time.perf_counter()
        if kind == "reference":
            rc = oracle.ref().ref_sort(oracle._ptr(work), n_s, rs, rks, threads)
            if rc:
                raise RuntimeError(f"ref_sort rc={rc}")
        else:
            oracle.lib().orc_msd_sort(oracle._ptr(work), n_s, rs, ks, None)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    ok = host_sorted(work, n_s, rs, ks, cores)
    del work
    what = "all" if n_s == n else f"first {n_s}"
    return {"value": n_s * len(times) / sum(times), "unit": UNIT,
            "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": f"{what} records of the {cfg_name.upper()} generator{proxy}; {len(times)} runs, "
                      f"median {statistics.median(times)*1e3:.1f} ms; {threads} threads "
                      f"({cores} physical cores); sorted={ok}",
            "ms_per_step": 1e3 * sum(times) / len(times), "steps": len(times),
            "records": n_s, "same_config": n_s == n, "threads": threads}


def reference_cap(cfg_name: str) -> int:
    """The whole config when this host can hold it (data + the reference's own
    aux buffer + headroom), else a 2^28-record prefix."""
    n, rs = CONFIGS[cfg_name][0], CONFIGS[cfg_name][1]
    need = 2 * n * rs + (16 << 30)
    return n if mem_available() >= need else min(n, 1 << 28)


# ------------------------------------------------------------------ GPU arm

def algorithmic_bytes(stats: dict, rs: int) -> dict:
    """2*rs per record per executed pass (read + write);
    histogram-only reads are overhead (1*rs per record read whole, 1 byte per
    record read from the digit array, which the scatter before wrote)."""
    nd = stats.get("hist_digit_records", 0)
    return {
        "scatter": 2 * rs * stats.get("scatter_records", 0),
        "local_sort": 2 * rs * stats.get("local_records", 0),
        "copy_back": 2 * rs * stats.get("copy_records", 0),
        "tile_hist": rs * stats.get("hist_records", 0) + nd,
    }


def kernel_table(kt: dict, ab: dict) -> dict:
    return {k: {"launches": l, "ms": round(t, 3),
                "GBps": round(ab[k] / (t / 1e3) / 1e9, 1) if ab.get(k) and t else None}
            for k, (l, t) in kt.items()}


def ncu_traffic(cfg_name: str) -> dict:
    """DRAM bytes per launch per kernel class from the committed ncu launch list
    of this config's bench command (scripts/traffic_from_launches.py; the file
    is regenerated with every evidence run)."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg_name}.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def dominant(kt: dict, ab: dict, peak: float, peak_src: str, traffic: dict | None = None) -> dict | None:
    """Roofline of the kernel class with the most device time (live CUDA events)."""
    if not kt:
        return None
    dom = max(kt, key=lambda k: kt[k][1])
    dl, dt = kt[dom]
    db = ab.get(dom, 0)
    achieved = db / (dt / 1e3) / 1e9 if dt else 0.0
    tr = (traffic or {}).get(dom)
    return {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": tr,
            "traffic_source": (traffic or {}).get("_source") if tr else None,
            "algorithmic_bytes_per_launch": db / max(dl, 1), "launches": dl, "peak_source": peak_src}


def sort_roofline(ab: dict, total_ms: float, steps: int, peak: float, n: int, rs: int,
                  n_gpus: int = 1) -> dict:
    alg = ab.get("scatter", 0) + ab.get("local_sort", 0) + ab.get("copy_back", 0) + \
        ab.get("partition", 0) + ab.get("partition_exchange", 0)
    gbs = alg / (total_ms / 1e3) / 1e9
    return {"achieved": round(gbs, 1), "peak": peak * n_gpus, "unit": "GB/s",
            "frac": round(gbs / (peak * n_gpus), 4), "algorithmic_bytes_per_step": alg / steps,
            "passes_per_record": round(alg / steps / (2 * rs * n), 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-cap", type=int, default=0,
                    help="records of the reference run (0: the whole config when host RAM allows)")
    ap.add_argument("--exchange", default="both", choices=["both", "p2p", "nccl"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "gpu" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n_total, rs, ks, dist_kind, seed, desc = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return 0
        return reference_arm(args, n_total, rs, ks, desc)

    import torch

    import paper_1612_02557_b200 as rg
    # RADULS_BENCH_BACKEND=gloo + RADULS_BENCH_DEVICE=0: every rank on one shared
    # device (the -m gpu test of this N>1 path on a one-GPU box; ranks meet only
    # at host barriers, no kernel waits on another rank). Default: NCCL, GPU = local rank.
    backend = os.environ.get("RADULS_BENCH_BACKEND", "nccl")
    dev_index = int(os.environ.get("RADULS_BENCH_DEVICE", local_rank))
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    coll_dev = dev if backend == "nccl" else torch.device("cpu")
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lay = rg.RecordLayout(rs, ks)
    n_local = n_total // world
    base = rank * n_local
    if rank == world - 1:
        n_local = n_total - base
    peak, peak_src = load_peaks()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def gather(obj):
        if world == 1:
            return [obj]
        out = [None] * world
        torch.distributed.all_gather_object(out, obj)
        return out

    stream = torch.cuda.current_stream(dev)
    rg.set_profiling(False)

    def run_workload(cfg_name: str, exchanges, steps: int, warmup: int, clocks=None) -> dict:
        """One configuration, device-resident: per exchange (N>1) warm-up +
        timed steps, per-rank kernel times, exchange timings, launches, and
        the verification of the last step's output (untimed). Returns
        {exchange: summary} (+ "_regions": the timed regions)."""
        wn_total, wrs, wks, wdist, wseed, _ = CONFIGS[cfg_name]
        wlay = rg.RecordLayout(wrs, wks)
        wn_local = wn_total // world
        wbase = rank * wn_local
        if rank == world - 1:
            wn_local = wn_total - wbase
        data = torch.empty(wn_local * wrs, dtype=torch.uint8, device=dev)
        tmp = torch.empty_like(data) if world == 1 else None
        rg.generate(wn_local, wlay, dist=wdist, seed=wseed, index_base=wbase, out=data)
        digest_in = rg.digest(data, wn_local, wrs)

        def one_step(exchange, timings):
            rg.generate(wn_local, wlay, dist=wdist, seed=wseed, index_base=wbase, out=data)
            torch.cuda.synchronize(dev)
            barrier()
            torch.cuda.synchronize(dev)
            c0 = rg.launch_count()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if world == 1:
                rg.sort(data, wn_local, wlay, tmp=tmp, stream=stream)
                out, n_out = data, wn_local
            else:
                from paper_1612_02557_b200.distributed import sort_distributed
                out, n_out = sort_distributed(data, wn_local, wlay, timings=timings, exchange=exchange)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            return e0.elapsed_time(e1), out, n_out, rg.launch_count() - c0

        def measure(exchange):
            for _ in range(warmup):
                _, out, n_out, _ = one_step(exchange, {})
                del out
            rg.set_profiling(True)
            kt: dict = {}
            st: dict = {}
            xs = {"exchange_ms": 0.0, "partition_ms": 0.0, "sent_bytes": 0, "plan_s": 0.0}
            step_ms = []
            launches = 0
            t_region0 = time.time()
            for _ in range(steps):
                tim: dict = {}
                ms, out, n_out, nl = one_step(exchange, tim)
                launches += nl
                step_ms.append(max_over_ranks(ms))
                for k, (l, t) in rg.last_kernel_times().items():  # this rank's (local) sort
                    kt.setdefault(k, [0, 0.0])
                    kt[k][0] += l
                    kt[k][1] += t
                for k, v in rg.last_stats().items():
                    st[k] = st.get(k, 0) + v
                for k in ("exchange_ms", "partition_ms", "sent_bytes", "plan_s"):
                    if tim.get(k) is not None:
                        xs[k] += tim[k]
            t_region = (t_region0, time.time())
            rg.set_profiling(False)
            # verification (untimed): order, digest, and at N>1 the rank seams
            viol, _ = rg.check_sorted(out, n_out, wlay)
            d_out = rg.digest(out, n_out, wrs)
            first = bytes(out[:wks].cpu().numpy()) if n_out else None
            last = bytes(out[(n_out - 1) * wrs:(n_out - 1) * wrs + wks].cpu().numpy()) if n_out else None
            del out
            mine = {"viol": viol, "d_in": digest_in, "d_out": d_out, "n_out": n_out, "first": first,
                    "last": last, "kt": kt, "st": st, "xs": xs, "launches": launches, "n_local": wn_local}
            return step_ms, t_region, gather(mine)

        def verify(rows) -> dict:
            m = (1 << 128) - 1
            din = sum(r["d_in"][0] + (r["d_in"][1] << 64) for r in rows) & m
            dout = sum(r["d_out"][0] + (r["d_out"][1] << 64) for r in rows) & m
            seams = True
            prev = None
            for r in rows:
                if r["n_out"]:
                    if prev is not None and prev > r["first"]:
                        seams = False
                    prev = r["last"]
            tot = sum(r["n_out"] for r in rows)
            ok = all(r["viol"] == 0 for r in rows) and din == dout and seams and tot == wn_total
            return {"ok": ok, "inversions": sum(r["viol"] for r in rows), "digest_equal": din == dout,
                    "rank_seams_ordered": seams, "records_out": tot}

        def summarise(ex, step_ms, rows) -> dict:
            total_ms = sum(step_ms)
            ab_all: dict = {}
            per_rank = []
            worst = None
            for r in rows:
                ab = algorithmic_bytes(r["st"], wrs)
                kt = {k: tuple(v) for k, v in r["kt"].items()}
                if ex is not None:  # the partition pass of the exchange: one read + one write of n_local
                    cls = "partition_exchange" if ex == "p2p" else "partition"
                    ms_p = r["xs"]["exchange_ms"] if ex == "p2p" else r["xs"]["partition_ms"]
                    kt[cls] = (steps, ms_p)
                    ab[cls] = 2 * wrs * r["n_local"] * steps
                for k, v in ab.items():
                    ab_all[k] = ab_all.get(k, 0) + v
                roof = dominant(kt, ab, peak, peak_src, ncu_traffic(cfg_name) if world == 1 else None)
                per_rank.append({"kernel": roof["kernel"], "frac": roof["frac"]} if roof else None)
                if roof and (worst is None or roof["frac"] < worst[0]["frac"]):
                    worst = (roof, kt, ab)
            out = {"workload": CONFIGS[cfg_name][5],
                   "value": wn_total * steps / (total_ms / 1e3), "unit": UNIT,
                   "ms_per_step": total_ms / steps, "steps": steps, "verified": verify(rows),
                   "roofline": worst[0] if worst else None,
                   "roofline_sort": sort_roofline(ab_all, total_ms, steps, peak, wn_total, wrs, world),
                   "kernels": kernel_table(worst[1], worst[2]) if worst else None,
                   "gpu_launches": sum(r["launches"] for r in rows),
                   "stats_per_step": {k: v // steps for k, v in rows[0]["st"].items()} or None}
            if world > 1:
                out["roofline"]["per_rank_frac"] = [q["frac"] if q else None for q in per_rank]
                out["roofline"]["rank"] = "slowest rank (lowest frac)"
                sent = max(r["xs"]["sent_bytes"] for r in rows) / steps
                t_ex = max(r["xs"]["exchange_ms"] for r in rows) / steps
                gbs = sent / (t_ex / 1e3) / 1e9 if t_ex else None
                out["nvlink"] = {"exchange": ex, "sent_bytes_per_gpu": sent, "t_exchange_ms": round(t_ex, 3),
                                 "GBps": round(gbs, 1) if gbs else None, "peak": 900.0,
                                 "peak_source": "NVLink 5 per direction per GPU (nominal)",
                                 "frac": round(gbs / 900.0, 4) if gbs else None,
                                 "what": ("the fused partition+store kernel (reads local records, stores "
                                          "each destination's share into its window over NVLink)"
                                          if ex == "p2p" else "NCCL all_to_all_single"),
                                 "plan_ms": round(1e3 * max(r["xs"]["plan_s"] for r in rows) / steps, 3)}
            return out

        res = {}
        regions = []
        for ex in exchanges:
            step_ms, region, rows = measure(ex)
            regions.append(region)
            res[ex] = summarise(ex, step_ms, rows)
            if world > 1:  # the next exchange (and e2e) gets the memory back
                from paper_1612_02557_b200.distributed import release_peer_windows
                release_peer_windows()
                torch.cuda.empty_cache()
        del data, tmp
        torch.cuda.empty_cache()
        res["_regions"] = regions
        return res

    clocks = ClockSampler(dev_index)
    clocks.start()  # before the warm-up: nvidia-smi's start-up stays outside the timed region
    exchanges = [None] if world == 1 else (["p2p", "nccl"] if args.exchange == "both" else [args.exchange])
    summ = run_workload(args.config, exchanges, args.steps, args.warmup)
    regions = summ.pop("_regions")
    clk = clocks.stop((regions[0][0], regions[-1][1]))
    best = max(summ, key=lambda e: summ[e]["value"])
    head = summ[best]

    # ---------------- C1-C4 beside the headline: same run, same box (N>1: the headline's exchange)
    per_config = None
    if not args.no_per_config:
        per_config = {}
        for name in sorted(CONFIGS):
            if name == args.config:
                continue
            try:
                time.sleep(3)  # let the HBM/power state settle after the previous config
                r = run_workload(name, [best], 3, 3)
                r.pop("_regions")
                per_config[name] = r[best]
            except Exception as ex:  # noqa: BLE001
                per_config[name] = {"error": str(ex)[:200]}

    # ---------------- e2e through the host-memory drop-in
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(rg, torch, dev, lay, n_local, base, dist_kind, seed, args.e2e_steps, world,
                      n_total, max_over_ranks, barrier, best)
        if world == 1 and e2e.get("value"):
            # the same with the drop-in's device buffers kept between calls
            # (raduls_gpu_set_host_cache(1)); the headline above uses the
            # default, which frees them before each call returns
            rg.set_host_cache(True)
            try:
                c = run_e2e(rg, torch, dev, lay, n_local, base, dist_kind, seed, args.e2e_steps, world,
                            n_total, max_over_ranks, barrier, best)
                e2e["cached_buffers"] = {"value": c.get("value"), "ms_per_step": c.get("ms_per_step")}
            finally:
                rg.set_host_cache(False)

    # ---------------- CPU baseline (rank 0, N=1): the reference sorter on the host cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = run_cpu_reference(args.config, args.cpu_cap or reference_cap(args.config), 1, 0)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "same_config")}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (SURVEY.md §8(d) counter-based generator, regenerated on device "
                    "before each step, untimed)",
            "config": {"workload": desc, "n_records": n_total, "record_size": rs, "key_size": ks,
                       "parallelism": "single GPU" if world == 1 else
                       f"{world} GPUs: key-range partition, exchange={best} "
                       "(p2p: partition kernel stores into peer windows over NVLink; "
                       "nccl: local partition + NCCL all-to-all)",
                       "l2": "inputs >> 126 MB L2 (no flush needed)"},
            "verified": head["verified"]["ok"] if world > 1 else head["verified"]["ok"],
            "verification": head["verified"],
            "roofline": head["roofline"], "roofline_sort": head["roofline_sort"],
            "kernels": head["kernels"],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": head["gpu_launches"], "clocks": clk,
            "stats_per_step": head["stats_per_step"],
        }
        if world > 1:
            line["nvlink"] = head["nvlink"]
            line["exchanges"] = {e: {k: summ[e][k] for k in ("value", "ms_per_step", "verified", "roofline",
                                                              "roofline_sort", "nvlink", "gpu_launches")}
                                 for e in summ}
            line["exchange"] = best
        if per_config:
            line["per_config"] = per_config
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def reference_arm(args, n_total, rs, ks, desc) -> int:
    """bench.py --impl reference: the reference CPU sorter on the host cores, on
    the same config as the GPU arm (the whole config when host RAM allows;
    timed runs capped so the arm ends in a few minutes), plus a T=1 figure and
    the C1 pair."""
    cap = args.cpu_cap or reference_cap(args.config)
    full = cap >= n_total
    steps = max(1, min(args.steps, 4)) if full else max(1, args.steps)
    warmup = min(args.warmup, 1) if full else args.warmup
    r = run_cpu_reference(args.config, cap, steps, warmup)
    extra = {}
    try:  # T=1 on C1, and C1 whole at the physical cores: the same-config pair
        r1 = run_cpu_reference("c1", CONFIGS["c1"][0], 1, 0, threads=1)
        extra["t1_c1"] = {k: r1[k] for k in ("value", "unit", "threads", "sample")}
        rc1 = run_cpu_reference("c1", CONFIGS["c1"][0], 3, 1)
        extra["c1"] = {k: rc1[k] for k in ("value", "unit", "threads", "sample", "ms_per_step")}
    except Exception as ex:  # noqa: BLE001
        extra["error"] = str(ex)[:200]
    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": r["steps"], "steps_requested": args.steps, "warmup": warmup,
            "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (SURVEY.md §8(d) counter-based generator)",
            "impl": "reference",
            "config": {"workload": desc, "n_records": n_total, "record_size": rs,
                       "key_size": ks, "sample_records": r["records"], "same_config": r["same_config"]},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference_extra": extra}
    print(json.dumps(line), flush=True)
    return 0


def run_e2e(rg, torch, dev, lay, n_local, base, dist_kind, seed, steps, world, n_total,
            max_over_ranks, barrier, exchange=None):
    """Same metric through the host-memory API: pinned host input, H2D + sort + D2H
    inside the timed region (raduls_gpu_sort_host at N=1; H2D + distributed sort
    + D2H into a pinned result buffer at N>1), after one untimed warm-up call."""
    rs = lay.record_size
    # N>1: one pinned buffer per rank for the input and this rank's key range
    # of the output (which may be a little larger than its input share)
    cap = n_local if world == 1 else int(n_local * 1.25 + (1 << 20))
    try:
        host = torch.empty(cap * rs, dtype=torch.uint8, pin_memory=True)
    except RuntimeError as ex:
        return {"value": None, "unit": UNIT, "error": f"pinned alloc failed: {ex}"[:200]}
    times = []
    for step in range(steps + 1):  # step 0: untimed warm-up (library buffers, windows)
        # pristine input into the pinned buffer (untimed), generated on the device
        # in 4 GiB chunks so the library's own device buffers still fit
        chunk = max(1, (4 << 30) // rs)
        for c0 in range(0, n_local, chunk):
            cn = min(chunk, n_local - c0)
            g = rg.generate(cn, lay, dist=dist_kind, seed=seed, index_base=base + c0, device=dev)
            host[c0 * rs:(c0 + cn) * rs].copy_(g)
            del g
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            rg.sort(host.numpy(), n_local, lay)  # raduls_gpu_sort_host: H2D, sort, D2H
        else:
            from paper_1612_02557_b200.distributed import sort_distributed
            d = host[:n_local * rs].to(dev, non_blocking=True)
            out, n_out = sort_distributed(d, n_local, lay, exchange=exchange)
            del d
            if host.numel() < n_out * rs:  # (skewed keys: a bigger range than planned for)
                host = torch.empty(n_out * rs, dtype=torch.uint8, pin_memory=True)
            host[:n_out * rs].copy_(out[:n_out * rs])
            torch.cuda.synchronize(dev)
            del out
        dt = max_over_ranks(time.perf_counter() - t0)
        if step:
            times.append(dt)
        barrier()
    del host
    torch.cuda.empty_cache()
    return {"value": n_total * len(times) / sum(times), "unit": UNIT,
            "h2d_bytes_per_step": n_total * rs, "d2h_bytes_per_step": n_total * rs,
            "ms_per_step": 1e3 * sum(times) / len(times), "steps": len(times), "warmup": 1,
            "path": "raduls_gpu_sort_host (pinned host buffer; device buffers allocated and freed "
                    "inside every call, as the reference's aux)" if world == 1 else
                    f"H2D + sort_distributed(exchange={exchange}) + D2H"}


if __name__ == "__main__":
    sys.exit(main())
