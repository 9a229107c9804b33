#!/usr/bin/env python
"""bench.py — sorted records/sec of the B200 MSD record sort (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
    python bench.py --impl reference ...      # the reference CPU sorter arm

A "step" is one complete sort of one batch: at N=1 the whole workload
(default C5: 2^32 records of 16 B, the paper's headline scale, BASELINE.json
configs[4]) through libraduls_gpu.so; at N>1 (torchrun, one rank per GPU) the
same total partitioned across ranks by key range (strong scaling) and
exchanged once with an NCCL all-to-all (paper_1612_02557_b200/distributed.py).

Timing: inputs are regenerated on the device before every step (untimed:
the sort is in place); the timed region is the sort call only, bracketed
by a barrier and torch.cuda.synchronize(), CUDA events on the sort's stream,
max over ranks. Inputs (1-64 GiB) exceed the 126 MB L2, so no flush is
needed. Per-kernel CUDA-event times of the timed steps give the live
roofline of the dominant kernel; `e2e` repeats the measurement through the
host-memory drop-in (pinned host buffer, H2D + sort + D2H inside the timed
region); `cpu_baseline` times the reference CPU sorter (oracle/_ref, the
unmodified reference library compiled here) on a bounded sample on the
box's host cores.
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

def cpu_sample(cfg_name: str, n_sample: int):
    import numpy as np

    import oracle
    n, rs, ks, dist, seed, _ = CONFIGS[cfg_name]
    n_s = min(n, n_sample)
    a = oracle.generate(n_s, rs, ks, dist, seed, 0)
    return a, n_s, rs, ks, np


def run_cpu_reference(cfg_name: str, n_sample: int, steps: int, warmup: int) -> dict:
    """The reference CPU sorter on the host cores (oracle/_ref when built, else the
    plain-C port). Returns a dict with records/s over `steps` timed runs."""
    import oracle
    a, n_s, rs, ks, np = cpu_sample(cfg_name, n_sample)
    threads = os.cpu_count() or 1
    kind = "reference" if oracle.ref_available() else "port"
    proxy = ""
    rks = ks
    if kind == "reference" and ks not in (8, 16):
        rks = 16  # the reference rejects ks=24: (32,16) proxy, exact on these inputs
        proxy = f" (run as layout ({rs},16): the reference rejects key_size={ks})"
    work = np.empty_like(a)
    times = []
    for i in range(warmup + steps):
        work[:] = a
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
    ok, _ = oracle.check_sorted(work, rs, ks)
    return {"value": n_s * len(times) / sum(times), "unit": UNIT,
            "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": f"first {n_s} records of the {cfg_name.upper()} generator{proxy}; "
                      f"median run {statistics.median(times)*1e3:.1f} ms; sorted={ok}",
            "ms_per_step": 1e3 * sum(times) / len(times), "steps": len(times)}


# ------------------------------------------------------------------ GPU arm

def algorithmic_bytes(stats: dict, rs: int) -> dict:
    """2*rs per record per executed pass (read + write);
    histogram-only reads are overhead (1*rs per record read whole, 1 byte per
    record read from the digit array, which the scatter before wrote)."""
    nd = stats.get("hist_digit_records", 0)
    return {
        "scatter": 2 * rs * stats["scatter_records"],
        "local_sort": 2 * rs * stats["local_records"],
        "copy_back": 2 * rs * stats["copy_records"],
        "tile_hist": rs * stats["hist_records"] + nd,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample", type=int, default=1 << 26)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "gpu" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n_total, rs, ks, dist_kind, seed, desc = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return 0
        r = run_cpu_reference(args.config, args.cpu_sample, max(1, args.steps), args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": r["steps"], "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u8", "data": "synthetic (SURVEY.md §8(d) counter-based generator)",
                "impl": "reference",
                "config": {"workload": desc, "n_records": n_total, "record_size": rs,
                           "key_size": ks, "sample_records": min(n_total, args.cpu_sample)},
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch

    import paper_1612_02557_b200 as rg
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    lay = rg.RecordLayout(rs, ks)
    n_local = n_total // world
    base = rank * n_local
    if rank == world - 1:
        n_local = n_total - base

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---------------- device-resident measurement
    data = torch.empty(n_local * rs, dtype=torch.uint8, device=dev)
    tmp = torch.empty_like(data) if world == 1 else None
    stream = torch.cuda.current_stream(dev)
    rg.set_profiling(False)

    def one_step(timed: bool):
        rg.generate(n_local, lay, dist=dist_kind, seed=seed, index_base=base, out=data)
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if world == 1:
            rg.sort(data, n_local, lay, tmp=tmp, stream=stream)
            out, n_out = data, n_local
        else:
            from paper_1612_02557_b200.distributed import sort_distributed
            out, n_out = sort_distributed(data, n_local, lay)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return e0.elapsed_time(e1), out, n_out

    clocks = ClockSampler(local_rank)
    clocks.start()  # before the warm-up: nvidia-smi's start-up stays outside the timed region
    for _ in range(args.warmup):
        _, out, n_out = one_step(False)
        del out
    digest_in = None
    if world == 1:
        rg.generate(n_local, lay, dist=dist_kind, seed=seed, index_base=base, out=data)
        digest_in = rg.digest(data, n_local, rs)
    rg.set_profiling(True)
    kt_sum: dict[str, list] = {}
    stats_sum: dict[str, int] = {}
    step_ms = []
    t_region0 = time.time()
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        ms, out, n_out = one_step(True)
        step_ms.append(max_over_ranks(ms))
        if world == 1:
            for k, (l, t) in rg.last_kernel_times().items():
                kt_sum.setdefault(k, [0, 0.0])
                kt_sum[k][0] += l
                kt_sum[k][1] += t
            for k, v in rg.last_stats().items():
                stats_sum[k] = stats_sum.get(k, 0) + v
    wall = time.perf_counter() - wall0
    clk = clocks.stop((t_region0, time.time()))
    rg.set_profiling(False)
    # verify the last step (untimed)
    viol, _ = rg.check_sorted(out, n_out, lay)
    verified = viol == 0
    if world == 1:
        verified = verified and rg.digest(out, n_out, rs) == digest_in
    if world > 1:
        t = torch.tensor([0 if verified else 1], device=dev)
        torch.distributed.all_reduce(t)
        verified = int(t.item()) == 0
    del out
    total_ms = sum(step_ms)
    value = n_total * args.steps / (total_ms / 1e3)

    # ---------------- roofline of the dominant kernel (live CUDA-event times)
    peak, peak_src = load_peaks()
    roofline = None
    kernels = {}
    if world == 1 and kt_sum:
        ab = algorithmic_bytes(stats_sum, rs)
        for k, (l, t) in kt_sum.items():
            b = ab.get(k, 0)
            kernels[k] = {"launches": l, "ms": round(t, 3),
                          "GBps": round(b / (t / 1e3) / 1e9, 1) if b and t else None}
        dom = max(kt_sum, key=lambda k: kt_sum[k][1])
        dl, dt = kt_sum[dom]
        db = ab.get(dom, 0)
        achieved = db / (dt / 1e3) / 1e9 if dt else 0.0
        traffic = None
        tfile = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
        if os.path.exists(tfile):
            try:
                with open(tfile) as f:
                    traffic = json.load(f).get(dom)
            except Exception:  # noqa: BLE001
                traffic = None
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4),
                    "traffic": traffic, "algorithmic_bytes_per_launch": db / max(dl, 1),
                    "launches": dl, "peak_source": peak_src}
        sort_alg = ab["scatter"] + ab["local_sort"] + ab["copy_back"]
        sort_gbs = sort_alg / (total_ms / 1e3) / 1e9
        roofline_sort = {"achieved": round(sort_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(sort_gbs / peak, 4),
                         "algorithmic_bytes_per_step": sort_alg / args.steps,
                         "passes_per_record": round(sort_alg / args.steps / (2 * rs * n_total), 3)}
    else:
        roofline_sort = None
    gpu_launches = sum(v[0] for v in kt_sum.values()) if kt_sum else None
    if world > 1:
        gpu_launches = None  # counted per rank only in single-GPU runs

    del data, tmp
    torch.cuda.empty_cache()

    # ---------------- e2e through the host-memory drop-in
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(rg, torch, dev, lay, n_local, base, dist_kind, seed, args.e2e_steps, world,
                      n_total, max_over_ranks, barrier)

    # ---------------- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = run_cpu_reference(args.config, args.cpu_sample, 3, 1)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (SURVEY.md §8(d) counter-based generator, regenerated on device "
                    "before each step, untimed)",
            "config": {"workload": desc, "n_records": n_total, "record_size": rs, "key_size": ks,
                       "parallelism": "single GPU" if world == 1 else
                       f"{world} GPUs: key-range partition + NCCL all-to-all",
                       "l2": "inputs >> 126 MB L2 (no flush needed)"},
            "verified": verified,
            "wall_s_timed_region": wall,
            "roofline": roofline, "roofline_sort": roofline_sort, "kernels": kernels or None,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk,
            "stats_per_step": {k: v // args.steps for k, v in stats_sum.items()} or None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_e2e(rg, torch, dev, lay, n_local, base, dist_kind, seed, steps, world, n_total,
            max_over_ranks, barrier):
    """Same metric through the host-memory API: pinned host input, H2D + sort + D2H
    inside the timed region (raduls_gpu_sort_host at N=1; H2D + distributed sort
    + D2H into a pinned result buffer at N>1), after one untimed warm-up call."""
    rs = lay.record_size
    nbytes = n_local * rs
    try:
        host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    except RuntimeError as ex:
        return {"value": None, "unit": UNIT, "error": f"pinned alloc failed: {ex}"[:200]}
    times = []
    res = None  # N>1: pinned result buffer, allocated outside the timed region
    if world > 1:
        res = torch.empty(int(n_local * 1.25 + (1 << 20)) * rs, dtype=torch.uint8, pin_memory=True)
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
            d = host.to(dev, non_blocking=True)
            out, n_out = sort_distributed(d, n_local, lay)
            del d
            if res.numel() < n_out * rs:  # (skewed keys: a bigger range than planned for)
                res = torch.empty(n_out * rs, dtype=torch.uint8, pin_memory=True)
            res[:n_out * rs].copy_(out[:n_out * rs])
            torch.cuda.synchronize(dev)
            del out
        dt = max_over_ranks(time.perf_counter() - t0)
        if step:
            times.append(dt)
        barrier()
    del host, res
    torch.cuda.empty_cache()
    return {"value": n_total * len(times) / sum(times), "unit": UNIT,
            "h2d_bytes_per_step": n_total * rs, "d2h_bytes_per_step": n_total * rs,
            "ms_per_step": 1e3 * sum(times) / len(times), "steps": len(times), "warmup": 1,
            "path": "raduls_gpu_sort_host (pinned host buffer)" if world == 1 else
                    "H2D + sort_distributed + D2H"}


if __name__ == "__main__":
    sys.exit(main())
