"""Benchmark harness with the reference's CSV schema, so its tooling
(``speedup_report``) consumes GPU rows unchanged.

Mirrors P/include/raduls/bench.hpp:17-71 and P/src/bench.cpp:22-211:

* ``csv_header()`` — the exact header
  ``algo,n,record_size,key_size,distribution,threads,wall_time,verified,repeat_index``;
* ``write_csv_row`` — same field order and ``%.9f`` wall time;
* ``run_bench(req, csv, log, now)`` — one dataset (generated, or loaded from a
  raw record file), then algos x threads x repeats on a fresh copy each, the
  clock read exactly twice per run around the sort call (``now`` is
  injectable, bench.hpp:52-56), optional verification outside the bracket;
  returns 0 when every verification passed, else 1;
* ``speedup_report(csv_in, out, log)`` — per-algorithm medians and speedups
  against the threads=1 row (bench.cpp:162-211).

Algorithms (the reference's are raduls | lsd1 | lsd4 | oracle, bench.cpp:24-47):

* ``raduls_gpu``        — MSD sort through the host drop-in (H2D + sort + D2H
  inside the bracket: the reference's call shape, host memory in and out);
* ``raduls_gpu_device`` — the same sort on device-resident data (copied in
  before the bracket; the bracket ends after a device synchronize);
* ``lsd1_gpu`` / ``lsd4_gpu`` — the LSD baseline through its host drop-in,
  LsdConfig{64} / LsdConfig{256} as the reference's lsd1 / lsd4.

``threads`` is the GPU count of the row (1: this harness runs one device).
Verification (``digest``) uses the library's device checkers: sortedness
(check_sorted, verify.cpp:27-35) plus the order-independent multiset digest
(array_digest, verify.cpp:37-50). ``full`` additionally requires the MSD and
LSD outputs to be byte-identical (both are stable).
"""
from __future__ import annotations

import io
import statistics
import sys
import time
from dataclasses import dataclass, field
from typing import Callable, TextIO

import numpy as np

from . import raduls as R
from .records import RecordArray, load_file

__all__ = ["BenchRequest", "RunResult", "csv_header", "write_csv_row", "run_bench",
           "speedup_report", "KNOWN_ALGOS"]

KNOWN_ALGOS = ("raduls_gpu", "raduls_gpu_device", "lsd1_gpu", "lsd4_gpu")
_CSV_HEADER = "algo,n,record_size,key_size,distribution,threads,wall_time,verified,repeat_index"


@dataclass
class BenchRequest:
    algos: list = field(default_factory=lambda: ["raduls_gpu"])
    n: int = 0
    layout: R.RecordLayout = field(default_factory=R.RecordLayout)
    dist: int = R.DIST_UNIFORM           # DIST_UNIFORM | DIST_SKEW (§8(d) generator)
    seed: int = 0
    threads: list = field(default_factory=lambda: [1])
    repeats: int = 3
    input_path: str = ""                 # when set, load records instead of generating
    verify: str = "none"                 # none | digest | full


@dataclass
class RunResult:
    algo: str = ""
    n: int = 0
    record_size: int = 0
    key_size: int = 0
    distribution: str = ""
    threads: int = 0
    wall_time: float = 0.0  # seconds, sort call only
    verified: bool = True
    repeat_index: int = 0


def csv_header() -> str:
    return _CSV_HEADER


def write_csv_row(out: TextIO, r: RunResult) -> None:
    out.write(f"{r.algo},{r.n},{r.record_size},{r.key_size},{r.distribution},{r.threads},"
              f"{r.wall_time:.9f},{'true' if r.verified else 'false'},{r.repeat_index}\n")


def _monotonic_ns() -> int:
    return time.monotonic_ns()


def _dataset(req: BenchRequest, log: TextIO) -> tuple[RecordArray, str]:
    if req.input_path:
        ds = load_file(req.input_path, req.layout)
        log.write(f"loaded {ds.size()} records from {req.input_path}\n")
        return ds, "file"
    ds = RecordArray(req.layout, req.n)
    name = "uniform" if req.dist == R.DIST_UNIFORM else "zipf"
    if req.n:
        dev = R.generate(req.n, req.layout, dist=req.dist, seed=req.seed)
        ds.buf[:] = dev.cpu().numpy()
    log.write(f"generated {ds.size()} {name} records (seed {req.seed})\n")
    return ds, name


def _device_checks(buf: np.ndarray, n: int, layout: R.RecordLayout):
    torch = R._torch()
    d = torch.from_numpy(buf).cuda() if buf.size else torch.empty(0, dtype=torch.uint8,
                                                                 device="cuda")
    if n == 0:
        return (0, 0), 0
    return R.digest(d, n, layout.record_size), R.check_sorted(d, n, layout)[0]


def run_bench(req: BenchRequest, csv: TextIO, log: TextIO,
              now: Callable[[], int] | None = None) -> int:
    for a in req.algos:
        if a not in KNOWN_ALGOS:
            raise ValueError(f"unknown algorithm: {a}")
    if not req.layout.valid():
        raise R._layout_error(req.layout)
    now = now or _monotonic_ns
    ds, dist_name = _dataset(req, log)
    n, layout = ds.size(), ds.layout
    want_digest = None
    if req.verify != "none":
        want_digest, _ = _device_checks(ds.buf, n, layout)
    reference_out = None  # first stable output, for verify == "full"

    torch = R._torch()
    work = RecordArray(layout, n)
    dev = dev_tmp = None
    if "raduls_gpu_device" in req.algos:
        dev = torch.empty(max(n * layout.record_size, 1), dtype=torch.uint8, device="cuda")
        dev_tmp = torch.empty_like(dev)
    csv.write(csv_header() + "\n")
    all_ok = True
    for algo in req.algos:
        for t in req.threads:
            for rep in range(req.repeats):
                work.buf[:] = ds.buf
                if algo == "raduls_gpu_device":
                    if n:
                        dev[:n * layout.record_size].copy_(torch.from_numpy(work.buf))
                    torch.cuda.synchronize()
                t0 = now()
                if algo == "raduls_gpu":
                    R.sort(work.buf, n, layout)
                elif algo == "raduls_gpu_device":
                    R.sort(dev, n, layout, tmp=dev_tmp)
                    torch.cuda.synchronize()
                elif algo == "lsd1_gpu":
                    R.lsd_sort(work.buf, n, layout, R.LsdConfig(64, t))
                else:
                    R.lsd_sort(work.buf, n, layout, R.LsdConfig(256, t))
                t1 = now()
                if algo == "raduls_gpu_device" and n:
                    work.buf[:] = dev[:n * layout.record_size].cpu().numpy()
                row = RunResult(algo, n, layout.record_size, layout.key_size, dist_name, t,
                                (t1 - t0) * 1e-9, True, rep)
                if req.verify != "none":
                    dg, inversions = _device_checks(work.buf, n, layout)
                    ok = inversions == 0 and dg == want_digest
                    if req.verify == "full":
                        if reference_out is None:
                            reference_out = work.buf.copy()
                        ok = ok and np.array_equal(work.buf, reference_out)
                    row.verified = ok
                    if not ok:
                        all_ok = False
                        log.write(f"verification FAILED: algo={algo} threads={t} repeat={rep}\n")
                write_csv_row(csv, row)
    return 0 if all_ok else 1


def speedup_report(csv_in: TextIO, out: TextIO, log: TextIO) -> int:
    line = csv_in.readline()
    if not line:
        log.write("empty CSV input\n")
        return 0
    header = line.rstrip("\n").split(",")
    try:
        ai, ti, wi = header.index("algo"), header.index("threads"), header.index("wall_time")
    except ValueError:
        log.write("CSV is missing algo/threads/wall_time columns\n")
        return 0
    order: list = []
    samples: dict = {}
    need = max(ai, ti, wi) + 1
    for line in csv_in:
        line = line.rstrip("\n")
        if not line:
            continue
        f = line.split(",")
        if len(f) < need:
            continue
        if f[ai] not in samples:
            order.append(f[ai])
            samples[f[ai]] = {}
        samples[f[ai]].setdefault(int(f[ti]), []).append(float(f[wi]))
    out.write("algo,threads,median_wall_time,speedup\n")
    for algo in order:
        by_t = samples[algo]
        if 1 not in by_t:
            log.write(f"no threads=1 baseline for {algo}, skipped\n")
            continue
        base = statistics.median(by_t[1])
        for t in sorted(by_t):
            m = statistics.median(by_t[t])
            out.write(f"{algo},{t},{m:.9f},{(base / m if m > 0 else 0.0):.4f}\n")
    return 0


def main(argv=None) -> int:
    """``python -m paper_1612_02557_b200.harness run --algo raduls_gpu,lsd1_gpu --n N
    [--record-size 16 --key-size 8 --dist uniform|zipf --seed S --repeats K
    --input FILE --verify none|digest|full]`` -> CSV on stdout;
    ``... speedup < results.csv`` -> the speedup table."""
    import argparse
    p = argparse.ArgumentParser(prog="raduls_gpu_bench")
    sub = p.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--algo", default="raduls_gpu")
    r.add_argument("--n", type=int, default=0)
    r.add_argument("--record-size", type=int, default=16)
    r.add_argument("--key-size", type=int, default=8)
    r.add_argument("--dist", choices=["uniform", "zipf"], default="uniform")
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--repeats", type=int, default=3)
    r.add_argument("--input", default="")
    r.add_argument("--verify", choices=["none", "digest", "full"], default="none")
    sub.add_parser("speedup")
    a = p.parse_args(argv)
    if a.cmd == "speedup":
        return speedup_report(sys.stdin, sys.stdout, sys.stderr)
    req = BenchRequest(algos=a.algo.split(","), n=a.n,
                       layout=R.RecordLayout(a.record_size, a.key_size),
                       dist=R.DIST_UNIFORM if a.dist == "uniform" else R.DIST_SKEW,
                       seed=a.seed, repeats=a.repeats, input_path=a.input, verify=a.verify)
    buf = io.StringIO()
    rc = run_bench(req, buf, sys.stderr)
    sys.stdout.write(buf.getvalue())
    return rc


if __name__ == "__main__":
    sys.exit(main())
