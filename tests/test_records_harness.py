"""Record files (P/src/datagen.cpp:120-144) and the CSV bench harness
(P/src/bench.cpp:22-211). CPU tests mirror P/tests/test_datagen.cpp:138-166
and P/tests/test_bench.cpp:137-162; the run_bench cases (GPU) mirror
test_bench.cpp:59-135 with the fake clock."""
import io
import os

import numpy as np
import pytest

import paper_1612_02557_b200 as rg
from paper_1612_02557_b200 import harness
from helpers import make_input


def test_file_round_trip(tmp_path):
    """test_datagen.cpp:138-166."""
    path = str(tmp_path / "raduls_datagen_test.bin")
    lay = rg.RecordLayout(16, 8)
    a = rg.RecordArray(lay, 12345)
    a.buf[:] = make_input(12345, 16, 8, 6)
    rg.save_file(path, a)
    b = rg.load_file(path, lay)
    assert b.size() == 12345 and np.array_equal(a.buf, b.buf)
    assert b.buf.ctypes.data % 64 == 0  # allocate_record_bytes alignment
    rg.save_file(path, rg.RecordArray(lay, 0))
    assert rg.load_file(path, lay).size() == 0
    with open(path, "wb") as f:
        f.write(b"0123456789")
    with pytest.raises(rg.FormatError, match="16"):
        rg.load_file(path, lay)
    with pytest.raises(rg.IoError):
        rg.load_file("/nonexistent/raduls.bin", lay)
    with pytest.raises(ValueError, match="unsupported record layout"):
        rg.load_file(path, rg.RecordLayout(8, 16))
    with pytest.raises(rg.IoError):
        rg.save_file("/nonexistent/dir/raduls.bin", a)


def test_record_array_views():
    lay = rg.RecordLayout(24, 16)
    a = rg.RecordArray(lay, 5)
    a.records()[:] = np.arange(5 * 24, dtype=np.uint8).reshape(5, 24)
    assert np.array_equal(a.record(3), np.arange(72, 96, dtype=np.uint8))
    c = a.clone()
    c.buf[0] = 99
    assert a.buf[0] == 0 and a.byte_size() == 120 and not a.empty()


def test_csv_header_and_row_format():
    assert harness.csv_header() == ("algo,n,record_size,key_size,distribution,threads,"
                                    "wall_time,verified,repeat_index")
    out = io.StringIO()
    harness.write_csv_row(out, harness.RunResult("raduls_gpu", 100, 16, 8, "uniform", 1,
                                                 0.5, True, 2))
    assert out.getvalue() == "raduls_gpu,100,16,8,uniform,1,0.500000000,true,2\n"


def test_speedup_report_medians_and_missing_baselines():
    """test_bench.cpp:137-162, same rows, same expectations."""
    csv = io.StringIO(harness.csv_header() + "\n"
                      "fast,100,16,8,uniform,1,10.0,true,0\n"
                      "fast,100,16,8,uniform,1,10.0,true,1\n"
                      "fast,100,16,8,uniform,2,5.0,true,0\n"
                      "fast,100,16,8,uniform,2,20.0,true,1\n"
                      "nobase,100,16,8,uniform,2,1.0,true,0\n")
    out, log = io.StringIO(), io.StringIO()
    assert harness.speedup_report(csv, out, log) == 0
    rows = [r for r in out.getvalue().splitlines() if r]
    assert len(rows) == 3
    assert rows[0] == "algo,threads,median_wall_time,speedup"
    f1, f2 = rows[1].split(","), rows[2].split(",")
    assert f1[:2] == ["fast", "1"] and float(f1[3]) == pytest.approx(1.0)
    assert f2[1] == "2" and float(f2[2]) == pytest.approx(12.5)
    assert float(f2[3]) == pytest.approx(0.8)
    assert "nobase" in log.getvalue()
    assert harness.speedup_report(io.StringIO(""), out, log) == 0
    assert "empty CSV input" in log.getvalue()


def test_unknown_algorithm_rejected():
    with pytest.raises(ValueError, match="unknown algorithm"):
        harness.run_bench(harness.BenchRequest(algos=["bogus"], n=10), io.StringIO(),
                          io.StringIO())


def counting_clock():
    calls = [0]

    def now():
        calls[0] += 1
        return calls[0] * 1_000_000_000
    return now, calls


@pytest.mark.gpu
def test_wall_time_covers_the_sort_call_only(torch_cuda):
    """test_bench.cpp:59-98: two clock reads per run, Cartesian row order."""
    req = harness.BenchRequest(algos=["raduls_gpu", "lsd1_gpu"], n=5000,
                               layout=rg.RecordLayout(16, 8), threads=[1, 2], repeats=2,
                               verify="full")
    now, calls = counting_clock()
    csv, log = io.StringIO(), io.StringIO()
    assert harness.run_bench(req, csv, log, now) == 0, log.getvalue()
    rows = [r for r in csv.getvalue().splitlines() if r]
    assert len(rows) == 9 and rows[0] == harness.csv_header()
    want_algo = ["raduls_gpu"] * 4 + ["lsd1_gpu"] * 4
    want_t = ["1", "1", "2", "2"] * 2
    want_rep = ["0", "1"] * 4
    for i in range(8):
        f = rows[i + 1].split(",")
        assert len(f) == 9
        assert f[0] == want_algo[i] and f[1] == "5000" and f[2] == "16" and f[3] == "8"
        assert f[4] == "uniform" and f[5] == want_t[i] and f[8] == want_rep[i]
        assert float(f[6]) == pytest.approx(1.0) and f[7] == "true"
    assert calls[0] == 16


@pytest.mark.gpu
def test_identical_requests_identical_rows(torch_cuda):
    """test_bench.cpp:100-117 (skewed distribution, fake clock)."""
    req = harness.BenchRequest(algos=["lsd4_gpu", "raduls_gpu_device"], n=2000,
                               layout=rg.RecordLayout(24, 8), dist=rg.DIST_SKEW, seed=99,
                               threads=[2], repeats=1, verify="digest")
    a, b = io.StringIO(), io.StringIO()
    harness.run_bench(req, a, io.StringIO(), counting_clock()[0])
    harness.run_bench(req, b, io.StringIO(), counting_clock()[0])
    assert a.getvalue() == b.getvalue()
    assert all(r.endswith(",true,0") for r in a.getvalue().splitlines()[1:])


@pytest.mark.gpu
def test_zero_records_and_file_input(torch_cuda, tmp_path):
    """test_bench.cpp:119-135 plus the --input path (bench.cpp:86-90)."""
    csv = io.StringIO()
    assert harness.run_bench(harness.BenchRequest(n=0, repeats=1, verify="digest"), csv,
                             io.StringIO()) == 0
    f = csv.getvalue().splitlines()[1].split(",")
    assert f[1] == "0" and f[7] == "true"
    path = str(tmp_path / "in.bin")
    arr = rg.RecordArray(rg.RecordLayout(32, 24), 3000)
    arr.buf[:] = make_input(3000, 32, 24, 17, universe=100)
    rg.save_file(path, arr)
    csv = io.StringIO()
    req = harness.BenchRequest(algos=["raduls_gpu", "raduls_gpu_device", "lsd4_gpu"],
                               layout=rg.RecordLayout(32, 24), repeats=1, input_path=path,
                               verify="full")
    assert harness.run_bench(req, csv, io.StringIO()) == 0
    rows = csv.getvalue().splitlines()[1:]
    assert len(rows) == 3 and all(r.split(",")[4] == "file" for r in rows)
    assert os.path.getsize(path) == 3000 * 32
