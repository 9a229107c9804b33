"""CPU: the C-ABI library loads and exports every entry point include/raduls_gpu.h
declares; host-side argument validation works without a GPU (errors are
reported before any device work, like the reference's std::invalid_argument,
P/include/raduls/detail/dispatch.hpp:37-39)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1612_02557_b200 as rg
from paper_1612_02557_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "raduls_gpu.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(raduls_gpu_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), f"{name} missing from libraduls_gpu.so"
    assert set(_lib.EXPORTED) <= set(names)


def test_no_oracle_in_product():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_1612_02557_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in src and "liboracle" not in src, f


def test_layout_validation_matches_reference_table():
    L = _lib.load()
    # reference valid set (P/include/raduls/layout.hpp:22-27) plus widened key sizes
    for rs, ks in [(8, 8), (16, 8), (16, 16), (24, 8), (24, 16), (32, 8), (32, 16), (32, 24),
                   (16, 1), (32, 32)]:
        assert L.raduls_gpu_layout_valid(rs, ks) == 1
        assert rg.RecordLayout(rs, ks).valid()
    for rs, ks in [(8, 16), (12, 8), (16, 12 + 8), (40, 8), (0, 8), (16, 0)]:
        assert L.raduls_gpu_layout_valid(rs, ks) == 0


def test_invalid_arguments_rejected_without_gpu():
    L = _lib.load()
    assert L.raduls_gpu_sort(None, None, 10, 12, 8, None) == _lib.EINVAL
    assert L.raduls_gpu_sort(None, None, 10, 16, 17, None) == _lib.EINVAL
    assert L.raduls_gpu_sort(None, None, 2**62, 16, 8, None) == _lib.EINVAL  # size overflow
    assert L.raduls_gpu_sort(None, None, 10, 16, 8, None) == _lib.EINVAL      # null data
    assert L.raduls_gpu_sort(8, None, 10, 16, 8, None) == _lib.EINVAL         # misaligned
    assert L.raduls_gpu_sort_host(None, None, 10, 8, 8) == _lib.EINVAL
    assert L.raduls_gpu_sort(None, None, 1, 16, 8, None) == _lib.OK           # n < 2: no-op
    assert L.raduls_gpu_sort_host(None, None, 0, 16, 8) == _lib.OK
    assert "invalid" in _lib.strerror(_lib.EINVAL)
    with pytest.raises(ValueError, match="unsupported record layout"):
        rg.sort(np.zeros(64, dtype=np.uint8), 2, rg.RecordLayout(8, 16))


def test_version_and_stats_struct():
    L = _lib.load()
    assert L.raduls_gpu_version() >= 0x000100
    assert C.sizeof(_lib.Stats) == 4 + 4 + 8 * 8  # (round 2: + bitmap_spill_groups)


def test_stats_struct_fields_match_the_header():
    """The ctypes mirror of raduls_gpu_stats has the header's fields, in order
    and with the header's widths (an ABI drift would misread every counter)."""
    txt = open(HEADER).read()
    body = re.search(r"typedef struct \{(.*?)\} raduls_gpu_stats;", txt, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(uint32_t|uint64_t)\s+(\w+)\s*;", body)
    want = [(name, C.c_uint32 if t == "uint32_t" else C.c_uint64) for t, name in fields]
    assert want == list(_lib.Stats._fields_)
    assert want[-1][0] == "bitmap_spill_groups"


def test_lsd_rejects_bad_config_and_layouts_without_gpu():
    """test_lsd.cpp:69-77: lane sizes 63 and 0, layout (8, 16) -> invalid_argument."""
    L = _lib.load()
    buf = np.zeros(64, dtype=np.uint8)
    for lane in (63, 0):
        with pytest.raises(ValueError, match="multiple of 64"):
            rg.lsd_sort(buf, 2, rg.RecordLayout(16, 8), rg.LsdConfig(lane, 1))
    with pytest.raises(ValueError, match="unsupported record layout"):
        rg.lsd_sort(buf, 2, rg.RecordLayout(8, 16), rg.LsdConfig(64, 1))
    assert L.raduls_gpu_lsd_sort(None, None, 10, 12, 8, None) == _lib.EINVAL
    assert L.raduls_gpu_lsd_sort(8, None, 10, 16, 8, None) == _lib.EINVAL       # misaligned
    assert L.raduls_gpu_lsd_sort(None, None, 1, 16, 8, None) == _lib.OK         # n < 2
    assert L.raduls_gpu_lsd_sort_host(None, None, 10, 16, 8) == _lib.EINVAL
    assert L.raduls_gpu_lsd_sort_host(None, None, 1, 16, 8) == _lib.OK


def test_sort_multi_rejects_bad_arguments_without_gpu():
    L = _lib.load()
    dev = (C.c_int * 1)(0)
    ptrs = (C.c_void_p * 1)(None)
    n = np.zeros(1, dtype=np.uint64)
    nout = np.zeros(1, dtype=np.uint64)
    args = (dev, ptrs, n.ctypes.data_as(_lib._u64p), ptrs, nout.ctypes.data_as(_lib._u64p), 10)
    assert L.raduls_gpu_sort_multi(0, *args, 16, 8) == _lib.EINVAL      # no devices
    assert L.raduls_gpu_sort_multi(1, *args, 12, 8) == _lib.EINVAL      # layout
    assert L.raduls_gpu_sort_multi(1, *args, 16, 8) == _lib.EINVAL      # null output


def test_partition_phases_and_samples_reject_bad_arguments_without_gpu():
    """raduls_gpu_partition_plan / _store and the sample entry points validate
    before touching a device (include/raduls_gpu.h)."""
    L = _lib.load()
    cnt = np.zeros(2, dtype=np.uint64)
    ao = np.zeros(8, dtype=np.uint64)
    cp, ap = cnt.ctypes.data_as(_lib._u64p), ao.ctypes.data_as(_lib._u64p)
    assert L.raduls_gpu_partition_plan(None, 10, 12, 8, 0, 16, 2, cp, ap, None) == _lib.EINVAL  # layout
    assert L.raduls_gpu_partition_plan(None, 10, 16, 8, 0, None, 2, cp, ap, None) == _lib.EINVAL  # no map
    assert L.raduls_gpu_partition_plan(None, 10, 16, 8, 0, 16, 0, cp, ap, None) == _lib.EINVAL  # 0 ranks
    assert L.raduls_gpu_partition_plan(None, 10, 16, 8, 0, 16, 2, None, ap, None) == _lib.EINVAL
    assert L.raduls_gpu_partition_plan(8, 10, 16, 8, 0, 16, 2, cp, ap, None) == _lib.EINVAL  # misaligned
    assert L.raduls_gpu_partition_store(None, 10, 12, 8, cp, None) == _lib.EINVAL
    assert L.raduls_gpu_partition_store(None, 10, 16, 8, None, None) == _lib.EINVAL
    assert L.raduls_gpu_sample_andor(None, 10, 12, 64, ap, None) == _lib.EINVAL
    assert L.raduls_gpu_sample_andor(None, 10, 16, 64, None, None) == _lib.EINVAL
    assert L.raduls_gpu_sample_prefix_histogram(None, 10, 16, 17, 0, 64, 16, None) == _lib.EINVAL
    assert L.raduls_gpu_sample_prefix_histogram(8, 10, 16, 8, 0, 64, 16, None) == _lib.EINVAL
