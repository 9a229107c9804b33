"""ctypes binding of libraduls_gpu.so (C-ABI in include/raduls_gpu.h).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, every entry point raises. The library is loaded from this package
directory only (never from site-packages), so the driver can see which .so
the tests and the bench actually used.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# RADULS_GPU_LIB=checked selects the checked build (libraduls_gpu_checked.so,
# bounds/alignment/deadlock checks and poisoned scratch; tests/test_gpu_checked.py)
LIB_PATH = os.path.join(HERE, "libraduls_gpu_checked.so" if os.environ.get("RADULS_GPU_LIB") == "checked"
                        else "libraduls_gpu.so")

OK, EINVAL, ENOMEM, ECUDA, ENCCL, EINTERNAL = 0, 1, 2, 3, 4, 5

EXPORTED = [
    "raduls_gpu_strerror",
    "raduls_gpu_layout_valid",
    "raduls_gpu_version",
    "raduls_gpu_sort",
    "raduls_gpu_sort_host",
    "raduls_gpu_lsd_sort",
    "raduls_gpu_lsd_sort_host",
    "raduls_gpu_last_stats",
    "raduls_gpu_split",
    "raduls_gpu_histogram",
    "raduls_gpu_generate",
    "raduls_gpu_digest",
    "raduls_gpu_check_sorted",
    "raduls_gpu_prefix_histogram",
    "raduls_gpu_partition",
    "raduls_gpu_release",
    "raduls_gpu_set_profiling",
    "raduls_gpu_last_kernel_times",
    "raduls_gpu_andor",
    "raduls_gpu_sort_multi",
    "raduls_gpu_partition_to",
    "raduls_gpu_partition_plan",
    "raduls_gpu_partition_store",
    "raduls_gpu_sample_andor",
    "raduls_gpu_sample_prefix_histogram",
    "raduls_gpu_ipc_alloc",
    "raduls_gpu_ipc_open",
    "raduls_gpu_ipc_close",
    "raduls_gpu_free",
    "raduls_gpu_rank_mode",
    "raduls_gpu_digit_andor",
    "raduls_gpu_partition_store_pieces",
    "raduls_gpu_launch_count",
    "raduls_gpu_set_host_cache",
    "raduls_gpu_set_pivots",
    "raduls_gpu_check_report",
    "raduls_gpu_sort_segments",
]


class Stats(C.Structure):
    _fields_ = [
        ("levels", C.c_uint32),
        ("scatter_launches", C.c_uint32),
        ("hist_records", C.c_uint64),
        ("scatter_records", C.c_uint64),
        ("local_records", C.c_uint64),
        ("copy_records", C.c_uint64),
        ("fallback_groups", C.c_uint64),
        ("skipped_levels", C.c_uint64),
        ("hist_digit_records", C.c_uint64),
        ("bitmap_spill_groups", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("launches", C.c_uint32), ("ms", C.c_double)]


_lock = threading.Lock()
_lib = None

_vp = C.c_void_p
_u32 = C.c_uint32
_u64 = C.c_uint64
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)


def load(build_if_missing: bool = False):
    """Return the loaded library; raise RuntimeError when it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if build_if_missing:
                from . import build as _b
                _b.build()
            else:
                raise RuntimeError(
                    f"{LIB_PATH} is not built; run `python -m paper_1612_02557_b200.build` "
                    "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.raduls_gpu_strerror.restype = C.c_char_p
        L.raduls_gpu_strerror.argtypes = [C.c_int]
        L.raduls_gpu_layout_valid.argtypes = [_u32, _u32]
        L.raduls_gpu_version.restype = _u32
        L.raduls_gpu_sort.argtypes = [_vp, _vp, _u64, _u32, _u32, _vp]
        L.raduls_gpu_sort_host.argtypes = [_vp, _vp, _u64, _u32, _u32]
        L.raduls_gpu_lsd_sort.argtypes = [_vp, _vp, _u64, _u32, _u32, _vp]
        L.raduls_gpu_lsd_sort_host.argtypes = [_vp, _vp, _u64, _u32, _u32]
        L.raduls_gpu_last_stats.argtypes = [C.POINTER(Stats)]
        L.raduls_gpu_split.argtypes = [_vp, _vp, _u64, _u32, _u32, _u64p, _vp]
        L.raduls_gpu_histogram.argtypes = [_vp, _u64, _u32, _u32, _u64p, _u64p, _vp]
        L.raduls_gpu_generate.argtypes = [_vp, _u64, _u32, _u32, _u32, _u64, _u64, _vp]
        L.raduls_gpu_digest.argtypes = [_vp, _u64, _u32, _u64p, _u64p, _vp]
        L.raduls_gpu_check_sorted.argtypes = [_vp, _u64, _u32, _u32, _u64p, _u64p, _vp]
        L.raduls_gpu_prefix_histogram.argtypes = [_vp, _u64, _u32, _u32, _u32, _vp, _vp]
        L.raduls_gpu_partition.argtypes = [_vp, _vp, _u64, _u32, _u32, _u32, _vp, _u32, _u64p, _vp]
        L.raduls_gpu_release.restype = None
        L.raduls_gpu_set_profiling.argtypes = [C.c_int]
        L.raduls_gpu_andor.argtypes = [_vp, _u64, _u32, _u64p, _vp]
        L.raduls_gpu_partition_to.argtypes = [_vp, _u64, _u32, _u32, _u32, _vp, _u32, _u64p, _u64p, _vp]
        L.raduls_gpu_partition_plan.argtypes = [_vp, _u64, _u32, _u32, _u32, _vp, _u32, _u64p, _u64p, _vp]
        L.raduls_gpu_partition_store.argtypes = [_vp, _u64, _u32, _u32, _u64p, _vp]
        L.raduls_gpu_sample_andor.argtypes = [_vp, _u64, _u32, _u32, _u64p, _vp]
        L.raduls_gpu_sample_prefix_histogram.argtypes = [_vp, _u64, _u32, _u32, _u32, _u32, _vp, _vp]
        L.raduls_gpu_ipc_alloc.argtypes = [_u64, C.POINTER(_vp), C.c_char_p]
        L.raduls_gpu_ipc_open.argtypes = [C.c_char_p, C.POINTER(_vp)]
        L.raduls_gpu_ipc_close.argtypes = [_vp]
        L.raduls_gpu_free.argtypes = [_vp]
        L.raduls_gpu_rank_mode.argtypes = [C.POINTER(C.c_int)]
        L.raduls_gpu_launch_count.argtypes = [_u64p]
        L.raduls_gpu_set_host_cache.argtypes = [C.c_int]
        L.raduls_gpu_set_pivots.argtypes = [_u32, _vp, _vp, _u32]
        L.raduls_gpu_check_report.argtypes = [_u64p]
        L.raduls_gpu_sort_segments.argtypes = [_vp, _vp, _u64, _u32, _u32, _u32, _u64p, _vp, _vp]
        L.raduls_gpu_digit_andor.argtypes = [_vp, _u64, _u32, _u32, _u32, _vp, _u32, _vp, _u64p, _vp]
        L.raduls_gpu_partition_store_pieces.argtypes = [_vp, _u64, _u32, _u32, _u32, _vp, _u64p, _u64p,
                                                        _vp]
        L.raduls_gpu_sort_multi.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(_vp), _u64p,
                                            C.POINTER(_vp), _u64p, _u64, _u32, _u32]
        L.raduls_gpu_last_kernel_times.argtypes = [C.POINTER(KernelTime), C.c_int,
                                                   C.POINTER(C.c_int)]
        _lib = L
        return L


def strerror(code: int) -> str:
    return load().raduls_gpu_strerror(code).decode()
