"""Python mirror of the reference's public sort interface, backed by the
B200 C-ABI (include/raduls_gpu.h).

Reference names kept (P = /root/reference/proj):

* ``RecordLayout``     — P/include/raduls/layout.hpp:16-28 (widened: any
  key_size in [1, record_size]; the reference takes 8 or 16 only).
* ``SchedulerConfig``  — P/include/raduls/scheduler.hpp:23-32. Accepted for
  signature compatibility; its knobs steer CPU thread scheduling only and
  never change output (P/tests/test_scheduler.cpp:171-177), so the GPU path
  ignores them.
* ``sort(data, n, layout, cfg)`` — P/include/raduls/scheduler.hpp:60-65.
  ``data`` may be a CUDA ``torch.uint8`` tensor (sorted in place on the
  device) or host memory (numpy array / bytearray / ``RecordArray``; sorted in
  place through H2D -> device sort -> D2H).
* ``LsdConfig`` / ``lsd_sort(data, n, layout, cfg)`` — the reference's LSD
  baseline, P/include/raduls/lsd.hpp:12-22 (stable; equals ``sort``'s output).
* errors: ``ValueError`` for unsupported layouts (the reference's
  ``std::invalid_argument``, dispatch.hpp:37-39), ``ResourceError`` (a
  ``MemoryError``; the reference's ``raduls::resource_error``,
  errors.hpp:12-22), ``CudaError`` for device failures.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = [
    "RecordLayout", "SchedulerConfig", "TinyPolicy", "BigBinFraction", "ResourceError",
    "CudaError", "sort", "sort_device", "split", "histogram", "generate", "digest",
    "check_sorted", "last_stats", "DIST_UNIFORM", "DIST_SKEW", "local_capacity",
    "set_profiling", "last_kernel_times", "LsdConfig", "lsd_sort", "rank_mode", "launch_count", "set_host_cache",
]

DIST_UNIFORM = 0
DIST_SKEW = 1


class ResourceError(MemoryError):
    """Device or pinned memory could not be allocated; the input is untouched."""


class CudaError(RuntimeError):
    """A CUDA runtime call inside the library failed."""


@dataclass(frozen=True)
class RecordLayout:
    record_size: int = 16
    key_size: int = 8

    def payload_size(self) -> int:
        return self.record_size - self.key_size

    def valid(self) -> bool:
        return bool(_valid(self.record_size, self.key_size))


def _valid(rs: int, ks: int) -> bool:
    return rs in (8, 16, 24, 32) and 1 <= ks <= rs


@dataclass
class BigBinFraction:
    num: int = 2
    den: int = 3


@dataclass
class TinyPolicy:
    tiny_threshold: int = 384
    insertion_threshold: int = 32
    narrowing_factor_limit: int = 16
    narrowed_tiny_threshold: int = 32
    intro_vs_shell_override: int = 0


@dataclass
class SchedulerConfig:
    threads: int = 1
    l2_cache_bytes: int = 262144
    big_bin_threshold: BigBinFraction = field(default_factory=BigBinFraction)
    queue_cutoff_divisor: int = 4096
    chunk_multiplier: int = 8
    first_chunk_divisor: int = 64
    buffer_bytes: int = 256
    tiny: TinyPolicy = field(default_factory=TinyPolicy)


@dataclass
class LsdConfig:
    """P/include/raduls/lsd.hpp:12-15. ``buffer_bytes_per_digit`` (write-
    combining lane size) must be a positive multiple of 64 as in the reference
    (lsd.cpp:13-14); like ``threads`` it steers the CPU scatter only."""
    buffer_bytes_per_digit: int = 64
    threads: int = 1


def _raise(rc: int, what: str) -> None:
    if rc == _lib.OK:
        return
    msg = f"{what}: {_lib.strerror(rc)}"
    if rc == _lib.EINVAL:
        raise ValueError(msg)
    if rc == _lib.ENOMEM:
        raise ResourceError(msg)
    raise CudaError(msg)


def _layout_error(layout: RecordLayout) -> ValueError:
    return ValueError(f"unsupported record layout: record_size={layout.record_size} "
                      f"key_size={layout.key_size}")


def _torch():
    import torch  # noqa: PLC0415  (torch is plumbing: device memory + streams)
    return torch


def _is_cuda_tensor(x) -> bool:
    try:
        torch = _torch()
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _check_device_tensor(data, tmp) -> None:
    """uint8, contiguous, and tmp on data's device: n counts bytes / rs, and
    the library reads the tensor's memory from data_ptr() on."""
    torch = _torch()
    for name, t in (("data", data), ("tmp", tmp)):
        if t is None:
            continue
        if t.dtype != torch.uint8:
            raise TypeError(f"{name} must be a torch.uint8 tensor (got {t.dtype})")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    if tmp is not None and tmp.device != data.device:
        raise ValueError("tmp must be on data's device")


def _stream_ptr(stream, device=None) -> int | None:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream(device).cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def sort_device(d_data: int, d_tmp: int | None, n: int, layout: RecordLayout,
                stream: int | None = None) -> None:
    """Raw device-pointer entry (raduls_gpu_sort)."""
    if not layout.valid():
        raise _layout_error(layout)
    rc = _lib.load().raduls_gpu_sort(d_data, d_tmp, n, layout.record_size, layout.key_size,
                                     stream)
    _raise(rc, "raduls_gpu_sort")


def sort(data, n: int | None = None, layout: RecordLayout = RecordLayout(),
         cfg: SchedulerConfig | None = None, *, tmp=None, stream=None) -> None:
    """Sort ``n`` fixed-size records in place, non-decreasing by key.

    Mirrors ``raduls::sort(uint8_t* data, size_t n, const RecordLayout&,
    const SchedulerConfig&)``. ``tmp`` (device tensor of the same byte size)
    is the optional caller-owned scratch of the C-ABI.
    """
    if not layout.valid():
        raise _layout_error(layout)
    rs = layout.record_size
    if hasattr(data, "layout") and hasattr(data, "buf") and n is None:  # RecordArray
        return sort(data.buf, data.n, data.layout, cfg, tmp=tmp, stream=stream)
    if _is_cuda_tensor(data):
        _check_device_tensor(data, tmp)
        if n is None:
            n = data.numel() // rs
        if data.numel() < n * rs:
            raise ValueError("data holds fewer than n records")
        tptr = tmp.data_ptr() if tmp is not None else None
        if tmp is not None and tmp.numel() < n * rs:
            raise ValueError("tmp holds fewer than n records")
        torch = _torch()
        with torch.cuda.device(data.device):  # the library works on the current device
            st = _stream_ptr(stream, data.device)
            rc = _lib.load().raduls_gpu_sort(data.data_ptr(), tptr, n, rs, layout.key_size, st)
        _raise(rc, "raduls_gpu_sort")
        return None
    # host memory
    if isinstance(data, (bytearray, memoryview)):
        arr = np.frombuffer(data, dtype=np.uint8)
    else:
        arr = data
    if not isinstance(arr, np.ndarray) or arr.dtype != np.uint8 or not arr.flags["C_CONTIGUOUS"]:
        raise TypeError("host data must be a C-contiguous uint8 buffer")
    if n is None:
        n = arr.size // rs
    if arr.size < n * rs:
        raise ValueError("data holds fewer than n records")
    if not arr.flags["WRITEABLE"]:
        raise ValueError("host data is read-only")
    rc = _lib.load().raduls_gpu_sort_host(arr.ctypes.data, None, n, rs, layout.key_size)
    _raise(rc, "raduls_gpu_sort_host")
    return None


def last_stats() -> dict:
    s = _lib.Stats()
    _raise(_lib.load().raduls_gpu_last_stats(C.byref(s)), "raduls_gpu_last_stats")
    return s.as_dict()


def rank_mode() -> int:
    """The scatter's in-warp ranking on this device (raduls_gpu_rank_mode):
    0 = shared-memory atomics, used after the device self-test confirmed they
    are served in lane order; 1 = ballot ranking. The sort is stable either way."""
    m = C.c_int(-1)
    _raise(_lib.load().raduls_gpu_rank_mode(C.byref(m)), "raduls_gpu_rank_mode")
    return m.value


def set_host_cache(on: bool) -> None:
    """Keep the host drop-in's device staging buffers between calls
    (raduls_gpu_set_host_cache); off (default) frees them before each call returns."""
    _raise(_lib.load().raduls_gpu_set_host_cache(1 if on else 0), "raduls_gpu_set_host_cache")


def launch_count() -> int:
    """Kernel launches made by libraduls_gpu.so in this process so far."""
    c = C.c_uint64(0)
    _raise(_lib.load().raduls_gpu_launch_count(C.byref(c)), "raduls_gpu_launch_count")
    return c.value


def set_profiling(on: bool) -> None:
    """Per-kernel CUDA-event timing of subsequent sorts (raduls_gpu_set_profiling)."""
    _raise(_lib.load().raduls_gpu_set_profiling(1 if on else 0), "raduls_gpu_set_profiling")


def last_kernel_times() -> dict:
    """{kernel class: (launches, ms)} of the most recent sort (profiling on)."""
    buf = (_lib.KernelTime * 16)()
    cnt = C.c_int(0)
    _raise(_lib.load().raduls_gpu_last_kernel_times(buf, 16, C.byref(cnt)),
           "raduls_gpu_last_kernel_times")
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].ms))
            for i in range(min(cnt.value, 16))}


def split(src, dst, n: int, record_size: int, key_byte_offset: int, stream=None) -> np.ndarray:
    """One stable single-digit split (reference radix_split, kernels.hpp:157-167).
    Returns the 256-entry digit histogram."""
    h = np.zeros(256, dtype=np.uint64)
    rc = _lib.load().raduls_gpu_split(src.data_ptr(), dst.data_ptr(), n, record_size,
                                      key_byte_offset, h.ctypes.data_as(_lib._u64p),
                                      _stream_ptr(stream))
    _raise(rc, "raduls_gpu_split")
    return h


def histogram(data, n: int, layout: RecordLayout, stream=None) -> tuple[np.ndarray, np.ndarray]:
    """Histograms of key bytes 0..min(ks,8)-1 ([8,256] u64) and the AND/OR of
    every 64-bit record word ([8] u64: and at 2w, or at 2w+1)."""
    h = np.zeros((8, 256), dtype=np.uint64)
    ao = np.zeros(8, dtype=np.uint64)
    rc = _lib.load().raduls_gpu_histogram(data.data_ptr(), n, layout.record_size,
                                          layout.key_size, h.ctypes.data_as(_lib._u64p),
                                          ao.ctypes.data_as(_lib._u64p), _stream_ptr(stream))
    _raise(rc, "raduls_gpu_histogram")
    return h, ao


def generate(n: int, layout: RecordLayout, dist: int = DIST_UNIFORM, seed: int = 1,
             index_base: int = 0, out=None, device=None, stream=None):
    """Device generator of SURVEY.md §8(d); returns a CUDA uint8 tensor."""
    torch = _torch()
    if out is None:
        out = torch.empty(n * layout.record_size, dtype=torch.uint8,
                          device=device if device is not None else "cuda")
    rc = _lib.load().raduls_gpu_generate(out.data_ptr(), n, layout.record_size, layout.key_size,
                                         dist, seed, index_base, _stream_ptr(stream))
    _raise(rc, "raduls_gpu_generate")
    return out


def digest(data, n: int, record_size: int, stream=None) -> tuple[int, int]:
    lo, hi = C.c_uint64(), C.c_uint64()
    rc = _lib.load().raduls_gpu_digest(data.data_ptr(), n, record_size, C.byref(lo),
                                       C.byref(hi), _stream_ptr(stream))
    _raise(rc, "raduls_gpu_digest")
    return lo.value, hi.value


def check_sorted(data, n: int, layout: RecordLayout, stream=None) -> tuple[int, int]:
    """(number of adjacent inversions, first inversion index or 2**64-1)."""
    v, f = C.c_uint64(), C.c_uint64()
    rc = _lib.load().raduls_gpu_check_sorted(data.data_ptr(), n, layout.record_size,
                                             layout.key_size, C.byref(v), C.byref(f),
                                             _stream_ptr(stream))
    _raise(rc, "raduls_gpu_check_sorted")
    return v.value, f.value


# Local-sort group capacity per record size (mirrors local_cap<RS>() in
# csrc/raduls_gpu.cu; used by tests to aim at boundaries).
_LOCAL_CAP = {8: 18432, 16: 3584, 24: 2560, 32: 4608}


def local_capacity(record_size: int) -> int:
    return _LOCAL_CAP[record_size]


# Scatter / histogram tile per record size (mirrors ScatterCfg<RS>::kTile in
# csrc/k_scatter.cuh; tests aim at its boundaries).
_SCATTER_TILE = {8: 5120, 16: 2816, 24: 1792, 32: 1536}


def scatter_tile(record_size: int) -> int:
    return _SCATTER_TILE[record_size]


def _host_records(data, n, rs):
    if isinstance(data, (bytearray, memoryview)):
        arr = np.frombuffer(data, dtype=np.uint8)
    else:
        arr = data
    if not isinstance(arr, np.ndarray) or arr.dtype != np.uint8 or not arr.flags["C_CONTIGUOUS"]:
        raise TypeError("host data must be a C-contiguous uint8 buffer")
    if n is None:
        n = arr.size // rs
    if arr.size < n * rs:
        raise ValueError("data holds fewer than n records")
    if not arr.flags["WRITEABLE"]:
        raise ValueError("host data is read-only")
    return arr, n


def lsd_sort(data, n: int | None = None, layout: RecordLayout = RecordLayout(),
             cfg: LsdConfig | None = None, *, tmp=None, stream=None) -> None:
    """Stable LSD radix sort (``raduls::lsd_sort``, P/src/lsd.cpp:12-35) on the
    device: one stable byte split per key byte, least significant first
    (raduls_gpu_lsd_sort / raduls_gpu_lsd_sort_host). Same arguments and
    errors as ``sort``."""
    cfg = cfg or LsdConfig()
    if cfg.buffer_bytes_per_digit <= 0 or cfg.buffer_bytes_per_digit % 64:
        raise ValueError("LSD buffer size must be a positive multiple of 64 bytes")
    if not layout.valid():
        raise _layout_error(layout)
    rs = layout.record_size
    if hasattr(data, "layout") and hasattr(data, "buf") and n is None:  # RecordArray
        return lsd_sort(data.buf, data.n, data.layout, cfg, tmp=tmp, stream=stream)
    if _is_cuda_tensor(data):
        _check_device_tensor(data, tmp)
        if n is None:
            n = data.numel() // rs
        if data.numel() < n * rs:
            raise ValueError("data holds fewer than n records")
        if tmp is not None and tmp.numel() < n * rs:
            raise ValueError("tmp holds fewer than n records")
        tptr = tmp.data_ptr() if tmp is not None else None
        torch = _torch()
        with torch.cuda.device(data.device):
            rc = _lib.load().raduls_gpu_lsd_sort(data.data_ptr(), tptr, n, rs, layout.key_size,
                                                 _stream_ptr(stream, data.device))
        _raise(rc, "raduls_gpu_lsd_sort")
        return None
    arr, n = _host_records(data, n, rs)
    rc = _lib.load().raduls_gpu_lsd_sort_host(arr.ctypes.data, None, n, rs, layout.key_size)
    _raise(rc, "raduls_gpu_lsd_sort_host")
    return None
