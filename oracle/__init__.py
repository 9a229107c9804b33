"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product package ``paper_1612_02557_b200`` never imports it.

Two libraries:

* ``oracle/liboracle.so`` — the plain-C restatement of the reference hot path
  (``oracle/raduls_oracle.c``; each function cites the reference file:line it
  follows).
* ``oracle/_ref/libraduls_ref.so`` — the unmodified reference library compiled
  from ``/root/reference/proj/src`` by ``oracle/Makefile`` (optional: present
  when it was built in the container that had the reference mounted).

All arrays are numpy ``uint8`` buffers of ``n * rec_size`` bytes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libraduls_ref.so")

_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """Compile the C oracle (and the reference, when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u8p)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_rnd.restype = C.c_uint64
        L.orc_rnd.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
        L.orc_generate.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint64, C.c_uint64]
        L.orc_zipf_thresholds.argtypes = [C.c_double, C.c_uint32, _u64p]
        L.orc_histogram.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p]
        L.orc_exclusive_prefix_sum.argtypes = [_u64p, _u64p]
        L.orc_radix_split.argtypes = [_u8p, _u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p]
        L.orc_msd_sort.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u8p]
        L.orc_comparison_sort.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_is_tiny.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_digest.argtypes = [_u8p, C.c_uint64, C.c_uint32, _u64p, _u64p]
        L.orc_check_sorted.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p]
        L.orc_stable_sort.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_canonicalize.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_load_be64.restype = C.c_uint64
        L.orc_load_be64.argtypes = [_u8p]
        L.orc_store_be64.argtypes = [_u8p, C.c_uint64]
        L.orc_digit.restype = C.c_uint8
        L.orc_digit.argtypes = [_u8p, C.c_uint32, C.c_uint32]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference library itself (oracle/_ref). Raises if it was not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " not built (make -C oracle ref)")
        L = C.CDLL(REF_SO)
        L.ref_sort.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_lsd_sort.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint32]
        L.ref_oracle_sort.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32]
        L.ref_digest.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p, _u64p]
        L.ref_check_sorted.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p]
        L.ref_build_histogram.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          _u64p]
        L.ref_radix_split.argtypes = [_u8p, _u8p, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint32, _u64p]
        L.ref_buffered_split.argtypes = [_u8p, _u8p, C.c_uint64, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_uint32, _u64p]
        L.ref_is_tiny.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_generate.argtypes = [_u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_double, C.c_uint64, C.c_uint64, C.c_uint32]
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        _ref = L
    return _ref


# ---------------------------------------------------------------- numpy helpers

DIST_UNIFORM = 0
DIST_SKEW = 1  # C3: top 24 bits zero, Zipf(1.2) byte, 32 uniform bits


def seed_for_config(c: int) -> int:
    """seed_c = 0x5EED0000 + c (c = 1..5)."""
    return 0x5EED0000 + c


def generate(n: int, rs: int, ks: int, dist: int = DIST_UNIFORM, seed: int = 1,
             index_base: int = 0) -> np.ndarray:
    a = np.empty(n * rs, dtype=np.uint8)
    rc = lib().orc_generate(_ptr(a), n, rs, ks, dist, seed, index_base)
    if rc:
        raise ValueError(f"orc_generate: layout ({rs},{ks}) rejected")
    return a


def msd_sort(a: np.ndarray, rs: int, ks: int) -> np.ndarray:
    """The C restatement of raduls::sort (T = 1); returns a sorted copy."""
    out = a.copy()
    rc = lib().orc_msd_sort(_ptr(out), len(out) // rs, rs, ks, None)
    if rc == 1:
        raise ValueError(f"unsupported record layout: record_size={rs} key_size={ks}")
    if rc:
        raise MemoryError("orc_msd_sort")
    return out


def stable_sort(a: np.ndarray, rs: int, ks: int) -> np.ndarray:
    out = a.copy()
    if lib().orc_stable_sort(_ptr(out), len(out) // rs, rs, ks):
        raise MemoryError("orc_stable_sort")
    return out


def canonical(a: np.ndarray, rs: int, ks: int) -> np.ndarray:
    """Sort each equal-key run by full record bytes; raises if not key-sorted."""
    out = a.copy()
    if not lib().orc_canonicalize(_ptr(out), len(out) // rs, rs, ks):
        raise AssertionError("canonical(): input is not key-sorted")
    return out


def digest(a: np.ndarray, rs: int) -> tuple[int, int]:
    lo, hi = C.c_uint64(), C.c_uint64()
    lib().orc_digest(_ptr(a), len(a) // rs, rs, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def check_sorted(a: np.ndarray, rs: int, ks: int) -> tuple[bool, int]:
    v = C.c_uint64(0)
    ok = lib().orc_check_sorted(_ptr(a), len(a) // rs, rs, ks, C.byref(v))
    return bool(ok), v.value


def histogram(a: np.ndarray, rs: int, byte_offset: int) -> np.ndarray:
    h = np.zeros(256, dtype=np.uint64)
    lib().orc_histogram(_ptr(a), len(a) // rs, rs, byte_offset,
                        h.ctypes.data_as(_u64p))
    return h


def radix_split(a: np.ndarray, rs: int, byte_offset: int) -> tuple[np.ndarray, np.ndarray]:
    out = np.empty_like(a)
    h = np.zeros(256, dtype=np.uint64)
    lib().orc_radix_split(_ptr(a), _ptr(out), len(a) // rs, rs, byte_offset,
                          h.ctypes.data_as(_u64p))
    return out, h


def zipf_thresholds(s: float = 1.2, universe: int = 256) -> np.ndarray:
    t = np.zeros(universe, dtype=np.uint64)
    lib().orc_zipf_thresholds(s, universe, t.ctypes.data_as(_u64p))
    return t


# ---------------------------------------------------------------- reference helpers

def ref_sort(a: np.ndarray, rs: int, ks: int, threads: int = 1) -> np.ndarray:
    """Run the unmodified reference raduls::sort on a copy (oracle/_ref)."""
    out = a.copy()
    rc = ref().ref_sort(_ptr(out), len(out) // rs, rs, ks, threads)
    if rc == 1:
        raise ValueError(f"unsupported record layout: record_size={rs} key_size={ks}")
    if rc:
        raise RuntimeError(f"ref_sort failed rc={rc}")
    return out


def ref_digest(a: np.ndarray, rs: int, ks: int) -> tuple[int, int]:
    lo, hi = C.c_uint64(), C.c_uint64()
    rc = ref().ref_digest(_ptr(a), len(a) // rs, rs, ks, C.byref(lo), C.byref(hi))
    if rc:
        raise ValueError("ref_digest rejected the layout")
    return lo.value, hi.value


def host_cores() -> int:
    """Physical cores, by the method of P/tests/acceptance.cpp:52-66."""
    cores = set()
    phys, core = 0, -1
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("physical id"):
                    phys = int(line.split(":")[1])
                elif line.startswith("core id"):
                    core = int(line.split(":")[1])
                    cores.add((phys, core))
    except OSError:
        pass
    return len(cores) if cores else (os.cpu_count() or 1)
