"""Host record arrays and raw record files.

Mirrors (P = /root/reference/proj):

* ``RecordArray`` — P/include/raduls/record_array.hpp:15-61: an owning,
  contiguous buffer of ``n`` records of one layout (here a numpy uint8 array,
  64-B aligned like the reference's ``allocate_record_bytes``).
* ``load_file`` / ``save_file`` — P/src/datagen.cpp:120-144: raw header-less
  files of back-to-back records. ``load_file`` raises ``ValueError`` for an
  unsupported layout (``std::invalid_argument``), ``IoError`` when the file
  cannot be opened or read (``raduls::io_error``, errors.hpp:16-19) and
  ``FormatError`` when its length is not a multiple of the record size
  (``raduls::format_error``, errors.hpp:20-23).
"""
from __future__ import annotations

import os

import numpy as np

from .raduls import RecordLayout, _layout_error

__all__ = ["RecordArray", "IoError", "FormatError", "load_file", "save_file"]


class IoError(OSError):
    """A record file could not be opened, read or written."""


class FormatError(ValueError):
    """A record file's length is not a multiple of the record size."""


def _aligned_bytes(nbytes: int, align: int = 64) -> np.ndarray:
    raw = np.empty(nbytes + align, dtype=np.uint8)
    off = (-raw.ctypes.data) % align
    return raw[off:off + nbytes]


class RecordArray:
    """``n`` records of ``layout`` in one contiguous host buffer (``buf``)."""

    def __init__(self, layout: RecordLayout, n: int = 0, buf: np.ndarray | None = None):
        if not layout.valid():
            raise _layout_error(layout)
        self.layout = layout
        self.n = int(n)
        nbytes = self.n * layout.record_size
        if buf is None:
            buf = _aligned_bytes(nbytes)
        elif buf.dtype != np.uint8 or buf.size != nbytes or not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("buf must be a contiguous uint8 array of n * record_size bytes")
        self.buf = buf

    def size(self) -> int:
        return self.n

    def empty(self) -> bool:
        return self.n == 0

    def byte_size(self) -> int:
        return self.buf.size

    def record(self, i: int) -> np.ndarray:
        rs = self.layout.record_size
        return self.buf[i * rs:(i + 1) * rs]

    def records(self) -> np.ndarray:
        """(n, record_size) view."""
        return self.buf.reshape(self.n, self.layout.record_size)

    def clone(self) -> "RecordArray":
        out = RecordArray(self.layout, self.n)
        out.buf[:] = self.buf
        return out


def load_file(path: str, layout: RecordLayout) -> RecordArray:
    """Read a raw record file (datagen.cpp:120-135)."""
    if not layout.valid():
        raise _layout_error(layout)
    try:
        nbytes = os.path.getsize(path)
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    with f:
        if nbytes % layout.record_size:
            raise FormatError(f"{path}: size {nbytes} is not a multiple of record_size "
                              f"{layout.record_size}")
        out = RecordArray(layout, nbytes // layout.record_size)
        if nbytes and f.readinto(memoryview(out.buf)) != nbytes:
            raise IoError(f"short read from {path}")
    return out


def save_file(path: str, array: RecordArray) -> None:
    """Write the records back to back, no header (datagen.cpp:137-144)."""
    try:
        f = open(path, "wb")
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e
    with f:
        if array.byte_size() and f.write(memoryview(array.buf)) != array.byte_size():
            raise IoError(f"short write to {path}")
