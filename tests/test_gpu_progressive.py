"""Host drop-in with pinned buffers: the progressive sort (level 0 over the
whole array, then its children in key-range batches, each range copied back
to the host as soon as it is final while later ranges are still sorted).

RADULS_GPU_PROGRESSIVE_BYTES=0 forces it at test sizes; each case is checked
byte for byte against the oracle's stable sort, and against the same sort
with the progressive path off."""
import numpy as np
import pytest

import oracle
from helpers import make_input

pytestmark = pytest.mark.gpu


def _pinned_sort(rg, torch, a, rs, ks):
    pin = torch.empty(a.size, dtype=torch.uint8, pin_memory=True).numpy()
    pin[:] = a
    rg.sort(pin, a.size // rs, rg.RecordLayout(rs, ks))
    return pin.copy(), rg.last_stats()


def _check(rg, torch, monkeypatch, a, rs, ks):
    want = oracle.stable_sort(a, rs, ks)
    monkeypatch.setenv("RADULS_GPU_PROGRESSIVE_BYTES", "0")
    got, st = _pinned_sort(rg, torch, a, rs, ks)
    assert np.array_equal(got, want), f"progressive: mismatch (rs={rs} ks={ks})"
    monkeypatch.setenv("RADULS_GPU_PROGRESSIVE_BYTES", str(1 << 62))
    got2, st2 = _pinned_sort(rg, torch, a, rs, ks)
    assert np.array_equal(got2, want), f"level by level: mismatch (rs={rs} ks={ks})"
    # the same passes either way (batches only reorder the work)
    for k in ("scatter_records", "local_records", "hist_records", "hist_digit_records", "copy_records"):
        assert st[k] == st2[k], (k, st, st2)
    return st


@pytest.mark.parametrize("rs,ks,n", [(16, 8, 1 << 20), (8, 8, 1 << 23), (32, 24, 1 << 20),
                                     (24, 16, 1 << 20), (16, 16, 3_000_017)])
def test_progressive_uniform(rg, torch_cuda, monkeypatch, rs, ks, n):
    a = make_input(n, rs, ks, 0x9A0 + rs + n % 97)
    _check(rg, torch_cuda, monkeypatch, a, rs, ks)


def test_progressive_skewed_c3_shape(rg, torch_cuda, monkeypatch):
    """Constant leading bytes, Zipf byte: level 0 at byte 3, big and small
    children interleaved (small ones finished at level 0, inside the ranges)."""
    rs, ks = 16, 8
    a = make_input(1 << 21, rs, ks, 0x5EED0003, dist=oracle.DIST_SKEW)
    _check(rg, torch_cuda, monkeypatch, a, rs, ks)


def test_progressive_duplicates_and_equal_keys(rg, torch_cuda, monkeypatch):
    rs, ks, n = 16, 8, 1 << 20
    _check(rg, torch_cuda, monkeypatch, make_input(n, rs, ks, 5, universe=700), rs, ks)
    a = make_input(n, rs, ks, 6)
    a.reshape(n, rs)[:, :ks] = 9  # every key equal: level 0 finishes everything
    _check(rg, torch_cuda, monkeypatch, a, rs, ks)


def test_progressive_few_children(rg, torch_cuda, monkeypatch):
    """Byte 0 takes 3 values: fewer level-0 children than batches."""
    rs, ks, n = 16, 8, 1 << 20
    a = make_input(n, rs, ks, 7)
    a.reshape(n, rs)[:, 0] %= 3
    _check(rg, torch_cuda, monkeypatch, a, rs, ks)
