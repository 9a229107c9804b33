"""GPU parity of the digit array (levels histogrammed from the key byte the
previous scatter wrote, 1 byte per record instead of the whole record).

Every case is checked against the oracle's stable sort byte for byte, with
the digit array on (default) and off (RADULS_GPU_NO_DIGIT_ARRAY), and the
accounting says which levels read the digit array. The constant-byte cases
cover the planner's digit-array branch (k_plan: constancy read off the digit
totals; the segment re-queued at p + 1, the next level reading whole records).
"""
import numpy as np
import pytest

import oracle
from helpers import from_dev, make_input, to_dev

pytestmark = pytest.mark.gpu


def _sort(rg, torch, a, rs, ks):
    d = to_dev(torch, a)
    rg.sort(d, a.size // rs, rg.RecordLayout(rs, ks))
    torch.cuda.synchronize()
    return from_dev(d), rg.last_stats()


def _check(rg, torch, monkeypatch, a, rs, ks, expect_digit_levels=True):
    want = oracle.stable_sort(a, rs, ks)
    got, st = _sort(rg, torch, a, rs, ks)
    assert np.array_equal(got, want), f"digit array on: mismatch (rs={rs} ks={ks})"
    if expect_digit_levels:
        assert st["hist_digit_records"] > 0, st
    monkeypatch.setenv("RADULS_GPU_NO_DIGIT_ARRAY", "1")
    got2, st2 = _sort(rg, torch, a, rs, ks)
    monkeypatch.delenv("RADULS_GPU_NO_DIGIT_ARRAY")
    assert st2["hist_digit_records"] == 0
    assert np.array_equal(got2, want), f"digit array off: mismatch (rs={rs} ks={ks})"
    return st


@pytest.mark.parametrize("rs,ks,n", [(8, 8, 1 << 24), (16, 8, 1 << 21), (16, 16, 1 << 21),
                                     (24, 24, 1 << 20), (32, 24, 1 << 21), (32, 8, 1 << 21)])
def test_uniform_levels_read_the_digit_array(rg, torch_cuda, monkeypatch, rs, ks, n):
    a = make_input(n, rs, ks, 0xD16 + rs + ks)
    st = _check(rg, torch_cuda, monkeypatch, a, rs, ks)
    # every level after the first reads 1 byte per record
    assert st["hist_records"] == n, st


def test_constant_byte_after_a_split(rg, torch_cuda, monkeypatch):
    """Byte 0 takes 4 values, byte 1 is constant: the level on byte 1 sees one
    populated digit in the digit array and re-queues every segment at byte 2."""
    rs, ks, n = 16, 8, 1 << 20
    a = make_input(n, rs, ks, 41)
    r = a.reshape(n, rs)
    r[:, 0] &= 3
    r[:, 1] = 0x5A
    st = _check(rg, torch_cuda, monkeypatch, a, rs, ks)
    assert st["skipped_levels"] >= 4, st


def test_constant_last_key_byte_in_the_digit_array(rg, torch_cuda, monkeypatch):
    """ks = 2 and byte 1 constant: the digit-array level finds every key of a
    segment equal (finished where it lies, copied home from tmp)."""
    rs, ks, n = 16, 2, 1 << 18
    a = make_input(n, rs, ks, 42)
    r = a.reshape(n, rs)
    r[:, 0] &= 3
    r[:, 1] = 0x11
    st = _check(rg, torch_cuda, monkeypatch, a, rs, ks)
    assert st["copy_records"] > 0, st


def test_last_key_byte_split_from_the_digit_array(rg, torch_cuda, monkeypatch):
    rs, ks, n = 16, 2, 1 << 18
    a = make_input(n, rs, ks, 43)
    a.reshape(n, rs)[:, 0] &= 7
    _check(rg, torch_cuda, monkeypatch, a, rs, ks)


def test_mixed_level_falls_back_to_record_histograms(rg, torch_cuda, monkeypatch):
    """One segment's next byte is constant, the other's varies: the level after
    that mixes a re-queued segment with split ones and reads whole records."""
    rs, ks, n = 16, 8, 1 << 20
    a = make_input(n, rs, ks, 44)
    r = a.reshape(n, rs)
    r[:, 0] &= 1
    r[r[:, 0] == 0, 1] = 0x77
    st = _check(rg, torch_cuda, monkeypatch, a, rs, ks)
    assert st["skipped_levels"] >= 1, st


def test_skewed_c3_shape(rg, torch_cuda, monkeypatch):
    rs, ks = 16, 8
    a = make_input(1 << 21, rs, ks, 0x5EED0003, dist=oracle.DIST_SKEW)
    _check(rg, torch_cuda, monkeypatch, a, rs, ks)


def test_duplicate_heavy_digit_levels(rg, torch_cuda, monkeypatch):
    """Few distinct keys: large equal-key segments through digit-array levels."""
    rs, ks, n = 16, 8, 1 << 20
    a = make_input(n, rs, ks, 45, universe=1000)
    _check(rg, torch_cuda, monkeypatch, a, rs, ks, expect_digit_levels=False)
