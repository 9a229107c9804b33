"""Local-sort edge cases around the bucket geometry (k_local: 2^B buckets
spread over [min window, max window] by a multiplier every thread computes
in float, rounded down so that buckets stay monotone and below 2^B).

Single-group inputs (n <= the local capacity, so the whole input is one
local sort) with window ranges at the boundaries of the identity / multiplier
paths and at the full 32-bit range; each compared with the oracle's stable
sort byte for byte.
"""
import numpy as np
import pytest

import oracle
from helpers import from_dev, make_input, to_dev

pytestmark = pytest.mark.gpu


def _run(rg, torch, a, rs, ks):
    d = to_dev(torch, a)
    rg.sort(d, a.size // rs, rg.RecordLayout(rs, ks))
    torch.cuda.synchronize()
    got = from_dev(d)
    want = oracle.stable_sort(a, rs, ks)
    assert np.array_equal(got, want), f"mismatch (rs={rs} ks={ks} n={a.size // rs})"


def _set_window(a, rs, vals):
    """Key bytes 0..3 (the window at p = 0) <- big-endian vals."""
    n = a.size // rs
    r = a.reshape(n, rs)
    r[:, 0:4] = np.asarray(vals, dtype=">u4").view(np.uint8).reshape(n, 4)


@pytest.mark.parametrize("rs,ks,n", [(16, 8, 3000), (16, 8, 3584), (24, 16, 2500), (32, 24, 4600),
                                     (8, 8, 18000)])
@pytest.mark.parametrize("span", ["nbk-1", "nbk", "nbk+1", "full", "full-1", "tiny"])
def test_window_range_boundaries(rg, torch_cuda, rs, ks, n, span):
    a = make_input(n, rs, ks, 0xB0C + n + rs)
    B = min(int(np.ceil(np.log2(n))) + 1, 15 if rs == 8 else 13)
    nbk = 1 << B
    rng = np.random.default_rng(n * 7 + rs)
    if span == "full":
        lo, hi = 0, 0xFFFFFFFF
    elif span == "full-1":
        lo, hi = 1, 0xFFFFFFFF
    elif span == "tiny":
        lo, hi = 0x12345678, 0x12345679
    else:
        rm1 = {"nbk-1": nbk - 1, "nbk": nbk, "nbk+1": nbk + 1}[span]
        lo = 0x7FFF0000
        hi = lo + rm1
    w = rng.integers(lo, hi + 1, size=n, dtype=np.uint64)
    w[0], w[-1] = lo, hi  # the range's ends are present
    _set_window(a, rs, w.astype(np.uint32))
    _run(rg, torch_cuda, a, rs, ks)


def test_window_clusters_at_both_ends(rg, torch_cuda):
    """Half the windows at 0, half at 0xFFFFFFFF: two crowded buckets (the
    LSD fallback instance) next to empty ones."""
    rs, ks, n = 16, 8, 3000
    a = make_input(n, rs, ks, 77)
    w = np.where(np.arange(n) % 2 == 0, 0, 0xFFFFFFFF).astype(np.uint32)
    _set_window(a, rs, w)
    _run(rg, torch_cuda, a, rs, ks)
