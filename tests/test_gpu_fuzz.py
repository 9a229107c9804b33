"""Seeded randomized inputs across layouts, sizes and key shapes — each compared
byte for byte with the oracle's stable sort (P/src/verify.cpp:52-64). The
shapes aim at the seams of the small-bin chain (bitmap sort -> big instance ->
bucket sort -> LSD): duplicate rates from none to all-equal, constant and
low-entropy bytes at random key positions, sorted / reversed / nearly sorted
input, sizes around the group capacities.
"""
import numpy as np
import pytest

import oracle
from helpers import from_dev, make_input, to_dev

pytestmark = pytest.mark.gpu

LAYOUTS = [(8, 8), (8, 3), (16, 8), (16, 16), (16, 5), (24, 16), (24, 24), (32, 24), (32, 8), (32, 32)]


def _shape(rng, a, n, rs, ks):
    """Mutate the keys of `a` in place into one of several shapes; returns its name."""
    r = a.reshape(n, rs)
    kind = rng.integers(0, 9)
    if kind == 0:
        return "uniform"
    if kind == 1:  # every key one of u values
        u = int(rng.choice([1, 2, 7, 64, 1000, max(2, n // 3), n]))
        pick = r[rng.integers(0, min(u, n), size=n), :ks].copy()
        r[:, :ks] = pick
        return f"universe{u}"
    if kind == 2:  # some key bytes constant
        for b in rng.choice(ks, size=rng.integers(1, ks + 1), replace=False):
            r[:, b] = rng.integers(0, 256)
        return "constant-bytes"
    if kind == 3:  # low-entropy bytes (few values per byte)
        for b in range(ks):
            vals = rng.integers(0, 256, size=rng.integers(1, 5)).astype(np.uint8)
            r[:, b] = vals[rng.integers(0, vals.size, size=n)]
        return "low-entropy"
    if kind in (4, 5, 6):  # sorted / reversed / nearly sorted
        order = np.lexsort(tuple(r[:, b] for b in range(ks - 1, -1, -1)))
        s = r[order].copy()
        if kind == 5:
            s = s[::-1].copy()
        if kind == 6:
            for _ in range(max(1, n // 50)):
                i, j = rng.integers(0, n, size=2)
                s[[i, j]] = s[[j, i]]
        r[:] = s
        return ["sorted", "reversed", "nearly-sorted"][kind - 4]
    if kind == 7:  # keys equal in the first bytes, differing late (beyond a 4-byte window)
        cut = int(rng.integers(0, ks))
        r[:, :cut] = rng.integers(0, 256)
        return f"late-varying{cut}"
    # kind 8: a hot key among uniform ones
    hot = rng.random(n) < rng.choice([0.1, 0.5, 0.9])
    r[hot, :ks] = r[0, :ks]
    return "hot-key"


@pytest.mark.parametrize("case", range(72))
def test_random_shapes_match_the_oracle(rg, torch_cuda, case):
    rng = np.random.default_rng(0xF022 + case)
    rs, ks = LAYOUTS[case % len(LAYOUTS)]
    cap = rg.local_capacity(rs)
    n = int(rng.choice([2, 17, 255, 2047, 2049, cap - 1, cap, cap + 1, 2 * cap + 5, 20_000, 70_000,
                        150_000, 400_000]))
    a = make_input(n, rs, ks, 0xF0220000 + case)
    name = _shape(rng, a, n, rs, ks)
    d = to_dev(torch_cuda, a)
    rg.sort(d, n, rg.RecordLayout(rs, ks))
    torch_cuda.cuda.synchronize()
    got = from_dev(d)
    want = oracle.stable_sort(a, rs, ks)
    assert np.array_equal(got, want), f"case {case}: rs={rs} ks={ks} n={n} shape={name}"
