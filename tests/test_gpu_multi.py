"""raduls_gpu_sort_multi (one process, G devices) against the oracle.

This run has one GPU, so the device is listed G times: every phase of the
multi-device plan (global constant prefix, 16-bit prefix histograms, the
count-balanced bucket map, stable partition, peer-copy exchange, local sort)
runs with G ranks; the phases meet only at host joins, so no kernel waits on
another rank. The per-device counts are checked against the Python plan
(distributed.balanced_bucket_map), which the gloo tests pin independently.
"""
import numpy as np
import pytest

import oracle
from helpers import from_dev, make_input, to_dev

from paper_1612_02557_b200 import distributed as D

pytestmark = pytest.mark.gpu


def expected_counts(parts, rs, ks, G):
    allr = np.concatenate([p.reshape(-1, rs) for p in parts])
    ao = np.zeros((1, 8), dtype=np.uint64)
    if allr.size:
        words = allr.view("<u8") if rs % 8 == 0 else None
        for w in range(rs // 8):
            ao[0, 2 * w] = np.bitwise_and.reduce(words[:, w])
            ao[0, 2 * w + 1] = np.bitwise_or.reduce(words[:, w])
    else:
        ao[0, 0::2] = np.uint64(2**64 - 1)
    p0 = D.first_varying_byte(ao, ks)
    if p0 >= ks:
        p0 = 0
    hi = allr[:, p0].astype(np.int64) if p0 < ks else np.zeros(len(allr), np.int64)
    lo = allr[:, p0 + 1].astype(np.int64) if p0 + 1 < ks else np.zeros(len(allr), np.int64)
    hist = np.bincount((hi << 8) | lo, minlength=D.NBUCKETS)
    bmap = D.balanced_bucket_map(hist, G)
    return np.bincount(bmap[(hi << 8) | lo], minlength=G)


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("rs,ks,universe", [(16, 8, 0), (32, 24, 5000), (8, 8, 300), (24, 16, 0)])
def test_sort_multi_equals_stable_sort_of_concatenation(rg, torch_cuda, G, rs, ks, universe):
    rng = np.random.default_rng(G * 100 + rs)
    sizes = [int(x) for x in rng.integers(0, 60000, size=G)]
    if G > 1:
        sizes[1] = 0  # an empty device
    parts = [make_input(n, rs, ks, 1000 * G + i + rs, universe=universe) for i, n in enumerate(sizes)]
    outs, counts = D.sort_multi([to_dev(torch_cuda, p) for p in parts], rg.RecordLayout(rs, ks))
    got = np.concatenate([from_dev(o)[:c * rs] for o, c in zip(outs, counts)])
    want = oracle.stable_sort(np.concatenate(parts), rs, ks)
    assert np.array_equal(got, want)
    assert counts == list(expected_counts(parts, rs, ks, G))


def test_sort_multi_skewed_and_balanced(rg, torch_cuda):
    """C3-shaped keys (three constant leading bytes): the plan starts at the
    first globally varying byte; uniform keys split evenly over the devices."""
    rs, ks, G = 16, 8, 4
    parts = [make_input(50000, rs, ks, 0x5EED0003 + i, dist=oracle.DIST_SKEW) for i in range(G)]
    outs, counts = D.sort_multi([to_dev(torch_cuda, p) for p in parts], rg.RecordLayout(rs, ks))
    got = np.concatenate([from_dev(o)[:c * rs] for o, c in zip(outs, counts)])
    assert np.array_equal(got, oracle.stable_sort(np.concatenate(parts), rs, ks))
    parts = [make_input(100000, rs, ks, 77 + i) for i in range(G)]
    outs, counts = D.sort_multi([to_dev(torch_cuda, p) for p in parts], rg.RecordLayout(rs, ks))
    assert sum(counts) == 400000 and max(counts) < 1.05 * 100000 and min(counts) > 0.95 * 100000


def test_sort_multi_capacity_too_small_writes_nothing(rg, torch_cuda):
    rs, ks = 16, 8
    parts = [make_input(10000, rs, ks, 5 + i) for i in range(2)]
    with pytest.raises(ValueError):
        D.sort_multi([to_dev(torch_cuda, p) for p in parts], rg.RecordLayout(rs, ks), capacity=5000)
