"""The bitmap local sort (csrc/k_local_bm.cuh) and its hand-over chain:

    k_local_bm (groups <= the primary capacity)
         (8-B records: k_local_bm8, records in registers)
      -> k_local_bm_med (single bins above it, 16-B records)
      -> k_local_list   (bucket sort: groups with a crowded bitmap word)
      -> k_local<.., true> (LSD fallback: crowded buckets)

Every case is compared byte for byte with the oracle's stable sort
(P/src/verify.cpp:52-64 oracle_sort); `bitmap_spill_groups` / `fallback_groups`
tell which link of the chain took the groups.
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


def _check(rg, torch, a, rs, ks):
    got, st = _sort(rg, torch, a, rs, ks)
    want = oracle.stable_sort(a, rs, ks)
    assert np.array_equal(got, want), f"mismatch (rs={rs} ks={ks} n={a.size // rs})"
    return st


@pytest.mark.parametrize("rs,ks", [(8, 8), (8, 5), (16, 8), (16, 16), (24, 16), (32, 24), (32, 8)])
@pytest.mark.parametrize("n", [2, 3, 31, 127, 128, 129, 1000, 1279, 1280, 1281, 1728, 2047, 2048, 2049, 2500, 3584, 16384,
                               18432])
def test_single_group_uniform_keys_stay_in_the_bitmap_sort(rg, torch_cuda, rs, ks, n):
    if n > rg.local_capacity(rs):
        pytest.skip("above the local-sort capacity of this record size")
    a = make_input(n, rs, ks, 0xB17 + 13 * n + rs)
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 0 and st["fallback_groups"] == 0, st
    assert st["local_records"] == n, st


@pytest.mark.parametrize("rs,ks", [(8, 8), (16, 8), (24, 16), (32, 24)])
def test_million_uniform_records_no_spill(rg, torch_cuda, rs, ks):
    n = 1 << 20
    a = make_input(n, rs, ks, 0xB17B17 + rs)
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 0, st


@pytest.mark.parametrize("rs,ks", [(8, 8), (16, 8), (24, 16), (32, 24)])
@pytest.mark.parametrize("copies", [2, 3, 8])
def test_every_key_repeated_stays_in_the_dirty_word_lists(rg, torch_cuda, rs, ks, copies):
    """Each key `copies` times: every cell is shared and every word dirty; the
    lists hold all records of a group (8-B records: up to 6144), so the dense
    pass orders them — equal keys in input order (stable) — without the
    bucket sort's LSD fallback."""
    n = 1 << 16
    a = make_input(n, rs, ks, 0xD0B1E + copies + rs)
    r = a.reshape(n, rs)
    base = r[: n // copies, :ks].copy()
    for c in range(copies):
        seg = r[c * (n // copies):(c + 1) * (n // copies)]
        seg[:, :ks] = base[: seg.shape[0]]
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["fallback_groups"] == 0, st
    if rs != 8 and copies <= 3:
        assert st["bitmap_spill_groups"] == 0, st


@pytest.mark.parametrize("rs,ks", [(8, 8), (16, 8)])
def test_sixty_four_copies_of_each_key_crowd_the_words(rg, torch_cuda, rs, ks):
    """64 copies of each key: one cell holds more than 32 records, the group
    is handed to the bucket sort and on to the LSD fallback."""
    n = 1 << 16
    a = make_input(n, rs, ks, 0xC40D + rs)
    r = a.reshape(n, rs)
    base = r[: n // 64, :ks].copy()
    r[:, :ks] = np.tile(base, (64, 1))
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] > 0, st


@pytest.mark.parametrize("rs,ks,n", [(8, 8, 12000), (16, 8, 1500), (16, 8, 3000), (24, 16, 2000),
                                     (32, 24, 4000)])
def test_few_distinct_keys_reach_the_lsd_fallback(rg, torch_cuda, rs, ks, n):
    """One group whose keys differ only in the last key byte (7 values): every
    window is equal, the one shared cell is crowded -> bucket sort -> crowded
    bucket -> LSD fallback."""
    a = make_input(n, rs, ks, 0xFA11 + rs)
    r = a.reshape(n, rs)
    rng = np.random.default_rng(5)
    r[:, :ks] = 0x42
    r[:, ks - 1] = rng.integers(0, 7, size=n).astype(np.uint8)
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 1 and st["fallback_groups"] == 1, st


@pytest.mark.parametrize("rs,ks", [(8, 8), (16, 8), (16, 16), (24, 16), (32, 24)])
def test_shared_cells_resolved_by_bytes_beyond_the_window(rg, torch_cuda, rs, ks):
    """Pairs of records with equal 4-byte windows that differ only in later key
    bytes (and exact duplicates): the dense dirty-word pass must compare the
    rest of the key and then the input index."""
    n = 1500
    a = make_input(n, rs, ks, 0xBE70 + rs)
    r = a.reshape(n, rs)
    rng = np.random.default_rng(11)
    for _ in range(40):
        i, j = rng.integers(0, n, size=2)
        r[j, :4] = r[i, :4]          # same window, later bytes differ
    for _ in range(20):
        i, j = rng.integers(0, n, size=2)
        r[j, :ks] = r[i, :ks]        # exact duplicate keys
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 0, st


def test_key_ends_inside_the_window(rg, torch_cuda):
    """ks - p < 4: the window is shorter than four bytes at the key's end."""
    for ks in (1, 2, 3, 5, 6, 7):
        n = 1200
        a = make_input(n, 16, ks, 0xE0D + ks)
        _check(rg, torch_cuda, a, 16, ks)


def test_medium_bins_take_the_big_instance(rg, torch_cuda):
    """16-B records: bins of ~3000 records (above the primary capacity of 2048,
    within the local-sort capacity) are groups of their own, sorted by the
    big instance over the device-counted list."""
    rs, ks = 16, 8
    bins = 48
    n = bins * 3000
    a = make_input(n, rs, ks, 0x3ED)
    r = a.reshape(n, rs)
    rng = np.random.default_rng(3)
    r[:, 0] = 0
    r[:, 1] = np.repeat(np.arange(bins, dtype=np.uint8), 3000)[rng.permutation(n)]
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 0, st
    assert st["local_records"] == n, st


def test_medium_bins_24_byte_records(rg, torch_cuda):
    """24-B records: bins of ~2000 records (above the primary capacity of 1280,
    within the local-sort capacity of 2560) take the big instance."""
    rs, ks = 24, 16
    bins = 40
    n = bins * 2000
    a = make_input(n, rs, ks, 0x24ED)
    r = a.reshape(n, rs)
    rng = np.random.default_rng(4)
    r[:, 0] = 7
    r[:, 1] = np.repeat(np.arange(bins, dtype=np.uint8), 2000)[rng.permutation(n)]
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 0 and st["local_records"] == n, st


@pytest.mark.parametrize("rs,ks,big,cnt", [(16, 8, 3000, 10), (24, 16, 2000, 10), (32, 24, 3000, 10),
                                            (32, 24, 3000, 200)])
def test_mixed_small_and_medium_bins(rg, torch_cuda, rs, ks, big, cnt):
    """`cnt` bins of `big` records (single-bin groups above the primary capacity)
    among 246 small bins: with few of them the primary instance runs first and
    hands them to the big instance's list; when they are the majority of the
    groups the host launches the big instance over the whole list."""
    small = 246 - cnt if cnt < 246 else 0
    sizes = [big] * cnt + [37] * small
    n = sum(sizes)
    a = make_input(n, rs, ks, 0x317ED + rs + cnt)
    r = a.reshape(n, rs)
    rng = np.random.default_rng(9)
    r[:, 0] = 3
    r[:, 1] = np.repeat(np.arange(len(sizes), dtype=np.uint8), sizes)[rng.permutation(n)]
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] == 0 and st["local_records"] == n, st


def test_clustered_windows_inside_the_digit_range(rg, torch_cuda):
    """The planner hands the group its digit range, so the cell grid spans
    whole digits: windows clustered in a sliver of that range share cells and
    the group goes to the bucket sort (which measures the range itself)."""
    rs, ks = 16, 8
    n = 1 << 16
    a = make_input(n, rs, ks, 0xC1A5)
    r = a.reshape(n, rs)
    r[:, 1:4] = 0x55          # bytes 1..3 constant: byte 0 splits, windows differ in the last byte only
    st = _check(rg, torch_cuda, a, rs, ks)
    assert st["bitmap_spill_groups"] > 0 and st["fallback_groups"] == 0, st


def test_bucket_sort_alone_still_matches(rg, torch_cuda, monkeypatch):
    """RADULS_GPU_LOCAL=bucket: the bucket sort takes every group (the local
    sort before the bitmap sort existed)."""
    monkeypatch.setenv("RADULS_GPU_LOCAL", "bucket")
    for rs, ks, n in [(8, 8, 1 << 18), (16, 8, 1 << 18), (32, 24, 1 << 17), (24, 16, 50000)]:
        a = make_input(n, rs, ks, 0xB0C4 + rs)
        st = _check(rg, torch_cuda, a, rs, ks)
        assert st["bitmap_spill_groups"] == 0, st
