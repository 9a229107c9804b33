"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar: key sequence bit-exact, equal-key runs the same record
multiset. The GPU sort is stable, so it must equal the oracle's *stable*
sort (oracle_sort, P/src/verify.cpp:52-64) byte for byte, and for distinct
keys it must equal the reference MSD (restated in oracle/raduls_oracle.c)
byte for byte. Patterns follow P/tests/acceptance.cpp:102-166 and
P/tests/test_scheduler.cpp:123-214.
"""
import os

import numpy as np
import pytest

import oracle
from helpers import ALL_LAYOUTS, EXTRA_LAYOUTS, from_dev, make_input, to_dev

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 2, 31, 32, 33, 100, 180, 383, 384, 385, 1000, 100000]


def gpu_sort(rg, torch, a, rs, ks, tmp=False):
    d = to_dev(torch, a)
    t = torch.empty_like(d) if tmp else None
    rg.sort(d, a.size // rs, rg.RecordLayout(rs, ks), tmp=t)
    torch.cuda.synchronize()
    return from_dev(d)


def assert_parity(got, a, rs, ks):
    want = oracle.stable_sort(a, rs, ks)
    if not np.array_equal(got, want):
        n = a.size // rs
        g, w = got.reshape(n, rs), want.reshape(n, rs)
        bad = np.nonzero((g != w).any(axis=1))[0]
        raise AssertionError(f"mismatch at {len(bad)} records, first {bad[:5]} "
                             f"(rs={rs} ks={ks} n={n})")


@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS + EXTRA_LAYOUTS)
def test_oracle_equivalence_sizes(rg, torch_cuda, rs, ks):
    """acceptance.cpp:102-136 pattern: layouts x boundary sizes x universes."""
    seed = 20260809 + rs * 100 + ks
    for i, n in enumerate(SIZES):
        universe = (0, 256, 2)[i % 3]
        a = make_input(n, rs, ks, seed + i, universe)
        got = gpu_sort(rg, torch_cuda, a, rs, ks, tmp=bool(i % 2))
        assert_parity(got, a, rs, ks)


@pytest.mark.parametrize("rs,ks", [(8, 8), (16, 8), (32, 24), (24, 16)])
def test_capacity_boundaries(rg, torch_cuda, rs, ks):
    """Inputs straddling the local-sort capacity and the scatter tile."""
    cap = rg.local_capacity(rs)
    for j, n in enumerate([cap - 1, cap, cap + 1, 2 * cap + 3, 70000]):
        a = make_input(n, rs, ks, 99 + j, (0, 256, 3)[j % 3])
        assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)


def test_distinct_keys_match_reference_msd_bytes(rg, torch_cuda):
    """Distinct keys: byte-identical to the reference MSD (test_scheduler.cpp:171-183)."""
    for rs, ks in ALL_LAYOUTS:
        a = make_input(200000, rs, ks, 555 + rs + ks)
        got = gpu_sort(rg, torch_cuda, a, rs, ks)
        assert np.array_equal(got, oracle.msd_sort(a, rs, ks))


def test_shape_extremes(rg, torch_cuda):
    """test_scheduler.cpp:142-169: all-equal, sorted, reverse, empty."""
    rs, ks = 16, 8
    equal = make_input(50000, rs, ks, 7, universe=1)
    assert np.array_equal(gpu_sort(rg, torch_cuda, equal, rs, ks), equal)  # stable identity
    srt = oracle.stable_sort(make_input(20000, rs, ks, 8), rs, ks)
    assert np.array_equal(gpu_sort(rg, torch_cuda, srt, rs, ks), srt)
    rev = srt.reshape(-1, rs)[::-1].copy().reshape(-1)
    assert_parity(gpu_sort(rg, torch_cuda, rev, rs, ks), rev, rs, ks)
    empty = np.zeros(0, dtype=np.uint8)
    assert gpu_sort(rg, torch_cuda, empty, rs, ks).size == 0


def test_hot_leading_byte(rg, torch_cuda):
    """test_scheduler.cpp:185-202: 80% of keys share the leading byte."""
    rs, ks, n = 16, 8, 300000
    a = make_input(n, rs, ks, 11)
    r = a.reshape(n, rs)
    hot = np.arange(n) % 5 != 0
    r[hot, 0] = 0xAB
    assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)


def test_constant_middle_bytes_skew(rg, torch_cuda):
    """C3-shaped input (leading constant bytes, Zipf byte): exercises (e)."""
    rs, ks = 16, 8
    a = make_input(1 << 20, rs, ks, 0x5EED0003, dist=oracle.DIST_SKEW)
    assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)
    st = rg.last_stats()
    # bytes 0-2 are constant: level 0 starts at byte 3 without moving a record
    # (a sort that split them would scatter every record three extra times)
    n = a.size // rs
    assert st["hist_records"] == n and st["scatter_records"] < 3 * n, st


def test_long_ties_force_fallback(rg, torch_cuda):
    """Keys equal on their first 20 bytes, different in the last 4: the local
    sort's 4-byte window ties and the full-key fallback must order them."""
    rs, ks, n = 32, 24, 9000
    a = make_input(n, rs, ks, 3)
    r = a.reshape(n, rs)
    r[:, 0:20] = 7
    assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)


def test_million_records_digest(rg, torch_cuda):
    """test_scheduler.cpp:204-214: 2^20 records, digest + sortedness on device."""
    rs, ks, n = 16, 8, 1 << 20
    a = make_input(n, rs, ks, 2718)
    d = to_dev(torch_cuda, a)
    before = rg.digest(d, n, rs)
    assert before == oracle.digest(a, rs)
    rg.sort(d, n, rg.RecordLayout(rs, ks))
    assert rg.digest(d, n, rs) == before
    assert rg.check_sorted(d, n, rg.RecordLayout(rs, ks))[0] == 0
    assert_parity(from_dev(d), a, rs, ks)


def test_host_dropin(rg):
    """raduls_gpu_sort_host: the (data, tmp, n, rs, ks) drop-in on host memory."""
    for rs, ks in [(16, 8), (32, 24), (8, 8)]:
        a = make_input(123457, rs, ks, 42 + rs, 1000)
        b = a.copy()
        rg.sort(b, a.size // rs, rg.RecordLayout(rs, ks))
        assert_parity(b, a, rs, ks)


def test_invalid_layouts_raise(rg, torch_cuda):
    buf = torch_cuda.zeros(64, dtype=torch_cuda.uint8, device="cuda")
    for rs, ks in [(8, 16), (12, 8), (40, 8), (16, 0)]:
        with pytest.raises(ValueError):
            rg.sort(buf, 2, rg.RecordLayout(rs, ks))


def test_varying_byte_missed_by_the_sample(rg, torch_cuda):
    """Level 0 guesses the first varying key byte from a strided sample; a more
    significant byte that varies only off the sample must still be honoured."""
    rs, ks, n = 16, 8, 1 << 20
    a = make_input(n, rs, ks, 12)
    r = a.reshape(n, rs)
    r[:, 0] = 0
    r[7, 0] = 1       # off the stride-16 sample
    r[1001, 0] = 2
    assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)


def test_pair_ties_beyond_the_window(rg, torch_cuda):
    """Records whose first four varying key bytes tie in pairs (and in triples)
    but differ further down the key: the local sort's window tie handling."""
    rs, ks = 32, 24
    for n, rep in [(1500, 2), (1500, 3), (4000, 2)]:
        a = make_input(n, rs, ks, 77 + rep)
        r = a.reshape(n, rs)
        r[:, 0:16] = 0
        # groups of `rep` records share bytes 16..19 (a bijective scramble of the
        # group id, so all four bytes vary); bytes 20..23 stay random
        base = (np.arange(n, dtype=np.uint64) // rep * np.uint64(2654435761)) % np.uint64(2**32)
        r[:, 16:20] = base.astype(">u4").view(np.uint8).reshape(n, 4)
        rng = np.random.default_rng(rep)
        r[:] = r[rng.permutation(n)]
        assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)


def test_cpp_dropin_shim(rg):
    """include/raduls_gpu.hpp from C++: raduls::gpu::sort with the reference's
    signature, invalid layouts -> std::invalid_argument (tests/cpp/dropin_main.cpp)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "dropin_main")
    if not os.path.exists(exe):
        import __graft_entry__
        __graft_entry__.build_cpp_dropin()
    for args in (["100000", "16", "8"], ["54321", "32", "24"], ["300000", "8", "8"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


CONFIG_GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "reference_configs.json")


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_size_configs_match_reference_hash(rg, torch_cuda, name):
    """BASELINE configs C1-C4 at full size, generated on the device, against the
    sha256 of the reference's canonical output (tests/golden/make_golden.py
    --configs, reference raduls::sort with T=8; C4 through the exact (32,16)
    proxy). The GPU sort is stable and payload word 0 is the record index, so
    its output is already canonical."""
    import hashlib
    import json
    gold = json.load(open(CONFIG_GOLDEN))[name]
    n, rs, ks, dist, seed = gold["n"], gold["rs"], gold["ks"], gold["dist"], gold["seed"]
    lay = rg.RecordLayout(rs, ks)
    d = rg.generate(n, lay, dist=dist, seed=seed)
    assert list(rg.digest(d, n, rs)) == gold["digest"]
    rg.sort(d, n, lay)
    torch_cuda.cuda.synchronize()
    assert rg.check_sorted(d, n, lay)[0] == 0
    assert list(rg.digest(d, n, rs)) == gold["digest"]
    h = hashlib.sha256()
    step = 1 << 30
    for o in range(0, n * rs, step):
        h.update(memoryview(d[o:o + step].cpu().numpy()))
    del d
    torch_cuda.cuda.empty_cache()
    assert h.hexdigest() == gold["canonical_sha"]


def test_host_dropin_streams_pageable_and_pinned(rg, torch_cuda):
    """raduls_gpu_sort_host on more than the pinned staging ring (5 x 32 MiB
    chunks): pageable buffers stream through staging, pinned ones go direct;
    an odd byte offset exercises 'any alignment' (scheduler.hpp:56-59)."""
    rs, ks, n = 16, 8, 10_000_000
    d = rg.generate(n, rg.RecordLayout(rs, ks), seed=0x5EED0001)
    a = d.cpu().numpy()
    want_sorted = d.clone()
    rg.sort(want_sorted, n, rg.RecordLayout(rs, ks))
    want = want_sorted.cpu().numpy()
    page = np.empty(a.size + 3, dtype=np.uint8)[3:]
    page[:] = a
    rg.sort(page, n, rg.RecordLayout(rs, ks))
    assert np.array_equal(page, want)
    pin = torch_cuda.empty(a.size, dtype=torch_cuda.uint8, pin_memory=True).numpy()
    pin[:] = a
    rg.sort(pin, n, rg.RecordLayout(rs, ks))
    assert np.array_equal(pin, want)
    page[:] = a
    rg.lsd_sort(page, n, rg.RecordLayout(rs, ks))
    assert np.array_equal(page, want)


def test_c5_full_size_matches_reference_group_hashes(rg, torch_cuda):
    """BASELINE C5 (2^32 x 16 B) on one GPU against the reference's chunked run
    (for each top-byte group [32g, 32g+32) the reference sorted
    that group's records, tests/golden/make_golden.py --c5). The sorted output
    is partitioned by top byte, so group g is the contiguous slice after groups
    0..g-1; its bytes must hash to the reference's canonical sha256."""
    import hashlib
    import json
    gold = json.load(open(CONFIG_GOLDEN))["c5"]
    n, rs, ks, dist, seed = gold["n"], gold["rs"], gold["ks"], gold["dist"], gold["seed"]
    free, _ = torch_cuda.cuda.mem_get_info()
    if free < 2 * n * rs + (4 << 30):
        pytest.skip(f"needs {2 * n * rs >> 30} GiB of free device memory")
    lay = rg.RecordLayout(rs, ks)
    d = rg.generate(n, lay, dist=dist, seed=seed)
    rg.sort(d, n, lay)
    torch_cuda.cuda.synchronize()
    assert rg.check_sorted(d, n, lay)[0] == 0
    off = 0
    step = 1 << 30
    for g in gold["groups"]:
        lo, hi = off * rs, (off + g["records"]) * rs
        first, last = d[lo:lo + rs].cpu().numpy(), d[hi - rs:hi].cpu().numpy()
        assert g["top_byte_lo"] <= first[0] and last[0] < g["top_byte_hi"]
        h = hashlib.sha256()
        for o in range(lo, hi, step):
            h.update(memoryview(d[o:min(o + step, hi)].cpu().numpy()))
        assert h.hexdigest() == g["canonical_sha"], f"group {g['top_byte_lo']}"
        off += g["records"]
    assert off == n
    del d
    torch_cuda.cuda.empty_cache()


def test_host_sort_out_of_core(rg, torch_cuda, monkeypatch):
    """raduls_gpu_sort_host beyond the device budget:
    RADULS_GPU_DEVICE_BUDGET forces the out-of-core plan (streamed AND/OR +
    16-bit prefix histogram, greedy contiguous parts, streamed stable
    partition into host scratch, per-part device sort) on inputs several times
    the budget; the result must equal the in-core sort byte for byte."""
    for rs, ks, dist, n in [(16, 8, oracle.DIST_UNIFORM, 6_000_000), (16, 8, oracle.DIST_SKEW, 3_000_000),
                            (32, 24, oracle.DIST_UNIFORM, 2_000_000), (8, 8, oracle.DIST_UNIFORM, 5_000_000)]:
        lay = rg.RecordLayout(rs, ks)
        d = rg.generate(n, lay, dist=dist, seed=0x5EED0000 + rs + dist)
        a = d.cpu().numpy()
        rg.sort(d, n, lay)
        want = d.cpu().numpy()
        monkeypatch.setenv("RADULS_GPU_DEVICE_BUDGET", str(96 << 20))
        b = a.copy()
        rg.sort(b, n, lay)
        assert np.array_equal(b, want), (rs, ks, dist)
        # caller-provided host scratch (the drop-in's tmp argument)
        c = a.copy()
        tmp = np.empty_like(a)
        rc = rg._lib.load().raduls_gpu_sort_host(c.ctypes.data, tmp.ctypes.data, n, rs, ks)
        assert rc == 0 and np.array_equal(c, want)
        monkeypatch.delenv("RADULS_GPU_DEVICE_BUDGET")
    # all keys equal: nothing moves
    monkeypatch.setenv("RADULS_GPU_DEVICE_BUDGET", str(96 << 20))
    e = make_input(3_000_000, 16, 8, 1, universe=1)
    f = e.copy()
    rg.sort(f, 3_000_000, rg.RecordLayout(16, 8))
    assert np.array_equal(f, e)


def test_host_sort_out_of_core_late_varying_top_byte(rg, torch_cuda, monkeypatch):
    """Out-of-core host sort whose first chunk has a constant top key byte that
    varies only in later chunks: the first pass guesses byte 1, the exact AND/OR
    forces a second prefix-histogram pass on byte 0 (back-to-back staged copies
    of a pageable buffer: a staging buffer must not be refilled while its last
    DMA is still reading it)."""
    rs, ks, n = 16, 8, 6_000_000
    a = make_input(n, rs, ks, 0xACE)
    r = a.reshape(n, rs)
    r[: n // 2, 0] = 0x42  # first half (and so the first chunks): constant byte 0
    want = oracle.stable_sort(a, rs, ks)
    monkeypatch.setenv("RADULS_GPU_DEVICE_BUDGET", str(96 << 20))
    b = a.copy()
    rg.sort(b, n, rg.RecordLayout(rs, ks))
    assert np.array_equal(b, want)


def test_host_sort_out_of_core_bucket_larger_than_device(rg, torch_cuda, monkeypatch):
    """One 16-bit key prefix holds more records than a device part: that part
    is sorted by the same out-of-core plan applied to its range (its next
    varying bytes), recursively, instead of failing with ENOMEM."""
    rs, ks, n = 16, 8, 6_000_000
    a = make_input(n, rs, ks, 0xB16)
    r = a.reshape(n, rs)
    hot = np.random.default_rng(3).random(n) < 0.55
    r[hot, 0], r[hot, 1] = 0x77, 0x33   # ~3.3 M records in one bucket (a part holds ~2.1 M)
    r[hot[: n // 3].nonzero()[0][:1000], 2] = 0x00  # and a few ties deeper down
    want = oracle.stable_sort(a, rs, ks)
    monkeypatch.setenv("RADULS_GPU_DEVICE_BUDGET", str(96 << 20))
    b = a.copy()
    rg.sort(b, n, rg.RecordLayout(rs, ks))
    assert np.array_equal(b, want)
    c = a.copy()
    tmp = np.empty_like(a)
    rc = rg._lib.load().raduls_gpu_sort_host(c.ctypes.data, tmp.ctypes.data, n, rs, ks)
    assert rc == 0 and np.array_equal(c, want)


def test_host_sort_frees_its_device_buffers(rg, torch_cuda):
    """The host drop-in frees its two n*rs device buffers before returning
    (the reference frees its per-call aux, msd_sorter.hpp:52), unless the
    caller opts into caching them (raduls_gpu_set_host_cache)."""
    rs, ks, n = 16, 8, 1 << 25  # 512 MiB of records: 1 GiB of device buffers
    a = make_input(n, rs, ks, 77)
    torch_cuda.cuda.synchronize()
    free0, _ = torch_cuda.cuda.mem_get_info()
    b = a.copy()
    rg.sort(b, n, rg.RecordLayout(rs, ks))
    free1, _ = torch_cuda.cuda.mem_get_info()
    assert free1 > free0 - (256 << 20)
    try:
        rg.set_host_cache(True)
        c = a.copy()
        rg.sort(c, n, rg.RecordLayout(rs, ks))
        free2, _ = torch_cuda.cuda.mem_get_info()
        assert free2 < free0 - (900 << 20)
        assert np.array_equal(b, c)
    finally:
        rg.set_host_cache(False)
    free3, _ = torch_cuda.cuda.mem_get_info()
    assert free3 > free0 - (256 << 20)


@pytest.mark.parametrize("rs,ks", [(8, 8), (16, 8), (24, 16), (32, 24)])
def test_scatter_tile_boundaries(rg, torch_cuda, rs, ks):
    """Sizes straddling multiples of the scatter tile above the local-sort
    capacity (so a scatter level runs), and the single-segment split."""
    tile, cap = rg.raduls.scatter_tile(rs), rg.local_capacity(rs)
    k0 = cap // tile + 1
    for j, n in enumerate([k0 * tile - 1, k0 * tile, k0 * tile + 1, (k0 + 3) * tile + 7]):
        a = make_input(n, rs, ks, 4242 + j, (0, 300, 2, 0)[j])
        assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)
        d = to_dev(torch_cuda, a)
        out = torch_cuda.empty_like(d)
        counts = rg.split(d, out, n, rs, 0)
        torch_cuda.cuda.synchronize()
        want = a.reshape(n, rs)[np.argsort(a.reshape(n, rs)[:, 0], kind="stable")].reshape(-1)
        assert np.array_equal(from_dev(out), want)
        assert list(counts) == list(np.bincount(a.reshape(n, rs)[:, 0], minlength=256))


def test_scratch_allocation_failure_leaves_input_untouched(rg, torch_cuda):
    """The reference's resource_error contract (P/include/raduls/record_array.hpp:
    21-28, scheduler.hpp:56-59): when the scratch array cannot be allocated the
    call fails with ResourceError and the records are untouched. Here the
    records take more than half of the free device memory, so the library's
    own d_tmp allocation (cudaMallocAsync, d_tmp = NULL) cannot succeed."""
    free, _ = torch_cuda.cuda.mem_get_info()
    rs, ks = 32, 8  # 32-B records: 60% of the device within the 2^32-record limit
    n = min(int(free * 0.6) // rs, 1 << 32)
    if n * rs * 2 <= free:  # pragma: no cover - a device this roomy cannot exercise it
        pytest.skip("not enough memory pressure")
    lay = rg.RecordLayout(rs, ks)
    d = rg.generate(n, lay, seed=7)
    before = rg.digest(d, n, rs)
    probe = d[:1 << 20].clone()
    with pytest.raises(rg.ResourceError):
        rg.sort(d, n, lay)
    torch_cuda.cuda.synchronize()
    assert rg.digest(d, n, rs) == before
    assert torch_cuda.equal(d[:1 << 20], probe)
    del d, probe
    torch_cuda.cuda.empty_cache()
    # the library still works afterwards
    a = make_input(100000, rs, ks, 3)
    assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)


def test_concurrent_callers_on_one_device(rg, torch_cuda):
    """Concurrent calls on disjoint arrays are safe (no global
    state in the reference, scheduler.hpp:56-61). ctypes drops the GIL, so the
    threads enter the library together and serialise on the device workspace."""
    import threading
    cases = [(16, 8, 150_000, 1), (32, 24, 60_000, 2), (8, 8, 200_000, 3), (24, 16, 90_000, 4),
             (16, 16, 5_000, 5), (16, 8, 400_000, 6)]
    inputs = [make_input(n, rs, ks, seed, universe=(0, 500)[seed % 2]) for rs, ks, n, seed in cases]
    devs = [to_dev(torch_cuda, a) for a in inputs]
    errors = []

    def work(i):
        try:
            rs, ks, n, _ = cases[i]
            for _ in range(3):  # repeated sorts of a sorted array stay put
                rg.sort(devs[i], n, rg.RecordLayout(rs, ks))
            torch_cuda.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (rs, ks, n, _), a, d in zip(cases, inputs, devs):
        assert_parity(from_dev(d), a, rs, ks)


def test_sort_on_a_caller_stream(rg, torch_cuda):
    """raduls_gpu_sort on the caller's stream is ordered after the caller's
    earlier work on that stream (the input is produced there)."""
    rs, ks, n = 16, 8, 300_000
    a = make_input(n, rs, ks, 9)
    s = torch_cuda.cuda.Stream()
    host = torch_cuda.from_numpy(a).pin_memory()
    with torch_cuda.cuda.stream(s):
        d = torch_cuda.empty(n * rs, dtype=torch_cuda.uint8, device="cuda")
        d.copy_(host, non_blocking=True)  # produced on s
        rg.sort(d, n, rg.RecordLayout(rs, ks), stream=s)
    s.synchronize()
    assert_parity(from_dev(d), a, rs, ks)


def test_device_tensor_arguments_are_checked(rg, torch_cuda):
    """Only contiguous uint8 tensors are sorted (n counts bytes / rs and the
    library reads from data_ptr() on); anything else is rejected up front."""
    torch = torch_cuda
    lay = rg.RecordLayout(16, 8)
    with pytest.raises(TypeError):
        rg.sort(torch.zeros(64, dtype=torch.int32, device="cuda"), 4, lay)
    with pytest.raises(ValueError):
        rg.sort(torch.zeros(128, dtype=torch.uint8, device="cuda")[::2], 4, lay)
    d = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(TypeError):
        rg.sort(d, 4, lay, tmp=torch.zeros(16, dtype=torch.int32, device="cuda"))


def test_scatter_rank_modes_are_both_stable(rg, torch_cuda, monkeypatch):
    """The scatter ranks with shared-memory atomics only after the device
    self-test (k_rank_selftest) confirmed lane-ordered service; the ballot
    ranker (stable by construction) is what the library falls back to. Both
    must give the stable sort byte for byte, on duplicate-heavy inputs where
    an unstable rank would reorder equal keys."""
    import subprocess
    import sys
    mode = rg.rank_mode()
    assert mode in (0, 1)
    cases = [(16, 8, 300_000, 7), (8, 8, 400_000, 3), (32, 24, 120_000, 50), (24, 16, 90_000, 2)]
    for rs, ks, n, universe in cases:
        a = make_input(n, rs, ks, 1234 + rs, universe)
        assert_parity(gpu_sort(rg, torch_cuda, a, rs, ks), a, rs, ks)
    # the ballot ranker, in a fresh process (the mode is chosen once per device)
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np, torch, oracle, paper_1612_02557_b200 as rg\n"
        "from helpers import make_input\n"
        "assert rg.rank_mode() == 1\n"
        "for rs, ks, n, u in %r:\n"
        "    a = make_input(n, rs, ks, 1234 + rs, u)\n"
        "    d = torch.from_numpy(a.copy()).cuda()\n"
        "    rg.sort(d, n, rg.RecordLayout(rs, ks)); torch.cuda.synchronize()\n"
        "    assert np.array_equal(d.cpu().numpy(), oracle.stable_sort(a, rs, ks)), (rs, ks)\n"
        "print('OK')\n" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           os.path.dirname(os.path.abspath(__file__)), cases))
    env = dict(os.environ, RADULS_GPU_STABLE_RANK="ballot")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
