"""GPU parity of the building-block kernels against the oracle.

* generator bit-identical to oracle orc_generate;
* histogram of bytes 0..7 == build_histogram (P/tests/test_kernels.cpp:62-85);
* single-digit split byte-identical to radix_split (P/tests/test_kernels.cpp:114-143,
  acceptance.cpp:138-166 kernel equivalence);
* digest / check_sorted == array_digest / check_sorted (P/src/verify.cpp:27-50);
* multi-GPU partition: stable grouping by destination rank.
"""
import numpy as np
import pytest

import oracle
from helpers import ALL_LAYOUTS, EXTRA_LAYOUTS, from_dev, make_input, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS + [(32, 24), (16, 3)])
@pytest.mark.parametrize("dist", [0, 1])
def test_generator_bit_identical(rg, torch_cuda, rs, ks, dist):
    for n, base in [(1, 0), (1000, 0), (77777, 123456789)]:
        d = rg.generate(n, rg.RecordLayout(rs, ks), dist=dist, seed=0x5EED0001, index_base=base)
        want = oracle.generate(n, rs, ks, dist, 0x5EED0001, base)
        assert np.array_equal(from_dev(d), want)


@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS + EXTRA_LAYOUTS)
def test_histogram_all_bytes(rg, torch_cuda, rs, ks):
    for n, uni in [(0, 0), (1, 0), (5000, 0), (100003, 256), (65536, 1)]:
        a = make_input(n, rs, ks, 17 + n, uni)
        h, ao = rg.histogram(to_dev(torch_cuda, a), n, rg.RecordLayout(rs, ks))
        for b in range(min(ks, 8)):
            assert np.array_equal(h[b], oracle.histogram(a, rs, b)), (b, n)
        if n:
            words = a.reshape(n, rs).view("<u8")
            for w in range(rs // 8):
                assert int(ao[2 * w]) == int(np.bitwise_and.reduce(words[:, w]))
                assert int(ao[2 * w + 1]) == int(np.bitwise_or.reduce(words[:, w]))


@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS)
def test_split_matches_radix_split(rg, torch_cuda, rs, ks):
    rng = np.random.default_rng(424242 + rs)
    for it in range(6):
        n = (1 << 20) if it == 0 else int(rng.integers(1, 300000))
        a = make_input(n, rs, ks, int(rng.integers(1 << 40)), 1000 if it % 3 == 0 else 0)
        off = int(rng.integers(0, ks))
        src = to_dev(torch_cuda, a)
        dst = torch_cuda.empty_like(src)
        h = rg.split(src, dst, n, rs, off)
        want, wh = oracle.radix_split(a, rs, off)
        assert np.array_equal(h, wh)
        assert np.array_equal(from_dev(dst), want)


def test_split_identity_on_identical_keys(rg, torch_cuda):
    """test_kernels.cpp:210-220."""
    rs, n = 16, 10000
    a = make_input(n, rs, 8, 1, universe=1)
    src = to_dev(torch_cuda, a)
    dst = torch_cuda.empty_like(src)
    rg.split(src, dst, n, rs, 7)
    assert np.array_equal(from_dev(dst), a)


@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS + [(32, 24)])
def test_digest_and_check_sorted(rg, torch_cuda, rs, ks):
    a = make_input(50001, rs, ks, 5, 300)
    d = to_dev(torch_cuda, a)
    assert rg.digest(d, 50001, rs) == oracle.digest(a, rs)
    v, f = rg.check_sorted(d, 50001, rg.RecordLayout(rs, ks))
    ok, first = oracle.check_sorted(a, rs, ks)
    assert (v == 0) == ok
    if not ok:
        assert f == first
    s = oracle.stable_sort(a, rs, ks)
    assert rg.check_sorted(to_dev(torch_cuda, s), 50001, rg.RecordLayout(rs, ks))[0] == 0


@pytest.mark.parametrize("rs,ks", [(16, 8), (8, 8), (32, 24)])
def test_partition_stable_by_rank(rg, torch_cuda, rs, ks):
    import ctypes as C
    n, ranks, pb = 200000, 5, 0
    a = make_input(n, rs, ks, 31 + rs, 0)
    src = to_dev(torch_cuda, a)
    dst = torch_cuda.empty_like(src)
    # contiguous bucket ranges -> ranks
    bucket_rank = (np.arange(65536) * ranks // 65536).astype(np.uint32)
    dmap = torch_cuda.from_numpy(bucket_rank.view(np.int32)).cuda()
    counts = np.zeros(ranks, dtype=np.uint64)
    L = rg._lib.load()
    rc = L.raduls_gpu_partition(src.data_ptr(), dst.data_ptr(), n, rs, ks, pb, dmap.data_ptr(),
                                ranks, counts.ctypes.data_as(C.POINTER(C.c_uint64)), None)
    assert rc == 0
    torch_cuda.cuda.synchronize()
    r = a.reshape(n, rs)
    pref = (r[:, 0].astype(np.int64) << 8) | r[:, 1]
    dest = bucket_rank[pref]
    order = np.argsort(dest, kind="stable")
    assert np.array_equal(counts, np.bincount(dest, minlength=ranks).astype(np.uint64))
    assert np.array_equal(from_dev(dst).reshape(n, rs), r[order])
    # prefix histogram
    hist = torch_cuda.zeros(65536, dtype=torch_cuda.int64, device="cuda")
    rc = L.raduls_gpu_prefix_histogram(src.data_ptr(), n, rs, ks, pb, hist.data_ptr(), None)
    assert rc == 0
    assert np.array_equal(hist.cpu().numpy(), np.bincount(pref, minlength=65536))


@pytest.mark.parametrize("rs,ks", [(16, 8), (8, 8), (24, 16), (32, 24)])
def test_partition_to_equals_partition(rg, torch_cuda, rs, ks):
    """raduls_gpu_partition_to (the partition fused with the exchange) writes
    each rank's stable range to its own destination buffer: identical to the
    ordinary partition output cut at the rank counts."""
    import ctypes as C
    from paper_1612_02557_b200 import _lib
    from helpers import make_input, to_dev, from_dev
    L = _lib.load()
    n, ranks = 100_003, 3
    a = make_input(n, rs, ks, 31 + rs, universe=(0 if rs != 8 else 5000))
    d = to_dev(torch_cuda, a)
    bmap = (np.arange(65536, dtype=np.uint32) * ranks // 65536).astype(np.uint32)
    dmap = torch_cuda.from_numpy(bmap.view(np.int32)).cuda()
    ref = torch_cuda.empty_like(d)
    counts = np.zeros(ranks, dtype=np.uint64)
    assert L.raduls_gpu_partition(d.data_ptr(), ref.data_ptr(), n, rs, ks, 0, dmap.data_ptr(), ranks,
                                  counts.ctypes.data_as(_lib._u64p), None) == 0
    outs = [torch_cuda.empty(int(c) * rs + 64, dtype=torch_cuda.uint8, device="cuda") for c in counts]
    dst = np.array([o.data_ptr() for o in outs], dtype=np.uint64)
    got = np.zeros(ranks, dtype=np.uint64)
    assert L.raduls_gpu_partition_to(d.data_ptr(), n, rs, ks, 0, dmap.data_ptr(), ranks,
                                     dst.ctypes.data_as(_lib._u64p), got.ctypes.data_as(_lib._u64p),
                                     None) == 0
    torch_cuda.cuda.synchronize()
    assert list(got) == list(counts)
    r = from_dev(ref)
    off = 0
    for o, c in zip(outs, counts):
        c = int(c)
        assert np.array_equal(from_dev(o)[:c * rs], r[off * rs:(off + c) * rs])
        off += c


@pytest.mark.parametrize("rs,ks", [(16, 8), (8, 8), (24, 16), (32, 24)])
def test_partition_plan_store_equals_partition(rg, torch_cuda, rs, ks):
    """raduls_gpu_partition_plan + raduls_gpu_partition_store (the two-phase
    fused partition of the sampled multi-GPU plan): same counts and same
    per-rank ranges as the ordinary partition; the plan's AND/OR is the
    array's; any other call in between invalidates the plan."""
    from paper_1612_02557_b200 import _lib
    from helpers import make_input, to_dev, from_dev
    L = _lib.load()
    n, ranks = 100_003, 3
    a = make_input(n, rs, ks, 41 + rs, universe=(0 if rs != 8 else 5000))
    d = to_dev(torch_cuda, a)
    bmap = (np.arange(65536, dtype=np.uint32) * ranks // 65536).astype(np.uint32)
    dmap = torch_cuda.from_numpy(bmap.view(np.int32)).cuda()
    ref = torch_cuda.empty_like(d)
    counts = np.zeros(ranks, dtype=np.uint64)
    assert L.raduls_gpu_partition(d.data_ptr(), ref.data_ptr(), n, rs, ks, 0, dmap.data_ptr(), ranks,
                                  counts.ctypes.data_as(_lib._u64p), None) == 0
    got = np.zeros(ranks, dtype=np.uint64)
    ao = np.zeros(8, dtype=np.uint64)
    assert L.raduls_gpu_partition_plan(d.data_ptr(), n, rs, ks, 0, dmap.data_ptr(), ranks,
                                       got.ctypes.data_as(_lib._u64p), ao.ctypes.data_as(_lib._u64p),
                                       None) == 0
    assert list(got) == list(counts)
    w = a.reshape(n, rs).view("<u8")
    for k in range(rs // 8):
        assert ao[2 * k] == np.bitwise_and.reduce(w[:, k]) and ao[2 * k + 1] == np.bitwise_or.reduce(w[:, k])
    outs = [torch_cuda.empty(int(c) * rs + 64, dtype=torch_cuda.uint8, device="cuda") for c in counts]
    dst = np.array([o.data_ptr() for o in outs], dtype=np.uint64)
    assert L.raduls_gpu_partition_store(d.data_ptr(), n, rs, ks, dst.ctypes.data_as(_lib._u64p), None) == 0
    torch_cuda.cuda.synchronize()
    r = from_dev(ref)
    off = 0
    for o, c in zip(outs, counts):
        c = int(c)
        assert np.array_equal(from_dev(o)[:c * rs], r[off * rs:(off + c) * rs])
        off += c
    # a second store of the same plan, or one after another call, is refused
    assert L.raduls_gpu_partition_store(d.data_ptr(), n, rs, ks, dst.ctypes.data_as(_lib._u64p), None) == _lib.EINVAL
    assert L.raduls_gpu_partition_plan(d.data_ptr(), n, rs, ks, 0, dmap.data_ptr(), ranks,
                                       got.ctypes.data_as(_lib._u64p), ao.ctypes.data_as(_lib._u64p),
                                       None) == 0
    tmp = to_dev(torch_cuda, a)
    rg.sort(tmp, n, rg.RecordLayout(rs, ks))
    assert L.raduls_gpu_partition_store(d.data_ptr(), n, rs, ks, dst.ctypes.data_as(_lib._u64p), None) == _lib.EINVAL


@pytest.mark.parametrize("rs,ks", [(16, 8), (8, 8), (32, 24)])
def test_sampled_andor_and_prefix_histogram(rg, torch_cuda, rs, ks):
    from paper_1612_02557_b200 import _lib
    from helpers import make_input, to_dev
    L = _lib.load()
    n, samples = 300_001, 4096
    a = make_input(n, rs, ks, 51 + rs)
    d = to_dev(torch_cuda, a)
    stride = max(1, n // samples)
    idx = np.minimum(n - 1, np.arange(samples, dtype=np.int64) * stride)
    recs = a.reshape(n, rs)[idx]
    ao = np.zeros(8, dtype=np.uint64)
    assert L.raduls_gpu_sample_andor(d.data_ptr(), n, rs, samples, ao.ctypes.data_as(_lib._u64p), None) == 0
    w = recs.view("<u8")
    for k in range(rs // 8):
        assert ao[2 * k] == np.bitwise_and.reduce(w[:, k]) and ao[2 * k + 1] == np.bitwise_or.reduce(w[:, k])
    pb = 1
    hist = torch_cuda.zeros(65536, dtype=torch_cuda.int64, device="cuda")
    assert L.raduls_gpu_sample_prefix_histogram(d.data_ptr(), n, rs, ks, pb, samples, hist.data_ptr(), None) == 0
    pref = (recs[:, pb].astype(np.int64) << 8) | recs[:, pb + 1].astype(np.int64)
    assert np.array_equal(hist.cpu().numpy(), np.bincount(pref, minlength=65536))


@pytest.mark.parametrize("rs,ks", [(16, 8), (8, 8), (32, 24)])
def test_sort_segments_matches_oracle(rg, torch_cuda, rs, ks):
    """raduls_gpu_sort_segments (the multi-GPU receiver's sort): records
    already grouped into key-ordered segments (here stably by key byte 0),
    each sorted from key byte 1 on; empty segments, and the 0x42 segment cut
    into below / equal-key / above parts (the equal part from key byte ks)."""
    from paper_1612_02557_b200.distributed import DeviceOps
    n = 400_000
    a = make_input(n, rs, ks, 31 + rs)
    r = a.reshape(n, rs)
    hot = bytes([0x42] * ks)
    r[: n // 10, :ks] = 0x42  # 10%: one key
    parts, sizes, fb = [], [], []
    for v in range(256):
        seg = r[r[:, 0] == v]  # stable: input order inside
        if v == 0x42:
            keys = [bytes(x[:ks]) for x in seg]
            for sel, f in (([k < hot for k in keys], 1), ([k == hot for k in keys], ks),
                           ([k > hot for k in keys], 1)):
                parts.append(seg[np.array(sel, dtype=bool)])
                sizes.append(int(np.sum(sel)))
                fb.append(f)
        else:
            parts.append(seg)
            sizes.append(len(seg))
            fb.append(1)
    part = np.concatenate(parts).reshape(-1)
    sizes[5:5] = [0, 0]  # empty segments are allowed anywhere
    fb[5:5] = [1, 2]
    assert sum(sizes) == n
    d = to_dev(torch_cuda, part)
    DeviceOps().sort_segments(d, n, rg.RecordLayout(rs, ks), sizes, fb)
    torch_cuda.cuda.synchronize()
    assert np.array_equal(from_dev(d), oracle.stable_sort(part, rs, ks))


def test_sort_segments_many_small_segments(rg, torch_cuda):
    """Hundreds of small key-ordered segments (below the local-sort capacity,
    some empty, some of one record), each from key byte 2."""
    from paper_1612_02557_b200.distributed import DeviceOps
    rs, ks, n = 16, 8, 200_000
    a = make_input(n, rs, ks, 777)
    r = a.reshape(n, rs)
    pre = (r[:, 0].astype(np.int64) << 8) | r[:, 1]
    order = np.argsort(pre, kind="stable")
    part = r[order].reshape(-1).copy()
    sizes = [int(c) for c in np.bincount(pre, minlength=65536)]  # ~3 records per 16-bit bucket
    d = to_dev(torch_cuda, part)
    DeviceOps().sort_segments(d, n, rg.RecordLayout(rs, ks), sizes, [2] * 65536)
    torch_cuda.cuda.synchronize()
    assert np.array_equal(from_dev(d), oracle.stable_sort(part, rs, ks))
