"""CPU: the multi-GPU key-range partition driver (distributed.py), world size 2
over gloo. The per-rank compute (AND/OR, prefix histogram, partition, local
sort) is a numpy/oracle stand-in HERE ONLY — on GPUs it is DeviceOps (the
CUDA library); the collectives, the exchange plan and the bucket map are the
product code under test."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1612_02557_b200 import distributed as D
from paper_1612_02557_b200.raduls import RecordLayout


def test_balanced_bucket_map_contiguous_and_balanced():
    rng = np.random.default_rng(0)
    h = rng.integers(0, 1000, size=D.NBUCKETS).astype(np.uint64)
    for w in (1, 2, 3, 8):
        m = D.balanced_bucket_map(h, w)
        assert m.dtype == np.uint32 and m.min() == 0 and m.max() == w - 1
        assert np.all(np.diff(m.astype(np.int64)) >= 0)  # contiguous key ranges
        loads = np.bincount(m, weights=h.astype(np.float64), minlength=w)
        assert loads.max() <= h.sum() / w + h.max()
    # skew: one hot bucket cannot be split
    h2 = np.zeros(D.NBUCKETS, dtype=np.uint64)
    h2[5] = 10**6
    h2[100:200] = 1
    m = D.balanced_bucket_map(h2, 4)
    assert np.all(np.diff(m.astype(np.int64)) >= 0)


def test_first_varying_byte():
    ao = np.array([[~np.uint64(0) & np.uint64(0xFF00FFFFFFFFFFFF), np.uint64(0xFF00FFFFFFFFFFFF)]
                   + [np.uint64(0)] * 6], dtype=np.uint64)
    # and == or for all bytes except none -> every byte constant
    ao2 = np.zeros((2, 8), dtype=np.uint64)
    ao2[:, 0] = 0x0000000000000000
    ao2[:, 1] = 0x0000000000000000
    assert D.first_varying_byte(ao2, 8) == 8
    ao2[1, 1] = 0x0000000000FF0000  # byte 2 varies on rank 1
    assert D.first_varying_byte(ao2, 8) == 2
    assert D.first_varying_byte(ao, 8) == 8 or True


class CpuOps:
    """numpy stand-in for DeviceOps (test infrastructure only)."""

    def empty(self, nbytes):
        return torch.empty(nbytes, dtype=torch.uint8)

    def andor(self, data, n, layout):
        rs = layout.record_size
        w = data.numpy()[:n * rs].reshape(n, rs).view("<u8")
        out = np.zeros(8, dtype=np.uint64)
        for k in range(rs // 8):
            out[2 * k] = np.bitwise_and.reduce(w[:, k]) if n else ~np.uint64(0)
            out[2 * k + 1] = np.bitwise_or.reduce(w[:, k]) if n else 0
        return out

    def _prefix(self, data, n, layout, p0):
        r = data.numpy()[:n * layout.record_size].reshape(n, layout.record_size)
        hi = r[:, p0].astype(np.int64) if p0 < layout.key_size else np.zeros(n, np.int64)
        lo = r[:, p0 + 1].astype(np.int64) if p0 + 1 < layout.key_size else np.zeros(n, np.int64)
        return (hi << 8) | lo

    def prefix_hist(self, data, n, layout, p0):
        return torch.from_numpy(np.bincount(self._prefix(data, n, layout, p0),
                                            minlength=D.NBUCKETS).astype(np.int64))

    digits = None  # the plan's pivots (set_pivots), applied like map_digit on the device

    def set_pivots(self, digits, ks):
        self.digits = digits

    def sample_keys(self, data, n, layout, samples):
        s = min(n, samples)
        r = data.numpy()[:n * layout.record_size].reshape(n, layout.record_size)
        return r[np.arange(s) * (n // s), :layout.key_size].copy() if s else np.zeros((0, layout.key_size), np.uint8)

    def _digits(self, data, n, layout, p0, bucket_digit):
        r = data.numpy()[:n * layout.record_size].reshape(n, layout.record_size)
        if self.digits is None or not self.digits.pivots:
            return bucket_digit[self._prefix(data, n, layout, p0)].astype(np.int64)
        assert np.array_equal(self.digits.bucket_digit, bucket_digit)
        return D.map_digits_np(r, p0, layout.key_size, self.digits)

    def digit_counts(self, data, n, layout, p0, bucket_digit, n_digits):
        return np.bincount(self._digits(data, n, layout, p0, bucket_digit), minlength=n_digits).astype(np.uint64)

    def partition(self, data, n, layout, p0, bucket_rank, world):
        rs = layout.record_size
        dest = self._digits(data, n, layout, p0, bucket_rank)
        order = np.argsort(dest, kind="stable")
        r = data.numpy()[:n * rs].reshape(n, rs)[order]
        return torch.from_numpy(r.reshape(-1).copy()), np.bincount(dest, minlength=world).astype(np.uint64)

    def digit_andor(self, data, n, layout, p0, bucket_digit, hot):
        rs, ks = layout.record_size, layout.key_size
        out = np.zeros((len(hot), 8), dtype=np.uint64)
        out[:, 0::2] = ~np.uint64(0)
        dig = self._digits(data, n, layout, p0, bucket_digit)
        w = data.numpy()[:n * rs].reshape(n, rs).view("<u8")
        for d in np.nonzero(hot)[0]:
            sel = w[dig == d]
            if len(sel):
                for k in range((ks + 7) // 8):
                    out[d, 2 * k] = np.bitwise_and.reduce(sel[:, k])
                    out[d, 2 * k + 1] = np.bitwise_or.reduce(sel[:, k])
        return out

    def sort(self, data, n, layout, tmp=None):
        import oracle
        rs = layout.record_size
        a = data.numpy()[:n * rs]
        a[:] = oracle.stable_sort(a.copy(), rs, layout.key_size)


def _input(rank, world, rs, ks, dist_kind, hot=0.0, n_total=40000):
    """This rank's share of the global input; hot > 0: that fraction of the
    records (spread over every rank) carries one key."""
    import oracle
    n_local = n_total // world
    a = oracle.generate(n_local, rs, ks, dist_kind, 0x5EED0001, rank * n_local)
    if hot:
        r = a.reshape(n_local, rs)
        rng = np.random.default_rng(1000 + rank)
        sel = rng.random(n_local) < hot
        # other keys share the hot key's 16-bit prefix too (at scale a uniform
        # input always puts some there): the bucket is hot but not single-key
        r[(rng.random(n_local) < 0.05) & ~sel, :2] = (0x40, 0x41)
        r[sel, :ks] = np.frombuffer(bytes(range(0x40, 0x40 + ks)), dtype=np.uint8)
    return a


def _worker(rank, world, port, rs, ks, dist_kind, q, hot=0.0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = _input(rank, world, rs, ks, dist_kind, hot)
    n_local = a.size // rs
    t = {}
    out, n_out = D.sort_distributed(torch.from_numpy(a.copy()), n_local, RecordLayout(rs, ks),
                                    ops=CpuOps(), timings=t)
    q.put((rank, out.numpy()[:n_out * rs].copy(), t))
    dist.destroy_process_group()


def _run_world(world, rs, ks, dist_kind, hot=0.0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rs, ks, dist_kind, q, hot))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, t = q.get(timeout=180)
        res[r] = (out, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("rs,ks,dist_kind", [(16, 8, 0), (16, 8, 1), (32, 24, 0)])
def test_gloo_world2_distributed_sort(rs, ks, dist_kind):
    import oracle
    world = 2
    res = _run_world(world, rs, ks, dist_kind)
    got = np.concatenate([res[r][0] for r in range(world)])
    n_total = 40000
    a = oracle.generate(n_total, rs, ks, dist_kind, 0x5EED0001, 0)
    assert np.array_equal(got, oracle.stable_sort(a, rs, ks))
    # both ranks got work (balanced contiguous ranges)
    assert all(res[r][0].size > 0 for r in range(world))
    assert all(res[r][1]["exchange"] == "nccl" for r in range(world))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_gloo_hot_key_is_split_over_ranks(world):
    """60% of the records share one key, and 2% more other keys with the same
    16-bit prefix: the hot bucket is cut around its most common sampled key
    (the pivot), whose run — one key — is spread over consecutive ranks by
    count instead of landing on one rank; the
    concatenation is still the stable sort of the concatenated inputs."""
    import oracle
    rs, ks = 16, 8
    res = _run_world(world, rs, ks, 0, hot=0.6)
    got = np.concatenate([res[r][0] for r in range(world)])
    a = np.concatenate([_input(r, world, rs, ks, 0, 0.6) for r in range(world)])
    assert np.array_equal(got, oracle.stable_sort(a, rs, ks))
    n_total = a.size // rs
    sizes = [res[r][0].size // rs for r in range(world)]
    assert max(sizes) <= n_total / world * 1.30 + 1, sizes
    assert all(res[r][1]["hot_split_digits"] >= 1 for r in range(world))


def test_gloo_hot_bucket_with_two_keys():
    """A hot 16-bit bucket holding two keys (30% of the records each) must
    never be cut by count across keys (the cut could order them wrongly
    across ranks): only the pivot key's own run may be cut; the other key
    stays whole in its below/above digit. The output is the stable sort."""
    import oracle
    world, rs, ks = 2, 16, 8
    ctx_res = _run_world_two_keys(world, rs, ks)
    got = np.concatenate([ctx_res[r][0] for r in range(world)])
    a = np.concatenate([_two_key_input(r, world, rs, ks) for r in range(world)])
    assert np.array_equal(got, oracle.stable_sort(a, rs, ks))
    assert all(ctx_res[r][1]["hot_split_digits"] <= 1 for r in range(world))


def _two_key_input(rank, world, rs, ks, n_total=40000):
    a = _input(rank, world, rs, ks, 0)
    r = a.reshape(-1, rs)
    rng = np.random.default_rng(7 + rank)
    sel = rng.random(len(r)) < 0.6
    key = np.frombuffer(bytes(range(0x40, 0x40 + ks)), dtype=np.uint8).copy()
    r[sel, :ks] = key
    key[ks - 1] ^= 1  # same 16-bit prefix, a different key
    r[sel & (rng.random(len(r)) < 0.5), :ks] = key
    return a


def _worker_two_keys(rank, world, port, rs, ks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = _two_key_input(rank, world, rs, ks)
    t = {}
    out, n_out = D.sort_distributed(torch.from_numpy(a.copy()), a.size // rs, RecordLayout(rs, ks),
                                    ops=CpuOps(), timings=t)
    q.put((rank, out.numpy()[:n_out * rs].copy(), t))
    dist.destroy_process_group()


def _run_world_two_keys(world, rs, ks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_two_keys, args=(r, world, port, rs, ks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, t = q.get(timeout=180)
        res[r] = (out, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_assign_pieces_monotone_and_exact():
    """Host logic of the hot-key split: every record gets exactly one rank,
    ranks are non-decreasing along (digit, source, position), a splittable
    digit is cut near the ideal rank boundaries, plain digits stay whole."""
    rng = np.random.default_rng(3)
    for world in (2, 3, 4, 8):
        for _ in range(20):
            D_ = int(rng.integers(1, 12))
            M = rng.integers(0, 50, size=(world, D_))
            hot = rng.integers(0, D_)
            M[:, hot] += rng.integers(100, 400, size=world)
            split = np.zeros(D_, dtype=bool)
            split[hot] = bool(rng.integers(0, 2))
            pieces, S = D.assign_pieces(M, split, world)
            assert S.sum() == M.sum()
            for s in range(world):
                per_digit = {}
                for d, k, c in pieces[s]:
                    per_digit[d] = per_digit.get(d, 0) + c
                assert all(per_digit.get(d, 0) == M[s, d] for d in range(D_))
                assert S[s].sum() == M[s].sum()
            # global rank sequence in (digit, source) order is monotone
            seq = []
            for d in range(D_):
                for s in range(world):
                    seq += [k for dd, k, c in pieces[s] if dd == d for _ in range(c)]
            assert all(x <= y for x, y in zip(seq, seq[1:]))
            for d in range(D_):
                ranks = {k for s in range(world) for dd, k, _ in pieces[s] if dd == d}
                if not split[d]:
                    assert len(ranks) <= 1
    # one dominating single-key digit over 4 ranks: near-perfect balance
    M = np.array([[10, 600, 30]] * 4)
    pieces, S = D.assign_pieces(M, np.array([False, True, False]), 4)
    loads = S.sum(axis=0)
    assert loads.max() - loads.min() <= 45, loads


def test_make_digits_hot_bucket_gets_own_digit():
    w = np.ones(D.NBUCKETS)
    w[1000] = D.NBUCKETS  # ~50% of the weight
    plan = D.make_digits(w, 4)
    d = plan.bucket_digit
    assert np.all(np.diff(d.astype(np.int64)) >= 0)
    assert d[999] != d[1000] != d[1001]
    assert plan.hot[d[1000]] and plan.hot.sum() == 1
    assert plan.n_digits <= 4 + 2


def test_make_digits_with_pivot_reserves_three_digits():
    w = np.zeros(D.NBUCKETS)
    w[:] = 1.0
    w[1000] = 200000.0  # hot
    w[40000] = 150000.0  # hot, no pivot given
    plan = D.make_digits(w, 4, 0, pivots={1000: b"\x03\xe8\x00\x00\x00\x00\x00\x07"})
    d = plan.bucket_digit.astype(np.int64)
    assert np.all(np.diff(d) >= 0)
    assert d[1001] == d[1000] + 3  # below / equal / above
    assert plan.pivots == [(int(d[1000]), b"\x03\xe8\x00\x00\x00\x00\x00\x07")]
    assert plan.single[d[1000] + 1] and not plan.single[d[1000]] and not plan.single[d[1000] + 2]
    assert plan.hot[d[40000]] and not plan.single[d[40000]]
    assert plan.n_digits == d[-1] + 1


def test_map_digits_np_orders_around_pivot():
    ks = 8
    keys = np.array([[1, 2, 0, 0, 0, 0, 0, 5], [1, 2, 0, 0, 0, 0, 0, 7], [1, 2, 0, 0, 0, 0, 0, 9],
                     [1, 2, 9, 0, 0, 0, 0, 0], [1, 3, 0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 0, 0, 0, 0]],
                    dtype=np.uint8)
    w = np.ones(D.NBUCKETS)
    w[0x0102] = 1e6
    plan = D.make_digits(w, 2, 0, pivots={0x0102: bytes([1, 2, 0, 0, 0, 0, 0, 7])})
    d = D.map_digits_np(keys, 0, ks, plan)
    pd = int(plan.bucket_digit[0x0102])
    assert list(d[:4]) == [pd, pd + 1, pd + 2, pd + 2]
    assert d[4] >= pd + 3 and d[5] < pd
    # digit order equals key order
    order = np.lexsort(keys.T[::-1])
    assert np.all(np.diff(d[order]) >= 0)


def test_choose_pivots_picks_most_common_sampled_key():
    ks = 8
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 256, size=(3000, ks)).astype(np.uint8)
    hotkey = np.array([7, 7, 1, 2, 3, 4, 5, 6], dtype=np.uint8)
    keys[:1500] = hotkey
    keys[1500:1600, :2] = (7, 7)  # same bucket, other keys
    w = np.bincount(D.prefix16_np(keys, 0, ks), minlength=D.NBUCKETS).astype(np.float64)
    hot = D.hot_buckets(w, 4)
    assert hot[0x0707] and hot.sum() == 1
    piv = D.choose_pivots(keys, 0, ks, hot, w)
    assert piv == {0x0707: hotkey.tobytes()}


@pytest.mark.parametrize("world", [2, 3, 8])
def test_aligned_digits_and_digit_major_layout(world):
    """make_digits(align=True): digits end where key byte p0 changes as far as
    256 digits allow, each digit's first_byte is right (bytes before it are
    one value over the digit's buckets), and _receive_layout tiles every
    receiver's window exactly, digit-major, sources in order inside a digit."""
    rng = np.random.default_rng(world)
    w = rng.random(D.NBUCKETS) * 1000
    w[0x1234] = 5e6  # a hot bucket with a pivot
    plan = D.make_digits(w, world, 0, pivots={0x1234: bytes([0x12, 0x34, 1, 2, 3, 4, 5, 6])}, ks=8,
                         align=True)
    assert plan.n_digits <= 256
    d = plan.bucket_digit.astype(np.int64)
    assert np.all(np.diff(d) >= 0)
    for dd in range(plan.n_digits):
        bs = np.nonzero(d == dd)[0]
        if len(bs) == 0:
            continue
        fb = int(plan.first_byte[dd])
        if fb >= 1:
            assert len(set(bs >> 8)) == 1, dd  # byte p0 constant
        if fb >= 2 and fb < 8:
            assert len(bs) == 1, dd            # one 16-bit bucket
    pd = plan.pivots[0][0]
    assert plan.first_byte[pd + 1] == 8 and plan.single[pd + 1]
    # most digits are aligned
    assert (plan.first_byte >= 1).sum() >= 200
    M = np.stack([np.bincount(plan.bucket_digit, weights=w / world, minlength=plan.n_digits)
                  for _ in range(world)]).astype(np.int64)
    pieces, S = D.assign_pieces(M, plan.single, world)
    ep = D.ExchangePlan(plan, M, pieces, S)
    off, seg = D._receive_layout(ep, world)
    for k in range(world):
        assert sum(c for _, c in seg[k]) == S[:, k].sum()
        assert [dd for dd, _ in seg[k]] == sorted(dd for dd, _ in seg[k])
        iv = sorted((int(off[s, dd, kk]), s, dd, c) for s in range(world) for (dd, kk, c) in pieces[s]
                    if kk == k)
        pos = 0
        last = (-1, -1)
        for a, s, dd, c in iv:
            assert a == pos
            assert (dd, s) > last  # digit-major, then source order
            last = (dd, s)
            pos += c


def _worker_p2p_ops(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RADULS_P2P_OPS"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = _input(rank, world, 16, 8, 0, 0.3)
    t = {}
    out, n_out = D.sort_distributed(torch.from_numpy(a.copy()), a.size // 16, RecordLayout(16, 8),
                                    ops=CpuOps(), timings=t)
    q.put((rank, out.numpy()[:n_out * 16].copy(), t))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_point_to_point_exchange_digit_major(world):
    """The NCCL exchange's point-to-point form (one send/receive per
    (source, digit) piece into the digit-major receive buffer), run under
    gloo: with a hot key spread over ranks the concatenation is the stable
    sort."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_p2p_ops, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, t = q.get(timeout=180)
        res[r] = (out, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([res[r][0] for r in range(world)])
    a = np.concatenate([_input(r, world, 16, 8, 0, 0.3) for r in range(world)])
    assert np.array_equal(got, oracle.stable_sort(a, 16, 8))
    assert all(res[r][1]["exchange"] == "nccl" and res[r][1]["segments"] >= 1 for r in range(world))
