"""Multi-process key-range sort with the fused partition + exchange (CUDA IPC
peer windows, raduls_gpu_partition_to) on the device.

This run has one GPU, so two (or three) processes share it: the metadata
collectives run on gloo, each process maps the others' receive windows
through CUDA IPC and the partition kernel of every rank stores its records
straight into them; no kernel waits on another rank (ranks meet only at host
barriers). Checked against the oracle's stable sort of the concatenated
inputs (rank order = input order of the concatenation).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _hot_input(data, n_local, rs, ks, rank, hot):
    """Overwrite the key of a `hot` fraction of this rank's records with one
    fixed key (a single-key bucket holding most of the records)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    sel = (torch.rand(n_local, generator=g) < hot).nonzero().flatten().to(data.device)
    key = torch.tensor([0x5A, 0x17, 0x33, 0x00, 0x42, 0x99, 0x01, 0xEE] * 3, dtype=torch.uint8,
                       device=data.device)[:ks]
    # 3% of the other records get the hot key's 16-bit prefix (as any uniform
    # input at scale does): the hot bucket is not single-key
    near = (torch.rand(n_local, generator=g) < 0.03).nonzero().flatten().to(data.device)
    data.view(n_local, rs)[near, :2] = key[:2]
    data.view(n_local, rs)[sel, :ks] = key


def _worker(rank, world, port, cfg, outdir, poke=False, exchange="p2p", hot=0.0, backend="gloo",
            special=""):
    import json

    import torch
    import torch.distributed as dist

    import paper_1612_02557_b200 as rg
    from paper_1612_02557_b200.distributed import release_peer_windows, sort_distributed
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
    n_total, rs, ks, dist_kind, seed = cfg
    lay = rg.RecordLayout(rs, ks)
    n_local = n_total // world
    base = rank * n_local
    if rank == world - 1:
        n_local = n_total - base
    for step in range(2):  # the second step reuses the cached windows
        if special == "empty_rank1" and rank == 1:
            n_local = 0
        data = rg.generate(max(n_local, 1), lay, dist=dist_kind, seed=seed, index_base=base)
        if special == "one_key":
            data.view(-1, rs)[:, :ks] = 0x5C
        if hot:
            _hot_input(data, n_local, rs, ks, rank, hot)
        if poke and rank == world - 1:
            # key byte 0 varies in one record only, past the strided AND/OR
            # sample: the sampled plan's prefix byte is wrong, the exact
            # AND/OR from the partition's histogram catches it (exact re-plan)
            data[(n_local - 1) * rs] = 1
        np.save(os.path.join(outdir, f"in{rank}.npy"), data[:n_local * rs].cpu().numpy())
        tim = {}
        out, n_out = sort_distributed(data, n_local, lay, exchange=exchange, timings=tim)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"out{rank}_{step}.npy"), out[:n_out * rs].cpu().numpy())
        with open(os.path.join(outdir, f"tim{rank}_{step}.json"), "w") as f:
            json.dump({k: v for k, v in tim.items() if isinstance(v, (int, float, str))}, f)
        dist.barrier()
    release_peer_windows()
    dist.destroy_process_group()


def _run(tmp_path, world, cfg, **kw):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cfg, str(tmp_path), kw.get("poke", False),
                                      kw.get("exchange", "p2p"), kw.get("hot", 0.0),
                                      kw.get("backend", "gloo"), kw.get("special", "")),
                       nprocs=world, join=True, start_method="spawn")


def _check(tmp_path, world, cfg):
    import json

    import oracle
    n_total, rs, ks, _, _ = cfg
    inputs = np.concatenate([np.load(tmp_path / f"in{r}.npy") for r in range(world)])
    want = oracle.stable_sort(inputs, rs, ks)
    for step in range(2):
        got = np.concatenate([np.load(tmp_path / f"out{r}_{step}.npy") for r in range(world)])
        assert got.size == inputs.size
        assert np.array_equal(got, want), f"step {step}"
    return [json.load(open(tmp_path / f"tim{r}_1.json")) for r in range(world)], \
        [np.load(tmp_path / f"out{r}_1.npy").size // rs for r in range(world)]


@pytest.mark.parametrize("world,cfg", [
    (2, (300_000, 16, 8, 0, 0x5EED0001)),
    (3, (200_001, 32, 24, 0, 0x5EED0004)),
    (2, (250_000, 16, 8, 1, 0x5EED0003)),   # C3-shaped: constant leading bytes, Zipf byte
    (2, (120_000, 8, 8, 0, 0x5EED0002)),
])
def test_distributed_p2p_exchange_matches_oracle(torch_cuda, tmp_path, world, cfg):
    _run(tmp_path, world, cfg)
    tim, _ = _check(tmp_path, world, cfg)
    assert all(t["exchange"] == "p2p" for t in tim)


@pytest.mark.parametrize("world,cfg", [
    (2, (300_000, 16, 8, 0, 0x5EED0001)),
    (3, (200_001, 32, 24, 0, 0x5EED0004)),
    (2, (250_000, 16, 8, 1, 0x5EED0003)),
])
def test_distributed_nccl_exchange_matches_oracle(torch_cuda, tmp_path, world, cfg):
    """exchange="nccl" with the CUDA DeviceOps: local partition by digit, then
    all_to_all_single (host-staged under gloo on this shared device)."""
    _run(tmp_path, world, cfg, exchange="nccl")
    tim, _ = _check(tmp_path, world, cfg)
    assert all(t["exchange"] == "nccl" for t in tim)
    assert all(t["exchange_ms"] is not None and t["partition_ms"] is not None for t in tim)


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_distributed_world1_nccl_group(torch_cuda, tmp_path, exchange):
    """A one-rank NCCL process group: the real NCCL all_to_all_single (and
    the p2p window path) on the device."""
    cfg = (400_000, 16, 8, 0, 0x5EED0005)
    _run(tmp_path, 1, cfg, exchange=exchange, backend="nccl")
    tim, _ = _check(tmp_path, 1, cfg)
    assert tim[0]["exchange"] == exchange


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_distributed_hot_single_key_is_split(torch_cuda, tmp_path, world, exchange):
    """60% of the records share one key: that single-key bucket is spread over
    ranks by count, so no rank receives much more
    than its share, and the concatenation is still the stable sort."""
    cfg = (240_000, 16, 8, 0, 0x5EED0001)
    _run(tmp_path, world, cfg, exchange=exchange, hot=0.6)
    tim, n_out = _check(tmp_path, world, cfg)
    assert all(t["hot_split_digits"] >= 1 for t in tim)
    assert max(n_out) <= cfg[0] / world * 1.05 + 16


def test_distributed_p2p_sample_misses_a_varying_byte(torch_cuda, tmp_path):
    world, cfg = 2, (250_000, 16, 8, 1, 0x5EED0003)  # bytes 0-2 constant except the poked record
    _run(tmp_path, world, cfg, poke=True)
    inputs = np.concatenate([np.load(tmp_path / f"in{r}.npy") for r in range(world)])
    assert inputs.reshape(-1, cfg[1])[:, 0].max() == 1
    _check(tmp_path, world, cfg)


def test_bench_multi_rank_line(torch_cuda, tmp_path):
    """bench.py's N>1 path (two ranks sharing this device over gloo): both
    exchanges timed, the line carries roofline, nvlink and a verified output."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RADULS_BENCH_BACKEND="gloo", RADULS_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "2",
           "--warmup", "3", "--no-e2e", "--no-per-config"]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["verified"] is True
    assert set(line["exchanges"]) == {"p2p", "nccl"}
    for e, r in line["exchanges"].items():
        assert r["verified"]["ok"], e
        assert r["nvlink"]["sent_bytes_per_gpu"] > 0 and r["nvlink"]["t_exchange_ms"] > 0
        assert r["roofline"]["frac"] > 0 and len(r["roofline"]["per_rank_frac"]) == 2
    assert line["gpu_launches"] > 0 and line["roofline_sort"]["frac"] > 0


@pytest.mark.parametrize("rs,ks", [(16, 8), (32, 24), (8, 8)])
def test_partition_pivot_digits_match_host(torch_cuda, rs, ks):
    """The device map_digit (pivot-cut hot buckets, csrc/common.cuh) against
    its host restatement (distributed.map_digits_np): per-digit counts and the
    stable partition's bytes, through raduls_gpu_partition with pivots set."""
    import paper_1612_02557_b200 as rg
    from paper_1612_02557_b200 import distributed as D
    n = 200_000
    lay = rg.RecordLayout(rs, ks)
    data = rg.generate(n, lay, seed=99)
    _hot_input(data, n, rs, ks, 0, 0.5)
    a = data.cpu().numpy().reshape(n, rs)
    w = np.bincount(D.prefix16_np(a, 0, ks), minlength=D.NBUCKETS).astype(np.float64)
    hot = D.hot_buckets(w, 4)
    piv = D.choose_pivots(a[::7, :ks].copy(), 0, ks, hot, w)
    assert len(piv) == 1
    plan = D.make_digits(w, 4, 0, pivots=piv)
    ops = D.DeviceOps()
    ops.set_pivots(plan, ks)
    try:
        out, counts = ops.partition(data, n, lay, 0, plan.bucket_digit, plan.n_digits)
        want_d = D.map_digits_np(a, 0, ks, plan)
        assert list(counts.astype(np.int64)) == list(np.bincount(want_d, minlength=plan.n_digits))
        order = np.argsort(want_d, kind="stable")
        assert np.array_equal(out[:n * rs].cpu().numpy().reshape(n, rs), a[order])
        c2 = ops.digit_counts(data, n, lay, 0, plan.bucket_digit, plan.n_digits)
        assert np.array_equal(c2.astype(np.int64), counts.astype(np.int64))
    finally:
        ops.set_pivots(D.make_digits(w, 4, 0), ks)  # clear


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_distributed_empty_rank_and_one_key(torch_cuda, tmp_path, exchange):
    """A rank with no records, and an input where every key is equal (one
    single-key bucket holding everything: spread over the ranks by count)."""
    cfg = (150_000, 16, 8, 0, 0x5EED0001)
    _run(tmp_path, 3, cfg, exchange=exchange, special="empty_rank1")
    _check(tmp_path, 3, cfg)
    _run(tmp_path / "k", 3, cfg, exchange=exchange, special="one_key") if (tmp_path / "k").mkdir() is None else None
    tim, n_out = _check(tmp_path / "k", 3, cfg)
    assert max(n_out) <= cfg[0] / 3 + 16  # one key, balanced by count
