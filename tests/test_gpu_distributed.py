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


def _worker(rank, world, port, cfg, outdir, poke=False):
    import torch
    import torch.distributed as dist

    import paper_1612_02557_b200 as rg
    from paper_1612_02557_b200.distributed import release_peer_windows, sort_distributed
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    n_total, rs, ks, dist_kind, seed = cfg
    lay = rg.RecordLayout(rs, ks)
    n_local = n_total // world
    base = rank * n_local
    if rank == world - 1:
        n_local = n_total - base
    for step in range(2):  # the second step reuses the cached windows
        data = rg.generate(n_local, lay, dist=dist_kind, seed=seed, index_base=base)
        if poke and rank == world - 1:
            # key byte 0 varies in one record only, past the strided AND/OR
            # sample: the sampled plan's prefix byte is wrong, the exact
            # AND/OR from the partition's histogram catches it (exact re-plan)
            data[(n_local - 1) * rs] = 1
        np.save(os.path.join(outdir, f"in{rank}.npy"), data.cpu().numpy())
        out, n_out = sort_distributed(data, n_local, lay, exchange="p2p")
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"out{rank}_{step}.npy"), out[:n_out * rs].cpu().numpy())
        dist.barrier()
    release_peer_windows()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, (300_000, 16, 8, 0, 0x5EED0001)),
    (3, (200_001, 32, 24, 0, 0x5EED0004)),
    (2, (250_000, 16, 8, 1, 0x5EED0003)),   # C3-shaped: constant leading bytes, Zipf byte
    (2, (120_000, 8, 8, 0, 0x5EED0002)),
])
def test_distributed_p2p_exchange_matches_oracle(torch_cuda, tmp_path, world, cfg):
    import torch.multiprocessing as mp

    import oracle
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cfg, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    n_total, rs, ks, _, _ = cfg
    inputs = np.concatenate([np.load(tmp_path / f"in{r}.npy") for r in range(world)])
    want = oracle.stable_sort(inputs, rs, ks)
    for step in range(2):
        got = np.concatenate([np.load(tmp_path / f"out{r}_{step}.npy") for r in range(world)])
        assert got.size == n_total * rs
        assert np.array_equal(got, want), f"step {step}"


def test_distributed_p2p_sample_misses_a_varying_byte(torch_cuda, tmp_path):
    import torch.multiprocessing as mp

    import oracle
    world, cfg = 2, (250_000, 16, 8, 1, 0x5EED0003)  # bytes 0-2 constant except the poked record
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cfg, str(tmp_path), True), nprocs=world,
                       join=True, start_method="spawn")
    n_total, rs, ks, _, _ = cfg
    inputs = np.concatenate([np.load(tmp_path / f"in{r}.npy") for r in range(world)])
    assert inputs.reshape(-1, rs)[:, 0].max() == 1
    want = oracle.stable_sort(inputs, rs, ks)
    for step in range(2):
        got = np.concatenate([np.load(tmp_path / f"out{r}_{step}.npy") for r in range(world)])
        assert np.array_equal(got, want), f"step {step}"
