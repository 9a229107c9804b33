"""Workload for compute-sanitizer (scripts/sanitize.sh) and for the checked build
(RADULS_GPU_LIB=checked; tests/test_gpu_checked.py): every kernel family of
libraduls_gpu.so on small C1-, C2-, C3- and C4-shaped inputs, checked against
the oracle so a run that "passes" the tool also sorted correctly.

Kernels reached: k_sample_andor, k_set_seg0/k_check_seg0, k_tile_hist (TMA
ring, rs 16/24/32), k_tile_hist_reg (rs 8), k_tile_hist_nd (digit-array
levels), k_tile_scan (look-back), k_plan, k_scatter (plain, digit-array
TMA at rs 32, map, peer; atomic and ballot ranking), k_local_bm (bitmap local
sort: clean and dirty words), k_local_bm_med (single bins above the primary
capacity), k_local_bm8 (8-B records), k_local_list (bucket sort over the
handed-over groups), k_local (the bucket sort alone with
RADULS_GPU_LOCAL=bucket, and the LSD fallback), k_copy_back, k_publish, k_rank_selftest, k_gen, k_digest,
k_check_sorted, k_andor, k_prefix_hist, k_sample_prefix_hist, k_map_to_u8.

    python scripts/sanitize_driver.py [--quick]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1612_02557_b200 as rg  # noqa: E402
from helpers import make_input  # noqa: E402


def check_sort(a, rs, ks, tag):
    n = a.size // rs
    d = torch.from_numpy(a.copy()).cuda()
    rg.sort(d, n, rg.RecordLayout(rs, ks))
    torch.cuda.synchronize()
    got = d.cpu().numpy()
    assert np.array_equal(got, oracle.stable_sort(a, rs, ks)), tag
    print("ok", tag, flush=True)


def main():
    quick = "--quick" in sys.argv
    sh = 1 if quick else 0
    # C1-shaped: (16,8) uniform, two scatter levels + local sort (+ digit array)
    check_sort(make_input(1 << (19 - sh), 16, 8, 0x5EED0001), 16, 8, "c1-shape")
    # C2-shaped: (8,8) key-only, register histogram + register local sort
    check_sort(make_input(1 << (20 - sh), 8, 8, 0x5EED0002), 8, 8, "c2-shape")
    # C3-shaped: skewed, constant leading bytes skipped, unbalanced bins
    check_sort(make_input(1 << (19 - sh), 16, 8, 0x5EED0003, dist=oracle.DIST_SKEW), 16, 8, "c3-shape")
    # C4-shaped: (32,24), digit-array TMA loads in the scatter
    check_sort(make_input(1 << (18 - sh), 32, 24, 0x5EED0004), 32, 24, "c4-shape")
    # (24,16)
    check_sort(make_input(1 << (17 - sh), 24, 16, 0x5EED0005), 24, 16, "rs24")
    # duplicate-heavy: shared cells outgrow the lists -> bucket sort; crowded
    # buckets -> the LSD fallback instance
    check_sort(make_input(200_000, 16, 8, 9, universe=3000), 16, 8, "fallback")
    check_sort(make_input(200_000, 8, 8, 9, universe=3000), 8, 8, "fallback-8")
    check_sort(make_input(150_000, 16, 8, 10, universe=60_000), 16, 8, "pairs")
    # bins of ~3000 16-B records: groups of their own for the big bitmap instance
    a = make_input(48 * 3000, 16, 8, 0x3ED)
    r = a.reshape(-1, 16)
    r[:, 0] = 0
    r[:, 1] = np.repeat(np.arange(48, dtype=np.uint8), 3000)[np.random.default_rng(3).permutation(48 * 3000)]
    check_sort(a, 16, 8, "medium-bins")
    # the bucket sort alone (every group), as before the bitmap sort
    os.environ["RADULS_GPU_LOCAL"] = "bucket"
    check_sort(make_input(1 << (18 - sh), 16, 8, 0x5EED0011), 16, 8, "bucket-16")
    check_sort(make_input(1 << (18 - sh), 8, 8, 0x5EED0012), 8, 8, "bucket-8")
    check_sort(make_input(1 << (17 - sh), 32, 24, 0x5EED0013), 32, 24, "bucket-32")
    del os.environ["RADULS_GPU_LOCAL"]
    # constant trailing key byte after a split -> copy-back of finished bins
    a = make_input(1 << 17, 16, 2, 42)
    r = a.reshape(-1, 16)
    r[:, 0] &= 3
    r[:, 1] = 0x11
    check_sort(a, 16, 2, "copy-back")
    # LSD baseline (ballot ranking) and the single split
    a = make_input(100_000, 16, 8, 5, universe=500)
    d = torch.from_numpy(a.copy()).cuda()
    rg.lsd_sort(d, 100_000, rg.RecordLayout(16, 8))
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), oracle.stable_sort(a, 16, 8))
    print("ok lsd", flush=True)
    src = torch.from_numpy(a.copy()).cuda()
    dst = torch.empty_like(src)
    rg.split(src, dst, 100_000, 16, 3)
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), oracle.radix_split(a, 16, 3)[0])
    print("ok split", flush=True)
    # multi-GPU building blocks on one device: partition (map), partition_to
    # (peer stores into this device's own buffers), histograms, AND/OR
    from paper_1612_02557_b200.distributed import DeviceOps, balanced_bucket_map
    n, rs, ks = 150_000, 16, 8
    a = make_input(n, rs, ks, 77)
    ops = DeviceOps()
    lay = rg.RecordLayout(rs, ks)
    d = torch.from_numpy(a.copy()).cuda()
    ops.andor(d, n, lay)
    h = ops.prefix_hist(d, n, lay, 0).cpu().numpy().astype(np.uint64)
    ops.sample_andor(d, n, lay, 4096)
    ops.sample_prefix_hist(d, n, lay, 0, 4096)
    bmap = balanced_bucket_map(h, 3)
    send, counts = ops.partition(d, n, lay, 0, bmap, 3)
    outs = [torch.empty(int(c) * rs + 16, dtype=torch.uint8, device="cuda") for c in counts]
    dst = np.array([o.data_ptr() for o in outs], dtype=np.uint64)
    got = ops.partition_to(d, n, lay, 0, bmap, 3, dst)
    assert np.array_equal(got, counts)
    cat = torch.cat([o[: int(c) * rs] for o, c in zip(outs, counts)])
    torch.cuda.synchronize()
    assert torch.equal(cat, send[: n * rs])
    c2, _ = ops.partition_plan(d, n, lay, 0, bmap, 3)
    ops.partition_store(d, n, lay, dst)
    torch.cuda.synchronize()
    print("ok partition", flush=True)
    g = rg.generate(1000, lay, seed=1)
    rg.digest(g, 1000, rs)
    rg.check_sorted(g, 1000, lay)
    print("ok utilities", flush=True)
    import ctypes as C
    rep = np.zeros(6, dtype=np.uint64)
    if rg._lib.load().raduls_gpu_check_report(rep.ctypes.data_as(C.POINTER(C.c_uint64))) == 1:
        print(f"checked build: calls {int(rep[5])} violations {int(rep[0])} timeouts {int(rep[4])}", flush=True)
        assert rep[0] == 0 and rep[4] == 0, rep
    print("DRIVER OK", flush=True)


if __name__ == "__main__":
    main()
