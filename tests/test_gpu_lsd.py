"""GPU LSD baseline (raduls_gpu_lsd_sort) against the oracle.

Patterns follow the reference's own LSD tests (P/tests/test_lsd.cpp:25-84):
byte-identical to the stable reference on payload-bearing layouts with heavy
key duplication, sorted input unchanged, agreement with the MSD sorter and the
oracle, rejection of bad buffer sizes and layouts.
"""
import numpy as np
import pytest

import oracle
from helpers import ALL_LAYOUTS, from_dev, make_input, to_dev

pytestmark = pytest.mark.gpu


def lsd_copy(rg, torch, a, rs, ks, cfg=None, tmp=False):
    d = to_dev(torch, a)
    t = torch.empty_like(d) if tmp else None
    rg.lsd_sort(d, a.size // rs, rg.RecordLayout(rs, ks), cfg, tmp=t)
    torch.cuda.synchronize()
    return from_dev(d)


@pytest.mark.parametrize("rs,ks", [(16, 8), (24, 16), (32, 8)])
def test_lsd_byte_identical_to_stable_reference(rg, torch_cuda, rs, ks):
    """test_lsd.cpp:25-40: n in {0,1,2,1000,100000}, universe 256, both lane sizes."""
    for i, n in enumerate([0, 1, 2, 1000, 100000]):
        a = make_input(n, rs, ks, 808 + i, universe=256)
        want = oracle.stable_sort(a, rs, ks)
        for buf in (64, 256):
            got = lsd_copy(rg, torch_cuda, a, rs, ks, rg.LsdConfig(buf, 4), tmp=bool(i % 2))
            assert np.array_equal(got, want), (rs, ks, n, buf)


@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS)
def test_lsd_all_layouts_match_msd(rg, torch_cuda, rs, ks):
    """LSD and MSD outputs are byte-identical (both stable), keys distinct or not."""
    for universe in (0, 3000):
        a = make_input(70000, rs, ks, 99 + rs + ks, universe=universe)
        got = lsd_copy(rg, torch_cuda, a, rs, ks)
        d = to_dev(torch_cuda, a)
        rg.sort(d, a.size // rs, rg.RecordLayout(rs, ks))
        assert np.array_equal(got, from_dev(d))
        assert np.array_equal(got, oracle.stable_sort(a, rs, ks))


def test_lsd_sorted_input_unchanged(rg, torch_cuda):
    """test_lsd.cpp:42-47."""
    rs, ks = 16, 8
    srt = oracle.stable_sort(make_input(50000, rs, ks, 4, universe=1000), rs, ks)
    assert np.array_equal(lsd_copy(rg, torch_cuda, srt, rs, ks), srt)


def test_lsd_agrees_with_msd_and_oracle(rg, torch_cuda):
    """test_lsd.cpp:49-67: (16,16), 200000 records, digest preserved."""
    rs, ks, n = 16, 16, 200000
    a = make_input(n, rs, ks, 5)
    got = lsd_copy(rg, torch_cuda, a, rs, ks, rg.LsdConfig(256, 4))
    assert oracle.digest(got, rs) == oracle.digest(a, rs)
    assert np.array_equal(got, oracle.stable_sort(a, rs, ks))


def test_lsd_constant_bytes_skipped(rg, torch_cuda):
    """Constant key bytes (C3 shape) take no pass; the result is unchanged."""
    rs, ks = 16, 8
    a = make_input(1 << 18, rs, ks, 0x5EED0003, dist=oracle.DIST_SKEW)
    assert np.array_equal(lsd_copy(rg, torch_cuda, a, rs, ks), oracle.stable_sort(a, rs, ks))


def test_lsd_host_dropin(rg):
    """raduls_gpu_lsd_sort_host: host memory in place."""
    for rs, ks in [(16, 8), (8, 8), (32, 24)]:
        a = make_input(54321, rs, ks, 31 + rs, universe=500)
        b = a.copy()
        rg.lsd_sort(b, a.size // rs, rg.RecordLayout(rs, ks))
        assert np.array_equal(b, oracle.stable_sort(a, rs, ks))


def test_lsd_cpp_shim(rg):
    """raduls::gpu::lsd_sort from C++ (tests/cpp/dropin_main.cpp, lsd mode)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "dropin_main")
    if not os.path.exists(exe):
        import __graft_entry__
        __graft_entry__.build_cpp_dropin()
    for args in (["100000", "16", "8", "lsd4"], ["30000", "32", "24", "lsd1"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
