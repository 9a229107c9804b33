"""CPU: pin the oracle (oracle/raduls_oracle.c) against the reference.

* the reference's own known-answer tests (P/tests/test_record.cpp:35-59,
  P/tests/test_kernels.cpp:87-112, acceptance.cpp:172-183) restated on the
  oracle;
* committed golden fixtures produced by the unmodified reference library
  (tests/golden/make_golden.py -> reference_small.json): the oracle's
  generator reproduces every input byte for byte, its MSD restatement
  reproduces the reference's output byte for byte (T = 1), and canonical()
  agrees;
* when oracle/_ref is built (this container), live reference comparisons.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from helpers import ALL_LAYOUTS, EXTRA_LAYOUTS, make_input

HERE = os.path.dirname(os.path.abspath(__file__))
SMALL = json.load(open(os.path.join(HERE, "golden", "reference_small.json")))


def sha(a):
    return hashlib.sha256(memoryview(a)).hexdigest()


def test_digit_and_be64_kats():
    k = SMALL["kats"]
    rec = np.frombuffer(bytes.fromhex(k["digit_key"]) + bytes(8), dtype=np.uint8).copy()
    L = oracle.lib()
    p = oracle._ptr(rec)
    assert L.orc_digit(p, 8, 7) == k["digit_7"]
    assert L.orc_digit(p, 8, 0) == k["digit_0"]
    assert L.orc_digit(p, 8, 4) == k["digit_4"]
    buf = np.zeros(8, dtype=np.uint8)
    L.orc_store_be64(oracle._ptr(buf), int(k["be64_value"], 16))
    assert buf.tobytes().hex() == k["be64_bytes"]
    assert L.orc_load_be64(oracle._ptr(buf)) == int(k["be64_value"], 16)
    rng = np.random.default_rng(1)
    for _ in range(100):
        v = int(rng.integers(0, 2**63)) * 2 + 1
        L.orc_store_be64(oracle._ptr(buf), v)
        assert L.orc_load_be64(oracle._ptr(buf)) == v


def test_prefix_sum_kat():
    k = SMALL["kats"]
    counts = np.zeros(256, dtype=np.uint64)
    counts[:3] = k["prefix_counts_head"]
    offs = np.zeros(256, dtype=np.uint64)
    oracle.lib().orc_exclusive_prefix_sum(counts.ctypes.data_as(oracle._u64p),
                                          offs.ctypes.data_as(oracle._u64p))
    assert list(offs[:4]) == k["prefix_offsets_head"]
    assert offs[255] == k["prefix_last"]


def test_mix64_and_is_tiny_kats():
    k = SMALL["kats"]
    for x, want in k["mix64"].items():
        assert oracle.lib().orc_mix64(int(x)) == want
    for b, p, want in k["is_tiny"]:
        assert oracle.lib().orc_is_tiny(b, p) == want


@pytest.mark.parametrize("case", SMALL["cases"], ids=lambda c: f"{c['rs']}-{c['ks']}-{c['n']}-{c['universe']}")
def test_oracle_matches_reference_fixture(case):
    rs, ks, n = case["rs"], case["ks"], case["n"]
    a = make_input(n, rs, ks, case["seed"], case["universe"])
    assert sha(a) == case["input_sha"], "generator drifted from the fixture"
    assert list(oracle.digest(a, rs)) == case["digest"]
    out = oracle.msd_sort(a, rs, ks)
    can = oracle.canonical(out, rs, ks)
    assert sha(can) == case["canonical_sha"]
    if case["source"] == "reference" and tuple(case["ref_layout"]) == (rs, ks):
        # same algorithm, T = 1: byte-identical, payload order included
        assert sha(out) == case["ref_sha"]
    assert sha(oracle.canonical(oracle.stable_sort(a, rs, ks), rs, ks)) == case["canonical_sha"]


@pytest.mark.parametrize("v", SMALL["vectors"], ids=lambda v: f"{v['rs']}-{v['ks']}")
def test_full_vectors(v):
    a = np.frombuffer(bytes.fromhex(v["input_hex"]), dtype=np.uint8).copy()
    out = oracle.msd_sort(a, v["rs"], v["ks"])
    assert out.tobytes().hex() == v["ref_output_hex"]


@pytest.mark.parametrize("s", SMALL["splits"], ids=lambda s: f"{s['rs']}-{s['ks']}")
def test_radix_split_fixture(s):
    a = make_input(s["n"], s["rs"], s["ks"], s["seed"], 0)
    out, h = oracle.radix_split(a, s["rs"], s["byte_offset"])
    assert sha(out) == s["out_sha"]
    assert sha(h.view(np.uint8)) == s["hist_sha"]


def test_zipf_thresholds_monotone():
    t = oracle.zipf_thresholds()
    assert t[-1] == 2**53
    assert np.all(np.diff(t.astype(np.float64)) > 0)
    a = oracle.generate(1 << 16, 16, 8, oracle.DIST_SKEW, 3)
    r = a.reshape(-1, 16)
    assert np.all(r[:, :3] == 0)  # top 24 bits zero
    frac0 = np.mean(r[:, 3] == 0)
    assert 0.2 < frac0 < 0.3  # Zipf(1.2) over 256 values: P(rank 1) ~ 0.254


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("rs,ks", ALL_LAYOUTS)
def test_live_reference_threads(rs, ks):
    """Distinct keys: byte-identical across thread counts (test_scheduler.cpp:171-183)
    and identical to the oracle restatement."""
    a = make_input(200_000, rs, ks, 555 + rs)
    o = oracle.msd_sort(a, rs, ks)
    for t in (1, 4):
        assert np.array_equal(oracle.ref_sort(a, rs, ks, t), o)


@pytest.mark.parametrize("rs,ks", EXTRA_LAYOUTS)
def test_widened_layouts_oracle_consistent(rs, ks):
    """Key sizes the reference rejects: the MSD restatement agrees with the
    stable sort on the key sequence and multiset."""
    for u in (0, 3):
        a = make_input(5000, rs, ks, 9 + rs + ks, u)
        out = oracle.msd_sort(a, rs, ks)
        assert oracle.check_sorted(out, rs, ks)[0]
        assert oracle.digest(out, rs) == oracle.digest(a, rs)
        assert np.array_equal(oracle.canonical(out, rs, ks),
                              oracle.canonical(oracle.stable_sort(a, rs, ks), rs, ks))


def test_reference_rejects_bad_layouts():
    for rs, ks in [(8, 16), (12, 8), (40, 8)]:
        with pytest.raises(ValueError):
            oracle.msd_sort(np.zeros(64, dtype=np.uint8), rs, ks)
