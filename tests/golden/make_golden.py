"""Generate tests/golden/*.json from the reference library itself.

Run in the build container, where /root/reference is mounted and
oracle/Makefile has compiled the unmodified reference into
oracle/_ref/libraduls_ref.so:

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --configs  # + full-size C1-C4 hashes (minutes)
    python tests/golden/make_golden.py --c5       # + C5 per-top-byte-group hashes (long)

Inputs come from the SURVEY.md §8(d) generator (oracle/raduls_oracle.c
orc_generate, bit-identical to the CUDA k_gen); outputs from the reference's
raduls::sort (P/include/raduls/scheduler.hpp:60-61). Stored: sha256 of each
input, of the reference output and of canonical(output) (equal-key runs
ordered by full record bytes), plus a few complete small
vectors and the reference's own known-answer values.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from helpers import ALL_LAYOUTS, make_input  # noqa: E402

SIZES = [0, 1, 2, 31, 33, 100, 383, 385, 1000, 5000, 100000]
UNIVERSES = [0, 256, 2]
CONFIGS = {  # name: (n, rs, ks, dist, seed) — SURVEY.md §8(d)
    "c1": (1 << 26, 16, 8, 0, 0x5EED0001),
    "c2": (1 << 30, 8, 8, 0, 0x5EED0002),
    "c3": (1 << 29, 16, 8, 1, 0x5EED0003),
    "c4": (1 << 28, 32, 24, 0, 0x5EED0004),
    "c5": (1 << 32, 16, 8, 0, 0x5EED0005),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(memoryview(a)).hexdigest()


def ref_layout(rs: int, ks: int) -> tuple[int, int]:
    """The reference only takes ks 8/16: wider keys run as (rs, 16) — exact when
    no two adjacent outputs share their 16-byte prefix (checked)."""
    return (rs, ks) if ks in (8, 16) else (rs, 16)


def ref_sorted(a: np.ndarray, rs: int, ks: int, threads: int) -> np.ndarray:
    rrs, rks = ref_layout(rs, ks)
    out = oracle.ref_sort(a, rrs, rks, threads)
    if rks != ks:
        n = a.size // rs
        r = out.reshape(n, rs)
        if n > 1 and np.any(np.all(r[1:, :rks] == r[:-1, :rks], axis=1)):
            raise RuntimeError("proxy layout not exact: adjacent 16-byte prefixes tie")
    return out


def gen_parallel(n: int, rs: int, ks: int, dist: int, seed: int, base: int = 0,
                 threads: int = 8) -> np.ndarray:
    out = np.empty(n * rs, dtype=np.uint8)
    step = (n + threads - 1) // threads

    def work(t):
        lo = t * step
        hi = min(n, lo + step)
        if hi > lo:
            part = out[lo * rs:hi * rs]
            rc = oracle.lib().orc_generate(oracle._ptr(part), hi - lo, rs, ks, dist, seed, base + lo)
            assert rc == 0

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def small_fixtures() -> dict:
    cases = []
    i = 0
    for rs, ks in ALL_LAYOUTS + [(32, 24)]:
        for n in SIZES:
            for u in UNIVERSES:
                seed = 1000 + i
                i += 1
                a = make_input(n, rs, ks, seed, u)
                source = "reference"
                try:
                    out = ref_sorted(a, rs, ks, 1)
                except RuntimeError:
                    # ks=24 with 16-byte-prefix ties: no reference layout can order it;
                    # fall back to the stable-sort restatement of oracle_sort
                    # (P/src/verify.cpp:52-64 with compare_keys, layout.hpp:52-55)
                    out = oracle.stable_sort(a, rs, ks)
                    source = "oracle_stable_sort"
                cases.append({"rs": rs, "ks": ks, "n": n, "universe": u, "seed": seed,
                              "input_sha": sha(a), "ref_sha": sha(out),
                              "canonical_sha": sha(oracle.canonical(out, rs, ks)),
                              "digest": list(oracle.digest(a, rs)),
                              "ref_layout": list(ref_layout(rs, ks)), "source": source})
    vectors = []
    for rs, ks in ALL_LAYOUTS:
        a = make_input(64, rs, ks, 77 + rs + ks, 16)
        out = ref_sorted(a, rs, ks, 1)
        vectors.append({"rs": rs, "ks": ks, "n": 64, "input_hex": a.tobytes().hex(),
                        "ref_output_hex": out.tobytes().hex()})
    R = oracle.ref()
    kats = {
        # P/tests/test_record.cpp:35-46: key bytes 01..08 -> digit 7 = 0x01, digit 0 = 0x08
        "digit_key": "0102030405060708", "digit_7": 1, "digit_0": 8, "digit_4": 4,
        # P/tests/test_record.cpp:48-59
        "be64_value": "0102030405060708", "be64_bytes": "0102030405060708",
        # P/tests/test_kernels.cpp:92-100: counts [3,0,2,0...] -> offsets [0,3,3,5,...,5]
        "prefix_counts_head": [3, 0, 2], "prefix_offsets_head": [0, 3, 3, 5], "prefix_last": 5,
        # mix64 (P/include/raduls/datagen.hpp:37-42) from the reference build
        "mix64": {str(x): int(R.ref_mix64(x)) for x in [0, 1, 2, 0x5EED0001, 2**63, 2**64 - 1]},
        # is_tiny table (P/tests/acceptance.cpp:172-183)
        "is_tiny": [[b, p, int(R.ref_is_tiny(b, p))] for b, p in
                    [(300, 1000), (383, 1000), (384, 1000), (100, 10000), (31, 31 * 16 + 1),
                     (32, 32 * 16 + 1), (100, 1600), (100, 1601), (0, 0), (383, 0), (384, 0)]],
    }
    # radix_split (P/include/raduls/kernels.hpp:157-167) byte-exact on a few inputs
    splits = []
    for rs, ks in ALL_LAYOUTS:
        a = make_input(3000, rs, ks, 4242 + rs, 0)
        off = (rs + ks) % ks
        out = np.empty_like(a)
        h = np.zeros(256, dtype=np.uint64)
        rc = R.ref_radix_split(oracle._ptr(a), oracle._ptr(out), 3000, rs, ks, off,
                               h.ctypes.data_as(oracle._u64p))
        assert rc == 0
        splits.append({"rs": rs, "ks": ks, "n": 3000, "seed": 4242 + rs, "byte_offset": off,
                       "out_sha": sha(out), "hist_sha": sha(h.view(np.uint8))})
    return {"generator": "SURVEY.md §8(d) (oracle/raduls_oracle.c orc_generate)",
            "reference": "oracle/_ref/libraduls_ref.so (raduls::sort, T=1)",
            "cases": cases, "vectors": vectors, "kats": kats, "splits": splits}


def config_fixture(name: str, threads: int = 8) -> dict:
    n, rs, ks, dist, seed = CONFIGS[name]
    a = gen_parallel(n, rs, ks, dist, seed)
    d = oracle.digest(a, rs)
    out = ref_sorted(a, rs, ks, threads)
    del a
    can = oracle.canonical(out, rs, ks)
    res = {"n": n, "rs": rs, "ks": ks, "dist": dist, "seed": seed, "digest": list(d),
           "ref_layout": list(ref_layout(rs, ks)), "canonical_sha": sha(can),
           "first_record_hex": can[:rs].tobytes().hex(),
           "last_record_hex": can[-rs:].tobytes().hex()}
    return res


def c5_fixture(threads: int = 8, groups: int = 8) -> dict:
    """Exact chunked oracle: the sorted C5 output is
    partitioned by the key's top byte; group g holds top bytes [g*256/G, (g+1)*256/G)."""
    n, rs, ks, dist, seed = CONFIGS["c5"]
    chunk = 1 << 26
    res = {"n": n, "rs": rs, "ks": ks, "dist": dist, "seed": seed, "groups": []}
    width = 256 // groups
    for g in range(groups):
        parts = []
        for c0 in range(0, n, chunk):
            a = gen_parallel(min(chunk, n - c0), rs, ks, dist, seed, c0, threads)
            r = a.reshape(-1, rs)
            sel = (r[:, 0] >= g * width) & (r[:, 0] < (g + 1) * width)
            parts.append(r[sel].copy())
        sub = np.concatenate(parts).reshape(-1)
        del parts
        out = ref_sorted(sub, rs, ks, threads)
        del sub
        can = oracle.canonical(out, rs, ks)
        res["groups"].append({"top_byte_lo": g * width, "top_byte_hi": (g + 1) * width,
                              "records": can.size // rs, "canonical_sha": sha(can)})
        print(f"c5 group {g}: {can.size // rs} records", flush=True)
        del out, can
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", action="store_true")
    ap.add_argument("--c5", action="store_true")
    args = ap.parse_args()
    if not oracle.ref_available():
        sys.exit("oracle/_ref/libraduls_ref.so missing: run `make -C oracle` with /root/reference mounted")
    with open(os.path.join(HERE, "reference_small.json"), "w") as f:
        json.dump(small_fixtures(), f, indent=1)
    print("wrote reference_small.json")
    if args.configs:
        path = os.path.join(HERE, "reference_configs.json")
        cur = json.load(open(path)) if os.path.exists(path) else {}
        for name in ["c1", "c2", "c3", "c4"]:
            cur[name] = config_fixture(name)
            print("config", name, cur[name]["canonical_sha"][:16], flush=True)
            with open(path, "w") as f:
                json.dump(cur, f, indent=1)
    if args.c5:
        path = os.path.join(HERE, "reference_configs.json")
        cur = json.load(open(path)) if os.path.exists(path) else {}
        cur["c5"] = c5_fixture()
        with open(path, "w") as f:
            json.dump(cur, f, indent=1)


if __name__ == "__main__":
    main()
