"""Test helpers: seeded inputs (via the oracle's generator) and device I/O."""
from __future__ import annotations

import numpy as np

import oracle

ALL_LAYOUTS = [(8, 8), (16, 8), (16, 16), (24, 8), (24, 16), (32, 8), (32, 16)]  # reference set
EXTRA_LAYOUTS = [(32, 24), (16, 1), (16, 3), (24, 24), (32, 32), (8, 5), (32, 12)]  # widened


def make_input(n: int, rs: int, ks: int, seed: int, universe: int = 0,
               dist: int = oracle.DIST_UNIFORM) -> np.ndarray:
    """Seeded records; with `universe` > 0 every key word is reduced mod universe
    (the duplicate-heavy inputs of P/tests/test_util.hpp:29-46)."""
    a = oracle.generate(n, rs, ks, dist, seed)
    if universe and n:
        r = a.reshape(n, rs)
        for w in range((ks + 7) // 8):
            lo, hi = 8 * w, min(8 * w + 8, rs)
            if hi - lo < 8:
                continue
            v = r[:, lo:hi].copy().view(">u8").reshape(n) % np.uint64(universe)
            r[:, lo:hi] = v.astype(">u8").view(np.uint8).reshape(n, 8)
        # bytes of a partial last key word: clear so the universe bound holds
        if ks % 8:
            r[:, (ks // 8) * 8:ks] = 0
    return a


def to_dev(torch, a: np.ndarray):
    return torch.from_numpy(a.copy()).cuda()


def from_dev(t) -> np.ndarray:
    return t.cpu().numpy()


def keys_of(a: np.ndarray, rs: int, ks: int) -> np.ndarray:
    n = a.size // rs
    return a.reshape(n, rs)[:, :ks]
