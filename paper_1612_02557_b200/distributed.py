"""Multi-GPU key-range partition sort; one process per GPU.

The reference is single-address-space (P/include/raduls/task_queue.hpp,
std::thread workers); MSD bins are independent once the top-prefix partition
is fixed (children tile the parent, P/include/raduls/kernels.hpp:82-94), so
the sort shards with ONE exchange step:

 1. AND/OR of the local key words, all-gathered -> the global first varying
    key byte p0 (constant leading bytes — C3's three zero bytes — are
    skipped, (e));
 2. 65 536-bucket histogram of the 16-bit prefix at key bytes (p0, p0+1),
    all-gathered: every rank learns the global distribution;
 3. bucket -> digit map (DigitPlan): contiguous bucket ranges balanced by
    record count, one digit per rank range; a hot bucket (more than
    1/(HOT_SHARE * world) of the records) gets a digit of its own, and when
    its records provably share one key (raduls_gpu_digit_andor) that digit is
    spread over consecutive ranks by count — SURVEY.md §8(e) step 4 "only a
    single-key bucket may be split" — so one hot key cannot overload a rank;
    equal keys keep their global (rank, position) order;
 4. stable local partition into per-destination send ranges on the device
    (the same tile histogram / look-back scan / scatter kernels as an MSD
    level);
 5. the exchange: by default the partition kernel itself stores every
    destination's records into that rank's receive window over NVLink (CUDA
    IPC mappings), so partition and all-to-all are one kernel; or a local
    partition plus one NCCL all-to-all;
 6. each rank sorts what it received (raduls_gpu_sort).

On the default (NVLink window) path, steps 1-2 read strided samples only
(plan_exchange_sampled): the map only has to be balanced. The exact
per-destination counts (for the window offsets) and the exact AND/OR (to
confirm p0) come from the partition's own tile histogram
(raduls_gpu_partition_plan) and are all-gathered before the stores
(raduls_gpu_partition_store), so the data is read twice before the local
sort (histogram + stores) instead of four times. A byte that varies only off
the sample makes every rank re-plan exactly (plan_exchange).

Rank r ends up holding the r-th contiguous key range, sorted; the concatenation
over ranks is the sorted whole. The collective plumbing is torch.distributed;
the per-rank compute is the CUDA library behind `DeviceOps`. `DeviceOps` is
the only product implementation; tests substitute a CPU stand-in for the
per-rank compute to exercise the host logic and collectives with gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .raduls import RecordLayout, _raise

NBUCKETS = 65536


# ---------------------------------------------------------------- host logic

def first_varying_byte(andor_per_rank: np.ndarray, ks: int) -> int:
    """andor_per_rank: [ranks, 8] u64 (and at 2w, or at 2w+1 per rank, little-endian
    record words). Returns the first key byte that is not constant over all
    ranks' records, or ks when every key is equal."""
    a = np.bitwise_and.reduce(andor_per_rank[:, 0::2].astype(np.uint64), axis=0)
    o = np.bitwise_or.reduce(andor_per_rank[:, 1::2].astype(np.uint64), axis=0)
    diff = a ^ o
    for b in range(ks):
        if (int(diff[b >> 3]) >> ((b & 7) * 8)) & 0xFF:
            return b
    return ks


def balanced_bucket_map(global_hist: np.ndarray, world: int) -> np.ndarray:
    """Contiguous bucket ranges per rank, balanced by record count: bucket b
    goes to the rank whose ideal share [r*N/W, (r+1)*N/W) holds the bucket's
    midpoint. Monotone in b, so rank r receives a contiguous key range."""
    h = np.asarray(global_hist, dtype=np.float64)
    c = np.cumsum(h)
    total = c[-1]
    if total == 0:
        return np.zeros(NBUCKETS, dtype=np.uint32)
    # mid = (prefix before b) + h_b / 2; rank = floor(mid * world / total),
    # in place and in the same operation order as the C++ planner
    c -= h
    c += h / 2.0
    c *= world
    c /= total
    r = c.astype(np.uint32)  # non-negative: truncation is floor
    np.minimum(r, world - 1, out=r)
    return r


HOT_SHARE = 4  # a bucket with more than total / (HOT_SHARE * world) records is hot
MAX_PIVOTS = 16  # raduls_gpu_set_pivots
SAMPLE_KEYS = 4096  # keys sampled per rank to find a hot bucket's pivot (its most common key)


@dataclass
class DigitPlan:
    """The partition's digits: digit = bucket_digit[16-bit prefix at p0],
    except in a pivot bucket, whose records get digit d, d+1 or d+2 for a key
    below, equal to or above the pivot key (map_digit, csrc/common.cuh).
    Digits are monotone in key order. hot[d]: a hot bucket's digit whose
    single-key-ness is unknown (checked with digit_andor before any split);
    single[d]: a pivot's equal digit — one key by construction."""
    p0: int
    bucket_digit: np.ndarray   # [65536] u32
    n_digits: int
    hot: np.ndarray            # [n_digits] bool
    single: np.ndarray = None  # [n_digits] bool
    pivots: list = None        # [(digit d of the "below" part, key bytes)]
    first_byte: np.ndarray = None  # [n_digits] u8: key bytes before it are equal within the digit

    def __post_init__(self):
        if self.single is None:
            self.single = np.zeros(self.n_digits, dtype=bool)
        if self.pivots is None:
            self.pivots = []


def hot_buckets(weights: np.ndarray, world: int) -> np.ndarray:
    w = np.asarray(weights, dtype=np.float64)
    total = w.sum()
    if world <= 1 or total <= 0:
        return np.zeros(NBUCKETS, dtype=bool)
    return w > total / (HOT_SHARE * world)


def make_digits(weights: np.ndarray, world: int, p0: int = 0, split_hot: bool = True,
                pivots: dict | None = None, ks: int | None = None, align: bool = False) -> DigitPlan:
    """Digits from global bucket weights (exact counts or sample estimates):
    each rank's contiguous bucket range (balanced_bucket_map) is one digit,
    except that every hot bucket is a digit of its own — three digits
    (below / equal / above) when `pivots` names a pivot key for it.

    align: digits also end where key byte p0 changes (every 256 buckets), as
    far as 256 digits allow (the lightest byte-p0 boundaries are dropped
    first), so that within most digits byte p0 is constant and the receiver
    can sort each digit's run from byte p0 + 1 on (first_byte; needs ks)."""
    w = np.asarray(weights, dtype=np.float64)
    rank = balanced_bucket_map(w, world).astype(np.int64)
    hot = hot_buckets(w, world) if split_hot else np.zeros(NBUCKETS, dtype=bool)
    piv = np.zeros(NBUCKETS, dtype=bool)
    if split_hot and pivots:
        for b in pivots:
            if hot[b]:
                piv[b] = True
    change = np.zeros(NBUCKETS, dtype=bool)
    change[1:] = (rank[1:] != rank[:-1]) | hot[1:] | hot[:-1]
    if align:
        budget = 256 - (1 + int(change.sum()) + 2 * int(piv.sum()))
        cand = [b for b in range(256, NBUCKETS, 256) if not change[b]]
        if budget < len(cand):  # keep the boundaries between the heaviest byte-p0 blocks
            blk = w.reshape(256, 256).sum(axis=1)
            cand.sort(key=lambda b: -(blk[(b >> 8) - 1] + blk[b >> 8]))
            cand = cand[:max(budget, 0)]
        change[cand] = True
    # digit of every bucket from the run lengths between cuts; two more digits
    # per earlier pivot bucket (its equal and above parts)
    cuts = np.flatnonzero(change)
    lengths = np.diff(np.concatenate([[0], cuts, [NBUCKETS]]))
    runs = np.arange(len(lengths), dtype=np.int64)
    pruns = np.searchsorted(cuts, np.flatnonzero(piv), side="right")  # the run of each pivot bucket
    run_digit = runs + 2 * np.searchsorted(pruns, runs, side="left")
    digit = np.repeat(run_digit.astype(np.uint32), lengths)
    n_digits = int(digit[-1]) + 1 + (2 if piv[-1] else 0)
    if n_digits > 256:  # too many ranks for separate hot digits: whole buckets only
        return make_digits(weights, world, p0, split_hot=False, ks=ks, align=align)
    dhot = np.zeros(n_digits, dtype=bool)
    single = np.zeros(n_digits, dtype=bool)
    plist = []
    for b in np.nonzero(hot)[0]:
        d = int(digit[b])
        if piv[b]:
            single[d + 1] = True
            plist.append((d, bytes(pivots[int(b)])))
        else:
            dhot[d] = True
    plan = DigitPlan(p0, digit, n_digits, dhot, single, plist)
    if ks is not None:
        # first key byte that may vary inside each digit's records
        # digit is non-decreasing in the bucket: each digit's bucket range
        dr = np.arange(n_digits)
        b_lo = np.searchsorted(digit, dr, side="left").astype(np.int64)
        b_hi = np.searchsorted(digit, dr, side="right").astype(np.int64) - 1
        has = b_hi >= b_lo
        fb = np.full(n_digits, p0, dtype=np.int64)
        fb[has & ((b_lo >> 8) == (b_hi >> 8))] = p0 + 1  # one value of byte p0
        fb[has & (b_lo == b_hi)] = p0 + 2                # one 16-bit bucket
        for d, _ in plist:
            fb[d] = fb[d + 2] = p0 + 2
            fb[d + 1] = ks  # the pivot key itself: one key
        plan.first_byte = np.minimum(fb, ks).astype(np.uint8)
    return plan


def prefix16_np(keys: np.ndarray, p0: int, ks: int) -> np.ndarray:
    """16-bit big-endian key prefix at bytes (p0, p0+1) of [n, >=ks] u8 keys."""
    hi = keys[:, p0].astype(np.int64) if p0 < ks else np.zeros(len(keys), np.int64)
    lo = keys[:, p0 + 1].astype(np.int64) if p0 + 1 < ks else np.zeros(len(keys), np.int64)
    return (hi << 8) | lo


def choose_pivots(keys: np.ndarray, p0: int, ks: int, hot: np.ndarray, weights: np.ndarray) -> dict:
    """Pivot key per hot bucket: the most common key among the sampled keys
    ([S, ks] u8, every rank's) that fall into it; at most MAX_PIVOTS, the
    heaviest buckets first."""
    if not hot.any() or len(keys) == 0:
        return {}
    pre = prefix16_np(keys, p0, ks)
    order = sorted(np.nonzero(hot)[0], key=lambda b: -weights[b])[:MAX_PIVOTS]
    out = {}
    for b in order:
        sel = keys[pre == b]
        if len(sel) == 0:
            continue
        u, c = np.unique(sel[:, :ks], axis=0, return_counts=True)
        out[int(b)] = u[int(np.argmax(c))].tobytes()
    return out


def map_digits_np(keys: np.ndarray, p0: int, ks: int, digits: "DigitPlan") -> np.ndarray:
    """Host restatement of map_digit (csrc/common.cuh) for [n, >=ks] u8 keys
    (the CPU stand-in of the tests and plan checks)."""
    d = digits.bucket_digit[prefix16_np(keys, p0, ks)].astype(np.int64)
    for pd, key in digits.pivots:
        sel = d == pd
        if not sel.any():
            continue
        k = keys[sel, :ks]
        pk = np.frombuffer(key, dtype=np.uint8)[:ks]
        neq = k != pk
        first = np.where(neq.any(axis=1), neq.argmax(axis=1), ks)
        rows = np.arange(len(k))
        below = np.zeros(len(k), dtype=bool)
        m = first < ks
        below[m] = k[rows[m], first[m]] < pk[first[m]]
        d[sel] = np.where(first == ks, pd + 1, np.where(below, pd, pd + 2))
    return d


def assign_pieces(M: np.ndarray, splittable: np.ndarray, world: int):
    """Destination ranks of every digit's records, from the exact counts
    M[source, digit]. Returns (pieces, S): pieces[s] is the list of
    (digit, rank, count) for source s in digit order (a digit's pieces in
    rank order), S[s, r] the records source s sends to rank r.

    Global order = digit order, inside a digit source order then position (the
    stable order of the concatenated inputs). A plain digit goes whole to the
    rank holding its midpoint; a splittable digit (one key) is cut at the
    ideal rank boundaries ceil(k N / world), clamped to the ranks of its
    plain neighbours so the ranks stay monotone."""
    M = np.asarray(M, dtype=np.int64)
    G, D = M.shape
    C = M.sum(axis=0)
    N = int(C.sum())
    P = np.concatenate([[0], np.cumsum(C)[:-1]]).astype(np.int64)
    rank = np.zeros(D, dtype=np.int64)
    if N:
        rank = np.minimum((2 * P + C) * world // (2 * N), world - 1)
    plain = ~np.asarray(splittable, dtype=bool)
    S = np.zeros((G, world), dtype=np.int64)
    # plain digits: whole, to rank[d] (vectorised)
    Mp = np.where(plain[None, :], M, 0)
    for r in range(world):
        S[:, r] = Mp[:, rank == r].sum(axis=1)
    per = {s_: [] for s_ in range(G)}  # s -> [(d, k, c)]
    for s_ in range(G):
        ds = np.nonzero(Mp[s_] > 0)[0]
        per[s_] = list(zip(ds.tolist(), rank[ds].tolist(), Mp[s_, ds].tolist()))
    split_ds = [d for d in np.nonzero(~plain & (C > 0))[0]]
    if split_ds:
        bound = [(k * N + world - 1) // world for k in range(world + 1)]  # first position of rank k
        live = np.nonzero(plain & (C > 0))[0]
        for d in split_ds:
            i = np.searchsorted(live, d)
            r_lo = int(rank[live[i - 1]]) if i > 0 else 0
            r_hi = int(rank[live[i]]) if i < len(live) else world - 1
            start = int(P[d])
            for s_ in range(G):
                a = start
                b = a + int(M[s_, d])
                start = b
                for k in range(r_lo, r_hi + 1):
                    lo = a if k == r_lo else max(a, bound[k])
                    hi = b if k == r_hi else min(b, bound[k + 1])
                    if hi > lo:
                        per[s_].append((int(d), k, hi - lo))
                        S[s_, k] += hi - lo
        for s_ in range(G):
            per[s_].sort(key=lambda t: (t[0], t[1]))
    pieces = [per[s_] for s_ in range(G)]
    return pieces, S


@dataclass
class ExchangePlan:
    digits: DigitPlan
    M: np.ndarray                # [world, n_digits] records source -> digit
    pieces: list                 # per source: [(digit, rank, count)] in digit order
    matrix: np.ndarray           # [world, world] records source -> destination rank

    @property
    def p0(self) -> int:
        return self.digits.p0

    def send_counts(self, rank: int) -> np.ndarray:
        return self.matrix[rank]

    def recv_counts(self, rank: int) -> np.ndarray:
        return self.matrix[:, rank]


# ---------------------------------------------------------------- per-rank compute

class DeviceOps:
    """Per-rank compute on the local GPU through the C-ABI (the product path)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.L = _lib.load()

    def empty(self, nbytes: int):
        return self.torch.empty(nbytes, dtype=self.torch.uint8, device=self.device)

    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def andor(self, data, n: int, layout: RecordLayout) -> np.ndarray:
        out = np.zeros(8, dtype=np.uint64)
        _raise(self.L.raduls_gpu_andor(data.data_ptr(), n, layout.record_size,
                                       out.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_andor")
        return out

    def prefix_hist(self, data, n: int, layout: RecordLayout, p0: int):
        h = self.torch.zeros(NBUCKETS, dtype=self.torch.int64, device=self.device)
        _raise(self.L.raduls_gpu_prefix_histogram(data.data_ptr(), n, layout.record_size,
                                                  layout.key_size, p0, h.data_ptr(),
                                                  self.stream()),
               "raduls_gpu_prefix_histogram")
        return h

    def partition(self, data, n: int, layout: RecordLayout, p0: int, bucket_rank: np.ndarray,
                  world: int):
        out = self.empty(n * layout.record_size)
        dmap = self.torch.from_numpy(bucket_rank.astype(np.int32)).to(self.device)
        counts = np.zeros(world, dtype=np.uint64)
        _raise(self.L.raduls_gpu_partition(data.data_ptr(), out.data_ptr(), n, layout.record_size,
                                           layout.key_size, p0, dmap.data_ptr(), world,
                                           counts.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_partition")
        return out, counts

    def partition_to(self, data, n: int, layout: RecordLayout, p0: int, bucket_rank: np.ndarray,
                     world: int, dst: np.ndarray) -> np.ndarray:
        """Partition fused with the exchange: rank r's records go to address dst[r]."""
        dmap = self.torch.from_numpy(bucket_rank.astype(np.int32)).to(self.device)
        counts = np.zeros(world, dtype=np.uint64)
        _raise(self.L.raduls_gpu_partition_to(data.data_ptr(), n, layout.record_size, layout.key_size,
                                              p0, dmap.data_ptr(), world,
                                              dst.ctypes.data_as(_lib._u64p),
                                              counts.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_partition_to")
        return counts

    def sample_andor(self, data, n: int, layout: RecordLayout, samples: int) -> np.ndarray:
        out = np.zeros(8, dtype=np.uint64)
        _raise(self.L.raduls_gpu_sample_andor(data.data_ptr(), n, layout.record_size, samples,
                                              out.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_sample_andor")
        return out

    def sample_prefix_hist(self, data, n: int, layout: RecordLayout, p0: int, samples: int):
        h = self.torch.zeros(NBUCKETS, dtype=self.torch.int64, device=self.device)
        _raise(self.L.raduls_gpu_sample_prefix_histogram(data.data_ptr(), n, layout.record_size,
                                                         layout.key_size, p0, samples, h.data_ptr(),
                                                         self.stream()),
               "raduls_gpu_sample_prefix_histogram")
        return h

    def partition_plan(self, data, n: int, layout: RecordLayout, p0: int, bucket_rank: np.ndarray,
                       world: int):
        """Exact per-destination counts and the AND/OR of every record word
        (one read); the stores follow in partition_store."""
        dmap = self.torch.from_numpy(bucket_rank.astype(np.int32)).to(self.device)
        counts = np.zeros(world, dtype=np.uint64)
        andor = np.zeros(8, dtype=np.uint64)
        _raise(self.L.raduls_gpu_partition_plan(data.data_ptr(), n, layout.record_size, layout.key_size,
                                                p0, dmap.data_ptr(), world,
                                                counts.ctypes.data_as(_lib._u64p),
                                                andor.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_partition_plan")
        return counts, andor

    def partition_store(self, data, n: int, layout: RecordLayout, dst: np.ndarray) -> None:
        _raise(self.L.raduls_gpu_partition_store(data.data_ptr(), n, layout.record_size, layout.key_size,
                                                 dst.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_partition_store")

    def digit_andor(self, data, n: int, layout: RecordLayout, p0: int, bucket_digit: np.ndarray,
                    hot: np.ndarray) -> np.ndarray:
        """[n_digits, 8] AND/OR of the key words of each flagged digit's records."""
        nd = len(hot)
        dmap = self.torch.from_numpy(bucket_digit.astype(np.int32)).to(self.device)
        flags = np.ascontiguousarray(hot.astype(np.uint8))
        out = np.zeros((nd, 8), dtype=np.uint64)
        _raise(self.L.raduls_gpu_digit_andor(data.data_ptr(), n, layout.record_size, layout.key_size, p0,
                                             dmap.data_ptr(), nd, flags.ctypes.data,
                                             out.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_digit_andor")
        return out

    def partition_store_pieces(self, data, n: int, layout: RecordLayout, digit: np.ndarray,
                               count: np.ndarray, dst: np.ndarray) -> None:
        digit = np.ascontiguousarray(digit, dtype=np.uint32)
        count = np.ascontiguousarray(count, dtype=np.uint64)
        dst = np.ascontiguousarray(dst, dtype=np.uint64)
        _raise(self.L.raduls_gpu_partition_store_pieces(data.data_ptr(), n, layout.record_size,
                                                        layout.key_size, len(digit), digit.ctypes.data,
                                                        count.ctypes.data_as(_lib._u64p),
                                                        dst.ctypes.data_as(_lib._u64p), self.stream()),
               "raduls_gpu_partition_store_pieces")

    def set_pivots(self, digits: DigitPlan, ks: int) -> None:
        """The plan's pivot keys for every later bucket-map call (raduls_gpu_set_pivots)."""
        k = len(digits.pivots)
        dg = np.array([d for d, _ in digits.pivots] or [0], dtype=np.uint32)
        keys = np.frombuffer(b"".join(key[:ks] for _, key in digits.pivots) or b"\0", dtype=np.uint8).copy()
        _raise(self.L.raduls_gpu_set_pivots(k, dg.ctypes.data, keys.ctypes.data, ks), "raduls_gpu_set_pivots")

    def sample_keys(self, data, n: int, layout: RecordLayout, samples: int) -> np.ndarray:
        """Key bytes of a strided sample of min(n, samples) records ([S, ks] u8)."""
        rs, ks = layout.record_size, layout.key_size
        s = min(n, samples)
        if s == 0:
            return np.zeros((0, ks), dtype=np.uint8)
        idx = (self.torch.arange(s, device=self.device, dtype=self.torch.int64) * (n // s))
        return data[:n * rs].view(n, rs)[idx, :ks].cpu().numpy()

    def digit_counts(self, data, n: int, layout: RecordLayout, p0: int, bucket_digit: np.ndarray,
                     n_digits: int) -> np.ndarray:
        """Exact records per digit (the partition's own histogram, pivots applied)."""
        counts, _ = self.partition_plan(data, n, layout, p0, bucket_digit, n_digits)
        return counts

    def sort_segments(self, data, n: int, layout: RecordLayout, sizes, first_bytes, tmp=None) -> None:
        """raduls_gpu_sort_segments: n records already in key-ordered segments."""
        sz = np.ascontiguousarray(sizes, dtype=np.uint64)
        fb = np.ascontiguousarray(first_bytes, dtype=np.uint8)
        _raise(self.L.raduls_gpu_sort_segments(data.data_ptr(), tmp.data_ptr() if tmp is not None else None,
                                               n, layout.record_size, layout.key_size, len(sz),
                                               sz.ctypes.data_as(_lib._u64p), fb.ctypes.data, self.stream()),
               "raduls_gpu_sort_segments")

    def sort(self, data, n: int, layout: RecordLayout, tmp=None) -> None:
        _raise(self.L.raduls_gpu_sort(data.data_ptr(), tmp.data_ptr() if tmp is not None else None,
                                      n, layout.record_size, layout.key_size, self.stream()),
               "raduls_gpu_sort")


# ---------------------------------------------------------------- driver

def _coll_device(data, group):
    """Metadata collectives run on the data's device under NCCL, on the host otherwise (gloo)."""
    import torch
    import torch.distributed as dist
    return data.device if dist.get_backend(group) == "nccl" else torch.device("cpu")


def _all_gather_np(arr: np.ndarray, dev, group) -> np.ndarray:
    """All-gather of a fixed-size u64/i64 numpy row -> [world, ...] numpy."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).to(dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return np.stack([o.cpu().numpy() for o in out]).view(arr.dtype)


def _key_bytes_constant(andor: np.ndarray, ks: int) -> bool:
    """andor: [8] u64 (and at 2w, or at 2w+1): every key byte constant?"""
    for b in range(ks):
        w = b >> 3
        if ((int(andor[2 * w]) ^ int(andor[2 * w + 1])) >> ((b & 7) * 8)) & 0xFF:
            return False
    return True


def _splittable(ops, data, n, layout, digits: DigitPlan, group) -> np.ndarray:
    """Digits whose records (over every rank) share one key: a pivot's equal
    digit by construction, a hot bucket without a pivot when digit_andor
    proves it."""
    split = digits.single.copy()
    if not digits.hot.any():
        return split
    ao = ops.digit_andor(data, n, layout, digits.p0, digits.bucket_digit, digits.hot)  # [D, 8]
    allao = _all_gather_np(ao.astype(np.uint64), _coll_device(data, group), group)  # [world, D, 8]
    a = np.bitwise_and.reduce(allao[:, :, 0::2], axis=0)
    o = np.bitwise_or.reduce(allao[:, :, 1::2], axis=0)
    comb = np.empty((digits.n_digits, 8), dtype=np.uint64)
    comb[:, 0::2], comb[:, 1::2] = a, o
    for d in np.nonzero(digits.hot)[0]:
        split[d] = _key_bytes_constant(comb[d], layout.key_size)
    return split


def _digits_with_pivots(ops, data, n: int, layout: RecordLayout, weights: np.ndarray, world: int,
                        p0: int, group) -> DigitPlan:
    """Digits from global bucket weights; every hot bucket is cut around its
    most common sampled key (a pivot), so that key's run can be spread over
    ranks by count even when the bucket holds other keys too. Arms the
    pivots on the device (ops.set_pivots)."""
    ks = layout.key_size
    hot = hot_buckets(weights, world)
    pivots = {}
    if hot.any() and hasattr(ops, "sample_keys"):
        k = ops.sample_keys(data, n, layout, SAMPLE_KEYS)
        row = np.zeros((SAMPLE_KEYS, 32), dtype=np.uint8)
        row[:len(k), :ks] = k
        cnt = np.array([len(k)], dtype=np.int64)
        flat = np.concatenate([cnt.view(np.uint8), row.reshape(-1)])
        allk = _all_gather_np(flat, _coll_device(data, group), group)
        keys = np.concatenate([allk[r, 8:].reshape(SAMPLE_KEYS, 32)[:int(allk[r, :8].view(np.int64)[0])]
                               for r in range(allk.shape[0])])
        pivots = choose_pivots(keys, p0, ks, hot, weights)
    digits = make_digits(weights, world, p0, pivots=pivots, ks=ks, align=True)
    if hasattr(ops, "set_pivots"):
        ops.set_pivots(digits, ks)
    return digits


def plan_exchange(ops, data, n: int, layout: RecordLayout, group=None) -> ExchangePlan:
    """Exact plan: full AND/OR and full 16-bit prefix histograms, all-gathered;
    per-source digit counts follow from the histograms (or, with pivots, from
    the partition's own histogram)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = _coll_device(data, group)
    # 1. global constant-prefix detection
    p0 = first_varying_byte(_all_gather_np(ops.andor(data, n, layout).astype(np.uint64), dev, group),
                            layout.key_size)
    if p0 >= layout.key_size:
        p0 = 0  # every key equal: any contiguous map is correct
    # 2. 16-bit prefix histograms, all-gathered
    h = ops.prefix_hist(data, n, layout, p0).cpu().numpy().astype(np.int64)
    hist = _all_gather_np(h, dev, group).astype(np.int64)  # [world, 65536]
    # 3. digits (hot buckets cut around pivots), single-key digits, exact counts, pieces
    digits = _digits_with_pivots(ops, data, n, layout, hist.sum(axis=0), world, p0, group)
    split = _splittable(ops, data, n, layout, digits, group)
    if digits.pivots:
        mine = np.asarray(ops.digit_counts(data, n, layout, p0, digits.bucket_digit, digits.n_digits),
                          dtype=np.uint64)
        M = _all_gather_np(mine, dev, group).astype(np.int64)
    else:
        M = np.stack([np.bincount(digits.bucket_digit, weights=hist[r].astype(np.float64),
                                  minlength=digits.n_digits) for r in range(world)]).astype(np.int64)
    pieces, S = assign_pieces(M, split, world)
    return ExchangePlan(digits, M, pieces, S)


SAMPLE_ANDOR = 1 << 16
SAMPLE_HIST = 1 << 20


def plan_exchange_sampled(ops, data, n: int, layout: RecordLayout, group=None):
    """The exchange plan without a full read of the data before the
    partition: the prefix byte and the digit map come from strided samples
    (the map only has to be balanced), and the exact per-digit counts plus
    the exact AND/OR come from the partition's own tile histogram
    (ops.partition_plan), all-gathered. Returns (plan, ok): ok is False on
    every rank when the exact AND/OR shows a more significant varying byte
    than the sample's (a byte that varies only off-sample); the caller then
    plans exactly (plan_exchange). On success the device holds the armed
    partition plan (partition_store_pieces follows)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    ks = layout.key_size
    dev = _coll_device(data, group)
    # 1. sampled AND/OR -> the guessed first varying key byte
    sao = ops.sample_andor(data, n, layout, SAMPLE_ANDOR).astype(np.uint64)
    p0 = first_varying_byte(_all_gather_np(sao, dev, group), ks)
    if p0 >= ks:
        p0 = 0
    # 2. sampled 16-bit prefix histograms, each weighted by its rank's record count
    h = ops.sample_prefix_hist(data, n, layout, p0, SAMPLE_HIST).cpu().numpy().astype(np.int64)
    row = np.concatenate([h, [n]]).astype(np.int64)
    rows = _all_gather_np(row, dev, group)
    weights = np.zeros(NBUCKETS, dtype=np.float64)
    for r in range(world):
        hr = rows[r, :NBUCKETS].astype(np.float64)
        if hr.sum() > 0:
            weights += hr * (float(rows[r, NBUCKETS]) / hr.sum())
    digits = _digits_with_pivots(ops, data, n, layout, weights, world, p0, group)
    split = _splittable(ops, data, n, layout, digits, group)
    # 3. exact per-digit counts and AND/OR from the partition's histogram, all-gathered
    counts, andor = ops.partition_plan(data, n, layout, p0, digits.bucket_digit, digits.n_digits)
    m = _all_gather_np(np.concatenate([counts.astype(np.uint64), andor.astype(np.uint64)]), dev, group)
    M = m[:, :digits.n_digits].astype(np.int64)
    p_exact = first_varying_byte(m[:, digits.n_digits:], ks)
    if p_exact >= ks:
        p_exact = 0
    pieces, S = assign_pieces(M, split, world)
    return ExchangePlan(digits, M, pieces, S), p_exact == p0


class _CudaBytes:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerWindows:
    """One receive window per rank in device memory, mapped by every other
    rank through CUDA IPC (one process per GPU on one node: NVLink P2P).
    ``ptrs[r]`` is rank r's window as seen from this process."""

    def __init__(self, nbytes: int, group=None):
        import torch.distributed as dist
        L = _lib.load()
        self.nbytes = nbytes
        self.rank = dist.get_rank(group)
        own = C.c_void_p()
        handle = C.create_string_buffer(64)
        _raise(L.raduls_gpu_ipc_alloc(nbytes, C.byref(own), handle), "raduls_gpu_ipc_alloc")
        self.own = own.value
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, handle.raw, group=group)
        self.ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(self.own)
                continue
            p = C.c_void_p()
            _raise(L.raduls_gpu_ipc_open(h, C.byref(p)), "raduls_gpu_ipc_open")
            self.ptrs.append(p.value)

    def close(self) -> None:
        L = _lib.load()
        for r, p in enumerate(self.ptrs):
            if r != self.rank:
                L.raduls_gpu_ipc_close(p)
        L.raduls_gpu_free(self.own)
        self.ptrs = []


_windows: dict = {}


def _peer_windows(nbytes: int, group, device):
    """Cached windows of at least nbytes; every rank asks for the same size
    (it comes from the exchanged histograms), so re-creation is collective.
    Returns None on every rank when any rank could not set its window up
    (the caller then exchanges through NCCL)."""
    import torch
    import torch.distributed as dist
    key = id(group)
    w = _windows.get(key)
    if w is not None and w.nbytes >= nbytes:
        return w
    if w is not None:
        w.close()
        _windows.pop(key, None)
    ok = 1
    try:
        w = PeerWindows(nbytes, group)
    except Exception:  # noqa: BLE001 - IPC unavailable: agree on the NCCL path below
        ok, w = 0, None
    dev = device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0:
        if w is not None:
            w.close()
        return None
    _windows[key] = w
    return w


def release_peer_windows() -> None:
    for w in _windows.values():
        w.close()
    _windows.clear()


def _receive_layout(plan: ExchangePlan, world: int):
    """Digit-major receive windows: receiver k holds its digits in digit
    order, each digit's records source by source (the stable order). Returns
    (offsets, segments): offsets[s, d, k] = record offset of source s's piece
    of digit d in receiver k's window; segments[k] = [(digit, records)] in
    window order."""
    G, D = len(plan.pieces), plan.digits.n_digits
    C = np.zeros((G, D, world), dtype=np.int64)
    for s_, pcs in enumerate(plan.pieces):
        for d, k, c in pcs:
            C[s_, d, k] += c
    T = C.sum(axis=0)                                   # [D, world]
    base = np.cumsum(T, axis=0) - T                     # digit-major, per receiver
    offsets = base[None, :, :] + (np.cumsum(C, axis=0) - C)
    segments = [[(int(d), int(T[d, k])) for d in np.nonzero(T[:, k])[0]] for k in range(world)]
    return offsets, segments


def _piece_destinations(plan: ExchangePlan, rank: int, rs: int, bases, offsets) -> tuple:
    """This source's pieces with their byte addresses in the receivers'
    windows (digit-major, _receive_layout)."""
    dg, ct, ds = [], [], []
    for d, k, c in plan.pieces[rank]:
        dg.append(d)
        ct.append(c)
        ds.append(bases[k] + int(offsets[rank, d, k]) * rs)
    return (np.array(dg, dtype=np.uint32), np.array(ct, dtype=np.uint64), np.array(ds, dtype=np.uint64))


def _split_digit_count(plan: ExchangePlan) -> int:
    """Digits whose records go to more than one rank (a hot key spread by count)."""
    ranks = {}
    for pcs in plan.pieces:
        for d, k, _ in pcs:
            ranks.setdefault(d, set()).add(k)
    return sum(1 for v in ranks.values() if len(v) > 1)


def _exchange_digit_major(recv, send, plan: ExchangePlan, offsets, rank: int, world: int, rs: int,
                          group) -> None:
    """The NCCL exchange into a digit-major receive buffer (the layout of
    _receive_layout): every (source, digit) piece lands at its place, so the
    receiver continues the MSD sort from the next byte. NCCL: one grouped
    batch of point-to-point sends and receives (pieces between a pair of
    ranks posted in the same digit order on both sides); a rank's pieces to
    itself are device copies. gloo (tests on one shared device or CPU): one
    all_to_all_single staged through host memory, rearranged on the host."""
    import os

    import torch.distributed as dist
    mine = plan.pieces[rank]
    # RADULS_P2P_OPS=1: the point-to-point form under gloo too (CPU tests of its
    # piece order and placement; gloo sends host tensors only)
    if dist.get_backend(group) == "nccl" or (os.environ.get("RADULS_P2P_OPS") == "1" and not send.is_cuda):
        ops_ = []
        pos = 0
        for d, k, c in mine:
            if k == rank:
                o = int(offsets[rank, d, rank])
                recv[o * rs:(o + c) * rs].copy_(send[pos * rs:(pos + c) * rs])
            else:
                ops_.append(dist.P2POp(dist.isend, send[pos * rs:(pos + c) * rs], k, group))
            pos += c
        for s_ in range(world):
            if s_ == rank:
                continue
            for d, k, c in plan.pieces[s_]:
                if k == rank:
                    o = int(offsets[s_, d, rank])
                    ops_.append(dist.P2POp(dist.irecv, recv[o * rs:(o + c) * rs], s_, group))
        if ops_:
            for r in dist.batch_isend_irecv(ops_):
                r.wait()
        return
    # gloo: source-major all_to_all_single (host-staged for CUDA tensors), then
    # each source's run of pieces (digit order) moved to its digit-major place
    n_out = int(plan.recv_counts(rank).sum())
    n_in = int(plan.send_counts(rank).sum())
    staged = recv.new_empty(max(n_out, 1) * rs, device="cpu")
    _all_to_all(staged[:n_out * rs], send[:n_in * rs], [int(c) * rs for c in plan.recv_counts(rank)],
                [int(c) * rs for c in plan.send_counts(rank)], group)
    out = staged.new_empty(max(n_out, 1) * rs)
    at = 0
    for s_ in range(world):
        for d, k, c in plan.pieces[s_]:
            if k == rank:
                o = int(offsets[s_, d, rank])
                out[o * rs:(o + c) * rs] = staged[at * rs:(at + c) * rs]
                at += c
    recv[:n_out * rs].copy_(out[:n_out * rs])


def _all_to_all(recv, send, out_splits, in_splits, group):
    """dist.all_to_all_single; gloo cannot move CUDA tensors, so there the
    exchange is staged through host memory (tests on one shared device)."""
    import torch.distributed as dist
    if dist.get_backend(group) != "nccl" and send.is_cuda:
        r = recv.new_empty(recv.numel(), device="cpu")
        dist.all_to_all_single(r, send.cpu(), output_split_sizes=out_splits,
                               input_split_sizes=in_splits, group=group)
        recv.copy_(r)
        return
    dist.all_to_all_single(recv, send, output_split_sizes=out_splits, input_split_sizes=in_splits,
                           group=group)


def _sort_received(ops, recv, n_out: int, layout: RecordLayout, plan: ExchangePlan, mine, tmp=None) -> int:
    """Sort this rank's digit-major receive buffer: its digits, in key order,
    are each one key range whose bytes before first_byte are equal — the
    exchange was the first MSD level, so the sort continues from there
    (raduls_gpu_sort_segments). Returns the number of segments."""
    fb = plan.digits.first_byte
    if fb is not None and hasattr(ops, "sort_segments") and len(mine) > 1:
        ops.sort_segments(recv, n_out, layout, [c for _, c in mine], [int(fb[d]) for d, _ in mine], tmp)
    elif tmp is not None:
        ops.sort(recv, n_out, layout, tmp)
    else:
        ops.sort(recv, n_out, layout)
    return len(mine)


def sort_distributed(data, n: int, layout: RecordLayout, ops=None, group=None,
                     timings: dict | None = None, exchange: str | None = None):
    """Sort `n` local records (uint8 tensor on this rank's device) across the
    process group. Returns (out tensor, n_out): this rank's contiguous key
    range, sorted.

    exchange="p2p" (default with DeviceOps on CUDA): the partition kernel
    stores every destination's records straight into that rank's receive
    window over NVLink (CUDA IPC; raduls_gpu_partition_store_pieces) — the
    partition and the all-to-all are one kernel. The returned tensor then
    aliases this rank's cached window and stays valid until the next call on
    the group. exchange="nccl": local partition by digit, then one grouped
    NCCL batch of per-piece sends and receives (_exchange_digit_major;
    host-staged under gloo). Either way the receive buffer is digit-major,
    so the local sort starts from the digits as pre-split segments.

    timings (optional dict) receives plan_s, exchange_ms (device time of the
    exchange: the fused partition kernel, or the all-to-all), partition_ms
    (nccl path), local_sort_s, sent_bytes (records leaving this rank * rs),
    recv_records and exchange ("p2p" or "nccl")."""
    import time

    import torch
    import torch.distributed as dist
    if ops is None:
        ops = DeviceOps(data.device)
    if exchange is None:
        exchange = "p2p" if isinstance(ops, DeviceOps) else "nccl"
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rs = layout.record_size
    cuda = data.is_cuda

    def event():
        if not cuda:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(data.device))
        return e

    def elapsed(e0, e1) -> float | None:
        if e0 is None:
            return None
        e1.synchronize()
        return e0.elapsed_time(e1)

    t0 = time.perf_counter()
    win = None
    if exchange == "p2p":
        plan, armed = plan_exchange_sampled(ops, data, n, layout, group)
        if not armed:  # a key byte varies only off the sample: plan exactly, re-arm the device plan
            plan = plan_exchange(ops, data, n, layout, group)
            counts, _ = ops.partition_plan(data, n, layout, plan.p0, plan.digits.bucket_digit,
                                           plan.digits.n_digits)
            if not np.array_equal(counts.astype(np.int64), plan.M[rank]):
                raise RuntimeError("partition counts disagree with the exchanged histograms")
        win = _peer_windows(max(int(plan.matrix.sum(axis=0).max()), 1) * rs, group, data.device)
        if win is None:  # IPC unavailable on some rank: the NCCL exchange below
            exchange = "nccl"
    else:
        plan = plan_exchange(ops, data, n, layout, group)
    n_out = int(plan.recv_counts(rank).sum())
    t1 = time.perf_counter()
    info = {"exchange": exchange, "plan_s": t1 - t0, "recv_records": n_out,
            "sent_bytes": int((plan.send_counts(rank).sum() - plan.send_counts(rank)[rank]) * rs),
            "hot_split_digits": _split_digit_count(plan)}
    if win is not None:
        offsets, segments = _receive_layout(plan, world)
        dg, ct, ds = _piece_destinations(plan, rank, rs, win.ptrs, offsets)
        if cuda:
            torch.cuda.synchronize(data.device)
        dist.barrier(group=group)  # every window free (previous results consumed)
        e0 = event()
        ops.partition_store_pieces(data, n, layout, dg, ct, ds)
        e1 = event()
        info["exchange_ms"] = elapsed(e0, e1)
        dist.barrier(group=group)  # every rank's stores into every window are complete
        t2 = time.perf_counter()
        recv = torch.as_tensor(_CudaBytes(win.own, max(n_out, 1) * rs), device=data.device)
        info["segments"] = _sort_received(ops, recv, n_out, layout, plan, segments[rank],
                                          ops.empty(max(n_out, 1) * rs))
    else:
        # local stable partition by digit (pieces of a digit stay in rank order)
        e0 = event()
        send, counts = ops.partition(data, n, layout, plan.p0, plan.digits.bucket_digit,
                                     plan.digits.n_digits)
        e1 = event()
        if not np.array_equal(np.asarray(counts, dtype=np.int64), plan.M[rank]):
            raise RuntimeError("partition counts disagree with the exchanged histograms")
        recv = ops.empty(max(n_out, 1) * rs)
        offsets, segments = _receive_layout(plan, world)
        e2 = event()
        _exchange_digit_major(recv, send, plan, offsets, rank, world, rs, group)
        e3 = event()
        info["partition_ms"] = elapsed(e0, e1)
        info["exchange_ms"] = elapsed(e2, e3)
        del send
        t2 = time.perf_counter()
        info["segments"] = _sort_received(ops, recv, n_out, layout, plan, segments[rank])
    if cuda:
        torch.cuda.synchronize(data.device)
    t3 = time.perf_counter()
    info["local_sort_s"] = t3 - t2
    if timings is not None:
        timings.update(info)
    return recv, n_out


# ---------------------------------------------------------------- one process, G devices

def sort_multi(inputs, layout: RecordLayout, capacity: int | None = None):
    """raduls_gpu_sort_multi: ``inputs`` is a list of CUDA uint8 tensors (one
    per device; a device may appear more than once), each holding whole
    records. Returns ``(outputs, counts)``: outputs[g] is a tensor on
    inputs[g]'s device whose first counts[g] records are the g-th contiguous
    key range, sorted (concatenated over g: the stable sort of the inputs in
    list order). ``capacity`` (records per output) defaults to the total."""
    import torch
    G = len(inputs)
    rs = layout.record_size
    n_in = np.array([t.numel() // rs for t in inputs], dtype=np.uint64)
    cap = int(n_in.sum()) if capacity is None else int(capacity)
    outs = [torch.empty(max(cap, 1) * rs, dtype=torch.uint8, device=t.device) for t in inputs]
    devs = (C.c_int * G)(*[t.device.index for t in inputs])
    din = (C.c_void_p * G)(*[t.data_ptr() for t in inputs])
    dout = (C.c_void_p * G)(*[t.data_ptr() for t in outs])
    n_out = np.zeros(G, dtype=np.uint64)
    for t in inputs:
        torch.cuda.synchronize(t.device)
    rc = _lib.load().raduls_gpu_sort_multi(G, devs, din, n_in.ctypes.data_as(_lib._u64p), dout,
                                           n_out.ctypes.data_as(_lib._u64p), cap, rs,
                                           layout.key_size)
    _raise(rc, "raduls_gpu_sort_multi")
    return outs, [int(x) for x in n_out]
