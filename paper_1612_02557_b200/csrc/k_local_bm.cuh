// (d) small-bin sort, bitmap form: the first-line local sort for records held
// in shared memory (16/24/32 B). Same contract as local_group (k_local.cuh):
// one CTA sorts one group of <= kCap records that share key bytes [0, p), by
// key bytes [p, ks), stable, straight into `data`, safe in place.
//
// Reference: the tiny-bin sorts (P/include/raduls/small_sorts.hpp:48-191) and
// finalize() (P/include/raduls/detail/msd_sorter.hpp:76-80).
//
// The bucket sort of k_local.cuh spends ~150 of its ~247 thread instructions
// per record on putting record ids into bucket order and ranking every record
// against its bucket's neighbours (dependent shared-memory loads). Here the
// 32-bit window of key bytes p..p+3 of every record is mapped linearly
// (monotone) onto a fine grid of ~16 n cells (8-B records: ~32 n), one BIT per
// cell; the window
// range comes with the group (the planner knows the digit range of byte p), so
// windows and cell bits are one pass with no barrier before it:
//   * cells: one atomicOr per record sets its cell's bit. A record that finds
//     the bit already set (two records in one cell: ~6% of random records)
//     bumps a u16 counter ("extras") of its 32-cell bitmap word;
//   * scan (bm_scan): warp-cooperative prefix sum over the words of
//     popc(word) + extras; the word's start is stored as a u16 in place of
//     its extras. A word holding a shared cell (a dirty word) turns its own
//     bitmap word into a descriptor {start, count, cursor} and its start
//     entry into 0x8000 | the first entry of its run in a dense list (u16
//     record ids; the list can hold every record of the group);
//   * rank: a record of a clean word is final at start + popc(bits below its
//     own) -- two independent shared-memory loads, no neighbour to compare
//     with, no id scatter -- and is stored to its place at once. Records of
//     dirty words (all of them, ~12%) append themselves to their word's run and
//     are ranked densely afterwards, each against the few entries of its own
//     run, by (window, key bytes beyond the window, input index): stable.
// No search for the varying key bytes: a window holding constant bytes only
// loses resolution. A group with more than kMaxBucket records in one word
// (duplicate-heavy, clustered or constant-byte keys) is handed
// untouched -- nothing has been written by then -- to the bucket sort
// (k_local_list below) through a device-counted list; that one searches the
// varying bytes and may hand the group on to the LSD fallback.
// Shapes: 16-B records, 256 threads, five CTAs per SM, groups of <= 2048
// records (a single bin between that and LocalCfg::kCap is a group of its
// own for the 512-thread instance, k_local_bm_med); 24-B records alike with
// groups of <= 1280; 32-B records in the bucket sort's shape; 8-B records in registers (k_local_bm8).
#pragma once

#include "k_local.cuh"

namespace rg {

// Shape knobs of the 16-B primary instance (A/B): threads per
// CTA, CTAs per SM, group capacity. The planner packs small bins into groups
// of at most this capacity (group_cap<RS>()); a single bin between it and the
// local-sort capacity (LocalCfg::kCap) is a group of its own, taken by the
// big instance (V = 1: the bucket sort's shape).
// Measured (C5 local sort, interleaved A/B, 32 cells per record): 512 threads
// x 2 CTAs per SM, cap 3584: 38.7 ms; 384 x 3, cap 2560: 36.8 ms; 256 x 5, cap
// 1792: 31.9 ms. With 16 cells per record the bitmap shrinks: six CTAs of <=
// 1728 records C5 30.05 vs 30.9 ms, C1 0.549 vs 0.594 ms; five CTAs of <= 2048
// records (the largest group whose grid stays 2^15 cells) C1 0.533, C3 4.66 vs
// 4.86 (its 1800-record bins stay in this instance), C5 30.4 vs 30.6 ms.
#ifndef RG_BM_THREADS
#define RG_BM_THREADS 256
#endif
#ifndef RG_BM_BLOCKS
#define RG_BM_BLOCKS 5
#endif
#ifndef RG_BM_CAP16
#define RG_BM_CAP16 2048
#endif
// RG_BM_WAIT1: thread 0 alone waits for the group's TMA copy, the block barrier
// hands the completion on (no spinning warps). RG_BM_PERSIST: the several-
// CTAs-per-SM shapes run as a resident grid walking the groups with its stride.
#ifndef RG_BM_WAIT1
#define RG_BM_WAIT1 0
#endif
#ifndef RG_BM_KNOWN
#define RG_BM_KNOWN 1
#endif
// L2 eviction hint of the final record stores (0 none, 1 evict_first, 2 evict_last)
#ifndef RG_HINT_LOCST
#define RG_HINT_LOCST 0
#endif
// RG_BM_CHUNKS (16/32-B records): the group's TMA copy is issued as one bulk
// copy per loop iteration's records (T records), each with its own mbarrier,
// and the first pass over the records waits chunk by chunk: it runs while the
// rest of the group is still arriving.
#ifndef RG_BM_CHUNKS
#define RG_BM_CHUNKS 0
#endif
#ifndef RG_BM_PERSIST
#define RG_BM_PERSIST 0
#endif
// the big 16-B instance (V = 1): threads, CTAs per SM, bitmap bits (0: as the primary)
#ifndef RG_BM_MED_THREADS
#define RG_BM_MED_THREADS 512
#endif
#ifndef RG_BM_MED_BLOCKS
#define RG_BM_MED_BLOCKS 2
#endif
#ifndef RG_BM_MED_BITS
#define RG_BM_MED_BITS 0
#endif
#ifndef RG_BM_MED_PREFETCH
#define RG_BM_MED_PREFETCH 1
#endif
// 24-B primary instance: RG_BM_THREADS threads, RG_BM_BLOCKS24 CTAs per SM,
// groups of <= RG_BM_CAP24 records (0: the bucket sort's shape, 512 threads x 2,
// cap 2560). Measured on 2^28 x 24 B: local sort 2.50 (1280 x 5) / 2.52 (1024 x
// 6) vs 3.36 ms; a single bin above the capacity goes to the 512-thread instance.
#ifndef RG_BM_CAP24
#define RG_BM_CAP24 1280
#endif
#ifndef RG_BM_BLOCKS24
#define RG_BM_BLOCKS24 5
#endif
#ifndef RG_BM_THREADS32
#define RG_BM_THREADS32 512
#endif
// 32-B primary instance in the small two-tier shape (0: off -- one 512-thread CTA
// per SM takes every group). Measured: 2^26 x 32 B (1024-record bins) local sort
// 1.01 vs 1.28 ms; C4's 4096-record bins are all above it, and the host then
// launches the big instance over the whole list (n_big_groups from the planner).
#ifndef RG_BM_CAP32
#define RG_BM_CAP32 1280
#endif
#ifndef RG_BM_BLOCKS32
#define RG_BM_BLOCKS32 4
#endif
#ifndef RG_BM_BITS
#define RG_BM_BITS 0
#endif
// cells per record aimed at (log2): shared-memory records 2^4 (measured 2^3 /
// 2^4 / 2^5: C5 local 33.0 / 30.4 / 30.9 ms, C4 5.94 / 5.14 / 5.34); 8-B
// records 2^5 (2^4: C2 local 8.13 vs 7.85 ms)
#ifndef RG_BM_CELL_LOG
#define RG_BM_CELL_LOG 4
#endif
#ifndef RG_BM8_CELL_LOG
#define RG_BM8_CELL_LOG 5
#endif

constexpr int ceil_log2_c(int n) {
    int b = 0;
    while ((1 << b) < n) ++b;
    return b;
}

template <int RS, int V = 0>
struct BmCfg {
    using L = LocalCfg<RS>;
    static_assert(!L::kRegRecords, "shared-memory records only");
    static constexpr bool kTuned = RS == 16 && V == 0;
    static constexpr bool kTuned24 = (RS == 24 && V == 0 && RG_BM_CAP24 != 0) || (RS == 32 && V == 0 && RG_BM_CAP32 != 0);
    static constexpr bool kMed = RS == 16 && V == 1;
    static constexpr int kThreads = (kTuned || kTuned24) ? RG_BM_THREADS
                                    : kMed ? RG_BM_MED_THREADS
                                           : RS == 32 ? RG_BM_THREADS32 : L::kThreads;
    static constexpr int kMinBlocks = kTuned ? RG_BM_BLOCKS
                                      : kTuned24 ? (RS == 24 ? RG_BM_BLOCKS24 : RG_BM_BLOCKS32)
                                                 : kMed ? RG_BM_MED_BLOCKS : L::kMinBlocks;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kCap = kTuned ? RG_BM_CAP16 : kTuned24 ? (RS == 24 ? RG_BM_CAP24 : RG_BM_CAP32) : L::kCap;
    static_assert(kCap <= L::kCap, "the bucket sort takes over whole groups");
    static constexpr int kIpt = (kCap + kThreads - 1) / kThreads;
    // cells per record aimed at, as a power of two: FB = ceil(log2 n) + kCellLog
    static constexpr int kCellLog = RG_BM_CELL_LOG;
    // cells = 2^kFineBits at most
    static constexpr int kFineBits = (kMed && RG_BM_MED_BITS) ? RG_BM_MED_BITS
                                     : RG_BM_BITS ? RG_BM_BITS : ceil_log2_c(kCap) + kCellLog;
    static constexpr int kWords = 1 << (kFineBits - 5);
    // scan: every warp owns kRows rows of 128 words
    static constexpr int kRows = (kWords + 128 * kWarps - 1) / (128 * kWarps);
    static_assert(kRows >= 1 && kRows <= 4, "scan rows per warp");
    // the dirty-record list holds every record if need be (u16 entries); a dirty
    // word's descriptor lives in its own bitmap word
    static constexpr int kRecBytes = ((kCap * RS + 16 + 127) / 128) * 128;
    static constexpr size_t kSmem = size_t(kRecBytes) + size_t(kWords) * 6 + ((size_t(kCap) * 2 + 15) / 16) * 16;
};

// Scan over the bitmap words of popc(word) + extras -> every word's start (u16
// in place of its extras). Warp q owns words [128 R q, 128 R (q + 1)) as R rows
// of 128 (those below nW); lane l reads words 4 l..4 l + 3 of each row
// (conflict-free 16-B / 8-B loads); row sums are scanned across the lanes two
// rows to a register (u16 halves: sums <= n < 32768). A word with extras (a
// shared cell) is dirty: its own bitmap word (its bits are not needed again:
// all its records go through the list) becomes its descriptor start | count
// << 16 | cursor << 24, and its start entry holds 0x8000 | the first list
// entry of its run; *s_alloc counts the records of dirty words, *s_crowd is
// set when one word holds more than kMaxBucket records. One block barrier
// inside; the caller syncs after it.
template <int W, int R>
__device__ __forceinline__ void bm_scan(uint32_t* bm, uint32_t* pre, uint32_t nW, uint32_t* s_scan,
                                        uint32_t* s_alloc, uint32_t* s_crowd) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        const uint4* bm4 = reinterpret_cast<const uint4*>(bm) + warp * (32 * R);
        uint2* pre2 = reinterpret_cast<uint2*>(pre) + warp * (32 * R);
        uint32_t sv[R];
#pragma unroll
        for (int v = 0; v < R; ++v) {
            sv[v] = 0;
            if ((uint32_t(warp) * R + v) * 128u < nW) {
                const uint4 a = bm4[v * 32 + lane];
                const uint2 x = pre2[v * 32 + lane];
                uint32_t s = __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
                if (x.x | x.y) s += (x.x & 0xFFFFu) + (x.x >> 16) + (x.y & 0xFFFFu) + (x.y >> 16);
                sv[v] = s;
            }
        }
        constexpr int NP = (R + 1) / 2;
        uint32_t pk[NP], ik[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) ik[q] = pk[q] = sv[2 * q] | ((2 * q + 1 < R ? sv[2 * q + 1 < R ? 2 * q + 1 : 0] : 0u) << 16);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, ik[q], off);
                if (lane >= off) ik[q] += y;
            }
        }
        uint32_t tk[NP], wtot = 0;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            tk[q] = __shfl_sync(0xFFFFFFFFu, ik[q], 31);
            wtot += (tk[q] & 0xFFFFu) + (tk[q] >> 16);
        }
        if (lane == 0) s_scan[warp] = wtot;
        __syncthreads();
        const uint32_t t = lane < W ? s_scan[lane] : 0u;
        uint32_t rowb = __reduce_add_sync(0xFFFFFFFFu, lane < warp ? t : 0u);
        {
#pragma unroll
            for (int v = 0; v < R; ++v) {
                if ((uint32_t(warp) * R + v) * 128u >= nW) break;  // warp-uniform
                const uint32_t exl = ik[v / 2] - pk[v / 2];  // exclusive over the lanes, per row
                const uint32_t ex = (v & 1) ? (exl >> 16) : (exl & 0xFFFFu);
                const uint32_t rt = (v & 1) ? (tk[v / 2] >> 16) : (tk[v / 2] & 0xFFFFu);
                const uint4 a = bm4[v * 32 + lane];
                const uint2 x = pre2[v * 32 + lane];
                const uint32_t c0 = __popc(a.x), c1 = __popc(a.y), c2 = __popc(a.z);
                uint32_t r0 = rowb + ex, r1 = r0 + c0, r2 = r1 + c1, r3 = r2 + c2;
                if (x.x | x.y) {  // rare: a dirty word among the four
                    const uint32_t e0 = x.x & 0xFFFFu, e1 = x.x >> 16, e2 = x.y & 0xFFFFu, e3 = x.y >> 16;
                    r1 += e0;
                    r2 += e0 + e1;
                    r3 += e0 + e1 + e2;
                    auto dirty = [&](uint32_t start, uint32_t cnt, uint32_t c) -> uint32_t {
                        if (cnt > kMaxBucket) *s_crowd = 1;  // duplicate-heavy: not for the quadratic ranking
                        const uint32_t off = atomicAdd(s_alloc, cnt);
                        bm[(uint32_t(warp) * R + v) * 128u + 4u * lane + c] = start | (min(cnt, 255u) << 16);
                        return 0x8000u | (off & 0x7FFFu);
                    };
                    if (e0) r0 = dirty(r0, c0 + e0, 0);
                    if (e1) r1 = dirty(r1, c1 + e1, 1);
                    if (e2) r2 = dirty(r2, c2 + e2, 2);
                    if (e3) r3 = dirty(r3, __popc(a.w) + e3, 3);
                }
                pre2[v * 32 + lane] = make_uint2(r0 | (r1 << 16), r2 | (r3 << 16));
                rowb += rt;
            }
        }
    }
}

// Whether groups larger than the primary instance's capacity exist (they go to
// the `med` list, sorted by the big instance).
template <int RS>
constexpr bool kBmHasBig = BmCfg<RS, 0>::kCap < LocalCfg<RS>::kCap;

struct GroupList {
    Group* list;
    unsigned int* n;
    uint32_t cap;
};

__device__ __forceinline__ void push_group(const GroupList& l, const Group& g) {
    const uint32_t i = atomicAdd(l.n, 1u);
    if (i < l.cap) l.list[i] = g;
}

template <int RS, int V, typename Mid>
__device__ __forceinline__ void local_group_bm(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group g, uint32_t ks,
    LevelCounters* __restrict__ ctr, const GroupList spill, const GroupList med, Mid&& mid) {
    using C = BmCfg<RS, V>;
    constexpr int T = C::kThreads, W = C::kWarps, IPT = C::kIpt, R = C::kRows;
    extern __shared__ __align__(128) uint8_t smem[];
    RG_CHK_POISON_SMEM(smem);
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem + C::kRecBytes);  // [kWords] cell bits
    uint32_t* pre = bm + C::kWords;                                   // [kWords] u16: extras, then starts
    uint16_t* dl = reinterpret_cast<uint16_t*>(pre + C::kWords / 2);  // [kCap] records of dirty words, run by run
    __shared__ uint32_t s_scan[W];
    __shared__ uint32_t s_wmin, s_wmax, s_alloc, s_crowd;
    constexpr bool kChunks = RG_BM_CHUNKS && RS % 16 == 0;  // (16-B aligned records: no head bytes)
    __shared__ __align__(8) unsigned long long s_barv[kChunks ? IPT : 1];
    unsigned long long& s_bar = s_barv[0];

    const uint32_t n = g.size;
    const uint8_t* gsrc = (g.parity ? tmp : data) + g.start * RS;
    uint8_t* dst = data + g.start * RS;
    const int lane = threadIdx.x & 31;
    if constexpr (V == 0 && kBmHasBig<RS>) {
        if (n > uint32_t(C::kCap)) {  // a single bin above this instance's capacity
            if (threadIdx.x == 0) push_group(med, g);
            return;
        }
    }
    const uint32_t klim = ks < uint32_t(RS) ? ks : uint32_t(RS);
    if (n <= 1 || g.p >= klim) {  // nothing to order (no key byte left: the input order stands)
        if (g.parity)
            for (uint32_t e = threadIdx.x; e < n; e += T) store_rec<RS>(dst, e, load_rec<RS>(gsrc, e));
        return;
    }

    // ---- 1. the group on chip (TMA), bitmap and counters zeroed meanwhile
    const uint32_t head = uint32_t(reinterpret_cast<uintptr_t>(gsrc) & 15u);
    const uint8_t* recs = smem + head;
    const bool chunks = kChunks && head == 0;  // (a base pointer that is only 8-B aligned: one copy)
    if (threadIdx.x == 0) {
        if (chunks) {
            const uint32_t bytes = n * RS;
            constexpr uint32_t CH = uint32_t(T) * RS;  // one loop iteration's records
#pragma unroll
            for (int j = 0; j < IPT; ++j)
                if (uint32_t(j) * CH < bytes) mbar_init(&s_barv[j], 1);
            fence_mbar_init();
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * CH < bytes) {
                    const uint32_t sz = min(CH, bytes - uint32_t(j) * CH);
                    mbar_arrive_expect_tx(&s_barv[j], sz);
                    tma_load_1d_h<RG_HINT_LOCAL>(smem + j * CH, gsrc + j * CH, sz, &s_barv[j]);
                }
            }
        } else {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const uint32_t bytes = n * RS;
        const uint32_t hb = head ? min(8u, bytes) : 0u;
        const uint32_t body = (bytes - hb) & ~15u;
        const uint32_t tail = bytes - hb - body;
        if (hb) *reinterpret_cast<uint2*>(smem + head) = *reinterpret_cast<const uint2*>(gsrc);
        if (tail)
            *reinterpret_cast<uint2*>(smem + head + hb + body) =
                *reinterpret_cast<const uint2*>(gsrc + hb + body);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_bar, body);
        for (uint32_t o = 0; o < body; o += 32768u)
            tma_load_1d_h<RG_HINT_LOCAL>(smem + head + hb + o, gsrc + hb + o, min(32768u, body - o), &s_bar);
        }
        s_wmin = 0xFFFFFFFFu;
        s_wmax = 0u;
        s_alloc = 0;
        s_crowd = 0;
    }
    // cells: 2^FB, ~2^kCellLog per record; at least one warp's scan span
    uint32_t FB = 32u + uint32_t(C::kCellLog) - __clz(n - 1);  // ceil(log2 n) + kCellLog (n >= 2)
    FB = FB < 12u ? 12u : (FB > uint32_t(C::kFineBits) ? uint32_t(C::kFineBits) : FB);
    const uint32_t nW = 1u << (FB - 5);  // a multiple of 128 (one scan row)
    {
        uint4* z = reinterpret_cast<uint4*>(bm);
#pragma unroll
        for (int q = 0; q < (C::kWords / 4 + T - 1) / T; ++q)
            if (q * T + threadIdx.x < nW / 4) z[q * T + threadIdx.x] = make_uint4(0, 0, 0, 0);
        uint4* z2 = reinterpret_cast<uint4*>(pre);
#pragma unroll
        for (int q = 0; q < (C::kWords / 8 + T - 1) / T; ++q)
            if (q * T + threadIdx.x < nW / 8) z2[q * T + threadIdx.x] = make_uint4(0, 0, 0, 0);
    }
    if (chunks) {
        __syncthreads();  // (the first pass waits per chunk)
    } else if constexpr (RG_BM_WAIT1) {
        if (threadIdx.x == 0) mbar_wait(&s_bar, 0);
        __syncthreads();
    } else {
        __syncthreads();
        mbar_wait(&s_bar, 0);
    }

    // ---- 2./3. windows: key bytes p..p+3 (fewer at the key's end), big-endian,
    // one byte permute per record; their range; cell bits. No search for the varying
    // bytes: a window holding constant bytes only loses resolution, and a
    // group it cannot resolve is handed to the bucket sort
    const uint32_t nwin = klim - g.p < 4u ? klim - g.p : 4u;
    const bool beyond = g.p + 4u < klim;
    uint32_t Ldef[4] = {g.p, g.p + 1, g.p + 2, g.p + 3};
    const WindowSel ws = make_window_sel(Ldef, nwin, RS / 4, false);
    // The planner's groups carry the digit range [d0, d1] of byte p (pad: d0 |
    // d1 << 8 | 1 << 16): the window range is known without a min/max pass, so
    // windows and cell bits are one pass (RG_BM_KNOWN).
    const bool known = RG_BM_KNOWN && (g.pad & 0x10000u) != 0u;
    const uint32_t ncell = 1u << FB;
    uint32_t fc[IPT];
    // cell = umulhi(w - wmin, mul): monotone in w and < 2^FB (mul rounded down
    // with a 1e-6 margin over the float error; k_local.cuh's bucket geometry)
    auto mul_of = [&](uint32_t rm1) {
        return rm1 < ncell ? 0u
                           : uint32_t(__fdiv_rz(float(ncell) * 4294967296.0f, float(rm1) + 1.0f) * 0.999999f);
    };
    // one bit per occupied cell; a record finding its cell taken counts itself
    // in the word's extras (u16 halves of pre)
    auto mark = [&](uint32_t f) {
        const uint32_t bit = 1u << (f & 31u);
        const uint32_t old = atomicOr(&bm[f >> 5], bit);
        if (old & bit) atomicAdd(&pre[f >> 6], 1u << ((f >> 1) & 16u));
    };
    uint32_t wmin, mul;
    if (known) {
        const uint32_t d0 = g.pad & 0xFFu, d1 = (g.pad >> 8) & 0xFFu;
        wmin = d0 << 24;
        mul = mul_of(((d1 - d0 + 1u) << 24) - 1u);
        mid();
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T >= n) break;  // block-uniform
            if (chunks) mbar_wait(&s_barv[j], 0);
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) {
                const uint32_t d = rec_window<RS>(ld_smem_rec<RS>(recs, e), ws) - wmin;
                const uint32_t f = min(mul ? __umulhi(d, mul) : d, ncell - 1u);
                fc[j] = f;
                mark(f);
            }
        }
    } else {
        uint32_t wv[IPT];
        uint32_t smn = 0xFFFFFFFFu, smx = 0u;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T >= n) break;  // block-uniform
            if (chunks) mbar_wait(&s_barv[j], 0);
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) {
                const uint32_t w = rec_window<RS>(ld_smem_rec<RS>(recs, e), ws);
                wv[j] = w;
                smn = min(smn, w);
                smx = max(smx, w);
            }
        }
        smn = __reduce_min_sync(0xFFFFFFFFu, smn);
        smx = __reduce_max_sync(0xFFFFFFFFu, smx);
        if (lane == 0) {
            atomicMin(&s_wmin, smn);
            atomicMax(&s_wmax, smx);
        }
        __syncthreads();
        wmin = s_wmin;
        const uint32_t rm1 = s_wmax - wmin;  // range - 1
        if (rm1 == 0 && !beyond) {           // every key equal: stable order is the input order
            if (g.parity) {
#pragma unroll
                for (int j = 0; j < IPT; ++j) {
                    if (uint32_t(j) * T >= n) break;
                    const uint32_t e = uint32_t(j) * T + threadIdx.x;
                    if (e < n) store_rec<RS>(dst, e, ld_smem_rec<RS>(recs, e));
                }
            }
            return;
        }
        mul = mul_of(rm1);
        mid();
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T >= n) break;
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) {
                const uint32_t d = wv[j] - wmin;
                const uint32_t f = min(mul ? __umulhi(d, mul) : d, ncell - 1u);
                fc[j] = f;
                mark(f);
            }
        }
    }
    __syncthreads();

    // ---- 4. scan (bm_scan): word starts; a dirty word's descriptor in its bitmap word
    bm_scan<W, R>(bm, pre, nW, s_scan, &s_alloc, &s_crowd);
    __syncthreads();
    const uint32_t nd = s_alloc;  // records of dirty words (<= n: the list holds them all)
    if (s_crowd) {
        // block-uniform; nothing written yet: the bucket sort takes the group
        if (threadIdx.x == 0) {
            push_group(spill, g);
            atomicAdd(&ctr->bm_spill, 1u);
        }
        return;
    }

    // ---- 5. clean words: final position = the word's start + bits below the
    // record's own; stored at once (one uncoalesced vector store per record,
    // the group's lines complete in L2). Dirty words: into the word's list run
    // (cursor in the descriptor's top byte).
    const uint16_t* pre16 = reinterpret_cast<const uint16_t*>(pre);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (uint32_t(j) * T >= n) break;
        const uint32_t e = uint32_t(j) * T + threadIdx.x;
        if (e < n) {
            const uint32_t f = fc[j], word = f >> 5;
            const uint32_t pv = pre16[word];
            const uint32_t m = bm[word];
            if (pv < 0x8000u) {
                const uint32_t pos = pv + __popc(m & ((1u << (f & 31u)) - 1u));
                store_rec_h<RS, RG_HINT_LOCST>(dst, pos, ld_smem_rec<RS>(recs, e));
            } else {
                const uint32_t old = atomicAdd(&bm[word], 1u << 24);
                dl[(pv & 0x7FFFu) + (old >> 24)] = uint16_t(e);
            }
        }
    }
    if (nd == 0) {
        if (threadIdx.x == 0) atomicAdd(&ctr->moved_local, (unsigned long long)n);
        return;
    }
    __syncthreads();
    // ---- 6. dirty words, densely from the list: each entry finds its word again
    // (window -> cell) and ranks itself among the word's run by (window, key
    // bytes beyond the window, input index)
    {
        auto window_of = [&](uint32_t e) { return rec_window<RS>(ld_smem_rec<RS>(recs, e), ws); };
        auto cmp_rest = [&](uint32_t a, uint32_t b) -> int {
            for (uint32_t q = g.p + 4u; q < klim; ++q) {
                const uint32_t x = recs[size_t(a) * RS + q], y = recs[size_t(b) * RS + q];
                if (x != y) return x < y ? -1 : 1;
            }
            return 0;
        };
        for (uint32_t i = threadIdx.x; i < nd; i += T) {
            const uint32_t e = dl[i];
            const uint32_t w = window_of(e);
            const uint32_t dd = w - wmin;
            const uint32_t word = min(mul ? __umulhi(dd, mul) : dd, ncell - 1u) >> 5;
            const uint32_t desc = bm[word];
            const uint32_t start = desc & 0xFFFFu, cnt = (desc >> 16) & 0xFFu;
            const uint32_t off = pre16[word] & 0x7FFFu;
            uint32_t rank = 0;
            for (uint32_t q = off; q < off + cnt; ++q) {
                if (q == i) continue;
                const uint32_t e2 = dl[q];
                const uint32_t w2 = window_of(e2);
                bool lt;
                if (w2 != w) {
                    lt = w2 < w;
                } else {
                    const int c = beyond ? cmp_rest(e2, e) : 0;
                    lt = c < 0 || (c == 0 && e2 < e);
                }
                rank += lt;
            }
            store_rec<RS>(dst, start + rank, ld_smem_rec<RS>(recs, e));
        }
    }
    if (threadIdx.x == 0) atomicAdd(&ctr->moved_local, (unsigned long long)n);
}

// Bitmap local sort launch: the shapes of k_local (several CTAs per SM: a CTA
// per group, the group half a resident wave ahead prefetched into L2; one CTA per
// SM: persistent, groups round-robin, next descriptor by cp.async).
// V = 1: the big instance over the whole group list (the host launches it
// instead when most groups are single bins above the primary capacity).
template <int RS, int V = 0>
__global__ void __launch_bounds__(BmCfg<RS, V>::kThreads, BmCfg<RS, V>::kMinBlocks) k_local_bm(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group* __restrict__ groups,
    uint32_t n_groups, uint32_t ks, LevelCounters* __restrict__ ctr, GroupList spill, GroupList med,
    uint32_t ahead) {
    if constexpr (BmCfg<RS, V>::kMinBlocks > 1 && !RG_BM_PERSIST) {
        if (threadIdx.x == 0 && blockIdx.x + ahead < n_groups)
            prefetch_group_l2<RS>(data, tmp, groups[blockIdx.x + ahead]);
        local_group_bm<RS, V>(data, tmp, groups[blockIdx.x], ks, ctr, spill, med, [] {});
        return;
    }
    __shared__ __align__(16) Group s_g[2];
    uint32_t i = blockIdx.x;
    if (i >= n_groups) return;
    if (threadIdx.x == 0) s_g[0] = groups[i];
    __syncthreads();
    for (int buf = 0; i < n_groups; buf ^= 1) {
        const uint32_t nx = i + gridDim.x;
        const bool more = nx < n_groups;
        if (threadIdx.x == 0 && more) {
            for (int q = 0; q < int(sizeof(Group) / 8); ++q)
                cp_async8(reinterpret_cast<uint8_t*>(&s_g[buf ^ 1]) + 8 * q,
                          reinterpret_cast<const uint8_t*>(&groups[nx]) + 8 * q);
        }
        const Group g = s_g[buf];
        auto mid = [&] {
            if (threadIdx.x == 0 && more) {
                cp_async_wait_all();
                prefetch_group_l2<RS>(data, tmp, s_g[buf ^ 1]);
            }
        };
        local_group_bm<RS, V>(data, tmp, g, ks, ctr, spill, med, mid);
        if (threadIdx.x == 0 && more) cp_async_wait_all();
        __syncthreads();
        i = nx;
    }
}

// The big instance over the device-counted `med` list (groups above the
// primary instance's capacity), launched right behind k_local_bm with a fixed
// grid; CTAs walk the list with the grid's stride.
template <int RS>
__global__ void __launch_bounds__(BmCfg<RS, 1>::kThreads, BmCfg<RS, 1>::kMinBlocks) k_local_bm_med(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, GroupList med, uint32_t ks,
    LevelCounters* __restrict__ ctr, GroupList spill) {
    const uint32_t n = min(*med.n, med.cap);
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        const uint32_t nx = i + gridDim.x;
        auto mid = [&] {  // the CTA's next group toward L2 while this one is sorted
            if (RG_BM_MED_PREFETCH && threadIdx.x == 0 && nx < n) prefetch_group_l2<RS>(data, tmp, med.list[nx]);
        };
        local_group_bm<RS, 1>(data, tmp, med.list[i], ks, ctr, spill, med, mid);
        __syncthreads();  // shared memory free for the next group
    }
}

// ---------------------------------------------------------------- 8-B records
//
// The bitmap sort for 8-B records (BASELINE C2: bins of ~16 K records, one
// group each): records stay in registers (coalesced global loads), one CTA of
// 1024 threads per SM, persistent. The cell of a record is recomputed from its
// registers where needed (no per-record cell array); final positions are kept
// in registers (u16 pairs), dirty-word records get theirs from the dense list
// pass; the output is staged through shared memory (over the dead bitmap) in
// final order and stored coalesced.
struct Bm8Cfg {
    static constexpr int RS = 8;
    static constexpr int kThreads = 1024;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kCap = LocalCfg<8>::kCap;
    static constexpr int kIpt = (kCap + kThreads - 1) / kThreads;
    static constexpr int kCellLog = RG_BM8_CELL_LOG;
#ifndef RG_BM8_BITS
#define RG_BM8_BITS 19
#endif
    static constexpr int kFineBits = RG_BM8_BITS;  // 2^19 cells: 28-32 per record at C2's bins
    static constexpr int kWords = 1 << (kFineBits - 5);
    static constexpr int kRows = (kWords + 128 * kWarps - 1) / (128 * kWarps);
    static_assert(kRows >= 1 && kRows <= 4, "scan rows per warp");
    // records of dirty words: {e, window} and their final positions (u16); a
    // dirty word's descriptor lives in its bitmap word. (The records are in
    // registers: with the windows in the list the dense pass needs no global
    // loads -- re-reading them from L2 instead cost C2's local sort +11%.)
    static constexpr int kDirty = 6144;
    static constexpr size_t kBmBytes = size_t(kWords) * 6 + size_t(kDirty) * (8 + 2);
    static constexpr size_t kStageBytes = size_t(kCap) * RS;
    static constexpr size_t kSmem = kBmBytes > kStageBytes ? kBmBytes : kStageBytes;
    static_assert(kCap < 32768, "positions are u15");
};

template <typename Mid>
__device__ __forceinline__ void local_group_bm8(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group g, uint32_t ks,
    LevelCounters* __restrict__ ctr, const GroupList spill, Mid&& mid) {
    using C = Bm8Cfg;
    constexpr int RS = 8;
    constexpr int T = C::kThreads, W = C::kWarps, IPT = C::kIpt, R = C::kRows;
    extern __shared__ __align__(128) uint8_t smem[];
    RG_CHK_POISON_SMEM(smem);
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem);              // [kWords] cell bits
    uint32_t* pre = bm + C::kWords;                                // [kWords] u16: extras, then starts
    uint2* dl = reinterpret_cast<uint2*>(pre + C::kWords / 2);     // [kDirty] {e, window}, run by run
    uint16_t* dfin = reinterpret_cast<uint16_t*>(dl + C::kDirty);  // [kDirty] final position of list entry i
    __shared__ uint32_t s_scan[W];
    __shared__ uint32_t s_wmin, s_wmax, s_alloc, s_crowd;

    const uint32_t n = g.size;
    const uint8_t* gsrc = (g.parity ? tmp : data) + g.start * RS;
    uint8_t* dst = data + g.start * RS;
    const int lane = threadIdx.x & 31;
    const uint32_t klim = ks < uint32_t(RS) ? ks : uint32_t(RS);
    if (n <= 1 || g.p >= klim) {
        if (g.parity)
            for (uint32_t e = threadIdx.x; e < n; e += T) store_rec<RS>(dst, e, load_rec<RS>(gsrc, e));
        return;
    }

    // ---- 1. records into registers; bitmap and counters zeroed
    Rec<RS> r[IPT];
    {
        const uint8_t* tsrc = gsrc + size_t(threadIdx.x) * RS;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T >= n) break;  // block-uniform
            if (uint32_t(j) * T + threadIdx.x < n) r[j] = load_rec_stream<RS>(tsrc, uint64_t(j) * T);
        }
    }
    if (threadIdx.x == 0) {
        s_wmin = 0xFFFFFFFFu;
        s_wmax = 0u;
        s_alloc = 0;
        s_crowd = 0;
    }
    uint32_t FB = 32u + uint32_t(C::kCellLog) - __clz(n - 1);  // ceil(log2 n) + kCellLog (n >= 2)
    FB = FB < 12u ? 12u : (FB > uint32_t(C::kFineBits) ? uint32_t(C::kFineBits) : FB);
    const uint32_t nW = 1u << (FB - 5);
    {
        uint4* z = reinterpret_cast<uint4*>(bm);
#pragma unroll
        for (int q = 0; q < (C::kWords / 4 + T - 1) / T; ++q)
            if (q * T + threadIdx.x < nW / 4) z[q * T + threadIdx.x] = make_uint4(0, 0, 0, 0);
        uint4* z2 = reinterpret_cast<uint4*>(pre);
#pragma unroll
        for (int q = 0; q < (C::kWords / 8 + T - 1) / T; ++q)
            if (q * T + threadIdx.x < nW / 8) z2[q * T + threadIdx.x] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();

    // ---- 2./3. windows (key bytes p..p+3, one byte permute), cell bits
    const uint32_t nwin = klim - g.p < 4u ? klim - g.p : 4u;
    const bool beyond = g.p + 4u < klim;
    uint32_t Ldef[4] = {g.p, g.p + 1, g.p + 2, g.p + 3};
    const WindowSel ws = make_window_sel(Ldef, nwin, RS / 4, true);
    const bool known = RG_BM_KNOWN && (g.pad & 0x10000u) != 0u;
    const uint32_t ncell = 1u << FB;
    auto mul_of = [&](uint32_t rm1) {
        return rm1 < ncell ? 0u
                           : uint32_t(__fdiv_rz(float(ncell) * 4294967296.0f, float(rm1) + 1.0f) * 0.999999f);
    };
    auto mark = [&](uint32_t f) {
        const uint32_t bit = 1u << (f & 31u);
        const uint32_t old = atomicOr(&bm[f >> 5], bit);
        if (old & bit) atomicAdd(&pre[f >> 6], 1u << ((f >> 1) & 16u));
    };
    uint32_t wmin, mul;
    if (known) {
        const uint32_t d0 = g.pad & 0xFFu, d1 = (g.pad >> 8) & 0xFFu;
        wmin = d0 << 24;
        mul = mul_of(((d1 - d0 + 1u) << 24) - 1u);
    } else {
        uint32_t smn = 0xFFFFFFFFu, smx = 0u;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T >= n) break;
            if (uint32_t(j) * T + threadIdx.x < n) {
                const uint32_t w = rec_window<RS>(r[j], ws);
                smn = min(smn, w);
                smx = max(smx, w);
            }
        }
        smn = __reduce_min_sync(0xFFFFFFFFu, smn);
        smx = __reduce_max_sync(0xFFFFFFFFu, smx);
        if (lane == 0) {
            atomicMin(&s_wmin, smn);
            atomicMax(&s_wmax, smx);
        }
        __syncthreads();
        wmin = s_wmin;
        const uint32_t rm1 = s_wmax - wmin;
        if (rm1 == 0 && !beyond) {  // every key equal: stable order is the input order
            if (g.parity) {
#pragma unroll
                for (int j = 0; j < IPT; ++j) {
                    if (uint32_t(j) * T >= n) break;
                    const uint32_t e = uint32_t(j) * T + threadIdx.x;
                    if (e < n) store_rec<RS>(dst, e, r[j]);
                }
            }
            return;
        }
        mul = mul_of(rm1);
    }
    auto cell_of = [&](const Rec<RS>& v) -> uint32_t {
        const uint32_t d = rec_window<RS>(v, ws) - wmin;
        return min(mul ? __umulhi(d, mul) : d, ncell - 1u);
    };
    mid();
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (uint32_t(j) * T >= n) break;
        if (uint32_t(j) * T + threadIdx.x < n) mark(cell_of(r[j]));
    }
    __syncthreads();

    // ---- 4. scan (bm_scan): word starts; a dirty word's descriptor in its bitmap word
    bm_scan<W, R>(bm, pre, nW, s_scan, &s_alloc, &s_crowd);
    __syncthreads();
    const uint32_t nd = s_alloc;  // records of dirty words
    if (s_crowd || nd > uint32_t(C::kDirty)) {
        // block-uniform; nothing written yet: the bucket sort takes the group
        if (threadIdx.x == 0) {
            push_group(spill, g);
            atomicAdd(&ctr->bm_spill, 1u);
        }
        return;
    }

    // ---- 5. final positions into registers (u16 pairs); records of dirty
    // words go to their word's list run and remember their list slot
    const uint16_t* pre16 = reinterpret_cast<const uint16_t*>(pre);
    uint32_t pp[(IPT + 1) / 2];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if ((j & 1) == 0) pp[j / 2] = 0;
        if (uint32_t(j) * T >= n) continue;  // block-uniform
        const uint32_t e = uint32_t(j) * T + threadIdx.x;
        if (e < n) {
            const uint32_t f = cell_of(r[j]), word = f >> 5;
            const uint32_t pv = pre16[word];
            const uint32_t m = bm[word];
            uint32_t pos;
            if (pv < 0x8000u) {
                pos = pv + __popc(m & ((1u << (f & 31u)) - 1u));
            } else {
                const uint32_t old = atomicAdd(&bm[word], 1u << 24);
                const uint32_t slot = (pv & 0x7FFFu) + (old >> 24);
                dl[slot] = make_uint2(e, rec_window<RS>(r[j], ws));
                pos = 0x8000u | slot;
            }
            pp[j / 2] |= pos << ((j & 1) * 16);
        }
    }
    if (nd) {
        __syncthreads();
        // ---- 6. dirty words, densely from the list: each entry finds its word
        // (window -> cell) and ranks itself among the word's run by (window, key
        // bytes beyond the window, input index)
        auto cmp_rest = [&](uint32_t a, uint32_t b) -> int {
            for (uint32_t q = g.p + 4u; q < klim; ++q) {
                const uint32_t x = gsrc[size_t(a) * RS + q], y = gsrc[size_t(b) * RS + q];
                if (x != y) return x < y ? -1 : 1;
            }
            return 0;
        };
        for (uint32_t i = threadIdx.x; i < nd; i += T) {
            const uint2 me = dl[i];
            const uint32_t e = me.x, w = me.y;
            const uint32_t dd = w - wmin;
            const uint32_t word = min(mul ? __umulhi(dd, mul) : dd, ncell - 1u) >> 5;
            const uint32_t desc = bm[word];
            const uint32_t start = desc & 0xFFFFu, cnt = (desc >> 16) & 0xFFu;
            const uint32_t off = pre16[word] & 0x7FFFu;
            uint32_t rank = 0;
            for (uint32_t q = off; q < off + cnt; ++q) {
                if (q == i) continue;
                const uint2 o = dl[q];
                bool lt;
                if (o.y != w) {
                    lt = o.y < w;
                } else {
                    const int c = beyond ? cmp_rest(o.x, e) : 0;
                    lt = c < 0 || (c == 0 && o.x < e);
                }
                rank += lt;
            }
            dfin[i] = uint16_t(start + rank);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const uint32_t pos = (pp[j / 2] >> ((j & 1) * 16)) & 0xFFFFu;
            if (pos & 0x8000u) {
                const uint32_t fin = dfin[pos & 0x7FFFu];
                pp[j / 2] = (pp[j / 2] & ~(0xFFFFu << ((j & 1) * 16))) | (fin << ((j & 1) * 16));
            }
        }
    }
    __syncthreads();  // the bitmap structures are dead: the stage takes their place

    // ---- 7. output staged in final order, stored coalesced (all reads of the
    // source are done: safe in place)
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (uint32_t(j) * T >= n) break;
        if (uint32_t(j) * T + threadIdx.x < n)
            st_smem_rec<RS>(smem, (pp[j / 2] >> ((j & 1) * 16)) & 0xFFFFu, r[j]);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += T) store_rec<RS>(dst, i, ld_smem_rec<RS>(smem, i));
    if (threadIdx.x == 0) atomicAdd(&ctr->moved_local, (unsigned long long)n);
}

__global__ void __launch_bounds__(Bm8Cfg::kThreads, 1) k_local_bm8(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group* __restrict__ groups,
    uint32_t n_groups, uint32_t ks, LevelCounters* __restrict__ ctr, GroupList spill) {
    __shared__ __align__(16) Group s_g[2];
    uint32_t i = blockIdx.x;
    if (i >= n_groups) return;
    if (threadIdx.x == 0) s_g[0] = groups[i];
    __syncthreads();
    for (int buf = 0; i < n_groups; buf ^= 1) {
        const uint32_t nx = i + gridDim.x;
        const bool more = nx < n_groups;
        if (threadIdx.x == 0 && more) {
            for (int q = 0; q < int(sizeof(Group) / 8); ++q)
                cp_async8(reinterpret_cast<uint8_t*>(&s_g[buf ^ 1]) + 8 * q,
                          reinterpret_cast<const uint8_t*>(&groups[nx]) + 8 * q);
        }
        const Group g = s_g[buf];
        auto mid = [&] {
            if (threadIdx.x == 0 && more) {
                cp_async_wait_all();
                prefetch_group_l2<8>(data, tmp, s_g[buf ^ 1]);
            }
        };
        local_group_bm8(data, tmp, g, ks, ctr, spill, mid);
        if (threadIdx.x == 0 && more) cp_async_wait_all();
        __syncthreads();  // shared memory free for the next group; its descriptor visible
        i = nx;
    }
}

// The bucket sort (local_group) over a device-counted list: the groups the
// bitmap sort handed over. Launched right behind k_local_bm with a fixed grid
// (no host read of the count); CTAs walk the list with the grid's stride.
template <int RS>
__global__ void __launch_bounds__(LocalCfg<RS>::kThreads, LocalCfg<RS>::kMinBlocks) k_local_list(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group* __restrict__ list,
    const unsigned int* __restrict__ n_list, uint32_t list_cap, uint32_t ks,
    LevelCounters* __restrict__ ctr, Group* __restrict__ spill, unsigned int* __restrict__ n_spill,
    uint32_t spill_cap) {
    const uint32_t n = min(*n_list, list_cap);
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        local_group<RS, false>(data, tmp, list[i], ks, ctr, spill, n_spill, spill_cap, [] {});
        __syncthreads();  // shared memory free for the next group
    }
}

}  // namespace rg
