// Device-side pass planner: turns one level's per-segment digit totals into
// the next level's work lists, without a host round trip per segment.
//
// Reference: child_bins (P/include/raduls/kernels.hpp:82-94) — children tile
// the parent in digit order, advance the digit and flip the buffer parity —
// plus the bin routing of MsdSorter (P/include/raduls/detail/msd_sorter.hpp:
// 89-214: size 0 skipped, size 1 finalized, tiny bins comparison-sorted, the
// last digit finalized, the rest recursed/queued) and is_tiny
// (P/include/raduls/small_sorts.hpp:31-37). The reference's thread-share
// policy (scheduler.cpp:8-38) and task queues (task_queue.hpp) have no GPU
// counterpart: size classes decide instead —
//   * size <= kCap (local-sort capacity)   -> packed into local-sort groups,
//   * larger                               -> next level (histogram, then scatter),
// and (e) a segment whose key byte p is constant is not scattered at all: it is
// re-queued at the first varying byte (or finished when none varies), keeping
// its buffer parity.
#pragma once

#include "common.cuh"
#include "k_local.cuh"

namespace rg {

struct PlanArgs {
    Seg* segs;                           // this level; action written here
    unsigned long long* seg_tot;         // [nseg][256]: in digit totals, out exclusive digit bases
    const unsigned long long* seg_andor;  // [nseg][8]
    Group* groups;
    CopyRange* copies;
    Seg* next;
    unsigned long long* next_andor;
    uint32_t* next_tile_seg;
    LevelCounters* ctr;
    uint32_t ks;
    uint32_t tile;       // tile partition (records)
    uint32_t cap_local;  // local-sort capacity (records): larger children go to the next level
    uint32_t cap_group;  // small children are packed into groups of at most this (<= cap_local)
    uint32_t side;       // this level was histogrammed from the digit array (no AND/OR)
};

__device__ __forceinline__ uint32_t andor_byte_varies(const unsigned long long* ao, uint32_t b) {
    const unsigned long long x = ao[2 * (b >> 3)] ^ ao[2 * (b >> 3) + 1];
    return uint32_t((x >> ((b & 7u) * 8u)) & 0xFFull);
}

// A batch of a level's segments (src, contiguous, with contiguous tiles from
// tb0 on) as a level of its own: segments renumbered from 0, tile bases from
// 0, and the tile -> segment map rebuilt. One block per segment.
__global__ void k_rebase_segs(const Seg* __restrict__ src, uint32_t tb0, Seg* __restrict__ dst,
                              uint32_t* __restrict__ tile_seg, uint32_t tile) {
    const uint32_t i = blockIdx.x;
    Seg g = src[i];
    g.tile_base -= tb0;
    g.action = 0;
    if (threadIdx.x == 0) dst[i] = g;
    const uint32_t nt = uint32_t((g.size + tile - 1) / tile);
    for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) tile_seg[g.tile_base + t] = i;
}

__global__ void k_init_andor(unsigned long long* andor, uint32_t rows) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows * 8) andor[i] = (i & 1) ? 0ull : ~0ull;
}

// Emit copy-back ranges covering [start, start+size) (whole block).
__device__ void emit_copies(const PlanArgs& A, uint64_t start, uint64_t size, uint32_t* s_base) {
    const uint64_t nchunks = (size + kCopyTile - 1) / kCopyTile;
    if (threadIdx.x == 0) {
        *s_base = atomicAdd(&A.ctr->n_copy, uint32_t(nchunks));
        atomicAdd(&A.ctr->moved_copy, (unsigned long long)size);
    }
    __syncthreads();
    for (uint64_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
        CopyRange r;
        r.start = start + c * kCopyTile;
        r.size = uint32_t(min(uint64_t(kCopyTile), size - c * kCopyTile));
        r.pad = 0;
        A.copies[*s_base + c] = r;
    }
}

// Allocate one next-level segment and its tiles (single thread).
__device__ uint32_t emit_next(const PlanArgs& A, uint64_t start, uint64_t size, uint32_t p,
                              uint32_t parity, uint32_t* tile_base) {
    const uint32_t idx = atomicAdd(&A.ctr->n_next, 1u);
    const uint32_t nt = uint32_t((size + A.tile - 1) / A.tile);
    const uint32_t tb = atomicAdd(&A.ctr->n_next_tiles, nt);
    Seg s;
    s.start = start;
    s.size = size;
    s.p = p;
    s.parity = parity;
    s.tile_base = tb;
    s.action = 0;
    A.next[idx] = s;
    *tile_base = tb;
    return idx;
}

// Block-cooperative initialisation of a next-level segment's tile map and AND/OR.
__device__ __forceinline__ void init_next(const PlanArgs& A, uint32_t idx, uint32_t tb, uint64_t size) {
    const uint32_t nt = uint32_t((size + A.tile - 1) / A.tile);
    for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) A.next_tile_seg[tb + t] = idx;
    if (threadIdx.x < 8) A.next_andor[uint64_t(idx) * 8 + threadIdx.x] = (threadIdx.x & 1) ? 0ull : ~0ull;
}

// Level 0 without host round trips. k_set_seg0: the whole array as one
// segment at the first key byte that varies in the strided sample (0 if none).
__global__ void k_set_seg0(const unsigned long long* __restrict__ andor, uint32_t ks, uint64_t n,
                           Seg* __restrict__ seg) {
    const uint32_t b = threadIdx.x;  // one warp
    const bool varies = b < ks && andor_byte_varies(andor, b);
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, varies);
    if (b == 0) {
        Seg s0;
        s0.start = 0;
        s0.size = n;
        s0.p = m ? __ffs(m) - 1 : 0u;
        s0.parity = 0;
        s0.tile_base = 0;
        s0.action = 0;
        *seg = s0;
    }
}

// After the level-0 histogram: a more significant byte than the sample's
// guess varies (it varies only off the sample) -> flag = 0x100 | that byte;
// the host then redoes level 0 on it. Never the other way round: a byte that
// varies in the sample varies in the array.
__global__ void k_check_seg0(const unsigned long long* __restrict__ andor, const Seg* __restrict__ seg,
                             uint32_t ks, unsigned long long* __restrict__ flag) {
    const uint32_t b = threadIdx.x;
    const bool varies = b < ks && andor_byte_varies(andor, b);
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, varies);
    if (b == 0) {
        const uint32_t pg = m ? __ffs(m) - 1 : ks;
        *flag = (pg < ks && pg != seg->p) ? (0x100ull | pg) : 0ull;
    }
}

__global__ void __launch_bounds__(256) k_plan(PlanArgs A) {
    __shared__ unsigned long long s_cnt[kRadix], s_off[kRadix];
    __shared__ unsigned long long s_wsum[8];
    __shared__ uint32_t s_action, s_pnext, s_base, s_ngroups, s_tb0;
    __shared__ uint32_t s_next_idx[kRadix], s_next_tb[kRadix];
    __shared__ uint32_t s_wbig[8], s_wtiles[8], s_nb_base, s_nt_base;
    __shared__ uint64_t s_gstart[kRadix];
    __shared__ uint32_t s_gdig[kRadix];
    __shared__ uint32_t s_gsize[kRadix], s_P[kRadix + 1], s_nbig[kRadix], s_open[kRadix], s_end[kRadix];
    __shared__ uint32_t s_wsz[8];
    const uint32_t s = blockIdx.x;
    const Seg g = A.segs[s];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (A.side) {
        // byte p histogrammed from the digit array: it varies iff more than one
        // digit is populated; if it does not, the segment is re-queued at p + 1
        // (whose first varying byte the next level's record histogram finds)
        const uint32_t nz = __syncthreads_count(A.seg_tot[uint64_t(s) * kRadix + tid] != 0ull);
        if (tid == 0) {
            s_pnext = g.p + 1;
            s_action = nz > 1 ? 2u : (g.p + 1 >= A.ks ? 0u : 1u);
        }
    } else if (tid < 32) {  // first varying key byte >= p (AND/OR of the segment)
        const unsigned long long* ao = A.seg_andor + uint64_t(s) * 8;
        const uint32_t b = g.p + lane;
        const bool varies = b < A.ks && andor_byte_varies(ao, b);
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, varies);
        if (lane == 0) {
            const uint32_t pn = m ? g.p + __ffs(m) - 1 : A.ks;
            s_pnext = pn;
            s_action = pn >= A.ks ? 0u : (pn > g.p ? 1u : 2u);
        }
    }
    __syncthreads();
    const uint32_t action = s_action;
    if (action != 0 && g.size <= A.cap_local) {
        // a segment that fits one local-sort group (only the caller-given
        // segments of raduls_gpu_sort_segments are this small): sorted as one
        // group from byte p, no scatter
        if (tid == 0) {
            Group gr;
            gr.start = g.start;
            gr.size = uint32_t(g.size);
            gr.p = g.p;
            gr.parity = g.parity;
            gr.pad = 0;
            A.groups[atomicAdd(&A.ctr->n_groups, 1u)] = gr;
            if (g.size > A.cap_group) atomicAdd(&A.ctr->n_big_groups, 1u);
        }
        return;
    }
    if (action == 0) {  // all keys equal: finished where it lies
        if (g.parity) emit_copies(A, g.start, g.size, &s_base);
        return;
    }
    if (action == 1) {  // (e) constant byte p: skip it without moving a record
        if (tid == 0) {
            s_base = emit_next(A, g.start, g.size, s_pnext, g.parity, &s_tb0);
            atomicAdd(&A.ctr->n_skip, 1u);
        }
        __syncthreads();
        init_next(A, s_base, s_tb0, g.size);
        return;
    }

    // action 2: scatter on byte p. Exclusive digit bases (u64 block scan).
    unsigned long long* tot = A.seg_tot + uint64_t(s) * kRadix;
    const unsigned long long c = tot[tid];
    unsigned long long x = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    unsigned long long wbase = 0;
    for (int k = 0; k < warp; ++k) wbase += s_wsum[k];
    const unsigned long long off = wbase + x - c;
    tot[tid] = off;
    s_cnt[tid] = c;
    s_off[tid] = off;
    if (tid == 0) {
        A.segs[s].action = kActScatter;
        atomicAdd(&A.ctr->n_scatter_segs, 1u);
        atomicAdd(&A.ctr->moved_scatter, (unsigned long long)g.size);
    }
    __syncthreads();
    const uint32_t cp = 1u - g.parity;
    if (g.p + 1 >= A.ks) {  // last key byte: every child is final after this split
        if (cp) emit_copies(A, g.start, g.size, &s_base);
        return;
    }
    // big children -> next level: block-scan the flags and tile counts so the
    // whole block allocates with two atomics
    const unsigned long long cs = s_cnt[tid];
    const bool big = cs > A.cap_local;
    const uint32_t nt_child = big ? uint32_t((cs + A.tile - 1) / A.tile) : 0u;
    {
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, big);
        uint32_t t = nt_child;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
            if (lane >= o) t += y;
        }
        if (lane == 31) s_wbig[warp] = __popc(bal), s_wtiles[warp] = t;
        __syncthreads();
        if (tid == 0) {
            uint32_t nb = 0, nt = 0;
            for (int k = 0; k < 8; ++k) {
                const uint32_t a = s_wbig[k], b = s_wtiles[k];
                s_wbig[k] = nb, s_wtiles[k] = nt;
                nb += a, nt += b;
            }
            s_nb_base = nb ? atomicAdd(&A.ctr->n_next, nb) : 0u;
            s_nt_base = nt ? atomicAdd(&A.ctr->n_next_tiles, nt) : 0u;
        }
        __syncthreads();
        s_next_idx[tid] = 0xFFFFFFFFu;
        if (big) {
            const uint32_t idx = s_nb_base + s_wbig[warp] + __popc(bal & lanemask_lt());
            const uint32_t tb = s_nt_base + s_wtiles[warp] + t - nt_child;
            Seg nx;
            nx.start = g.start + s_off[tid];
            nx.size = cs;
            nx.p = g.p + 1;
            nx.parity = cp;
            nx.tile_base = tb;
            nx.action = 0;
            A.next[idx] = nx;
            for (int w = 0; w < 8; w += 2) A.next_andor[uint64_t(idx) * 8 + w] = ~0ull,
                                             A.next_andor[uint64_t(idx) * 8 + w + 1] = 0ull;
            s_next_idx[tid] = idx;
            s_next_tb[tid] = tb;
        }
    }
    // small children -> greedy groups in digit order (a child joins the open
    // group while the group stays <= cap; a big child closes it). With the
    // exclusive prefix P of the small sizes, a group opened at digit d ends at
    // the first d' > d that is big or has P[d' + 1] - P[d] > cap: every digit
    // finds its own end by binary search (P is monotone), a suffix minimum
    // gives the next open digit, and thread 0 walks the ~n/cap-long chain.
    {
        const uint32_t cap = uint32_t(A.cap_group);  // (a child above it is a group of its own)
        const unsigned long long c = s_cnt[tid];
        const bool big = c > A.cap_local;
        const uint32_t sz = big ? 0u : uint32_t(c);
        // exclusive prefix of the small sizes (block scan over 256 digits)
        uint32_t x = sz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsz[warp] = x;
        __syncthreads();
        uint32_t wb = 0;
        for (int k = 0; k < warp; ++k) wb += s_wsz[k];
        s_P[tid] = wb + x - sz;
        if (tid == kRadix - 1) s_P[kRadix] = wb + x;
        // next big digit after d, next open (small, non-empty) digit >= d: suffix minima
        s_nbig[tid] = big ? tid : kRadix;
        s_open[tid] = sz ? tid : kRadix;
        __syncthreads();
        for (int o = 1; o < kRadix; o <<= 1) {
            const uint32_t nb = tid + o < kRadix ? s_nbig[tid + o] : kRadix;
            const uint32_t op = tid + o < kRadix ? s_open[tid + o] : kRadix;
            __syncthreads();
            s_nbig[tid] = min(s_nbig[tid], nb);
            s_open[tid] = min(s_open[tid], op);
            __syncthreads();
        }
        // end of a group opened here: first d' in (d, next big) with P[d'+1] > P[d] + cap
        if (sz) {
            const uint32_t lim = tid + 1 < kRadix ? s_nbig[tid + 1] : kRadix;  // first big after d
            const uint32_t bound = s_P[tid] + cap;
            uint32_t lo = tid + 1, hi = lim;  // answer in [lo, hi]; hi = lim: no overflow before it
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_P[mid + 1] > bound) hi = mid;
                else lo = mid + 1;
            }
            s_end[tid] = lo;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t ng = 0, nbig = 0;
            for (uint32_t d0 = s_open[0]; d0 < uint32_t(kRadix);) {
                const uint32_t e = s_end[d0];
                s_gstart[ng] = g.start + s_off[d0];
                s_gsize[ng] = s_P[e] - s_P[d0];
                s_gdig[ng] = d0 | ((e - 1u) << 8) | 0x10000u;  // byte p of the group's records lies in [d0, e)
                nbig += s_gsize[ng] > A.cap_group;
                ++ng;
                d0 = e < uint32_t(kRadix) ? s_open[e] : uint32_t(kRadix);
            }
            s_ngroups = ng;
            s_base = ng ? atomicAdd(&A.ctr->n_groups, ng) : 0u;
            if (nbig) atomicAdd(&A.ctr->n_big_groups, nbig);
        }
    }
    __syncthreads();
    if (tid < int(s_ngroups)) {
        Group gr;
        gr.start = s_gstart[tid];
        gr.size = s_gsize[tid];
        gr.p = g.p;
        gr.parity = cp;
        gr.pad = s_gdig[tid];
        A.groups[s_base + tid] = gr;
    }
    // tile -> segment map of the big children: one warp per child
    for (int d = warp; d < kRadix; d += 8) {
        const uint32_t idx = s_next_idx[d];
        if (idx == 0xFFFFFFFFu) continue;
        const uint32_t nt = uint32_t((s_cnt[d] + A.tile - 1) / A.tile);
        const uint32_t tb = s_next_tb[d];
        for (uint32_t t = lane; t < nt; t += 32) A.next_tile_seg[tb + t] = idx;
    }
}

}  // namespace rg
