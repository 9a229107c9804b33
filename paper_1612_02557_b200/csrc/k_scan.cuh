// (b) Decoupled-lookback device-wide exclusive scan of bin offsets.
//
// Reference: compute_offsets inside buffered_radix_split
// (P/include/raduls/kernels.hpp:198-209), run by one thread behind a
// std::barrier: for every digit d and chunk c (digit-major, chunk-minor)
//     chunk_base[c][d] = sum over chunks c' < c of chunk_hist[c'][d]
//                        + sum over digits d' < d of the total count of d'.
// Here the chunks are the scatter tiles of every segment of an MSD level.
// k_tile_scan computes, for every tile t and digit d, the exclusive prefix of
// tile_cnt over the earlier tiles of the same segment (tile_off[t][d]) and the
// per-segment digit totals — a segmented scan along the tile axis done with
// decoupled look-back: each CTA scans kScanChunk consecutive tiles (one thread
// per digit), publishes its running sum at once (aggregate, or inclusive when
// the chunk holds its segment's first tile), then walks back over earlier
// chunks' {flag, value} words until it meets an inclusive one. The digit-major
// term is added by the planner (k_plan) from the totals.
#pragma once

#include "common.cuh"

namespace rg {

#ifndef RG_SCAN_CHUNK
#define RG_SCAN_CHUNK 64
#endif
#ifndef RG_SCAN_LOOK
#define RG_SCAN_LOOK 4
#endif
constexpr int kScanChunk = RG_SCAN_CHUNK;

// Look-back over earlier chunks' status words for digit d, starting at chunk
// c-1, until an inclusive prefix; returns the exclusive prefix.
__device__ __forceinline__ unsigned long long lookback_chunks(const unsigned long long* status,
                                                              int64_t c, int d) {
    constexpr int kLook = RG_SCAN_LOOK;
    unsigned long long excl = 0;
    int64_t t = c - 1;
    while (true) {
        unsigned long long v[kLook];
#pragma unroll
        for (int q = 0; q < kLook; ++q)
            v[q] = (t - q >= 0) ? ld_volatile_u64(status + uint64_t(t - q) * kRadix + d) : kFlagIncl;
        bool done = false;
        int used = 0;
#pragma unroll
        for (int q = 0; q < kLook; ++q) {
            if (done || used != q) continue;
            const unsigned long long flag = v[q] & ~kValueMask;
            if (flag == 0) continue;  // not yet published: re-poll from here
            excl += v[q] & kValueMask;
            ++used;
            if (flag == kFlagIncl) done = true;
        }
        if (done) return excl;
        t -= used;
    }
}

template <int kTile>
__global__ void __launch_bounds__(256) k_tile_scan(const Seg* __restrict__ segs,
                                                   const uint32_t* __restrict__ tile_seg,
                                                   const uint16_t* __restrict__ tile_cnt,
                                                   uint32_t n_tiles, uint32_t* __restrict__ tile_off,
                                                   unsigned long long* __restrict__ seg_tot,
                                                   unsigned long long* __restrict__ status,
                                                   LevelCounters* __restrict__ ctr) {
    __shared__ uint32_t s_chunk;
    __shared__ uint32_t s_seg[kScanChunk];
    __shared__ uint8_t s_head[kScanChunk], s_last[kScanChunk];
    if (threadIdx.x == 0) s_chunk = atomicAdd(&ctr->scan_ticket, 1u);
    __syncthreads();
    const uint32_t c = s_chunk;
    const uint32_t t0 = c * kScanChunk;
    const uint32_t tn = min(uint32_t(kScanChunk), n_tiles - t0);
    if (threadIdx.x < tn) {
        const uint32_t t = t0 + threadIdx.x;
        const uint32_t s = tile_seg[t];
        const Seg g = segs[s];
        const uint32_t nt = uint32_t((g.size + kTile - 1) / kTile);
        s_seg[threadIdx.x] = s;
        s_head[threadIdx.x] = t == g.tile_base;
        s_last[threadIdx.x] = t == g.tile_base + nt - 1;
    }
    __syncthreads();
    const int d = threadIdx.x;
    const uint16_t* cnt = tile_cnt + uint64_t(t0) * kRadix + d;
    // pass 1: the chunk's trailing segmented sum (independent loads, unrolled)
    unsigned long long run = 0;
    int first_head = kScanChunk;
#pragma unroll 16
    for (int q = 0; q < kScanChunk; ++q) {
        if (uint32_t(q) < tn) {
            if (s_head[q]) {
                run = 0;
                if (first_head == kScanChunk) first_head = q;
            }
            run += cnt[uint64_t(q) * kRadix];
        }
    }
    unsigned long long excl = 0;
    unsigned long long* my = status + uint64_t(c) * kRadix + d;
    if (first_head < kScanChunk) {
        // the trailing run starts at a segment head inside this chunk: its
        // prefix is complete, publish it at once
        st_volatile_u64(my, kFlagIncl | run);
        // tiles before the head continue a segment begun in an earlier chunk
        if (first_head > 0) excl = lookback_chunks(status, int64_t(c), d);
    } else {
        st_volatile_u64(my, kFlagAgg | run);
        excl = lookback_chunks(status, int64_t(c), d);
        st_volatile_u64(my, kFlagIncl | (excl + run));
    }
    // pass 2: per-tile exclusive offsets (the counts again, now cache-hot)
    unsigned long long loc = excl;
#pragma unroll 16
    for (int q = 0; q < kScanChunk; ++q) {
        if (uint32_t(q) < tn) {
            if (s_head[q]) loc = 0;
            const uint32_t k = cnt[uint64_t(q) * kRadix];
            tile_off[uint64_t(t0 + q) * kRadix + d] = uint32_t(loc);
            if (s_last[q]) seg_tot[uint64_t(s_seg[q]) * kRadix + d] = loc + k;
            loc += k;
        }
    }
}

}  // namespace rg
