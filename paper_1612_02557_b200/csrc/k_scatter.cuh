// (b) decoupled-lookback exclusive scan of bin offsets + (c) warp-ranked,
// shared-memory-staged scatter with coalesced vector stores.
//
// Reference: buffered_radix_split (P/include/raduls/kernels.hpp:175-264) —
// chunk histograms (:212-218), digit-major/chunk-minor offsets computed by one
// thread behind a std::barrier (:198-209), then 256 per-thread write-combining
// lanes flushed with SSE2 streaming stores (:221-245, :134-151). The result is
// the stable split of radix_split (kernels.hpp:157-167).
//
// B200 design (one CTA per tile of kTile records, tiles claimed through a
// dynamic ticket so every predecessor of a tile is already running):
//   1. coalesced vector loads of the tile (warp-striped: warp w owns a
//      contiguous run of 32*ITEMS records, lane-interleaved);
//   2. warp multisplit ranking with __match_any_sync: each lane learns how many
//      earlier lanes of its warp (in input order) share its digit;
//   3. per-warp counts -> per-digit tile counts and tile-local exclusive
//      offsets (digit-major, warp-minor: keeps the split stable);
//   4. decoupled look-back across the tiles of the same segment, one thread per
//      digit, over 64-bit {flag, count} status words — the GPU replacement for
//      the reference's barrier + compute_offsets;
//   5. records are staged in shared memory in digit order, then each thread
//      writes consecutive staged records to consecutive destinations, so a
//      digit run becomes one contiguous span of 16-B (or 8-B) vector stores —
//      the analogue of the reference's 256-B write-combining lanes.
// Segment-aware: a launch scatters any number of segments (MSD bins); each tile
// belongs to one segment and looks back only within it.
#pragma once

#include "common.cuh"

namespace rg {

template <int RS>
struct ScatterCfg {
    static constexpr int kThreads = 256;
    static constexpr int kItems = RS == 8 ? 16 : RS == 16 ? 8 : RS == 24 ? 5 : 4;
    static constexpr int kTile = kThreads * kItems;
    static constexpr int kWarps = kThreads / 32;
};

// Block-wide exclusive scan of one u32 per thread over the first 256 threads
// (blockDim >= 256). Returns the exclusive prefix; *total gets the sum.
__device__ __forceinline__ uint32_t scan256_exclusive(uint32_t v, uint32_t* s_warp,
                                                      uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
    }
    if (threadIdx.x < 256 && lane == 31) s_warp[warp] = x;
    __syncthreads();
    uint32_t wsum = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t c = s_warp[k];
        wsum += (k < warp) ? c : 0u;
        tot += c;
    }
    __syncthreads();
    *total = tot;
    return wsum + x - v;
}

// Digit of a record: key byte p (MSD split), or — kMap — the destination rank
// of its 16-bit key prefix at bytes (p, p+1) through a 65536-entry map (the
// multi-GPU key-range partition).
template <int RS, bool kMap>
__device__ __forceinline__ uint32_t scatter_digit(const Rec<RS>& r, uint32_t p, uint32_t ks,
                                                  const uint8_t* __restrict__ map) {
    if constexpr (kMap) {
        const uint32_t hi = p < ks ? rec_byte<RS>(r, p) : 0u;
        const uint32_t lo = p + 1 < ks ? rec_byte<RS>(r, p + 1) : 0u;
        return __ldg(map + ((hi << 8) | lo));
    } else {
        return rec_byte<RS>(r, p);
    }
}

template <int RS, bool kMap = false>
__global__ void __launch_bounds__(ScatterCfg<RS>::kThreads) k_scatter(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Seg* __restrict__ segs,
    const unsigned long long* __restrict__ seg_off,  // [nseg][256] exclusive digit offsets
    const unsigned long long* __restrict__ stile_base, const uint32_t* __restrict__ tile_seg,
    unsigned long long* __restrict__ status,  // [ntiles][256], zeroed
    LevelCounters* __restrict__ ctr, uint32_t ks = 0, const uint8_t* __restrict__ map = nullptr) {
    using C = ScatterCfg<RS>;
    constexpr int T = C::kThreads, IT = C::kItems, W = C::kWarps;
    __shared__ __align__(16) uint8_t s_recs[C::kTile * RS];
    __shared__ uint8_t s_dig[C::kTile];
    __shared__ uint32_t s_wcnt[W][kRadix];
    __shared__ uint32_t s_lstart[kRadix];
    __shared__ long long s_gdelta[kRadix];
    __shared__ uint32_t s_scan[8];
    __shared__ uint32_t s_tile;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile_ticket, 1u);
    for (int i = threadIdx.x; i < W * kRadix; i += T) (&s_wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t s = tile_seg[tile];
    const Seg g = segs[s];
    const uint64_t k = uint64_t(tile) - stile_base[s];
    const uint64_t t0 = k * C::kTile;
    const uint32_t tn = uint32_t(min(uint64_t(C::kTile), g.size - t0));
    const uint8_t* src = (g.parity ? tmp : data) + (g.start + t0) * RS;
    uint8_t* dst = (g.parity ? data : tmp);
    const uint32_t p = g.p;

    // 1-2: load + warp multisplit rank
    Rec<RS> r[IT];
    uint32_t pk[IT];  // digit (9 bits, 0x100 = invalid) | (rank within warp) << 9
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const uint32_t i = uint32_t(warp * IT + j) * 32u + lane;
        const bool valid = i < tn;
        if (valid) {
            r[j] = load_rec_stream<RS>(src, i);
        } else {
#pragma unroll
            for (int q = 0; q < Rec<RS>::kWords; ++q) r[j].w[q] = 0;
        }
        const uint32_t d = valid ? scatter_digit<RS, kMap>(r[j], p, ks, map) : 0x100u;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader && valid) {
            old = s_wcnt[warp][d];
            s_wcnt[warp][d] = old + __popc(peers);
        }
        old = __shfl_sync(0xFFFFFFFFu, old, leader);
        __syncwarp();
        pk[j] = d | ((old + __popc(peers & lt)) << 9);
    }
    __syncthreads();

    // 3: per-digit tile totals, warp-exclusive offsets, tile-local starts
    uint32_t tcount = 0;
    if (threadIdx.x < kRadix) {
        const int d = threadIdx.x;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t c = s_wcnt[w][d];
            s_wcnt[w][d] = tcount;
            tcount += c;
        }
    }
    // 4a: publish aggregate (or inclusive, for a segment's first tile) early
    unsigned long long* my_status = status + uint64_t(tile) * kRadix;
    if (threadIdx.x < kRadix)
        st_volatile_u64(my_status + threadIdx.x, (k == 0 ? kFlagIncl : kFlagAgg) | tcount);
    uint32_t total;
    const uint32_t lstart = scan256_exclusive(threadIdx.x < kRadix ? tcount : 0u, s_scan, &total);
    if (threadIdx.x < kRadix) s_lstart[threadIdx.x] = lstart;
    __syncthreads();

    // 5a: stage records in digit order
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const uint32_t d = pk[j] & 0x1FFu;
        if (d < 256u) {
            const uint32_t slot = s_lstart[d] + s_wcnt[warp][d] + (pk[j] >> 9);
            st_smem_rec<RS>(s_recs, slot, r[j]);
            s_dig[slot] = uint8_t(d);
        }
    }

    // 4b: look-back within the segment (one thread per digit)
    if (threadIdx.x < kRadix) {
        const int d = threadIdx.x;
        uint64_t excl = 0;
        if (k > 0) {
            int64_t t = int64_t(tile) - 1;
            while (true) {
                const uint64_t v = ld_volatile_u64(status + uint64_t(t) * kRadix + d);
                const uint64_t flag = v & ~kValueMask;
                if (flag == 0) continue;  // predecessor not published yet
                excl += v & kValueMask;
                if (flag == kFlagIncl) break;
                --t;
            }
            st_volatile_u64(my_status + d, kFlagIncl | (excl + tcount));
        }
        s_gdelta[d] = (long long)(g.start + seg_off[uint64_t(s) * kRadix + d] + excl) -
                      (long long)s_lstart[d];
    }
    __syncthreads();

    // 5b: coalesced write-out of the staged tile
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const uint32_t slot = uint32_t(j) * T + threadIdx.x;
        if (slot < tn) {
            const Rec<RS> v = ld_smem_rec<RS>(s_recs, slot);
            const uint32_t d = s_dig[slot];
            store_rec<RS>(dst, uint64_t(s_gdelta[d] + (long long)slot), v);
        }
    }
}

}  // namespace rg
