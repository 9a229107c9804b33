// (a) Digit histogramming in shared memory with warp-aggregated atomics, and
// (e) constant-digit detection.
//
// Reference: build_histogram (P/include/raduls/kernels.hpp:71-77) and the
// count loop of buffered_radix_split (kernels.hpp:212-218), which counts one
// digit per chunk into chunk_hist[c] so that compute_offsets (:198-209) can
// give every (chunk, digit) a disjoint destination range. Here a "chunk" is a
// scatter tile: k_tile_hist writes the 256 digit counts of every tile (the
// reference's chunk_hist) plus the AND/OR of every record word over the
// segment — a key byte is constant over a segment iff its AND byte equals its
// OR byte, which lets the planner skip it (no reference counterpart).
//
// Warp aggregation: each warp reduces AND/OR of the 32-bit word holding the
// digit with REDUX (__reduce_and_sync/__reduce_or_sync); for a digit that is
// constant across the warp one lane adds the warp's count instead of 32 lanes
// colliding on one shared-memory counter (C3's skewed byte and constant
// bytes would otherwise serialise the atomics 32 ways).
#pragma once

#include "common.cuh"
#include "k_scatter.cuh"

namespace rg {

// Warp-aggregated increment of byte-histogram `h` (256 bins) for this lane's
// value `b` (valid lanes only). `wand`/`wor` are the warp's AND/OR of the
// 32-bit word holding the byte, `shift` the byte's bit offset in that word.
__device__ __forceinline__ void warp_hist_add(uint32_t* h, uint32_t b, bool valid, uint32_t wand,
                                              uint32_t wor, uint32_t shift, uint32_t nvalid) {
    if ((((wand ^ wor) >> shift) & 0xFFu) == 0u) {
        if (lane_id() == 0 && nvalid) atomicAdd(&h[(wor >> shift) & 0xFFu], nvalid);
    } else if (valid) {
        atomicAdd(&h[b], 1u);
    }
}

// AND/OR of every 64-bit record word over a sample of the array (stride
// sampling): the first key byte that varies in the sample varies globally, so
// it is the level-0 digit unless a more significant byte varies only outside
// the sample (then the host re-histograms; the result is never wrong).
template <int RS>
__global__ void __launch_bounds__(256) k_sample_andor(const uint8_t* __restrict__ data, uint64_t n,
                                                      uint64_t stride, uint32_t samples,
                                                      unsigned long long* __restrict__ andor) {
    constexpr int KW = RS / 8;
    uint64_t a[KW], o[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < samples; s += gridDim.x * blockDim.x) {
        const uint64_t i = min(n - 1, uint64_t(s) * stride);
        const Rec<RS> r = load_rec<RS>(data, i);
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            const uint64_t v = rec_word64<RS>(r, w);
            a[w] &= v;
            o[w] |= v;
        }
    }
#pragma unroll
    for (int w = 0; w < KW; ++w) {
        for (int off = 16; off; off >>= 1) {
            a[w] &= __shfl_xor_sync(0xFFFFFFFFu, a[w], off);
            o[w] |= __shfl_xor_sync(0xFFFFFFFFu, o[w], off);
        }
        if (lane_id() == 0) {
            atomicAnd(&andor[2 * w], a[w]);
            atomicOr(&andor[2 * w + 1], o[w]);
        }
    }
}

// AND/OR of every 64-bit record word over the whole array (grid-stride).
template <int RS>
__global__ void __launch_bounds__(256) k_andor(const uint8_t* __restrict__ data, uint64_t n,
                                               unsigned long long* __restrict__ andor) {
    constexpr int KW = RS / 8;
    uint64_t a[KW], o[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const Rec<RS> r = load_rec_stream<RS>(data, i);
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            const uint64_t v = rec_word64<RS>(r, w);
            a[w] &= v;
            o[w] |= v;
        }
    }
#pragma unroll
    for (int w = 0; w < KW; ++w) {
        for (int off = 16; off; off >>= 1) {
            a[w] &= __shfl_xor_sync(0xFFFFFFFFu, a[w], off);
            o[w] |= __shfl_xor_sync(0xFFFFFFFFu, o[w], off);
        }
        if (lane_id() == 0) {
            atomicAnd(&andor[2 * w], a[w]);
            atomicOr(&andor[2 * w + 1], o[w]);
        }
    }
}

// Per-tile digit counts of byte segs[s].p for every tile of every segment of
// the level, plus AND/OR of every record word per segment, over the scatter's
// tile partition (kTile records, tile -> segment through tile_seg, tile index
// inside the segment = tile - segs[s].tile_base). tile_cnt: [ntiles][256]
// u16. seg_andor: [nseg][8] u64 (and at 2w, or at 2w+1), pre-initialised.
// kMap: the digit is the destination rank of the record's 16-bit key prefix
// at bytes (p, p+1) through a 65536-entry map (multi-GPU partition); the
// AND/OR is computed there too (the multi-GPU plan verifies its prefix byte).
//
// Persistent and warp-specialised like k_scatter: a producer warp takes tiles
// round-robin and TMA-loads them (cp.async.bulk + mbarrier) into a 2-stage
// shared-memory ring, so every SM always has tile
// loads in flight; 8 consumer warps histogram a tile from shared memory
// (warp-aggregated atomics into per-stage counts) while the next one lands,
// and a drain warp writes out each finished tile's counts and AND/OR, so
// consumer warps never wait on each other (measured against a block barrier +
// drain per tile: 6.41 vs 6.06 TB/s at C5, 6.64 vs 6.39 at C4). Tuning knobs
// measured at C5/C4: 1 CTA x 4 stages 3.9-4.6 TB/s, 4 CTAs x 1 stage 6.2,
// 512 consumers 5.0-5.7, 128 consumers 4.5-6.3 — the default is 2 x 2 x 256.
#ifndef RG_HIST_THREADS
#define RG_HIST_THREADS 256
#endif
#ifndef RG_HIST_STAGES
#define RG_HIST_STAGES 2
#endif
#ifndef RG_HIST_CTAS
#define RG_HIST_CTAS 2
#endif
template <int RS>
struct HistCfg {
    static constexpr int kThreads = RG_HIST_THREADS;  // consumer threads
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kTile = ScatterCfg<RS>::kTile;
    static constexpr int kItems = (kTile + kThreads - 1) / kThreads;
    static constexpr int kStages = RG_HIST_STAGES;
    static constexpr int kCtas = RG_HIST_CTAS;  // resident per SM (grid = kCtas x SMs)
    static constexpr int kBufBytes = ScatterCfg<RS>::kBufBytes;
    static constexpr size_t kSmem = size_t(kStages) * kBufBytes;
};

struct HistTile {
    uint32_t tile;  // >= n_tiles: none
    uint32_t seg, tn, p, head;
};

// kKey1: AND/OR of record word 0 only (the sort with ks <= 8: the other
// words are payload, whose bytes the planner never reads; C5 -1.7%).
template <int RS, bool kMap = false, bool kKey1 = false>
__global__ void __launch_bounds__(HistCfg<RS>::kThreads + 64, HistCfg<RS>::kCtas) k_tile_hist(
    const uint8_t* __restrict__ data, const uint8_t* __restrict__ tmp, const Seg* __restrict__ segs,
    const uint32_t* __restrict__ tile_seg, uint16_t* __restrict__ tile_cnt,
    unsigned long long* __restrict__ seg_andor, LevelCounters* __restrict__ ctr, uint32_t n_tiles,
    uint32_t ks = 0, const uint8_t* __restrict__ map = nullptr) {
    using C = HistCfg<RS>;
    constexpr int T = C::kThreads, W = C::kWarps, IT = C::kItems, S = C::kStages, KW = RS / 8;
    extern __shared__ __align__(128) uint8_t smem[];
    RG_CHK_POISON_SMEM(smem);
    __shared__ __align__(16) uint32_t s_h[S][kRadix];
    __shared__ unsigned long long s_and[S][W][KW], s_or[S][W][KW];
    // full: the tile landed (TMA); done: every consumer warp counted it; empty: drained
    __shared__ __align__(8) unsigned long long s_full[S], s_done[S], s_empty[S];
    __shared__ HistTile s_info[S];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < uint32_t(S * kRadix); i += blockDim.x) (&s_h[0][0])[i] = 0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&s_full[q], 1);
            mbar_init(&s_done[q], W);
            mbar_init(&s_empty[q], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == W) {  // ------------------------------------------------ producer
        if (lane != 0) return;
        // tiles round-robin (a histogram has no write locality to keep), the
        // next tile's metadata loaded while this one's buffer frees up
        uint32_t tile = blockIdx.x;
        uint32_t s = tile < n_tiles ? tile_seg[tile] : 0u;
        Seg g = tile < n_tiles ? segs[s] : Seg{};
        for (uint32_t it = 0;; ++it) {
            const int b = it % S;
            const uint32_t tnext = tile + gridDim.x;
            const uint32_t snext = tnext < n_tiles ? tile_seg[tnext] : 0u;
            if (it >= uint32_t(S)) mbar_wait(&s_empty[b], ((it / S) - 1) & 1u);
            HistTile ti;
            ti.tile = tile;
            if (tile >= n_tiles) {
                s_info[b] = ti;
                mbar_arrive_expect_tx(&s_full[b], 0);
                return;
            }
            const uint64_t k = uint64_t(tile) - g.tile_base;
            const uint8_t* gsrc = (g.parity ? tmp : data) + (g.start + k * C::kTile) * RS;
            ti.seg = s;
            ti.tn = uint32_t(min(uint64_t(C::kTile), g.size - k * C::kTile));
            ti.p = g.p;
            const uint32_t bytes = ti.tn * RS;
            const uint32_t head = uint32_t(reinterpret_cast<uintptr_t>(gsrc) & 15u);  // 0 or 8
            const uint32_t hb = head ? min(8u, bytes) : 0u;
            const uint32_t body = (bytes - hb) & ~15u;
            const uint32_t tail = bytes - hb - body;
            ti.head = head;
            uint8_t* sb = smem + b * C::kBufBytes + head;
            if (hb) *reinterpret_cast<uint2*>(sb) = *reinterpret_cast<const uint2*>(gsrc);
            if (tail)
                *reinterpret_cast<uint2*>(sb + hb + body) = *reinterpret_cast<const uint2*>(gsrc + hb + body);
            fence_proxy_async_smem();
            s_info[b] = ti;
            mbar_arrive_expect_tx(&s_full[b], body);
            if (body) tma_load_1d_h<RG_HINT_HIST>(sb + hb, gsrc + hb, body, &s_full[b]);
            const Seg gnext = tnext < n_tiles ? segs[snext] : g;
            tile = tnext;
            s = snext;
            g = gnext;
        }
    }

    if (warp == W + 1) {  // ------------------------------------------- drain
        // per tile: the 256 counts out (and cleared), the segment's AND/OR,
        // then the buffer back to the producer. Consumer warps never wait on
        // one another: each only signals `done` for the tile it counted.
        unsigned long long recs = 0;
        for (uint32_t it = 0;; ++it) {
            const int b = it % S;
            mbar_wait(&s_done[b], (it / S) & 1u);
            const HistTile ti = s_info[b];
            if (ti.tile >= n_tiles) break;
            uint4* hv = reinterpret_cast<uint4*>(s_h[b]) + lane * 2;  // digits 8 lane .. 8 lane + 7
            const uint4 x = hv[0], y = hv[1];
            hv[0] = make_uint4(0, 0, 0, 0);
            hv[1] = make_uint4(0, 0, 0, 0);
            uint4 o;
            o.x = (x.x & 0xFFFFu) | (x.y << 16);
            o.y = (x.z & 0xFFFFu) | (x.w << 16);
            o.z = (y.x & 0xFFFFu) | (y.y << 16);
            o.w = (y.z & 0xFFFFu) | (y.w << 16);
            *reinterpret_cast<uint4*>(tile_cnt + uint64_t(ti.tile) * kRadix + lane * 8) = o;
            if (lane < KW) {  // (kMap too: the multi-GPU plan checks its prefix byte with it)
                unsigned long long ra = ~0ull, ro = 0ull;
                for (int q = 0; q < W; ++q) ra &= s_and[b][q][lane], ro |= s_or[b][q][lane];
                atomicAnd(&seg_andor[uint64_t(ti.seg) * 8 + 2 * lane], ra);
                atomicOr(&seg_andor[uint64_t(ti.seg) * 8 + 2 * lane + 1], ro);
            }
            recs += ti.tn;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
        }
        if (lane == 0 && recs) atomicAdd(&ctr->hist_records, recs);
        return;
    }

    // ------------------------------------------------------------ consumers
    for (uint32_t it = 0;; ++it) {
        const int b = it % S;
        mbar_wait(&s_full[b], (it / S) & 1u);
        const HistTile ti = s_info[b];
        if (ti.tile >= n_tiles) {
            if (lane == 0) mbar_arrive(&s_done[b]);  // the drain warp sees the end too
            break;
        }
        const uint8_t* tile = smem + b * C::kBufBytes + ti.head;
        const uint32_t tn = ti.tn, p = ti.p;
        uint32_t* hb = s_h[b];
        uint64_t a[KW], o[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t i = uint32_t(warp * IT + j) * 32u + lane;  // warp-striped
            const bool valid = i < tn;
            Rec<RS> r;
            if (valid) r = ld_smem_rec<RS, false>(tile, i);  // (the half-swapped order measured +4% here)
            else
#pragma unroll
                for (int q = 0; q < Rec<RS>::kWords; ++q) r.w[q] = 0;
            if constexpr (kMap) {
                if (valid)
                    atomicAdd(&hb[map_digit([&](uint32_t b) { return rec_byte<RS>(r, b); }, p, ks, map)], 1u);
            } else {
                const uint32_t nvalid = __popc(__ballot_sync(0xFFFFFFFFu, valid));
                const uint32_t word = rec_word32<RS>(r, p >> 2);
                const uint32_t wa = __reduce_and_sync(0xFFFFFFFFu, valid ? word : ~0u);
                const uint32_t wo = __reduce_or_sync(0xFFFFFFFFu, valid ? word : 0u);
                const uint32_t shf = (p & 3u) * 8u;
                warp_hist_add(hb, (word >> shf) & 0xFFu, valid, wa, wo, shf, nvalid);
            }
            if (valid) {
#pragma unroll
                for (int w = 0; w < (kKey1 ? 1 : KW); ++w) {
                    const uint64_t v = rec_word64<RS>(r, w);
                    a[w] &= v;
                    o[w] |= v;
                }
            }
        }
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            for (int off = 16; off; off >>= 1) {
                a[w] &= __shfl_xor_sync(0xFFFFFFFFu, a[w], off);
                o[w] |= __shfl_xor_sync(0xFFFFFFFFu, o[w], off);
            }
            if (lane == 0) s_and[b][warp][w] = a[w], s_or[b][warp][w] = o[w];
        }
        __syncwarp();  // the warp's counts and partials before its arrival
        if (lane == 0) mbar_arrive(&s_done[b]);
    }
}

// 8-B records: one CTA per tile, all loads in flight in registers (measured
// 5.2 TB/s at C2 against 4.4 for the TMA-fed kernel, whose 8 consumer warps
// cannot keep up with 16 records each). Threads of a CTA: ~8 records in
// flight per thread (16 at 8 B), a multiple of 32, >= 256 for the digit counts.
template <int RS, int kTile>
struct HistRegCfg {
    static constexpr int kIt = RS == 8 ? 16 : 8;
    static constexpr int kThreads = ((kTile + kIt - 1) / kIt + 31) / 32 * 32 < 256
                                        ? 256
                                        : ((kTile + kIt - 1) / kIt + 31) / 32 * 32;
};

template <int RS, int kTile, bool kMap = false>
__global__ void __launch_bounds__(HistRegCfg<RS, kTile>::kThreads) k_tile_hist_reg(const uint8_t* __restrict__ data,
                                                   const uint8_t* __restrict__ tmp,
                                                   const Seg* __restrict__ segs,
                                                   const uint32_t* __restrict__ tile_seg,
                                                   uint16_t* __restrict__ tile_cnt,
                                                   unsigned long long* __restrict__ seg_andor,
                                                   LevelCounters* __restrict__ ctr, uint32_t ks,
                                                   const uint8_t* __restrict__ map,
                                                   uint32_t ahead) {  // ~ resident CTAs: 4 per SM
    constexpr int KW = RS / 8;
    constexpr int HT = HistRegCfg<RS, kTile>::kThreads, HW = HT / 32;
    constexpr int IT = (kTile + HT - 1) / HT;
    __shared__ uint32_t sh[kRadix];
    __shared__ unsigned long long s_and[HW][KW], s_or[HW][KW];
    if (threadIdx.x < kRadix) sh[threadIdx.x] = 0;
    const uint32_t tile = blockIdx.x;
    const uint32_t s = tile_seg[tile];
    const Seg g = segs[s];
    const uint64_t k = uint64_t(tile) - g.tile_base;
    const uint8_t* src = (g.parity ? tmp : data) + (g.start + k * kTile) * RS;
    const uint32_t tn = uint32_t(min(uint64_t(kTile), g.size - k * kTile));
    const uint32_t p = g.p;
    // 8-B records: pull the tile one resident wave ahead toward L2 (its CTA
    // then starts on L2 hits; measured +4% at C2, a loss at 16 B)
    if (RS == 8 && threadIdx.x == 0 && tile + ahead < gridDim.x) {
        const uint32_t t2 = tile + ahead;
        const Seg g2 = segs[tile_seg[t2]];
        const uint64_t k2 = uint64_t(t2) - g2.tile_base;
        const uint64_t n2 = min(uint64_t(kTile), g2.size - k2 * kTile);
        const uintptr_t a0 = reinterpret_cast<uintptr_t>((g2.parity ? tmp : data) + (g2.start + k2 * kTile) * RS);
        const uintptr_t a = (a0 + 15) & ~uintptr_t(15), e = (a0 + n2 * RS) & ~uintptr_t(15);
        if (e > a) {
            RG_CHK_G(reinterpret_cast<const void*>(a), uint32_t(e - a), kChkPrefetch);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(uint32_t(e - a)) : "memory");
        }
    }
    Rec<RS> r[IT];
#pragma unroll
    for (int j = 0; j < IT; ++j) {  // all loads in flight
        const uint32_t i = uint32_t(j) * HT + threadIdx.x;
        if (i < tn) {
            r[j] = load_rec_stream<RS>(src, i);
        } else {
#pragma unroll
            for (int q = 0; q < Rec<RS>::kWords; ++q) r[j].w[q] = 0;
        }
    }
    __syncthreads();
    uint64_t a[KW], o[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const uint32_t i = uint32_t(j) * HT + threadIdx.x;
        const bool valid = i < tn;
        if constexpr (kMap) {
            if (valid)
                atomicAdd(&sh[map_digit([&](uint32_t b) { return rec_byte<RS>(r[j], b); }, p, ks, map)], 1u);
        } else {
            const uint32_t nvalid = __popc(__ballot_sync(0xFFFFFFFFu, valid));
            const uint32_t word = rec_word32<RS>(r[j], p >> 2);
            const uint32_t wa = __reduce_and_sync(0xFFFFFFFFu, valid ? word : ~0u);
            const uint32_t wo = __reduce_or_sync(0xFFFFFFFFu, valid ? word : 0u);
            const uint32_t shf = (p & 3u) * 8u;
            warp_hist_add(sh, (word >> shf) & 0xFFu, valid, wa, wo, shf, nvalid);
        }
        if (valid) {
#pragma unroll
            for (int w = 0; w < KW; ++w) {
                const uint64_t v = rec_word64<RS>(r[j], w);
                a[w] &= v;
                o[w] |= v;
            }
        }
    }
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < KW; ++w) {
        for (int off = 16; off; off >>= 1) {
            a[w] &= __shfl_xor_sync(0xFFFFFFFFu, a[w], off);
            o[w] |= __shfl_xor_sync(0xFFFFFFFFu, o[w], off);
        }
        if (lane_id() == 0) s_and[warp][w] = a[w], s_or[warp][w] = o[w];
    }
    __syncthreads();
    if (threadIdx.x < KW) {
        unsigned long long ra = ~0ull, ro = 0ull;
        for (int q = 0; q < HW; ++q) ra &= s_and[q][threadIdx.x], ro |= s_or[q][threadIdx.x];
        atomicAnd(&seg_andor[uint64_t(s) * 8 + 2 * threadIdx.x], ra);
        atomicOr(&seg_andor[uint64_t(s) * 8 + 2 * threadIdx.x + 1], ro);
    }
    if (threadIdx.x == 0) atomicAdd(&ctr->hist_records, (unsigned long long)tn);
    if (threadIdx.x < kRadix) tile_cnt[uint64_t(tile) * kRadix + threadIdx.x] = uint16_t(sh[threadIdx.x]);
}

// Tile histogram of a level whose key bytes were written by the previous
// level's scatter into the digit array `nd` (one byte per record position:
// the byte p of every record of every segment of this level). The histogram
// then reads 1 byte per record instead of the whole record (rs bytes): at C5
// 4.3 GB instead of 68.7 GB per level. One warp per tile (tiles round-robin
// over all warps), warp-private shared-memory counts, 16-B vector loads of
// the tile's bytes, counts flushed as u16 like k_tile_hist. No AND/OR: the
// planner reads constancy of byte p off the digit totals (one non-zero digit).
constexpr int kNdWarps = 8;
#ifndef RG_ND_CH
#define RG_ND_CH 6
#endif

template <int kTile>
__global__ void __launch_bounds__(kNdWarps * 32, 4) k_tile_hist_nd(
    const uint8_t* __restrict__ nd, const Seg* __restrict__ segs, const uint32_t* __restrict__ tile_seg,
    uint16_t* __restrict__ tile_cnt, LevelCounters* __restrict__ ctr, uint32_t n_tiles) {
    __shared__ __align__(16) uint32_t s_h[kNdWarps][kRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* h = s_h[warp];
#pragma unroll
    for (int q = 0; q < kRadix / 32; ++q) h[q * 32 + lane] = 0;
    __syncwarp();
    const uint32_t nwarps = gridDim.x * kNdWarps;
    uint32_t tile = blockIdx.x * kNdWarps + warp;
    unsigned long long recs = 0;
    Seg g = tile < n_tiles ? segs[tile_seg[tile]] : Seg{};
    constexpr int kIt = (kTile + 15) / 512 + 1;  // 16-B vectors per lane covering a tile (any alignment)
    constexpr int kCh = RG_ND_CH;
    while (tile < n_tiles) {
        const uint32_t tnext = tile + nwarps;
        const Seg gnext = tnext < n_tiles ? segs[tile_seg[tnext]] : g;  // next tile's metadata in flight
        const uint64_t k = uint64_t(tile) - g.tile_base;
        const uint64_t start = g.start + k * kTile;
        const uint32_t tn = uint32_t(min(uint64_t(kTile), g.size - k * kTile));
        const uint64_t a0 = start & ~uint64_t(15), end = start + tn;
#pragma unroll
        for (int j0 = 0; j0 < kIt; j0 += kCh) {  // kCh vectors per lane in flight (register budget)
            uint4 v[kCh];
#pragma unroll
            for (int j = 0; j < kCh; ++j) {
                const uint64_t off = a0 + uint64_t((j0 + j) * 32 + lane) * 16;
                if (j0 + j < kIt && off < end) {
                    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                        : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w)
                        : "l"(nd + off));
                }
            }
#pragma unroll
            for (int j = 0; j < kCh; ++j) {
                const uint64_t off = a0 + uint64_t((j0 + j) * 32 + lane) * 16;
                if (j0 + j >= kIt || off >= end) continue;
                const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
                if (off >= start && off + 16 <= end) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) atomicAdd(&h[(w[q >> 2] >> ((q & 3) * 8)) & 0xFFu], 1u);
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const uint64_t pos = off + q;
                        if (pos >= start && pos < end) atomicAdd(&h[(w[q >> 2] >> ((q & 3) * 8)) & 0xFFu], 1u);
                    }
                }
            }
        }
        __syncwarp();
        uint4* hv = reinterpret_cast<uint4*>(h) + lane * 2;  // digits 8 lane .. 8 lane + 7
        const uint4 x = hv[0], y = hv[1];
        hv[0] = make_uint4(0, 0, 0, 0);
        hv[1] = make_uint4(0, 0, 0, 0);
        uint4 o;
        o.x = (x.x & 0xFFFFu) | (x.y << 16);
        o.y = (x.z & 0xFFFFu) | (x.w << 16);
        o.z = (y.x & 0xFFFFu) | (y.y << 16);
        o.w = (y.z & 0xFFFFu) | (y.w << 16);
        *reinterpret_cast<uint4*>(tile_cnt + uint64_t(tile) * kRadix + lane * 8) = o;
        __syncwarp();
        recs += tn;
        tile = tnext;
        g = gnext;
    }
    if (lane == 0 && recs) atomicAdd(&ctr->hist_digit_records, recs);
}

}  // namespace rg
