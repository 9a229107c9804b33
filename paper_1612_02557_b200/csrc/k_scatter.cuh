// (c) Scatter pass: warp-ranked, shared-memory-staged, coalesced vector stores.
//
// Reference: the scatter loop of buffered_radix_split
// (P/include/raduls/kernels.hpp:221-245): records are copied into one of 256
// per-thread write-combining lanes by digit and every full lane is flushed as
// one contiguous block with SSE2 streaming stores (flush_block, :134-151), at
// destinations fixed beforehand by compute_offsets (:198-209). The result is
// the stable split of radix_split (kernels.hpp:157-167).
//
// B200 design — persistent and warp-specialised:
//   * warp 8 (producer) claims tiles in order through a global ticket, skips tiles of segments the planner did not split,
//     and TMA-loads each tile (cp.async.bulk, mbarrier transaction count) into
//     one of two shared-memory buffers;
//   * warps 0-7 (consumers) rank the tile's records by digit inside their warp
//     (warp_rank, common.cuh; warp-striped input order, warp-private counters,
//     digit-major/warp-minor offsets): kRank 1 -- peers of a digit from eight
//     ballots, rank = counter + popc(peers & lanemask_lt), stable by
//     construction; kRank 0 -- one shared-memory atomic per record, stable only
//     if the hardware serves the lanes of one atomic in lane order, so it is
//     launched only after k_rank_selftest confirmed that on the device
//     (atomic_rank_ok, raduls_gpu.cu; C5 scatter 73.6 vs 94.7 ms). They then
//     build a slot map in digit order, and write the records out in
//     that order: consecutive slots of one digit go to consecutive destinations,
//     so every digit run becomes one contiguous span of 16-B (8-B) vector
//     stores — the GPU analogue of the 256-B write-combining lanes.
// With `nd` (the digit array), records whose child is split again next level
// also store their next key byte at their destination index, so that level's
// histogram reads 1 byte per record instead of the record (k_tile_hist_nd).
// Destinations come from k_tile_scan (per-tile digit offsets inside the
// segment, the decoupled-lookback scan) and k_plan (digit bases): no tile waits
// on another, so prefetching the next tile cannot stall anyone.
#pragma once

#include "common.cuh"

namespace rg {

#ifndef RG_SC_NDSMEM
#define RG_SC_NDSMEM 1
#endif
#ifndef RG_SC_STAGES
#define RG_SC_STAGES 2
#endif
#ifndef RG_HINT_NDST
#define RG_HINT_NDST 0
#endif
#ifndef RG_SC_EARLY8
#define RG_SC_EARLY8 1
#endif
#ifndef RG_SC_EARLY16
#define RG_SC_EARLY16 0
#endif
#ifndef RG_SC_CTAS
#define RG_SC_CTAS 2
#endif
#ifndef RG_SC_U4
#define RG_SC_U4 11
#endif
#ifndef RG_SC_ITEMS16
#define RG_SC_ITEMS16 11
#endif
constexpr int kScUnroll = RG_SC_U4;  // write-out loop unroll (11 vs 4: C1 -1%, C2 -1.2%, C5 -0.5%)

template <int RS>
struct ScatterCfg {
    static constexpr int kThreads = 256;
    static constexpr int kItems = RS == 8 ? 20 : RS == 16 ? RG_SC_ITEMS16 : RS == 24 ? 7 : 6;
    static constexpr int kTile = kThreads * kItems;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kStages = RG_SC_STAGES;  // tile buffers in the TMA ring
    static constexpr int kCtas = RG_SC_CTAS;      // resident per SM (grid = kCtas x SMs)
    static constexpr int kBufBytes = ((kTile * RS + 16 + 127) / 128) * 128;  // + alignment slack
    static constexpr size_t kSmem = size_t(kStages) * kBufBytes + size_t(kTile) * 4;  // ring + slot map
    // plain split (no map): + the tile's digit bytes per stage, u16 slot map
    static constexpr int kNdBytes = ((kTile + 32 + 15) / 16) * 16;
    // (32-B records only: their record byte reads are 8-way bank-conflicted;
    // measured a loss at 8/16/24 B, where the u16 map's digit re-extraction
    // and the second bulk copy cost more than the 2-4-way conflicts saved)
    static constexpr bool kNdSmem = RG_SC_NDSMEM && RS == 32;
    static constexpr size_t kSmemPlain = kNdSmem ? size_t(kStages) * (kBufBytes + kNdBytes) + size_t(kTile) * 2
                                                 : kSmem;
};

// Exclusive scan of one u32 per thread over the 256 consumer threads (named
// barrier 1; every consumer thread must call it). Returns the exclusive prefix; *total gets the sum.
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
    bar_sync_named(1, 256);
    uint32_t wsum = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t c = s_warp[k];
        wsum += (k < warp) ? c : 0u;
        tot += c;
    }
    bar_sync_named(1, 256);
    *total = tot;
    return wsum + x - v;
}

// Digit of a staged record: key byte p (MSD split), or — kMap — the
// destination digit of its 16-bit key prefix at bytes (p, p+1) through the
// partition map (map_digit: 65536 entries + pivot keys; the multi-GPU
// key-range partition).
template <int RS, bool kMap>
__device__ __forceinline__ uint32_t scatter_digit_smem(const uint8_t* rec, uint32_t p, uint32_t ks,
                                                       const uint8_t* __restrict__ map) {
    if constexpr (kMap) {
        return map_digit([&](uint32_t b) { return uint32_t(rec[b]); }, p, ks, map);
    } else {
        return rec[p];
    }
}

// Per-tile facts resolved by the issuing thread when the tile is claimed.
struct TileInfo {
    uint32_t tile;    // ticket (status row); >= n_tiles: none
    uint32_t seg;
    uint32_t tn;      // records in the tile
    uint32_t p;
    uint32_t parity;
    uint32_t head;    // byte offset of the tile inside its smem buffer (0 or 8)
    uint64_t k;       // tile index inside the segment
    uint64_t gstart;  // first record of the tile (global record index)
    uint64_t seg_start;
    uint64_t seg_size;
    uint32_t ndh;  // offset of the tile's first digit byte in its stage's digit buffer (nd_in)
    uint32_t pad;
};

// kPeer (the multi-GPU partition): digit d's records are
// stored straight to dig_dst[d] — a peer GPU's receive buffer over NVLink (P2P
// or CUDA-IPC mapped), at this source's offset there — so the all-to-all is
// carried out by the partition's own coalesced stores, tile by tile, instead
// of a separate collective. A digit whose run is split across several
// destinations (one hot key spread over ranks by count) has bit 63 set in
// dig_dst[d] and its pieces at pieces[dig_dst[d] & 0x7FFFFFFF ...]: the
// record at index i of the digit's run goes to the first piece with
// i < end, at address adj + i * RS.
struct Piece {
    unsigned long long end;  // exclusive end index of the piece inside the digit's run
    unsigned long long adj;  // destination address of the piece's first record - its start index * RS
};

// kRank: warp_rank mode (0: atomic ranks, device-checked; 1: ballot ranks).
template <int RS, bool kMap = false, bool kPeer = false, int kRank = 0>
__global__ void __launch_bounds__(ScatterCfg<RS>::kThreads + 32, ScatterCfg<RS>::kCtas) k_scatter(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Seg* __restrict__ segs,
    const unsigned long long* __restrict__ seg_base,  // [nseg][256] exclusive digit bases
    const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_off,  // [ntiles][256]
    uint32_t n_tiles, unsigned int* __restrict__ ticket, uint32_t ks = 0,
    const uint8_t* __restrict__ map = nullptr,
    const unsigned long long* __restrict__ dig_dst = nullptr, uint8_t* __restrict__ nd = nullptr,
    uint32_t cap_local = 0, const uint8_t* __restrict__ nd_in = nullptr,
    const Piece* __restrict__ pieces = nullptr) {
    using C = ScatterCfg<RS>;
    constexpr int T = C::kThreads, IT = C::kItems, W = C::kWarps;
    extern __shared__ __align__(128) uint8_t smem[];
    RG_CHK_POISON_SMEM(smem);
    uint8_t* buf0 = smem;
    constexpr int S = C::kStages;
    // Plain split: the digits can come TMA-loaded from nd_in (this level's
    // digit array) into a per-stage byte buffer — conflict-free byte reads
    // instead of 4-way bank-conflicted reads of the records — and the slot
    // map is u16 (record index | nd flag << 15; step 4 re-reads the digit from
    // the record it loads anyway).
    constexpr bool kU16 = !kMap && C::kNdSmem;
    uint8_t* snd = smem + S * C::kBufBytes;  // [S][kNdBytes] (kU16)
    // slot map: record index | digit << 16 | nd flag << 24, in digit order (u32), or (kU16) u16
    uint32_t* s_map = reinterpret_cast<uint32_t*>(smem + S * C::kBufBytes);
    uint16_t* s_map16 = reinterpret_cast<uint16_t*>(smem + S * (C::kBufBytes + C::kNdBytes));
    __shared__ uint32_t s_wcnt[W][kRadix];  // per-warp digit counts, then tile-local slot starts
    // destination of slot 0 of each digit, relative to the segment start (segments hold < 2^32 records)
    __shared__ uint32_t s_gdelta[kRadix];
    __shared__ unsigned long long s_pdst[kPeer ? kRadix : 1];  // digit's destination - its base
    __shared__ uint32_t s_scan[8];
    __shared__ __align__(8) unsigned long long s_full[C::kStages], s_empty[C::kStages];
    __shared__ TileInfo s_info[C::kStages];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&s_full[q], 1);
            mbar_init(&s_empty[q], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == W) {  // ------------------------------------------------ producer
        if (lane != 0) return;
        // Tiles are claimed in order through a global ticket, so all CTAs work
        // on a narrow window of consecutive tiles: the bucket frontiers each
        // tile writes stay few and L2-resident until neighbouring tiles
        // complete their lines (a static round-robin lets 296 persistent CTAs
        // drift thousands of tiles apart on 2^32-record inputs, and the
        // half-written lines that get evicted cost read-modify-write traffic).
        uint32_t it = 0;
        while (true) {
            const uint32_t tile = atomicAdd(ticket, 1u);
            Seg g;
            uint32_t s = 0;
            if (tile < n_tiles) {
                s = tile_seg[tile];
                g = segs[s];
                if (g.action != kActScatter) continue;  // constant byte / finished: not split
            }
            const int b = it % S;
            if (it >= uint32_t(S)) mbar_wait(&s_empty[b], ((it / S) - 1) & 1u);
            ++it;
            TileInfo ti;
            ti.tile = tile;
            if (tile >= n_tiles) {
                s_info[b] = ti;
                mbar_arrive_expect_tx(&s_full[b], 0);
                return;
            }
            ti.seg = s;
            ti.k = uint64_t(tile) - g.tile_base;
            ti.seg_start = g.start;
            ti.seg_size = g.size;
            ti.gstart = g.start + ti.k * C::kTile;
            ti.tn = uint32_t(min(uint64_t(C::kTile), g.size - ti.k * C::kTile));
            ti.p = g.p;
            ti.parity = g.parity;
            const uint8_t* gsrc = (g.parity ? tmp : data) + ti.gstart * RS;
            const uint32_t bytes = ti.tn * RS;
            const uint32_t head = uint32_t(reinterpret_cast<uintptr_t>(gsrc) & 15u);  // 0 or 8
            const uint32_t hb = head ? min(8u, bytes) : 0u;
            const uint32_t body = (bytes - hb) & ~15u;
            const uint32_t tail = bytes - hb - body;  // 0 or 8
            ti.head = head;
            uint8_t* sb = buf0 + b * C::kBufBytes + head;
            if (hb) *reinterpret_cast<uint2*>(sb) = *reinterpret_cast<const uint2*>(gsrc);
            if (tail)
                *reinterpret_cast<uint2*>(sb + hb + body) =
                    *reinterpret_cast<const uint2*>(gsrc + hb + body);
            uint32_t ndb = 0;
            uint64_t nda = 0;
            if (kU16 && nd_in) {  // the tile's digit bytes, 16-B aligned around [gstart, gstart + tn)
                nda = ti.gstart & ~uint64_t(15);
                ndb = uint32_t(((ti.gstart + ti.tn + 15) & ~uint64_t(15)) - nda);
                ti.ndh = uint32_t(ti.gstart - nda);
            }
            fence_proxy_async_smem();
            s_info[b] = ti;
            mbar_arrive_expect_tx(&s_full[b], body + ndb);
            if (body) tma_load_1d_h<RG_HINT_SC>(sb + hb, gsrc + hb, body, &s_full[b]);
            if (ndb) tma_load_1d(snd + b * C::kNdBytes, nd_in + nda, ndb, &s_full[b]);
        }
    }

    // ------------------------------------------------------------ consumers
    for (uint32_t it = 0;; ++it) {
        const int b = it % S;
#pragma unroll
        for (int q = 0; q < kRadix / 32; ++q) s_wcnt[warp][q * 32 + lane] = 0;
        mbar_wait(&s_full[b], (it / S) & 1u);
        const TileInfo ti = s_info[b];
        if (ti.tile >= n_tiles) break;
        // this thread's digit: base inside the segment + offset of the tile.
        // kEarly 1 (8-B records): issued now, consumed after the ranking, the
        // tile offset by cp.async into s_gdelta (free since the last tile's
        // write-out) so ptxas cannot sink the load past the named barriers.
        // Measured in one process, interleaved (scripts/ab_interleave.py):
        // C2 scatter -3%; at 16 B the same change costs +3-7% (C5 77.9 vs
        // 75.1 ms), so kEarly 0 loads and resolves them here.
        constexpr int kEarly = RS == 8 ? RG_SC_EARLY8 : RG_SC_EARLY16;
        const unsigned long long my_sb = seg_base[uint64_t(ti.seg) * kRadix + threadIdx.x];
        uint32_t my_toff = 0, big = 0;
        uint64_t my_se = 0;
        if constexpr (kEarly == 1) {
            cp_async4(&s_gdelta[threadIdx.x], tile_off + uint64_t(ti.tile) * kRadix + threadIdx.x);
            if (nd)
                my_se = threadIdx.x + 1 < kRadix ? seg_base[uint64_t(ti.seg) * kRadix + threadIdx.x + 1]
                                                 : ti.seg_size;
        } else {
            my_toff = tile_off[uint64_t(ti.tile) * kRadix + threadIdx.x];
            if (nd) {
                const uint64_t se = threadIdx.x + 1 < kRadix ? seg_base[uint64_t(ti.seg) * kRadix + threadIdx.x + 1]
                                                             : ti.seg_size;
                big = se - my_sb > cap_local ? (1u << 24) : 0u;
            }
        }
        const uint8_t* tile = buf0 + b * C::kBufBytes + ti.head;
        const uint32_t tn = ti.tn, p = ti.p;
        __syncwarp();

        // 1: stable rank inside the warp (warp_rank, common.cuh): items are
        // warp-striped in input order and the counters are per warp, so ranks
        // follow input order by construction (lane order inside one call from
        // popc(peers & lanemask_lt), not from the order atomics are served).
        uint32_t pk[IT];  // digit | rank << 9 ; 0x100 = invalid
        const uint8_t* sdig = snd + b * C::kNdBytes + ti.ndh;
        const bool dig_nd = kU16 && nd_in != nullptr;
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t i = uint32_t(warp * IT + j) * 32u + lane;
            const bool valid = i < tn;
            uint32_t d = 0;
            if (valid) d = dig_nd ? uint32_t(sdig[i]) : scatter_digit_smem<RS, kMap>(tile + size_t(i) * RS, p, ks, map);
            const uint32_t rk = warp_rank<kRank>(&s_wcnt[warp][0], d, valid);  // every lane calls it
            pk[j] = valid ? (d | (rk << 9)) : 0x100u;
        }
        bar_sync_named(1, T);

        // 2: per-digit tile totals, warp-exclusive offsets, tile-local starts
        if constexpr (kEarly != 0) big = (nd && my_se - my_sb > cap_local) ? (1u << 24) : 0u;
        uint32_t tcount = 0, wc[W];
        {
            const int d = threadIdx.x;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                wc[w] = s_wcnt[w][d];
                tcount += wc[w];
            }
        }
        uint32_t total;
        const uint32_t lstart = scan256_exclusive(tcount, s_scan, &total);
        {  // warp w's first slot of digit d; bit 24: the digit's child is split
           // next level, so its records' next key byte goes to nd
            const int d = threadIdx.x;
            uint32_t run = lstart;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                s_wcnt[w][d] = run | big;
                run += wc[w];
            }
        }
        if constexpr (kEarly == 1) {
            cp_async_wait_all();  // this thread's own element
            my_toff = s_gdelta[threadIdx.x];
        }
        s_gdelta[threadIdx.x] = uint32_t(my_sb) + my_toff - lstart;
        if constexpr (kPeer) {
            const unsigned long long dd = dig_dst[threadIdx.x];
            // split digit: flag | first piece << 32 | the digit's base in the segment
            s_pdst[threadIdx.x] = (dd >> 63) ? ((dd & 0xFFFFFFFF00000000ull) | uint32_t(my_sb))
                                             : dd - (ti.seg_start + my_sb) * RS;
        }
        bar_sync_named(1, T);

        // 3: slot map (digit order) in shared memory
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t d = pk[j] & 0x1FFu;
            if (d < 256u) {
                const uint32_t sw = s_wcnt[warp][d] + (pk[j] >> 9);
                const uint32_t idx = uint32_t(warp * IT + j) * 32u + lane;
                if constexpr (kU16) s_map16[sw & 0xFFFFFFu] = uint16_t(idx | ((sw >> 9) & 0x8000u));
                else s_map[sw & 0xFFFFFFu] = idx | (d << 16) | (sw & (1u << 24));
            }
        }
        bar_sync_named(1, T);

        // 4: write-out in digit order: consecutive slots of a digit go to
        // consecutive destinations (coalesced vector stores)
        uint8_t* dst = (ti.parity ? data : tmp) + ti.seg_start * RS;
#pragma unroll kScUnroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t slot = uint32_t(j) * T + threadIdx.x;
            if (slot < tn) {
                uint32_t m, d;
                Rec<RS> v;
                if constexpr (kU16) {
                    const uint32_t m16 = s_map16[slot];
                    v = ld_smem_rec<RS>(tile, m16 & 0x7FFFu);
                    d = rec_byte<RS>(v, p);
                    m = m16 << 9;  // nd flag -> bit 24
                } else {
                    m = s_map[slot];
                    v = ld_smem_rec<RS>(tile, m & 0xFFFFu);
                    d = (m >> 16) & 0xFFu;
                }
                if constexpr (kPeer) {
                    const unsigned long long pd = s_pdst[d];
                    const uint32_t di = s_gdelta[d] + slot;
                    if (!(pd >> 63)) {
                        store_rec<RS>(reinterpret_cast<uint8_t*>(pd + ti.seg_start * RS), di, v);
                    } else {  // a digit split over several destinations (rare)
                        const uint32_t idx = di - uint32_t(pd);
                        const Piece* pc = pieces + ((pd >> 32) & 0x7FFFFFFFu);
                        while (idx >= pc->end) ++pc;
                        store_rec<RS>(reinterpret_cast<uint8_t*>(pc->adj), idx, v);
                    }
                } else {
                    const uint32_t di = s_gdelta[d] + slot;
                    store_rec_h<RS, RG_HINT_SCST>(dst, di, v);
                    if (m >> 24) {
                        if constexpr (RG_HINT_NDST == 0) {
                            RG_CHK_G(nd + ti.seg_start + di, 1, kChkDigitStore),
                            nd[ti.seg_start + di] = uint8_t(rec_byte<RS>(v, p + 1));
                        } else {
                            uint64_t pol;
                            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                            asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(nd + ti.seg_start + di),
                                         "r"(rec_byte<RS>(v, p + 1)), "l"(pol)
                                         : "memory");
                        }
                    }
                }
            }
        }
        bar_sync_named(1, T);  // buffer b, map and counters free for reuse
        if (threadIdx.x == 0) mbar_arrive(&s_empty[b]);
    }
}

}  // namespace rg
