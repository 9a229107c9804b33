// (a) Digit histogramming in shared memory with warp-aggregated atomics, and
// (e) constant-digit detection.
//
// Reference: build_histogram (P/include/raduls/kernels.hpp:71-77) and the count
// loop of buffered_radix_split (kernels.hpp:212-218). The reference counts one
// digit per split; here one read of the whole array counts the first eight key
// bytes at once and reduces the bitwise AND / OR of every key word, so a key
// byte is constant over the array iff its AND byte equals its OR byte — the
// reference has no counterpart for that skip.
//
// Warp aggregation: each warp first reduces AND/OR of its 32 records' key word
// with REDUX (__reduce_and_sync/__reduce_or_sync). For a byte that is constant
// across the warp one lane adds the warp's count to the shared bin instead of
// 32 lanes colliding on the same shared-memory address (C3's three all-zero
// leading bytes would otherwise serialise every atomic 32 ways).
#pragma once

#include "common.cuh"

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

// Whole-array histograms of record bytes 0..nb-1 (nb = min(ks, 8)) plus the
// AND/OR of every 64-bit record word. hist: [8][256] u64, andor: [2*4] u64
// (and[w] at 2w, or[w] at 2w+1). Both must be initialised by the caller
// (hist 0, and ~0, or 0).
template <int RS>
__global__ void __launch_bounds__(256) k_histo_all(const uint8_t* __restrict__ data, uint64_t n,
                                                   uint32_t nb,
                                                   unsigned long long* __restrict__ hist,
                                                   unsigned long long* __restrict__ andor) {
    constexpr int KW = RS / 8;
    __shared__ uint32_t sh[8][kRadix];
    __shared__ unsigned long long s_and[8][KW], s_or[8][KW];
    for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();

    uint64_t a[KW], o[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;

    constexpr int U = 4;  // records in flight per thread
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
    for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x * U; base < n; base += stride) {
        Rec<RS> r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + uint64_t(u) * blockDim.x + threadIdx.x;
            if (i < n) {
                r[u] = load_rec_stream<RS>(data, i);
            } else {
#pragma unroll
                for (int k = 0; k < Rec<RS>::kWords; ++k) r[u].w[k] = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + uint64_t(u) * blockDim.x + threadIdx.x;
            const bool valid = i < n;
            const uint32_t nvalid = __popc(__ballot_sync(0xFFFFFFFFu, valid));
            const uint32_t lo = r[u].w[0], hi = r[u].w[1];
            const uint32_t al = __reduce_and_sync(0xFFFFFFFFu, valid ? lo : ~0u);
            const uint32_t ol = __reduce_or_sync(0xFFFFFFFFu, valid ? lo : 0u);
            const uint32_t ah = __reduce_and_sync(0xFFFFFFFFu, valid ? hi : ~0u);
            const uint32_t oh = __reduce_or_sync(0xFFFFFFFFu, valid ? hi : 0u);
            for (uint32_t b = 0; b < nb; ++b) {  // nb is uniform
                const uint32_t word = b < 4 ? lo : hi;
                const uint32_t sh_ = (b & 3u) * 8u;
                warp_hist_add(sh[b], (word >> sh_) & 0xFFu, valid, b < 4 ? al : ah,
                              b < 4 ? ol : oh, sh_, nvalid);
            }
            if (valid) {
#pragma unroll
                for (int w = 0; w < KW; ++w) {
                    const uint64_t v = rec_word64<RS>(r[u], w);
                    a[w] &= v;
                    o[w] |= v;
                }
            }
        }
    }
    // block reduce AND/OR
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
        for (int k = 0; k < int(blockDim.x >> 5); ++k) ra &= s_and[k][threadIdx.x], ro |= s_or[k][threadIdx.x];
        atomicAnd(&andor[2 * threadIdx.x], ra);
        atomicOr(&andor[2 * threadIdx.x + 1], ro);
    }
    for (uint32_t i = threadIdx.x; i < nb * kRadix; i += blockDim.x) {
        const uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(&hist[i], (unsigned long long)c);
    }
}

// Per-segment histogram of record byte segs[s].p, plus the AND/OR of every
// record word over the segment. One CTA per histogram tile of kHistTile
// records; tile -> segment through htile_seg. seg_hist: [nseg][256] u64,
// seg_andor: [nseg][8] u64 (and at 2w, or at 2w+1); both pre-initialised.
constexpr int kHistThreads = 256;
constexpr int kHistItems = 16;
constexpr int kHistTile = kHistThreads * kHistItems;

template <int RS>
__global__ void __launch_bounds__(kHistThreads) k_seg_hist(
    const uint8_t* __restrict__ data, const uint8_t* __restrict__ tmp, const Seg* __restrict__ segs,
    const uint32_t* __restrict__ htile_seg, unsigned long long* __restrict__ seg_hist,
    unsigned long long* __restrict__ seg_andor) {
    constexpr int KW = RS / 8;
    __shared__ uint32_t sh[kRadix];
    __shared__ unsigned long long s_and[kHistThreads / 32][KW], s_or[kHistThreads / 32][KW];
    sh[threadIdx.x] = 0;
    const uint32_t s = htile_seg[blockIdx.x];
    const Seg g = segs[s];
    const uint64_t k = uint64_t(blockIdx.x) - g.htile_base;
    const uint8_t* src = (g.parity ? tmp : data) + g.start * RS;
    const uint64_t t0 = k * kHistTile;
    const uint64_t tn = min(uint64_t(kHistTile), g.size - t0);
    const uint32_t p = g.p;
    __syncthreads();

    uint64_t a[KW], o[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
#pragma unroll 4
    for (int j = 0; j < kHistItems; ++j) {
        const uint64_t i = uint64_t(j) * kHistThreads + threadIdx.x;
        const bool valid = i < tn;
        Rec<RS> r;
        if (valid) {
            r = load_rec_stream<RS>(src, t0 + i);
        } else {
#pragma unroll
            for (int q = 0; q < Rec<RS>::kWords; ++q) r.w[q] = 0;
        }
        const uint32_t nvalid = __popc(__ballot_sync(0xFFFFFFFFu, valid));
        // word holding byte p (select chain, p uniform)
        uint32_t word = r.w[0];
#pragma unroll
        for (int q = 1; q < Rec<RS>::kWords; ++q) word = (p >> 2) == uint32_t(q) ? r.w[q] : word;
        const uint32_t wa = __reduce_and_sync(0xFFFFFFFFu, valid ? word : ~0u);
        const uint32_t wo = __reduce_or_sync(0xFFFFFFFFu, valid ? word : 0u);
        const uint32_t shf = (p & 3u) * 8u;
        warp_hist_add(sh, (word >> shf) & 0xFFu, valid, wa, wo, shf, nvalid);
        if (valid) {
#pragma unroll
            for (int w = 0; w < KW; ++w) {
                const uint64_t v = rec_word64<RS>(r, w);
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
        for (int q = 0; q < kHistThreads / 32; ++q) ra &= s_and[q][threadIdx.x], ro |= s_or[q][threadIdx.x];
        atomicAnd(&seg_andor[uint64_t(s) * 8 + 2 * threadIdx.x], ra);
        atomicOr(&seg_andor[uint64_t(s) * 8 + 2 * threadIdx.x + 1], ro);
    }
    const uint32_t c = sh[threadIdx.x];
    if (c) atomicAdd(&seg_hist[uint64_t(s) * kRadix + threadIdx.x], (unsigned long long)c);
}

}  // namespace rg
