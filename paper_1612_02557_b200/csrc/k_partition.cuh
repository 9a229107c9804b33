// Multi-GPU key-range partition helpers (no reference
// counterpart — the reference is single-address-space). A rank holds N/G
// records; the 16-bit big-endian key prefix at bytes (pb, pb+1) selects a
// bucket, a host-built map assigns contiguous bucket ranges to ranks, and the
// records are split stably into G contiguous send ranges by k_tile_hist /
// k_tile_scan / k_scatter with kMap = true (the same passes as an MSD level).
#pragma once

#include "common.cuh"

namespace rg {

template <int RS>
__device__ __forceinline__ uint32_t prefix16(const Rec<RS>& r, uint32_t pb, uint32_t ks) {
    const uint32_t hi = pb < ks ? rec_byte<RS>(r, pb) : 0u;
    const uint32_t lo = pb + 1 < ks ? rec_byte<RS>(r, pb + 1) : 0u;
    return (hi << 8) | lo;
}

// 65536-bucket prefix histogram, accumulated into hist (u64). Warp-aggregated
// global atomics (a hot bucket costs one atomic per warp, not per record).
template <int RS>
__global__ void __launch_bounds__(256) k_prefix_hist(const uint8_t* __restrict__ data, uint64_t n,
                                                     uint32_t ks, uint32_t pb,
                                                     unsigned long long* __restrict__ hist) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
        const uint64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const uint32_t b = valid ? prefix16<RS>(load_rec_stream<RS>(data, i), pb, ks) : 0x10000u;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
        if (valid && (threadIdx.x & 31) == uint32_t(__ffs(peers) - 1))
            atomicAdd(&hist[b], (unsigned long long)__popc(peers));
    }
}

// k_prefix_hist over a strided sample of `samples` records (record
// min(n - 1, s * stride)): the multi-GPU plan's bucket map only needs to be
// balanced, not exact (the exact per-rank counts come from the partition's
// own tile histogram).
template <int RS>
__global__ void __launch_bounds__(256) k_sample_prefix_hist(const uint8_t* __restrict__ data, uint64_t n,
                                                            uint64_t stride, uint32_t samples, uint32_t ks,
                                                            uint32_t pb, unsigned long long* __restrict__ hist) {
    for (uint32_t base = blockIdx.x * blockDim.x; base < samples; base += gridDim.x * blockDim.x) {
        const uint32_t s = base + threadIdx.x;
        const bool valid = s < samples;
        const uint32_t b = valid ? prefix16<RS>(load_rec<RS>(data, min(n - 1, uint64_t(s) * stride)), pb, ks)
                                 : 0x10000u;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
        if (valid && (threadIdx.x & 31) == uint32_t(__ffs(peers) - 1))
            atomicAdd(&hist[b], (unsigned long long)__popc(peers));
    }
}

// AND/OR of the key words (64-bit words holding key bytes) of the records
// whose bucket maps to a flagged digit: hot[d] = slot + 1 (<= kHotSlots), 0 =
// not flagged. out[slot][8]: and at 2w, or at 2w+1 (words w >= ceil(ks/8)
// untouched). The multi-GPU plan uses it to prove that a hot bucket holds a
// single key before spreading it over ranks by count.
constexpr int kHotSlots = 32;

template <int RS>
__global__ void __launch_bounds__(256) k_digit_andor(const uint8_t* __restrict__ data, uint64_t n, uint32_t ks,
                                                     uint32_t pb, const uint8_t* __restrict__ map,
                                                     const uint8_t* __restrict__ hot,
                                                     unsigned long long* __restrict__ out) {
    constexpr int KW = RS / 8;
    __shared__ uint8_t s_hot[256];
    __shared__ unsigned long long s_a[kHotSlots][KW], s_o[kHotSlots][KW];
    s_hot[threadIdx.x] = hot[threadIdx.x];
    for (uint32_t i = threadIdx.x; i < kHotSlots * KW; i += blockDim.x) {
        (&s_a[0][0])[i] = ~0ull;
        (&s_o[0][0])[i] = 0ull;
    }
    __syncthreads();
    const uint32_t kw = (ks + 7) / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    // thread-private accumulators for the last hot slot seen (a hot key makes
    // most records land in one slot: no shared-memory atomic per record)
    uint32_t cur = 0;
    unsigned long long a[KW], o[KW];
    auto flush = [&] {
        if (!cur) return;
#pragma unroll
        for (int w = 0; w < KW; ++w)
            if (uint32_t(w) < kw) {
                atomicAnd(&s_a[cur - 1][w], a[w]);
                atomicOr(&s_o[cur - 1][w], o[w]);
            }
    };
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const Rec<RS> r = load_rec_stream<RS>(data, i);
        const uint32_t h = s_hot[map_digit([&](uint32_t b) { return rec_byte<RS>(r, b); }, pb, ks, map)];
        if (!h) continue;
        if (h != cur) {
            flush();
            cur = h;
#pragma unroll
            for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
        }
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            a[w] &= rec_word64<RS>(r, w);
            o[w] |= rec_word64<RS>(r, w);
        }
    }
    flush();
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kHotSlots * KW; i += blockDim.x) {
        const uint32_t h = i / KW, w = i % KW;
        if (w < kw && (&s_o[0][0])[i] != 0ull) atomicOr(&out[h * 8 + 2 * w + 1], (&s_o[0][0])[i]);
        if (w < kw && (&s_a[0][0])[i] != ~0ull) atomicAnd(&out[h * 8 + 2 * w], (&s_a[0][0])[i]);
    }
}

__global__ void k_map_to_u8(const uint32_t* __restrict__ in, uint8_t* __restrict__ out,
                            uint32_t n_ranks, unsigned int* __restrict__ bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 65536) {
        const uint32_t r = in[i];
        if (r >= n_ranks) atomicOr(bad, 1u);
        out[i] = uint8_t(r < n_ranks ? r : 0);
    }
}

}  // namespace rg
