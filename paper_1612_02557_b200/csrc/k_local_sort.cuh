// (d) segmented small-bin sort for the MSD tail.
//
// Reference: the tiny-bin comparison sorts (P/include/raduls/small_sorts.hpp:
// 48-191: insertion / Shell {8,1} / introsort, chosen by TinyPolicy :14-45),
// the plain radix_split used for bins that fit half of L2 (kernels.hpp:157-167
// via msd_sorter.hpp:188-196) and finalize()'s copy back to the caller's buffer
// (msd_sorter.hpp:76-80).
//
// B200 design: one 1024-thread CTA sorts a *group* — one or more adjacent
// complete segments (bins) of at most kCap records in total, all sharing key
// bytes [0, p). Sorting the group by key bytes [p, ks) equals sorting each bin
// on its own, because the bins are contiguous and already in key order.
//   1. coalesced load of the group; AND/OR of the key words over the group
//      gives the non-constant key bytes L = l0 < l1 < ... in [p, ks);
//   2. the first <= 4 of them are packed big-endian into a 32-bit window per
//      record, kept in shared memory;
//   3. stable LSD passes (warp multisplit with __match_any_sync, per-warp
//      counters, digit-major/warp-minor offsets) over the window bytes sort a
//      16-bit permutation in shared memory;
//   4. if more than four key bytes vary, adjacent records that tie on the window
//      are compared on the remaining bytes; any inversion sends the group through
//      a full stable LSD over every byte of L (rare on real keys, always correct);
//   5. records are gathered in sorted order (the group was just read, so this hits
//      L2), held in registers until the whole group is read, then written with
//      coalesced vector stores straight into the caller's buffer — no separate
//      copy-back pass, and safe when source and destination are the same buffer.
// The whole sort is stable (stable splits + stable local sort), so its output
// equals a stable sort by key; with distinct keys it is byte-identical to the
// reference's (unstable) MSD output.
#pragma once

#include "common.cuh"

namespace rg {

template <int RS>
struct LocalCfg {
    static constexpr int kThreads = 1024;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kIpt = RS == 8 ? 20 : RS == 16 ? 10 : RS == 24 ? 7 : 5;
    static constexpr int kCap = kThreads * kIpt;  // records per group (C_local)
    static constexpr size_t kSmem = size_t(kCap) * (4 + 2 + 2) + size_t(kWarps) * kRadix * 4 + 2048;
};

struct LocalShared {
    uint32_t* win;    // [cap]
    uint16_t* pa;     // [cap]
    uint16_t* pb;     // [cap]
    uint32_t* wcnt;   // [warps][256]
};

// One stable LSD pass: pout <- pin ordered by digit(pin[pos]). Positions are
// split into 32 contiguous warp chunks (multiples of 32) processed in order.
template <int IPT, bool kIdentity, typename DigitFn>
__device__ __forceinline__ void lsd_pass(uint32_t n, const uint16_t* pin, uint16_t* pout,
                                         uint32_t* wcnt, uint32_t* s_tot, DigitFn digit_of) {
    constexpr int W = 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t chunk = ((n + W * 32 - 1) / (W * 32)) * 32;  // per-warp positions
    const uint32_t steps = chunk / 32;
    uint32_t* my = wcnt + warp * kRadix;
#pragma unroll
    for (int q = 0; q < kRadix / 32; ++q) my[q * 32 + lane] = 0;
    __syncwarp();
    const uint32_t lt = lanemask_lt();
    uint32_t pk[IPT];
#pragma unroll
    for (int s = 0; s < IPT; ++s) {
        pk[s] = 0xFFFFFFFFu;
        if (uint32_t(s) < steps) {
            const uint32_t pos = warp * chunk + s * 32 + lane;
            const bool valid = pos < n;
            const uint32_t e = valid ? (kIdentity ? pos : uint32_t(pin[pos])) : 0u;
            const uint32_t d = valid ? digit_of(e) : 0x100u;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (lane == leader && valid) {
                old = my[d];
                my[d] = old + __popc(peers);
            }
            old = __shfl_sync(0xFFFFFFFFu, old, leader);
            __syncwarp();
            if (valid) pk[s] = d | ((old + __popc(peers & lt)) << 8);
        }
    }
    __syncthreads();
    // digit-major, warp-minor exclusive offsets: thread t -> digit t>>2, warps (t&3)*8..+7
    {
        const uint32_t d = threadIdx.x >> 2, q = threadIdx.x & 3;
        uint32_t part = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) part += wcnt[(q * 8 + w) * kRadix + d];
        // exclusive scan across the 4 quarter-threads of this digit (consecutive lanes)
        uint32_t x = part;
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, 1, 4);
        if (q >= 1) x += y;
        y = __shfl_up_sync(0xFFFFFFFFu, x, 2, 4);
        if (q >= 2) x += y;
        const uint32_t qexcl = x - part;
        if (q == 3) s_tot[d] = x;  // digit total
        __syncthreads();
        // warp 0: exclusive scan of the 256 digit totals (8 per lane)
        if (warp == 0) {
            uint32_t v[8], sum = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = s_tot[lane * 8 + i], sum += v[i];
            uint32_t xs = sum;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t z = __shfl_up_sync(0xFFFFFFFFu, xs, off);
                if (lane >= off) xs += z;
            }
            uint32_t run = xs - sum;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                s_tot[256 + lane * 8 + i] = run;
                run += v[i];
            }
        }
        __syncthreads();
        uint32_t run = s_tot[256 + d] + qexcl;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            uint32_t* c = &wcnt[(q * 8 + w) * kRadix + d];
            const uint32_t cnt = *c;
            *c = run;
            run += cnt;
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < IPT; ++s) {
        if (pk[s] != 0xFFFFFFFFu) {
            const uint32_t d = pk[s] & 0xFFu;
            const uint32_t pos = warp * chunk + s * 32 + lane;
            const uint32_t e = kIdentity ? pos : uint32_t(pin[pos]);
            pout[my[d] + (pk[s] >> 8)] = uint16_t(e);
        }
    }
    __syncthreads();
}

// Key byte `b` of record `e` of the group, read from global memory (fallback path).
template <int RS>
__device__ __forceinline__ uint32_t gbyte(const uint8_t* src, uint32_t e, uint32_t b) {
    return src[size_t(e) * RS + b];
}

template <int RS>
__global__ void __launch_bounds__(1024, 1) k_local_sort(uint8_t* __restrict__ data,
                                                        uint8_t* __restrict__ tmp,
                                                        const Group* __restrict__ groups,
                                                        uint32_t ks,
                                                        LevelCounters* __restrict__ ctr) {
    using C = LocalCfg<RS>;
    constexpr int T = C::kThreads, IPT = C::kIpt;
    constexpr int KW = RS / 8;
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* win = reinterpret_cast<uint32_t*>(smem);
    uint16_t* pa = reinterpret_cast<uint16_t*>(win + C::kCap);
    uint16_t* pb = pa + C::kCap;
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(pb + C::kCap);
    __shared__ uint32_t s_tot[512];
    __shared__ unsigned long long s_and[32][KW], s_or[32][KW];
    __shared__ uint32_t s_L[32];
    __shared__ uint32_t s_nL, s_flag;

    const Group g = groups[blockIdx.x];
    const uint32_t n = g.size;
    const uint8_t* src = (g.parity ? tmp : data) + g.start * RS;
    uint8_t* dst = data + g.start * RS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (n <= 1) {  // a single record: move home if it lives in tmp
        if (n == 1 && g.parity && threadIdx.x == 0) store_rec<RS>(dst, 0, load_rec<RS>(src, 0));
        return;
    }

    // 1. load keys, AND/OR reduce
    uint64_t a[KW], o[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t i = uint32_t(j) * T + threadIdx.x;
        if (i < n) {
            const Rec<RS> r = load_rec<RS>(src, i);
#pragma unroll
            for (int w = 0; w < KW; ++w) {
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
        if (lane == 0) s_and[warp][w] = a[w], s_or[warp][w] = o[w];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t diff[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            uint64_t ra = ~0ull, ro = 0ull;
            for (int q = 0; q < 32; ++q) ra &= s_and[q][w], ro |= s_or[q][w];
            diff[w] = ra ^ ro;
        }
        uint32_t nL = 0;
        for (uint32_t b = g.p; b < ks; ++b) {
            uint64_t dw = diff[0];
#pragma unroll
            for (int w = 1; w < KW; ++w) dw = (b >> 3) == uint32_t(w) ? diff[w] : dw;
            if ((dw >> ((b & 7) * 8)) & 0xFF) s_L[nL++] = b;
        }
        s_nL = nL;
        s_flag = 0;
    }
    __syncthreads();
    const uint32_t nL = s_nL;
    const uint32_t nwin = nL < 4 ? nL : 4;

    uint16_t* sorted = pa;  // identity when nL == 0
    if (nL > 0) {
        // 2. windows: bytes L[0..nwin) packed big-endian into the top of a u32
        const uint32_t L0 = s_L[0], L1 = s_L[nwin > 1 ? 1 : 0], L2 = s_L[nwin > 2 ? 2 : 0],
                       L3 = s_L[nwin > 3 ? 3 : 0];
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const uint32_t i = uint32_t(j) * T + threadIdx.x;
            if (i < n) {
                const Rec<RS> r = load_rec<RS>(src, i);  // L1/L2 hit: just loaded
                uint32_t wv = rec_byte<RS>(r, L0) << 24;
                if (nwin > 1) wv |= rec_byte<RS>(r, L1) << 16;
                if (nwin > 2) wv |= rec_byte<RS>(r, L2) << 8;
                if (nwin > 3) wv |= rec_byte<RS>(r, L3);
                win[i] = wv;
            }
        }
        __syncthreads();
        // 3. LSD over the window bytes, least significant first
        uint16_t *pin = pa, *pout = pb;
        bool first = true;
        for (int q = int(nwin) - 1; q >= 0; --q) {
            const uint32_t shift = 24u - 8u * uint32_t(q);
            auto dig = [&](uint32_t e) { return (win[e] >> shift) & 0xFFu; };
            if (first)
                lsd_pass<IPT, true>(n, pin, pout, wcnt, s_tot, dig);
            else
                lsd_pass<IPT, false>(n, pin, pout, wcnt, s_tot, dig);
            first = false;
            uint16_t* t = pin;
            pin = pout;
            pout = t;
        }
        sorted = pin;
        // 4. ties beyond the window
        if (nL > 4) {
            for (uint32_t pos = threadIdx.x + 1; pos < n; pos += T) {
                const uint32_t ea = sorted[pos - 1], eb = sorted[pos];
                if (win[ea] == win[eb]) {
                    for (uint32_t q = 4; q < nL; ++q) {
                        const uint32_t ba = gbyte<RS>(src, ea, s_L[q]);
                        const uint32_t bb = gbyte<RS>(src, eb, s_L[q]);
                        if (ba != bb) {
                            if (bb < ba) s_flag = 1;
                            break;
                        }
                    }
                }
            }
            __syncthreads();
            if (s_flag) {  // full stable LSD over every varying byte
                if (threadIdx.x == 0) atomicAdd(&ctr->fallback_groups, 1ull);
                pin = pa;
                pout = pb;
                first = true;
                for (int q = int(nL) - 1; q >= 0; --q) {
                    const uint32_t b = s_L[q];
                    if (q >= 4) {
                        auto dig = [&](uint32_t e) { return gbyte<RS>(src, e, b); };
                        if (first)
                            lsd_pass<IPT, true>(n, pin, pout, wcnt, s_tot, dig);
                        else
                            lsd_pass<IPT, false>(n, pin, pout, wcnt, s_tot, dig);
                    } else {
                        const uint32_t shift = 24u - 8u * uint32_t(q);
                        auto dig = [&](uint32_t e) { return (win[e] >> shift) & 0xFFu; };
                        if (first)
                            lsd_pass<IPT, true>(n, pin, pout, wcnt, s_tot, dig);
                        else
                            lsd_pass<IPT, false>(n, pin, pout, wcnt, s_tot, dig);
                    }
                    first = false;
                    uint16_t* t = pin;
                    pin = pout;
                    pout = t;
                }
                sorted = pin;
            }
        }
    } else if (!g.parity) {
        return;  // every key equal and already home: stable order == input order
    }

    // 5. gather in sorted order (all reads before any write), coalesced stores
    Rec<RS> out[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t pos = uint32_t(j) * T + threadIdx.x;
        if (pos < n) out[j] = load_rec<RS>(src, nL > 0 ? uint32_t(sorted[pos]) : pos);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t pos = uint32_t(j) * T + threadIdx.x;
        if (pos < n) store_rec<RS>(dst, pos, out[j]);
    }
    if (threadIdx.x == 0) atomicAdd(&ctr->moved_local, (unsigned long long)n);
}

// Finished records that ended in tmp move home (reference finalize(),
// msd_sorter.hpp:76-80). One CTA per range of <= kCopyTile records.
constexpr int kCopyTile = 8192;

template <int RS>
__global__ void __launch_bounds__(256) k_copy_back(uint8_t* __restrict__ data,
                                                   const uint8_t* __restrict__ tmp,
                                                   const CopyRange* __restrict__ ranges) {
    const CopyRange c = ranges[blockIdx.x];
    const uint64_t bytes = uint64_t(c.size) * RS;
    const uint8_t* s = tmp + c.start * RS;
    uint8_t* d = data + c.start * RS;
    if constexpr (RS % 16 == 0) {
        for (uint64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
    } else {
        for (uint64_t i = threadIdx.x; i < bytes / 8; i += blockDim.x)
            reinterpret_cast<uint2*>(d)[i] = reinterpret_cast<const uint2*>(s)[i];
    }
}

}  // namespace rg
