// (d) segmented small-bin sort for the MSD tail.
//
// Reference: the tiny-bin comparison sorts (P/include/raduls/small_sorts.hpp:
// 48-191: insertion / Shell {8,1} / introsort, chosen by TinyPolicy :14-45),
// the plain radix_split used for bins that fit half of L2 (kernels.hpp:157-167
// via msd_sorter.hpp:188-196) and finalize()'s copy back to the caller's buffer
// (msd_sorter.hpp:76-80).
//
// B200 design: one 1024-thread CTA sorts a *group* — one or more adjacent
// complete segments (bins) of at most kCap records, all sharing key bytes
// [0, p). Sorting the group by key bytes [p, ks) equals sorting each bin on its
// own, because the bins are contiguous and already in key order.
//   1. every record of the group is loaded once (coalesced) and stays in
//      registers until the end, so the sort is safe in place (source ==
//      destination buffer);
//   2. AND/OR of the key words over the group gives the varying key bytes
//      L = l0 < l1 < ... in [p, ks); the first <= 4 are packed big-endian into
//      a 32-bit window w per record (shared memory);
//   3. fast path — one counting pass: ~n buckets spread linearly over the
//      group's window range [min w, max w] (so buckets hold ~1 record for
//      uniformly distributed bytes), shared-memory histogram, scan,
//      scatter of record ids into bucket order; then every record ranks itself
//      inside its bucket by (w, remaining key bytes, input index). That is a
//      comparison sort of ~1-2 records per bucket — the GPU counterpart of the
//      reference's radix split followed by insertion sort of tiny bins;
//   4. robust path, when a bucket would hold more than kMaxBucket records
//      (duplicate-heavy or adversarial keys): stable LSD passes over the
//      window bytes (ballot multisplit ranking), then over the bytes beyond
//      the window if adjacent records still tie;
//   5. each thread stores its own records at their final positions.
// Every path orders equal keys by input index, so the whole MSD sort is
// stable: its output equals a stable sort by key, and for distinct keys it is
// byte-identical to the reference's (unstable) MSD output.
#pragma once

#include "common.cuh"

namespace rg {

template <int RS>
struct LocalCfg {
    static constexpr int kThreads = 1024;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kIpt = RS == 8 ? 20 : RS == 16 ? 10 : RS == 24 ? 7 : 5;
    static constexpr int kCap = kThreads * kIpt;  // records per group (C_local)
    static constexpr int kBucketBits = RS == 8 ? 14 : RS == 16 ? 14 : 13;
    static constexpr int kCntBytes =
        (1 << kBucketBits) * 2 > kWarps * kRadix * 4 ? (1 << kBucketBits) * 2 : kWarps * kRadix * 4;
    static constexpr size_t kSmem = size_t(kCap) * (4 + 2 + 2) + size_t(kCntBytes);
};

constexpr uint32_t kMaxBucket = 32;

// Block-wide exclusive scan of one u32 per thread (blockDim 1024).
__device__ __forceinline__ uint32_t block_scan_excl_1024(uint32_t v, uint32_t* s_w,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_w[lane];
        uint32_t z = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, z, off);
            if (lane >= off) z += y;
        }
        s_w[32 + lane] = z - w;
        if (lane == 31) s_w[64] = z;
    }
    __syncthreads();
    const uint32_t r = s_w[32 + warp] + x - v;
    *total = s_w[64];
    __syncthreads();
    return r;
}

// One stable LSD pass: pout <- pin ordered by digit(pin[pos]). Positions are
// split into 32 contiguous warp chunks (multiples of 32) processed in order;
// ranking by ballot multisplit with warp-private counters (digit-major,
// warp-minor offsets keep it stable).
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
            const uint32_t d = valid ? digit_of(e) : 0u;
            const uint32_t peers = match_digit8(d, valid);
            const uint32_t before = valid ? my[d] : 0u;
            __syncwarp();
            if (valid && uint32_t(lane) == 31u - __clz(peers)) my[d] = before + __popc(peers);
            __syncwarp();
            if (valid) pk[s] = d | ((before + __popc(peers & lt)) << 8);
        }
    }
    __syncthreads();
    // digit-major, warp-minor exclusive offsets: thread t -> digit t>>2, warps (t&3)*8..+7
    {
        const uint32_t d = threadIdx.x >> 2, q = threadIdx.x & 3;
        uint32_t part = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) part += wcnt[(q * 8 + w) * kRadix + d];
        uint32_t x = part;
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, 1, 4);
        if (q >= 1) x += y;
        y = __shfl_up_sync(0xFFFFFFFFu, x, 2, 4);
        if (q >= 2) x += y;
        const uint32_t qexcl = x - part;
        if (q == 3) s_tot[d] = x;
        __syncthreads();
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

// Key byte `b` of group record `e`, read from global memory (L2-resident: the
// group was just loaded).
template <int RS>
__device__ __forceinline__ uint32_t gbyte(const uint8_t* src, uint32_t e, uint32_t b) {
    return src[size_t(e) * RS + b];
}

// -1/0/+1: compare records a, b of the group on the varying key bytes beyond
// the window (L[4..nL)).
template <int RS>
__device__ __forceinline__ int cmp_beyond(const uint8_t* src, uint32_t a, uint32_t b,
                                          const uint32_t* L, uint32_t nL) {
    for (uint32_t q = 4; q < nL; ++q) {
        const uint32_t x = gbyte<RS>(src, a, L[q]), y = gbyte<RS>(src, b, L[q]);
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

// kFallback = false: the fast path; a group whose buckets overflow kMaxBucket
// is appended to `spill` untouched (nothing written) and sorted later by the
// kFallback = true instance (stable LSD only), launched once per sort on the
// collected list. Keeping the LSD code out of the fast kernel keeps the
// group's records in registers without spilling.
template <int RS, bool kFallback>
__global__ void __launch_bounds__(1024, 1) k_local_sort(uint8_t* __restrict__ data,
                                                        uint8_t* __restrict__ tmp,
                                                        const Group* __restrict__ groups,
                                                        uint32_t ks,
                                                        LevelCounters* __restrict__ ctr,
                                                        Group* __restrict__ spill,
                                                        unsigned int* __restrict__ n_spill,
                                                        uint32_t spill_cap) {
    using C = LocalCfg<RS>;
    constexpr int T = C::kThreads, IPT = C::kIpt;
    constexpr int KW = RS / 8;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* win = reinterpret_cast<uint32_t*>(smem);              // [cap]
    uint16_t* slot = reinterpret_cast<uint16_t*>(win + C::kCap);    // [cap]  (LSD: pa)
    uint16_t* fpos = slot + C::kCap;                                // [cap]  (LSD: pb)
    uint32_t* cnt = reinterpret_cast<uint32_t*>(fpos + C::kCap);    // packed u16 pairs / LSD wcnt
    __shared__ uint32_t s_tot[512];
    __shared__ unsigned long long s_and[32][KW], s_or[32][KW];
    __shared__ uint32_t s_L[32];
    __shared__ uint32_t s_nL, s_flag, s_maxb, s_wmin, s_wmax;
    __shared__ uint32_t s_scan[65];

    const Group g = groups[blockIdx.x];
    const uint32_t n = g.size;
    const uint8_t* src = (g.parity ? tmp : data) + g.start * RS;
    uint8_t* dst = data + g.start * RS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (n <= 1) {  // a single record: move home if it lives in tmp
        if (n == 1 && g.parity && threadIdx.x == 0) store_rec<RS>(dst, 0, load_rec<RS>(src, 0));
        return;
    }

    // 1. load the group into registers; AND/OR of every record word
    Rec<RS> r[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t e = uint32_t(j) * T + threadIdx.x;
        if (e < n) r[j] = load_rec_stream<RS>(src, e);
    }
    {
        uint64_t a[KW], o[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T + threadIdx.x < n) {
#pragma unroll
                for (int w = 0; w < KW; ++w) {
                    const uint64_t v = rec_word64<RS>(r[j], w);
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
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: varying key bytes in [p, ks)
        uint32_t diffb = 0;  // lane b: byte b varies
        {
            const uint32_t b = lane;
            if (b >= g.p && b < ks && b < uint32_t(RS)) {
                unsigned long long ra = ~0ull, ro = 0ull;
                for (int q = 0; q < 32; ++q) {
                    unsigned long long xa = s_and[q][0], xo = s_or[q][0];
#pragma unroll
                    for (int w = 1; w < KW; ++w)
                        if ((b >> 3) == uint32_t(w)) xa = s_and[q][w], xo = s_or[q][w];
                    ra &= xa;
                    ro |= xo;
                }
                diffb = uint32_t(((ra ^ ro) >> ((b & 7) * 8)) & 0xFF);
            }
        }
        const uint32_t vm = __ballot_sync(0xFFFFFFFFu, diffb != 0);
        if (diffb) s_L[__popc(vm & lanemask_lt())] = lane;
        if (lane == 0) {
            s_wmin = 0xFFFFFFFFu;
            s_wmax = 0u;
            s_nL = __popc(vm);
            s_flag = 0;
            s_maxb = 0;
        }
    }
    __syncthreads();
    const uint32_t nL = s_nL;
    if (nL == 0) {  // every key equal: stable order is the input order
        if (g.parity) {
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                if (e < n) store_rec<RS>(dst, e, r[j]);
            }
        }
        return;
    }
    const uint32_t nwin = nL < 4 ? nL : 4;

    // 2. 32-bit windows
    {
        const uint32_t L0 = s_L[0], L1 = s_L[nwin > 1 ? 1 : 0], L2 = s_L[nwin > 2 ? 2 : 0],
                       L3 = s_L[nwin > 3 ? 3 : 0];
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) {
                uint32_t wv = rec_byte<RS>(r[j], L0) << 24;
                if (nwin > 1) wv |= rec_byte<RS>(r[j], L1) << 16;
                if (nwin > 2) wv |= rec_byte<RS>(r[j], L2) << 8;
                if (nwin > 3) wv |= rec_byte<RS>(r[j], L3);
                win[e] = wv;
            }
        }
    }
    // bucket geometry: nbk ~ n buckets spread linearly over the window range
    // [wmin, wmax] of the group (block min/max), so uniformly distributed key
    // bytes give ~1 record per bucket whatever the group's digit span.
    {
        uint32_t mn = 0xFFFFFFFFu, mx = 0u;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) {
                const uint32_t w = win[e];
                mn = min(mn, w);
                mx = max(mx, w);
            }
        }
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0) {
            atomicMin(&s_wmin, mn);
            atomicMax(&s_wmax, mx);
        }
    }
    uint32_t B = 32u - __clz(n - 1);  // ceil(log2 n)
    B = B < 1 ? 1 : (B > uint32_t(C::kBucketBits) ? uint32_t(C::kBucketBits) : B);
    const uint32_t nbk = 1u << B;
    const bool beyond = nL > 4;
    // 3a. bucket histogram (packed u16 pairs)
    for (uint32_t i = threadIdx.x; i < nbk / 2; i += T) cnt[i] = 0;
    __syncthreads();
    const uint32_t wmin = s_wmin;
    const uint32_t range = s_wmax - wmin;
    // bucket(w) = floor((w - wmin) * nbk / (range + 1)), monotone in w, < nbk
    const bool exact = uint64_t(range) + 1 <= nbk;
    const unsigned long long mul =
        exact ? 0ull : (((unsigned long long)nbk << 32) / (uint64_t(range) + 1));
    auto bucket_of = [&](uint32_t w) -> uint32_t {
        const uint32_t d = w - wmin;
        return exact ? d : uint32_t((uint64_t(d) * mul) >> 32);
    };
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t e = uint32_t(j) * T + threadIdx.x;
        if (e < n) {
            const uint32_t b = bucket_of(win[e]);
            atomicAdd(&cnt[b >> 1], 1u << ((b & 1) * 16));
        }
    }
    __syncthreads();
    // 3b. exclusive scan over nbk buckets; each thread owns a contiguous run
    {
        const uint32_t per = nbk > uint32_t(T) ? nbk / T : 1u;  // buckets per thread (even or 1)
        const uint32_t b0 = threadIdx.x * per;
        uint32_t sum = 0, mx = 0;
        if (b0 < nbk) {
            for (uint32_t b = b0; b < b0 + per; ++b) {
                const uint32_t c = (cnt[b >> 1] >> ((b & 1) * 16)) & 0xFFFFu;
                sum += c;
                mx = c > mx ? c : mx;
            }
        }
        uint32_t total;
        uint32_t run = block_scan_excl_1024(sum, s_scan, &total);
        // max bucket
        for (int off = 16; off; off >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
        if (lane == 0 && mx) atomicMax(&s_maxb, mx);
        if (b0 < nbk) {
            for (uint32_t b = b0; b < b0 + per; b += (per >= 2 ? 2 : 1)) {
                if (per >= 2) {
                    const uint32_t w = cnt[b >> 1];
                    const uint32_t c0 = w & 0xFFFFu, c1 = w >> 16;
                    cnt[b >> 1] = run | ((run + c0) << 16);
                    run += c0 + c1;
                } else {
                    // per == 1 (nbk <= 1024): owner of the even bucket rewrites the pair
                    const uint32_t w = cnt[b >> 1];
                    if ((b & 1) == 0) {
                        const uint32_t c0 = w & 0xFFFFu;
                        cnt[b >> 1] = run | ((run + c0) << 16);
                    }
                }
            }
        }
    }
    __syncthreads();
    const bool fast = !kFallback && s_maxb <= kMaxBucket;
    if (!kFallback && !fast) {  // hand the untouched group to the LSD instance
        if (threadIdx.x == 0) {
            const uint32_t i = atomicAdd(n_spill, 1u);
            if (i < spill_cap) spill[i] = g;
            atomicAdd(&ctr->fallback_groups, 1ull);
        }
        return;
    }

    if (fast) {
        // 3c. scatter record ids into bucket order (cursor = packed start)
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) {
                const uint32_t b = bucket_of(win[e]);
                const uint32_t old = atomicAdd(&cnt[b >> 1], 1u << ((b & 1) * 16));
                slot[(old >> ((b & 1) * 16)) & 0xFFFFu] = uint16_t(e);
            }
        }
        __syncthreads();
        // 3d. order inside each bucket: cnt now holds bucket ends. Thread t
        // owns the contiguous bucket run [b0, b0+per): work ~ sum(size^2),
        // no divergence on the largest bucket of a warp.
        {
            const uint32_t per = nbk > uint32_t(T) ? nbk / T : 1u;
            const uint32_t b0 = threadIdx.x * per;
            if (b0 < nbk) {
                auto end_of = [&](uint32_t b) { return (cnt[b >> 1] >> ((b & 1) * 16)) & 0xFFFFu; };
                uint32_t st = b0 ? end_of(b0 - 1) : 0u;
                for (uint32_t b = b0; b < b0 + per; ++b) {
                    const uint32_t en = end_of(b);
                    if (en - st == 1) {
                        fpos[slot[st]] = uint16_t(st);
                    } else if (en > st) {
                        for (uint32_t q = st; q < en; ++q) {
                            const uint32_t e = slot[q];
                            const uint32_t w = win[e];
                            uint32_t rank = 0;
                            for (uint32_t q2 = st; q2 < en; ++q2) {
                                const uint32_t e2 = slot[q2];
                                const uint32_t w2 = win[e2];
                                bool less = w2 < w;
                                if (w2 == w && e2 != e) {
                                    const int c = beyond ? cmp_beyond<RS>(src, e2, e, s_L, nL) : 0;
                                    less = c < 0 || (c == 0 && e2 < e);
                                }
                                rank += less;
                            }
                            fpos[e] = uint16_t(st + rank);
                        }
                    }
                    st = en;
                }
            }
        }
        __syncthreads();
    } else if constexpr (kFallback) {
        // 4. robust stable LSD over the window bytes, then beyond if needed
        uint16_t *pin = slot, *pout = fpos;
        bool first = true;
        for (int q = int(nwin) - 1; q >= 0; --q) {
            const uint32_t sh = 24u - 8u * uint32_t(q);
            auto dig = [&](uint32_t e) { return (win[e] >> sh) & 0xFFu; };
            if (first)
                lsd_pass<IPT, true>(n, pin, pout, cnt, s_tot, dig);
            else
                lsd_pass<IPT, false>(n, pin, pout, cnt, s_tot, dig);
            first = false;
            uint16_t* t = pin;
            pin = pout;
            pout = t;
        }
        if (beyond) {
            for (uint32_t pos = threadIdx.x + 1; pos < n; pos += T) {
                const uint32_t ea = pin[pos - 1], eb = pin[pos];
                if (win[ea] == win[eb] && cmp_beyond<RS>(src, ea, eb, s_L, nL) > 0) s_flag = 1;
            }
            __syncthreads();
            if (s_flag) {  // full stable LSD over every varying byte
                first = true;
                for (int q = int(nL) - 1; q >= 0; --q) {
                    const uint32_t b = s_L[q];
                    if (q >= 4) {
                        auto dig = [&](uint32_t e) { return gbyte<RS>(src, e, b); };
                        if (first)
                            lsd_pass<IPT, true>(n, pin, pout, cnt, s_tot, dig);
                        else
                            lsd_pass<IPT, false>(n, pin, pout, cnt, s_tot, dig);
                    } else {
                        const uint32_t sh = 24u - 8u * uint32_t(q);
                        auto dig = [&](uint32_t e) { return (win[e] >> sh) & 0xFFu; };
                        if (first)
                            lsd_pass<IPT, true>(n, pin, pout, cnt, s_tot, dig);
                        else
                            lsd_pass<IPT, false>(n, pin, pout, cnt, s_tot, dig);
                    }
                    first = false;
                    uint16_t* t = pin;
                    pin = pout;
                    pout = t;
                }
            }
        }
        // inverse permutation into pout (e -> final position)
        for (uint32_t pos = threadIdx.x; pos < n; pos += T) pout[pin[pos]] = uint16_t(pos);
        __syncthreads();
        fpos = pout;
    }

    // 5. every record to its final position (all reads of src are done)
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t e = uint32_t(j) * T + threadIdx.x;
        if (e < n) store_rec<RS>(dst, fpos[e], r[j]);
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
