// (d) segmented small-bin sort, shared-memory variant (record sizes 16/24/32).
//
// Same contract and algorithm as k_local_sort (k_local_sort.cuh; reference
// small_sorts.hpp:48-191, msd_sorter.hpp:76-80, 188-196), but the group's
// records live in shared memory instead of registers:
//   * one TMA bulk copy (cp.async.bulk, mbarrier transaction count) brings the
//     whole contiguous group on chip — no per-thread loads, no registers held;
//   * keys, windows, buckets and ranks are all computed from shared memory;
//   * the output loop walks final positions in order (coalesced vector
//     stores) and reads each record from its shared-memory slot, which is
//     in-place safe because the group is entirely on chip before any store.
// Low register and moderate shared-memory use let two CTAs share an SM
// (record size 16), so one group's HBM traffic overlaps another's sorting.
#pragma once

#include "common.cuh"
#include "k_local_sort.cuh"

namespace rg {

template <int RS>
struct LocalSmemCfg {
    static constexpr int kThreads = 512;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kCap = RS == 16 ? 3584 : RS == 24 ? 2560 : 4608;
    static constexpr int kIpt = (kCap + kThreads - 1) / kThreads;
    static constexpr int kBucketBits = 13;  // nbk <= 8192
    static constexpr int kCntBytes = 16384;  // max(8192 * 2, kWarps * 256 * 4)
    static constexpr int kRecBytes = ((kCap * RS + 16 + 127) / 128) * 128;
    static constexpr size_t kSmem = size_t(kRecBytes) + size_t(kCap) * (4 + 2 + 2) + kCntBytes;
    static_assert((1 << kBucketBits) * 2 <= kCntBytes && kWarps * kRadix * 4 <= kCntBytes, "cnt");
};

// Stable LSD pass for W warps (T = 32 W threads, T >= 256, T % 256 == 0).
template <int IPT, int W, bool kIdentity, typename DigitFn>
__device__ __forceinline__ void lsd_pass_w(uint32_t n, const uint16_t* pin, uint16_t* pout,
                                           uint32_t* wcnt, uint32_t* s_tot, DigitFn digit_of) {
    constexpr int T = W * 32;
    constexpr int TPD = T / 256;       // threads per digit in the offset scan
    constexpr int WPT = W / TPD;       // warps per such thread
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t chunk = ((n + T - 1) / T) * 32;  // per-warp positions
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
    {
        const uint32_t d = threadIdx.x / TPD, q = threadIdx.x % TPD;
        uint32_t part = 0;
#pragma unroll
        for (int w = 0; w < WPT; ++w) part += wcnt[(q * WPT + w) * kRadix + d];
        uint32_t x = part;
#pragma unroll
        for (int o = 1; o < TPD; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o, TPD);
            if (q >= uint32_t(o)) x += y;
        }
        const uint32_t qexcl = x - part;
        if (q == TPD - 1) s_tot[d] = x;
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
        for (int w = 0; w < WPT; ++w) {
            uint32_t* c = &wcnt[(q * WPT + w) * kRadix + d];
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

// Block-wide exclusive scan, any blockDim that is a multiple of 32 (<= 1024).
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* s_w, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < nw ? s_w[lane] : 0u;
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

template <int RS, bool kFallback>
__global__ void __launch_bounds__(512, 2) k_local_smem(uint8_t* __restrict__ data,
                                                       uint8_t* __restrict__ tmp,
                                                       const Group* __restrict__ groups, uint32_t ks,
                                                       LevelCounters* __restrict__ ctr,
                                                       Group* __restrict__ spill,
                                                       unsigned int* __restrict__ n_spill,
                                                       uint32_t spill_cap) {
    using C = LocalSmemCfg<RS>;
    constexpr int T = C::kThreads, W = C::kWarps, IPT = C::kIpt;
    constexpr int KW = RS / 8;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* recbuf = smem;
    uint32_t* win = reinterpret_cast<uint32_t*>(smem + C::kRecBytes);
    uint16_t* slot = reinterpret_cast<uint16_t*>(win + C::kCap);
    uint16_t* perm = slot + C::kCap;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(perm + C::kCap);
    __shared__ uint32_t s_tot[512];
    __shared__ uint32_t s_scan[65];
    __shared__ unsigned long long s_and[W][KW], s_or[W][KW];
    __shared__ uint32_t s_L[32];
    __shared__ uint32_t s_nL, s_flag, s_maxb, s_wmin, s_wmax;
    __shared__ __align__(8) unsigned long long s_bar;

    const Group g = groups[blockIdx.x];
    const uint32_t n = g.size;
    const uint8_t* gsrc = (g.parity ? tmp : data) + g.start * RS;
    uint8_t* dst = data + g.start * RS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (n <= 1) {
        if (n == 1 && g.parity && threadIdx.x == 0) store_rec<RS>(dst, 0, load_rec<RS>(gsrc, 0));
        return;
    }

    // 1. the whole group into shared memory with TMA (8-B edges by hand)
    const uint32_t head = uint32_t(reinterpret_cast<uintptr_t>(gsrc) & 15u);  // 0 or 8
    const uint8_t* recs = recbuf + head;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const uint32_t bytes = n * RS;
        const uint32_t hb = head ? min(8u, bytes) : 0u;
        const uint32_t body = (bytes - hb) & ~15u;
        const uint32_t tail = bytes - hb - body;
        if (hb) *reinterpret_cast<uint2*>(recbuf + head) = *reinterpret_cast<const uint2*>(gsrc);
        if (tail)
            *reinterpret_cast<uint2*>(recbuf + head + hb + body) =
                *reinterpret_cast<const uint2*>(gsrc + hb + body);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_bar, body);
        for (uint32_t o = 0; o < body; o += 32768u)
            tma_load_1d(recbuf + head + hb + o, gsrc + hb + o, min(32768u, body - o), &s_bar);
        s_wmin = 0xFFFFFFFFu;
        s_wmax = 0u;
        s_flag = 0;
        s_maxb = 0;
    }
    __syncthreads();
    mbar_wait(&s_bar, 0);

    // 2. AND/OR of the record words -> varying key bytes L in [p, ks)
    {
        uint64_t a[KW], o[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) a[w] = ~0ull, o[w] = 0ull;
        for (uint32_t e = threadIdx.x; e < n; e += T) {
            const Rec<RS> r = ld_smem_rec<RS>(recs, e);
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
            if (lane == 0) s_and[warp][w] = a[w], s_or[warp][w] = o[w];
        }
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t diffb = 0;
        const uint32_t b = lane;
        if (b >= g.p && b < ks && b < uint32_t(RS)) {
            unsigned long long ra = ~0ull, ro = 0ull;
            for (int q = 0; q < W; ++q) {
                unsigned long long xa = s_and[q][0], xo = s_or[q][0];
#pragma unroll
                for (int w = 1; w < KW; ++w)
                    if ((b >> 3) == uint32_t(w)) xa = s_and[q][w], xo = s_or[q][w];
                ra &= xa;
                ro |= xo;
            }
            diffb = uint32_t(((ra ^ ro) >> ((b & 7) * 8)) & 0xFF);
        }
        const uint32_t vm = __ballot_sync(0xFFFFFFFFu, diffb != 0);
        if (diffb) s_L[__popc(vm & lanemask_lt())] = lane;
        if (lane == 0) s_nL = __popc(vm);
    }
    __syncthreads();
    const uint32_t nL = s_nL;
    if (nL == 0) {  // every key equal: stable order is the input order
        if (g.parity)
            for (uint32_t e = threadIdx.x; e < n; e += T) store_rec<RS>(dst, e, ld_smem_rec<RS>(recs, e));
        return;
    }
    const uint32_t nwin = nL < 4 ? nL : 4;
    const bool beyond = nL > 4;

    // 3. 32-bit windows (bytes L0..L3, big-endian) and their range
    {
        const uint32_t L0 = s_L[0], L1 = s_L[nwin > 1 ? 1 : 0], L2 = s_L[nwin > 2 ? 2 : 0],
                       L3 = s_L[nwin > 3 ? 3 : 0];
        uint32_t mn = 0xFFFFFFFFu, mx = 0u;
        for (uint32_t e = threadIdx.x; e < n; e += T) {
            const uint8_t* rp = recs + size_t(e) * RS;
            uint32_t wv = uint32_t(rp[L0]) << 24;
            if (nwin > 1) wv |= uint32_t(rp[L1]) << 16;
            if (nwin > 2) wv |= uint32_t(rp[L2]) << 8;
            if (nwin > 3) wv |= uint32_t(rp[L3]);
            win[e] = wv;
            mn = min(mn, wv);
            mx = max(mx, wv);
        }
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0) {
            atomicMin(&s_wmin, mn);
            atomicMax(&s_wmax, mx);
        }
    }
    uint32_t B = 32u - __clz(n - 1);
    B = B < 1 ? 1 : (B > uint32_t(C::kBucketBits) ? uint32_t(C::kBucketBits) : B);
    const uint32_t nbk = 1u << B;
    for (uint32_t i = threadIdx.x; i < nbk / 2; i += T) cnt[i] = 0;
    __syncthreads();
    const uint32_t wmin = s_wmin;
    const uint32_t range = s_wmax - wmin;
    const bool exact = uint64_t(range) + 1 <= nbk;
    const unsigned long long mul = exact ? 0ull : (((unsigned long long)nbk << 32) / (uint64_t(range) + 1));
    auto bucket_of = [&](uint32_t w) -> uint32_t {
        const uint32_t d = w - wmin;
        return exact ? d : uint32_t((uint64_t(d) * mul) >> 32);
    };
    auto end_of = [&](uint32_t b) { return (cnt[b >> 1] >> ((b & 1) * 16)) & 0xFFFFu; };
    // -1/0/+1 on the varying bytes beyond the window, from shared memory
    auto cmp_rest = [&](uint32_t a, uint32_t b) -> int {
        for (uint32_t q = 4; q < nL; ++q) {
            const uint32_t x = recs[size_t(a) * RS + s_L[q]], y = recs[size_t(b) * RS + s_L[q]];
            if (x != y) return x < y ? -1 : 1;
        }
        return 0;
    };

    // 4. bucket histogram, scan (packed u16 pairs), largest bucket
    for (uint32_t e = threadIdx.x; e < n; e += T) {
        const uint32_t b = bucket_of(win[e]);
        atomicAdd(&cnt[b >> 1], 1u << ((b & 1) * 16));
    }
    __syncthreads();
    {
        const uint32_t per = nbk > uint32_t(T) ? nbk / T : 1u;
        const uint32_t b0 = threadIdx.x * per;
        uint32_t sum = 0, mx = 0;
        if (b0 < nbk) {
            for (uint32_t b = b0; b < b0 + per; ++b) {
                const uint32_t c = end_of(b);  // still counts here
                sum += c;
                mx = c > mx ? c : mx;
            }
        }
        uint32_t total;
        uint32_t run = block_scan_excl(sum, s_scan, &total);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0 && mx) atomicMax(&s_maxb, mx);
        if (b0 < nbk) {
            if (per >= 2) {
                for (uint32_t b = b0; b < b0 + per; b += 2) {
                    const uint32_t w = cnt[b >> 1];
                    const uint32_t c0 = w & 0xFFFFu, c1 = w >> 16;
                    cnt[b >> 1] = run | ((run + c0) << 16);
                    run += c0 + c1;
                }
            } else if ((b0 & 1) == 0) {
                const uint32_t c0 = cnt[b0 >> 1] & 0xFFFFu;
                cnt[b0 >> 1] = run | ((run + c0) << 16);
            }
        }
    }
    __syncthreads();

    if (!kFallback && s_maxb <= kMaxBucket) {
        // 5. record ids into bucket order (cnt: starts -> ends)
        for (uint32_t e = threadIdx.x; e < n; e += T) {
            const uint32_t b = bucket_of(win[e]);
            const uint32_t old = atomicAdd(&cnt[b >> 1], 1u << ((b & 1) * 16));
            slot[(old >> ((b & 1) * 16)) & 0xFFFFu] = uint16_t(e);
        }
        __syncthreads();
        // 6. rank inside the bucket, one slot per thread (lane-contiguous slots)
        for (uint32_t q = threadIdx.x; q < n; q += T) {
            const uint32_t e = slot[q];
            const uint32_t w = win[e];
            const uint32_t b = bucket_of(w);
            const uint32_t en = end_of(b);
            const uint32_t st = b ? end_of(b - 1) : 0u;
            uint32_t rank = 0;
            for (uint32_t q2 = st; q2 < en; ++q2) {
                const uint32_t e2 = slot[q2];
                const uint32_t w2 = win[e2];
                bool less = w2 < w;
                if (w2 == w && e2 != e) {
                    const int c = beyond ? cmp_rest(e2, e) : 0;
                    less = c < 0 || (c == 0 && e2 < e);
                }
                rank += less;
            }
            perm[st + rank] = uint16_t(e);
        }
        __syncthreads();
    } else {
        if (!kFallback) {  // crowded buckets: hand the untouched group to the LSD instance
            if (threadIdx.x == 0) {
                const uint32_t i = atomicAdd(n_spill, 1u);
                if (i < spill_cap) spill[i] = g;
                atomicAdd(&ctr->fallback_groups, 1ull);
            }
            return;
        }
        if constexpr (kFallback) {
            // stable LSD over the window bytes, then every varying byte if ties remain
            uint16_t *pin = slot, *pout = perm;
            bool first = true;
            for (int q = int(nwin) - 1; q >= 0; --q) {
                const uint32_t sh = 24u - 8u * uint32_t(q);
                auto dig = [&](uint32_t e) { return (win[e] >> sh) & 0xFFu; };
                if (first)
                    lsd_pass_w<IPT, W, true>(n, pin, pout, cnt, s_tot, dig);
                else
                    lsd_pass_w<IPT, W, false>(n, pin, pout, cnt, s_tot, dig);
                first = false;
                uint16_t* t = pin;
                pin = pout;
                pout = t;
            }
            if (beyond) {
                for (uint32_t pos = threadIdx.x + 1; pos < n; pos += T) {
                    const uint32_t ea = pin[pos - 1], eb = pin[pos];
                    if (win[ea] == win[eb] && cmp_rest(ea, eb) > 0) s_flag = 1;
                }
                __syncthreads();
                if (s_flag) {
                    first = true;
                    for (int q = int(nL) - 1; q >= 0; --q) {
                        const uint32_t bb = s_L[q];
                        auto dig = [&](uint32_t e) { return uint32_t(recs[size_t(e) * RS + bb]); };
                        if (first)
                            lsd_pass_w<IPT, W, true>(n, pin, pout, cnt, s_tot, dig);
                        else
                            lsd_pass_w<IPT, W, false>(n, pin, pout, cnt, s_tot, dig);
                        first = false;
                        uint16_t* t = pin;
                        pin = pout;
                        pout = t;
                    }
                }
            }
            if (pin != perm)
                for (uint32_t i = threadIdx.x; i < n; i += T) perm[i] = pin[i];
            __syncthreads();
        }
    }

    // 7. final positions in order: coalesced stores of records read from shared memory
#pragma unroll 4
    for (uint32_t f = threadIdx.x; f < n; f += T) store_rec<RS>(dst, f, ld_smem_rec<RS>(recs, perm[f]));
    if (threadIdx.x == 0) atomicAdd(&ctr->moved_local, (unsigned long long)n);
}

}  // namespace rg
