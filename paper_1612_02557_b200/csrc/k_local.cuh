// (d) segmented small-bin sort for the MSD tail.
//
// Reference: the tiny-bin comparison sorts (P/include/raduls/small_sorts.hpp:
// 48-191: insertion / Shell {8,1} / introsort chosen by TinyPolicy :14-45), the
// plain radix_split used for bins that fit half of L2 (kernels.hpp:157-167 via
// msd_sorter.hpp:188-196) and finalize()'s copy back to the caller's buffer
// (msd_sorter.hpp:76-80).
//
// One CTA sorts a *group*: one or more adjacent complete segments (bins) of at
// most kCap records that share key bytes [0, p). Sorting the group by key bytes
// [p, ks) equals sorting each bin on its own (the bins are contiguous and
// already in key order). The whole group is held on chip before anything is
// written, so the sort is safe in place (source == destination buffer):
//   * record sizes 16/24/32: one TMA bulk copy (cp.async.bulk + mbarrier) puts
//     the group in shared memory; the output walks final positions in order
//     (coalesced vector stores) reading records from shared memory;
//   * record size 8 (groups up to 18 K records, BASELINE C2's 16 K-record
//     bins): records stay in registers; the output is staged through shared
//     memory in final order, then written with coalesced stores.
// Steps: AND/OR of the key words (REDUX) -> the varying key bytes
// L = l0 < l1 < ... in [p, ks); their first <= 4 form a big-endian 32-bit
// window w per record (one byte permute when they sit in two adjacent words);
// one counting pass over ~2n buckets spread linearly over [min w, max w]
// (histogram with packed u16 counters, vectorised conflict-free scan, scatter
// of record ids); then every record ranks itself inside its bucket, branch-
// free for buckets of <= 3 records, by (w, remaining key bytes, input index);
// larger buckets go to a short list ranked afterwards. Duplicate-heavy groups
// (a bucket over kMaxBucket) are handed untouched to the kFallback instance: a
// stable LSD over every varying byte. Every path orders equal keys by input
// index, so the sort is stable.
#pragma once

#include "common.cuh"

namespace rg {

constexpr uint32_t kMaxBucket = 32;

// output loop unroll (measured vs 4: 8 at 16 B C1 -3%, C3 -3%, C5 -4%;
// 2 at 32 B C4 -1.7%, where 8 costs +5%)
#ifndef RG_LOC_OUTU
#define RG_LOC_OUTU 0
#endif
template <int RS>
constexpr int kLocOutUnroll = RG_LOC_OUTU ? RG_LOC_OUTU : (RS == 32 ? 2 : 8);
#ifndef RG_LOC_OUT8U
#define RG_LOC_OUT8U 0
#endif
constexpr int kLocOut8Unroll = RG_LOC_OUT8U;  // 8-B staged output loop
#ifndef RG_LOC_KEYW
#define RG_LOC_KEYW 1
#endif

template <int RS>
struct LocalCfg {
    static constexpr bool kRegRecords = RS == 8;  // records in registers (else shared memory)
    // 16/24-B records: small CTAs, four per SM, so one group's HBM traffic and
    // barriers overlap other groups' work; 32-B records keep 4608-record groups
    // (BASELINE C4's ~4 K-record bins) at one CTA per SM.
    // RG_LOC8_CAP / _THREADS / _BLOCKS / _BITS: the 8-B shape, as knobs for
    // the measured alternative of a third scatter level at C2 (a smaller cap
    // makes C2's ~16 K-record bins split once more)
#ifndef RG_LOC8_CAP
#define RG_LOC8_CAP 18432
#endif
#ifndef RG_LOC8_THREADS
#define RG_LOC8_THREADS 1024
#endif
#ifndef RG_LOC8_BLOCKS
#define RG_LOC8_BLOCKS 1
#endif
#ifndef RG_LOC8_BITS
#define RG_LOC8_BITS 15
#endif
    static constexpr int kThreads = kRegRecords ? RG_LOC8_THREADS : 512;
    static constexpr int kMinBlocks = (RS == 16 || RS == 24) ? 2 : RS == 8 ? RG_LOC8_BLOCKS : 1;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kCap = RS == 8 ? RG_LOC8_CAP : RS == 16 ? 3584 : RS == 24 ? 2560 : 4608;
    static constexpr int kIpt = (kCap + kThreads - 1) / kThreads;
    static constexpr int kBucketBits = RS == 8 ? RG_LOC8_BITS : 13;
    // packed u16 bucket counters, four pad words per 64 buckets (conflict-free LDS.128 scan)
    static constexpr int kCntWords = (1 << kBucketBits) / 2 + (1 << kBucketBits) / 16;
    static constexpr int kCntBytes = (kCntWords * 4 > kWarps * kRadix * 4) ? kCntWords * 4
                                                                             : kWarps * kRadix * 4;
    static constexpr int kRecBytes = kRegRecords ? 0 : ((kCap * RS + 16 + 127) / 128) * 128;
    // RG_LOC_LIST=1 (shared-memory records): singletons placed during the id
    // scatter, records of multi-record buckets appended to a CTA list (kList
    // u16 entries fit beside two CTAs per SM at 16/24 B) and ranked densely
    // from it. Fewer instructions, but each list entry is a chain of four
    // dependent shared-memory loads with ~2.5 entries per thread, against
    // three with seven independent records per thread in the per-record pass:
    // measured slower (interleaved A/B, one box: C5 local 50.3 vs 47.3 ms, C1
    // +5%, C4 +9%, C2 unchanged); off by default.
#ifndef RG_LOC_LIST
#define RG_LOC_LIST 0
#endif
    static constexpr int kList = (kRegRecords || !RG_LOC_LIST) ? 0 : RS == 32 ? kCap : 2560;
    static constexpr int kTotWords = (kList / 2 > 512) ? kList / 2 : 512;
    static constexpr int kBmWords = kList ? (1 << kBucketBits) / 32 : 1;
    static constexpr size_t kSmem = size_t(kRecBytes) + size_t(kCap) * (4 + 2 + 2) + kCntBytes;
};

// Block-wide exclusive scan (blockDim a multiple of 32, <= 1024): one
// barrier; every warp then adds up the totals of the warps before it itself.
template <bool kTrailingSync = true>
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
    // lane q holds warp q's total; the warp's base is the sum over q < warp
    const uint32_t t = lane < nw ? s_w[lane] : 0u;
    const uint32_t base = __reduce_add_sync(0xFFFFFFFFu, lane < warp ? t : 0u);
    *total = __reduce_add_sync(0xFFFFFFFFu, t);
    if (kTrailingSync) __syncthreads();  // s_w may be reused
    return base + x - v;
}

// Stable LSD pass for W warps (T = 32 W threads, T % 256 == 0): pout <- pin
// ordered by digit(pin[pos]); ballot multisplit with warp-private counters,
// digit-major / warp-minor offsets.
template <int IPT, int W, bool kIdentity, typename DigitFn>
__device__ __forceinline__ void lsd_pass_w(uint32_t n, const uint16_t* pin, uint16_t* pout,
                                           uint32_t* wcnt, uint32_t* s_tot, DigitFn digit_of) {
    constexpr int T = W * 32;
    constexpr int TPD = T / 256;  // threads per digit in the offset scan
    constexpr int WPT = W / TPD;  // warps per such thread
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

// One group, by the whole CTA (called per group by the persistent k_local).
// `mid` is called by every thread once the bucket geometry is known (the
// persistent launch uses it to prefetch the next group off the critical path).
template <int RS, bool kFallback, typename Mid>
__device__ __forceinline__ void local_group(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group g,
    uint32_t ks, LevelCounters* __restrict__ ctr, Group* __restrict__ spill,
    unsigned int* __restrict__ n_spill, uint32_t spill_cap, Mid&& mid) {
    using C = LocalCfg<RS>;
    constexpr bool REG = C::kRegRecords;
    // RG_LOC_DIRECT (shared-memory records): each record is stored to its final
    // place when it is ranked (its own slot read from shared memory, one
    // uncoalesced 16-B global store; the group's lines fill up in L2 within
    // microseconds) instead of through perm and a coalesced output loop that
    // gathers records at random from shared memory (~10.4 wavefronts per 32
    // records against 4). Interleaved A/B (profiles/r2_ab_direct*.log): C5
    // local 44.5 vs 46.7 ms, C3 -3%, C1 -2.3%, C4 unchanged.
#ifndef RG_LOC_DIRECT
#define RG_LOC_DIRECT 1
#endif
    constexpr bool kDirect = RG_LOC_DIRECT && !REG;
    constexpr int T = C::kThreads, W = C::kWarps, IPT = C::kIpt;
    constexpr int KW = RS / 8;
    extern __shared__ __align__(128) uint8_t smem[];
    RG_CHK_POISON_SMEM(smem);
    // [perm][win][slot][cnt]: win..cnt is one span, the 8-B output's staging area
    uint16_t* perm = reinterpret_cast<uint16_t*>(smem + C::kRecBytes);  // [cap] final order / fpos
    uint32_t* win = reinterpret_cast<uint32_t*>(perm + C::kCap);        // [cap]
    uint16_t* slot = reinterpret_cast<uint16_t*>(win + C::kCap);        // [cap] bucket order
    uint32_t* cnt = reinterpret_cast<uint32_t*>(slot + C::kCap);        // packed u16 pairs
    __shared__ uint32_t s_tot[C::kTotWords];  // LSD totals / deferred lists / the multi-bucket list (u16)
    __shared__ uint32_t s_bm[C::kBmWords];     // kList: singleton-bucket bitmap
    __shared__ uint32_t s_lcnt;                // kList: multi-bucket list length
    __shared__ uint32_t s_scan[65];
    __shared__ uint32_t s_and[W][2 * KW], s_or[W][2 * KW];
    __shared__ uint32_t s_Lw[W][32];  // per-warp copy of the varying key bytes
    __shared__ uint32_t s_flag, s_maxb, s_wmin, s_wmax, s_wmin2, s_wmax2;
    __shared__ uint32_t s_wq[W];  // per-warp deferred-record list lengths
    __shared__ __align__(8) unsigned long long s_bar;

    const uint32_t n = g.size;
    const uint8_t* gsrc = (g.parity ? tmp : data) + g.start * RS;
    uint8_t* dst = data + g.start * RS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (n <= 1) {
        if (n == 1 && g.parity && threadIdx.x == 0) store_rec<RS>(dst, 0, load_rec<RS>(gsrc, 0));
        return;
    }

    // ---- 1. the group on chip
    const uint32_t head = REG ? 0u : uint32_t(reinterpret_cast<uintptr_t>(gsrc) & 15u);
    const uint8_t* recs = smem + head;  // shared-memory records (REG == false)
    Rec<RS> r[REG ? IPT : 1];
    if constexpr (REG) {
        const uint8_t* tsrc = gsrc + size_t(threadIdx.x) * RS;  // constant offsets per j
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (uint32_t(j) * T >= n) break;  // block-uniform
            const uint32_t e = uint32_t(j) * T + threadIdx.x;
            if (e < n) r[j] = load_rec_stream<RS>(tsrc, uint64_t(j) * T);
        }
    } else if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const uint32_t bytes = n * RS;
        const uint32_t hb = head ? min(8u, bytes) : 0u;
        const uint32_t body = (bytes - hb) & ~15u;
        const uint32_t tail = bytes - hb - body;
        if (hb) *reinterpret_cast<uint2*>(smem + head) = *reinterpret_cast<const uint2*>(gsrc);
        if (tail)
            *reinterpret_cast<uint2*>(smem + head + hb + body) =
                *reinterpret_cast<const uint2*>(gsrc + hb + body);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_bar, body);
        for (uint32_t o = 0; o < body; o += 32768u)
            tma_load_1d_h<RG_HINT_LOCAL>(smem + head + hb + o, gsrc + hb + o, min(32768u, body - o), &s_bar);
    }
    if (threadIdx.x == 0) {
        s_wmin = 0xFFFFFFFFu;
        s_wmax = 0u;
        s_wmin2 = 0xFFFFFFFFu;
        s_wmax2 = 0u;
        s_flag = 0;
        for (int q = 0; q < W; ++q) s_wq[q] = 0;
        s_maxb = 0;
        s_lcnt = 0;
    }
    if constexpr (C::kList > 0)
        for (uint32_t q = threadIdx.x; q < uint32_t(C::kBmWords); q += T) s_bm[q] = 0;
    // bucket counters zeroed now (first used by the histogram, several barriers on)
    for (uint32_t i = threadIdx.x; i < uint32_t(C::kCntWords + 3) / 4; i += T)
        reinterpret_cast<uint4*>(cnt)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if constexpr (!REG) mbar_wait(&s_bar, 0);
    auto rec_of = [&](int j, uint32_t e) -> Rec<RS> {
        if constexpr (REG) return r[j];
        else return ld_smem_rec<RS>(recs, e);
    };

    // ---- 2. AND/OR of the record words (REDUX) -> varying key bytes L.
    // Shared-memory records: the same pass computes the window of the default
    // varying bytes p..p+3 (what random keys have), kept if L confirms it, so
    // the records are read once instead of twice.
    constexpr bool KEEP = !REG;
    uint32_t wv[KEEP ? IPT : 1];
    uint32_t smn = 0xFFFFFFFFu, smx = 0u;
    uint32_t Ldef[4] = {g.p, g.p + 1, g.p + 2, g.p + 3};
    const WindowSel wsd = make_window_sel(Ldef, 4, RS / 4, false);
    // (16/24-B records; measured a loss at 32 B, whose kernel is register-bound)
    const bool spec = KEEP && RS <= 24 && g.p + 4 <= ks && g.p + 4 <= uint32_t(RS) && wsd.fast;
    // only the words holding key bytes (payload words cannot vary the
    // order): the first half when ks <= rs / 2, e.g. BASELINE C1/C3/C5
    const uint32_t nk = (RG_LOC_KEYW && RS >= 16 && ks <= uint32_t(4 * KW)) ? uint32_t(KW) : uint32_t(2 * KW);
    {
        uint32_t a[2 * KW], o[2 * KW];
#pragma unroll
        for (int w = 0; w < 2 * KW; ++w) a[w] = ~0u, o[w] = 0u;
        auto andor = [&](auto specc, auto nkc) {
            constexpr int NK = decltype(nkc)::value;
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                if (e < n) {
                    const Rec<RS> v = rec_of(j, e);
#pragma unroll
                    for (int w = 0; w < NK; ++w) a[w] &= v.w[w], o[w] |= v.w[w];
                    if constexpr (decltype(specc)::value) {
                        const uint32_t w = rec_window<RS>(v, wsd);
                        wv[KEEP ? j : 0] = w;
                        win[e] = w;
                        smn = min(smn, w);
                        smx = max(smx, w);
                    }
                }
            }
        };
        if (nk == uint32_t(KW)) {
            if (spec) andor(BoolC<KEEP>{}, IntC<KW>{});
            else andor(BoolC<false>{}, IntC<KW>{});
        } else {
            if (spec) andor(BoolC<KEEP>{}, IntC<2 * KW>{});
            else andor(BoolC<false>{}, IntC<2 * KW>{});
        }
#pragma unroll
        for (int w = 0; w < 2 * KW; ++w) {
            if (uint32_t(w) < nk) {  // (the rest stay ~0 / 0: constant)
                a[w] = __reduce_and_sync(0xFFFFFFFFu, a[w]);
                o[w] = __reduce_or_sync(0xFFFFFFFFu, o[w]);
            }
        }
        if (lane < 2 * KW) {
            uint32_t av = a[0], ov = o[0];
#pragma unroll
            for (int w = 1; w < 2 * KW; ++w)
                if (lane == w) av = a[w], ov = o[w];
            s_and[warp][lane] = av;
            s_or[warp][lane] = ov;
        }
        if (spec) {  // the default windows' range, complete at the barrier below
            smn = __reduce_min_sync(0xFFFFFFFFu, smn);
            smx = __reduce_max_sync(0xFFFFFFFFu, smx);
            if (lane == 0) {
                atomicMin(&s_wmin, smn);
                atomicMax(&s_wmax, smx);
            }
        }
    }
    __syncthreads();
    // every warp derives the varying bytes itself (no second block barrier)
    uint32_t* s_L = s_Lw[warp];
    uint32_t nL;
    {
        // lane q < W holds warp q's partials; REDUX combines them per word
        const uint32_t b = lane;  // key byte b lives in 32-bit word b/4
        uint32_t dsel = 0;
#pragma unroll
        for (int w = 0; w < 2 * KW; ++w) {
            if (uint32_t(w) < nk) {
                const uint32_t ra = __reduce_and_sync(0xFFFFFFFFu, lane < W ? s_and[lane][w] : ~0u);
                const uint32_t ro = __reduce_or_sync(0xFFFFFFFFu, lane < W ? s_or[lane][w] : 0u);
                if ((b >> 2) == uint32_t(w)) dsel = ra ^ ro;
            }
        }
        uint32_t diffb = 0;
        if (b >= g.p && b < ks && b < uint32_t(RS)) diffb = (dsel >> ((b & 3) * 8)) & 0xFFu;
        const uint32_t vm = __ballot_sync(0xFFFFFFFFu, diffb != 0);
        if (diffb) s_L[__popc(vm & lanemask_lt())] = lane;
        nL = __popc(vm);
        __syncwarp();
    }
    if (nL == 0) {  // every key equal: stable order is the input order
        if (g.parity) {
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                if (e < n) store_rec<RS>(dst, e, rec_of(j, e));
            }
        }
        return;
    }
    const uint32_t nwin = nL < 4 ? nL : 4;
    const bool beyond = nL > 4;
    const bool spec_ok = spec && nwin == 4 && s_L[0] == g.p && s_L[1] == g.p + 1 && s_L[2] == g.p + 2 &&
                         s_L[3] == g.p + 3;  // warp-uniform and equal in every warp

    // ---- 3. windows (registers + shared memory), their range
    // windows / buckets kept in registers when records are not (register budget)
    // spec_ok: windows and range came with the AND/OR pass (no barrier here)
    if (!spec_ok) {
        const uint32_t L0 = s_L[0], L1 = s_L[nwin > 1 ? 1 : 0], L2 = s_L[nwin > 2 ? 2 : 0],
                       L3 = s_L[nwin > 3 ? 3 : 0];
        const WindowSel ws = make_window_sel(s_L, nwin, RS / 4, RS == 8);
        uint32_t mn = 0xFFFFFFFFu, mx = 0u;
        auto windows = [&](auto fastc) {
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                uint32_t w = 0;
                if (e < n) {
                    // whole-record vector load from shared memory: lanes hit consecutive banks
                    const Rec<RS> v = rec_of(j, e);
                    if constexpr (decltype(fastc)::value) {
                        w = rec_window<RS>(v, ws);
                    } else {
                        w = rec_byte<RS>(v, L0) << 24;
                        if (nwin > 1) w |= rec_byte<RS>(v, L1) << 16;
                        if (nwin > 2) w |= rec_byte<RS>(v, L2) << 8;
                        if (nwin > 3) w |= rec_byte<RS>(v, L3);
                    }
                    win[e] = w;
                    mn = min(mn, w);
                    mx = max(mx, w);
                }
                if constexpr (KEEP) wv[j] = w;
            }
        };
        if (RS == 8 || ws.fast) windows(BoolC<true>{});
        else windows(BoolC<RS == 8>{});
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0) {
            atomicMin(&s_wmin2, mn);
            atomicMax(&s_wmax2, mx);
        }
        __syncthreads();
    }
    // bucket geometry, computed by every thread (no serial step, no barrier):
    // 2^B buckets spread linearly over [wmin, wmax] by bucket = umulhi(w - wmin,
    // mul). Any mul keeps buckets monotone in w; mul <= nbk 2^32 / range
    // (rounded down with a 1e-6 margin over the float error) keeps them < nbk.
    uint32_t B = 33u - __clz(n - 1);  // ceil(log2 n) + 1: ~0.5 records per bucket
    B = B < 1 ? 1 : (B > uint32_t(C::kBucketBits) ? uint32_t(C::kBucketBits) : B);
    const uint32_t nbk = 1u << B;
    const uint32_t wmin = spec_ok ? s_wmin : s_wmin2;
    const uint32_t rm1 = (spec_ok ? s_wmax : s_wmax2) - wmin;  // range - 1
    const uint32_t mul =
        rm1 < nbk ? 0u : uint32_t(__fdiv_rz(float(nbk) * 4294967296.0f, float(rm1) + 1.0f) * 0.999999f);
    auto bucket_of = [&](uint32_t w) -> uint32_t {  // monotone in w, < nbk
        const uint32_t d = w - wmin;
        return mul ? __umulhi(d, mul) : d;
    };
    // packed counter word of bucket b (u16 pairs, padded: +4 words per 64 buckets)
    auto cw = [&](uint32_t b) -> uint32_t& { return cnt[(b >> 1) + ((b >> 6) << 2)]; };
    // the same counter as a u16 (little-endian halves: even bucket low)
    const uint16_t* cnt16 = reinterpret_cast<const uint16_t*>(cnt);
    auto end_of = [&](uint32_t b) -> uint32_t { return cnt16[b + ((b >> 6) << 3)]; };
    auto cmp_rest = [&](uint32_t a, uint32_t b) -> int {  // bytes beyond the window
        for (uint32_t q = 4; q < nL; ++q) {
            uint32_t x, y;
            if constexpr (REG) {
                x = gsrc[size_t(a) * RS + s_L[q]];
                y = gsrc[size_t(b) * RS + s_L[q]];
            } else {
                x = recs[size_t(a) * RS + s_L[q]];
                y = recs[size_t(b) * RS + s_L[q]];
            }
            if (x != y) return x < y ? -1 : 1;
        }
        return 0;
    };

    mid();
    // ---- 4. bucket histogram (packed u16 pairs, zeroed at the start), scan, largest bucket
    // KEEP: per record (padded u16 counter index | bucket << 16), the address
    // math done once for the histogram, the id scatter and the rank
    auto i16_of = [](uint32_t b) { return b + ((b >> 6) << 3); };
    uint32_t bk[KEEP ? IPT : 1];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (uint32_t(j) * T >= n) break;  // block-uniform
        const uint32_t e = uint32_t(j) * T + threadIdx.x;
        if (e < n) {
            if constexpr (KEEP) {
                const uint32_t b = bucket_of(wv[j]), i = i16_of(b);
                bk[j] = i | (b << 16);
                atomicAdd(&cnt[i >> 1], 1u << ((i & 1) * 16));
            } else {
                const uint32_t b = bucket_of(win[e]);
                atomicAdd(&cw(b), 1u << ((b & 1) * 16));
            }
        }
    }
    __syncthreads();
    {
        const uint32_t per = nbk > uint32_t(T) ? nbk / T : 1u;
        const uint32_t b0 = threadIdx.x * per;
        uint32_t sum = 0, mx = 0;
        // per >= 8: the thread's per/2 counter words are contiguous and 16-B
        // aligned; the pad words make the LDS.128 of 8 threads conflict-free.
        // Packed u16 pairs are summed as u32 (each half stays < 65536).
        uint4* pv = reinterpret_cast<uint4*>(&cw(b0));
        const uint32_t nv = per / 8;
        // kList: bit b of s_bm = bucket b holds exactly one record
        auto ones = [](uint32_t w) {  // the two u16 halves == 1 -> bits 0, 1
            return uint32_t((w & 0xFFFFu) == 1u) | (uint32_t((w >> 16) == 1u) << 1);
        };
        if (per >= 8) {
            uint32_t S = 0, M = 0, bits = 0;
            for (uint32_t v = 0; v < nv; ++v) {
                const uint4 q = pv[v];
                S += q.x + q.y + q.z + q.w;
                M = __vmaxu2(M, __vmaxu2(__vmaxu2(q.x, q.y), __vmaxu2(q.z, q.w)));
                if constexpr (C::kList > 0) {
                    const uint32_t m8 = ones(q.x) | (ones(q.y) << 2) | (ones(q.z) << 4) | (ones(q.w) << 6);
                    bits |= m8 << ((v * 8u) & 31u);
                    if (((v * 8u + 8u) & 31u) == 0u || v + 1 == nv) {
                        const uint32_t bb0 = b0 + ((v * 8u) & ~31u);
                        atomicOr(&s_bm[bb0 >> 5], bits << (bb0 & 31u));
                        bits = 0;
                    }
                }
            }
            sum = (S & 0xFFFFu) + (S >> 16);
            mx = max(M & 0xFFFFu, M >> 16);
        } else if (b0 < nbk) {
            uint32_t bits = 0;
            for (uint32_t b = b0; b < b0 + per; ++b) {
                const uint32_t c = end_of(b);  // still counts
                sum += c;
                mx = c > mx ? c : mx;
                bits |= uint32_t(c == 1u) << (b - b0);
            }
            if constexpr (C::kList > 0)
                if (bits) atomicOr(&s_bm[b0 >> 5], bits << (b0 & 31u));
        }
        uint32_t total;
        uint32_t run = block_scan_excl<false>(sum, s_scan, &total);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0 && mx) atomicMax(&s_maxb, mx);
        // counts -> (start of even bucket | start of odd bucket << 16)
        auto starts = [&](uint32_t w) {
            const uint32_t o = run * 0x10001u + (w << 16);
            run += (w * 0x10001u) >> 16;
            return o;
        };
        if (per >= 8) {
            for (uint32_t v = 0; v < nv; ++v) {
                uint4 q = pv[v];
                q.x = starts(q.x);
                q.y = starts(q.y);
                q.z = starts(q.z);
                q.w = starts(q.w);
                pv[v] = q;
            }
        } else if (b0 < nbk) {
            if (per >= 2) {
                for (uint32_t b = b0; b < b0 + per; b += 2) {
                    const uint32_t w = cw(b);
                    const uint32_t c0 = w & 0xFFFFu, c1 = w >> 16;
                    cw(b) = run | ((run + c0) << 16);
                    run += c0 + c1;
                }
            } else if ((b0 & 1) == 0) {
                const uint32_t c0 = cw(b0) & 0xFFFFu;
                cw(b0) = run | ((run + c0) << 16);
            }
        }
    }
    __syncthreads();

    if (!kFallback && s_maxb <= kMaxBucket) {
        auto less = [&](uint32_t w2, uint32_t e2, uint32_t w, uint32_t e) -> bool {
            if (w2 != w) return w2 < w;
            const int c = beyond ? cmp_rest(e2, e) : 0;
            return c < 0 || (c == 0 && e2 < e);
        };
        auto place = [&](uint32_t e, uint32_t f) {
            if constexpr (REG) perm[e] = uint16_t(f);  // e -> final position
            else if constexpr (kDirect) store_rec<RS>(dst, f, ld_smem_rec<RS>(recs, e));  // now, uncoalesced
            else perm[f] = uint16_t(e);                // final position -> e
        };
        auto rank_slow = [&](uint32_t e, uint32_t w, uint32_t st, uint32_t en) {
            uint32_t rank = 0;
            for (uint32_t q2 = st; q2 < en; ++q2) {
                const uint32_t e2 = slot[q2];
                if (e2 != e) rank += less(win[e2], e2, w, e);
            }
            return rank;
        };
        // rank of record e (window w) in its bucket [st, en) of <= 3 records:
        // branch-free; the bucket's slots are read clamped (a slot equal to e
        // counts nothing); equal windows with key bytes beyond them take the
        // full comparison
        auto rank3 = [&](uint32_t e, uint32_t w, uint32_t st, uint32_t en) -> uint32_t {
            const uint32_t sz = en - st, last = en - 1;
            // a bucket of one needs no neighbour: its lanes skip the loads
            uint32_t e1 = e, e2 = e, e3 = e, w1 = w, w2 = w, w3 = w;
            if (sz > 1) {
                e1 = slot[st];
                e2 = slot[min(st + 1, last)];
                e3 = slot[min(st + 2, last)];
                w1 = win[e1];
                w2 = win[e2];
                w3 = win[e3];
            }
            const bool u1 = e1 != e, u2 = e2 != e && e2 != e1, u3 = e3 != e && e3 != e2;
            // (window, index) order as one 64-bit compare
            const uint64_t k = (uint64_t(w) << 32) | e;
            uint32_t rank = 0;
            rank += u1 && ((uint64_t(w1) << 32) | e1) < k;
            rank += u2 && ((uint64_t(w2) << 32) | e2) < k;
            rank += u3 && ((uint64_t(w3) << 32) | e3) < k;
            const bool tie = (u1 && w1 == w) || (u2 && w2 == w) || (u3 && w3 == w);
            if (beyond && tie) rank = rank_slow(e, w, st, en);
            return rank;
        };
        bool listed = false;
        if constexpr (C::kList > 0) {
            // ---- 5. record ids into bucket order (cnt: starts -> ends). A
            // record alone in its bucket (~2/3 of them at ~0.44 records per
            // bucket) is final at its slot: placed now, never ranked. The others
            // go to a CTA-wide list (warp-aggregated appends), ranked densely
            // after the barrier -- no pass over all records for the ranking.
            uint16_t* clst = reinterpret_cast<uint16_t*>(s_tot);
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                bool multi = false;
                if (e < n) {
                    const uint32_t i = bk[j] & 0xFFFFu, b = (bk[j] >> 16) & 0x1FFFu;
                    const uint32_t old = atomicAdd(&cnt[i >> 1], 1u << ((i & 1) * 16));
                    const uint32_t pos = (old >> ((i & 1) * 16)) & 0xFFFFu;
                    if ((s_bm[b >> 5] >> (b & 31u)) & 1u) {
                        place(e, pos);
                    } else {
                        slot[pos] = uint16_t(e);
                        multi = true;
                    }
                }
                const uint32_t mm = __ballot_sync(0xFFFFFFFFu, multi);
                if (mm) {
                    const uint32_t leader = uint32_t(__ffs(mm) - 1);
                    uint32_t base = 0;
                    if (uint32_t(lane) == leader) base = atomicAdd(&s_lcnt, uint32_t(__popc(mm)));
                    base = __shfl_sync(0xFFFFFFFFu, base, leader);
                    if (multi) {
                        const uint32_t q = base + __popc(mm & lanemask_lt());
                        if (q < uint32_t(C::kList)) clst[q] = uint16_t(e);
                    }
                }
            }
            __syncthreads();
            const uint32_t nl = s_lcnt;
            if (nl <= uint32_t(C::kList)) {  // block-uniform
                listed = true;
                // ---- 6. order inside the multi-record buckets
                for (uint32_t q = threadIdx.x; q < nl; q += T) {
                    const uint32_t e = clst[q];
                    const uint32_t w = win[e];
                    const uint32_t bb = bucket_of(w);
                    const uint32_t en = end_of(bb);
                    const uint32_t st = bb ? end_of(bb - 1) : 0u;
                    place(e, st + (en - st <= 3 ? rank3(e, w, st, en) : rank_slow(e, w, st, en)));
                }
            }
            // (list overflow: the per-record pass below; every multi-record
            // bucket's slots are filled, singletons place themselves again)
        } else {
            // ---- 5. record ids into bucket order (cnt: starts -> ends)
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                if (e < n) {
                    uint32_t i;  // the bucket's u16 counter index
                    if constexpr (KEEP) i = bk[j] & 0xFFFFu;
                    else i = i16_of(bucket_of(win[e]));
                    const uint32_t old = atomicAdd(&cnt[i >> 1], 1u << ((i & 1) * 16));
                    slot[(old >> ((i & 1) * 16)) & 0xFFFFu] = uint16_t(e);
                }
            }
            __syncthreads();
        }
        if (!listed) {
            // ---- 6. order inside buckets (~1 record each), per record: size-1
            // bucket -> its start; size 2-3 -> rank3; larger buckets (a few
            // percent) go to a per-warp list (s_tot: 1024 u16 split over the
            // warps) ranked densely by the same warp after its loop; s_wq (the
            // lengths) are 0 from the start
            constexpr uint32_t kWq = 1024 / W;
            uint16_t* lst = reinterpret_cast<uint16_t*>(s_tot) + warp * kWq;
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                if (e < n) {
                    uint32_t w, bb, en, st;
                    if constexpr (KEEP) {
                        w = wv[j];
                        bb = (bk[j] >> 16) & 0x1FFFu;
                        const uint32_t i = bk[j] & 0xFFFFu;  // bucket bb - 1 sits 1 (9 across a pad) below
                        en = cnt16[i];
                        st = bb ? cnt16[i - ((bb & 63) ? 1u : 9u)] : 0u;
                    } else {
                        w = win[e];
                        bb = bucket_of(w);
                        en = end_of(bb);
                        st = bb ? end_of(bb - 1) : 0u;
                    }
                    if (en - st <= 3) {
                        place(e, st + rank3(e, w, st, en));
                    } else {
                        const uint32_t i = atomicAdd(&s_wq[warp], 1u);
                        if (i < kWq) lst[i] = uint16_t(e);
                        else place(e, st + rank_slow(e, w, st, en));  // list full: rank inline
                    }
                }
            }
            __syncwarp();
            {
                const uint32_t nl = min(s_wq[warp], kWq);
                for (uint32_t i = lane; i < nl; i += 32) {
                    const uint32_t e = lst[i];
                    const uint32_t w = win[e];
                    const uint32_t bb = bucket_of(w);
                    const uint32_t en = end_of(bb);
                    const uint32_t st = bb ? end_of(bb - 1) : 0u;
                    place(e, st + rank_slow(e, w, st, en));
                }
            }
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
                        auto dig = [&](uint32_t e) -> uint32_t {
                            if constexpr (REG) return gsrc[size_t(e) * RS + bb];
                            else return recs[size_t(e) * RS + bb];
                        };
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
            // pin: final position -> e. Into perm in the layout the output step expects.
            if constexpr (REG) {
                for (uint32_t i = threadIdx.x; i < n; i += T) pout[pin[i]] = uint16_t(i);
                __syncthreads();
                if (pout != perm)
                    for (uint32_t i = threadIdx.x; i < n; i += T) perm[i] = pout[i];
            } else if (pin != perm) {
                for (uint32_t i = threadIdx.x; i < n; i += T) perm[i] = pin[i];
            }
            __syncthreads();
        }
    }

    // ---- 7. output (all reads of the source are done)
    if constexpr (REG) {
        // stage through shared memory (win..cnt, free now) so the global stores
        // are coalesced instead of one scattered 8-B store per lane; chunks of
        // final positions when the group outgrows the span
        constexpr uint32_t CC = uint32_t(size_t(C::kCap) * 6 + C::kCntBytes) / RS;
        uint8_t* stage = reinterpret_cast<uint8_t*>(win);
        for (uint32_t c0 = 0; c0 < n; c0 += CC) {
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                if (uint32_t(j) * T >= n) break;  // block-uniform
                const uint32_t e = uint32_t(j) * T + threadIdx.x;
                if (e < n) {
                    const uint32_t f = perm[e];
                    if (CC >= uint32_t(C::kCap) || (f >= c0 && f < c0 + CC))
                        st_smem_rec<RS>(stage, f - c0, r[j]);
                }
            }
            __syncthreads();
            const uint32_t cn = min(CC, n - c0);
#if RG_LOC_OUT8U
#pragma unroll kLocOut8Unroll
#endif
            for (uint32_t i = threadIdx.x; i < cn; i += T)
                store_rec<RS>(dst, c0 + i, ld_smem_rec<RS>(stage, i));
            if (c0 + CC < n) __syncthreads();
        }
    } else {
        if constexpr (!(kDirect && !kFallback)) {  // (kDirect: every record was stored when placed)
#pragma unroll kLocOutUnroll<RS>
            for (uint32_t f = threadIdx.x; f < n; f += T)
                store_rec<RS>(dst, f, ld_smem_rec<RS>(recs, perm[f]));
        }
    }
    if (threadIdx.x == 0) atomicAdd(&ctr->moved_local, (unsigned long long)n);
}

// Pull a group's bytes toward L2 (cp.async.bulk.prefetch.L2): issued one group
// ahead, so the next group's TMA copy / loads are served from L2 while this
// group is being sorted.
template <int RS>
__device__ __forceinline__ void prefetch_group_l2(const uint8_t* data, const uint8_t* tmp, const Group& g) {
    const uintptr_t src = reinterpret_cast<uintptr_t>((g.parity ? tmp : data) + g.start * RS);
    uintptr_t a = (src + 15) & ~uintptr_t(15);
    const uintptr_t e = (src + uintptr_t(g.size) * RS) & ~uintptr_t(15);
    for (; a < e; a += 32768) {
        const uint32_t sz = uint32_t(min(uintptr_t(32768), e - a));
        RG_CHK_G(reinterpret_cast<const void*>(a), sz, kChkPrefetch);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    }
}

// Local sort launch. One CTA per SM (8- and 32-B records): persistent, one
// resident CTA per SM, groups assigned round-robin (no atomics). The next group's descriptor is
// copied into shared memory with cp.async while the current group is sorted,
// and once its bucket geometry is known thread 0 prefetches the next group's
// records into L2 (cp.async.bulk.prefetch.L2), so a group's start no longer
// waits on a dependent descriptor load and a cold HBM read.
template <int RS, bool kFallback>
__global__ void __launch_bounds__(LocalCfg<RS>::kThreads, LocalCfg<RS>::kMinBlocks) k_local(
    uint8_t* __restrict__ data, uint8_t* __restrict__ tmp, const Group* __restrict__ groups,
    uint32_t n_groups, uint32_t ks, LevelCounters* __restrict__ ctr, Group* __restrict__ spill,
    unsigned int* __restrict__ n_spill, uint32_t spill_cap, uint32_t ahead) {
    if constexpr (LocalCfg<RS>::kMinBlocks > 1) {
        // two CTAs per SM already overlap one group's start with the other's
        // sort: one group per CTA (measured 4% faster than this loop), the
        // group one resident wave later (ahead = resident CTAs: 2 per SM)
        // prefetched into L2
        if (threadIdx.x == 0 && blockIdx.x + ahead < n_groups)
            prefetch_group_l2<RS>(data, tmp, groups[blockIdx.x + ahead]);
        local_group<RS, kFallback>(data, tmp, groups[blockIdx.x], ks, ctr, spill, n_spill, spill_cap,
                                   [] {});
        return;
    }
    __shared__ __align__(16) Group s_g[2];
    uint32_t i = blockIdx.x;
    if (i >= n_groups) return;
    if (threadIdx.x == 0) s_g[0] = groups[i];
    __syncthreads();
    for (int buf = 0; i < n_groups; buf ^= 1) {
        const uint32_t nx = i + gridDim.x;
        const bool more = nx < n_groups;
        if (threadIdx.x == 0 && more) {
            static_assert(sizeof(Group) % 8 == 0, "Group copied in 8-B pieces");
            for (int q = 0; q < int(sizeof(Group) / 8); ++q)
                cp_async8(reinterpret_cast<uint8_t*>(&s_g[buf ^ 1]) + 8 * q,
                          reinterpret_cast<const uint8_t*>(&groups[nx]) + 8 * q);
        }
        const Group g = s_g[buf];
        auto mid = [&] {
            if (threadIdx.x == 0 && more) {
                cp_async_wait_all();
                prefetch_group_l2<RS>(data, tmp, s_g[buf ^ 1]);
            }
        };
        local_group<RS, kFallback>(data, tmp, g, ks, ctr, spill, n_spill, spill_cap, mid);
        if (threadIdx.x == 0 && more) cp_async_wait_all();
        __syncthreads();  // shared memory free for the next group; its descriptor visible
        i = nx;
    }
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
    if (threadIdx.x == 0) {
        RG_CHK_G(s, uint32_t(bytes), kChkLoad);
        RG_CHK_G(d, uint32_t(bytes), kChkStore);
    }
    if constexpr (RS % 16 == 0) {
        for (uint64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
    } else {
        for (uint64_t i = threadIdx.x; i < bytes / 8; i += blockDim.x)
            reinterpret_cast<uint2*>(d)[i] = reinterpret_cast<const uint2*>(s)[i];
    }
}

}  // namespace rg
