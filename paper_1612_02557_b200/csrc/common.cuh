// Shared device-side definitions for the B200 MSD record sort.
//
// Record model (reference P/include/raduls/layout.hpp:1-81, P = /root/reference/proj):
//   * a record is RS bytes (RS in {8,16,24,32}), key = its first `ks` bytes,
//     most significant byte first; key order == memcmp order (layout.hpp:52-55);
//   * the MSD digit processed at "byte position" p is record byte p, i.e. the
//     reference's digit(rec, ks-1-p) (layout.hpp:32-39).
// Records move as whole 8/16-byte vectors (copy_record, layout.hpp:70-73).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rg {

constexpr int kRadix = 256;

// ---------------------------------------------------------------- record vectors

// A record held in registers as RS/4 little-endian 32-bit words.
template <int RS>
struct Rec {
    static_assert(RS % 8 == 0 && RS >= 8 && RS <= 32, "record size");
    static constexpr int kWords = RS / 4;
    uint32_t w[kWords];
};

// ---------------------------------------------------------------- checked build
//
// RG_CHECKED (python -m paper_1612_02557_b200.build --checked ->
// libraduls_gpu_checked.so): the stand-in for compute-sanitizer, which this
// GPU pool does not run. Every global record access (vector loads/stores,
// TMA bulk copies and L2 prefetches, digit-array stores) is checked against
// the device ranges the current call registered (its data, tmp, digit arrays,
// destinations); TMA copies also for the 16-B alignment the hardware needs.
// mbarrier waits are bounded (a deadlock is counted instead of hanging the
// GPU); dynamic shared memory and the scratch buffers are poisoned (0xA5)
// before use, so a read of anything not written first changes the output;
// and with jitter on, random __nanosleep at every producer/consumer hand-off
// perturbs warp interleavings so an ordering race shows up as a parity
// failure. The C-ABI returns RADULS_GPU_EINTERNAL from any call that
// recorded a violation (raduls_gpu_check_report has the details).
#ifdef RG_CHECKED
constexpr unsigned int kChkRanges = 1024;
struct ChkState {
    unsigned long long fails, first_addr, deadlocks;
    unsigned int first_site, first_bytes;
    unsigned int n, jitter;
    unsigned long long lo[kChkRanges], hi[kChkRanges];  // sorted by lo, disjoint (merged on the host)
};
__device__ ChkState g_chk;

__device__ __noinline__ void chk_fail(uint32_t site, const void* p, uint32_t bytes) {
    if (atomicAdd(&g_chk.fails, 1ull) == 0) {
        g_chk.first_addr = reinterpret_cast<unsigned long long>(p);
        g_chk.first_site = site;
        g_chk.first_bytes = bytes;
    }
}

__device__ __forceinline__ void chk_global(const void* p, uint32_t bytes, uint32_t site) {
    const uint32_t n = *(volatile unsigned int*)&g_chk.n;
    if (n == 0 || !__isGlobal(p)) return;
    const unsigned long long a = reinterpret_cast<unsigned long long>(p);
    uint32_t l = 0, h = n;  // the last range starting at or below a
    while (h - l > 1) {
        const uint32_t m = (l + h) >> 1;
        if (g_chk.lo[m] <= a) l = m;
        else h = m;
    }
    if (g_chk.lo[l] <= a && a + bytes <= g_chk.hi[l]) return;
    chk_fail(site, p, bytes);
}

__device__ __forceinline__ void chk_jitter() {
    if (*(volatile unsigned int*)&g_chk.jitter) {
        unsigned long long h = clock64() ^ (uint64_t(blockIdx.x) << 20) ^ threadIdx.x;
        h *= 0x9E3779B97F4A7C15ull;
        __nanosleep(uint32_t(h >> 54));  // 0-1023 ns
    }
}

__device__ __forceinline__ void chk_poison_smem(uint8_t* smem) {
    uint32_t sz;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(sz));
    for (uint32_t i = threadIdx.x * 4u; i + 4u <= sz; i += blockDim.x * 4u)
        *reinterpret_cast<uint32_t*>(smem + i) = 0xA5A5A5A5u;
    __syncthreads();
}
#define RG_CHK_G(p, bytes, site) ::rg::chk_global((p), (bytes), (site))
#define RG_CHK_JITTER() ::rg::chk_jitter()
#define RG_CHK_POISON_SMEM(smem) ::rg::chk_poison_smem(smem)
#else
#define RG_CHK_G(p, bytes, site) ((void)0)
#define RG_CHK_JITTER() ((void)0)
#define RG_CHK_POISON_SMEM(smem) ((void)0)
#endif
// check sites (raduls_gpu_check_report)
enum : uint32_t {
    kChkLoad = 1, kChkLoadStream = 2, kChkStore = 3, kChkStoreHint = 4, kChkTmaSrc = 5, kChkTmaAlign = 6,
    kChkDigitStore = 7, kChkPrefetch = 8
};

template <int RS>
__device__ __forceinline__ Rec<RS> load_rec(const uint8_t* base, uint64_t idx) {
    Rec<RS> r;
    const uint8_t* p = base + idx * RS;
    RG_CHK_G(p, RS, kChkLoad);
    if constexpr (RS % 16 == 0) {
#pragma unroll
        for (int v = 0; v < RS / 16; ++v) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(p) + v);
            r.w[4 * v + 0] = q.x;
            r.w[4 * v + 1] = q.y;
            r.w[4 * v + 2] = q.z;
            r.w[4 * v + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int v = 0; v < RS / 8; ++v) {
            const uint2 q = __ldg(reinterpret_cast<const uint2*>(p) + v);
            r.w[2 * v + 0] = q.x;
            r.w[2 * v + 1] = q.y;
        }
    }
    return r;
}

// Same, but through L1-bypassing loads: for buffers written by an earlier
// kernel in the same sort (no stale-L1 issue across launches, but keeps the
// streaming data out of L1).
template <int RS>
__device__ __forceinline__ Rec<RS> load_rec_stream(const uint8_t* base, uint64_t idx) {
    Rec<RS> r;
    const uint8_t* p = base + idx * RS;
    RG_CHK_G(p, RS, kChkLoadStream);
    if constexpr (RS % 16 == 0) {
#pragma unroll
        for (int v = 0; v < RS / 16; ++v) {
            uint4 q;
            asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                         : "l"(reinterpret_cast<const uint4*>(p) + v));
            r.w[4 * v + 0] = q.x;
            r.w[4 * v + 1] = q.y;
            r.w[4 * v + 2] = q.z;
            r.w[4 * v + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int v = 0; v < RS / 8; ++v) {
            uint2 q;
            asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                         : "=r"(q.x), "=r"(q.y)
                         : "l"(reinterpret_cast<const uint2*>(p) + v));
            r.w[2 * v + 0] = q.x;
            r.w[2 * v + 1] = q.y;
        }
    }
    return r;
}

template <int RS>
__device__ __forceinline__ void store_rec(uint8_t* base, uint64_t idx, const Rec<RS>& r) {
    uint8_t* p = base + idx * RS;
    RG_CHK_G(p, RS, kChkStore);
    if constexpr (RS % 16 == 0) {
#pragma unroll
        for (int v = 0; v < RS / 16; ++v)
            reinterpret_cast<uint4*>(p)[v] =
                make_uint4(r.w[4 * v], r.w[4 * v + 1], r.w[4 * v + 2], r.w[4 * v + 3]);
    } else {
#pragma unroll
        for (int v = 0; v < RS / 8; ++v)
            reinterpret_cast<uint2*>(p)[v] = make_uint2(r.w[2 * v], r.w[2 * v + 1]);
    }
}

// Shared-memory record slots (same vector widths).
template <int RS>
__device__ __forceinline__ void st_smem_rec(uint8_t* s, uint32_t slot, const Rec<RS>& r) {
    store_rec<RS>(s, slot, r);
}

#ifndef RG_LD32_ALT
#define RG_LD32_ALT 1
#endif
template <int RS, bool kAlt = true>
__device__ __forceinline__ Rec<RS> ld_smem_rec(const uint8_t* s, uint32_t slot) {
    Rec<RS> r;
    const uint8_t* p = s + size_t(slot) * RS;
    if constexpr (RS == 32 && RG_LD32_ALT && kAlt) {
        // 32-B records: lanes of consecutive slots load the first half in
        // groups of four and the second half in the next four, so each 16-B
        // load instruction covers all eight 16-B bank groups of a quarter-warp
        // (plain order: two-way conflicts at the 32-B stride)
        const uint32_t h = (slot >> 2) & 1u;
        const uint4 q0 = reinterpret_cast<const uint4*>(p)[h];
        const uint4 q1 = reinterpret_cast<const uint4*>(p)[h ^ 1u];
        const uint4 a = h ? q1 : q0, b = h ? q0 : q1;
        r.w[0] = a.x, r.w[1] = a.y, r.w[2] = a.z, r.w[3] = a.w;
        r.w[4] = b.x, r.w[5] = b.y, r.w[6] = b.z, r.w[7] = b.w;
        return r;
    }
    if constexpr (RS % 16 == 0) {
#pragma unroll
        for (int v = 0; v < RS / 16; ++v) {
            const uint4 q = reinterpret_cast<const uint4*>(p)[v];
            r.w[4 * v + 0] = q.x;
            r.w[4 * v + 1] = q.y;
            r.w[4 * v + 2] = q.z;
            r.w[4 * v + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int v = 0; v < RS / 8; ++v) {
            const uint2 q = reinterpret_cast<const uint2*>(p)[v];
            r.w[2 * v + 0] = q.x;
            r.w[2 * v + 1] = q.y;
        }
    }
    return r;
}

// 32-bit word `wi` (runtime, warp-uniform) of a register-held record via a
// binary tree of selects on the bits of wi — written so that the compiler
// cannot turn it back into a dynamically indexed (local-memory) array access.
template <int LO, int N, int RS>
__device__ __forceinline__ uint32_t rec_word_tree(const Rec<RS>& r, uint32_t wi) {
    if constexpr (N == 1) {
        return r.w[LO];
    } else {
        constexpr int H = N / 2;
        const uint32_t a = rec_word_tree<LO, H, RS>(r, wi);
        const uint32_t b = rec_word_tree<LO + H, N - H, RS>(r, wi);
        return wi < uint32_t(LO + H) ? a : b;
    }
}

template <int RS>
__device__ __forceinline__ uint32_t rec_word32(const Rec<RS>& r, uint32_t wi) {
    return rec_word_tree<0, Rec<RS>::kWords, RS>(r, wi);
}

// Record byte `p` (runtime, warp-uniform) from a register-held record.
template <int RS>
__device__ __forceinline__ uint32_t rec_byte(const Rec<RS>& r, uint32_t p) {
    return (rec_word32<RS>(r, p >> 2) >> ((p & 3u) * 8u)) & 0xFFu;
}

// Big-endian window of up to four record bytes L0 < L1 < L2 < L3 that all lie
// in the 32-bit words q, q+1 (always true for 8-B records with q = 0): one
// byte permute instead of four byte extractions. `sel`/`mask` come from
// make_window_sel; the selector picks (L0, L1, L2, L3) into bytes (3, 2, 1, 0).
template <bool B>
struct BoolC {
    static constexpr bool value = B;
};

template <int V>
struct IntC {
    static constexpr int value = V;
};

struct WindowSel {
    uint32_t q, sel, mask;
    bool fast;
};
__device__ __forceinline__ WindowSel make_window_sel(const uint32_t* L, uint32_t nwin,
                                                     uint32_t rs_words, bool force_q0) {
    WindowSel s;
    s.q = force_q0 ? 0u : (L[0] >> 2);
    if (s.q + 1 >= rs_words && rs_words >= 2) s.q = rs_words - 2;
    s.sel = 0;
    s.fast = true;
    for (uint32_t k = 0; k < nwin; ++k) {
        const uint32_t rel = L[k] - 4 * s.q;
        if (rel >= 8) s.fast = false;
        s.sel |= (rel & 7u) << (4 * (3 - k));
    }
    s.mask = nwin >= 4 ? 0xFFFFFFFFu : (0xFFFFFFFFu << (8 * (4 - nwin)));
    return s;
}
template <int RS>
__device__ __forceinline__ uint32_t rec_window(const Rec<RS>& r, const WindowSel& s) {
    if constexpr (RS == 8) return __byte_perm(r.w[0], r.w[1], s.sel) & s.mask;
    else
        return __byte_perm(rec_word32<RS>(r, s.q), rec_word32<RS>(r, s.q + 1), s.sel) & s.mask;
}

// Little-endian 64-bit word k (record bytes 8k..8k+7).
template <int RS>
__device__ __forceinline__ uint64_t rec_word64(const Rec<RS>& r, int k) {
    return uint64_t(r.w[2 * k]) | (uint64_t(r.w[2 * k + 1]) << 32);
}

// ---------------------------------------------------------------- misc

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// ---------------------------------------------------------------- TMA / mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Orders this thread's earlier generic-proxy shared-memory accesses (made
// visible to it by a preceding __syncthreads) before its next async-proxy
// (TMA) write into the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// 1-D TMA bulk copy global -> shared (16-B aligned addresses, size % 16 == 0),
// completion signalled as transaction bytes on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            unsigned long long* bar) {
    RG_CHK_G(src, bytes, kChkTmaSrc);
#ifdef RG_CHECKED
    if ((smem_u32(dst) | uint32_t(reinterpret_cast<uintptr_t>(src)) | bytes) & 15u) chk_fail(kChkTmaAlign, src, bytes);
#endif
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// The same with an L2 eviction-priority hint (kHint 0: none; 1: evict_first,
// for streams read once, so they leave L2 before the scatter's half-written
// destination lines).
template <int kHint>
__device__ __forceinline__ void tma_load_1d_h(void* dst, const void* src, uint32_t bytes,
                                              unsigned long long* bar) {
    if constexpr (kHint == 0) {
        tma_load_1d(dst, src, bytes, bar);
    } else {
        RG_CHK_G(src, bytes, kChkTmaSrc);
#ifdef RG_CHECKED
        if ((smem_u32(dst) | uint32_t(reinterpret_cast<uintptr_t>(src)) | bytes) & 15u)
            chk_fail(kChkTmaAlign, src, bytes);
#endif
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(dst)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
            : "memory");
    }
}

#ifndef RG_HINT_SC
#define RG_HINT_SC 0
#endif
#ifndef RG_HINT_HIST
#define RG_HINT_HIST 1
#endif
#ifndef RG_HINT_SCST
#define RG_HINT_SCST 2
#endif

// Record store with an L2 eviction-priority hint (1: evict_first, 2: evict_last).
template <int RS, int kHint>
__device__ __forceinline__ void store_rec_h(uint8_t* base, uint64_t idx, const Rec<RS>& r) {
    if constexpr (kHint == 0 || RS % 16 != 0) {
        store_rec<RS>(base, idx, r);
    } else {
        uint64_t pol;
        if constexpr (kHint == 1)
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        else
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        uint8_t* p = base + idx * RS;
        RG_CHK_G(p, RS, kChkStoreHint);
#pragma unroll
        for (int v = 0; v < RS / 16; ++v)
            asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p + 16 * v),
                         "r"(r.w[4 * v]), "r"(r.w[4 * v + 1]), "r"(r.w[4 * v + 2]), "r"(r.w[4 * v + 3]),
                         "l"(pol)
                         : "memory");
    }
}
#ifndef RG_HINT_LOCAL
#define RG_HINT_LOCAL 0
#endif

// Asynchronous global -> shared copy of 8 bytes (LDGSTS, no register round
// trip); cp_async_wait_all() completes this thread's outstanding copies.
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok = 0;
    RG_CHK_JITTER();
#ifdef RG_CHECKED
    uint32_t spins = 0;
#endif
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(phase)
            : "memory");
#ifdef RG_CHECKED
        if (!ok && ++spins == (1u << 22)) {  // seconds: a lost arrival or transaction
            atomicAdd(&g_chk.deadlocks, 1ull);
            return;
        }
#endif
    } while (!ok);
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named barrier over the first `nthreads` threads (consumer warps only).
__device__ __forceinline__ void bar_sync_named(uint32_t id, uint32_t nthreads) {
    RG_CHK_JITTER();
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warp multisplit peer mask for an 8-bit digit: lanes of this warp holding the
// same digit (valid lanes only). Eight ballots instead of MATCH.ANY, whose
// result latency dominated the first profile (ncu: short_sb stalls on the
// BREV consuming it, profiles/r1_local_sort_match.txt).
__device__ __forceinline__ uint32_t match_digit8(uint32_t d, bool valid) {
    uint32_t m = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bit);
        m &= bit ? bal : ~bal;
    }
    return m;
}

// Stable in-warp rank of digit d: the number of this warp's earlier items
// (earlier calls, then lower lanes of this call) holding d. `cnt` is the
// warp's private 256-entry counter table. Every lane of the warp calls it.
//   kMode 0: one shared-memory atomic per item. Ranks follow lane order only
//            if the hardware serves the conflicting lanes of one atomic in
//            lane order, which PTX does not promise: the library runs it only
//            after k_rank_selftest has checked that behaviour on the device
//            (else it uses kMode 1). Measured C5 scatter 73.6 ms vs 94.7 ms
//            with kMode 1 and 110.2 ms with kMode 2 (same box, interleaved);
//   kMode 1: peers from eight ballots (match_digit8), rank = counter +
//            popc(peers & lanemask_lt), the highest peer lane advances the
//            counter (stable by construction);
//   kMode 2: the same with MATCH.ANY for the peer mask.
template <int kMode>
__device__ __forceinline__ uint32_t warp_rank(uint32_t* cnt, uint32_t d, bool valid) {
    if constexpr (kMode == 0) {
        return valid ? atomicAdd(&cnt[d], 1u) : 0u;
    } else {
        uint32_t peers;
        if constexpr (kMode == 1) {
            peers = match_digit8(d, valid);
        } else {
            peers = __match_any_sync(0xFFFFFFFFu, valid ? d : 0x100u);
            if (!valid) peers = 0;
        }
        const uint32_t before = valid ? cnt[d] : 0u;
        __syncwarp();
        if (valid && lane_id() == 31u - __clz(peers)) cnt[d] = before + __popc(peers);
        __syncwarp();
        return before + __popc(peers & lanemask_lt());
    }
}

// Device check of what kMode 0 relies on (run once per device before the first
// sort): every warp ranks pseudo-random digit streams -- all lanes equal, 2-64
// distinct values, alternating patterns -- with kMode 0 and kMode 1 on two
// private counter tables; any rank that differs sets *bad.
__global__ void __launch_bounds__(256) k_rank_selftest(uint32_t rounds, unsigned int* __restrict__ bad) {
    __shared__ uint32_t t0[8][256], t1[8][256];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint32_t q = lane; q < 256; q += 32) t0[warp][q] = t1[warp][q] = 0;
    __syncwarp();
    uint32_t diff = 0;
    for (uint32_t it = 0; it < rounds; ++it) {
        uint32_t h = (it * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^ (warp * 0xC2B2AE35u) ^ (lane * 0x27D4EB2Fu);
        h ^= h >> 15;
        h *= 0x2C1B3C6Du;
        h ^= h >> 12;
        const uint32_t kind = it % 8;
        uint32_t d;
        if (kind == 0) d = it & 0xFFu;                        // all lanes one digit
        else if (kind == 1) d = (lane & 1u) ? 7u : 200u;      // alternating
        else if (kind == 2) d = lane < 16 ? 3u : 250u;        // halves
        else d = (h >> 8) % (2u << kind) * 37u & 0xFFu;       // 4..256 distinct values
        const bool valid = kind != 7 || (h & 7u) != 0;        // some lanes idle
        const uint32_t r0 = warp_rank<0>(&t0[warp][0], d, valid);
        const uint32_t r1 = warp_rank<1>(&t1[warp][0], d, valid);
        diff |= valid && r0 != r1;
        if ((it & 255u) == 255u) {  // keep the counters small
            __syncwarp();
            for (uint32_t q = lane; q < 256; q += 32) t0[warp][q] = t1[warp][q] = 0;
            __syncwarp();
        }
    }
    if (__any_sync(0xFFFFFFFFu, diff) && lane == 0) atomicOr(bad, 1u);
}

// Multi-GPU partition digits --------------------------------
//
// The map buffer: map[b] (b < 65536) = digit of the 16-bit key prefix at bytes
// (p, p+1); map[kMapPivotSlot + d] = pivot slot + 1 when digit d is a hot
// bucket cut around a pivot key (0 otherwise); the pivot keys (kMaxPivots x 32
// B, the key's first ks bytes) follow. A record of a pivot digit gets digit
// d, d + 1 or d + 2 for a key below, equal to or above the pivot (memcmp
// order, P/include/raduls/layout.hpp:52-55): the equal run holds one key, so
// the plan may spread it over ranks by count.
constexpr uint32_t kMapPivotSlot = 65536;
constexpr uint32_t kMaxPivots = 16;
constexpr uint32_t kMapPivotKeys = kMapPivotSlot + 256;
constexpr uint32_t kMapBytes = kMapPivotKeys + kMaxPivots * 32;

// byte_at(i): key byte i of the record (any i < ks).
template <typename ByteAt>
__device__ __forceinline__ uint32_t map_digit(ByteAt byte_at, uint32_t p, uint32_t ks,
                                              const uint8_t* __restrict__ map) {
    const uint32_t hi = p < ks ? byte_at(p) : 0u;
    const uint32_t lo = p + 1 < ks ? byte_at(p + 1) : 0u;
    const uint32_t d = __ldg(map + ((hi << 8) | lo));
    const uint32_t pv = __ldg(map + kMapPivotSlot + d);
    if (pv == 0) return d;
    const uint8_t* key = map + kMapPivotKeys + (pv - 1) * 32u;
    for (uint32_t b = 0; b < ks; ++b) {
        const uint32_t x = byte_at(b), y = __ldg(key + b);
        if (x != y) return x < y ? d : d + 2;
    }
    return d + 1;
}

// Device segment descriptors -------------------------------------------------

// A contiguous run of records [start, start+size) that still needs ordering by
// key bytes >= p; `parity` says which working buffer holds it (0: caller's
// data, 1: tmp). Mirrors the reference's Bin (P/include/raduls/kernels.hpp:60-67)
// with the digit expressed as a record byte offset.
struct Seg {
    uint64_t start;
    uint64_t size;
    uint32_t p;
    uint32_t parity;
    uint32_t tile_base;  // first tile (histogram + scatter partition) of this segment
    uint32_t action;     // set by the planner: kActScatter when this level splits it
};

constexpr uint32_t kActScatter = 2;

// A run of one or more complete, adjacent small segments sorted by one CTA;
// all its records share key bytes [0, p).
struct Group {
    uint64_t start;
    uint32_t size;
    uint32_t p;
    uint32_t parity;
    uint32_t pad;  // 0, or d0 | d1 << 8 | 1 << 16: key byte p of every record lies in [d0, d1]
};

// A range of finished records living in tmp that must move home.
struct CopyRange {
    uint64_t start;
    uint32_t size;
    uint32_t pad;
};

// Per-level counters (device, zeroed before the planner runs).
struct LevelCounters {
    uint32_t n_groups;         // local-sort groups emitted
    uint32_t n_copy;           // copy-back ranges emitted
    uint32_t n_next;           // next-level segments
    uint32_t n_next_tiles;     // tiles of next-level segments
    uint32_t n_scatter_segs;   // segments scattered this level
    uint32_t scan_ticket;      // dynamic chunk id dispenser for k_tile_scan
    uint32_t scatter_ticket;   // in-order tile dispenser for k_scatter
    uint32_t hist_ticket;      // in-order tile dispenser for k_tile_hist
    unsigned long long moved_scatter;    // records moved by this level's scatter
    unsigned long long moved_local;      // records moved by local sorts
    unsigned long long moved_copy;       // records moved by copy-back
    unsigned long long fallback_groups;  // local-sort groups that needed the LSD fallback
    unsigned long long hist_records;     // records read by this level's tile histogram
    unsigned long long hist_digit_records;  // records histogrammed from the digit array (1 byte each)
    uint32_t n_skip;                     // segments re-queued at a later byte without a split
    uint32_t bm_spill;                   // groups the bitmap local sort handed to the bucket sort
    uint32_t n_big_groups;               // groups above the bitmap sort's primary capacity (single bins)
    uint32_t pad;
};

// Decoupled look-back status word: [63:62] flag, [61:0] value.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagIncl = 2ull << 62;
constexpr uint64_t kValueMask = (1ull << 62) - 1;

}  // namespace rg
