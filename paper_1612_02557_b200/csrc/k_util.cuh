// Device-side generator and verifiers.
//
//   k_gen          — the counter-based input generator of SURVEY.md §8(d), bit
//                    identical to oracle/raduls_oracle.c orc_generate(): key words
//                    big-endian (store_be64, P/include/raduls/layout.hpp:47-49),
//                    payload word 0 = record index (P/src/datagen.cpp:75-80),
//                    mix64 = the splitmix64 finalizer (P/include/raduls/datagen.hpp:37-42).
//   k_digest       — array_digest (P/src/verify.cpp:37-50): order-independent
//                    128-bit sum of per-record hashes.
//   k_check_sorted — check_sorted (P/src/verify.cpp:27-35): count of adjacent
//                    inversions and the first one.
#pragma once

#include "common.cuh"

namespace rg {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t rnd(uint64_t seed, uint64_t i, uint32_t w) {
    return mix64(seed ^ mix64(4 * i + w));
}

__device__ __forceinline__ uint64_t bswap64(uint64_t v) {
    const uint32_t lo = uint32_t(v), hi = uint32_t(v >> 32);
    return (uint64_t(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}

struct GenParams {
    uint64_t n;
    uint64_t seed;
    uint64_t index_base;
    uint32_t ks;
    uint32_t dist;           // 0 uniform, 1 C3 skew (Zipf(1.2) byte under 24 zero bits)
    const unsigned long long* thr;  // [256] Zipf thresholds (dist 1)
};

template <int RS>
__global__ void __launch_bounds__(256) k_gen(uint8_t* __restrict__ out, GenParams P) {
    constexpr int WORDS = RS / 8;
    __shared__ unsigned long long s_thr[256];
    if (P.dist == 1) s_thr[threadIdx.x] = P.thr[threadIdx.x];
    __syncthreads();
    const uint32_t key_words = (P.ks + 7) / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < P.n; j += stride) {
        const uint64_t i = P.index_base + j;
        uint64_t v[WORDS];
#pragma unroll
        for (int w = 0; w < WORDS; ++w) {
            if (uint32_t(w) < key_words) {
                if (P.dist == 1 && w == 0) {
                    const uint64_t u = rnd(P.seed, i, 0) >> 11;
                    // first k with u < thr[k] (thresholds ascending, thr[255] = 2^53)
                    uint32_t lo = 0, hi = 255;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (u < s_thr[mid]) hi = mid; else lo = mid + 1;
                    }
                    v[w] = (uint64_t(lo) << 32) | (rnd(P.seed, i, 1) & 0xFFFFFFFFull);
                } else {
                    v[w] = rnd(P.seed, i, P.dist == 1 ? w + 1 : w);
                }
            } else if (uint32_t(w) == key_words) {
                v[w] = i;
            } else {
                v[w] = mix64(i ^ (0xa5a5a5a5a5a5a5a5ull + uint64_t(w)));
            }
        }
        uint8_t* rec = out + j * RS;
        if constexpr (RS % 16 == 0) {
#pragma unroll
            for (int q = 0; q < WORDS / 2; ++q) {
                const uint64_t a = bswap64(v[2 * q]), b = bswap64(v[2 * q + 1]);
                reinterpret_cast<uint4*>(rec)[q] =
                    make_uint4(uint32_t(a), uint32_t(a >> 32), uint32_t(b), uint32_t(b >> 32));
            }
        } else {
#pragma unroll
            for (int q = 0; q < WORDS; ++q) {
                const uint64_t a = bswap64(v[q]);
                reinterpret_cast<uint2*>(rec)[q] = make_uint2(uint32_t(a), uint32_t(a >> 32));
            }
        }
    }
}

__device__ __forceinline__ uint64_t hash_mix(uint64_t x) {
    x = (x ^ (x >> 33)) * 0xff51afd7ed558ccdull;
    x = (x ^ (x >> 33)) * 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}

// acc[0] = low 64 bits, acc[1] = high 64 bits of the 128-bit digest sum.
template <int RS>
__global__ void __launch_bounds__(256) k_digest(const uint8_t* __restrict__ data, uint64_t n,
                                                unsigned long long* __restrict__ acc) {
    constexpr int WORDS = RS / 8;
    uint64_t lo = 0, hi = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const Rec<RS> r = load_rec_stream<RS>(data, i);
        uint64_t h = 0x8824a3d6f1e2c4b9ull;
#pragma unroll
        for (int w = 0; w < WORDS; ++w) h = hash_mix(h ^ (rec_word64<RS>(r, w) * 0x9ddfea08eb382d69ull));
        const uint64_t l = hash_mix(h ^ 0xc3a5c85c97cb3127ull);
        const uint64_t u = hash_mix(h ^ 0xb492b66fbe98f273ull);
        const uint64_t nl = lo + l;
        hi += u + (nl < lo ? 1 : 0);
        lo = nl;
    }
    // warp reduce 128-bit
    for (int off = 16; off; off >>= 1) {
        const uint64_t ol = __shfl_xor_sync(0xFFFFFFFFu, lo, off);
        const uint64_t oh = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
        const uint64_t nl = lo + ol;
        hi += oh + (nl < lo ? 1 : 0);
        lo = nl;
    }
    if ((threadIdx.x & 31) == 0) {
        const unsigned long long old = atomicAdd(&acc[0], (unsigned long long)lo);
        const uint64_t carry = (old + lo < old) ? 1 : 0;
        atomicAdd(&acc[1], (unsigned long long)(hi + carry));
    }
}

// Big-endian key word w of a record (bytes 8w..8w+7), with bytes at or beyond
// ks cleared.
template <int RS>
__device__ __forceinline__ uint64_t key_word_be(const Rec<RS>& r, int w, uint32_t ks) {
    uint64_t v = bswap64(rec_word64<RS>(r, w));
    const int rem = int(ks) - 8 * w;
    if (rem >= 8) return v;
    if (rem <= 0) return 0;
    return v & (~0ull << (8 * (8 - rem)));
}

// out[0] += number of i with key(i+1) < key(i); out[1] = min such i (init ~0).
template <int RS>
__global__ void __launch_bounds__(256) k_check_sorted(const uint8_t* __restrict__ data, uint64_t n,
                                                      uint32_t ks,
                                                      unsigned long long* __restrict__ out) {
    constexpr int WORDS = RS / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    unsigned long long cnt = 0, first = ~0ull;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i + 1 < n; i += stride) {
        const Rec<RS> a = load_rec<RS>(data, i);
        const Rec<RS> b = load_rec<RS>(data, i + 1);
        int cmp = 0;
#pragma unroll
        for (int w = 0; w < WORDS; ++w) {
            if (cmp == 0) {
                const uint64_t ka = key_word_be<RS>(a, w, ks), kb = key_word_be<RS>(b, w, ks);
                cmp = ka < kb ? -1 : (ka > kb ? 1 : 0);
            }
        }
        if (cmp > 0) {
            ++cnt;
            if (i < first) first = i;
        }
    }
    for (int off = 16; off; off >>= 1) {
        cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
        const unsigned long long f = __shfl_xor_sync(0xFFFFFFFFu, first, off);
        first = f < first ? f : first;
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicAdd(&out[0], cnt);
        atomicMin(&out[1], first);
    }
}

}  // namespace rg
