// C++ caller of the drop-in shim (include/raduls_gpu.hpp), written like the
// reference's own callers (P/src/bench.cpp:30-47 run_algo; P/tests/
// test_scheduler.cpp:16-22 sort_copy): generate records, raduls::gpu::sort,
// verify sortedness + multiset with the library's own checkers.
// Usage: dropin_main <n> <record_size> <key_size> [lsd]   (exit 0 = OK)
// With "lsd": raduls::gpu::lsd_sort (P/include/raduls/lsd.hpp:16-22) instead,
// after checking that bad lane sizes throw (test_lsd.cpp:69-77).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "raduls_gpu.hpp"

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000;
    const uint32_t rs = argc > 2 ? std::atoi(argv[2]) : 16, ks = argc > 3 ? std::atoi(argv[3]) : 8;
    const bool lsd = argc > 4 && std::strcmp(argv[4], "lsd") == 0;
    raduls::gpu::RecordLayout layout{rs, ks};
    std::vector<uint8_t> data(n * rs);
    std::mt19937_64 eng(42);
    for (auto& b : data) b = uint8_t(eng());
    // bad layouts throw std::invalid_argument before touching the data
    try {
        raduls::gpu::sort(data.data(), n, raduls::gpu::RecordLayout{8, 16});
        std::puts("FAIL: invalid layout accepted");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    if (lsd) {
        for (size_t lane : {size_t(63), size_t(0)}) {
            try {
                raduls::gpu::lsd_sort(data.data(), n, layout, raduls::gpu::LsdConfig{lane, 1});
                std::puts("FAIL: bad LSD lane size accepted");
                return 1;
            } catch (const std::invalid_argument&) {
            }
        }
    }
    std::vector<uint8_t> before = data;
    if (lsd)
        raduls::gpu::lsd_sort(data.data(), n, layout, raduls::gpu::LsdConfig{256, 4});
    else
        raduls::gpu::sort(data.data(), n, layout);
    for (size_t i = 0; i + 1 < n; ++i)
        if (std::memcmp(&data[i * rs], &data[(i + 1) * rs], ks) > 0) {
            std::printf("FAIL: inversion at %zu\n", i);
            return 1;
        }
    // same multiset: order-independent digest (verify.cpp:37-50 restated)
    uint64_t lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
    std::vector<uint8_t>* bufs[2] = {&before, &data};
    uint64_t* out[2][2] = {{&lo0, &hi0}, {&lo1, &hi1}};
    for (int k = 0; k < 2; ++k) {
        // host-side digest restated as in verify.cpp:37-50
        unsigned __int128 acc = 0;
        for (size_t i = 0; i < n; ++i) {
            uint64_t h = 0x8824a3d6f1e2c4b9ULL;
            for (uint32_t w = 0; w < rs / 8; ++w) {
                uint64_t v;
                std::memcpy(&v, &(*bufs[k])[i * rs + 8 * w], 8);
                uint64_t x = h ^ (v * 0x9ddfea08eb382d69ULL);
                x = (x ^ (x >> 33)) * 0xff51afd7ed558ccdULL;
                x = (x ^ (x >> 33)) * 0xc4ceb9fe1a85ec53ULL;
                h = x ^ (x >> 33);
            }
            auto mix = [](uint64_t x) {
                x = (x ^ (x >> 33)) * 0xff51afd7ed558ccdULL;
                x = (x ^ (x >> 33)) * 0xc4ceb9fe1a85ec53ULL;
                return x ^ (x >> 33);
            };
            acc += ((unsigned __int128)mix(h ^ 0xb492b66fbe98f273ULL) << 64) | mix(h ^ 0xc3a5c85c97cb3127ULL);
        }
        *out[k][0] = uint64_t(acc);
        *out[k][1] = uint64_t(acc >> 64);
    }
    if (lo0 != lo1 || hi0 != hi1) {
        std::puts("FAIL: multiset changed");
        return 1;
    }
    std::printf("OK n=%zu rs=%u ks=%u\n", n, rs, ks);
    return 0;
}
