// C++ caller of the drop-in shim (include/raduls_gpu.hpp), written like the
// reference's own callers: run_algo below has the shape of the reference
// bench's dispatcher (P/src/bench.cpp:32-47) with only the namespace switched
// to raduls::gpu; the RecordArray overload and a SchedulerConfig carrying a
// TinyPolicy are used as P/tests/test_scheduler.cpp:16-22 does. Generates
// records, sorts, verifies sortedness + multiset with a host digest.
// Usage: dropin_main <n> <record_size> <key_size> [raduls|lsd1|lsd4]   (exit 0 = OK)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "raduls_gpu.hpp"

using namespace raduls::gpu;  // the one line a reference caller changes

struct BenchRequest {  // the two fields run_algo reads (P/src/bench.hpp)
    size_t l2_bytes = 262144;
    size_t buffer_bytes = 256;
};

static void run_algo(const std::string& algo, uint8_t* data, size_t n, const RecordLayout& layout,
                     unsigned threads, const BenchRequest& req) {
    if (algo == "raduls") {
        SchedulerConfig cfg;
        cfg.threads = threads;
        cfg.l2_cache_bytes = req.l2_bytes;
        cfg.buffer_bytes = req.buffer_bytes;
        sort(data, n, layout, cfg);
    } else if (algo == "lsd1") {
        lsd_sort(data, n, layout, LsdConfig{64, threads});
    } else if (algo == "lsd4") {
        lsd_sort(data, n, layout, LsdConfig{256, threads});
    } else {
        throw std::invalid_argument("unknown algorithm: " + algo);
    }
}

static bool sorted_by_key(const uint8_t* d, size_t n, uint32_t rs, uint32_t ks) {
    for (size_t i = 0; i + 1 < n; ++i)
        if (std::memcmp(d + i * rs, d + (i + 1) * rs, ks) > 0) {
            std::printf("FAIL: inversion at %zu\n", i);
            return false;
        }
    return true;
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000;
    const uint32_t rs = argc > 2 ? std::atoi(argv[2]) : 16, ks = argc > 3 ? std::atoi(argv[3]) : 8;
    const std::string algo = argc > 4 ? argv[4] : "raduls";
    const bool lsd = algo != "raduls";
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
    run_algo(algo, data.data(), n, layout, 4, BenchRequest{});
    if (!sorted_by_key(data.data(), n, rs, ks)) return 1;
    // RecordArray overload (scheduler.hpp:63-65), a config with a TinyPolicy
    {
        RecordArray arr(layout, n);
        std::memcpy(arr.data(), before.data(), arr.byte_size());
        if (reinterpret_cast<uintptr_t>(arr.data()) % 64) {
            std::puts("FAIL: RecordArray storage not 64-B aligned");
            return 1;
        }
        SchedulerConfig cfg;
        cfg.tiny.tiny_threshold = 100;
        cfg.tiny.intro_vs_shell_override = 50;
        sort(arr, cfg);
        if (std::memcmp(arr.data(), data.data(), arr.byte_size()) != 0) {
            std::puts("FAIL: RecordArray sort differs from the pointer sort");
            return 1;
        }
        RecordArray c = arr.clone();
        if (c.size() != n || std::memcmp(c.data(), arr.data(), c.byte_size()) != 0) {
            std::puts("FAIL: RecordArray clone");
            return 1;
        }
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
