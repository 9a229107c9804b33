// raduls_gpu.hpp — C++ drop-in for the reference's public sort API on top of
// the C-ABI in raduls_gpu.h (header-only; link with -lraduls_gpu).
//
// Mirrors, name for name:
//   struct raduls::RecordLayout        /root/reference/proj/include/raduls/layout.hpp:16-28
//   struct raduls::SchedulerConfig     /root/reference/proj/include/raduls/scheduler.hpp:23-32
//   raduls::sort(uint8_t*, size_t, const RecordLayout&, const SchedulerConfig&)
//                                      /root/reference/proj/include/raduls/scheduler.hpp:60-61
//   raduls::resource_error             /root/reference/proj/include/raduls/errors.hpp:12-22
//   struct raduls::LsdConfig, raduls::lsd_sort(uint8_t*, size_t, const RecordLayout&, const LsdConfig&)
//                                      /root/reference/proj/include/raduls/lsd.hpp:12-22
// inside namespace raduls::gpu, so a caller switches implementations by
// changing the namespace (e.g. the reference bench's run_algo, bench.cpp:30-47,
// gains an "raduls_gpu" case calling raduls::gpu::sort). Error mapping:
// RADULS_GPU_EINVAL -> std::invalid_argument (dispatch.hpp:37-39),
// RADULS_GPU_ENOMEM -> resource_error, anything else -> std::runtime_error.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "raduls_gpu.h"

namespace raduls::gpu {

struct RecordLayout {
    uint32_t record_size = 16;  // 8, 16, 24 or 32
    uint32_t key_size = 8;      // 1..record_size (the reference: 8 or 16)
    constexpr uint32_t payload_size() const { return record_size - key_size; }
    bool valid() const { return raduls_gpu_layout_valid(record_size, key_size) != 0; }
};

struct BigBinFraction {
    uint32_t num = 2;
    uint32_t den = 3;
};

// Accepted for signature compatibility. The reference's knobs steer CPU thread
// scheduling and never change the sorted content (test_scheduler.cpp:171-177);
// the GPU planner ignores them.
struct SchedulerConfig {
    unsigned threads = 1;
    size_t l2_cache_bytes = 262144;
    BigBinFraction big_bin_threshold{};
    size_t queue_cutoff_divisor = 4096;
    unsigned chunk_multiplier = 8;
    unsigned first_chunk_divisor = 64;
    size_t buffer_bytes = 256;
};

struct resource_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void throw_on_error(int rc, const char* what) {
    if (rc == RADULS_GPU_OK) return;
    const std::string msg = std::string(what) + ": " + raduls_gpu_strerror(rc);
    if (rc == RADULS_GPU_EINVAL) throw std::invalid_argument(msg);
    if (rc == RADULS_GPU_ENOMEM) throw resource_error(msg);
    throw std::runtime_error(msg);
}

// Host-memory drop-in: sorts n records of `data` in place (H2D -> device sort -> D2H).
inline void sort(uint8_t* data, size_t n, const RecordLayout& layout,
                 const SchedulerConfig& /*cfg*/ = {}) {
    if (!layout.valid())
        throw std::invalid_argument("unsupported record layout: record_size=" +
                                    std::to_string(layout.record_size) +
                                    " key_size=" + std::to_string(layout.key_size));
    throw_on_error(raduls_gpu_sort_host(data, nullptr, n, layout.record_size, layout.key_size),
                   "raduls_gpu_sort_host");
}

// LSD baseline (lsd.hpp:12-22). The lane size must be a positive multiple of 64
// as in the reference (lsd.cpp:13-14); it and `threads` steer the CPU scatter only.
struct LsdConfig {
    size_t buffer_bytes_per_digit = 64;
    unsigned threads = 1;
};

inline void lsd_sort(uint8_t* data, size_t n, const RecordLayout& layout, const LsdConfig& cfg = {}) {
    if (cfg.buffer_bytes_per_digit == 0 || cfg.buffer_bytes_per_digit % 64 != 0)
        throw std::invalid_argument("LSD buffer size must be a positive multiple of 64 bytes");
    if (!layout.valid())
        throw std::invalid_argument("unsupported record layout: record_size=" +
                                    std::to_string(layout.record_size) +
                                    " key_size=" + std::to_string(layout.key_size));
    throw_on_error(raduls_gpu_lsd_sort_host(data, nullptr, n, layout.record_size, layout.key_size),
                   "raduls_gpu_lsd_sort_host");
}

// Device-resident variant: d_data/d_tmp are device pointers (d_tmp may be null).
inline void sort_device(void* d_data, void* d_tmp, size_t n, const RecordLayout& layout,
                        void* stream = nullptr) {
    throw_on_error(raduls_gpu_sort(d_data, d_tmp, n, layout.record_size, layout.key_size, stream),
                   "raduls_gpu_sort");
}

}  // namespace raduls::gpu
