// raduls_gpu.hpp — C++ drop-in for the reference's public sort API on top of
// the C-ABI in raduls_gpu.h (header-only; link with -lraduls_gpu).
//
// Mirrors, name for name:
//   struct raduls::RecordLayout        /root/reference/proj/include/raduls/layout.hpp:16-28
//   struct raduls::TinyPolicy          /root/reference/proj/include/raduls/small_sorts.hpp:14-25
//   struct raduls::SchedulerConfig     /root/reference/proj/include/raduls/scheduler.hpp:23-32
//   raduls::sort(uint8_t*, size_t, const RecordLayout&, const SchedulerConfig&)
//                                      /root/reference/proj/include/raduls/scheduler.hpp:60-61
//   raduls::sort(RecordArray&, const SchedulerConfig&)
//                                      /root/reference/proj/include/raduls/scheduler.hpp:63-65
//   class raduls::RecordArray, allocate_record_bytes
//                                      /root/reference/proj/include/raduls/record_array.hpp:15-61
//   raduls::resource_error             /root/reference/proj/include/raduls/errors.hpp:12-22
//   struct raduls::LsdConfig, raduls::lsd_sort(uint8_t*, size_t, const RecordLayout&, const LsdConfig&)
//                                      /root/reference/proj/include/raduls/lsd.hpp:12-22
// inside namespace raduls::gpu, so a caller switches implementations by
// changing the namespace (e.g. the reference bench's run_algo, bench.cpp:30-47,
// gains an "raduls_gpu" case calling raduls::gpu::sort). Error mapping:
// RADULS_GPU_EINVAL -> std::invalid_argument (dispatch.hpp:37-39),
// RADULS_GPU_ENOMEM -> resource_error, anything else -> std::runtime_error.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <memory>
#include <new>
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

// The reference's tiny-bin policy (which comparison sort finishes a bin).
// Accepted and ignored like the scheduler knobs: the GPU's small-bin sort is
// stable and its output does not depend on it.
struct TinyPolicy {
    size_t tiny_threshold = 384;
    size_t insertion_threshold = 32;
    size_t narrowing_factor_limit = 16;
    size_t narrowed_tiny_threshold = 32;
    size_t intro_vs_shell_override = 0;  // 0: derive from the key size

    size_t intro_vs_shell_threshold(size_t key_size) const {
        if (intro_vs_shell_override) return intro_vs_shell_override;
        return std::clamp<size_t>(100 + 5 * key_size, 100, 180);
    }
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
    TinyPolicy tiny{};
};

struct resource_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// 64-B aligned owning record storage (record_array.hpp:15-61): same
// allocation contract -- resource_error instead of std::bad_alloc.
struct AlignedFree {
    void operator()(uint8_t* p) const { ::operator delete[](p, std::align_val_t{64}); }
};

using AlignedBytes = std::unique_ptr<uint8_t[], AlignedFree>;

inline AlignedBytes allocate_record_bytes(size_t bytes) {
    try {
        return AlignedBytes(new (std::align_val_t{64}) uint8_t[bytes ? bytes : 1]);
    } catch (const std::bad_alloc&) {
        throw resource_error("cannot allocate " + std::to_string(bytes) + " bytes of record storage");
    }
}

class RecordArray {
  public:
    RecordArray() = default;
    RecordArray(const RecordLayout& layout, size_t n)
        : layout_(layout), n_(n), buf_(allocate_record_bytes(n * layout.record_size)) {}
    RecordArray(RecordArray&&) noexcept = default;
    RecordArray& operator=(RecordArray&&) noexcept = default;
    RecordArray(const RecordArray&) = delete;
    RecordArray& operator=(const RecordArray&) = delete;

    uint8_t* data() { return buf_.get(); }
    const uint8_t* data() const { return buf_.get(); }
    uint8_t* record(size_t i) { return buf_.get() + i * layout_.record_size; }
    const uint8_t* record(size_t i) const { return buf_.get() + i * layout_.record_size; }
    size_t size() const { return n_; }
    size_t byte_size() const { return n_ * layout_.record_size; }
    const RecordLayout& layout() const { return layout_; }
    bool empty() const { return n_ == 0; }

    RecordArray clone() const {
        RecordArray c(layout_, n_);
        if (byte_size()) std::memcpy(c.data(), data(), byte_size());
        return c;
    }

  private:
    RecordLayout layout_{};
    size_t n_ = 0;
    AlignedBytes buf_{};
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

inline void sort(RecordArray& array, const SchedulerConfig& cfg = {}) {
    sort(array.data(), array.size(), array.layout(), cfg);
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
