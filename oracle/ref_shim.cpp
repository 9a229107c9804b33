// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// extern "C" face of the *unmodified* RADULS reference library, compiled from
// the sources where they lie under /root/reference/proj (see oracle/Makefile,
// target `ref`). Output goes to oracle/_ref/libraduls_ref.so, which is
// git-ignored and travels to the GPU box with the snapshot so tests, smoke()
// and bench.py's reference arm can run the real reference there.
//
// Every function forwards to the reference's public API:
//   raduls::sort                 P/include/raduls/scheduler.hpp:60-61, P/src/scheduler.cpp:40-45
//   raduls::lsd_sort             P/include/raduls/lsd.hpp:22-26, P/src/lsd.cpp:12-35
//   raduls::oracle_sort          P/include/raduls/verify.hpp:53, P/src/verify.cpp:52-64
//   raduls::array_digest         P/src/verify.cpp:37-50
//   raduls::check_sorted         P/src/verify.cpp:27-35
//   raduls::radix_split          P/include/raduls/kernels.hpp:157-167
//   raduls::buffered_radix_split P/include/raduls/kernels.hpp:175-264
//   raduls::build_histogram      P/include/raduls/kernels.hpp:71-77
//   raduls::generate             P/src/datagen.cpp:86-118
// (P = /root/reference/proj). Exceptions never cross this boundary; they map
// to the same status codes the GPU C-ABI uses (include/raduls_gpu.h).
#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>

#include "raduls/datagen.hpp"
#include "raduls/detail/dispatch.hpp"
#include "raduls/kernels.hpp"
#include "raduls/lsd.hpp"
#include "raduls/scheduler.hpp"
#include "raduls/small_sorts.hpp"
#include "raduls/verify.hpp"

namespace {
constexpr int kOk = 0, kInval = 1, kNomem = 2, kOther = 9;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const std::invalid_argument&) {
        return kInval;
    } catch (const raduls::resource_error&) {
        return kNomem;
    } catch (const std::bad_alloc&) {
        return kNomem;
    } catch (...) {
        return kOther;
    }
}
}  // namespace

extern "C" {

int ref_sort(uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks, uint32_t threads) {
    return guarded([&] {
        raduls::SchedulerConfig cfg;
        cfg.threads = threads ? threads : 1;
        raduls::sort(data, size_t(n), raduls::RecordLayout{rs, ks}, cfg);
    });
}

int ref_lsd_sort(uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks, uint32_t buffer_bytes,
                 uint32_t threads) {
    return guarded([&] {
        raduls::lsd_sort(data, size_t(n), raduls::RecordLayout{rs, ks},
                         raduls::LsdConfig{buffer_bytes, threads ? threads : 1});
    });
}

int ref_oracle_sort(uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks) {
    return guarded([&] { raduls::oracle_sort(data, size_t(n), raduls::RecordLayout{rs, ks}); });
}

int ref_digest(const uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks, uint64_t* lo,
               uint64_t* hi) {
    return guarded([&] {
        const auto d = raduls::array_digest(data, size_t(n), raduls::RecordLayout{rs, ks});
        *lo = d.lo;
        *hi = d.hi;
    });
}

// Returns 1 when sorted, 0 otherwise (first violation in *first_violation);
// negative on an unsupported layout.
int ref_check_sorted(const uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks,
                     uint64_t* first_violation) {
    try {
        const auto r = raduls::check_sorted(data, size_t(n), raduls::RecordLayout{rs, ks});
        if (first_violation) *first_violation = r.first_violation;
        return r.ok ? 1 : 0;
    } catch (...) {
        return -1;
    }
}

int ref_build_histogram(const uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks,
                        uint32_t byte_index, uint64_t* counts256) {
    return guarded([&] {
        const auto h =
            raduls::build_histogram(data, size_t(n), raduls::RecordLayout{rs, ks}, byte_index);
        std::memcpy(counts256, h.counts.data(), 256 * sizeof(uint64_t));
    });
}

// One stable single-digit split at record byte offset `key_byte_offset`.
int ref_radix_split(const uint8_t* src, uint8_t* dst, uint64_t n, uint32_t rs, uint32_t ks,
                    uint32_t key_byte_offset, uint64_t* counts256) {
    return guarded([&] {
        raduls::detail::dispatch_layout(raduls::RecordLayout{rs, ks}, [&](auto rb, auto) {
            const auto h = raduls::radix_split<rb()>(src, dst, size_t(n), key_byte_offset);
            if (counts256) std::memcpy(counts256, h.counts.data(), 256 * sizeof(uint64_t));
        });
    });
}

int ref_buffered_split(const uint8_t* src, uint8_t* dst, uint64_t n, uint32_t rs, uint32_t ks,
                       uint32_t key_byte_offset, uint32_t threads, uint64_t* counts256) {
    return guarded([&] {
        raduls::detail::dispatch_layout(raduls::RecordLayout{rs, ks}, [&](auto rb, auto) {
            const unsigned t = threads ? threads : 1;
            const auto bounds = raduls::linear_growth_chunks(size_t(n), t);
            const auto h = raduls::buffered_radix_split<rb()>(src, dst, size_t(n),
                                                              key_byte_offset, bounds, t, 256);
            if (counts256) std::memcpy(counts256, h.counts.data(), 256 * sizeof(uint64_t));
        });
    });
}

int ref_is_tiny(uint64_t bin_size, uint64_t parent_size) {
    return raduls::is_tiny(size_t(bin_size), size_t(parent_size), raduls::TinyPolicy{}) ? 1 : 0;
}

// The reference's own generator (mt19937_64 shards); dist 0 uniform, 1 zipf.
int ref_generate(uint8_t* out, uint64_t n, uint32_t rs, uint32_t ks, uint32_t dist, double theta,
                 uint64_t universe, uint64_t seed, uint32_t threads) {
    return guarded([&] {
        raduls::GenSpec s;
        s.n = size_t(n);
        s.layout = raduls::RecordLayout{rs, ks};
        s.dist = dist ? raduls::Distribution::zipf : raduls::Distribution::uniform;
        s.theta = theta;
        s.universe = universe;
        s.seed = seed;
        auto a = raduls::generate(s, threads ? threads : 1);
        if (a.byte_size()) std::memcpy(out, a.data(), a.byte_size());
    });
}

uint64_t ref_mix64(uint64_t x) { return raduls::mix64(x); }

}  // extern "C"
