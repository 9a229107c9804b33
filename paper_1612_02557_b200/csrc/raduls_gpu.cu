// libraduls_gpu.so — C-ABI + C++ host planner of the B200 MSD record sort.
//
// Host side of the reference's MsdSorter (P/include/raduls/detail/msd_sorter.hpp:
// 41-233) and its entry raduls::sort (P/src/scheduler.cpp:40-45), re-designed
// for one GPU: instead of T worker threads draining priority queues of bins,
// the host runs a short loop over MSD *levels*; each level is a handful of
// kernel launches over device-resident segment lists:
//
//   level 0   k_sample_andor: first varying key byte of a strided sample
//   level L   k_tile_hist   per-tile digit counts + per-segment AND/OR (one read)
//             k_tile_scan   decoupled-lookback segmented scan -> per-tile offsets
//             k_plan        per segment: finish / skip a constant byte /
//                           scatter; children routed to groups or next level
//             k_scatter     one stable split of every scattered segment
//             k_local_sort  groups of small bins, sorted straight into `data`
//             k_copy_back   finished bins that ended in tmp
//
// One device->host read of the level counters per level sizes the next
// launches. See DESIGN.md for the data layout and the per-kernel rooflines.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/raduls_gpu.h"
#include "common.cuh"
#include "k_histogram.cuh"
#include "k_local.cuh"
#include "k_local_bm.cuh"
#include "k_partition.cuh"
#include "k_plan.cuh"
#include "k_scan.cuh"
#include "k_scatter.cuh"
#include "k_util.cuh"

namespace {

using namespace rg;

constexpr int kMaxLevels = 72;
// Key-range batches of a progressive sort (the host drop-in's overlapped
// device->host copy): the last batch's copy is the part left unoverlapped.
constexpr uint32_t kProgressiveBatches = 16;
// Per-call record limit: per-tile digit offsets are 32-bit (k_tile_scan).
constexpr uint64_t kMaxRecords = 1ull << 32;

struct CudaError {
    int code;
};

// A failed call is also recorded as the runtime's last error; clear it so a
// recoverable failure (an allocation) does not resurface at the next launch
// check of a later call. Sticky errors persist regardless.
#define RG_CHECK(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            if (std::getenv("RADULS_GPU_DEBUG"))                                        \
                std::fprintf(stderr, "raduls_gpu: %s failed: %s (%s:%d)\n", #expr,      \
                             cudaGetErrorString(e_), __FILE__, __LINE__);               \
            cudaGetLastError();                                                         \
            throw CudaError{e_ == cudaErrorMemoryAllocation ? RADULS_GPU_ENOMEM          \
                                                            : RADULS_GPU_ECUDA};         \
        }                                                                               \
    } while (0)

#define RG_LAUNCH_CHECK() RG_CHECK(cudaGetLastError())

// Every kernel launch of the library, process-wide (raduls_gpu_launch_count):
// bench.py reports how many of this library's kernels ran in its timed region.
static std::atomic<unsigned long long> g_launches{0};
static inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Host drop-ins: keep their two N*rs device buffers between calls
// (raduls_gpu_set_host_cache(1)) or free them before returning (default, like
// the reference's per-call aux buffer, P/include/raduls/detail/msd_sorter.hpp:52).
static std::atomic<int> g_host_cache{0};

// Checked build (RG_CHECKED; see common.cuh): the device ranges the current
// call may touch, the per-call violation check, the report.
#ifdef RG_CHECKED
struct ChkHost {
    std::mutex mu;
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    unsigned long long report[6] = {};  // fails, first_addr, site, bytes, deadlocks, checked calls
};
static ChkHost g_chk_host;
static void chk_upload(cudaStream_t st) {
    // RADULS_GPU_CHECK_SHRINK=B (negative control of the tests): every range
    // B bytes shorter, so a correct sort must be reported
    static const uint64_t shrink = std::getenv("RADULS_GPU_CHECK_SHRINK")
                                       ? std::strtoull(std::getenv("RADULS_GPU_CHECK_SHRINK"), nullptr, 10) : 0;
    std::vector<std::pair<uint64_t, uint64_t>> r = g_chk_host.ranges;
    for (auto& x : r) x.second = std::max(x.first, x.second - shrink);
    std::sort(r.begin(), r.end());
    std::vector<std::pair<uint64_t, uint64_t>> m;  // merged: sorted, disjoint
    for (auto& x : r) {
        if (!m.empty() && x.first <= m.back().second) m.back().second = std::max(m.back().second, x.second);
        else m.push_back(x);
    }
    static rg::ChkState h;  // (under g_chk_host.mu; copied before it is reused)
    const size_t k = std::min<size_t>(m.size(), rg::kChkRanges);
    for (size_t i = 0; i < k; ++i) h.lo[i] = m[i].first, h.hi[i] = m[i].second;
    h.n = unsigned(k);
    const size_t off = offsetof(rg::ChkState, n);
    RG_CHECK(cudaMemcpyToSymbol(rg::g_chk, reinterpret_cast<const char*>(&h) + off, sizeof(rg::ChkState) - off, off,
                                cudaMemcpyHostToDevice));
    (void)st;
}
// Replace (reset = true) or extend the registered ranges; enqueued on st.
static void chk_ranges(cudaStream_t st, std::initializer_list<std::pair<const void*, size_t>> r,
                       bool reset = true) {
    std::lock_guard<std::mutex> lk(g_chk_host.mu);
    if (reset) g_chk_host.ranges.clear();
    for (auto& x : r)
        if (x.first && x.second)
            g_chk_host.ranges.emplace_back(reinterpret_cast<uint64_t>(x.first),
                                           reinterpret_cast<uint64_t>(x.first) + x.second);
    chk_upload(st);
}
static void chk_begin() {
    cudaDeviceSynchronize();
    {
        std::lock_guard<std::mutex> lk(g_chk_host.mu);
        g_chk_host.ranges.clear();
    }
    static rg::ChkState h;  // zeros: no ranges, no counts (calls are serialised, g_chk_call)
    h.jitter = std::getenv("RADULS_GPU_CHECK_JITTER") ? 1u : 0u;
    cudaMemcpyToSymbol(rg::g_chk, &h, offsetof(rg::ChkState, lo));
}
// One checked call at a time per process: the device-side state (ranges,
// counters) is one per device and the host range list one per process, and
// a multi-device call runs a host thread per device.
static std::recursive_mutex g_chk_call;
// 0, or RADULS_GPU_EINTERNAL after printing the first violation
static int chk_end() {
    cudaDeviceSynchronize();
    rg::ChkState h;
    if (cudaMemcpyFromSymbol(&h, rg::g_chk, offsetof(rg::ChkState, lo)) != cudaSuccess) return RADULS_GPU_ECUDA;
    std::lock_guard<std::mutex> lk(g_chk_host.mu);
    g_chk_host.report[5]++;
    if (!h.fails && !h.deadlocks) return 0;
    if (!g_chk_host.report[0] && !g_chk_host.report[4]) {
        g_chk_host.report[1] = h.first_addr;
        g_chk_host.report[2] = h.first_site;
        g_chk_host.report[3] = h.first_bytes;
    }
    g_chk_host.report[0] += h.fails;
    g_chk_host.report[4] += h.deadlocks;
    std::fprintf(stderr, "raduls_gpu[checked]: %llu out-of-range/misaligned accesses (first: site %u, addr 0x%llx, %u B), "
                 "%llu barrier timeouts\n", h.fails, h.first_site, h.first_addr, h.first_bytes, h.deadlocks);
    return RADULS_GPU_EINTERNAL;
}
static void chk_ranges_vec(cudaStream_t st, const std::vector<std::pair<const void*, size_t>>& r) {
    std::lock_guard<std::mutex> lk(g_chk_host.mu);
    g_chk_host.ranges.clear();
    for (auto& x : r)
        if (x.first && x.second)
            g_chk_host.ranges.emplace_back(reinterpret_cast<uint64_t>(x.first),
                                           reinterpret_cast<uint64_t>(x.first) + x.second);
    chk_upload(st);
}
#define RG_CHK_RANGES_VEC(st, v) chk_ranges_vec((st), (v))
#define RG_CHK_RANGES(st, ...) chk_ranges((st), __VA_ARGS__)
#define RG_CHK_RANGES_ADD(st, ...) chk_ranges((st), __VA_ARGS__, false)
#else
#define RG_CHK_RANGES(st, ...) ((void)0)
#define RG_CHK_RANGES_ADD(st, ...) ((void)0)
#define RG_CHK_RANGES_VEC(st, v) ((void)0)
#endif

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
    void ensure(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n, 1);
        RG_CHECK(cudaMalloc(&p, want * sizeof(T)));
        cap = want;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// The host drop-ins' two n*rs device buffers. Mapped through the driver's
// virtual-memory API (cuMemCreate / cuMemMap, entry points looked up at run
// time) when available: unmapping one does not wait for the device, so the
// scratch buffer is released while the result's device->host copies are
// still running, and the whole release costs ~20 ms instead of cudaFree's
// device-wide wait plus 20-50 ms (profiles/r2_probe_vmm.txt). Else cudaMalloc.
struct VmmApi {
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemSetAccess) access = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemGetAllocationGranularity) gran = nullptr;
    bool ok = false;
    static const VmmApi& get() {
        static const VmmApi api = [] {
            VmmApi a;
            if (std::getenv("RADULS_GPU_NO_VMM")) return a;
            auto sym = [](const char* name) -> void* {
                void* p = nullptr;
                cudaDriverEntryPointQueryResult q{};
                if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
                    q != cudaDriverEntryPointSuccess) {
                    cudaGetLastError();
                    return nullptr;
                }
                return p;
            };
            a.create = reinterpret_cast<decltype(a.create)>(sym("cuMemCreate"));
            a.reserve = reinterpret_cast<decltype(a.reserve)>(sym("cuMemAddressReserve"));
            a.map = reinterpret_cast<decltype(a.map)>(sym("cuMemMap"));
            a.access = reinterpret_cast<decltype(a.access)>(sym("cuMemSetAccess"));
            a.unmap = reinterpret_cast<decltype(a.unmap)>(sym("cuMemUnmap"));
            a.release = reinterpret_cast<decltype(a.release)>(sym("cuMemRelease"));
            a.addr_free = reinterpret_cast<decltype(a.addr_free)>(sym("cuMemAddressFree"));
            a.gran = reinterpret_cast<decltype(a.gran)>(sym("cuMemGetAllocationGranularity"));
            a.ok = a.create && a.reserve && a.map && a.access && a.unmap && a.release && a.addr_free && a.gran;
            return a;
        }();
        return api;
    }
};

struct HostDevBuf {
    uint8_t* p = nullptr;
    size_t cap = 0;  // bytes
    size_t mapped = 0;
    CUmemGenericAllocationHandle h = 0;
    bool vmm = false;
    void ensure(size_t n) {
        if (n <= cap) return;
        release();
        const VmmApi& v = VmmApi::get();
        if (v.ok) {
            int dev = 0;
            RG_CHECK(cudaGetDevice(&dev));
            CUmemAllocationProp prop{};
            prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            prop.location.id = dev;
            size_t g = 0;
            if (v.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && g) {
                const size_t sz = (std::max<size_t>(n, 1) + g - 1) / g * g;
                CUdeviceptr va = 0;
                CUmemGenericAllocationHandle hh = 0;
                if (v.reserve(&va, sz, 0, 0, 0) == CUDA_SUCCESS) {
                    if (v.create(&hh, sz, &prop, 0) == CUDA_SUCCESS) {
                        CUmemAccessDesc ad{};
                        ad.location = prop.location;
                        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
                        if (v.map(va, sz, 0, hh, 0) == CUDA_SUCCESS) {
                            if (v.access(va, sz, &ad, 1) == CUDA_SUCCESS) {
                                p = reinterpret_cast<uint8_t*>(va);
                                cap = n;
                                mapped = sz;
                                h = hh;
                                vmm = true;
                                return;
                            }
                            v.unmap(va, sz);
                        }
                        v.release(hh);
                    }
                    v.addr_free(va, sz);
                }
                // out of device memory (or no VMM for this device): plain cudaMalloc below
            }
        }
        RG_CHECK(cudaMalloc(&p, std::max<size_t>(n, 1)));
        cap = n;
        vmm = false;
    }
    // The caller guarantees no queued work still uses the buffer (VMM:
    // unmapping does not wait; cudaFree waits for the whole device).
    void release() {
        if (!p) return;
        if (vmm) {
            const VmmApi& v = VmmApi::get();
            const CUdeviceptr va = reinterpret_cast<CUdeviceptr>(p);
            v.unmap(va, mapped);
            v.release(h);
            v.addr_free(va, mapped);
        } else {
            cudaFree(p);
        }
        p = nullptr;
        cap = mapped = 0;
        h = 0;
        vmm = false;
    }
};

// Optional per-kernel timing (raduls_gpu_set_profiling): CUDA events around
// every launch of the sort, on the launching stream, collected at the end of
// the sort (which synchronises anyway). Used by bench.py for the live
// roofline of the dominant kernel.
enum KClass { K_SAMPLE, K_HIST, K_SCAN, K_PLAN, K_SCATTER, K_LOCAL, K_COPY, K_INIT, K_NCLASS };
static const char* kClassName[K_NCLASS] = {"sample", "tile_hist", "tile_scan", "plan",
                                           "scatter", "local_sort", "copy_back", "init"};

struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> cls;  // per recorded pair
    size_t used = 0;
    double ms[K_NCLASS] = {};
    uint32_t launches[K_NCLASS] = {};
    void reset() {
        used = 0;
        cls.clear();
        for (int i = 0; i < K_NCLASS; ++i) ms[i] = 0, launches[i] = 0;
    }
    int begin(int c, cudaStream_t st) {
        if (!on) return -1;
        while (ev.size() < 2 * (used + 1)) {
            cudaEvent_t e;
            RG_CHECK(cudaEventCreate(&e));
            ev.push_back(e);
        }
        RG_CHECK(cudaEventRecord(ev[2 * used], st));
        cls.push_back(c);
        return int(used++);
    }
    void end(int i, cudaStream_t st) {
        if (i >= 0) RG_CHECK(cudaEventRecord(ev[2 * i + 1], st));
    }
    void collect() {  // after the stream has been synchronised
        for (size_t i = 0; i < used; ++i) {
            float t = 0.f;
            RG_CHECK(cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]));
            ms[cls[i]] += t;
            launches[cls[i]]++;
        }
        used = 0;
        cls.clear();
    }
};

// Host <-> device streaming for the host drop-ins.
// Pinned (page-locked or registered) caller buffers go straight to the DMA
// engine. Pageable ones -- the reference's callers pass plain heap memory --
// would cap cudaMemcpy at ~11 GB/s H2D / ~21 GB/s D2H on the B200 box, so they
// stream in chunks through a ring of pinned staging buffers: a small thread
// pool copies chunk i between the caller's memory and a staging buffer while
// the copy engine moves chunk i-1 (measurements in DESIGN.md).
class CopyPool {
  public:
    explicit CopyPool(unsigned n) {
        for (unsigned i = 0; i < n; ++i) th_.emplace_back([this, i] { run(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // memcpy split over the pool (the calling thread waits)
    void copy(uint8_t* dst, const uint8_t* src, size_t len) {
        if (len < (size_t(1) << 20) || th_.empty()) {
            std::memcpy(dst, src, len);
            return;
        }
        std::unique_lock<std::mutex> lk(m_);
        dst_ = dst;
        src_ = src;
        len_ = len;
        remaining_ = unsigned(th_.size());
        ++gen_;
        cv_.notify_all();
        done_.wait(lk, [&] { return remaining_ == 0; });
    }

  private:
    void run(unsigned id) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            uint8_t* d = dst_;
            const uint8_t* s = src_;
            const size_t len = len_, nt = th_.size();
            lk.unlock();
            size_t per = (len + nt - 1) / nt;
            per = (per + 4095) & ~size_t(4095);
            const size_t a = size_t(id) * per;
            if (a < len) std::memcpy(d + a, s + a, std::min(per, len - a));
            lk.lock();
            if (--remaining_ == 0) done_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    uint8_t* dst_ = nullptr;
    const uint8_t* src_ = nullptr;
    size_t len_ = 0;
    unsigned remaining_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

struct HostStager {
    static constexpr size_t kChunk = size_t(32) << 20;
    static constexpr int kRing = 3;
    uint8_t* stage[kRing] = {};
    cudaEvent_t ev[kRing] = {};
    CopyPool pool;

    static unsigned pool_threads() {
        const unsigned hw = std::thread::hardware_concurrency();
        return std::max(1u, std::min(8u, hw ? hw : 1u));
    }
    cudaStream_t copy = nullptr;  // device->host copies of finished key ranges (progressive sort)
    cudaEvent_t done = nullptr;
    HostStager() : pool(pool_threads()) {
        for (int i = 0; i < kRing; ++i) {
            RG_CHECK(cudaMallocHost(&stage[i], kChunk));
            RG_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        RG_CHECK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        RG_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    }
    ~HostStager() {
        if (copy) cudaStreamDestroy(copy);
        if (done) cudaEventDestroy(done);
        for (int i = 0; i < kRing; ++i) {
            if (stage[i]) cudaFreeHost(stage[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
    }
    static bool pinned(const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }
    void h2d(uint8_t* dev, const uint8_t* host, size_t bytes, cudaStream_t st) {
        if (pinned(host)) {
            RG_CHECK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
            return;
        }
        const size_t nchunks = (bytes + kChunk - 1) / kChunk;
        for (size_t c = 0; c < nchunks; ++c) {
            const int b = int(c % kRing);
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            // the staging buffer's last DMA -- from this call or an earlier
            // h2d/d2h, which may still be in flight -- must be done before the
            // host overwrites it (an event never recorded returns at once)
            RG_CHECK(cudaEventSynchronize(ev[b]));
            pool.copy(stage[b], host + off, len);
            RG_CHECK(cudaMemcpyAsync(dev + off, stage[b], len, cudaMemcpyHostToDevice, st));
            RG_CHECK(cudaEventRecord(ev[b], st));
        }
    }
    void d2h(uint8_t* host, const uint8_t* dev, size_t bytes, cudaStream_t st) {
        if (pinned(host)) {
            RG_CHECK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st));
            RG_CHECK(cudaStreamSynchronize(st));
            return;
        }
        const size_t nchunks = (bytes + kChunk - 1) / kChunk;
        // issue chunk c, then drain chunk c - (kRing - 1): kRing - 1 DMAs in flight
        for (size_t c = 0; c < nchunks + kRing - 1; ++c) {
            if (c < nchunks) {
                const int b = int(c % kRing);
                const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
                RG_CHECK(cudaMemcpyAsync(stage[b], dev + off, len, cudaMemcpyDeviceToHost, st));
                RG_CHECK(cudaEventRecord(ev[b], st));
            }
            if (c >= size_t(kRing - 1)) {
                const size_t j = c - (kRing - 1);
                if (j >= nchunks) continue;
                const int b = int(j % kRing);
                const size_t off = j * kChunk, len = std::min(kChunk, bytes - off);
                RG_CHECK(cudaEventSynchronize(ev[b]));
                pool.copy(host + off, stage[b], len);
            }
        }
    }
};

struct Workspace {
    int device = 0;
    Prof prof;
    std::mutex mu;
    DevBuf<unsigned long long> hist8, andor0, thr, acc;
    DevBuf<LevelCounters> ctr;
    DevBuf<Seg> segs[2];
    DevBuf<unsigned long long> seg_tot[2], seg_andor[2];
    DevBuf<uint32_t> tile_seg[2];
    DevBuf<uint16_t> tile_cnt;
    DevBuf<uint32_t> tile_off;
    DevBuf<unsigned long long> status;
    DevBuf<Group> groups, spill, spill_bm, spill_med;
    // [0]: groups for the LSD fallback, [1]: groups the bitmap sort handed to
    // the bucket sort, [2]: groups above the bitmap sort's primary capacity
    DevBuf<unsigned int> n_spill;
    DevBuf<CopyRange> copies;
    HostDevBuf host_data, host_tmp;
    DevBuf<uint8_t> map8;
    // partition pivots (raduls_gpu_set_pivots): the map buffer's pivot region
    // (kMapBytes - 65536 bytes) as uploaded with every bucket map
    std::array<uint8_t, kMapBytes - kMapPivotSlot> pivots{};
    uint32_t n_pivots = 0, pivot_max_digit = 0;
    DevBuf<unsigned long long> dig_dst;  // per-destination byte addresses (raduls_gpu_partition_to)
    DevBuf<Piece> pieces;
    DevBuf<unsigned long long> hot;       // raduls_gpu_digit_andor: slot flags + accumulators                // split digits' destination pieces (raduls_gpu_partition_store_pieces)
    DevBuf<uint8_t> nd;                  // digit array: next key byte per record position (sort_impl)
    DevBuf<Seg> bsegs;                   // level-1 segments of a progressive sort
    HostStager* stager = nullptr;  // host drop-ins, created on first use
    HostStager& host_stager() {
        if (!stager) stager = new HostStager();
        return *stager;
    }
    LevelCounters* h_ctr = nullptr;         // pinned [kMaxLevels]
    unsigned long long* h_small = nullptr;  // pinned scratch [4096]
    raduls_gpu_stats last{};
    bool attrs_set[33] = {};
    int rank_mode = -1;  // scatter ranking: -1 unchecked, 0 atomic (device-checked), 1 ballot
    // raduls_gpu_partition_plan -> raduls_gpu_partition_store hand-over
    struct PartPlan {
        bool pending = false;
        const void* src = nullptr;
        uint64_t n = 0;
        uint32_t rs = 0, ks = 0;
        unsigned long long tot[256] = {};
    } part;

    Workspace() {
        RG_CHECK(cudaMallocHost(&h_ctr, sizeof(LevelCounters) * kMaxLevels));
        RG_CHECK(cudaMallocHost(&h_small, sizeof(unsigned long long) * 4096));
        hist8.ensure(8 * kRadix);
        andor0.ensure(8);
        acc.ensure(4);
        ctr.ensure(kMaxLevels);
        thr.ensure(256);
    }
};

std::mutex g_mu;
std::map<int, Workspace*> g_ws;

Workspace& workspace() {
    int dev = 0;
    RG_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_ws.find(dev);
    if (it != g_ws.end()) return *it->second;
    auto* w = new Workspace();
    w->device = dev;
    g_ws[dev] = w;
    return *w;
}

bool layout_ok(uint32_t rs, uint32_t ks) {
    return (rs == 8 || rs == 16 || rs == 24 || rs == 32) && ks >= 1 && ks <= rs;
}

bool aligned_ok(const void* p, uint32_t rs) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    return (a % (rs % 16 == 0 ? 16 : 8)) == 0;
}

int grid_for(uint64_t n, int threads, int per_sm) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (n + threads - 1) / threads;
    return int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sms) * per_sm)));
}

// Local-sort group capacity: the register variant for 8-B records (C2 needs
// ~17 K-record groups), the shared-memory variant otherwise.
#ifndef RG_LOC_BM
#define RG_LOC_BM 1
#endif
#ifndef RG_LOC_BM8
#define RG_LOC_BM8 1
#endif
// L2 prefetch distance of the bitmap local sort, in resident waves (NUM / DEN).
// Measured (C5 local sort): 2 waves 30.4 ms, 1 wave 28.4, 1/2 wave 28.0-28.1,
// 1/4 wave 28.1.
#ifndef RG_BM_AHEAD_NUM
#define RG_BM_AHEAD_NUM 1
#endif
#ifndef RG_BM_AHEAD_DEN
#define RG_BM_AHEAD_DEN 2
#endif
template <int RS>
constexpr uint32_t local_cap() {
    return LocalCfg<RS>::kCap;
}
// Bound on a group packed from several small bins: the bitmap sort's primary
// capacity (a single bin above it, up to local_cap, is a group of its own).
template <int RS>
constexpr uint32_t group_cap() {
    if constexpr (RG_LOC_BM && RS != 8) return BmCfg<RS>::kCap;
    else return LocalCfg<RS>::kCap;
}

// Capacities for a sort of n records.
struct Caps {
    size_t seg, tiles, groups, copies;
};

template <int RS>
Caps caps_for(uint64_t n, uint64_t extra_segs = 0) {
    const uint64_t cap_local = local_cap<RS>();
    Caps c;
    c.seg = size_t(n / (cap_local + 1) + 2 + extra_segs);
    c.tiles = size_t(n / ScatterCfg<RS>::kTile + c.seg + 2);
    c.groups = size_t(3 * (n / group_cap<RS>()) + c.seg + 2);
    c.copies = size_t(n / kCopyTile + c.seg + 2);
    return c;
}

template <int RS>
void ensure_caps(Workspace& ws, uint64_t n, uint64_t extra_segs = 0) {
    const Caps c = caps_for<RS>(n, extra_segs);
    for (int b = 0; b < 2; ++b) {
        ws.segs[b].ensure(c.seg);
        ws.seg_tot[b].ensure(c.seg * kRadix);
        ws.seg_andor[b].ensure(c.seg * 8);
        ws.tile_seg[b].ensure(c.tiles);
    }
    ws.tile_cnt.ensure(c.tiles * kRadix);
    ws.tile_off.ensure(c.tiles * kRadix);
    ws.status.ensure((c.tiles / kScanChunk + 1) * kRadix);
    ws.groups.ensure(c.groups);
    ws.spill.ensure(c.groups);
    ws.spill_bm.ensure(c.groups);
    if constexpr (RS != 8) ws.spill_med.ensure(c.groups);
    ws.n_spill.ensure(4);  // ([0] read back as the low half of one 8-B word)
    ws.copies.ensure(c.copies);
}

template <int RS>
void set_attrs(Workspace& ws) {
    if (ws.attrs_set[RS]) return;
    RG_CHECK(cudaFuncSetAttribute(k_local<RS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(LocalCfg<RS>::kSmem)));
    RG_CHECK(cudaFuncSetAttribute(k_local<RS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(LocalCfg<RS>::kSmem)));
    RG_CHECK(cudaFuncSetAttribute(k_local_list<RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(LocalCfg<RS>::kSmem)));
    if constexpr (RS == 8) {
        RG_CHECK(cudaFuncSetAttribute(k_local_bm8, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(Bm8Cfg::kSmem)));
    } else {
        RG_CHECK(cudaFuncSetAttribute(k_local_bm<RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(BmCfg<RS>::kSmem)));
        if constexpr (kBmHasBig<RS>) {
            RG_CHECK(cudaFuncSetAttribute(k_local_bm_med<RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(BmCfg<RS, 1>::kSmem)));
            RG_CHECK(cudaFuncSetAttribute(k_local_bm<RS, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(BmCfg<RS, 1>::kSmem)));
        }
    }
    RG_CHECK(cudaFuncSetAttribute(k_tile_hist<RS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(HistCfg<RS>::kSmem)));
    RG_CHECK(cudaFuncSetAttribute(k_tile_hist<RS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(HistCfg<RS>::kSmem)));
    RG_CHECK(cudaFuncSetAttribute(k_tile_hist<RS, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(HistCfg<RS>::kSmem)));
    for (int r = 0; r < 2; ++r) {
        RG_CHECK(cudaFuncSetAttribute(r ? k_scatter<RS, false, false, 1> : k_scatter<RS, false, false, 0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(ScatterCfg<RS>::kSmemPlain)));
        RG_CHECK(cudaFuncSetAttribute(r ? k_scatter<RS, true, false, 1> : k_scatter<RS, true, false, 0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(ScatterCfg<RS>::kSmem)));
        RG_CHECK(cudaFuncSetAttribute(r ? k_scatter<RS, true, true, 1> : k_scatter<RS, true, true, 0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(ScatterCfg<RS>::kSmem)));
    }
    ws.attrs_set[RS] = true;
}

int sm_count() {
    int dev = 0, sms = 148;
    RG_CHECK(cudaGetDevice(&dev));
    RG_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}

// Tile histogram + segmented look-back scan of one level: per-tile digit
// offsets (ws.tile_off), per-segment digit totals (ws.seg_tot[cur]).
// nd_in: byte p of every record of the level, by record position (written
// by the previous level's scatter), so the histogram reads one byte per record.
template <int RS, bool kMap = false, bool kKey1 = false>
void level_counts(Workspace& ws, uint8_t* data, uint8_t* tmp, int cur, uint32_t ntiles, LevelCounters* c,
                  cudaStream_t st, uint32_t ks = 0, const uint8_t* map = nullptr,
                  const uint8_t* nd_in = nullptr) {
    constexpr int TILE = ScatterCfg<RS>::kTile;
    int pe = ws.prof.begin(K_HIST, st);
    if (nd_in) {
        const uint32_t grid = std::min<uint32_t>((ntiles + kNdWarps - 1) / kNdWarps, uint32_t(sm_count()) * 4);
        k_tile_hist_nd<TILE><<<grid, kNdWarps * 32, 0, st>>>(nd_in, ws.segs[cur].p, ws.tile_seg[cur].p,
                                                             ws.tile_cnt.p, c, ntiles);
        note_launch();
    } else if constexpr (RS == 8) {  // one CTA per tile (see k_tile_hist_reg)
        k_tile_hist_reg<RS, TILE, kMap><<<ntiles, HistRegCfg<RS, TILE>::kThreads, 0, st>>>(
            data, tmp, ws.segs[cur].p, ws.tile_seg[cur].p, ws.tile_cnt.p, ws.seg_andor[cur].p, c, ks, map,
            uint32_t(sm_count()) * 4);
        note_launch();
    } else {  // persistent, TMA-fed
        const uint32_t hgrid = std::min<uint32_t>(ntiles, uint32_t(sm_count()) * HistCfg<RS>::kCtas);
        k_tile_hist<RS, kMap, kKey1><<<hgrid, HistCfg<RS>::kThreads + 64, HistCfg<RS>::kSmem, st>>>(
            data, tmp, ws.segs[cur].p, ws.tile_seg[cur].p, ws.tile_cnt.p, ws.seg_andor[cur].p, c, ntiles, ks,
            map);
        note_launch();
    }
    RG_LAUNCH_CHECK();
    ws.prof.end(pe, st);
    const uint32_t nchunks = (ntiles + kScanChunk - 1) / kScanChunk;
    RG_CHECK(cudaMemsetAsync(ws.status.p, 0, size_t(nchunks) * kRadix * sizeof(unsigned long long), st));
    pe = ws.prof.begin(K_SCAN, st);
    k_tile_scan<TILE><<<nchunks, 256, 0, st>>>(ws.segs[cur].p, ws.tile_seg[cur].p, ws.tile_cnt.p, ntiles,
                                               ws.tile_off.p, ws.seg_tot[cur].p, ws.status.p, c);
    note_launch();
    RG_LAUNCH_CHECK();
    ws.prof.end(pe, st);
}

// Whether the scatter may rank with shared-memory atomics (warp_rank<0>):
// decided once per device by k_rank_selftest, overridable with
// RADULS_GPU_STABLE_RANK=ballot (always warp_rank<1>) for tests and A/B.
bool atomic_rank_ok(Workspace& ws) {
    if (ws.rank_mode < 0) {
        const char* e = std::getenv("RADULS_GPU_STABLE_RANK");
        if (e && std::strcmp(e, "ballot") == 0) {
            ws.rank_mode = 1;
        } else {
            unsigned int* d_bad = reinterpret_cast<unsigned int*>(ws.acc.p + 2);
            RG_CHECK(cudaMemset(d_bad, 0, sizeof(unsigned int)));
            k_rank_selftest<<<2 * sm_count(), 256>>>(4096, d_bad);
            note_launch();
            RG_LAUNCH_CHECK();
            unsigned int bad = 1;
            RG_CHECK(cudaMemcpy(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost));
            ws.rank_mode = bad ? 1 : 0;
        }
    }
    return ws.rank_mode == 0;
}

// stable_ballot: rank with ballots regardless of the device check (the LSD
// baseline and the single-split API, whose contract is stability itself).
template <int RS, bool kMap, bool kPeer = false>
void launch_scatter(Workspace& ws, uint8_t* data, uint8_t* tmp, int cur, uint32_t ntiles, uint32_t ks,
                    const uint8_t* map, LevelCounters* c, cudaStream_t st,
                    const unsigned long long* dig_dst = nullptr, uint8_t* nd = nullptr,
                    const uint8_t* nd_in = nullptr, bool stable_ballot = false,
                    const Piece* pieces = nullptr) {
    const uint32_t grid = std::min<uint32_t>(ntiles, uint32_t(sm_count()) * ScatterCfg<RS>::kCtas);
    const size_t smem = (kMap || kPeer) ? ScatterCfg<RS>::kSmem : ScatterCfg<RS>::kSmemPlain;
    const bool atomic = !stable_ballot && atomic_rank_ok(ws);
    const int pe = ws.prof.begin(K_SCATTER, st);
    if (atomic) {
        k_scatter<RS, kMap, kPeer, 0><<<grid, ScatterCfg<RS>::kThreads + 32, smem, st>>>(
            data, tmp, ws.segs[cur].p, ws.seg_tot[cur].p, ws.tile_seg[cur].p, ws.tile_off.p, ntiles,
            &c->scatter_ticket, ks, map, dig_dst, nd, local_cap<RS>(), nd_in, pieces);
    } else {
        k_scatter<RS, kMap, kPeer, 1><<<grid, ScatterCfg<RS>::kThreads + 32, smem, st>>>(
            data, tmp, ws.segs[cur].p, ws.seg_tot[cur].p, ws.tile_seg[cur].p, ws.tile_off.p, ntiles,
            &c->scatter_ticket, ks, map, dig_dst, nd, local_cap<RS>(), nd_in, pieces);
    }
    note_launch();
    RG_LAUNCH_CHECK();
    ws.prof.end(pe, st);
}

// RADULS_GPU_LOCAL=bucket: the bucket sort alone (k_local.cuh) for every group,
// as before the bitmap sort existed (tests and A/B).
bool bitmap_local() {
    if (!RG_LOC_BM) return false;
    const char* e = std::getenv("RADULS_GPU_LOCAL");
    return !(e && std::strcmp(e, "bucket") == 0);
}

// Launch the local sort over `ngroups` groups already in ws.groups.
template <int RS>
void launch_local(Workspace& ws, uint8_t* data, uint8_t* tmp, uint32_t ngroups, uint32_t ks,
                  LevelCounters* ctr, cudaStream_t st, uint32_t n_big = 0) {
    if (!ngroups) return;
    const int pe = ws.prof.begin(K_LOCAL, st);
    // one CTA per SM: persistent, groups round-robin; two per SM: a CTA per group
    const uint32_t grid = LocalCfg<RS>::kMinBlocks == 1 ? std::min<uint32_t>(ngroups, uint32_t(sm_count()))
                                                       : ngroups;
    if constexpr (RS == 8) {
        if (bitmap_local() && RG_LOC_BM8) {
            RG_CHECK(cudaMemsetAsync(ws.n_spill.p + 1, 0, 2 * sizeof(unsigned int), st));
            const GroupList spill{ws.spill_bm.p, ws.n_spill.p + 1, uint32_t(ws.spill_bm.cap)};
            const uint32_t pgrid = std::min<uint32_t>(ngroups, uint32_t(sm_count()));
            k_local_bm8<<<pgrid, Bm8Cfg::kThreads, Bm8Cfg::kSmem, st>>>(data, tmp, ws.groups.p, ngroups, ks,
                                                                       ctr, spill);
            note_launch();
            RG_LAUNCH_CHECK();
            k_local_list<RS><<<pgrid, LocalCfg<RS>::kThreads, LocalCfg<RS>::kSmem, st>>>(
                data, tmp, ws.spill_bm.p, ws.n_spill.p + 1, uint32_t(ws.spill_bm.cap), ks, ctr, ws.spill.p,
                ws.n_spill.p, uint32_t(ws.spill.cap));
            note_launch();
            RG_LAUNCH_CHECK();
            ws.prof.end(pe, st);
            return;
        }
    } else {
        if (bitmap_local()) {
            // the bitmap sort first; the groups it hands over (device-counted
            // list) go to the bucket sort right behind it, no host read between
            RG_CHECK(cudaMemsetAsync(ws.n_spill.p + 1, 0, 2 * sizeof(unsigned int), st));
            const GroupList spill{ws.spill_bm.p, ws.n_spill.p + 1, uint32_t(ws.spill_bm.cap)};
            const GroupList med{ws.spill_med.p, ws.n_spill.p + 2, uint32_t(ws.spill_med.cap)};
            const uint32_t bgrid =
                (BmCfg<RS>::kMinBlocks == 1 || RG_BM_PERSIST)
                    ? std::min<uint32_t>(ngroups, uint32_t(sm_count()) * BmCfg<RS>::kMinBlocks)
                    : ngroups;
            // most groups are single bins above the primary capacity: the big
            // instance takes the whole list itself (no hand-over pass)
            bool big_first = false;
            if constexpr (kBmHasBig<RS>) big_first = 2ull * n_big > ngroups;
            if (big_first) {
                if constexpr (kBmHasBig<RS>) {
                    const uint32_t ggrid = BmCfg<RS, 1>::kMinBlocks == 1
                                               ? std::min<uint32_t>(ngroups, uint32_t(sm_count()))
                                               : ngroups;
                    k_local_bm<RS, 1><<<ggrid, BmCfg<RS, 1>::kThreads, BmCfg<RS, 1>::kSmem, st>>>(
                        data, tmp, ws.groups.p, ngroups, ks, ctr, spill, med,
                        uint32_t(sm_count()) * BmCfg<RS, 1>::kMinBlocks);
                    note_launch();
                    RG_LAUNCH_CHECK();
                }
            } else {
                k_local_bm<RS><<<bgrid, BmCfg<RS>::kThreads, BmCfg<RS>::kSmem, st>>>(
                    data, tmp, ws.groups.p, ngroups, ks, ctr, spill, med,
                    uint32_t(sm_count()) * BmCfg<RS>::kMinBlocks * RG_BM_AHEAD_NUM / RG_BM_AHEAD_DEN);
                note_launch();
                RG_LAUNCH_CHECK();
                if constexpr (kBmHasBig<RS>) {
                    const uint32_t mgrid =
                        std::min<uint32_t>(ngroups, uint32_t(sm_count()) * BmCfg<RS, 1>::kMinBlocks);
                    k_local_bm_med<RS><<<mgrid, BmCfg<RS, 1>::kThreads, BmCfg<RS, 1>::kSmem, st>>>(
                        data, tmp, med, ks, ctr, spill);
                    note_launch();
                    RG_LAUNCH_CHECK();
                }
            }
            const uint32_t lgrid =
                std::min<uint32_t>(ngroups, uint32_t(sm_count()) * LocalCfg<RS>::kMinBlocks);
            k_local_list<RS><<<lgrid, LocalCfg<RS>::kThreads, LocalCfg<RS>::kSmem, st>>>(
                data, tmp, ws.spill_bm.p, ws.n_spill.p + 1, uint32_t(ws.spill_bm.cap), ks, ctr, ws.spill.p,
                ws.n_spill.p, uint32_t(ws.spill.cap));
            note_launch();
            RG_LAUNCH_CHECK();
            ws.prof.end(pe, st);
            return;
        }
    }
    k_local<RS, false><<<grid, LocalCfg<RS>::kThreads, LocalCfg<RS>::kSmem, st>>>(
        data, tmp, ws.groups.p, ngroups, ks, ctr, ws.spill.p, ws.n_spill.p, uint32_t(ws.spill.cap),
        uint32_t(sm_count()) * LocalCfg<RS>::kMinBlocks);
    note_launch();
    RG_LAUNCH_CHECK();
    ws.prof.end(pe, st);
}

// Groups the fast local sort handed over (duplicate-heavy keys): stable LSD.
// `n` = the spill count, read back with the level counters.
template <int RS>
void finish_spilled(Workspace& ws, uint8_t* data, uint8_t* tmp, uint32_t ks, LevelCounters* ctr,
                    cudaStream_t st, unsigned int n) {
    if (!n) return;
    if (n > ws.spill.cap) throw CudaError{RADULS_GPU_EINTERNAL};
    const int pe = ws.prof.begin(K_LOCAL, st);
    const uint32_t grid = LocalCfg<RS>::kMinBlocks == 1 ? std::min<uint32_t>(n, uint32_t(sm_count())) : n;
    k_local<RS, true><<<grid, LocalCfg<RS>::kThreads, LocalCfg<RS>::kSmem, st>>>(
        data, tmp, ws.spill.p, n, ks, ctr, nullptr, nullptr, 0,
        uint32_t(sm_count()) * LocalCfg<RS>::kMinBlocks);
    note_launch();
    RG_LAUNCH_CHECK();
    ws.prof.end(pe, st);
    RG_CHECK(cudaStreamSynchronize(st));
}

// Device -> pinned-host copy of a few words by a kernel (stores from the SMs
// over PCIe) instead of a DMA: the level loop's counter read-backs must not
// queue behind the multi-GB device->host copies the progressive host sort
// keeps on the copy engine. (Pinned host memory is device-accessible under UVA.)
__global__ void k_publish(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                          uint32_t words) {
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}
static_assert(sizeof(LevelCounters) % 8 == 0, "LevelCounters published as u64 words");

void publish(void* h_dst, const void* d_src, size_t bytes, cudaStream_t st) {
    k_publish<<<1, 64, 0, st>>>(static_cast<unsigned long long*>(h_dst),
                                static_cast<const unsigned long long*>(d_src), uint32_t((bytes + 7) / 8));
    note_launch();
    RG_LAUNCH_CHECK();
}

// The counters of `levels` levels and the spill count in one readback; the
// spilled groups (rare) get the LSD fallback and the counters are re-read.
template <int RS>
void read_counters_and_finish(Workspace& ws, uint8_t* data, uint8_t* tmp, uint32_t ks, LevelCounters* dctr,
                              uint32_t levels, cudaStream_t st) {
    unsigned int* hn = reinterpret_cast<unsigned int*>(ws.h_small + 4001);
    publish(ws.h_ctr, dctr, sizeof(LevelCounters) * levels, st);
    publish(hn, ws.n_spill.p, 8, st);  // (n_spill is the low half of an 8-B allocation)
    RG_CHECK(cudaStreamSynchronize(st));
    const unsigned int n = *hn;
    if (!n) return;
    finish_spilled<RS>(ws, data, tmp, ks, dctr, st, n);
    publish(ws.h_ctr, dctr, sizeof(LevelCounters) * levels, st);
    RG_CHECK(cudaStreamSynchronize(st));
}

// The digit arrays of a sort of n records, `stride` bytes apart: one, or two
// when the scatter also reads its digits from them (it then writes the next
// level's into the other); grown on demand, +16 B for the 16-B aligned
// vector / TMA over-reads. 0 if they cannot be allocated or
// RADULS_GPU_NO_DIGIT_ARRAY is set.
size_t digit_arrays(Workspace& ws, uint64_t n, int halves) {
    if (std::getenv("RADULS_GPU_NO_DIGIT_ARRAY")) return 0;
    const size_t stride = (size_t(n) + 16 + 255) & ~size_t(255);
    if (ws.nd.cap >= halves * stride) return stride;
    ws.nd.release();
    if (cudaMalloc(&ws.nd.p, halves * stride) != cudaSuccess) {
        cudaGetLastError();  // not sticky: clear it
        ws.nd.p = nullptr;
        return 0;
    }
    ws.nd.cap = halves * stride;
    return stride;
}

// on_final (optional): called with record ranges [begin, end) whose content
// in `data` is final once the work enqueued on `st` so far completes, in key
// order, covering [0, n) — the host drop-in overlaps their device->host copy
// with the rest of the sort. Without it (or when the level-0 split does not
// qualify) the sort runs level by level over all segments.
// seeds (optional, raduls_gpu_sort_segments): level 0 is the given list of
// contiguous, key-ordered segments {size, first key byte that may vary}
// instead of one segment over the whole array.
struct SegSeed {
    uint64_t size;
    uint32_t p;
};

template <int RS>
void sort_impl(Workspace& ws, uint8_t* data, uint8_t* tmp, uint64_t n, uint32_t ks,
               cudaStream_t st, const std::function<void(uint64_t, uint64_t)>* on_final = nullptr,
               const std::vector<SegSeed>* seeds = nullptr) {
    constexpr int TILE = ScatterCfg<RS>::kTile;
    raduls_gpu_stats stats{};
    ws.last = stats;
    ws.prof.reset();
    ws.part.pending = false;
    if (n < 2) return;  // msd_sorter.hpp:51
    if (seeds && seeds->size() == 1 && (*seeds)[0].p == 0) seeds = nullptr;  // the plain sort
    set_attrs<RS>(ws);
    ensure_caps<RS>(ws, n, seeds ? seeds->size() : 0);
    LevelCounters* dctr = ws.ctr.p;
    RG_CHECK(cudaMemsetAsync(ws.n_spill.p, 0, 4 * sizeof(unsigned int), st));
    RG_CHK_RANGES(st, {{data, size_t(n) * RS}, {tmp, size_t(n) * RS}});
#ifdef RG_CHECKED
    {  // poison the scratch: nothing may be read before this sort writes it
        if (tmp != data) RG_CHECK(cudaMemsetAsync(tmp, 0xA5, size_t(n) * RS, st));
        RG_CHECK(cudaMemsetAsync(ws.tile_cnt.p, 0xA5, ws.tile_cnt.cap * sizeof(uint16_t), st));
        RG_CHECK(cudaMemsetAsync(ws.tile_off.p, 0xA5, ws.tile_off.cap * sizeof(uint32_t), st));
        for (int b = 0; b < 2; ++b)
            RG_CHECK(cudaMemsetAsync(ws.seg_tot[b].p, 0xA5, ws.seg_tot[b].cap * sizeof(unsigned long long), st));
        RG_CHECK(cudaMemsetAsync(ws.groups.p, 0xA5, ws.groups.cap * sizeof(Group), st));
        RG_CHECK(cudaMemsetAsync(ws.copies.p, 0xA5, ws.copies.cap * sizeof(CopyRange), st));
        if (ws.nd.p) RG_CHECK(cudaMemsetAsync(ws.nd.p, 0xA5, ws.nd.cap, st));
    }
#endif

    if (n <= uint64_t(local_cap<RS>()) && !seeds) {  // one group sorts everything, in place
        Group g{0, uint32_t(n), 0, 0, 0};
        RG_CHECK(cudaMemcpyAsync(ws.groups.p, &g, sizeof g, cudaMemcpyHostToDevice, st));
        RG_CHECK(cudaMemsetAsync(dctr, 0, sizeof(LevelCounters), st));
        launch_local<RS>(ws, data, tmp, 1, ks, dctr, st, n > uint64_t(group_cap<RS>()) ? 1u : 0u);
        read_counters_and_finish<RS>(ws, data, tmp, ks, dctr, 1, st);
        ws.prof.collect();
        stats.levels = 1;
        stats.local_records = ws.h_ctr[0].moved_local;
        stats.fallback_groups = ws.h_ctr[0].fallback_groups;
        stats.bitmap_spill_groups = ws.h_ctr[0].bm_spill;
        ws.last = stats;
        return;
    }

    // ---- level 0: guess the first varying key byte from a strided sample,
    // histogram the whole array on it, confirm with the global AND/OR.
    {
        const int pi = ws.prof.begin(K_INIT, st);
        k_init_andor<<<1, 64, 0, st>>>(ws.andor0.p, 1);
        note_launch();
        RG_LAUNCH_CHECK();
        ws.prof.end(pi, st);
    }
    const uint32_t samples = uint32_t(std::min<uint64_t>(n, 65536));
    int pe = ws.prof.begin(K_SAMPLE, st);
    k_sample_andor<RS><<<64, 256, 0, st>>>(data, n, std::max<uint64_t>(1, n / samples), samples, ws.andor0.p);
    note_launch();
    RG_LAUNCH_CHECK();
    ws.prof.end(pe, st);
    // no host round trip: the guess goes straight into the level-0 segment,
    // and a check after the histogram flags (rarely) a more significant
    // varying byte; the flag is read with the level-0 plan's counters
    k_set_seg0<<<1, 32, 0, st>>>(ws.andor0.p, ks, n, ws.segs[0].p);
    note_launch();
    RG_LAUNCH_CHECK();
    const uint32_t nt0 = uint32_t((n + TILE - 1) / TILE);
    int cur = 0;
    unsigned long long* d_flag = ws.acc.p + 3;
    auto level0_counts = [&] {
        RG_CHECK(cudaMemsetAsync(ws.tile_seg[0].p, 0, nt0 * sizeof(uint32_t), st));
        const int pi = ws.prof.begin(K_INIT, st);
        k_init_andor<<<1, 64, 0, st>>>(ws.seg_andor[0].p, 1);
        note_launch();
        RG_LAUNCH_CHECK();
        ws.prof.end(pi, st);
        RG_CHECK(cudaMemsetAsync(dctr, 0, sizeof(LevelCounters), st));
        if (ks <= 8) level_counts<RS, false, true>(ws, data, tmp, 0, nt0, dctr, st);
        else level_counts<RS>(ws, data, tmp, 0, nt0, dctr, st);
        k_check_seg0<<<1, 32, 0, st>>>(ws.seg_andor[0].p, ws.segs[0].p, ks, d_flag);
        note_launch();
        RG_LAUNCH_CHECK();
    };
    uint32_t nseg = 1, ntiles = nt0;
    if (!seeds) {
        level0_counts();
    } else {
        // level 0 = the caller's segments (bsegs -> segs[0] and the tile map,
        // as a progressive batch is rebased), AND/OR rows reset, no sampled
        // guess and no redo flag
        std::vector<Seg> hs(seeds->size());
        uint64_t at = 0;
        uint32_t tb = 0;
        for (size_t i = 0; i < seeds->size(); ++i) {
            const uint64_t sz = (*seeds)[i].size;
            hs[i] = Seg{at, sz, std::min((*seeds)[i].p, ks), 0, tb, 0};
            at += sz;
            tb += uint32_t((sz + TILE - 1) / TILE);
        }
        if (at != n) throw CudaError{RADULS_GPU_EINVAL};
        nseg = uint32_t(hs.size());
        ntiles = tb;
        ws.bsegs.ensure(nseg);
        RG_CHECK(cudaMemcpyAsync(ws.bsegs.p, hs.data(), nseg * sizeof(Seg), cudaMemcpyHostToDevice, st));
        RG_CHECK(cudaMemsetAsync(d_flag, 0, sizeof(unsigned long long), st));
        RG_CHECK(cudaMemsetAsync(ws.tile_seg[0].p, 0, size_t(ntiles) * sizeof(uint32_t), st));
        k_rebase_segs<<<nseg, 256, 0, st>>>(ws.bsegs.p, 0, ws.segs[0].p, ws.tile_seg[0].p, TILE);
        note_launch();
        RG_LAUNCH_CHECK();
        k_init_andor<<<(nseg * 8 + 255) / 256, 256, 0, st>>>(ws.seg_andor[0].p, nseg);
        note_launch();
        RG_LAUNCH_CHECK();
        RG_CHECK(cudaMemsetAsync(dctr, 0, sizeof(LevelCounters), st));
        if (ntiles) {
            if (ks <= 8) level_counts<RS, false, true>(ws, data, tmp, 0, ntiles, dctr, st);
            else level_counts<RS>(ws, data, tmp, 0, ntiles, dctr, st);
        }
        RG_CHECK(cudaStreamSynchronize(st));  // hs (host) is read by the copy above
    }
    const Caps caps = caps_for<RS>(n, seeds ? seeds->size() : 0);
    // Digit arrays: the scatter writes the next key byte of every record whose
    // child is split again, so the next level's histogram reads 1 byte, not
    // rs, and its scatter takes its digits from there too. Best effort:
    // without the 2n extra bytes every level reads whole records.
    constexpr int nd_halves = ScatterCfg<RS>::kNdSmem ? 2 : 1;
    const size_t nd_stride = digit_arrays(ws, n, nd_halves);
    RG_CHK_RANGES_ADD(st, {{ws.nd.p, nd_stride ? ws.nd.cap : 0}});
    const uint8_t* nd_in = nullptr;  // this level's digits (null: read from the records)
    int nd_half = 0;
    // The level loop from `level` on (its counters at dctr + level); returns the
    // level count reached. stop_after_first: return after this level's
    // launches with cur / nseg / ntiles / nd_in describing the next level,
    // before its histogram.
    uint32_t last_skip = 0;  // n_skip of the last level run
    auto run_levels = [&](uint32_t level, bool stop_after_first) -> uint32_t {
    while (true) {
        if (level >= uint32_t(kMaxLevels)) throw CudaError{RADULS_GPU_EINTERNAL};
        LevelCounters* c = dctr + level;
        PlanArgs A;
        A.segs = ws.segs[cur].p;
        A.seg_tot = ws.seg_tot[cur].p;
        A.seg_andor = ws.seg_andor[cur].p;
        A.groups = ws.groups.p;
        A.copies = ws.copies.p;
        A.next = ws.segs[cur ^ 1].p;
        A.next_andor = ws.seg_andor[cur ^ 1].p;
        A.next_tile_seg = ws.tile_seg[cur ^ 1].p;
        A.ctr = c;
        A.ks = ks;
        A.tile = TILE;
        A.cap_local = local_cap<RS>();
        A.cap_group = group_cap<RS>();
        A.side = nd_in ? 1u : 0u;
        pe = ws.prof.begin(K_PLAN, st);
        k_plan<<<nseg, 256, 0, st>>>(A);
        note_launch();
        RG_LAUNCH_CHECK();
        ws.prof.end(pe, st);
        publish(ws.h_ctr + level, c, sizeof(LevelCounters), st);
        if (level == 0) publish(ws.h_small + 4000, d_flag, sizeof(unsigned long long), st);
        RG_CHECK(cudaStreamSynchronize(st));
        if (level == 0 && ws.h_small[4000]) {  // a more significant byte varies off the sample: redo level 0 on it
            Seg s0{0, n, uint32_t(ws.h_small[4000] & 0xFF), 0, 0, 0};
            RG_CHECK(cudaMemcpyAsync(ws.segs[0].p, &s0, sizeof s0, cudaMemcpyHostToDevice, st));
            level0_counts();
            continue;
        }
        const LevelCounters h = ws.h_ctr[level];
        if (h.n_groups > caps.groups || h.n_copy > caps.copies || h.n_next > caps.seg ||
            h.n_next_tiles > caps.tiles)
            throw CudaError{RADULS_GPU_EINTERNAL};
        // the next level reads its digits from nd iff every one of its
        // segments comes out of this level's scatter (none re-queued at a
        // later byte without a split)
        uint8_t* nd_out =
            (nd_stride && h.n_next && !h.n_skip) ? ws.nd.p + (nd_halves == 2 ? nd_half : 0) * nd_stride : nullptr;
        if (h.n_scatter_segs) {
            launch_scatter<RS, false>(ws, data, tmp, cur, ntiles, ks, nullptr, c, st, nullptr, nd_out,
                                      nd_halves == 2 ? nd_in : nullptr);
            stats.scatter_launches++;
        }
        launch_local<RS>(ws, data, tmp, h.n_groups, ks, c, st, h.n_big_groups);
        if (h.n_copy) {
            pe = ws.prof.begin(K_COPY, st);
            k_copy_back<RS><<<h.n_copy, 256, 0, st>>>(data, tmp, ws.copies.p);
            note_launch();
            RG_LAUNCH_CHECK();
            ws.prof.end(pe, st);
        }
        stats.scatter_records += h.moved_scatter;
        stats.copy_records += h.moved_copy;
        stats.skipped_levels += nseg - h.n_scatter_segs;
        ++level;
        last_skip = h.n_skip;
        if (!h.n_next) break;
        cur ^= 1;
        nseg = h.n_next;
        ntiles = h.n_next_tiles;
        nd_in = nd_out;
        nd_half ^= 1;
        if (stop_after_first) break;
        RG_CHECK(cudaMemsetAsync(dctr + level, 0, sizeof(LevelCounters), st));
        if (ks <= 8) level_counts<RS, false, true>(ws, data, tmp, cur, ntiles, dctr + level, st, ks, nullptr, nd_in);
        else level_counts<RS>(ws, data, tmp, cur, ntiles, dctr + level, st, ks, nullptr, nd_in);
    }
    return level;
    };
    // per-level accounting known only once the level's local sorts ran
    auto add_level_stats = [&](uint32_t l0, uint32_t l1) {
        for (uint32_t l = l0; l < l1; ++l) {
            stats.local_records += ws.h_ctr[l].moved_local;
            stats.fallback_groups += ws.h_ctr[l].fallback_groups;
            stats.bitmap_spill_groups += ws.h_ctr[l].bm_spill;
            stats.hist_records += ws.h_ctr[l].hist_records;
            stats.hist_digit_records += ws.h_ctr[l].hist_digit_records;
        }
    };
    const uint64_t prog_min = [] {
        const char* e = std::getenv("RADULS_GPU_PROGRESSIVE_BYTES");
        return e ? std::strtoull(e, nullptr, 10) : (uint64_t(256) << 20);
    }();
    if (on_final && n * RS >= prog_min && !seeds) {
        // Progressive: level 0 over the whole array, then its children (one
        // parent: in digit order = key order, tiles in the same order) in
        // batches of contiguous key ranges, each sorted to the end before the
        // next starts, so each range is final — and handed to on_final —
        // while later ranges are still being sorted.
        uint32_t levels = run_levels(0, true);
        const bool split = levels == 1 && nseg >= 2 && !last_skip && ws.h_ctr[0].n_scatter_segs == 1;
        read_counters_and_finish<RS>(ws, data, tmp, ks, dctr, 1, st);
        add_level_stats(0, 1);
        RG_CHECK(cudaMemsetAsync(ws.n_spill.p, 0, 4 * sizeof(unsigned int), st));
        if (!split) {  // nothing to batch (level 0 finished it, or skipped a constant byte)
            if (nseg && levels == 1 && ws.h_ctr[0].n_next) {
                RG_CHECK(cudaMemsetAsync(dctr + 1, 0, sizeof(LevelCounters), st));
                if (ks <= 8) level_counts<RS, false, true>(ws, data, tmp, cur, ntiles, dctr + 1, st, ks, nullptr, nd_in);
                else level_counts<RS>(ws, data, tmp, cur, ntiles, dctr + 1, st, ks, nullptr, nd_in);
                levels = run_levels(1, false);
                read_counters_and_finish<RS>(ws, data, tmp, ks, dctr, levels, st);
                add_level_stats(1, levels);
            }
            (*on_final)(0, n);
        } else {
            std::vector<Seg> hs(nseg);
            RG_CHECK(cudaMemcpyAsync(hs.data(), ws.segs[cur].p, nseg * sizeof(Seg), cudaMemcpyDeviceToHost, st));
            ws.bsegs.ensure(nseg);
            RG_CHECK(cudaMemcpyAsync(ws.bsegs.p, ws.segs[cur].p, nseg * sizeof(Seg), cudaMemcpyDeviceToDevice, st));
            RG_CHECK(cudaStreamSynchronize(st));
            const int cur1 = cur;
            const uint32_t nseg1 = nseg, ntiles1 = ntiles;
            const uint8_t* nd_in1 = nd_in;
            const int nd_half1 = nd_half;
            const uint32_t K = std::min<uint32_t>(nseg1, kProgressiveBatches);
            for (uint32_t b = 0; b < K; ++b) {
                const uint32_t s0 = uint32_t(uint64_t(b) * nseg1 / K), s1 = uint32_t(uint64_t(b + 1) * nseg1 / K);
                const uint32_t tb0 = hs[s0].tile_base, tb1 = b + 1 < K ? hs[s1].tile_base : ntiles1;
                const uint64_t p0 = b ? hs[s0].start : 0, p1 = b + 1 < K ? hs[s1].start : n;
                cur = cur1;
                nseg = s1 - s0;
                ntiles = tb1 - tb0;
                nd_in = nd_in1;
                nd_half = nd_half1;
                k_rebase_segs<<<nseg, 256, 0, st>>>(ws.bsegs.p + s0, tb0, ws.segs[cur].p, ws.tile_seg[cur].p, TILE);
                note_launch();
                RG_LAUNCH_CHECK();
                k_init_andor<<<(nseg * 8 + 255) / 256, 256, 0, st>>>(ws.seg_andor[cur].p, nseg);
                note_launch();
                RG_LAUNCH_CHECK();
                RG_CHECK(cudaMemsetAsync(dctr + 1, 0, sizeof(LevelCounters), st));
                if (ks <= 8) level_counts<RS, false, true>(ws, data, tmp, cur, ntiles, dctr + 1, st, ks, nullptr, nd_in);
                else level_counts<RS>(ws, data, tmp, cur, ntiles, dctr + 1, st, ks, nullptr, nd_in);
                const uint32_t lv = run_levels(1, false);
                levels = std::max(levels, lv);
                read_counters_and_finish<RS>(ws, data, tmp, ks, dctr, lv, st);
                add_level_stats(1, lv);
                RG_CHECK(cudaMemsetAsync(ws.n_spill.p, 0, 4 * sizeof(unsigned int), st));
                (*on_final)(p0, p1);
            }
        }
        ws.prof.collect();
        stats.levels = levels;
        ws.last = stats;
        return;
    }
    const uint32_t level = run_levels(0, false);
    read_counters_and_finish<RS>(ws, data, tmp, ks, dctr, level, st);
    ws.prof.collect();
    stats.levels = level;
    add_level_stats(0, level);
    ws.last = stats;
}

template <typename F>
int guarded(F&& f) {
    cudaGetLastError();  // a stale non-sticky error (e.g. a caller's failed allocation) is not ours
    try {
#ifdef RG_CHECKED
        std::lock_guard<std::recursive_mutex> serial(g_chk_call);
        chk_begin();
        f();
        return chk_end();
#else
        f();
        return RADULS_GPU_OK;
#endif
    } catch (const CudaError& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        return RADULS_GPU_ENOMEM;
    } catch (...) {
        return RADULS_GPU_EINTERNAL;
    }
}

template <typename F>
void dispatch_rs(uint32_t rs, F&& f) {
    switch (rs) {
        case 8: f(std::integral_constant<int, 8>{}); break;
        case 16: f(std::integral_constant<int, 16>{}); break;
        case 24: f(std::integral_constant<int, 24>{}); break;
        case 32: f(std::integral_constant<int, 32>{}); break;
        default: throw CudaError{RADULS_GPU_EINVAL};
    }
}

bool mul_overflows(uint64_t n, uint32_t rs) { return n > (~uint64_t(0)) / rs; }

void zipf_thresholds(double s, uint32_t universe, unsigned long long* thr) {
    // identical arithmetic to oracle/raduls_oracle.c orc_zipf_thresholds (checked by tests)
    double run = 0.0, total = 0.0;
    for (uint32_t r = 1; r <= universe; ++r) total += std::pow(double(r), -s);
    for (uint32_t k = 0; k < universe; ++k) {
        run += std::pow(double(k + 1), -s);
        const double t = run / total * 9007199254740992.0;
        thr[k] = (k + 1 == universe) ? 9007199254740992ull : (unsigned long long)t;
    }
}

// ---- multi-GPU key-range partition, host side of
// raduls_gpu_sort_multi: the same plan as paper_1612_02557_b200/distributed.py
// (first globally varying byte, 16-bit prefix histograms, contiguous
// count-balanced bucket ranges), with the metadata combined in host memory and
// the records exchanged by peer copies over NVLink.
constexpr uint32_t kPrefixBuckets = 65536;

uint32_t first_varying_byte_multi(const std::vector<std::array<uint64_t, 8>>& ao, uint32_t ks) {
    uint64_t a[4] = {~0ull, ~0ull, ~0ull, ~0ull}, o[4] = {0, 0, 0, 0};
    for (const auto& x : ao)
        for (int w = 0; w < 4; ++w) a[w] &= x[2 * w], o[w] |= x[2 * w + 1];
    for (uint32_t b = 0; b < ks; ++b)
        if (((a[b >> 3] ^ o[b >> 3]) >> ((b & 7) * 8)) & 0xFF) return b;
    return ks;
}

// bucket b -> the device whose ideal share [r N/G, (r+1) N/G) holds the
// bucket's midpoint (monotone: each device gets a contiguous key range; a
// bucket is never split, so equal keys stay together)
std::vector<uint32_t> balanced_bucket_map_multi(const std::vector<uint64_t>& hist, uint32_t g) {
    std::vector<uint32_t> map(kPrefixBuckets, 0);
    double total = 0;
    for (uint64_t h : hist) total += double(h);
    if (total == 0) return map;
    double before = 0;
    for (uint32_t b = 0; b < kPrefixBuckets; ++b) {
        const double h = double(hist[b]);
        const double mid = before + h / 2.0;
        int64_t r = int64_t(std::floor(mid * g / total));
        map[b] = uint32_t(std::min<int64_t>(std::max<int64_t>(r, 0), g - 1));
        before += h;
    }
    return map;
}

// run f(i) for i in [0, n) on n host threads; returns the first nonzero status
template <typename F>
int run_per_device(int n, F&& f) {
    std::vector<int> rc(n, RADULS_GPU_OK);
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i) th.emplace_back([&, i] { rc[i] = f(i); });
    for (auto& t : th) t.join();
    for (int i = 0; i < n; ++i)
        if (rc[i] != RADULS_GPU_OK) return rc[i];
    return RADULS_GPU_OK;
}

// Frees the host drop-ins' device buffers when the call ends (normally or by
// an error) unless the caller opted into caching them.
struct HostBufs {
    Workspace& ws;
    explicit HostBufs(Workspace& w) : ws(w) {}
    ~HostBufs() {
        if (g_host_cache.load()) return;
        cudaDeviceSynchronize();  // the progressive copies may still read host_data
        ws.host_data.release();
        ws.host_tmp.release();
    }
};

// Device memory a host sort may use: free memory plus the cached host-path
// buffers (reused), or RADULS_GPU_DEVICE_BUDGET bytes when set (tests force
// the out-of-core path with it).
uint64_t device_budget() {
    if (const char* v = std::getenv("RADULS_GPU_DEVICE_BUDGET")) return std::strtoull(v, nullptr, 10);
    size_t free_b = 0, total_b = 0;
    RG_CHECK(cudaMemGetInfo(&free_b, &total_b));
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lk(ws.mu);
    return uint64_t(free_b) + ws.host_data.cap + ws.host_tmp.cap;
}

}  // namespace

extern "C" {

const char* raduls_gpu_strerror(int code) {
    switch (code) {
        case RADULS_GPU_OK: return "ok";
        case RADULS_GPU_EINVAL: return "invalid argument (unsupported record layout, misaligned pointer or size overflow)";
        case RADULS_GPU_ENOMEM: return "out of memory";
        case RADULS_GPU_ECUDA: return "CUDA runtime error";
        case RADULS_GPU_ENCCL: return "NCCL error";
        case RADULS_GPU_EINTERNAL: return "internal error (planner invariant)";
        default: return "unknown status";
    }
}

int raduls_gpu_layout_valid(uint32_t rs, uint32_t ks) { return layout_ok(rs, ks) ? 1 : 0; }

uint32_t raduls_gpu_version(void) { return 0x000200u; }  // 0x0200: raduls_gpu_stats + bitmap_spill_groups

int raduls_gpu_sort(void* d_data, void* d_tmp, uint64_t n, uint32_t rs, uint32_t ks, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n > kMaxRecords) return RADULS_GPU_EINVAL;
    if (n >= 2 && (!d_data || !aligned_ok(d_data, rs) || (d_tmp && !aligned_ok(d_tmp, rs))))
        return RADULS_GPU_EINVAL;
    if (n < 2) return RADULS_GPU_OK;  // msd_sorter.hpp:51: nothing to do, nothing allocated
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        uint8_t* tmp = static_cast<uint8_t*>(d_tmp);
        bool own = false;
        if (n >= 2 && !tmp) {
            RG_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * rs, st));
            own = true;
        }
        try {
            dispatch_rs(rs, [&](auto R) {
                sort_impl<decltype(R)::value>(ws, static_cast<uint8_t*>(d_data), tmp, n, ks, st);
            });
        } catch (...) {
            if (own) cudaFreeAsync(tmp, st);
            throw;
        }
        if (own) RG_CHECK(cudaFreeAsync(tmp, st));
        RG_CHECK(cudaStreamSynchronize(st));
    });
}

// Host sort larger than the device budget: the
// multi-GPU plan applied to parts of one array. (1) a streamed pass over
// chunks: AND/OR and the 16-bit prefix histogram at the first chunk's guess of
// the first varying key byte (a second histogram pass only if the guess was
// wrong); (2) contiguous bucket ranges packed greedily into parts that fit the
// device; (3) a streamed stable partition of every chunk into the host scratch
// `tmp` at each part's running offset; (4) each part to the device, sorted,
// back to its final place in `data`. PCIe traffic: 3 reads + 2 writes of the
// array (4 + 2 when the guess misses).
static int sort_host_out_of_core(uint8_t* data, uint8_t* htmp, uint64_t n, uint32_t rs, uint32_t ks,
                                 uint64_t budget) {
    return guarded([&] {
        {  // the in-core host path's cached device buffers are not needed
            Workspace& ws = workspace();
            std::lock_guard<std::mutex> lk(ws.mu);
            ws.host_data.release();
            ws.host_tmp.release();
        }
        const uint64_t reserve = std::min<uint64_t>(budget / 4, uint64_t(1) << 30);
        uint64_t P = (budget - reserve) / (2 * rs + rs / 8 + 1);  // records per part (+ tmp + workspace)
        P = std::min<uint64_t>(P, kMaxRecords);
        if (P < (uint64_t(1) << 16)) throw CudaError{RADULS_GPU_ENOMEM};
        std::unique_ptr<uint8_t[]> own_tmp;
        if (!htmp) {
            own_tmp.reset(new uint8_t[n * rs]);
            htmp = own_tmp.get();
        }
        uint8_t *A = nullptr, *B = nullptr;
        unsigned long long* d_hist = nullptr;
        uint32_t* d_map = nullptr;
        struct Free {
            uint8_t **a, **b;
            unsigned long long** h;
            uint32_t** m;
            ~Free() {
                cudaFree(*a);
                cudaFree(*b);
                cudaFree(*h);
                cudaFree(*m);
            }
        } fr{&A, &B, &d_hist, &d_map};
        RG_CHECK(cudaMalloc(&A, P * rs));
        RG_CHECK(cudaMalloc(&B, P * rs));
        RG_CHECK(cudaMalloc(&d_hist, kPrefixBuckets * sizeof(unsigned long long)));
        RG_CHECK(cudaMalloc(&d_map, kPrefixBuckets * sizeof(uint32_t)));
        HostStager hs;
        cudaStream_t st = nullptr;
        auto check = [](int r) {
            if (r) throw CudaError{r};
        };
        // (1) AND/OR + prefix histogram at the guessed byte
        uint64_t all[8];
        for (int w = 0; w < 8; ++w) all[w] = (w & 1) ? 0ull : ~0ull;
        uint32_t guess = 0;
        auto hist_pass = [&](uint32_t p, bool andor) {
            RG_CHECK(cudaMemset(d_hist, 0, kPrefixBuckets * sizeof(unsigned long long)));
            for (uint64_t off = 0; off < n; off += P) {
                const uint64_t c = std::min(P, n - off);
                hs.h2d(A, data + off * rs, c * rs, st);
                if (andor) {
                    uint64_t h[8];
                    check(raduls_gpu_andor(A, c, rs, h, st));
                    for (int w = 0; w < 8; ++w) all[w] = (w & 1) ? (all[w] | h[w]) : (all[w] & h[w]);
                    if (off == 0) {
                        std::vector<std::array<uint64_t, 8>> one(1);
                        std::memcpy(one[0].data(), h, sizeof h);
                        p = guess = std::min(first_varying_byte_multi(one, ks), ks - 1);
                    }
                }
                check(raduls_gpu_prefix_histogram(A, c, rs, ks, p, reinterpret_cast<uint64_t*>(d_hist), st));
            }
        };
        hist_pass(0, true);
        std::vector<std::array<uint64_t, 8>> tot(1);
        std::memcpy(tot[0].data(), all, sizeof all);
        const uint32_t p0 = first_varying_byte_multi(tot, ks);
        if (p0 >= ks) return;  // every key equal: the stable order is the input order
        if (p0 != guess) hist_pass(p0, false);
        std::vector<uint64_t> hist(kPrefixBuckets);
        RG_CHECK(cudaMemcpy(hist.data(), d_hist, kPrefixBuckets * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        // (2) parts: contiguous bucket ranges of <= P records
        // A bucket larger than P is a part of its own ("big"): its records
        // share the 16-bit prefix, and it is sorted afterwards by the same
        // out-of-core plan applied to its range (the next varying bytes).
        std::vector<uint32_t> map(kPrefixBuckets);
        std::vector<uint64_t> psz(1, 0);
        for (uint32_t b = 0; b < kPrefixBuckets; ++b) {
            const bool big = hist[b] > P;
            if (psz.back() && (big || psz.back() + hist[b] > P || psz.back() > P)) psz.push_back(0);
            map[b] = uint32_t(psz.size() - 1);
            psz.back() += hist[b];
        }
        const uint32_t K = uint32_t(psz.size());
        if (K > 256) throw CudaError{RADULS_GPU_ENOMEM};
        std::vector<uint64_t> poff(K, 0), written(K, 0);
        for (uint32_t k = 1; k < K; ++k) poff[k] = poff[k - 1] + psz[k - 1];
        RG_CHECK(cudaMemcpy(d_map, map.data(), kPrefixBuckets * sizeof(uint32_t), cudaMemcpyHostToDevice));
        check(raduls_gpu_set_pivots(0, nullptr, nullptr, ks));  // whole buckets only here
        // (3) stable partition of every chunk into the parts' host ranges
        std::vector<uint64_t> cnt(K);
        for (uint64_t off = 0; off < n; off += P) {
            const uint64_t c = std::min(P, n - off);
            hs.h2d(A, data + off * rs, c * rs, st);
            check(raduls_gpu_partition(A, B, c, rs, ks, p0, d_map, K, cnt.data(), st));
            uint64_t run = 0;
            for (uint32_t k = 0; k < K; ++k) {
                // a part never outgrows the size its histogram promised
                // (a mismatch would overlap the next part in htmp)
                if (written[k] + cnt[k] > psz[k]) throw CudaError{RADULS_GPU_EINTERNAL};
                if (cnt[k]) hs.d2h(htmp + (poff[k] + written[k]) * rs, B + run * rs, cnt[k] * rs, st);
                written[k] += cnt[k];
                run += cnt[k];
            }
        }
        for (uint32_t k = 0; k < K; ++k)
            if (written[k] != psz[k]) throw CudaError{RADULS_GPU_EINTERNAL};
        // (4) every part: to the device, sorted, to its place in data. From
        // here on data is overwritten part by part; if anything fails, the
        // parts not yet written are copied back from htmp unsorted, so data
        // still holds the input's records (a permutation) when the error returns.
        uint32_t k = 0;
        try {
            for (; k < K; ++k) {
                if (!psz[k] || psz[k] > P) continue;  // big parts below
                hs.h2d(A, htmp + poff[k] * rs, psz[k] * rs, st);
                check(raduls_gpu_sort(A, B, psz[k], rs, ks, st));
                hs.d2h(data + poff[k] * rs, A, psz[k] * rs, st);
            }
            RG_CHECK(cudaStreamSynchronize(st));
            cudaFree(A), cudaFree(B), A = B = nullptr;  // the big parts' own plans allocate theirs
            for (k = 0; k < K; ++k) {
                if (psz[k] <= P) continue;
                // sort the range in place in htmp with data's (already
                // consumed) range as its scratch, then move it to data
                check(sort_host_out_of_core(htmp + poff[k] * rs, data + poff[k] * rs, psz[k], rs, ks, budget));
                std::memcpy(data + poff[k] * rs, htmp + poff[k] * rs, psz[k] * rs);
            }
        } catch (...) {
            cudaDeviceSynchronize();
            for (uint32_t q = 0; q < K; ++q)
                if ((q >= k || psz[q] > P) && psz[q]) std::memcpy(data + poff[q] * rs, htmp + poff[q] * rs, psz[q] * rs);
            throw;
        }
    });
}

int raduls_gpu_sort_host(uint8_t* data, uint8_t* tmp, uint64_t n, uint32_t rs, uint32_t ks) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || mul_overflows(2 * n, rs)) return RADULS_GPU_EINVAL;
    if (n < 2) return RADULS_GPU_OK;
    if (!data) return RADULS_GPU_EINVAL;
    uint64_t budget = 0;
    const int rc = guarded([&] { budget = device_budget(); });
    if (rc) return rc;
    const uint64_t bytes = n * rs;
    if (n > kMaxRecords || 2 * bytes + bytes / 8 + (uint64_t(1) << 30) > budget)
        return sort_host_out_of_core(data, tmp, n, rs, ks, budget);
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        HostBufs hb(ws);
        const bool timing = std::getenv("RADULS_GPU_HOST_TIMING") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        const auto ta = now();
        ws.host_data.ensure(bytes);
        if (timing)
            std::fprintf(stderr, "raduls_gpu_sort_host: data buffer %.1f ms\n",
                         std::chrono::duration<double, std::milli>(now() - ta).count());
        cudaStream_t st = nullptr;
        HostStager& hs = ws.host_stager();
        const auto t0 = now();
        hs.h2d(ws.host_data.p, data, bytes, st);
        ws.host_tmp.ensure(bytes);  // (pinned input: mapped while the copy runs)
        if (timing) RG_CHECK(cudaStreamSynchronize(st));
        const auto t1 = now();
        // pinned buffers: each key range is copied back as soon as it is final
        // (progressive sort), overlapping the copy with the rest of the sort
        const bool pinned = HostStager::pinned(data);
        uint64_t covered = 0;
        std::function<void(uint64_t, uint64_t)> fin = [&](uint64_t a, uint64_t b) {
            RG_CHECK(cudaEventRecord(hs.done, st));
            RG_CHECK(cudaStreamWaitEvent(hs.copy, hs.done, 0));
            RG_CHECK(cudaMemcpyAsync(data + a * rs, ws.host_data.p + a * rs, (b - a) * rs, cudaMemcpyDeviceToHost,
                                     hs.copy));
            covered += b - a;
        };
        dispatch_rs(rs, [&](auto R) {
            sort_impl<decltype(R)::value>(ws, ws.host_data.p, ws.host_tmp.p, n, ks, st, pinned ? &fin : nullptr);
        });
        // every kernel has finished (sort_impl ends synchronised); only the
        // result's copies may still run: the scratch goes now, under them
        if (!g_host_cache.load()) ws.host_tmp.release();
        const auto t2 = now();
        if (covered) {  // the sort handed over its ranges (all of them)
            RG_CHECK(cudaStreamSynchronize(hs.copy));
            if (covered != n) throw CudaError{RADULS_GPU_EINTERNAL};
        } else {  // not a progressive sort (small, or pageable buffer): copy back now
            hs.d2h(data, ws.host_data.p, bytes, st);
        }
        RG_CHECK(cudaStreamSynchronize(st));
        if (timing) {
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "raduls_gpu_sort_host: h2d %.1f ms, sort %.1f ms, d2h tail %.1f ms%s\n",
                         ms(t0, t1), ms(t1, t2), ms(t2, now()), covered ? " (progressive)" : "");
        }
    });
}

int raduls_gpu_last_stats(raduls_gpu_stats* out) {
    if (!out) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        *out = ws.last;
    });
}

}  // extern "C"

namespace {
// One-segment helper: histogram + scan of the whole array on byte p (or the
// mapped prefix), digit bases on the host; returns totals in h_tot[256].
template <int RS, bool kMap>
void single_segment_counts(Workspace& ws, uint8_t* src, uint64_t n, uint32_t p, uint32_t ks,
                           const uint8_t* map, unsigned long long* h_tot, cudaStream_t st) {
    constexpr int TILE = ScatterCfg<RS>::kTile;
    ws.part.pending = false;
    ensure_caps<RS>(ws, n);
    set_attrs<RS>(ws);
    Seg s0{0, n, p, 0, 0, 0};
    RG_CHECK(cudaMemcpyAsync(ws.segs[0].p, &s0, sizeof s0, cudaMemcpyHostToDevice, st));
    const uint32_t nt = uint32_t((n + TILE - 1) / TILE);
    RG_CHECK(cudaMemsetAsync(ws.tile_seg[0].p, 0, nt * sizeof(uint32_t), st));
    k_init_andor<<<1, 64, 0, st>>>(ws.seg_andor[0].p, 1);
    note_launch();
    RG_LAUNCH_CHECK();
    RG_CHECK(cudaMemsetAsync(ws.ctr.p, 0, sizeof(LevelCounters), st));
    level_counts<RS, kMap>(ws, src, src, 0, nt, ws.ctr.p, st, ks, map);
    RG_CHECK(cudaMemcpyAsync(h_tot, ws.seg_tot[0].p, kRadix * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             st));
    RG_CHECK(cudaStreamSynchronize(st));
}

// Scatter the single segment prepared by single_segment_counts from src into dst.
template <int RS, bool kMap, bool kPeer = false>
void single_segment_scatter(Workspace& ws, uint8_t* src, uint8_t* dst, uint64_t n, uint32_t ks,
                            const uint8_t* map, const unsigned long long* h_tot, cudaStream_t st,
                            const unsigned long long* dig_dst = nullptr, bool stable_ballot = false,
                            const Piece* pieces = nullptr) {
    constexpr int TILE = ScatterCfg<RS>::kTile;
    unsigned long long* off = ws.h_small + 1024;
    unsigned long long run = 0;
    for (int d = 0; d < 256; ++d) off[d] = run, run += h_tot[d];
    RG_CHECK(cudaMemcpyAsync(ws.seg_tot[0].p, off, kRadix * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                             st));
    const uint32_t act = kActScatter;
    RG_CHECK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(ws.segs[0].p) + offsetof(Seg, action), &act,
                             sizeof act, cudaMemcpyHostToDevice, st));
    const uint32_t nt = uint32_t((n + TILE - 1) / TILE);
    launch_scatter<RS, kMap, kPeer>(ws, src, dst, 0, nt, ks, map, ws.ctr.p, st, dig_dst, nullptr, nullptr,
                                    stable_ballot, pieces);
    RG_CHECK(cudaStreamSynchronize(st));
}

// LSD baseline (reference lsd_sort, P/src/lsd.cpp:12-35): ks stable splits
// from the least to the most significant key byte, ping-ponging between data
// and tmp; a byte whose split would not move anything (one digit holds every
// record) is skipped. Same stable result as the MSD sort.
template <int RS>
void lsd_impl(Workspace& ws, uint8_t* data, uint8_t* tmp, uint64_t n, uint32_t ks, cudaStream_t st) {
    uint8_t* src = data;
    uint8_t* dst = tmp;
    RG_CHK_RANGES(st, {{data, size_t(n) * RS}, {tmp, size_t(n) * RS}});
    for (uint32_t pass = 0; pass < ks; ++pass) {
        const uint32_t byte = ks - 1 - pass;
        unsigned long long* tot = ws.h_small;
        single_segment_counts<RS, false>(ws, src, n, byte, ks, nullptr, tot, st);
        bool moves = true;
        for (int d = 0; d < 256; ++d)
            if (tot[d] == n) moves = false;
        if (!moves) continue;
        single_segment_scatter<RS, false>(ws, src, dst, n, ks, nullptr, tot, st, nullptr, true);
        std::swap(src, dst);
    }
    if (src != data) RG_CHECK(cudaMemcpyAsync(data, src, n * RS, cudaMemcpyDeviceToDevice, st));
}


}  // namespace

extern "C" {

int raduls_gpu_lsd_sort(void* d_data, void* d_tmp, uint64_t n, uint32_t rs, uint32_t ks, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n > kMaxRecords) return RADULS_GPU_EINVAL;
    if (n >= 2 && (!d_data || !aligned_ok(d_data, rs) || (d_tmp && !aligned_ok(d_tmp, rs))))
        return RADULS_GPU_EINVAL;
    if (n < 2) return RADULS_GPU_OK;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        uint8_t* tmp = static_cast<uint8_t*>(d_tmp);
        bool own = false;
        if (!tmp) {
            RG_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * rs, st));
            own = true;
        }
        try {
            dispatch_rs(rs, [&](auto R) {
                lsd_impl<decltype(R)::value>(ws, static_cast<uint8_t*>(d_data), tmp, n, ks, st);
            });
        } catch (...) {
            if (own) cudaFreeAsync(tmp, st);
            throw;
        }
        if (own) RG_CHECK(cudaFreeAsync(tmp, st));
        RG_CHECK(cudaStreamSynchronize(st));
    });
}

int raduls_gpu_lsd_sort_host(uint8_t* data, uint8_t* /*tmp*/, uint64_t n, uint32_t rs, uint32_t ks) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n > kMaxRecords) return RADULS_GPU_EINVAL;
    if (n < 2) return RADULS_GPU_OK;
    if (!data) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        const size_t bytes = size_t(n) * rs;
        HostBufs hb(ws);
        ws.host_data.ensure(bytes);
        ws.host_tmp.ensure(bytes);
        cudaStream_t st = nullptr;
        HostStager& hs = ws.host_stager();
        hs.h2d(ws.host_data.p, data, bytes, st);
        dispatch_rs(rs, [&](auto R) {
            lsd_impl<decltype(R)::value>(ws, ws.host_data.p, ws.host_tmp.p, n, ks, st);
        });
        hs.d2h(data, ws.host_data.p, bytes, st);
        RG_CHECK(cudaStreamSynchronize(st));
    });
}


int raduls_gpu_sort_segments(void* d_data, void* d_tmp, uint64_t n, uint32_t rs, uint32_t ks, uint32_t n_segs,
                             const uint64_t* h_sizes, const uint8_t* h_first_byte, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n > kMaxRecords || (n_segs && (!h_sizes || !h_first_byte)))
        return RADULS_GPU_EINVAL;
    if (n >= 2 && (!d_data || !aligned_ok(d_data, rs) || (d_tmp && !aligned_ok(d_tmp, rs)))) return RADULS_GPU_EINVAL;
    std::vector<SegSeed> seeds;
    uint64_t total = 0;
    for (uint32_t i = 0; i < n_segs; ++i) {
        total += h_sizes[i];
        if (h_sizes[i]) seeds.push_back(SegSeed{h_sizes[i], h_first_byte[i]});
    }
    if (total != n) return RADULS_GPU_EINVAL;
    if (n < 2) return RADULS_GPU_OK;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        uint8_t* tmp = static_cast<uint8_t*>(d_tmp);
        bool own = false;
        if (!tmp) {
            RG_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * rs, st));
            own = true;
        }
        try {
            dispatch_rs(rs, [&](auto R) {
                sort_impl<decltype(R)::value>(ws, static_cast<uint8_t*>(d_data), tmp, n, ks, st, nullptr,
                                              seeds.size() > 1 ? &seeds : nullptr);
            });
        } catch (...) {
            if (own) cudaFreeAsync(tmp, st);
            throw;
        }
        if (own) RG_CHECK(cudaFreeAsync(tmp, st));
        RG_CHECK(cudaStreamSynchronize(st));
    });
}

int raduls_gpu_split(const void* d_src, void* d_dst, uint64_t n, uint32_t rs,
                     uint32_t key_byte_offset, uint64_t* h_counts, void* stream) {
    if (!layout_ok(rs, rs) || key_byte_offset >= rs || mul_overflows(n, rs) || n > kMaxRecords)
        return RADULS_GPU_EINVAL;
    if (n && (!aligned_ok(d_src, rs) || !aligned_ok(d_dst, rs))) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (h_counts) std::memset(h_counts, 0, 256 * sizeof(uint64_t));
        if (n == 0) return;
        RG_CHK_RANGES(st, {{d_src, size_t(n) * rs}, {d_dst, size_t(n) * rs}});
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src));
            unsigned long long* tot = ws.h_small;
            single_segment_counts<RSC, false>(ws, src, n, key_byte_offset, rs, nullptr, tot, st);
            if (h_counts) std::memcpy(h_counts, tot, 256 * sizeof(uint64_t));
            single_segment_scatter<RSC, false>(ws, src, static_cast<uint8_t*>(d_dst), n, rs, nullptr, tot, st,
                                               nullptr, true);
        });
    });
}

int raduls_gpu_histogram(const void* d_data, uint64_t n, uint32_t rs, uint32_t ks, uint64_t* h_hist,
                         uint64_t* h_andor, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n > kMaxRecords) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (h_hist) std::memset(h_hist, 0, 8 * 256 * sizeof(uint64_t));
        if (h_andor)
            for (int w = 0; w < 8; ++w) h_andor[w] = (w & 1) ? 0ull : ~0ull;
        if (!n) return;
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_data));
            for (uint32_t b = 0; b < std::min<uint32_t>(ks, 8); ++b) {
                single_segment_counts<RSC, false>(ws, src, n, b, ks, nullptr, ws.h_small, st);
                if (h_hist) std::memcpy(h_hist + 256 * b, ws.h_small, 256 * sizeof(uint64_t));
            }
            RG_CHECK(cudaMemcpyAsync(ws.h_small, ws.seg_andor[0].p, 8 * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, st));
            RG_CHECK(cudaStreamSynchronize(st));
            if (h_andor) std::memcpy(h_andor, ws.h_small, 8 * sizeof(uint64_t));
        });
    });
}

int raduls_gpu_generate(void* d_out, uint64_t n, uint32_t rs, uint32_t ks, uint32_t dist, uint64_t seed,
                        uint64_t index_base, void* stream) {
    if (!layout_ok(rs, ks) || dist > 1 || mul_overflows(n, rs)) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_out, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!n) return;
        if (dist == 1) {
            zipf_thresholds(1.2, 256, ws.h_small);
            RG_CHECK(cudaMemcpyAsync(ws.thr.p, ws.h_small, 256 * sizeof(unsigned long long),
                                     cudaMemcpyHostToDevice, st));
        }
        GenParams P{n, seed, index_base, ks, dist, ws.thr.p};
        RG_CHK_RANGES(st, {{d_out, size_t(n) * rs}});
        dispatch_rs(rs, [&](auto R) {
            k_gen<decltype(R)::value><<<grid_for(n, 256, 16), 256, 0, st>>>(static_cast<uint8_t*>(d_out), P);
            note_launch();
        });
        RG_LAUNCH_CHECK();
        RG_CHECK(cudaStreamSynchronize(st));  // thresholds live in pinned scratch
    });
}

int raduls_gpu_digest(const void* d_data, uint64_t n, uint32_t rs, uint64_t* lo, uint64_t* hi,
                      void* stream) {
    if (!layout_ok(rs, rs) || mul_overflows(n, rs)) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        RG_CHECK(cudaMemsetAsync(ws.acc.p, 0, 2 * sizeof(unsigned long long), st));
        RG_CHK_RANGES(st, {{d_data, size_t(n) * rs}});
        if (n) {
            dispatch_rs(rs, [&](auto R) {
                k_digest<decltype(R)::value><<<grid_for(n, 256, 8), 256, 0, st>>>(
                    static_cast<const uint8_t*>(d_data), n, ws.acc.p);
                note_launch();
            });
            RG_LAUNCH_CHECK();
        }
        RG_CHECK(cudaMemcpyAsync(ws.h_small, ws.acc.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        RG_CHECK(cudaStreamSynchronize(st));
        *lo = ws.h_small[0];
        *hi = ws.h_small[1];
    });
}

int raduls_gpu_check_sorted(const void* d_data, uint64_t n, uint32_t rs, uint32_t ks, uint64_t* violations,
                            uint64_t* first, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs)) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        unsigned long long init[2] = {0ull, ~0ull};
        RG_CHECK(cudaMemcpyAsync(ws.acc.p, init, sizeof init, cudaMemcpyHostToDevice, st));
        RG_CHK_RANGES(st, {{d_data, size_t(n) * rs}});
        if (n > 1) {
            dispatch_rs(rs, [&](auto R) {
                k_check_sorted<decltype(R)::value><<<grid_for(n, 256, 8), 256, 0, st>>>(
                    static_cast<const uint8_t*>(d_data), n, ks, ws.acc.p);
                note_launch();
            });
            RG_LAUNCH_CHECK();
        }
        RG_CHECK(cudaMemcpyAsync(ws.h_small, ws.acc.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        RG_CHECK(cudaStreamSynchronize(st));
        if (violations) *violations = ws.h_small[0];
        if (first) *first = ws.h_small[1];
    });
}

int raduls_gpu_prefix_histogram(const void* d_data, uint64_t n, uint32_t rs, uint32_t ks,
                                uint32_t prefix_byte, uint64_t* d_hist, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || !d_hist) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!n) return;
        dispatch_rs(rs, [&](auto R) {
            k_prefix_hist<decltype(R)::value><<<grid_for(n, 256, 8), 256, 0, st>>>(
                static_cast<const uint8_t*>(d_data), n, ks, prefix_byte,
                reinterpret_cast<unsigned long long*>(d_hist));
            note_launch();
        });
        RG_LAUNCH_CHECK();
    });
}

// Load the bucket -> rank map (u8) plus the pivot region and check them;
// false when an entry (or a pivot digit + 2) is >= n_ranks. Asynchronous up to
// the final check.
static bool load_rank_map(Workspace& ws, const uint32_t* d_bucket_rank, uint32_t n_ranks, cudaStream_t st) {
    if (ws.map8.cap < kMapBytes) ws.map8.ensure(kMapBytes);
    if (ws.n_pivots && ws.pivot_max_digit + 2 >= n_ranks) return false;
    RG_CHECK(cudaMemsetAsync(ws.acc.p, 0, sizeof(unsigned long long), st));
    k_map_to_u8<<<256, 256, 0, st>>>(d_bucket_rank, ws.map8.p, n_ranks, reinterpret_cast<unsigned int*>(ws.acc.p));
    note_launch();
    RG_LAUNCH_CHECK();
    unsigned char* hp = reinterpret_cast<unsigned char*>(ws.h_small + 3328);  // pinned staging (6 KB free)
    std::memcpy(hp, ws.pivots.data(), ws.pivots.size());
    RG_CHECK(cudaMemcpyAsync(ws.map8.p + kMapPivotSlot, hp, ws.pivots.size(), cudaMemcpyHostToDevice, st));
    RG_CHECK(cudaMemcpyAsync(ws.h_small + 2048, ws.acc.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    RG_CHECK(cudaStreamSynchronize(st));
    return uint32_t(ws.h_small[2048]) == 0;
}

int raduls_gpu_partition(const void* d_src, void* d_dst, uint64_t n, uint32_t rs, uint32_t ks,
                         uint32_t prefix_byte, const uint32_t* d_bucket_rank, uint32_t n_ranks,
                         uint64_t* h_rank_counts, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n_ranks < 1 || n_ranks > 256 || !d_bucket_rank ||
        n > kMaxRecords)
        return RADULS_GPU_EINVAL;
    if (n && (!aligned_ok(d_src, rs) || !aligned_ok(d_dst, rs))) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (h_rank_counts) std::memset(h_rank_counts, 0, n_ranks * sizeof(uint64_t));
        if (!load_rank_map(ws, d_bucket_rank, n_ranks, st)) throw CudaError{RADULS_GPU_EINVAL};
        if (!n) return;
        RG_CHK_RANGES(st, {{d_src, size_t(n) * rs}, {d_dst, size_t(n) * rs}});
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src));
            unsigned long long* tot = ws.h_small;
            single_segment_counts<RSC, true>(ws, src, n, prefix_byte, ks, ws.map8.p, tot, st);
            if (h_rank_counts) std::memcpy(h_rank_counts, tot, n_ranks * sizeof(uint64_t));
            single_segment_scatter<RSC, true>(ws, src, static_cast<uint8_t*>(d_dst), n, ks, ws.map8.p, tot, st);
        });
    });
}

int raduls_gpu_partition_to(const void* d_src, uint64_t n, uint32_t rs, uint32_t ks, uint32_t prefix_byte,
                            const uint32_t* d_bucket_rank, uint32_t n_ranks, const uint64_t* h_dst,
                            uint64_t* h_rank_counts, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n_ranks < 1 || n_ranks > 256 || !d_bucket_rank ||
        !h_dst || n > kMaxRecords)
        return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_src, rs)) return RADULS_GPU_EINVAL;
    for (uint32_t r = 0; r < n_ranks; ++r)
        if (h_dst[r] % (rs % 16 == 0 ? 16 : 8)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (h_rank_counts) std::memset(h_rank_counts, 0, n_ranks * sizeof(uint64_t));
        ws.dig_dst.ensure(kRadix);
        if (!load_rank_map(ws, d_bucket_rank, n_ranks, st)) throw CudaError{RADULS_GPU_EINVAL};
        unsigned long long* hd = ws.h_small + 3072;  // pinned staging for the destinations
        for (uint32_t r = 0; r < kRadix; ++r) hd[r] = r < n_ranks ? h_dst[r] : 0ull;
        RG_CHECK(cudaMemcpyAsync(ws.dig_dst.p, hd, kRadix * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
        if (!n) return;
#ifdef RG_CHECKED
        {
            std::vector<std::pair<const void*, size_t>> rr{{d_src, size_t(n) * rs}};
            for (uint32_t r = 0; r < n_ranks; ++r) rr.emplace_back(reinterpret_cast<const void*>(h_dst[r]), size_t(n) * rs);
            RG_CHK_RANGES_VEC(st, rr);
        }
#endif
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src));
            unsigned long long* tot = ws.h_small;
            single_segment_counts<RSC, true>(ws, src, n, prefix_byte, ks, ws.map8.p, tot, st);
            if (h_rank_counts) std::memcpy(h_rank_counts, tot, n_ranks * sizeof(uint64_t));
            single_segment_scatter<RSC, true, true>(ws, src, nullptr, n, ks, ws.map8.p, tot, st, ws.dig_dst.p);
        });
    });
}

int raduls_gpu_partition_plan(const void* d_src, uint64_t n, uint32_t rs, uint32_t ks, uint32_t prefix_byte,
                              const uint32_t* d_bucket_rank, uint32_t n_ranks, uint64_t* h_rank_counts,
                              uint64_t* h_andor, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n_ranks < 1 || n_ranks > 256 || !d_bucket_rank ||
        !h_rank_counts || !h_andor || n > kMaxRecords)
        return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_src, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        ws.part.pending = false;
        std::memset(h_rank_counts, 0, n_ranks * sizeof(uint64_t));
        for (int w = 0; w < 8; ++w) h_andor[w] = (w & 1) ? 0ull : ~0ull;
        if (!load_rank_map(ws, d_bucket_rank, n_ranks, st)) throw CudaError{RADULS_GPU_EINVAL};
        if (!n) return;
        RG_CHK_RANGES(st, {{d_src, size_t(n) * rs}});
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src));
            single_segment_counts<RSC, true>(ws, src, n, prefix_byte, ks, ws.map8.p, ws.part.tot, st);
        });
        RG_CHECK(cudaMemcpyAsync(ws.h_small + 2048, ws.seg_andor[0].p, 8 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, st));
        RG_CHECK(cudaStreamSynchronize(st));
        std::memcpy(h_andor, ws.h_small + 2048, 8 * sizeof(uint64_t));
        std::memcpy(h_rank_counts, ws.part.tot, n_ranks * sizeof(uint64_t));
        ws.part.pending = true;
        ws.part.src = d_src;
        ws.part.n = n;
        ws.part.rs = rs;
        ws.part.ks = ks;
    });
}

int raduls_gpu_partition_store(const void* d_src, uint64_t n, uint32_t rs, uint32_t ks, const uint64_t* h_dst,
                               void* stream) {
    if (!layout_ok(rs, ks) || !h_dst) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!n) return;
        if (!ws.part.pending || ws.part.src != d_src || ws.part.n != n || ws.part.rs != rs || ws.part.ks != ks)
            throw CudaError{RADULS_GPU_EINVAL};  // no matching plan on this device
        ws.part.pending = false;
        ws.dig_dst.ensure(kRadix);
        unsigned long long* hd = ws.h_small + 3072;  // pinned staging for the destinations
        for (uint32_t r = 0; r < kRadix; ++r) {
            hd[r] = ws.part.tot[r] ? h_dst[r] : 0ull;  // ranks without records: never dereferenced
            if (hd[r] % (rs % 16 == 0 ? 16 : 8)) throw CudaError{RADULS_GPU_EINVAL};
        }
        RG_CHECK(cudaMemcpyAsync(ws.dig_dst.p, hd, kRadix * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
#ifdef RG_CHECKED
        {
            std::vector<std::pair<const void*, size_t>> rr{{d_src, size_t(n) * rs}};
            for (uint32_t r = 0; r < kRadix; ++r)
                if (ws.part.tot[r]) rr.emplace_back(reinterpret_cast<const void*>(h_dst[r]), ws.part.tot[r] * rs);
            RG_CHK_RANGES_VEC(st, rr);
        }
#endif
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src));
            single_segment_scatter<RSC, true, true>(ws, src, nullptr, n, ks, ws.map8.p, ws.part.tot, st,
                                                    ws.dig_dst.p);
        });
    });
}

int raduls_gpu_partition_store_pieces(const void* d_src, uint64_t n, uint32_t rs, uint32_t ks, uint32_t n_pieces,
                                      const uint32_t* h_piece_digit, const uint64_t* h_piece_count,
                                      const uint64_t* h_piece_dst, void* stream) {
    if (!layout_ok(rs, ks) || (n_pieces && (!h_piece_digit || !h_piece_count || !h_piece_dst)))
        return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!n) return;
        if (!ws.part.pending || ws.part.src != d_src || ws.part.n != n || ws.part.rs != rs || ws.part.ks != ks)
            throw CudaError{RADULS_GPU_EINVAL};  // no matching plan on this device
        // pieces in digit order; every digit's pieces add up to its planned count
        const uint32_t align = rs % 16 == 0 ? 16 : 8;
        std::vector<Piece> table;
        unsigned long long* hd = ws.h_small + 3072;  // pinned staging for the destinations
        for (uint32_t d = 0; d < kRadix; ++d) hd[d] = 0ull;
        std::vector<uint64_t> sum(kRadix, 0);
        uint32_t i = 0;
        int last = -1;
        while (i < n_pieces) {
            const uint32_t d = h_piece_digit[i];
            if (d >= kRadix || int(d) <= last) throw CudaError{RADULS_GPU_EINVAL};
            last = int(d);
            uint32_t j = i;
            while (j < n_pieces && h_piece_digit[j] == d) ++j;
            for (uint32_t k = i; k < j; ++k) {
                if (h_piece_dst[k] % align) throw CudaError{RADULS_GPU_EINVAL};
                sum[d] += h_piece_count[k];
            }
            if (j - i == 1) {
                hd[d] = h_piece_dst[i];
            } else {
                hd[d] = (1ull << 63) | (uint64_t(table.size()) << 32);
                uint64_t start = 0;
                for (uint32_t k = i; k < j; ++k) {
                    if (!h_piece_count[k]) continue;
                    table.push_back(Piece{start + h_piece_count[k], h_piece_dst[k] - start * rs});
                    start += h_piece_count[k];
                }
                if (table.empty() || (table.back().end != sum[d])) throw CudaError{RADULS_GPU_EINVAL};
            }
            i = j;
        }
        for (uint32_t d = 0; d < kRadix; ++d)
            if (sum[d] != ws.part.tot[d]) throw CudaError{RADULS_GPU_EINVAL};  // pieces != the plan's counts
        ws.part.pending = false;
        ws.dig_dst.ensure(kRadix);
        RG_CHECK(cudaMemcpyAsync(ws.dig_dst.p, hd, kRadix * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
#ifdef RG_CHECKED
        {
            std::vector<std::pair<const void*, size_t>> rr{{d_src, size_t(n) * rs}};
            for (uint32_t k = 0; k < n_pieces; ++k)
                if (h_piece_count[k])
                    rr.emplace_back(reinterpret_cast<const void*>(h_piece_dst[k]), h_piece_count[k] * rs);
            RG_CHK_RANGES_VEC(st, rr);
        }
#endif
        if (!table.empty()) {
            ws.pieces.ensure(table.size());
            RG_CHECK(cudaMemcpyAsync(ws.pieces.p, table.data(), table.size() * sizeof(Piece), cudaMemcpyHostToDevice,
                                     st));
        }
        dispatch_rs(rs, [&](auto R) {
            constexpr int RSC = decltype(R)::value;
            uint8_t* src = const_cast<uint8_t*>(static_cast<const uint8_t*>(d_src));
            single_segment_scatter<RSC, true, true>(ws, src, nullptr, n, ks, ws.map8.p, ws.part.tot, st,
                                                    ws.dig_dst.p, false, table.empty() ? nullptr : ws.pieces.p);
        });
    });
}

int raduls_gpu_digit_andor(const void* d_src, uint64_t n, uint32_t rs, uint32_t ks, uint32_t prefix_byte,
                           const uint32_t* d_bucket_digit, uint32_t n_digits, const uint8_t* h_hot,
                           uint64_t* h_andor, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || n_digits < 1 || n_digits > 256 || !d_bucket_digit ||
        !h_hot || !h_andor)
        return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_src, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        for (uint32_t d = 0; d < n_digits; ++d)
            for (int w = 0; w < 8; ++w) h_andor[8 * d + w] = (w & 1) ? 0ull : ~0ull;
        // hot digits -> compact slots
        uint8_t* hslot = reinterpret_cast<uint8_t*>(ws.h_small + 3584);  // pinned, 256 B
        std::vector<uint32_t> slot_digit;
        for (uint32_t d = 0; d < kRadix; ++d) {
            hslot[d] = 0;
            if (d < n_digits && h_hot[d]) {
                if (slot_digit.size() >= size_t(kHotSlots)) throw CudaError{RADULS_GPU_EINVAL};
                slot_digit.push_back(d);
                hslot[d] = uint8_t(slot_digit.size());
            }
        }
        ws.part.pending = false;  // the bucket map below replaces a pending plan's
        if (!load_rank_map(ws, d_bucket_digit, n_digits, st)) throw CudaError{RADULS_GPU_EINVAL};
        if (!n || slot_digit.empty()) return;
        ws.hot.ensure(256 + kHotSlots * 8 * 8);
        uint8_t* d_hot = reinterpret_cast<uint8_t*>(ws.hot.p);
        unsigned long long* d_out = ws.hot.p + 32;
        unsigned long long* init = ws.h_small + 2304;  // pinned [kHotSlots * 8]
        for (int i = 0; i < kHotSlots * 8; ++i) init[i] = (i & 1) ? 0ull : ~0ull;
        RG_CHECK(cudaMemcpyAsync(d_hot, hslot, 256, cudaMemcpyHostToDevice, st));
        RG_CHECK(cudaMemcpyAsync(d_out, init, kHotSlots * 8 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                                 st));
        dispatch_rs(rs, [&](auto R) {
            k_digit_andor<decltype(R)::value><<<grid_for(n, 256, 8), 256, 0, st>>>(
                static_cast<const uint8_t*>(d_src), n, ks, prefix_byte, ws.map8.p, d_hot, d_out);
            note_launch();
        });
        RG_LAUNCH_CHECK();
        RG_CHECK(cudaMemcpyAsync(init, d_out, kHotSlots * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        RG_CHECK(cudaStreamSynchronize(st));
        for (size_t k = 0; k < slot_digit.size(); ++k)
            for (int w = 0; w < 8; ++w) h_andor[8 * slot_digit[k] + w] = init[8 * k + w];
    });
}

int raduls_gpu_sample_andor(const void* d_data, uint64_t n, uint32_t rs, uint32_t samples, uint64_t* h_andor,
                            void* stream) {
    if (!layout_ok(rs, rs) || mul_overflows(n, rs) || !h_andor) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        k_init_andor<<<1, 64, 0, st>>>(ws.andor0.p, 1);
        note_launch();
        RG_LAUNCH_CHECK();
        const uint32_t sm = uint32_t(std::min<uint64_t>(n, std::max<uint32_t>(samples, 1)));
        if (n) {
            dispatch_rs(rs, [&](auto R) {
                k_sample_andor<decltype(R)::value><<<64, 256, 0, st>>>(
                    static_cast<const uint8_t*>(d_data), n, std::max<uint64_t>(1, n / sm), sm, ws.andor0.p);
                note_launch();
            });
            RG_LAUNCH_CHECK();
        }
        RG_CHECK(cudaMemcpyAsync(ws.h_small, ws.andor0.p, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        RG_CHECK(cudaStreamSynchronize(st));
        std::memcpy(h_andor, ws.h_small, 8 * sizeof(uint64_t));
    });
}

int raduls_gpu_sample_prefix_histogram(const void* d_data, uint64_t n, uint32_t rs, uint32_t ks,
                                       uint32_t prefix_byte, uint32_t samples, uint64_t* d_hist, void* stream) {
    if (!layout_ok(rs, ks) || mul_overflows(n, rs) || !d_hist) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!n || !samples) return;
        const uint32_t sm = uint32_t(std::min<uint64_t>(n, samples));
        dispatch_rs(rs, [&](auto R) {
            k_sample_prefix_hist<decltype(R)::value><<<grid_for(sm, 256, 4), 256, 0, st>>>(
                static_cast<const uint8_t*>(d_data), n, std::max<uint64_t>(1, n / sm), sm, ks, prefix_byte,
                reinterpret_cast<unsigned long long*>(d_hist));
            note_launch();
        });
        RG_LAUNCH_CHECK();
    });
}

int raduls_gpu_ipc_alloc(uint64_t bytes, void** d_ptr, uint8_t* handle) {
    if (!d_ptr || !handle) return RADULS_GPU_EINVAL;
    return guarded([&] {
        void* p = nullptr;
        RG_CHECK(cudaMalloc(&p, std::max<uint64_t>(bytes, 256)));
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            throw CudaError{RADULS_GPU_ECUDA};
        }
        std::memcpy(handle, &h, sizeof h);
        *d_ptr = p;
    });
}

int raduls_gpu_ipc_open(const uint8_t* handle, void** d_ptr) {
    if (!d_ptr || !handle) return RADULS_GPU_EINVAL;
    return guarded([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        RG_CHECK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int raduls_gpu_ipc_close(void* d_ptr) {
    return guarded([&] { RG_CHECK(cudaIpcCloseMemHandle(d_ptr)); });
}

int raduls_gpu_free(void* d_ptr) {
    return guarded([&] { RG_CHECK(cudaFree(d_ptr)); });
}

int raduls_gpu_andor(const void* d_data, uint64_t n, uint32_t rs, uint64_t* h_andor, void* stream) {
    if (!layout_ok(rs, rs) || mul_overflows(n, rs) || !h_andor) return RADULS_GPU_EINVAL;
    if (n && !aligned_ok(d_data, rs)) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        k_init_andor<<<1, 64, 0, st>>>(ws.andor0.p, 1);
        note_launch();
        RG_LAUNCH_CHECK();
        if (n) {
            dispatch_rs(rs, [&](auto R) {
                k_andor<decltype(R)::value><<<grid_for(n, 256, 8), 256, 0, st>>>(
                    static_cast<const uint8_t*>(d_data), n, ws.andor0.p);
                note_launch();
            });
            RG_LAUNCH_CHECK();
        }
        RG_CHECK(cudaMemcpyAsync(ws.h_small, ws.andor0.p, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        RG_CHECK(cudaStreamSynchronize(st));
        std::memcpy(h_andor, ws.h_small, 8 * sizeof(uint64_t));
    });
}

int raduls_gpu_set_profiling(int on) {
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        ws.prof.on = on != 0;
    });
}

int raduls_gpu_set_pivots(uint32_t n_pivots, const uint32_t* digits, const uint8_t* keys, uint32_t ks) {
    if (n_pivots > kMaxPivots || ks < 1 || ks > 32 || (n_pivots && (!digits || !keys))) return RADULS_GPU_EINVAL;
    for (uint32_t i = 0; i < n_pivots; ++i) {
        if (digits[i] + 2 > 255) return RADULS_GPU_EINVAL;
        for (uint32_t j = 0; j < i; ++j)  // a pivot digit and its two successors belong to one pivot
            if (digits[i] + 2 >= digits[j] && digits[j] + 2 >= digits[i]) return RADULS_GPU_EINVAL;
    }
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        ws.pivots.fill(0);
        ws.pivot_max_digit = 0;
        for (uint32_t i = 0; i < n_pivots; ++i) {
            ws.pivots[digits[i]] = uint8_t(i + 1);
            std::memcpy(ws.pivots.data() + (kMapPivotKeys - kMapPivotSlot) + 32 * i, keys + size_t(i) * ks, ks);
            ws.pivot_max_digit = std::max(ws.pivot_max_digit, digits[i]);
        }
        ws.n_pivots = n_pivots;
    });
}

int raduls_gpu_check_report(uint64_t* out6) {
    if (!out6) return RADULS_GPU_EINVAL;
#ifdef RG_CHECKED
    std::lock_guard<std::mutex> lk(g_chk_host.mu);
    for (int i = 0; i < 6; ++i) out6[i] = g_chk_host.report[i];
    return 1;
#else
    for (int i = 0; i < 6; ++i) out6[i] = 0;
    return 0;
#endif
}

int raduls_gpu_set_host_cache(int on) {
    g_host_cache.store(on ? 1 : 0);
    if (!on) {
        return guarded([&] {
            Workspace& ws = workspace();
            std::lock_guard<std::mutex> lk(ws.mu);
            ws.host_data.release();
            ws.host_tmp.release();
        });
    }
    return RADULS_GPU_OK;
}

int raduls_gpu_launch_count(uint64_t* count) {
    if (!count) return RADULS_GPU_EINVAL;
    *count = g_launches.load(std::memory_order_relaxed);
    return RADULS_GPU_OK;
}

int raduls_gpu_rank_mode(int* mode) {
    if (!mode) return RADULS_GPU_EINVAL;
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        *mode = atomic_rank_ok(ws) ? 0 : 1;
    });
}

int raduls_gpu_last_kernel_times(raduls_gpu_kernel_time* out, int capacity, int* count) {
    return guarded([&] {
        Workspace& ws = workspace();
        std::lock_guard<std::mutex> lk(ws.mu);
        int k = 0;
        for (int c = 0; c < K_NCLASS; ++c) {
            if (!ws.prof.launches[c]) continue;
            if (out && k < capacity) {
                std::memset(&out[k], 0, sizeof out[k]);
                std::snprintf(out[k].name, sizeof out[k].name, "%s", kClassName[c]);
                out[k].launches = ws.prof.launches[c];
                out[k].ms = ws.prof.ms[c];
            }
            ++k;
        }
        if (count) *count = k;
    });
}

void raduls_gpu_release(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_ws) {
        Workspace* w = kv.second;
        std::lock_guard<std::mutex> lk2(w->mu);
        w->hist8.release(); w->andor0.release(); w->thr.release(); w->acc.release(); w->ctr.release();
        for (int b = 0; b < 2; ++b) {
            w->segs[b].release(); w->seg_tot[b].release(); w->seg_andor[b].release(); w->tile_seg[b].release();
        }
        w->tile_cnt.release(); w->tile_off.release(); w->status.release(); w->groups.release(); w->spill.release(); w->spill_bm.release(); w->spill_med.release(); w->n_spill.release();
        w->copies.release(); w->host_data.release(); w->host_tmp.release(); w->map8.release(); w->dig_dst.release(); w->pieces.release(); w->hot.release();
        w->nd.release(); w->bsegs.release();
        delete w->stager;
        if (w->h_ctr) cudaFreeHost(w->h_ctr);
        if (w->h_small) cudaFreeHost(w->h_small);
        delete w;
    }
    g_ws.clear();
}

int raduls_gpu_sort_multi(int n_dev, const int* devices, void* const* d_in, const uint64_t* n_in,
                          void* const* d_out, uint64_t* n_out, uint64_t out_capacity_recs,
                          uint32_t rs, uint32_t ks) {
    if (!layout_ok(rs, ks) || n_dev < 1 || n_dev > 256 || !devices || !d_in || !n_in || !d_out || !n_out)
        return RADULS_GPU_EINVAL;
    uint64_t total = 0;
    for (int g = 0; g < n_dev; ++g) {
        if (mul_overflows(n_in[g], rs) || n_in[g] > kMaxRecords) return RADULS_GPU_EINVAL;
        if (n_in[g] && (!d_in[g] || !aligned_ok(d_in[g], rs))) return RADULS_GPU_EINVAL;
        if (!d_out[g] || !aligned_ok(d_out[g], rs)) return RADULS_GPU_EINVAL;
        total += n_in[g];
    }
    if (mul_overflows(out_capacity_recs, rs)) return RADULS_GPU_EINVAL;
    const uint32_t G = uint32_t(n_dev);
    // 1. the first key byte that varies over all devices' records
    std::vector<std::array<uint64_t, 8>> ao(G);
    int rc = run_per_device(n_dev, [&](int g) {
        if (cudaSetDevice(devices[g]) != cudaSuccess) return int(RADULS_GPU_ECUDA);
        uint64_t* h = ao[g].data();
        for (int w = 0; w < 8; ++w) h[w] = (w & 1) ? 0ull : ~0ull;
        return n_in[g] ? raduls_gpu_andor(d_in[g], n_in[g], rs, h, nullptr) : int(RADULS_GPU_OK);
    });
    if (rc) return rc;
    uint32_t p0 = first_varying_byte_multi(ao, ks);
    if (p0 >= ks) p0 = 0;  // every key equal: any contiguous map is correct
    // 2. 16-bit prefix histograms at (p0, p0 + 1)
    std::vector<std::vector<uint64_t>> hist(G, std::vector<uint64_t>(kPrefixBuckets, 0));
    rc = run_per_device(n_dev, [&](int g) {
        return guarded([&] {
            RG_CHECK(cudaSetDevice(devices[g]));
            if (!n_in[g]) return;
            uint64_t* d_hist = nullptr;
            RG_CHECK(cudaMalloc(&d_hist, kPrefixBuckets * sizeof(uint64_t)));
            int r = RADULS_GPU_OK;
            if (cudaMemset(d_hist, 0, kPrefixBuckets * sizeof(uint64_t)) != cudaSuccess) r = RADULS_GPU_ECUDA;
            if (!r) r = raduls_gpu_prefix_histogram(d_in[g], n_in[g], rs, ks, p0, d_hist, nullptr);
            if (!r && cudaMemcpy(hist[g].data(), d_hist, kPrefixBuckets * sizeof(uint64_t),
                                 cudaMemcpyDeviceToHost) != cudaSuccess)
                r = RADULS_GPU_ECUDA;
            cudaFree(d_hist);
            if (r) throw CudaError{r};
        });
    });
    if (rc) return rc;
    // 3. contiguous count-balanced bucket ranges; who sends what to whom
    std::vector<uint64_t> global(kPrefixBuckets, 0);
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t b = 0; b < kPrefixBuckets; ++b) global[b] += hist[g][b];
    const std::vector<uint32_t> map = balanced_bucket_map_multi(global, G);
    // digits: each device's bucket range, cut further where key byte p0
    // changes as far as 256 digits allow (the lightest byte-p0 boundaries
    // dropped first) — the exchange is then the first MSD level, and each
    // device sorts its digits as pre-split segments (raduls_gpu_sort_segments)
    std::vector<uint8_t> cut(kPrefixBuckets, 0);
    uint32_t ncut = 0;
    for (uint32_t bk = 1; bk < kPrefixBuckets; ++bk)
        if (map[bk] != map[bk - 1]) cut[bk] = 1, ++ncut;
    {
        std::vector<uint32_t> cand;
        for (uint32_t bk = 256; bk < kPrefixBuckets; bk += 256)
            if (!cut[bk]) cand.push_back(bk);
        const uint32_t budget = 255 - std::min<uint32_t>(ncut, 255);
        if (cand.size() > budget) {
            std::vector<double> blk(256, 0.0);
            for (uint32_t bk = 0; bk < kPrefixBuckets; ++bk) blk[bk >> 8] += double(global[bk]);
            std::stable_sort(cand.begin(), cand.end(), [&](uint32_t x, uint32_t y) {
                return blk[(x >> 8) - 1] + blk[x >> 8] > blk[(y >> 8) - 1] + blk[y >> 8];
            });
            cand.resize(budget);
        }
        for (uint32_t bk : cand) cut[bk] = 1;
    }
    std::vector<uint32_t> digit(kPrefixBuckets, 0);
    for (uint32_t bk = 1; bk < kPrefixBuckets; ++bk) digit[bk] = digit[bk - 1] + cut[bk];
    const uint32_t D = digit[kPrefixBuckets - 1] + 1;
    std::vector<uint32_t> drank(D, 0), dlo(D, kPrefixBuckets), dhi(D, 0);
    for (uint32_t bk = 0; bk < kPrefixBuckets; ++bk) {
        const uint32_t d = digit[bk];
        drank[d] = map[bk];
        dlo[d] = std::min(dlo[d], bk);
        dhi[d] = std::max(dhi[d], bk);
    }
    std::vector<uint8_t> dfirst(D);
    for (uint32_t d = 0; d < D; ++d) {
        const uint32_t f = dlo[d] == dhi[d] ? p0 + 2 : (dlo[d] >> 8) == (dhi[d] >> 8) ? p0 + 1 : p0;
        dfirst[d] = uint8_t(std::min(f, ks));
    }
    std::vector<std::vector<uint64_t>> dcnt(G, std::vector<uint64_t>(D, 0));  // [src][digit]
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t bk = 0; bk < kPrefixBuckets; ++bk) dcnt[g][digit[bk]] += hist[g][bk];
    std::vector<std::vector<uint64_t>> cnt(G, std::vector<uint64_t>(G, 0));  // [src][dst]
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t d = 0; d < D; ++d) cnt[g][drank[d]] += dcnt[g][d];
    std::vector<uint64_t> recv(G, 0);
    for (uint32_t g = 0; g < G; ++g)
        for (uint32_t r = 0; r < G; ++r) recv[r] += cnt[g][r];
    for (uint32_t r = 0; r < G; ++r)
        if (recv[r] > out_capacity_recs || recv[r] > kMaxRecords) return RADULS_GPU_EINVAL;  // nothing written yet
    // digit-major output: device r holds its digits in order, each digit's
    // records source by source (the stable order); dat[g][d] = record offset
    // of source g's run of digit d in d_out[drank[d]]
    std::vector<std::vector<uint64_t>> dat(G, std::vector<uint64_t>(D, 0));
    std::vector<std::vector<uint64_t>> seg_size(G);
    std::vector<std::vector<uint8_t>> seg_first(G);
    {
        std::vector<uint64_t> pos(G, 0);
        for (uint32_t d = 0; d < D; ++d) {
            const uint32_t r = drank[d];
            uint64_t tot = 0;
            for (uint32_t g = 0; g < G; ++g) {
                dat[g][d] = pos[r] + tot;
                tot += dcnt[g][d];
            }
            pos[r] += tot;
            if (tot) {
                seg_size[r].push_back(tot);
                seg_first[r].push_back(dfirst[d]);
            }
        }
    }
    // 4. peer access between every pair of distinct devices (NVLink P2P)
    bool p2p = true;
    rc = guarded([&] {
        for (uint32_t g = 0; g < G; ++g)
            for (uint32_t r = 0; r < G; ++r) {
                if (devices[g] == devices[r]) continue;
                int ok = 0;
                RG_CHECK(cudaDeviceCanAccessPeer(&ok, devices[g], devices[r]));
                if (!ok) {
                    p2p = false;
                    continue;
                }
                RG_CHECK(cudaSetDevice(devices[g]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[r], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) throw CudaError{RADULS_GPU_ECUDA};
                cudaGetLastError();
            }
    });
    if (rc) return rc;
    // scratch per device (the partition output when P2P is missing; the local sort's tmp)
    std::vector<uint8_t*> part(G, nullptr);
    auto free_parts = [&] {
        for (uint32_t g = 0; g < G; ++g)
            if (part[g]) {
                cudaSetDevice(devices[g]);
                cudaFree(part[g]);
            }
    };
    // 5. the exchange. With P2P: ONE kernel per source device — the stable
    // partition stores every destination's records straight into that device's
    // d_out over NVLink (k_scatter<kPeer>). Without: partition locally, then
    // peer copies.
    rc = run_per_device(n_dev, [&](int g) {
        return guarded([&] {
            RG_CHECK(cudaSetDevice(devices[g]));
            const uint64_t bytes = std::max<uint64_t>(std::max(n_in[g], recv[g]) * rs, rs);
            RG_CHECK(cudaMalloc(&part[g], bytes));
            if (!n_in[g]) return;
            uint32_t* d_map = nullptr;
            RG_CHECK(cudaMalloc(&d_map, kPrefixBuckets * sizeof(uint32_t)));
            int r = cudaMemcpy(d_map, digit.data(), kPrefixBuckets * sizeof(uint32_t), cudaMemcpyHostToDevice) ==
                            cudaSuccess
                        ? int(RADULS_GPU_OK)
                        : int(RADULS_GPU_ECUDA);
            std::vector<uint64_t> got(D, 0), dst(D, 0);
            for (uint32_t d = 0; d < D; ++d)
                dst[d] = reinterpret_cast<uint64_t>(static_cast<uint8_t*>(d_out[drank[d]]) + dat[g][d] * rs);
            if (!r) r = raduls_gpu_set_pivots(0, nullptr, nullptr, ks);  // whole buckets only here
            if (!r) {
                if (p2p)
                    r = raduls_gpu_partition_to(d_in[g], n_in[g], rs, ks, p0, d_map, D, dst.data(), got.data(),
                                                nullptr);
                else
                    r = raduls_gpu_partition(d_in[g], part[g], n_in[g], rs, ks, p0, d_map, D, got.data(), nullptr);
            }
            cudaFree(d_map);
            if (r) throw CudaError{r};
            for (uint32_t d = 0; d < D; ++d)
                if (got[d] != dcnt[g][d]) throw CudaError{RADULS_GPU_EINTERNAL};
            RG_CHECK(cudaDeviceSynchronize());  // peer stores complete before the sort reads them
        });
    });
    if (!rc && !p2p) {
        rc = guarded([&] {
            std::vector<cudaStream_t> st(G);
            for (uint32_t g = 0; g < G; ++g) {
                RG_CHECK(cudaSetDevice(devices[g]));
                RG_CHECK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
            }
            for (uint32_t g = 0; g < G; ++g) {  // the local partition is digit-ordered: one copy per run
                uint64_t send = 0;
                RG_CHECK(cudaSetDevice(devices[g]));
                for (uint32_t d = 0; d < D; ++d) {
                    const uint64_t k = dcnt[g][d];
                    const uint32_t r = drank[d];
                    if (k)
                        RG_CHECK(cudaMemcpyPeerAsync(static_cast<uint8_t*>(d_out[r]) + dat[g][d] * rs, devices[r],
                                                     part[g] + send * rs, devices[g], k * rs, st[g]));
                    send += k;
                }
            }
            for (uint32_t g = 0; g < G; ++g) {
                RG_CHECK(cudaSetDevice(devices[g]));
                RG_CHECK(cudaStreamSynchronize(st[g]));
                RG_CHECK(cudaStreamDestroy(st[g]));
            }
        });
    }
    if (rc) {
        free_parts();
        return rc;
    }
    // 6. each device sorts its key range (the partition buffer is its scratch)
    rc = run_per_device(n_dev, [&](int g) {
        if (cudaSetDevice(devices[g]) != cudaSuccess) return int(RADULS_GPU_ECUDA);
        n_out[g] = recv[g];
        return raduls_gpu_sort_segments(d_out[g], part[g], recv[g], rs, ks, uint32_t(seg_size[g].size()),
                                        seg_size[g].data(), seg_first[g].data(), nullptr);
    });
    free_parts();
    (void)total;
    return rc;
}

}  // extern "C"
