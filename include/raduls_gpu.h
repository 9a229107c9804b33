/*
 * raduls_gpu.h — C-ABI of the B200-native MSD record sort (libraduls_gpu.so).
 *
 * Drop-in for the reference entry point
 *     void raduls::sort(uint8_t* data, size_t n, const RecordLayout& layout,
 *                       const SchedulerConfig& cfg = {});
 * (/root/reference/proj/include/raduls/scheduler.hpp:56-61,
 *  /root/reference/proj/src/scheduler.cpp:40-45)
 * in the (input buffer, temp buffer, n_recs, rec_size, key_size) shape named by
 * BASELINE.json. Plain pointers and sizes only; no exceptions cross the ABI.
 *
 * Record model (reference layout.hpp:1-81): a record is rec_size bytes
 * (8, 16, 24 or 32); the key is its first key_size bytes (1..rec_size), most
 * significant byte first, compared as memcmp. The reference accepts only
 * key_size 8 or 16 (layout.hpp:22-27); this library also takes any other
 * key_size <= rec_size (e.g. 24, BASELINE config C4).
 *
 * Result: records ordered non-decreasingly by key, in the caller's buffer.
 * The sort is stable (equal keys keep their input order). The reference's MSD
 * is not stable (Shell/introsort tails, small_sorts.hpp:166-167), so for
 * equal keys only the key sequence and the per-run record multiset are
 * comparable — which is the parity definition.
 *
 * Status codes (errors are reported before any write to `data`):
 */
#ifndef RADULS_GPU_H
#define RADULS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RADULS_GPU_OK = 0,
    RADULS_GPU_EINVAL = 1,   /* bad layout, misaligned pointer, n*rec_size overflow
                                (reference: std::invalid_argument, dispatch.hpp:37-39) */
    RADULS_GPU_ENOMEM = 2,   /* device/pinned allocation failed, input untouched
                                (reference: raduls::resource_error, record_array.hpp:21-28) */
    RADULS_GPU_ECUDA = 3,    /* a CUDA runtime call failed */
    RADULS_GPU_ENCCL = 4,    /* reserved for the multi-GPU exchange */
    RADULS_GPU_EINTERNAL = 5 /* planner capacity invariant violated (bug) */
};

/* Human-readable text for a status code. */
const char* raduls_gpu_strerror(int code);

/* 1 if (rec_size, key_size) is supported, else 0. */
int raduls_gpu_layout_valid(uint32_t rec_size, uint32_t key_size);

/* Library/ABI version, e.g. 0x000100 for 0.1.0. */
uint32_t raduls_gpu_version(void);

/*
 * Device-resident sort (replaces raduls::sort; scheduler.hpp:60-61).
 *   d_data : n_recs*rec_size bytes of device memory (16-B aligned for rec_size
 *            16/32, 8-B aligned for 8/24); sorted in place.
 *   d_tmp  : scratch of the same size, or NULL: the library then allocates it
 *            (cudaMallocAsync on `stream`) and frees it before returning, like
 *            the reference's internal aux array (msd_sorter.hpp:52).
 *   stream : a cudaStream_t (NULL = legacy default stream).
 * The call blocks until the sort has completed on `stream` (the MSD planner
 * reads a few counters back per level), mirroring the synchronous reference.
 * Calls on the same device are serialised (one shared workspace per device).
 */
int raduls_gpu_sort(void* d_data, void* d_tmp, uint64_t n_recs, uint32_t rec_size,
                    uint32_t key_size, void* stream);

/*
 * Host drop-in mirroring raduls::sort(data, n, layout, cfg): `data` is host
 * memory (any alignment); H2D -> device sort -> D2H. `tmp` is ignored (the
 * device scratch is library-owned); pass NULL.
 */
int raduls_gpu_sort_host(uint8_t* data, uint8_t* tmp, uint64_t n_recs, uint32_t rec_size,
                         uint32_t key_size);

/*
 * LSD baseline (replaces raduls::lsd_sort; P/include/raduls/lsd.hpp:16-22,
 * P/src/lsd.cpp:12-35): key_size stable byte splits, least significant first,
 * ping-ponging between d_data and d_tmp (NULL: library-allocated), result in
 * d_data. Bytes that are constant over the input are skipped. Stable, so the
 * output equals raduls_gpu_sort's byte for byte. Blocking like raduls_gpu_sort.
 */
int raduls_gpu_lsd_sort(void* d_data, void* d_tmp, uint64_t n_recs, uint32_t rec_size,
                        uint32_t key_size, void* stream);
/* Host-memory LSD drop-in (raduls::lsd_sort(data, n, layout, cfg)): H2D ->
 * raduls_gpu_lsd_sort -> D2H, like raduls_gpu_sort_host. */
int raduls_gpu_lsd_sort_host(uint8_t* data, uint8_t* tmp, uint64_t n_recs, uint32_t rec_size,
                             uint32_t key_size);

/* Accounting of the most recent sort on the calling thread's device. */
typedef struct {
    uint32_t levels;            /* planner levels executed */
    uint32_t scatter_launches;  /* k_scatter launches */
    uint64_t hist_records;      /* records read by histogram passes (k_histo_all + k_seg_hist) */
    uint64_t scatter_records;   /* records moved by scatter passes (1 read + 1 write each) */
    uint64_t local_records;     /* records moved by local sorts */
    uint64_t copy_records;      /* records moved by copy-back */
    uint64_t fallback_groups;   /* local-sort groups that needed the full-key fallback */
    uint64_t skipped_levels;    /* segment-levels skipped as constant digits (e) */
    uint64_t hist_digit_records; /* records histogrammed from the digit array (1 byte each; the
                                    scatter before wrote that byte) instead of from the records */
    uint64_t bitmap_spill_groups; /* local-sort groups the bitmap sort handed to the bucket sort
                                     (duplicate-heavy or clustered keys) */
} raduls_gpu_stats;

int raduls_gpu_last_stats(raduls_gpu_stats* out);

/* Per-kernel device time of the most recent sort, when profiling is on
 * (CUDA events recorded around every launch on the sort's stream; adds a few
 * microseconds per launch). Classes: sample, tile_hist, tile_scan, plan,
 * scatter, local_sort, copy_back. */
typedef struct {
    char name[16];
    uint32_t launches;
    double ms;
} raduls_gpu_kernel_time;

int raduls_gpu_set_profiling(int on);
int raduls_gpu_last_kernel_times(raduls_gpu_kernel_time* out, int capacity, int* count);

/* raduls_gpu_sort on records that are already partitioned into n_segs
 * contiguous, key-ordered segments (every key of segment i <= every key of
 * segment i + 1; h_sizes sum to n): the segments are sorted independently,
 * as the first MSD level's children, starting at key byte h_first_byte[i]
 * (key bytes before it must be equal within segment i). The multi-GPU
 * exchange delivers each rank's range in this form, so the receiver skips
 * the level the exchange already did. Zero-size segments are allowed. */
int raduls_gpu_sort_segments(void* d_data, void* d_tmp, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                             uint32_t n_segs, const uint64_t* h_sizes, const uint8_t* h_first_byte, void* stream);

/* How the scatter ranks records inside a warp on the current device (decided
 * on first use): 0 = one shared-memory atomic per record, used only after a
 * device self-test (k_rank_selftest) confirmed that the conflicting lanes of
 * one atomic are served in lane order; 1 = ballot ranking (stable by
 * construction; also forced by RADULS_GPU_STABLE_RANK=ballot). Either way the
 * sort is stable. The LSD baseline and raduls_gpu_split always use 1. */
int raduls_gpu_rank_mode(int* mode);

/* Kernel launches made by this library in this process so far (every kernel,
 * every entry point; a relaxed process-wide counter). */
int raduls_gpu_launch_count(uint64_t* count);

/* Checked build only (libraduls_gpu_checked.so, built with -DRG_CHECKED; the
 * stand-in for compute-sanitizer): returns 1 and fills out6 = {violations,
 * first violating address, its check site, its size, barrier timeouts,
 * checked calls} accumulated over the process; any call that recorded a
 * violation returned RADULS_GPU_EINTERNAL. The production library returns 0
 * (zeros). */
int raduls_gpu_check_report(uint64_t* out6);

/* The host drop-ins (raduls_gpu_sort_host, raduls_gpu_lsd_sort_host) stage the
 * records in two device buffers of n*rec_size bytes. Default (0): freed before
 * the call returns, as the reference frees its per-call aux buffer
 * (msd_sorter.hpp:52). 1: kept and reused by later calls of the same or a
 * smaller size until raduls_gpu_set_host_cache(0) or raduls_gpu_release(). */
int raduls_gpu_set_host_cache(int on);

/*
 * Building blocks (tests, benchmarks and the multi-GPU driver). All device
 * pointers; asynchronous on `stream` unless noted.
 */

/* One stable single-digit split of d_src into d_dst by record byte
 * `key_byte_offset` (reference radix_split, kernels.hpp:157-167);
 * h_counts (host, 256 u64, may be NULL) receives the digit histogram.
 * Synchronous. */
int raduls_gpu_split(const void* d_src, void* d_dst, uint64_t n_recs, uint32_t rec_size,
                     uint32_t key_byte_offset, uint64_t* h_counts, void* stream);

/* Histograms of record bytes 0..min(key_size,8)-1 (reference build_histogram,
 * kernels.hpp:71-77) and AND/OR of every 64-bit record word. Synchronous.
 * h_hist: host [8][256] u64; h_andor: host [8] u64 (and at 2w, or at 2w+1). */
int raduls_gpu_histogram(const void* d_data, uint64_t n_recs, uint32_t rec_size,
                         uint32_t key_size, uint64_t* h_hist, uint64_t* h_andor, void* stream);

/* SURVEY.md §8(d) generator; dist 0 uniform, 1 = C3 skew. Record i gets
 * global index index_base + i. */
int raduls_gpu_generate(void* d_out, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                        uint32_t dist, uint64_t seed, uint64_t index_base, void* stream);

/* AND / OR of every 64-bit record word over the array (h_andor: host [8] u64,
 * and at 2w, or at 2w+1); a key byte is constant iff its AND and OR bytes
 * agree. Synchronous. */
int raduls_gpu_andor(const void* d_data, uint64_t n_recs, uint32_t rec_size, uint64_t* h_andor,
                     void* stream);

/* array_digest (reference verify.cpp:37-50). Synchronous. */
int raduls_gpu_digest(const void* d_data, uint64_t n_recs, uint32_t rec_size, uint64_t* lo,
                      uint64_t* hi, void* stream);

/* check_sorted (reference verify.cpp:27-35): *violations = number of adjacent
 * inversions, *first = first one (or UINT64_MAX). Synchronous. */
int raduls_gpu_check_sorted(const void* d_data, uint64_t n_recs, uint32_t rec_size,
                            uint32_t key_size, uint64_t* violations, uint64_t* first,
                            void* stream);

/*
 * Multi-GPU key-range partition; one process per GPU,
 * exchange done by the caller (NCCL all-to-all).
 *
 * raduls_gpu_prefix_histogram: d_hist (device, 65536 u64, accumulated into)
 *   counts records by the 16-bit big-endian value of key bytes
 *   (prefix_byte, prefix_byte+1) — bytes at or beyond key_size read as 0.
 * raduls_gpu_partition: stable scatter of d_src into d_dst grouped by
 *   destination rank = d_bucket_rank[16-bit prefix] (< n_ranks <= 256);
 *   h_rank_counts (host, n_ranks u64) receives the per-rank record counts.
 *   Synchronous.
 */
int raduls_gpu_prefix_histogram(const void* d_data, uint64_t n_recs, uint32_t rec_size,
                                uint32_t key_size, uint32_t prefix_byte, uint64_t* d_hist,
                                void* stream);
int raduls_gpu_partition(const void* d_src, void* d_dst, uint64_t n_recs, uint32_t rec_size,
                         uint32_t key_size, uint32_t prefix_byte, const uint32_t* d_bucket_rank,
                         uint32_t n_ranks, uint64_t* h_rank_counts, void* stream);

/*
 * The partition fused with the exchange: like
 * raduls_gpu_partition, but destination rank r's records are stored by the
 * partition kernel itself, in stable order, to the byte address h_dst[r] —
 * typically a peer GPU's receive buffer reached over NVLink (peer access
 * enabled, or a raduls_gpu_ipc_open mapping), at this source's offset there.
 * h_dst[r] must be 16-B aligned (8-B for record sizes 8 and 24). Synchronous.
 */
int raduls_gpu_partition_to(const void* d_src, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                            uint32_t prefix_byte, const uint32_t* d_bucket_rank, uint32_t n_ranks,
                            const uint64_t* h_dst, uint64_t* h_rank_counts, void* stream);

/*
 * The same partition in two phases, so that a multi-GPU plan can exchange the
 * exact per-destination counts before any record moves (the bucket map can
 * then come from a sample):
 *   raduls_gpu_partition_plan: per-destination record counts (h_rank_counts,
 *     n_ranks entries) of the stable partition by d_bucket_rank[16-bit prefix
 *     at prefix_byte], and the AND/OR of every record word (h_andor, 8 u64:
 *     and at 2w, or at 2w+1), in one read of d_src; the per-tile offsets stay
 *     in the calling thread's device workspace;
 *   raduls_gpu_partition_store: the stores of that plan (same d_src, n, layout),
 *     rank r's records to the byte address h_dst[r] (as raduls_gpu_partition_to).
 * Any other call of this library on the device in between invalidates the
 * plan (store then returns RADULS_GPU_EINVAL). Synchronous.
 * raduls_gpu_sample_andor / raduls_gpu_sample_prefix_histogram: AND/OR (to
 * the host) and the 16-bit prefix histogram (accumulated into d_hist, 65536
 * u64) of a strided sample of `samples` records — inputs for the bucket map.
 */
int raduls_gpu_partition_plan(const void* d_src, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                              uint32_t prefix_byte, const uint32_t* d_bucket_rank, uint32_t n_ranks,
                              uint64_t* h_rank_counts, uint64_t* h_andor, void* stream);
int raduls_gpu_partition_store(const void* d_src, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                               const uint64_t* h_dst, void* stream);

/*
 * Hot keys ("only a single-key bucket may be split"):
 * a plan may give a hot 16-bit bucket its own digit and spread that digit's
 * records over several destinations by count, provided the bucket holds one
 * key only.
 *   raduls_gpu_digit_andor: AND/OR of the key words (64-bit words holding key
 *     bytes) of the records whose bucket maps to a digit d with h_hot[d] != 0
 *     (at most 32 such digits); h_andor: host [n_digits][8] u64 (and at 2w,
 *     or at 2w+1; ~0/0 for digits without records or not flagged). The digit
 *     holds a single key iff and == or on every key byte. Synchronous;
 *     cancels a pending raduls_gpu_partition_plan.
 *   raduls_gpu_partition_store_pieces: the stores of the pending plan, with
 *     each digit's run cut into pieces: n_pieces entries (h_piece_digit[i],
 *     h_piece_count[i], h_piece_dst[i]) in increasing digit order; a digit's
 *     pieces take its records in stable order, count by count, each to its
 *     own byte address (16-B aligned; 8-B for record sizes 8 and 24). The
 *     counts of every digit must add up to the plan's count for it.
 *     Synchronous.
 */
/*
 * Pivots for hot buckets whose records do not share one key: with pivot i
 * set on digit h_digits[i], a record whose bucket maps to that digit gets
 * digit d, d + 1 or d + 2 as its key (first key_size bytes, memcmp order) is
 * below, equal to or above h_keys[i * key_size ...] — so the equal run, one
 * key, may be cut into pieces by count. A plan then numbers its digits with
 * d + 1 and d + 2 reserved for the pivot. At most 16 pivots; their digit
 * triples must not overlap. The pivots apply to every bucket-map call of this
 * library on the current device (partition, partition_to, partition_plan,
 * digit_andor) until replaced; n_pivots = 0 clears them.
 */
int raduls_gpu_set_pivots(uint32_t n_pivots, const uint32_t* h_digits, const uint8_t* h_keys, uint32_t key_size);

int raduls_gpu_digit_andor(const void* d_src, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                           uint32_t prefix_byte, const uint32_t* d_bucket_digit, uint32_t n_digits,
                           const uint8_t* h_hot, uint64_t* h_andor, void* stream);
int raduls_gpu_partition_store_pieces(const void* d_src, uint64_t n_recs, uint32_t rec_size,
                                      uint32_t key_size, uint32_t n_pieces, const uint32_t* h_piece_digit,
                                      const uint64_t* h_piece_count, const uint64_t* h_piece_dst,
                                      void* stream);
int raduls_gpu_sample_andor(const void* d_data, uint64_t n_recs, uint32_t rec_size, uint32_t samples,
                            uint64_t* h_andor, void* stream);
int raduls_gpu_sample_prefix_histogram(const void* d_data, uint64_t n_recs, uint32_t rec_size, uint32_t key_size,
                                       uint32_t prefix_byte, uint32_t samples, uint64_t* d_hist, void* stream);

/*
 * CUDA IPC for the multi-process exchange: raduls_gpu_ipc_alloc allocates
 * device memory and returns its 64-byte IPC handle; a peer process maps it
 * with raduls_gpu_ipc_open (lazy peer access) and unmaps with
 * raduls_gpu_ipc_close; raduls_gpu_free releases the allocation.
 */
int raduls_gpu_ipc_alloc(uint64_t bytes, void** d_ptr, uint8_t* handle);
int raduls_gpu_ipc_open(const uint8_t* handle, void** d_ptr);
int raduls_gpu_ipc_close(void* d_ptr);
int raduls_gpu_free(void* d_ptr);

/*
 * Multi-GPU sort in one call: G devices, one host thread
 * per device. Device g holds n_in[g] records at d_in[g] (left unchanged). On
 * return d_out[g] (capacity out_capacity_recs records) holds n_out[g] records:
 * the g-th contiguous key range, sorted; the concatenation over g is the
 * stable sort of the inputs concatenated in device order. Plan: the first
 * key byte varying over all devices, 16-bit prefix histograms, contiguous
 * count-balanced bucket ranges (a bucket is never split); the stable device
 * partition stores each destination's records straight into that device's
 * d_out over NVLink (raduls_gpu_partition_to; peer copies when P2P is
 * unavailable); local sort.
 * EINVAL (nothing written) when a device would receive more than
 * out_capacity_recs records. A device may be listed more than once.
 */
int raduls_gpu_sort_multi(int n_dev, const int* devices, void* const* d_in, const uint64_t* n_in,
                          void* const* d_out, uint64_t* n_out, uint64_t out_capacity_recs,
                          uint32_t rec_size, uint32_t key_size);

/* Release the cached per-device workspace (optional): level metadata (~0.7 B
 * per record) and the digit array(s) (1 B per record, 2 B at rec_size 32)
 * that a sort grows on demand and keeps for the next call. */
void raduls_gpu_release(void);

#ifdef __cplusplus
}
#endif
#endif /* RADULS_GPU_H */
