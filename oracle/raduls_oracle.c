/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library;
 * the product (paper_1612_02557_b200/) never links or calls it.
 *
 * Plain-C restatement of the RADULS reference algorithm for the hot path
 * `raduls::sort` (P = /root/reference/proj):
 *
 *   record model ........ P/include/raduls/layout.hpp:16-81
 *   histogram/scan/split  P/include/raduls/kernels.hpp:35-94,157-167
 *   tiny-bin sorts ...... P/include/raduls/small_sorts.hpp:14-191
 *   MSD orchestration ... P/include/raduls/detail/msd_sorter.hpp:50-214 (T = 1 path)
 *   verification ........ P/src/verify.cpp:27-64
 *   input generator ..... SURVEY.md §8(d) counter-based generator, built on
 *                         mix64 (P/include/raduls/datagen.hpp:37-42) and the
 *                         payload convention of P/src/datagen.cpp:75-80.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer tests (P/tests/test_record.cpp:35-59,
 * P/tests/test_kernels.cpp:87-143) and, byte for byte, against the reference
 * library itself compiled from /root/reference by oracle/Makefile
 * (oracle/_ref/libraduls_ref.so) through the committed fixtures in
 * tests/golden/ (made by tests/golden/make_golden.py).
 *
 * Generalisation beyond the reference: any key_size in [1, record_size] and
 * record_size a multiple of 8 up to 32. Keys compare as memcmp over key_size
 * bytes (layout.hpp:52-55), which equals key_less<8|16> (layout.hpp:57-68)
 * where the reference is defined.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2

/* ------------------------------------------------------------------ record model */

static int layout_ok(uint32_t rs, uint32_t ks) {
    /* rs in {8,16,24,32}; 1 <= ks <= rs  (layout.hpp:22-27, widened to any ks) */
    return (rs == 8 || rs == 16 || rs == 24 || rs == 32) && ks >= 1 && ks <= rs;
}

int orc_layout_valid(uint32_t rs, uint32_t ks) { return layout_ok(rs, ks); }

uint64_t orc_load_be64(const uint8_t* p) { /* layout.hpp:41-45 */
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v = (v << 8) | p[i];
    return v;
}

void orc_store_be64(uint8_t* p, uint64_t v) { /* layout.hpp:47-49 */
    for (int i = 7; i >= 0; --i) {
        p[i] = (uint8_t)v;
        v >>= 8;
    }
}

/* digit(rec, byte_index) = rec[ks-1-byte_index]  (layout.hpp:32-39) */
uint8_t orc_digit(const uint8_t* rec, uint32_t ks, uint32_t byte_index) {
    return rec[ks - 1 - byte_index];
}

static inline int key_less(const uint8_t* a, const uint8_t* b, uint32_t ks) {
    return memcmp(a, b, ks) < 0; /* compare_keys, layout.hpp:52-55 */
}

static inline void swap_rec(uint8_t* a, uint8_t* b, uint32_t rs) { /* layout.hpp:75-81 */
    uint8_t t[32];
    memcpy(t, a, rs);
    memcpy(a, b, rs);
    memcpy(b, t, rs);
}

/* ------------------------------------------------------------------ generator (§8(d)) */

uint64_t orc_mix64(uint64_t x) { /* datagen.hpp:37-42 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t orc_rnd(uint64_t seed, uint64_t i, uint32_t w) {
    return orc_mix64(seed ^ orc_mix64(4 * i + w));
}

/* Integer inverse-CDF thresholds of Zipf(s) over `universe` ranks:
 * thr[k] = floor(CDF_k / CDF_universe * 2^53), thr[universe-1] = 2^53. */
void orc_zipf_thresholds(double s, uint32_t universe, uint64_t* thr) {
    double run = 0.0, total = 0.0;
    for (uint32_t r = 1; r <= universe; ++r) total += pow((double)r, -s);
    for (uint32_t k = 0; k < universe; ++k) {
        run += pow((double)(k + 1), -s);
        double t = run / total * 9007199254740992.0; /* 2^53 */
        thr[k] = (k + 1 == universe) ? 9007199254740992ULL : (uint64_t)t;
    }
}

/* dist 0: uniform keys. dist 1: C3 skew — top 24 bits zero, next 8 bits a
 * Zipf(s=1.2) rank over 256 values, low 32 bits uniform.
 * Record i (global index index_base + j) gets key words written big-endian
 * (store_be64, D1 of SURVEY.md), payload word 0 = i, further payload words as
 * datagen.cpp:79. */
int orc_generate(uint8_t* out, uint64_t n, uint32_t rs, uint32_t ks, uint32_t dist, uint64_t seed,
                 uint64_t index_base) {
    if (!layout_ok(rs, ks)) return ORC_EINVAL;
    uint64_t thr[256];
    if (dist == 1) orc_zipf_thresholds(1.2, 256, thr);
    const uint32_t words = rs / 8;
    const uint32_t key_words = (ks + 7) / 8;
    for (uint64_t j = 0; j < n; ++j) {
        const uint64_t i = index_base + j;
        uint8_t* rec = out + j * rs;
        for (uint32_t w = 0; w < words; ++w) {
            uint64_t v;
            if (w < key_words) {
                if (dist == 1 && w == 0) {
                    const uint64_t u = orc_rnd(seed, i, 0) >> 11;
                    uint32_t k = 0;
                    while (u >= thr[k]) ++k;
                    v = ((uint64_t)k << 32) | (orc_rnd(seed, i, 1) & 0xFFFFFFFFULL);
                } else {
                    v = orc_rnd(seed, i, dist == 1 ? w + 1 : w);
                }
            } else if (w == key_words) {
                v = i;
            } else {
                v = orc_mix64(i ^ (0xa5a5a5a5a5a5a5a5ULL + w));
            }
            orc_store_be64(rec + 8 * w, v);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ kernels */

/* build_histogram (kernels.hpp:71-77), by record byte offset */
void orc_histogram(const uint8_t* base, uint64_t n, uint32_t rs, uint32_t byte_offset,
                   uint64_t* counts) {
    memset(counts, 0, 256 * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ++counts[base[i * rs + byte_offset]];
}

/* exclusive_prefix_sum (kernels.hpp:47-55) */
void orc_exclusive_prefix_sum(const uint64_t* counts, uint64_t* offsets) {
    uint64_t run = 0;
    for (int d = 0; d < 256; ++d) {
        offsets[d] = run;
        run += counts[d];
    }
}

/* radix_split (kernels.hpp:157-167): stable counting split src -> dst */
void orc_radix_split(const uint8_t* src, uint8_t* dst, uint64_t n, uint32_t rs,
                     uint32_t byte_offset, uint64_t* counts_out) {
    uint64_t counts[256], cur[256];
    orc_histogram(src, n, rs, byte_offset, counts);
    orc_exclusive_prefix_sum(counts, cur);
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t* rec = src + i * rs;
        memcpy(dst + (cur[rec[byte_offset]]++) * rs, rec, rs);
    }
    if (counts_out) memcpy(counts_out, counts, sizeof counts);
}

/* ------------------------------------------------------------------ small sorts */

/* insertion_sort (small_sorts.hpp:47-60), stable */
static void insertion_sort(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
    uint8_t tmp[32];
    for (uint64_t i = 1; i < n; ++i) {
        memcpy(tmp, base + i * rs, rs);
        uint64_t j = i;
        while (j > 0 && key_less(tmp, base + (j - 1) * rs, ks)) {
            memcpy(base + j * rs, base + (j - 1) * rs, rs);
            --j;
        }
        memcpy(base + j * rs, tmp, rs);
    }
}

/* shell_sort with gaps {8, 1} (small_sorts.hpp:62-79) */
static void shell_sort(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
    static const uint64_t gaps[2] = {8, 1};
    uint8_t tmp[32];
    for (int g = 0; g < 2; ++g) {
        const uint64_t gap = gaps[g];
        for (uint64_t i = gap; i < n; ++i) {
            memcpy(tmp, base + i * rs, rs);
            uint64_t j = i;
            while (j >= gap && key_less(tmp, base + (j - gap) * rs, ks)) {
                memcpy(base + j * rs, base + (j - gap) * rs, rs);
                j -= gap;
            }
            memcpy(base + j * rs, tmp, rs);
        }
    }
}

/* sift_down / heap_sort (small_sorts.hpp:83-106) */
static void sift_down(uint8_t* base, uint64_t start, uint64_t end, uint32_t rs, uint32_t ks) {
    uint64_t root = start;
    for (;;) {
        uint64_t child = 2 * root + 1;
        if (child >= end) return;
        if (child + 1 < end && key_less(base + child * rs, base + (child + 1) * rs, ks)) ++child;
        if (!key_less(base + root * rs, base + child * rs, ks)) return;
        swap_rec(base + root * rs, base + child * rs, rs);
        root = child;
    }
}

static void heap_sort(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
    if (n < 2) return;
    for (uint64_t i = n / 2; i-- > 0;) sift_down(base, i, n, rs, ks);
    for (uint64_t i = n - 1; i > 0; --i) {
        swap_rec(base, base + i * rs, rs);
        sift_down(base, 0, i, rs, ks);
    }
}

/* partition_median3 (small_sorts.hpp:108-133) */
static uint64_t partition_median3(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
#define R(i) (base + (uint64_t)(i) * rs)
    const uint64_t mid = n / 2, last = n - 1;
    if (key_less(R(mid), R(0), ks)) swap_rec(R(mid), R(0), rs);
    if (key_less(R(last), R(mid), ks)) {
        swap_rec(R(last), R(mid), rs);
        if (key_less(R(mid), R(0), ks)) swap_rec(R(mid), R(0), rs);
    }
    swap_rec(R(0), R(mid), rs);
    uint64_t lo = 1, hi = n;
    for (;;) {
        while (key_less(R(lo), R(0), ks)) ++lo;
        --hi;
        while (key_less(R(0), R(hi), ks)) --hi;
        if (lo >= hi) return lo;
        swap_rec(R(lo), R(hi), rs);
        ++lo;
    }
#undef R
}

/* intro_rec / introspective_sort (small_sorts.hpp:135-175) */
static void intro_rec(uint8_t* base, uint64_t n, unsigned depth_left, uint64_t limit, uint32_t rs,
                      uint32_t ks) {
    while (n > limit) {
        if (depth_left == 0) {
            heap_sort(base, n, rs, ks);
            return;
        }
        --depth_left;
        const uint64_t cut = partition_median3(base, n, rs, ks);
        if (cut < n - cut) {
            intro_rec(base, cut, depth_left, limit, rs, ks);
            base += cut * rs;
            n -= cut;
        } else {
            intro_rec(base + cut * rs, n - cut, depth_left, limit, rs, ks);
            n = cut;
        }
    }
    insertion_sort(base, n, rs, ks);
}

static unsigned log2_floor(uint64_t n) {
    unsigned r = 0;
    while (n >>= 1) ++r;
    return r;
}

/* TinyPolicy defaults (small_sorts.hpp:14-25) */
enum { TINY = 384, INSERTION_MAX = 32, NARROW_FACTOR = 16, NARROWED_TINY = 32 };

/* is_tiny (small_sorts.hpp:31-37) */
int orc_is_tiny(uint64_t bin_size, uint64_t parent_size) {
    uint64_t threshold = TINY;
    if (parent_size > 0 && parent_size > (uint64_t)NARROW_FACTOR * bin_size)
        threshold = NARROWED_TINY;
    return bin_size < threshold;
}

static uint64_t intro_vs_shell(uint32_t ks) { /* clamp(100 + 5 ks, 100, 180) */
    uint64_t t = 100 + 5 * (uint64_t)ks;
    return t > 180 ? 180 : t;
}

/* comparison_sort (small_sorts.hpp:177-191) */
void orc_comparison_sort(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
    if (n < 2) return;
    if (n <= INSERTION_MAX)
        insertion_sort(base, n, rs, ks);
    else if (n <= intro_vs_shell(ks))
        shell_sort(base, n, rs, ks);
    else
        intro_rec(base, n, 2 * log2_floor(n), INSERTION_MAX, rs, ks);
}

/* ------------------------------------------------------------------ MSD driver */

typedef struct {
    uint8_t* primary;
    uint8_t* aux;
    uint64_t n;
    uint32_t rs, ks;
} Msd;

typedef struct { /* Bin (kernels.hpp:60-67), next_byte as a significance index */
    uint64_t start, end;
    int next_byte;
    int parity;
} Bin;

static uint8_t* arr(Msd* m, int parity) { return parity ? m->aux : m->primary; }

static void finalize(Msd* m, Bin b) { /* msd_sorter.hpp:76-80 */
    if (b.parity && b.end > b.start)
        memcpy(m->primary + b.start * m->rs, m->aux + b.start * m->rs, (b.end - b.start) * m->rs);
}

static void split(Msd* m, Bin b, uint64_t* counts) {
    const uint32_t off = m->ks - 1 - (uint32_t)b.next_byte; /* offset_of, msd_sorter.hpp:69-71 */
    orc_radix_split(arr(m, b.parity) + b.start * m->rs, arr(m, 1 - b.parity) + b.start * m->rs,
                    b.end - b.start, m->rs, off, counts);
}

static void child_bins(const uint64_t* counts, Bin parent, Bin* out) { /* kernels.hpp:82-94 */
    uint64_t pos = parent.start;
    for (int d = 0; d < 256; ++d) {
        out[d].start = pos;
        pos += counts[d];
        out[d].end = pos;
        out[d].next_byte = parent.next_byte - 1;
        out[d].parity = 1 - parent.parity;
    }
}

static int is_big(uint64_t size, uint64_t n) { /* is_big_bin with T = 1: 3*size > 2*n */
    return (unsigned __int128)size * 3 > (unsigned __int128)2 * n;
}

/* msd_radix_bins (msd_sorter.hpp:180-214) */
static void msd_radix_bins(Msd* m, Bin b) {
    const uint64_t size = b.end - b.start;
    if (size <= 1) {
        finalize(m, b);
        return;
    }
    uint64_t counts[256];
    Bin kids[256];
    split(m, b, counts);
    child_bins(counts, b, kids);
    if (b.next_byte == 0) {
        Bin whole = {b.start, b.end, 0, 1 - b.parity};
        finalize(m, whole);
        return;
    }
    for (int d = 0; d < 256; ++d) {
        const Bin c = kids[d];
        const uint64_t cs = c.end - c.start;
        if (cs == 0) continue;
        if (orc_is_tiny(cs, size)) {
            orc_comparison_sort(arr(m, c.parity) + c.start * m->rs, cs, m->rs, m->ks);
            finalize(m, c);
        } else {
            msd_radix_bins(m, c);
        }
    }
}

/* big_partition_pass (msd_sorter.hpp:144-165); its non-big children are
 * queued and later served by msd_radix_bins (queue order never changes
 * content because bins are disjoint). */
static void big_partition_pass(Msd* m, Bin b) {
    uint64_t counts[256];
    Bin kids[256];
    split(m, b, counts);
    child_bins(counts, b, kids);
    if (b.next_byte == 0) {
        Bin whole = {b.start, b.end, 0, 1 - b.parity};
        finalize(m, whole);
        return;
    }
    for (int d = 0; d < 256; ++d) {
        const Bin c = kids[d];
        const uint64_t cs = c.end - c.start;
        if (cs == 0) continue;
        if (cs == 1) {
            finalize(m, c);
            continue;
        }
        if (is_big(cs, m->n))
            big_partition_pass(m, c);
        else
            msd_radix_bins(m, c);
    }
}

/* raduls::sort restated for T = 1 (scheduler.cpp:40-45 -> msd_sorter.hpp:50-126).
 * aux may be NULL (allocated here, like msd_sorter.hpp:52). */
int orc_msd_sort(uint8_t* data, uint64_t n, uint32_t rs, uint32_t ks, uint8_t* aux) {
    if (!layout_ok(rs, ks)) return ORC_EINVAL; /* dispatch.hpp:37-39 */
    if (n < 2) return ORC_OK;                 /* msd_sorter.hpp:51 */
    uint8_t* own = NULL;
    if (!aux) {
        own = (uint8_t*)malloc(n * rs);
        if (!own) return ORC_ENOMEM;
        aux = own;
    }
    Msd m = {data, aux, n, rs, ks};
    const Bin whole = {0, n, (int)ks - 1, 0};
    uint64_t counts[256];
    Bin kids[256];
    split(&m, whole, counts); /* first_pass, msd_sorter.hpp:89-126 */
    child_bins(counts, whole, kids);
    if (whole.next_byte == 0) {
        Bin all = {0, n, 0, 1};
        finalize(&m, all);
    } else {
        for (int d = 0; d < 256; ++d) { /* classify_bins with T = 1 */
            const Bin c = kids[d];
            const uint64_t cs = c.end - c.start;
            if (cs == 0) continue;
            if (is_big(cs, n)) {
                big_partition_pass(&m, c);
            } else if (cs == 1) {
                finalize(&m, c);
            } else {
                msd_radix_bins(&m, c);
            }
        }
    }
    free(own);
    return ORC_OK;
}

/* ------------------------------------------------------------------ verification */

static inline uint64_t load_le64(const uint8_t* p) {
    uint64_t v;
    memcpy(&v, p, 8);
    return v;
}

static inline uint64_t hash_mix(uint64_t x) {
    x = (x ^ (x >> 33)) * 0xff51afd7ed558ccdULL;
    x = (x ^ (x >> 33)) * 0xc4ceb9fe1a85ec53ULL;
    return x ^ (x >> 33);
}

/* array_digest (verify.cpp:37-50): sum mod 2^128 of one 128-bit hash per record */
void orc_digest(const uint8_t* base, uint64_t n, uint32_t rs, uint64_t* lo, uint64_t* hi) {
    unsigned __int128 acc = 0;
    const uint32_t words = rs / 8;
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t* rec = base + i * rs;
        uint64_t h = 0x8824a3d6f1e2c4b9ULL;
        for (uint32_t w = 0; w < words; ++w)
            h = hash_mix(h ^ (load_le64(rec + 8 * w) * 0x9ddfea08eb382d69ULL));
        const uint64_t l = hash_mix(h ^ 0xc3a5c85c97cb3127ULL);
        const uint64_t u = hash_mix(h ^ 0xb492b66fbe98f273ULL);
        acc += ((unsigned __int128)u << 64) | l;
    }
    *lo = (uint64_t)acc;
    *hi = (uint64_t)(acc >> 64);
}

/* check_sorted (verify.cpp:27-35): 1 if sorted, else 0 with the first i where
 * key(i+1) < key(i) */
int orc_check_sorted(const uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks,
                     uint64_t* first_violation) {
    for (uint64_t i = 0; i + 1 < n; ++i)
        if (key_less(base + (i + 1) * rs, base + i * rs, ks)) {
            if (first_violation) *first_violation = i;
            return 0;
        }
    return 1;
}

/* oracle_sort (verify.cpp:52-64): stable sort by key — bottom-up merge sort */
int orc_stable_sort(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
    if (n < 2) return ORC_OK;
    uint8_t* buf = (uint8_t*)malloc(n * rs);
    if (!buf) return ORC_ENOMEM;
    uint8_t *a = base, *b = buf;
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            uint64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            uint64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                if (key_less(a + j * rs, a + i * rs, ks))
                    memcpy(b + (k++) * rs, a + (j++) * rs, rs);
                else
                    memcpy(b + (k++) * rs, a + (i++) * rs, rs);
            }
            if (i < mid) memcpy(b + k * rs, a + i * rs, (mid - i) * rs), k += mid - i;
            if (j < hi) memcpy(b + k * rs, a + j * rs, (hi - j) * rs);
        }
        uint8_t* t = a;
        a = b;
        b = t;
    }
    if (a != base) memcpy(base, a, n * rs);
    free(buf);
    return ORC_OK;
}

/* canonical(x): sort every maximal equal-key run of a key-sorted array by the
 * full record bytes (SURVEY.md §0 parity definition). Returns 0 if the input
 * was not key-sorted. */
static uint32_t g_cmp_rs;
static int full_cmp(const void* x, const void* y) { return memcmp(x, y, g_cmp_rs); }

int orc_canonicalize(uint8_t* base, uint64_t n, uint32_t rs, uint32_t ks) {
    if (!orc_check_sorted(base, n, rs, ks, NULL)) return 0;
    g_cmp_rs = rs;
    uint64_t i = 0;
    while (i < n) {
        uint64_t j = i + 1;
        while (j < n && memcmp(base + j * rs, base + i * rs, ks) == 0) ++j;
        if (j - i > 1) qsort(base + i * rs, j - i, rs, full_cmp);
        i = j;
    }
    return 1;
}
