/*
 * qms_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference QuickMergesort hot path
 * (/root/reference/proj/core/include/qmsort/) in plain C, used as the parity
 * checker for the B200 sort.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path (paper_1804_10062_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against
 *   - the reference's own golden vectors (Fig. 1 array, test_sort.cpp:24,37-45;
 *     swap_merge examples, test_merge.cpp:48-85; generator patterns,
 *     test_dataset.cpp:18-24),
 *   - outputs of the reference itself compiled here from /root/reference into
 *     oracle/_ref/ (oracle/Makefile), frozen under tests/golden/.
 *
 * Every function cites the reference routine it restates.  The element types
 * are the five BASELINE.json configs: int32, uint32, uint64, float64 and a
 * 32-byte record of four uint64 words compared lexicographically.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct { uint64_t w[4]; } qmso_rec32;

enum { QMSO_I32 = 0, QMSO_U32 = 1, QMSO_U64 = 2, QMSO_F64 = 3, QMSO_REC32 = 4, QMSO_I64 = 5 };
enum { QMSO_PIVOT_MEDIAN_OF_3 = 0, QMSO_PIVOT_MEDIAN_OF_SQRT_N = 1 };

/* ------------------------------------------------------------------------ */
/* Comparators: "less" per element type; greater = swapped arguments.       */
/* ------------------------------------------------------------------------ */
static inline int lt_i32(const int32_t *a, const int32_t *b) { return *a < *b; }
static inline int lt_i64(const int64_t *a, const int64_t *b) { return *a < *b; }
static inline int lt_u32(const uint32_t *a, const uint32_t *b) { return *a < *b; }
static inline int lt_u64(const uint64_t *a, const uint64_t *b) { return *a < *b; }
static inline int lt_f64(const double *a, const double *b) { return *a < *b; }
static inline int lt_rec(const qmso_rec32 *a, const qmso_rec32 *b) {
    for (int i = 0; i < 4; ++i)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i];
    return 0;
}

/*
 * QMSO_DEFINE(SFX, T, LESS) instantiates the QuickMergesort routines for one
 * element type T with comparator LESS(const T*, const T*).
 */
#define QMSO_DEFINE(SFX, T, LESS)                                                        \
    static inline void swp_##SFX(T *a, T *b) { T t = *a; *a = *b; *b = t; }             \
                                                                                         \
    /* binary_insertion_sort: small_sort.hpp:33-55 */                                    \
    static void bins_##SFX(T *a, size_t n, int g) {                                      \
        for (size_t i = 1; i < n; ++i) {                                                 \
            size_t lo = 0, hi = i;                                                       \
            while (lo < hi) {                                                            \
                size_t mid = lo + (hi - lo) / 2;                                         \
                int c = g ? LESS(&a[mid], &a[i]) : LESS(&a[i], &a[mid]);                 \
                if (c) hi = mid; else lo = mid + 1;                                      \
            }                                                                            \
            if (lo == i) continue;                                                       \
            T v = a[i];                                                                  \
            memmove(&a[lo + 1], &a[lo], (i - lo) * sizeof(T));                           \
            a[lo] = v;                                                                   \
        }                                                                                \
    }                                                                                    \
    static inline int cmp_##SFX(const T *x, const T *y, int g) {                         \
        return g ? LESS(y, x) : LESS(x, y);                                              \
    }                                                                                    \
    /* sort2/sort3/sort4: small_sort.hpp:59-86 */                                        \
    static inline void s2_##SFX(T *a, T *b, int g) { if (cmp_##SFX(b, a, g)) swp_##SFX(a, b); } \
    static void small_sort_##SFX(T *a, size_t n, int g) { /* small_sort.hpp:92-111 */    \
        switch (n) {                                                                     \
            case 0: case 1: return;                                                      \
            case 2: s2_##SFX(a, a + 1, g); return;                                       \
            case 3:                                                                      \
                s2_##SFX(a, a + 1, g);                                                   \
                if (cmp_##SFX(a + 2, a + 1, g)) {                                        \
                    swp_##SFX(a + 1, a + 2);                                             \
                    s2_##SFX(a, a + 1, g);                                               \
                }                                                                        \
                return;                                                                  \
            case 4:                                                                      \
                s2_##SFX(a, a + 1, g);                                                   \
                s2_##SFX(a + 2, a + 3, g);                                               \
                if (cmp_##SFX(a + 2, a, g)) { swp_##SFX(a, a + 2); swp_##SFX(a + 1, a + 3); } \
                if (cmp_##SFX(a + 2, a + 1, g)) {                                        \
                    swp_##SFX(a + 1, a + 2);                                             \
                    s2_##SFX(a + 2, a + 3, g);                                           \
                }                                                                        \
                return;                                                                  \
            default: bins_##SFX(a, n, g); return;                                        \
        }                                                                                \
    }                                                                                    \
                                                                                         \
    /* swap_merge: merge.hpp:64-97 (paper Fig. 2 `merge`).  run1 = [b1,e1) merges   */   \
    /* with run2 occupying the tail of out = [t,te); displaced slots park in run1. */   \
    static void swap_merge_##SFX(T *b1, T *e1, T *t, T *te, int g) {                     \
        size_t n1 = (size_t)(e1 - b1);                                                   \
        if (n1 == 0) return;                                                             \
        T *i1 = b1, *i2 = t + n1, *res = t;                                              \
        T first_displaced = *t;                                                          \
        while (i1 != e1 && i2 != te) {                                                   \
            T *src = cmp_##SFX(i2, i1, g) ? i2++ : i1++; /* ties take run1 (76) */      \
            *res = *src;                                                                 \
            ++res;                                                                       \
            *src = *res;                                                                 \
        }                                                                                \
        while (i1 != e1) {                                                               \
            *res = *i1;                                                                  \
            ++res;                                                                       \
            if (res != te) *i1 = *res;                                                   \
            ++i1;                                                                        \
        }                                                                                \
        *(e1 - 1) = first_displaced;                                                     \
    }                                                                                    \
                                                                                         \
    /* mergesort_into: merge.hpp:103-119 (Fig. 2 `msort`), X = small_sort below 10 */   \
    static void msort_into_##SFX(T *b, T *e, T *tgt, int g) {                            \
        size_t n = (size_t)(e - b);                                                      \
        if (n == 0) return;                                                              \
        if (n < 10) { /* base_case_reached, merge.hpp:51-55 */                           \
            small_sort_##SFX(b, n, g);                                                   \
            for (size_t i = 0; i < n; ++i) swp_##SFX(b + i, tgt + i);                    \
            return;                                                                      \
        }                                                                                \
        size_t q = n / 2;                                                                \
        msort_into_##SFX(b + q, e, tgt + q, g);                                          \
        msort_into_##SFX(b, b + q, b + q, g);                                            \
        swap_merge_##SFX(b + q, b + 2 * q, tgt, tgt + n, g);                             \
    }                                                                                    \
                                                                                         \
    /* mergesort_with_temp: merge.hpp:124-135 (Fig. 2 `out`) */                          \
    static void msort_temp_##SFX(T *b, T *e, T *tmp, int g) {                            \
        size_t n = (size_t)(e - b);                                                      \
        if (n < 2) return;                                                               \
        size_t q = n / 2, r = n - q;                                                     \
        msort_into_##SFX(b + q, e, tmp, g);                                              \
        msort_into_##SFX(b, b + q, b + r, g);                                            \
        swap_merge_##SFX(tmp, tmp + r, b, e, g);                                         \
    }                                                                                    \
                                                                                         \
    /* median_of_3_index: partition.hpp:21-30 */                                         \
    static size_t mo3_##SFX(T *a, size_t i, size_t j, size_t k, int g) {                 \
        size_t t;                                                                        \
        if (cmp_##SFX(&a[j], &a[i], g)) { t = i; i = j; j = t; }                         \
        if (cmp_##SFX(&a[k], &a[j], g)) {                                                \
            t = j; j = k; k = t;                                                         \
            if (cmp_##SFX(&a[j], &a[i], g)) { t = i; i = j; j = t; }                     \
        }                                                                                \
        return j;                                                                        \
    }                                                                                    \
                                                                                         \
    /* Exact k-th smallest (1-based) of a[0..s) by quickselect; stands in for        */ \
    /* select_kth (selection.hpp:131-203): same rank, same returned element value.  */ \
    static size_t select_##SFX(T *a, size_t s, size_t k, int g) {                        \
        size_t lo = 0, hi = s; /* [lo,hi) holds rank k-1 */                              \
        size_t want = k - 1;                                                             \
        while (hi - lo > 1) {                                                            \
            size_t p = mo3_##SFX(a, lo, lo + (hi - lo) / 2, hi - 1, g);                  \
            swp_##SFX(&a[lo], &a[p]);                                                    \
            size_t lt = lo, i = lo + 1, gt = hi; /* three_way, partition.hpp:196-230 */  \
            T pv = a[lo];                                                                \
            while (i < gt) {                                                             \
                if (cmp_##SFX(&a[i], &pv, g)) { swp_##SFX(&a[lt], &a[i]); ++lt; ++i; }   \
                else if (cmp_##SFX(&pv, &a[i], g)) { --gt; swp_##SFX(&a[i], &a[gt]); }   \
                else ++i;                                                                \
            }                                                                            \
            if (want < lt) hi = lt;                                                      \
            else if (want >= gt) lo = gt;                                                \
            else return want;                                                            \
        }                                                                                \
        return want;                                                                     \
    }                                                                                    \
                                                                                         \
    /* median_of_sqrt_pivot: partition.hpp:235-251 */                                    \
    static size_t mosqrt_##SFX(T *a, size_t n, int g) {                                  \
        size_t root = 1;                                                                 \
        while ((root + 1) * (root + 1) <= n) ++root;                                     \
        size_t s = 2 * (root / 2) + 1, stride = n / s;                                   \
        for (size_t i = 0; i < s; ++i)                                                   \
            if (i * stride != i) swp_##SFX(&a[i], &a[i * stride]);                       \
        return select_##SFX(a, s, (s + 1) / 2, g);                                       \
    }                                                                                    \
                                                                                         \
    /* Hoare partition around a[piv]: restates block_partition's contract          */   \
    /* (partition.hpp:37-164): pivot lands at the split, [0,split) !> pivot,       */   \
    /* (split,n) !< pivot, equal keys may fall on either side.                      */   \
    static size_t partition_##SFX(T *a, size_t n, size_t piv, int g) {                  \
        swp_##SFX(&a[0], &a[piv]);                                                       \
        T pv = a[0];                                                                     \
        size_t i = 0, j = n;                                                             \
        for (;;) {                                                                       \
            do { ++i; } while (i < n && cmp_##SFX(&a[i], &pv, g));                       \
            do { --j; } while (cmp_##SFX(&pv, &a[j], g));                                \
            if (i >= j) break;                                                           \
            swp_##SFX(&a[i], &a[j]);                                                     \
        }                                                                                \
        swp_##SFX(&a[0], &a[j]);                                                         \
        return j;                                                                        \
    }                                                                                    \
                                                                                         \
    /* quickmergesort_impl: sort.hpp:128-201 with the qms() preset (sort.hpp:37)    */  \
    static void qms_##SFX(T *a, size_t n_all, int g, int pivot) {                        \
        T *begin = a, *end = a + n_all;                                                  \
        for (;;) {                                                                       \
            size_t n = (size_t)(end - begin);                                            \
            if (n <= 1) return;                                                          \
            if (n < 10) { small_sort_##SFX(begin, n, g); return; } /* driver_cutoff */  \
            size_t piv = (pivot == QMSO_PIVOT_MEDIAN_OF_SQRT_N)                          \
                             ? mosqrt_##SFX(begin, n, g)                                 \
                             : mo3_##SFX(begin, 0, n / 2, n - 1, g);                     \
            size_t split = partition_##SFX(begin, n, piv, g);                            \
            size_t left_n = split, right_n = n - split - 1;                              \
            /* choose_mergesort_side: sort.hpp:101-110 (larger_when_feasible) */         \
            int left_smaller = left_n <= right_n;                                        \
            size_t larger_n = left_smaller ? right_n : left_n;                           \
            size_t temp_n = left_smaller ? left_n : right_n;                             \
            int side_left = (temp_n >= larger_n - larger_n / 2) ? !left_smaller : left_smaller; \
            if (side_left) {                                                             \
                msort_temp_##SFX(begin, begin + left_n, begin + split + 1, g);           \
                begin += split + 1;                                                      \
            } else {                                                                     \
                msort_temp_##SFX(begin + split + 1, end, begin, g);                      \
                end = begin + split;                                                     \
            }                                                                            \
        }                                                                                \
    }

QMSO_DEFINE(i32, int32_t, lt_i32)
QMSO_DEFINE(i64, int64_t, lt_i64)
QMSO_DEFINE(u32, uint32_t, lt_u32)
QMSO_DEFINE(u64, uint64_t, lt_u64)
QMSO_DEFINE(f64, double, lt_f64)
QMSO_DEFINE(rec, qmso_rec32, lt_rec)

/* ------------------------------------------------------------------------ */
/* Exported entry points (ctypes).                                          */
/* ------------------------------------------------------------------------ */

/* Sort data[0..n) of dtype in place; greater != 0 sorts by std::greater.
 * Returns 0, or -1 for a bad dtype. */
int qmso_sort(int dtype, int greater, int pivot, void *data, size_t n) {
    switch (dtype) {
        case QMSO_I32: qms_i32((int32_t *)data, n, greater, pivot); return 0;
        case QMSO_I64: qms_i64((int64_t *)data, n, greater, pivot); return 0;
        case QMSO_U32: qms_u32((uint32_t *)data, n, greater, pivot); return 0;
        case QMSO_U64: qms_u64((uint64_t *)data, n, greater, pivot); return 0;
        case QMSO_F64: qms_f64((double *)data, n, greater, pivot); return 0;
        case QMSO_REC32: qms_rec((qmso_rec32 *)data, n, greater, pivot); return 0;
    }
    return -1;
}

/* swap_merge on int64 test vectors (test_merge.cpp:48-85 golden examples).
 * data holds the whole array; run1 = [b1,e1), out = [t,te) as indices. */
void qmso_swap_merge_i64(int64_t *data, size_t b1, size_t e1, size_t t, size_t te) {
    swap_merge_i64(data + b1, data + e1, data + t, data + te, 0);
}

/* Is data[0..n) sorted (non-decreasing under less, or under greater)? */
int qmso_is_sorted(int dtype, int greater, const void *data, size_t n) {
    for (size_t i = 1; i < n; ++i) {
        int bad = 0;
        switch (dtype) {
            case QMSO_I32: bad = cmp_i32((const int32_t *)data + i, (const int32_t *)data + i - 1, greater); break;
            case QMSO_I64: bad = cmp_i64((const int64_t *)data + i, (const int64_t *)data + i - 1, greater); break;
            case QMSO_U32: bad = cmp_u32((const uint32_t *)data + i, (const uint32_t *)data + i - 1, greater); break;
            case QMSO_U64: bad = cmp_u64((const uint64_t *)data + i, (const uint64_t *)data + i - 1, greater); break;
            case QMSO_F64: bad = cmp_f64((const double *)data + i, (const double *)data + i - 1, greater); break;
            case QMSO_REC32: bad = cmp_rec((const qmso_rec32 *)data + i, (const qmso_rec32 *)data + i - 1, greater); break;
            default: return -1;
        }
        if (bad) return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Seeded generators: rng.hpp:10-38 (SplitMix64, bounded) and the           */
/* dataset.hpp:62-99 recipes as pinned in SURVEY.md 8(d).                   */
/* ------------------------------------------------------------------------ */
#define QMSO_GAMMA 0x9E3779B97F4A7C15ull
static inline uint64_t sm_mix(uint64_t z) { /* rng.hpp:14-19 finaliser */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* j-th output (0-based) of SplitMix64(seed): counter form. */
uint64_t qmso_sm(uint64_t seed, uint64_t j) { return sm_mix(seed + (j + 1) * QMSO_GAMMA); }

/* bounded(): rng.hpp:26-38, 128-bit multiply with rejection */
static uint64_t bounded_seq(uint64_t *state, uint64_t n) {
    if (n <= 1) return 0;
    *state += QMSO_GAMMA;
    unsigned __int128 mul = (unsigned __int128)sm_mix(*state) * n;
    uint64_t low = (uint64_t)mul;
    if (low < n) {
        uint64_t threshold = (0 - n) % n;
        while (low < threshold) {
            *state += QMSO_GAMMA;
            mul = (unsigned __int128)sm_mix(*state) * n;
            low = (uint64_t)mul;
        }
    }
    return (uint64_t)(mul >> 64);
}

/* generate_input({random_perm}, n, seed) (dataset.hpp:66-73), as int64 1..n. */
void qmso_gen_perm_i64(int64_t *v, size_t n, uint64_t seed) {
    for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(i + 1);
    uint64_t st = seed;
    for (size_t i = n; i > 1; --i) {
        size_t j = (size_t)bounded_seq(&st, i);
        int64_t t = v[i - 1]; v[i - 1] = v[j]; v[j] = t;
    }
}

/* generate_input({random_dup, m}, n, seed) (dataset.hpp:90-95). */
void qmso_gen_randomdup_i64(int64_t *v, size_t n, uint64_t seed, uint64_t m) {
    uint64_t st = seed;
    for (size_t i = 0; i < n; ++i) v[i] = (int64_t)(bounded_seq(&st, m ? m : 1) + 1);
}

/* Config recipes; `start` is the global index of element 0
 * so that shard r of P can generate its own slice. */
void qmso_gen_u32_uniform(uint32_t *v, size_t n, uint64_t seed, uint64_t start) {
    for (size_t i = 0; i < n; ++i) v[i] = (uint32_t)(qmso_sm(seed, start + i) >> 32);
}
void qmso_gen_u64_uniform(uint64_t *v, size_t n, uint64_t seed, uint64_t start) {
    for (size_t i = 0; i < n; ++i) v[i] = qmso_sm(seed, start + i);
}
void qmso_gen_rec32(qmso_rec32 *v, size_t n, uint64_t seed, uint64_t start) {
    for (size_t i = 0; i < n; ++i) {
        uint64_t g = start + i;
        v[i].w[0] = qmso_sm(seed, 4 * g) >> 52;
        v[i].w[1] = qmso_sm(seed, 4 * g + 1);
        v[i].w[2] = qmso_sm(seed, 4 * g + 2);
        v[i].w[3] = qmso_sm(seed, 4 * g + 3);
    }
}
/* f64 stress cases: 0 sorted, 1 reverse, 2 sixteen-distinct, 3 gaussian,
 * 4 organ-pipe. */
void qmso_gen_f64(double *v, size_t n, uint64_t seed, int kind) {
    for (size_t i = 0; i < n; ++i) {
        switch (kind) {
            case 0: v[i] = (double)(i + 1); break;
            case 1: v[i] = (double)(n - i); break;
            case 2: v[i] = (double)((qmso_sm(seed, i) >> 60) + 1); break;
            case 4: v[i] = (double)((i + 1) < (n - i) ? (i + 1) : (n - i)); break;
            case 3: {
                uint64_t k = i / 2;
                double u1 = (double)((qmso_sm(seed, 2 * k) >> 11) + 1) * 0x1.0p-53;
                double u2 = (double)(qmso_sm(seed, 2 * k + 1) >> 11) * 0x1.0p-53;
                double r = sqrt(-2.0 * log(u1));
                double x = (i & 1) ? r * sin(6.283185307179586 * u2) : r * cos(6.283185307179586 * u2);
                v[i] = (x == 0.0) ? 0.0 : x; /* canonicalise -0.0 */
                break;
            }
        }
    }
}
