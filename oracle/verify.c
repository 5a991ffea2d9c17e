/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Invariants of a sort result that hold at any size (used where the full
 * serial oracle is too slow, e.g. 2^31 keys): output nondecreasing; output is a
 * permutation of the input (count + order-independent multiset hash); pair
 * output stable (payload = original index increases within equal keys);
 * sampled order statistics against the unsorted input.
 */
#include <stdlib.h>
#include "oracle.h"

static inline uint64_t h64(uint64_t z) {  /* SplitMix64 finaliser */
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

int or_is_nondecreasing_u32(const uint32_t* a, size_t n) {
    int ok = 1;
    #pragma omp parallel for reduction(&&:ok) schedule(static)
    for (long long i = 1; i < (long long)n; ++i) ok = ok && (a[i - 1] <= a[i]);
    return ok;
}

int or_is_nondecreasing_u64(const uint64_t* a, size_t n) {
    int ok = 1;
    #pragma omp parallel for reduction(&&:ok) schedule(static)
    for (long long i = 1; i < (long long)n; ++i) ok = ok && (a[i - 1] <= a[i]);
    return ok;
}

void or_multiset_hash_u32(const uint32_t* a, size_t n, uint64_t* out) {
    uint64_t s = 0, x = 0;
    #pragma omp parallel for reduction(+:s) reduction(^:x) schedule(static)
    for (long long i = 0; i < (long long)n; ++i) { uint64_t h = h64(a[i]); s += h; x ^= h; }
    out[0] = n; out[1] = s; out[2] = x;
}

void or_multiset_hash_u64(const uint64_t* a, size_t n, uint64_t* out) {
    uint64_t s = 0, x = 0;
    #pragma omp parallel for reduction(+:s) reduction(^:x) schedule(static)
    for (long long i = 0; i < (long long)n; ++i) { uint64_t h = h64(a[i]); s += h; x ^= h; }
    out[0] = n; out[1] = s; out[2] = x;
}

void or_multiset_hash_pairs_u64_u32(const uint64_t* k, const uint32_t* v, size_t n, uint64_t* out) {
    uint64_t s = 0, x = 0;
    #pragma omp parallel for reduction(+:s) reduction(^:x) schedule(static)
    for (long long i = 0; i < (long long)n; ++i) {
        uint64_t h = h64(h64(k[i]) ^ (0x100000001B3ULL * (uint64_t)v[i] + 0x9E3779B97F4A7C15ULL));
        s += h; x ^= h;
    }
    out[0] = n; out[1] = s; out[2] = x;
}

int or_pairs_stable_u64_u32(const uint64_t* k, const uint32_t* v, size_t n) {
    int ok = 1;
    #pragma omp parallel for reduction(&&:ok) schedule(static)
    for (long long i = 1; i < (long long)n; ++i)
        ok = ok && (k[i - 1] < k[i] || (k[i - 1] == k[i] && v[i - 1] < v[i]));
    return ok;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

/* For m sampled (pos, val) of a claimed sorted output: val is the pos-th
 * smallest key of a[] iff #{x < val} <= pos < #{x <= val}.  One pass over a[]
 * with a binary search into the sorted distinct sample values. */
size_t or_check_order_stats_u32(const uint32_t* a, size_t n, const uint64_t* pos,
                                const uint32_t* val, size_t m) {
    if (m == 0) return 0;
    uint32_t* sv = (uint32_t*)malloc(m * sizeof(uint32_t));
    uint64_t* lt = (uint64_t*)calloc(m, sizeof(uint64_t));
    uint64_t* le = (uint64_t*)calloc(m, sizeof(uint64_t));
    if (!sv || !lt || !le) { free(sv); free(lt); free(le); return m; }
    for (size_t i = 0; i < m; ++i) sv[i] = val[i];
    qsort(sv, m, sizeof(uint32_t), cmp_u32);
    size_t u = 0;
    for (size_t i = 0; i < m; ++i) if (i == 0 || sv[i] != sv[u - 1]) sv[u++] = sv[i];
    #pragma omp parallel
    {
        uint64_t* llt = (uint64_t*)calloc(u, sizeof(uint64_t));
        uint64_t* lle = (uint64_t*)calloc(u, sizeof(uint64_t));
        #pragma omp for schedule(static)
        for (long long i = 0; i < (long long)n; ++i) {
            uint32_t x = a[i];
            /* first sample value >= x  */
            size_t lo = 0, hi = u;
            while (lo < hi) { size_t mid = (lo + hi) / 2; if (sv[mid] < x) lo = mid + 1; else hi = mid; }
            /* x < sv[q] for q > lo (and for q = lo if sv[lo] > x); x <= sv[q] for q >= lo */
            if (lo < u) { lle[lo]++; if (sv[lo] > x) llt[lo]++; else if (lo + 1 < u) llt[lo + 1]++; }
        }
        #pragma omp critical
        for (size_t q = 0; q < u; ++q) { lt[q] += llt[q]; le[q] += lle[q]; }
        free(llt); free(lle);
    }
    /* prefix: #{x <= sv[q]} = Σ_{q'<=q} le-marks; #{x < sv[q]} = Σ_{q'<=q} lt-marks */
    for (size_t q = 1; q < u; ++q) { lt[q] += lt[q - 1]; le[q] += le[q - 1]; }
    size_t bad = 0;
    for (size_t i = 0; i < m; ++i) {
        size_t lo = 0, hi = u;
        while (lo < hi) { size_t mid = (lo + hi) / 2; if (sv[mid] < val[i]) lo = mid + 1; else hi = mid; }
        if (!(lt[lo] <= pos[i] && pos[i] < le[lo])) ++bad;
    }
    free(sv); free(lt); free(le);
    return bad;
}
