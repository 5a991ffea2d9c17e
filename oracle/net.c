/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * BTN and OET: the paper's two network sorts over p sorted blocks of N = n/p
 * keys, simulated for p processors inside one process.
 *
 *   BTN (§2, cost PAPER.md:741-763 §3.2): "a p-processor
 *       bitonic sorter can sort n keys in lg(p)(lg(p)+1)/2 stages"; each of the
 *       p 'keys' is a sorted sequence of n/p regular keys; "a comparison of two
 *       'keys' on two processors gets resolved by merging the two n/p sorted
 *       sequences ... and then assigning the lower half, the smaller keys, to the
 *       lower indexed ... and the upper half to the higher indexed processor".
 *       Local initial sorting is SR4.
 *   OET (§2, cost PAPER.md:717-738 §3.2): p-wide p-round
 *       odd-even transposition sort of the p sorted blocks; in one round the
 *       pairs of adjacent processors merge-split, "the smaller n/p keys ... to
 *       the lower-indexed, and the latter to the next-indexed processor".
 *
 * Readings (R32-R34):
 *   R32 the bitonic network is the standard one: for stage
 *       k = 1..lg p, substage j = k..1, processor i pairs with i XOR 2^{j-1};
 *       the pair's direction is ascending iff bit k of i is 0; ascending keeps
 *       the smaller half at the lower index, descending at the higher index.
 *   R33 OET round t = 0..p-1 pairs (0,1),(2,3),... for even t and
 *       (1,2),(3,4),... for odd t.
 *   R34 every block has the same size N (the paper's n/p; SPEC.md "~n/p" is
 *       read as equal blocks, p | n); a merge-split merges the lower-indexed
 *       block first on ties (stable merge), each side keeps N keys; values move
 *       with their keys.  OET is then stable; BTN is not (a descending exchange
 *       hands the later equal keys to the lower index) — its values are only
 *       permuted with their keys.
 *
 * Each merge-split below is the plain definition: a two-finger merge of the two
 * blocks into a 2N scratch, then the halves are copied out.
 */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* merge blocks lo (index i) and hi (index i' > i); keep_low_at_lo: the smaller
 * N keys go to lo (ascending exchange), else to hi */
#define DEFINE_MERGE_SPLIT(NAME, KT)                                                         \
    static void NAME(KT* lo, uint32_t* vlo, KT* hi, uint32_t* vhi, size_t N, int keep_low_at_lo, \
                     KT* tk, uint32_t* tv) {                                                 \
        size_t a = 0, b = 0, o = 0;                                                          \
        while (a < N || b < N) {                                                             \
            int take_lo = b >= N || (a < N && lo[a] <= hi[b]); /* ties: lower index */       \
            if (take_lo) {                                                                   \
                tk[o] = lo[a];                                                               \
                if (tv) tv[o] = vlo[a];                                                      \
                ++a;                                                                         \
            } else {                                                                         \
                tk[o] = hi[b];                                                               \
                if (tv) tv[o] = vhi[b];                                                      \
                ++b;                                                                         \
            }                                                                                \
            ++o;                                                                             \
        }                                                                                    \
        KT* small_dst = keep_low_at_lo ? lo : hi;                                            \
        KT* large_dst = keep_low_at_lo ? hi : lo;                                            \
        memcpy(small_dst, tk, N * sizeof(KT));                                               \
        memcpy(large_dst, tk + N, N * sizeof(KT));                                           \
        if (tv) {                                                                            \
            uint32_t* vs = keep_low_at_lo ? vlo : vhi;                                       \
            uint32_t* vl = keep_low_at_lo ? vhi : vlo;                                       \
            memcpy(vs, tv, N * 4);                                                           \
            memcpy(vl, tv + N, N * 4);                                                       \
        }                                                                                    \
    }

DEFINE_MERGE_SPLIT(merge_split_u32, uint32_t)
DEFINE_MERGE_SPLIT(merge_split_u64, uint64_t)

static int is_pow2(int p) { return p >= 1 && (p & (p - 1)) == 0; }

static int lg(int p) {
    int m = 0;
    while ((1 << m) < p) ++m;
    return m;
}

/* the common driver: mode 0 BTN, 1 OET; kb key bytes */
static int net_sort(int mode, int kb, int p, int b, void* keys, uint32_t* vals, size_t N, int max_stages,
                    int* stages) {
    if (p < 1 || !keys || (mode == 0 && !is_pow2(p)) || (kb == 4 && vals)) return -1;
    if (stages) *stages = 0;
    /* local initial sorting: SR-b of every block */
    for (int k = 0; k < p; ++k) {
        int rc;
        if (kb == 4) rc = or_sr_u32((uint32_t*)keys + (size_t)k * N, N, b, -1);
        else if (vals) rc = or_sr_pairs_u64_u32((uint64_t*)keys + (size_t)k * N, vals + (size_t)k * N, N, b, -1);
        else rc = or_sr_u64((uint64_t*)keys + (size_t)k * N, N, b, -1);
        if (rc) return -1;
    }
    void* tk = malloc(2 * N * (size_t)kb + 8);
    uint32_t* tv = vals ? (uint32_t*)malloc(2 * N * 4 + 8) : NULL;
    if (!tk || (vals && !tv)) {
        free(tk);
        free(tv);
        return -1;
    }
#define BLK(i) ((char*)keys + (size_t)(i) * N * (size_t)kb)
#define VBLK(i) (vals ? vals + (size_t)(i) * N : NULL)
#define XCHG(i, i2, asc)                                                                                  \
    do {                                                                                                  \
        if (kb == 4)                                                                                      \
            merge_split_u32((uint32_t*)BLK(i), NULL, (uint32_t*)BLK(i2), NULL, N, asc, (uint32_t*)tk, NULL); \
        else                                                                                              \
            merge_split_u64((uint64_t*)BLK(i), VBLK(i), (uint64_t*)BLK(i2), VBLK(i2), N, asc, (uint64_t*)tk, \
                            tv);                                                                          \
    } while (0)
    int done = 0;
    if (mode == 0) {
        const int m = lg(p);
        for (int k = 1; k <= m; ++k)
            for (int j = k; j >= 1; --j) {
                if (max_stages >= 0 && done >= max_stages) goto out;
                for (int i = 0; i < p; ++i) {
                    const int partner = i ^ (1 << (j - 1));
                    if (partner <= i) continue; /* each pair once, from its lower index */
                    const int ascending = ((i >> k) & 1) == 0;
                    XCHG(i, partner, ascending);
                }
                ++done;
            }
    } else {
        for (int t = 0; t < p; ++t) {
            if (max_stages >= 0 && done >= max_stages) goto out;
            for (int i = t % 2; i + 1 < p; i += 2) XCHG(i, i + 1, 1);
            ++done;
        }
    }
out:
#undef XCHG
#undef VBLK
#undef BLK
    if (stages) *stages = done;
    free(tk);
    free(tv);
    return 0;
}

int or_btn_u32(int p, int b, uint32_t* keys, size_t N, int max_stages, int* stages) {
    return net_sort(0, 4, p, b, keys, NULL, N, max_stages, stages);
}
int or_btn_u64(int p, int b, uint64_t* keys, uint32_t* vals, size_t N, int max_stages, int* stages) {
    return net_sort(0, 8, p, b, keys, vals, N, max_stages, stages);
}
int or_oet_u32(int p, int b, uint32_t* keys, size_t N, int max_stages, int* stages) {
    return net_sort(1, 4, p, b, keys, NULL, N, max_stages, stages);
}
int or_oet_u64(int p, int b, uint64_t* keys, uint32_t* vals, size_t N, int max_stages, int* stages) {
    return net_sort(1, 8, p, b, keys, vals, N, max_stages, stages);
}
