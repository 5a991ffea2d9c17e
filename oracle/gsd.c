/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * GSD(X, n, p): deterministic regular oversampling sort
 * (§3.3, Algorithm 1), simulated for p processors inside one process.  Each
 * step below is one line of Algorithm 1, in the paper's order and notation:
 *
 *   1 LocalSorting   X_k = SR-b(k-th block)
 *   2 SampleSelect   r = ⌈ω⌉, s = r·p; T_k = rp−1 evenly spaced keys of X_k
 *                    partitioning it into rp segments, plus max(X_k);
 *                    T = sort(∪ T_k)  (rp² keys)
 *   3 SplitterSelect S_i = (i·s)-th smallest of T, 1 ≤ i ≤ p−1
 *   4 Split          X_{k,j} by binary search of S in X_k;
 *                    processor k sends X_{k,j} to processor j
 *   5 Merging        Y_j = p-way merge of X_{0,j}, …, X_{p−1,j}
 *
 * Readings where the paper is silent:
 *   R10 sample position of the i-th key: ⌈N_k·i/s⌉ − 1 (0-based), i = 1..s−1,
 *       then N_k − 1 (the maximum).  An empty block contributes s copies of
 *       the +∞ composite (KEY_MAX, k, POS_INF).
 *   R11 the sample is sorted with a library sort (composites are a total order,
 *       so any exact sort gives the same T; BTN is only how the paper sorts it).
 *   R12 S_i = T[i·s − 1] (0-based).
 *   R14/R15 elements are compared as composites (key, rank k, position in X_k),
 *       lexicographically; bucket j = {e : S_{j−1} <_c e ≤_c S_j}, S_0 = −∞,
 *       S_p = +∞ ("≤ splitter goes to the lower bucket").  This is
 *       also how duplicates are handled (the paper's promised discussion,
 *       PAPER.md:911-912, is absent).
 *   R16 ties in the merge go to the lower source rank, so a pair sort whose
 *       payload is the global index stays globally stable.
 *
 * Step 4 is written as its plain definition: count the composites of X_k that
 * are ≤_c S_j by a linear scan (the paper's binary search returns the same
 * number because X_k is sorted).  Step 5 repeatedly takes the smallest head,
 * lowest source rank on ties.
 *
 * GER(X, n, p) (Algorithm "GER") is the same skeleton with
 * step 2 replaced by random oversampling: "the sample consists of sp−1 keys
 * selected uniformly at random from the keys of all X_k".
 * Readings (R28-R30):
 *   R28 draw i = 0..sp−2: z_i = SplitMix64 in counter form (this file's own
 *       copy: z = seed + (i+1)·0x9E3779B97F4A7C15, then the standard finaliser),
 *       global position q_i = ⌊z_i · n / 2^64⌋ of the concatenation X_0‖…‖X_{p−1}
 *       of the sorted blocks (with replacement: equal draws give equal composites);
 *   R29 the key drawn at q_i is the composite (X_k[q_i − off_k], k, q_i − off_k),
 *       off_k = N_0 + … + N_{k−1} — so splitting, duplicates and stability are
 *       exactly GSD's (R14-R16); n = 0 gives +∞ composites;
 *   R30 s = 2⌈ω⌉²⌈lg n⌉ with ω = lg lg n unless the caller fixes s.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

#define POS_INF UINT64_MAX

typedef struct { uint64_t key, rank, pos; } composite_t;

static int comp_cmp(const composite_t* a, const composite_t* b) {
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->rank != b->rank) return a->rank < b->rank ? -1 : 1;
    if (a->pos != b->pos) return a->pos < b->pos ? -1 : 1;
    return 0;
}
static int comp_qsort(const void* a, const void* b) {
    return comp_cmp((const composite_t*)a, (const composite_t*)b);
}

/* SplitMix64 (this file's copy; pinned by tests/test_oracle_gsd.py against the
 * published vector): the i-th output of the sequential generator seeded `seed`. */
static uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t or_splitmix64_at(uint64_t seed, uint64_t i) { return splitmix64_at(seed, i); }

/* mode 0: GSD, s = r·p samples per block (regular);  mode 1: GER, s·p − 1 random
 * samples of the whole input (R28-R29).  Everything else is shared. */
static int sample_sort_u64(int p, int mode, size_t s, uint64_t seed, int b,
                           const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
                           uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
                           uint64_t* splitters, uint64_t* counts) {
    if (p < 1 || s < 1 || (b != 8 && b != 16)) return -1;
    int rc = 0;
    const size_t M = mode == 0 ? s * (size_t)p : s * (size_t)p - 1;  /* sample size */
    uint64_t** X = (uint64_t**)calloc((size_t)p, sizeof(uint64_t*));
    uint32_t** V = (uint32_t**)calloc((size_t)p, sizeof(uint32_t*));
    composite_t* T = (composite_t*)malloc((M ? M : 1) * sizeof(composite_t));
    composite_t* S = (composite_t*)malloc((size_t)p * sizeof(composite_t));
    size_t* cut = (size_t*)malloc((size_t)p * ((size_t)p + 1) * sizeof(size_t));
    size_t* head = (size_t*)malloc((size_t)p * sizeof(size_t));
    if (!X || !V || !T || !S || !cut || !head) { rc = -1; goto done; }

    /* Step 1: LocalSorting — X_k = SR-b(block k) (stable: pairs keep order). */
    for (int k = 0; k < p; ++k) {
        X[k] = (uint64_t*)malloc((N[k] ? N[k] : 1) * sizeof(uint64_t));
        if (!X[k]) { rc = -1; goto done; }
        memcpy(X[k], keys[k], N[k] * sizeof(uint64_t));
        if (vals) {
            V[k] = (uint32_t*)malloc((N[k] ? N[k] : 1) * sizeof(uint32_t));
            if (!V[k]) { rc = -1; goto done; }
            memcpy(V[k], vals[k], N[k] * sizeof(uint32_t));
            if (or_sr_pairs_u64_u32(X[k], V[k], N[k], b, -1)) { rc = -1; goto done; }
        } else if (or_sr_u64(X[k], N[k], b, -1)) { rc = -1; goto done; }
    }

    /* Step 2 (GER): sp−1 keys drawn uniformly at random from all X_k (R28, R29). */
    if (mode == 1) {
        size_t n = 0;
        for (int k = 0; k < p; ++k) n += N[k];
        for (size_t i = 0; i < M; ++i) {
            composite_t c = { UINT64_MAX, 0, POS_INF };
            if (n) {
                const uint64_t q = (uint64_t)(((unsigned __int128)splitmix64_at(seed, i) * n) >> 64);
                uint64_t off = 0;
                for (int k = 0; k < p; ++k) {   /* owner: off_k <= q < off_k + N_k */
                    if (q < off + N[k]) { c.key = X[k][q - off]; c.rank = (uint64_t)k; c.pos = q - off; break; }
                    off += N[k];
                }
            }
            T[i] = c;
        }
    }
    /* Step 2 (GSD): Sample selection — T_k (R10), then T = sort(∪ T_k) (R11). */
    for (int k = 0; k < p && mode == 0; ++k) {
        composite_t* Tk = T + (size_t)k * s;
        for (size_t i = 1; i <= s; ++i) {
            composite_t c;
            if (N[k] == 0) { c.key = UINT64_MAX; c.rank = (uint64_t)k; c.pos = POS_INF; }
            else {
                size_t pos = (i < s) ? (size_t)((N[k] * i + s - 1) / s) - 1   /* ⌈N·i/s⌉−1 */
                                     : N[k] - 1;                               /* the maximum */
                c.key = X[k][pos]; c.rank = (uint64_t)k; c.pos = pos;
            }
            Tk[i - 1] = c;
        }
    }
    qsort(T, M, sizeof(composite_t), comp_qsort);

    /* Step 3: Splitter selection — S_i = T[i·s − 1], 1 ≤ i ≤ p−1 (R12). */
    for (int i = 1; i < p; ++i) {
        S[i] = T[(size_t)i * s - 1];
        if (splitters) {
            splitters[3 * (i - 1) + 0] = S[i].key;
            splitters[3 * (i - 1) + 1] = S[i].rank;
            splitters[3 * (i - 1) + 2] = S[i].pos;
        }
    }

    /* Step 4: Split — cut[k][j] = #{e ∈ X_k : e ≤_c S_j} (R14), cut[k][0] = 0,
     * cut[k][p] = N_k; X_{k,j} = X_k[cut[k][j], cut[k][j+1]). */
    for (int k = 0; k < p; ++k) {
        size_t* ck = cut + (size_t)k * (p + 1);
        ck[0] = 0; ck[p] = N[k];
        for (int j = 1; j < p; ++j) {
            size_t c = 0;
            for (size_t q = 0; q < N[k]; ++q) {
                composite_t e = { X[k][q], (uint64_t)k, q };
                if (comp_cmp(&e, &S[j]) <= 0) ++c;
            }
            ck[j] = c;
        }
        for (int j = 0; j < p; ++j) if (counts) counts[(size_t)k * p + j] = ck[j + 1] - ck[j];
    }

    /* Step 5: Merging — Y_j = p-way merge of X_{k,j}, ties to the lower k (R16). */
    for (int j = 0; j < p; ++j) {
        size_t total = 0;
        for (int k = 0; k < p; ++k) {
            size_t* ck = cut + (size_t)k * (p + 1);
            head[k] = ck[j];
            total += ck[j + 1] - ck[j];
        }
        Ylen[j] = total;
        if (total > Ycap) { rc = -2; continue; }
        for (size_t o = 0; o < total; ++o) {
            int best = -1;
            for (int k = 0; k < p; ++k) {
                size_t end = cut[(size_t)k * (p + 1) + j + 1];
                if (head[k] >= end) continue;
                if (best < 0 || X[k][head[k]] < X[best][head[best]]) best = k;
            }
            Y_keys[j][o] = X[best][head[best]];
            if (vals) Y_vals[j][o] = V[best][head[best]];
            head[best]++;
        }
    }

done:
    if (X) for (int k = 0; k < p; ++k) free(X[k]);
    if (V) for (int k = 0; k < p; ++k) free(V[k]);
    free(X); free(V); free(T); free(S); free(cut); free(head);
    return rc;
}

/*
 * GVR(X, n, p): PAPER.md:988-1016 (Algorithm GVR), in its order:
 *   1 SampleSelection  s·p − 1 keys drawn uniformly at random from the (unsorted)
 *                      blocks X_k — the GER draws (R28) with positions in the
 *                      unsorted X_k, composites (key, k, position) (R29); T = sort
 *   2 SplitterSelect   S_i = T[i·s − 1], 1 ≤ i ≤ p−1
 *   3 Split            each key's destination j = #{i : S_i <_c (x, k, q)} ("binary
 *                      search of X_k into S"), then a count-sort of X_k by destination
 *                      (stable) gives the unordered X_{k,j}; processor k sends X_{k,j}
 *   4 LocalSorting     Y_j = X_{0,j} ‖ … ‖ X_{p−1,j} sorted by SR-b (stable), so equal
 *                      keys keep (source rank, position) order (R16)
 */
static int gvr_u64(int p, size_t s, uint64_t seed, int b,
                   const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
                   uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
                   uint64_t* splitters, uint64_t* counts) {
    if (p < 1 || s < 1 || (b != 8 && b != 16)) return -1;
    const size_t M = s * (size_t)p - 1;
    composite_t* T = (composite_t*)malloc((M ? M : 1) * sizeof(composite_t));
    composite_t* S = (composite_t*)malloc((size_t)p * sizeof(composite_t));
    if (!T || !S) { free(T); free(S); return -1; }
    size_t n = 0;
    for (int k = 0; k < p; ++k) n += N[k];

    /* Step 1: sample of the unsorted blocks (R28, R29), sorted as composites. */
    for (size_t i = 0; i < M; ++i) {
        composite_t c = { UINT64_MAX, 0, POS_INF };
        if (n) {
            const uint64_t q = (uint64_t)(((unsigned __int128)splitmix64_at(seed, i) * n) >> 64);
            uint64_t off = 0;
            for (int k = 0; k < p; ++k) {
                if (q < off + N[k]) { c.key = keys[k][q - off]; c.rank = (uint64_t)k; c.pos = q - off; break; }
                off += N[k];
            }
        }
        T[i] = c;
    }
    qsort(T, M, sizeof(composite_t), comp_qsort);

    /* Step 2: splitters. */
    for (int i = 1; i < p; ++i) {
        S[i] = T[(size_t)i * s - 1];
        if (splitters) {
            splitters[3 * (i - 1) + 0] = S[i].key;
            splitters[3 * (i - 1) + 1] = S[i].rank;
            splitters[3 * (i - 1) + 2] = S[i].pos;
        }
    }

    /* Steps 3-4: destinations, X_{k,j} in source order, Y_j = concatenation sorted. */
    int rc = 0;
    for (int j = 0; j < p; ++j) Ylen[j] = 0;
    for (int k = 0; k < p; ++k) {
        for (int j = 0; j < p; ++j) if (counts) counts[(size_t)k * p + j] = 0;
        for (size_t q = 0; q < N[k]; ++q) {
            composite_t e = { keys[k][q], (uint64_t)k, q };
            int j = 0;
            for (int i = 1; i < p; ++i) if (comp_cmp(&S[i], &e) < 0) j = i;  /* S_i <_c e */
            if (counts) counts[(size_t)k * p + j]++;
            if (Ylen[j] < Ycap) {
                Y_keys[j][Ylen[j]] = keys[k][q];
                if (vals) Y_vals[j][Ylen[j]] = vals[k][q];
            } else rc = -2;
            Ylen[j]++;
        }
    }
    for (int j = 0; j < p && rc == 0; ++j) {
        if (vals) { if (or_sr_pairs_u64_u32(Y_keys[j], Y_vals[j], Ylen[j], b, -1)) rc = -1; }
        else if (or_sr_u64(Y_keys[j], Ylen[j], b, -1)) rc = -1;
    }
    free(T); free(S);
    return rc;
}

int or_gvr_u64(int p, size_t s, uint64_t seed, int b,
               const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
               uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts) {
    return gvr_u64(p, s, seed, b, keys, vals, N, Y_keys, Y_vals, Ycap, Ylen, splitters, counts);
}

int or_gsd_u64(int p, int r, int b,
               const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
               uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts) {
    if (p < 1 || r < 1) return -1;
    return sample_sort_u64(p, 0, (size_t)r * (size_t)p, 0, b, keys, vals, N, Y_keys, Y_vals, Ycap, Ylen,
                           splitters, counts);
}

int or_ger_u64(int p, size_t s, uint64_t seed, int b,
               const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
               uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts) {
    return sample_sort_u64(p, 1, s, seed, b, keys, vals, N, Y_keys, Y_vals, Ycap, Ylen, splitters, counts);
}

/* u32 keys: the same algorithm on zero-extended keys (b-bit digits of a u32 key
 * and of its zero extension agree; the extra high rounds see one digit). */
static int sample_sort_u32(int p, int mode, size_t s, uint64_t seed, int b,
                           const uint32_t* const* keys, const size_t* N,
                           uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
                           uint64_t* splitters, uint64_t* counts) {
    if (p < 1) return -1;
    int rc = 0;
    uint64_t** K = (uint64_t**)calloc((size_t)p, sizeof(uint64_t*));
    uint64_t** Y = (uint64_t**)calloc((size_t)p, sizeof(uint64_t*));
    if (!K || !Y) { free(K); free(Y); return -1; }
    for (int k = 0; k < p && !rc; ++k) {
        K[k] = (uint64_t*)malloc((N[k] ? N[k] : 1) * sizeof(uint64_t));
        Y[k] = (uint64_t*)malloc((Ycap ? Ycap : 1) * sizeof(uint64_t));
        if (!K[k] || !Y[k]) rc = -1;
        else for (size_t i = 0; i < N[k]; ++i) K[k][i] = keys[k][i];
    }
    if (!rc) rc = mode == 2 ? gvr_u64(p, s, seed, b, (const uint64_t* const*)K, NULL, N, Y, NULL, Ycap, Ylen,
                                      splitters, counts)
                            : sample_sort_u64(p, mode, s, seed, b, (const uint64_t* const*)K, NULL, N, Y, NULL, Ycap,
                                              Ylen, splitters, counts);
    if (rc == 0)
        for (int j = 0; j < p; ++j)
            for (size_t i = 0; i < Ylen[j]; ++i) Y_keys[j][i] = (uint32_t)Y[j][i];
    for (int k = 0; k < p; ++k) { free(K[k]); free(Y[k]); }
    free(K); free(Y);
    return rc;
}

int or_gsd_u32(int p, int r, int b,
               const uint32_t* const* keys, const size_t* N,
               uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts) {
    if (p < 1 || r < 1) return -1;
    return sample_sort_u32(p, 0, (size_t)r * (size_t)p, 0, b, keys, N, Y_keys, Ycap, Ylen, splitters, counts);
}

int or_ger_u32(int p, size_t s, uint64_t seed, int b,
               const uint32_t* const* keys, const size_t* N,
               uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts) {
    return sample_sort_u32(p, 1, s, seed, b, keys, N, Y_keys, Ycap, Ylen, splitters, counts);
}

int or_gvr_u32(int p, size_t s, uint64_t seed, int b,
               const uint32_t* const* keys, const size_t* N,
               uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts) {
    return sample_sort_u32(p, 2, s, seed, b, keys, N, Y_keys, Ycap, Ylen, splitters, counts);
}
