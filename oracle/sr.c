/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * SR-b: serial LSD radix sort as a sequence of count-sort rounds.
 * PAPER.md:653-671 (§3.2, "Serial radix-r radix-sort: SR4"): "The radix used is
 * r=256 i.e. it is a four-round count-sort.  In each round of count-sort the
 * input is read twice, first during the initial counting process and last when
 * the output is to be generated, and the output is generated once."
 * PR2's radix r = 2^16 gives the b = 16 variant.
 *
 * Readings: R1 digit t = (x >> t·b) & (r−1), t = 0 first (LSD);
 * R2 keys unsigned; R3 equal digits keep input order (count-sort is stable);
 * R4 b ∈ {8, 16} only.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

/* One count-sort round over digit `t`:
 *   1. count digit occurrences (first read of the input)
 *   2. exclusive prefix of the counts = first output slot of each digit
 *   3. read the input again in order, write each key to its digit's next slot */
#define DEFINE_ROUND(NAME, KT)                                                       \
static void NAME(const KT* in, KT* out, const uint32_t* vin, uint32_t* vout,          \
                 size_t n, int t, int b, size_t* cnt) {                               \
    const size_t R = (size_t)1 << b;                                                  \
    const int shift = t * b;                                                          \
    memset(cnt, 0, R * sizeof(size_t));                                               \
    for (size_t i = 0; i < n; ++i) cnt[(in[i] >> shift) & (R - 1)]++;                 \
    size_t run = 0;                                                                   \
    for (size_t d = 0; d < R; ++d) { size_t c = cnt[d]; cnt[d] = run; run += c; }      \
    for (size_t i = 0; i < n; ++i) {                                                  \
        size_t d = (in[i] >> shift) & (R - 1);                                        \
        size_t o = cnt[d]++;                                                          \
        out[o] = in[i];                                                               \
        if (vin) vout[o] = vin[i];                                                    \
    }                                                                                 \
}
DEFINE_ROUND(round_u32, uint32_t)
DEFINE_ROUND(round_u64, uint64_t)

/* Whole sort: rounds t = 0 .. P-1 with a ping-pong buffer; the last round's
 * output is copied back so the result is in a[] (and v[]). */
#define DEFINE_SR(NAME, KT, KEYBITS, ROUND)                                           \
static int NAME(KT* a, uint32_t* v, size_t n, int b, int rounds) {                    \
    if (b != 8 && b != 16) return -1;                                                 \
    if (n == 0) return 0;                                                             \
    if (!a) return -1;                                                                \
    const int P = (KEYBITS) / b;                                                      \
    if (rounds < 0 || rounds > P) rounds = P;                                         \
    size_t* cnt = (size_t*)malloc(((size_t)1 << b) * sizeof(size_t));                \
    KT* tmp = (KT*)malloc(n * sizeof(KT));                                            \
    uint32_t* vtmp = v ? (uint32_t*)malloc(n * sizeof(uint32_t)) : NULL;              \
    if (!cnt || !tmp || (v && !vtmp)) { free(cnt); free(tmp); free(vtmp); return -1; }\
    KT* src = a; KT* dst = tmp; uint32_t* vsrc = v; uint32_t* vdst = vtmp;            \
    for (int t = 0; t < rounds; ++t) {                                                \
        ROUND(src, dst, vsrc, vdst, n, t, b, cnt);                                    \
        KT* s = src; src = dst; dst = s;                                              \
        uint32_t* vs = vsrc; vsrc = vdst; vdst = vs;                                  \
    }                                                                                 \
    if (src != a) {                                                                   \
        memcpy(a, src, n * sizeof(KT));                                               \
        if (v) memcpy(v, vsrc, n * sizeof(uint32_t));                                 \
    }                                                                                 \
    free(cnt); free(tmp); free(vtmp);                                                 \
    return 0;                                                                         \
}
DEFINE_SR(sr_u32, uint32_t, 32, round_u32)
DEFINE_SR(sr_u64, uint64_t, 64, round_u64)

int or_sr_u32(uint32_t* a, size_t n, int b, int rounds) { return sr_u32(a, NULL, n, b, rounds); }
int or_sr_u64(uint64_t* a, size_t n, int b, int rounds) { return sr_u64(a, NULL, n, b, rounds); }
int or_sr_pairs_u64_u32(uint64_t* a, uint32_t* v, size_t n, int b, int rounds) {
    if (n && !v) return -1;
    return sr_u64(a, v, n, b, rounds);
}

/* Counting step of every round at once (the "initial counting
 * process"), i.e. the digit histogram of each round. */
int or_hist_u32(const uint32_t* a, size_t n, int b, uint64_t* out) {
    if (b != 8 && b != 16) return -1;
    const size_t R = (size_t)1 << b; const int P = 32 / b;
    memset(out, 0, (size_t)P * R * sizeof(uint64_t));
    for (int t = 0; t < P; ++t)
        for (size_t i = 0; i < n; ++i) out[(size_t)t * R + ((a[i] >> (t * b)) & (R - 1))]++;
    return 0;
}

int or_hist_u64(const uint64_t* a, size_t n, int b, uint64_t* out) {
    if (b != 8 && b != 16) return -1;
    const size_t R = (size_t)1 << b; const int P = 64 / b;
    memset(out, 0, (size_t)P * R * sizeof(uint64_t));
    for (int t = 0; t < P; ++t)
        for (size_t i = 0; i < n; ++i) out[(size_t)t * R + ((a[i] >> (t * b)) & (R - 1))]++;
    return 0;
}
