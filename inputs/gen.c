/*
 * Seeded synthetic inputs shared by the oracle side and the CUDA side.
 *
 * This module holds NO arithmetic of the sorting method (no digits, counts,
 * prefixes, splitters, merges): it only produces the key/value arrays the
 * workloads of BASELINE.json describe.  Both the oracle (oracle/) and the GPU
 * path (paper_1808_10292_b200/) consume what it writes; neither imports the
 * other.
 *
 * Generator: SplitMix64 (Steele, Lea, Flood 2014), counter form:
 *     z_i = mix(seed + (i + 1) * 0x9E3779B97F4A7C15)
 *     mix(z): z ^= z >> 30; z *= 0xBF58476D1CE4E5B9;
 *             z ^= z >> 27; z *= 0x94D049BB133111EB; z ^= z >> 31
 * (constants as in SPEC.md:316).  z_i equals the i-th sequential output of the
 * stateful generator seeded with `seed`, so any shard [start, start+count) of a
 * global stream is generated independently.
 *
 * The paper never states its key distribution ("integers");
 * the distributions below are BASELINE.json configs[0..4].
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define SM64_GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t sm64_mix(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

static inline uint64_t sm64_at(uint64_t seed, uint64_t i) {
    return sm64_mix(seed + (i + 1) * SM64_GOLDEN);
}

uint64_t inp_splitmix64_at(uint64_t seed, uint64_t i) { return sm64_at(seed, i); }
uint64_t inp_splitmix64_mix(uint64_t z) { return sm64_mix(z); }

/* u32 distributions (configs[0..3]) */
enum {
    INP_U32_UNIFORM   = 0,  /* (u32)(z_i >> 32): uniform over [0, 2^32)         cfg 1,3,4 */
    INP_U32_MOD16     = 1,  /* (z_i >> 32) & 15: 16 distinct keys                cfg 3   */
    INP_U32_GAUSS     = 2,  /* rounded |N(2^31, (2^28)^2)|, clamped to u32       cfg 3   */
    INP_U32_SORTED    = 3,  /* stratified ascending draw                         cfg 3   */
    INP_U32_REVERSED  = 4,  /* the SORTED draw read backwards                    cfg 3   */
    INP_U32_EQUAL     = 5,  /* all keys = (u32)(z_0 >> 32)                       cfg 3   */
    INP_U32_HALF      = 6,  /* (u32)(z_i >> 33): uniform over [0, 2^31)          cfg 2   */
};

/* u64 distributions (configs[4]) */
enum {
    INP_U64_UNIFORM = 0,    /* z_i: uniform over [0, 2^64)                        cfg 5   */
    INP_U64_MOD1024 = 1,    /* z_i mod 1024: narrow range, exercises stability    cfg 5 variant */
};

/* Stratified ascending key for global index i of n_total:
 * lo_i = floor(i * 2^32 / n_total); key = lo_i + (z_i >> 32) mod (lo_{i+1} - lo_i).
 * key_i lies in [lo_i, lo_{i+1}), so the sequence is nondecreasing without
 * sorting anything (requires 1 <= n_total <= 2^32). */
static inline uint32_t sorted_key(uint64_t seed, uint64_t i, uint64_t n_total) {
    uint64_t lo = (uint64_t)(((unsigned __int128)i << 32) / n_total);
    uint64_t hi = (uint64_t)(((unsigned __int128)(i + 1) << 32) / n_total);
    uint64_t w = hi - lo;                   /* >= 1 when n_total <= 2^32 */
    return (uint32_t)(lo + ((sm64_at(seed, i) >> 32) % w));
}

static inline uint32_t gauss_key(uint64_t seed, uint64_t i) {
    const double two53 = 1.0 / 9007199254740992.0;  /* 2^-53 */
    double u1 = (double)((sm64_at(seed, 2 * i) >> 11) + 1) * two53;   /* (0, 1] */
    double u2 = (double)(sm64_at(seed, 2 * i + 1) >> 11) * two53;     /* [0, 1) */
    double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
    double x = 2147483648.0 + 268435456.0 * g;      /* mean 2^31, sigma 2^28 */
    long long r = llrint(x);
    if (r < 0) r = -r;
    if (r > 4294967295LL) r = 4294967295LL;
    return (uint32_t)r;
}

/* Fill out[0..count) with keys of global indices start .. start+count-1.
 * Returns 0 on success, -1 on a bad distribution or size. */
int inp_gen_u32(uint32_t* out, uint64_t start, uint64_t count, uint64_t seed,
                int dist, uint64_t n_total) {
    if (dist < 0 || dist > 6) return -1;
    if ((dist == INP_U32_SORTED || dist == INP_U32_REVERSED) &&
        (n_total == 0 || n_total > (1ULL << 32) || start + count > n_total)) return -1;
    const uint32_t eq = (uint32_t)(sm64_at(seed, 0) >> 32);
    #pragma omp parallel for schedule(static)
    for (long long k = 0; k < (long long)count; ++k) {
        uint64_t i = start + (uint64_t)k;
        uint32_t v;
        switch (dist) {
            case INP_U32_UNIFORM:  v = (uint32_t)(sm64_at(seed, i) >> 32); break;
            case INP_U32_MOD16:    v = (uint32_t)(sm64_at(seed, i) >> 32) & 15u; break;
            case INP_U32_GAUSS:    v = gauss_key(seed, i); break;
            case INP_U32_SORTED:   v = sorted_key(seed, i, n_total); break;
            case INP_U32_REVERSED: v = sorted_key(seed, n_total - 1 - i, n_total); break;
            case INP_U32_EQUAL:    v = eq; break;
            default:               v = (uint32_t)(sm64_at(seed, i) >> 33); break;
        }
        out[k] = v;
    }
    return 0;
}

int inp_gen_u64(uint64_t* out, uint64_t start, uint64_t count, uint64_t seed, int dist) {
    if (dist < 0 || dist > 1) return -1;
    #pragma omp parallel for schedule(static)
    for (long long k = 0; k < (long long)count; ++k) {
        uint64_t z = sm64_at(seed, start + (uint64_t)k);
        out[k] = dist == INP_U64_UNIFORM ? z : (z & 1023u);
    }
    return 0;
}

/* payload = original global index (configs[4]: "payload=original index") */
int inp_iota_u32(uint32_t* out, uint64_t start, uint64_t count) {
    #pragma omp parallel for schedule(static)
    for (long long k = 0; k < (long long)count; ++k) out[k] = (uint32_t)(start + (uint64_t)k);
    return 0;
}
