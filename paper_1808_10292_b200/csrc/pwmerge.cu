// GSD step 5 as ONE pass: a stable p-way merge of p sorted runs (PAPER.md:800-803,
// "Subsequences X_{k,j} ... are merged into Y_j using p-way merging"), reading the
// runs wherever they are (the peers' blocks over NVLink in the pull merge) and
// writing Y_j once — against ⌈log2 p⌉ read+write passes of the 2-way tree.
//
// The output is cut into chunks by a regular sample of the runs, the same device
// the paper uses one level up (GSD's own splitters):
//   1 k_pw_sample  every m-th element of run k (the last of each m-block) becomes
//                  a sample, tagged (k, t);
//   2 the samples (p sorted lists, laid out run by run) are sorted stably by key
//                  (radix sort: composite order — key, then run) into Sm, and
//                  k_pw_pos records where each run's samples landed;
//   3 k_pw_bounds  chunk boundary i is the composite b_i = Sm[i·c − 1]; for every
//                  run k, cnt[i][k] = #elements of run k that are ≤ b_i.  The
//                  samples bracket it: if q run-k samples precede Sm position i·c,
//                  cnt ∈ [q·m, min((q+1)·m − 1, len_k)], found by a binary search of
//                  ≤ m elements (a handful of remote reads);
//   4 k_pw_merge   one CTA per chunk: its p pieces [cnt[i−1][k], cnt[i][k]) are
//                  staged in shared memory, merged there by a ⌈log2 p⌉-level tree
//                  of merge-path merges (left = lower runs: ties stay stable), and
//                  stored coalesced at Σ_k cnt[i−1][k].  Per level every merged
//                  pair gets its own IT-output thread slots: warps 0-6 merge the
//                  regular slots forwards (one search, IT unrolled unchecked
//                  steps), warp 7 the last kPwSpecial slots of every pair
//                  backwards from their end co-rank (where a run runs out).
// A chunk holds at most c·m + p·(m − 1) elements (each run contributes its
// bracketed samples plus less than one block), so the shared-memory tile is fixed.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "merge.h"

namespace rs {
namespace {

#ifndef RS_PW_M
#define RS_PW_M 128
#endif
#ifndef RS_PW_C
#define RS_PW_C 0  // 0: 32 samples per chunk for 4-byte keys without values, else 16
#endif
#ifndef RS_PW_IT
// outputs per thread slot; odd, so neighbouring threads' merge-path positions fall
// in different banks.  k_pw_merge at 2^28 outputs, p = 8, ncu-serialised us
// (scripts/gpu_pw_ab.sh): round-1 tree (IT 19, slots straddling pairs) 1169;
// per-pair slots + unrolled unchecked steps + backwards special slots, IT/special
// 19/2 1174, 19/3 1121, 21/3 1106, 23/3 1097, 23/4 1100, 25/3 1106, 27/2 1174
#define RS_PW_IT 23
#endif
constexpr int kPwM = RS_PW_M;  // sample stride m
constexpr int kPwCMax = 32;     // samples per chunk c (PwRuns::c) at most
constexpr int kPwMaxP = 32;   // runs handled by the single-pass merge (shared-memory tile)
// threads x samples per chunk, k_pw_merge at 2^28 outputs, p = 8 (scripts/gpu_pw_ab.sh, us):
// 256 x 32 1101 (kept), 256 x 16 1375, 128 x 16 1206, 128 x 32 1400, 512 x 32 1500, 512 x 16 2343
#ifndef RS_PW_T
#define RS_PW_T 256
#endif
constexpr int kPwT = RS_PW_T;  // threads per merge CTA (warps 0..W-2 regular slots, the last warp the special ones)
constexpr int kPwLevels = 5;  // ⌈log2 kPwMaxP⌉
#ifndef RS_PW_SPECIAL
#define RS_PW_SPECIAL 3
#endif
constexpr int kPwSpecial = RS_PW_SPECIAL;  // slots per merged pair merged backwards from its end

struct PwRuns {
    const void* k[kPwMaxP];
    const uint32_t* v[kPwMaxP];
    uint64_t len[kPwMaxP];
    uint64_t soff[kPwMaxP + 1];  // sample offsets (run k's samples at [soff[k], soff[k+1]))
    int p;
    int c;  // samples per chunk
};

__device__ __forceinline__ int run_of(const PwRuns& R, uint64_t j) {  // soff[k] <= j < soff[k+1]
    int lo = 0, hi = R.p - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (R.soff[mid] <= j) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <typename K>
__global__ void k_pw_sample(PwRuns R, K* __restrict__ sk, uint32_t* __restrict__ sv) {
    const uint64_t M = R.soff[R.p];
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (uint64_t)gridDim.x * blockDim.x) {
        const int k = run_of(R, j);
        const uint64_t t = j - R.soff[k];
        sk[j] = static_cast<const K*>(R.k[k])[(t + 1) * kPwM - 1];
        sv[j] = ((uint32_t)k << 24) | (uint32_t)t;
    }
}

// pos[soff[k] + t] = merged index of run k's sample t
__global__ void k_pw_pos(PwRuns R, const uint32_t* __restrict__ smv, uint64_t M, uint32_t* __restrict__ pos) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = smv[j];
        pos[R.soff[v >> 24] + (v & 0xFFFFFFu)] = (uint32_t)j;
    }
}

// cnt[i * p + k] for boundaries i = 0 .. nch (row 0: nothing, row nch: the whole run)
template <typename K>
__global__ void k_pw_bounds(PwRuns R, const K* __restrict__ smk, const uint32_t* __restrict__ smv,
                            const uint32_t* __restrict__ pos, uint64_t nch, uint32_t* __restrict__ cnt) {
    const int p = R.p;
    const uint64_t total = (nch + 1) * (uint64_t)p;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = x / p;
        const int k = (int)(x % p);
        if (i == 0 || i == nch) {
            cnt[x] = i == 0 ? 0u : (uint32_t)R.len[k];
            continue;
        }
        const uint64_t bj = i * R.c - 1;  // boundary b_i = Sm[bj]
        const K bv = smk[bj];
        const int bk = (int)(smv[bj] >> 24);
        const uint64_t bpos = ((uint64_t)(smv[bj] & 0xFFFFFFu) + 1) * kPwM - 1;
        // q = run-k samples with merged index < i·c
        const uint32_t* pk = pos + R.soff[k];
        uint64_t lo = 0, hi = R.soff[k + 1] - R.soff[k];
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (pk[mid] < i * R.c) lo = mid + 1;
            else hi = mid;
        }
        const uint64_t q = lo;
        const K* rk = static_cast<const K*>(R.k[k]);
        uint64_t a = q * kPwM, b = min((q + 1) * kPwM - 1, R.len[k]);  // answer in [a, b]
        while (a < b) {  // first position whose element is > b_i (composite)
            const uint64_t mid = (a + b) >> 1;
            const K e = rk[mid];
            const bool le = e < bv || (e == bv && (k < bk || (k == bk && mid <= bpos)));
            if (le) a = mid + 1;
            else b = mid;
        }
        cnt[i * p + k] = (uint32_t)a;
    }
}

template <typename K>
__device__ __forceinline__ K lds(uint32_t addr) {  // a shared-memory load from a shared address
    if (sizeof(K) == 4) {
        uint32_t x;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(addr) : "memory");
        return (K)x;
    } else {
        unsigned long long x;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x) : "r"(addr) : "memory");
        return (K)x;
    }
}

template <typename K, bool V>
__global__ void __launch_bounds__(kPwT) k_pw_merge(PwRuns R, const uint32_t* __restrict__ cnt, int cap,
                                                   K* __restrict__ out, uint32_t* __restrict__ vout) {
    extern __shared__ __align__(16) unsigned char pw_smem[];
    K* X = reinterpret_cast<K*>(pw_smem);
    K* Y = X + cap;
    uint32_t* XV = reinterpret_cast<uint32_t*>(Y + cap);
    uint32_t* YV = XV + (V ? cap : 0);
    __shared__ uint32_t s_seg[kPwMaxP + 1];  // piece offsets in the chunk
    __shared__ uint32_t s_reg[kPwLevels][kPwMaxP / 2 + 1];  // prefix of regular slots per pair
    __shared__ uint32_t s_spc[kPwLevels][kPwMaxP / 2 + 1];  // prefix of special slots per pair
    __shared__ uint64_t s_o;
    const int p = R.p, tid = threadIdx.x;
    const uint64_t i = blockIdx.x;
    // piece table: in EVERY warp, lanes k < p load their bounds (L2 hits) and one
    // warp scan gives the pieces' offsets in the chunk, so each warp starts staging
    // its pieces at once (no CTA barrier behind warp 0's global loads: that wait was
    // 18 % of the kernel's stall samples); warp 0 also writes the tables the merge
    // levels read after the staging barrier
    const int warp = tid >> 5, lane = tid & 31;
    uint32_t c0 = 0, len = 0;
    if (lane < p) {
        c0 = cnt[i * p + lane];
        len = cnt[(i + 1) * p + lane] - c0;
    }
    uint32_t incl = len;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    const uint32_t excl = incl - len, total = __shfl_sync(0xffffffffu, incl, 31);
    const int E = (int)total;
    RS_DCHECK(E < cap);  // (the merge reads one slot past the last element)
    if (warp == 0) {
        uint64_t o = c0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) o += __shfl_xor_sync(0xffffffffu, o, d);
        if (lane < p) s_seg[lane] = excl;
        if (lane == 0) {
            s_seg[p] = total;
            s_o = o;
        }
        // thread-slot tables of every merge level: pair q of level L (stride 2^L)
        // has ⌈len/IT⌉ slots; its last kPwSpecial are "special" (near the runs'
        // ends, merged backwards) and numbered after all regular ones, so they
        // share one or two warps and their code path diverges only there
        for (int L = 0, st = 1; st < p; ++L, st *= 2) {
            const int npair = ((p + st - 1) / st + 1) / 2;
            const int ia = min(2 * lane * st, p), ib = min((2 * lane + 2) * st, p);
            const uint32_t qa = __shfl_sync(0xffffffffu, excl, ia & 31), qb = __shfl_sync(0xffffffffu, excl, ib & 31);
            const uint32_t va = ia >= 32 ? total : qa, vb = ib >= 32 ? total : qb;
            const uint32_t ns = lane < npair ? (vb - va + RS_PW_IT - 1) / RS_PW_IT : 0u;
            uint32_t sp = min(ns, (uint32_t)kPwSpecial), rg = ns - sp;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, rg, d), z = __shfl_up_sync(0xffffffffu, sp, d);
                if (lane >= d) {
                    rg += y;
                    sp += z;
                }
            }
            if (lane < npair) {
                s_reg[L][lane + 1] = rg;
                s_spc[L][lane + 1] = sp;
            }
            if (lane == 0) s_reg[L][0] = s_spc[L][0] = 0;
        }
    }
    // stage the pieces: with p >= 8 warps, warp w copies pieces w, w + 8, ...; with
    // fewer pieces than warps, piece k is copied by warps k, k + p, ... together
    // (p = 2: four warps per piece, not one warp walking 8 latency-bound batches);
    // each lane keeps SB independent (remote) loads in flight before writing shared memory
    {
// (k_pw_merge at c4 sizes, us: one warp per piece 3712 / 1744 / 1101 at p = 2 / 4 / 8;
// grouped 2262 / 1552 / 1102; batches of SB = 12: 3025 / 1943 / 1215, SB = 16: 2351 / 1631 / 1087;
// 8 for grouped pieces and 16 for one warp per piece in one kernel: 2469 / 1655 / 1088, pairs
// at 2^30: 3972 / 2782 / 1804 vs 3403 / 2767 / 1812 — the deeper path's registers cost every p)
#ifndef RS_PW_SB
#define RS_PW_SB 8
#endif
        constexpr int SB = RS_PW_SB, NW = kPwT / 32;
#ifdef RS_PW_STAGE_ONE_WARP
        const bool grouped = false;  // (A/B: the round-2 one-warp-per-piece staging)
#else
        const bool grouped = p < NW;
#endif
        const int k0 = grouped ? warp % p : warp;
        const int gi = grouped ? warp / p : 0, gn = grouped ? (NW - k0 + p - 1) / p : 1;
        for (int k = k0; k < p; k += grouped ? p : NW) {
            const int s0 = (int)__shfl_sync(0xffffffffu, excl, k), ln = (int)__shfl_sync(0xffffffffu, len, k);
            const uint32_t off = __shfl_sync(0xffffffffu, c0, k);
            const K* src = static_cast<const K*>(R.k[k]) + off;
            const uint32_t* vs = V ? R.v[k] + off : nullptr;
            for (int b = gi * 32 * SB; b < ln; b += gn * 32 * SB) {
                K r[SB];
                uint32_t rv[V ? SB : 1];
#pragma unroll
                for (int j = 0; j < SB; ++j) {
                    const int e = b + j * 32 + lane;
                    if (e < ln) {
                        r[j] = src[e];
                        if (V) rv[V ? j : 0] = vs[e];
                    }
                }
#pragma unroll
                for (int j = 0; j < SB; ++j) {
                    const int e = b + j * 32 + lane;
                    if (e < ln) {
                        X[s0 + e] = r[j];
                        if (V) XV[s0 + e] = rv[V ? j : 0];
                    }
                }
            }
        }
    }
    __syncthreads();
    // merge tree in shared memory: segments [seg[j], seg[j+1]) -> pairs -> ...
    // Each level gives every merged pair its own ⌈len/IT⌉ thread slots, so a
    // thread's IT outputs never straddle two pairs: one merge-path search, then
    // (unless a run ends inside the slot) IT unrolled steps without bound checks
    // on shared addresses — compare, select, store, reload the consumed head.
    int nseg = p, stride = 1;  // current segment j covers pieces [j·stride, min((j+1)·stride, p))
    K* src = X;
    K* dst = Y;
    uint32_t* vsrc = XV;
    uint32_t* vdst = YV;
    constexpr int IT = RS_PW_IT;  // outputs per thread slot
    constexpr uint32_t KB = (uint32_t)sizeof(K);
    for (int L = 0; nseg > 1; ++L) {
        const int npair = (nseg + 1) >> 1;
        const uint32_t sbase = smem_addr(src);
        const int nreg = (int)s_reg[L][npair], nslot = nreg + (int)s_spc[L][npair];
        // warps 0..6 take the regular slots, warp 7 the special ones
        const bool special = tid >= kPwT - 32;
        const int nmine = special ? nslot - nreg : nreg;
        for (int u = special ? tid - (kPwT - 32) : tid; u < nmine; u += special ? 32 : kPwT - 32) {
            const uint32_t* tab = special ? s_spc[L] : s_reg[L];
            int q = 0;  // the pair owning slot u
            while (q + 1 < npair && u >= (int)tab[q + 1]) ++q;
            const int a0 = (int)s_seg[2 * q * stride];
            const int a1 = (int)s_seg[min((2 * q + 1) * stride, p)];
            const int b1 = (int)s_seg[min((2 * q + 2) * stride, p)];
            const int slot = (u - (int)tab[q]) + (special ? (int)(s_reg[L][q + 1] - s_reg[L][q]) : 0);
            const int o0 = a0 + slot * IT;
            const int oend = min(o0 + IT, b1);
            const int la = a1 - a0, lb = b1 - a1;
            if (la == 0 || lb == 0) {  // an unpaired (or empty-sided) segment moves as it is
                for (int o = o0; o < oend; ++o) {
                    dst[o] = src[o];
                    if (V) vdst[o] = vsrc[o];
                }
                continue;
            }
            // merge path: the co-rank (pa, pb) of output position d of the pair
            auto corank = [&](int d, int& pa, int& pb) {
                int lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
                const uint32_t sa = sbase + (uint32_t)a0 * KB, sb = sbase + (uint32_t)(a1 + d - 1) * KB;
                while (lo < hi) {  // A[mid] at sa + mid·|K| against B[d − 1 − mid] at sb − mid·|K|
                    const int mid = (lo + hi) >> 1;
                    const uint32_t off = (uint32_t)mid * KB;
                    if (lds<K>(sa + off) <= lds<K>(sb - off)) lo = mid + 1;
                    else hi = mid;
                }
                pa = a0 + lo;
                pb = a1 + d - lo;
            };
            const int r = oend - o0;
            int pa, pb;
            if (special) {
                // backwards from the slot's end co-rank (the pair's last slot: the runs'
                // ends, an empty search): unchecked while r steps cannot pass either
                // run's start; ties leave B first
                corank(oend - a0, pa, pb);
                if (pa - a0 > r && pb - a1 > r) {
                    uint32_t sa = sbase + (uint32_t)(pa - 1) * KB, sb = sbase + (uint32_t)(pb - 1) * KB;
                    K ha = lds<K>(sa), hb = lds<K>(sb);
                    for (int o = oend - 1; o >= o0; --o) {
                        const bool takeB = hb >= ha;
                        const uint32_t from = takeB ? sb : sa;
                        dst[o] = takeB ? hb : ha;
                        if (V) vdst[o] = vsrc[(from - sbase) / KB];
                        const uint32_t nxt = from - KB;
                        const K nv = lds<K>(nxt);
                        sb = takeB ? nxt : sb;
                        sa = takeB ? sa : nxt;
                        hb = takeB ? nv : hb;
                        ha = takeB ? ha : nv;
                    }
                    continue;
                }
            }
            corank(o0 - a0, pa, pb);
            // absolute positions; a head past its run's end is read (the tile has one
            // slot of slack past E) but never selected
            K ha = src[pa], hb = src[pb];
            if (r == IT && a1 - pa >= IT && b1 - pb >= IT) {  // no run ends inside the slot
                uint32_t sa = sbase + (uint32_t)pa * KB, sb = sbase + (uint32_t)pb * KB;
#pragma unroll
                for (int k = 0; k < IT; ++k) {
                    const bool takeA = ha <= hb;
                    const uint32_t from = takeA ? sa : sb;
                    dst[o0 + k] = takeA ? ha : hb;
                    if (V) vdst[o0 + k] = vsrc[(from - sbase) / KB];
                    const uint32_t nxt = from + KB;
                    const K nv = lds<K>(nxt);
                    sa = takeA ? nxt : sa;
                    sb = takeA ? sb : nxt;
                    ha = takeA ? nv : ha;
                    hb = takeA ? hb : nv;
                }
            } else if (pa == a1 || pb == b1) {  // one run is spent: the other one's tail
                const int sh = pa == a1 ? 0 : lb;  // B[o − a1 + a0 − la] = src[o]; A: src[o − lb]
                for (int o = o0; o < oend; ++o) {
                    dst[o] = src[o - sh];
                    if (V) vdst[o] = vsrc[o - sh];
                }
            } else {
                for (int o = o0; o < oend; ++o) {  // a run ends inside the slot: bound-checked
                    const bool takeA = pb >= b1 || (pa < a1 && ha <= hb);
                    const int from = takeA ? pa : pb;
                    dst[o] = takeA ? ha : hb;
                    if (V) vdst[o] = vsrc[from];
                    const K nv = src[from + 1];
                    pa += takeA;
                    pb += !takeA;
                    ha = takeA ? nv : ha;
                    hb = takeA ? hb : nv;
                }
            }
        }
        __syncthreads();
        nseg = (nseg + 1) / 2;
        stride *= 2;
        K* t = src;
        src = dst;
        dst = t;
        uint32_t* tv = vsrc;
        vsrc = vdst;
        vdst = tv;
    }
    // coalesced store of the merged chunk
    const uint64_t o = s_o;
    for (int e = tid; e < E; e += kPwT) {
        out[o + e] = src[e];
        if (V) vout[o + e] = vsrc[e];
    }
}

constexpr int pw_cap(int p, int c) { return c * kPwM + p * kPwM; }
constexpr int pw_cap_padded(int p, int c) { return pw_cap(p, c) + 1; }  // one slot of slack
int pw_c(int key_bytes, bool hv) { return RS_PW_C ? RS_PW_C : (key_bytes == 4 && !hv ? 32 : 16); }

struct PwLayout {
    void *sk, *mk;            // samples, sorted samples (M keys each)
    uint32_t *sv, *mv;        // their tags
    uint32_t* pos;            // M
    uint32_t* cnt;            // (nch + 1) * p
    void* sort_ws;            // local_sort scratch for the sample
    size_t sort_ws_bytes;
    size_t bytes;
};

PwLayout pw_layout(void* ws, int key_bytes, uint64_t M, uint64_t nch, int p) {
    PwLayout L{};
    Carver c(ws);
    const size_t M1 = std::max<uint64_t>(M, 1);
    L.sk = c.take(M1 * key_bytes);
    L.mk = c.take(M1 * key_bytes);
    L.sv = static_cast<uint32_t*>(c.take(M1 * 4));
    L.mv = static_cast<uint32_t*>(c.take(M1 * 4));
    L.pos = static_cast<uint32_t*>(c.take(M1 * 4));
    L.cnt = static_cast<uint32_t*>(c.take((nch + 1) * (size_t)p * 4));
    L.sort_ws_bytes = local_ws_bytes(key_bytes, true, M1, 8);
    L.sort_ws = c.take(L.sort_ws_bytes);
    L.bytes = c.used();
    return L;
}

template <typename K, bool V>
rs_status_t pway(const PwRuns& R, uint64_t M, void* scratch, K* out, uint32_t* vout, cudaStream_t st) {
    const int p = R.p;
    const uint64_t nch = std::max<uint64_t>(1, (M + R.c - 1) / R.c);
    const PwLayout L = pw_layout(scratch, sizeof(K), M, nch, p);
    const unsigned g = (unsigned)std::min<uint64_t>((M + 255) / 256 + 1, 8192);
    {
        LaunchScope ls("pw_sample", st);
        if (M) k_pw_sample<K><<<g, 256, 0, st>>>(R, static_cast<K*>(L.sk), L.sv);
    }
    if (M) {
        // the samples, laid out run by run, sorted stably by key: ties stay in (run, t)
        // order, i.e. the composite order (a radix sort beats a merge tree at this size)
        rs_status_t s = local_sort(sizeof(K), L.sk, L.sv, M, 8, (int)sizeof(K) * 8, L.mk, L.mv, L.sort_ws,
                                   L.sort_ws_bytes, st);
        if (s != RS_OK) return s;
        LaunchScope ls("pw_pos", st);
        k_pw_pos<<<g, 256, 0, st>>>(R, L.mv, M, L.pos);
    }
    {
        LaunchScope ls("pw_bounds", st);
        const unsigned gb = (unsigned)std::min<uint64_t>(((nch + 1) * p + 255) / 256, 65535);
        k_pw_bounds<K><<<gb, 256, 0, st>>>(R, static_cast<const K*>(L.mk), L.mv, L.pos, nch, L.cnt);
    }
    const int cap = pw_cap_padded(p, R.c);
    const size_t smem = (size_t)cap * (2 * sizeof(K) + (V ? 8 : 0));
    {
        rs_status_t s = kernel_setup(reinterpret_cast<const void*>(k_pw_merge<K, V>), kPwT,
                                     (size_t)pw_cap_padded(kPwMaxP, kPwCMax) * (2 * sizeof(K) + (V ? 8 : 0)), nullptr);
        if (s != RS_OK) return s;
    }
    {
        LaunchScope ls("pw_merge", st);
        k_pw_merge<K, V><<<(unsigned)nch, kPwT, smem, st>>>(R, L.cnt, cap, out, vout);
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

}  // namespace

bool pway_applicable(int p, const std::vector<uint64_t>& len) {
    if (p < 2 || p > kPwMaxP) return false;
    for (uint64_t l : len)
        if (l >= (1ull << 31) || l / kPwM >= (1ull << 24)) return false;
    return true;
}

size_t pway_scratch_bytes(int key_bytes, uint64_t total, int p) {
    const uint64_t M = total / kPwM + (uint64_t)p;
    return pw_layout(nullptr, key_bytes, M, M + 2, p).bytes;  // nch <= M / c + 1
}

rs_status_t merge_pway(int key_bytes, const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                       const std::vector<uint64_t>& len, void* scratch, size_t scratch_bytes, void* out,
                       uint32_t* vout, cudaStream_t st) {
    const int p = (int)len.size();
    if (!pway_applicable(p, len)) return fail(RS_EINVAL, "p-way merge: p out of range or a run too long");
    PwRuns R{};
    R.p = p;
    R.c = pw_c(key_bytes, vout != nullptr);
    R.soff[0] = 0;
    uint64_t total = 0;
    for (int k = 0; k < p; ++k) {
        R.k[k] = rk[k];
        R.v[k] = rv.empty() ? nullptr : rv[k];
        R.len[k] = len[k];
        R.soff[k + 1] = R.soff[k] + len[k] / kPwM;
        total += len[k];
    }
    if (total == 0) return RS_OK;
    const uint64_t M = R.soff[p];
    if (scratch_bytes < pway_scratch_bytes(key_bytes, total, p)) return fail(RS_EINVAL, "p-way merge scratch too small");
    const bool V = vout != nullptr;
    if (key_bytes == 4)
        return V ? pway<uint32_t, true>(R, M, scratch, static_cast<uint32_t*>(out), vout, st)
                 : pway<uint32_t, false>(R, M, scratch, static_cast<uint32_t*>(out), nullptr, st);
    return V ? pway<uint64_t, true>(R, M, scratch, static_cast<uint64_t*>(out), vout, st)
             : pway<uint64_t, false>(R, M, scratch, static_cast<uint64_t*>(out), nullptr, st);
}

}  // namespace rs
