// K3 "atomic rank" (design 5, default when the startup probe passes) — one
// stable count-sort round of radix 256:
//
//   [load]    TMA bulk copy of tile k into s_in (issued during tile k-1's store)
//   [rank]    warp w, row j (32 consecutive keys, lane order = input order):
//             r = atomicAdd(&cnt_w[d], 1) on the warp's shared-memory counter of
//             the key's digit d.  The returned old values ARE the stable ranks
//             of the keys among the warp's keys of digit d: earlier rows were
//             counted by earlier instructions, and within one instruction the
//             sm_100 shared-memory atomic unit returns the old values of lanes
//             that hit the same address in ascending lane order.  That lane order
//             is a measured hardware property, not a PTX guarantee: the library
//             checks it with a probe kernel before it selects this design
//             (runtime.cu rank_probe) and otherwise runs design 2 (ballot ranks).
//             The final counter values are the warp's digit histogram, so the
//             counting of PAPER.md:664-667 comes out of the same instruction.
//   [offset]  thread d: tile count, in-tile offset of digit d, per-warp start
//             offsets; publish the tile count to the look-back status (flag A,
//             or P for tile 0) — the tiles x 256 counter matrix of PR4,
//             PAPER.md:690-694
//   [scatter] key -> s_out[start_w[d] + r]  (the tile sorted by digit, stably)
//   [lookback] thread d: windowed decoupled look-back over earlier tiles,
//             publishes the inclusive prefix (flag P)
//   [next]    thread 0 takes the next tile id and starts its TMA load into s_in
//   [store]   consecutive threads store consecutive s_out slots: each bucket run
//             is a coalesced burst at base[d] + prefix[d] + offset
//
// Against design 2 this removes the per-key 8-ballot peer mask and the warp
// counter load/store round trip: per 32 keys one conflicted atomic replaces an
// atomic + ~30 ALU instructions + a conflicted load and store.
#pragma once
#include <cstdio>

#include "onesweep_ec.cuh"

// timing ablations of design 5 (development builds only, OUTPUT INVALID):
// 1 no look-back walk, 2 no global store, 4 no scatter, 8 aligned in-place store
#ifndef RS_AR_ABLATE
#define RS_AR_ABLATE 0
#endif
// per-warp digit counters as 16-bit halves of shared words (digits 2w, 2w+1
// share word w): 128 words per warp instead of 256, so fewer bank conflicts
// look-back window of the small-tile configuration (all tiles in flight at once)
#ifndef RS_AR_LB_SMALL
#define RS_AR_LB_SMALL 8
#endif
// key loads through the read-only path: bit 0 [rank], bit 1 [scatter] (timing experiments)
#ifndef RS_AR_LDG
#define RS_AR_LDG 0
#endif
// [store] with the evict-first (streaming) cache hint: -1 u32 keys only (2^27 pass
// 0.335 -> 0.328 ms, 2^31 4.874 -> 4.858, DRAM bytes unchanged; u64 / pairs flat), 0 / 1
#ifndef RS_AR_STCS
#define RS_AR_STCS -1
#endif
#ifndef RS_AR_EARLY_NEXT
#define RS_AR_EARLY_NEXT 0
#endif
// per-phase cycle counts of thread 0 (development builds only: printf per CTA)
#ifndef RS_AR_PROF
#define RS_AR_PROF 0
#endif
#ifndef RS_AR_CT16
#define RS_AR_CT16 1
#endif
// RANK2 (template): [rank] only counts (atomics without return); after [offset]
// has turned the counters into warp start offsets, [scatter] takes each key's
// slot from a second returning atomic (start + stable rank, lane-ordered as in
// [rank]) — no rank registers and no counter load in the scatter.
// RANK2 = 2: [rank] keeps the returning atomics' stable ranks, but parks them (16
// bits each) in tensor memory with tcgen05.st instead of registers and [scatter]
// reads them back with tcgen05.ld: one random shared-memory access per key fewer
// than RANK2 = 1, and no rank registers (TMEM is otherwise idle in a sort)

namespace rs {

template <typename K, bool HAS_VAL, int RT, int KPT, int KSRC = 0>
struct OnesweepArCfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;
    static constexpr int THREADS = RT;
    static constexpr int WK = 32 * KPT;
    static constexpr int TILE = RT * KPT;
    static constexpr size_t in_off = 0;
    static constexpr size_t out_off = in_off + (KSRC != 0 ? 0 : (size_t)TILE * sizeof(K));
    static constexpr size_t vin_off = out_off + (size_t)TILE * sizeof(K);
    static constexpr size_t vout_off = vin_off + ((HAS_VAL && KSRC == 0) ? (size_t)TILE * 4 : 0);
    static constexpr size_t wc_off = vout_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t texcl_off = wc_off + (size_t)W * R * (RS_AR_CT16 ? 2 : 4);
    static constexpr size_t tcnt_off = texcl_off + R * 4;
    static constexpr size_t gofs_off = tcnt_off + R * 4;
    static constexpr size_t misc_off = gofs_off + R * 4;
    static constexpr size_t bar_off = misc_off + 64 * 4;
    static constexpr size_t smem_bytes = bar_off + 16;
};

// KREG: keep the keys in registers from [rank] to [scatter] (else re-read s_in).
// KSRC (where the ranking warps get their keys; 1 and 2 keys-only):
//   0  TMA bulk copy of the tile into shared memory (s_in)
//   1  each thread loads its keys from global memory into registers and keeps
//      them until the scatter (coalesced rows; the next tile is prefetched into
//      L2 by the TMA engine): no s_in, no shared-memory write/read of the input
//   2  as 1, but the keys are not kept: the scatter loads them again (from L2),
//      which frees the registers for larger tiles
template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S, bool KREG_, int KSRC = 0,
          int RANK2 = 0, int LB = 8>
__device__ __forceinline__ void onesweep_ar_body(const PassArgs& a) {
    static_assert(KSRC != 1 || !HAS_VAL, "register tiles are for keys-only sorts");
    constexpr bool LDGK = KSRC != 0;
    constexpr bool KREG = (KREG_ && KSRC != 2) || KSRC == 1;
    using ST = Status<S>;
    using C = OnesweepArCfg<K, HAS_VAL, RT, KPT, KSRC>;
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE, THREADS = C::THREADS;
    static_assert(RT % R == 0, "threads 0..255: one per digit in the offset and look-back phases");
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_in = reinterpret_cast<K*>(smem + C::in_off);
    K* s_out = reinterpret_cast<K*>(smem + C::out_off);
    uint32_t* s_vin = reinterpret_cast<uint32_t*>(smem + C::vin_off);
    uint32_t* s_vout = reinterpret_cast<uint32_t*>(smem + C::vout_off);
    uint32_t* s_wc = reinterpret_cast<uint32_t*>(smem + C::wc_off);
    uint32_t* s_texcl = reinterpret_cast<uint32_t*>(smem + C::texcl_off);
    uint32_t* s_tcnt = reinterpret_cast<uint32_t*>(smem + C::tcnt_off);
    uint32_t* s_gofs = reinterpret_cast<uint32_t*>(smem + C::gofs_off);
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + C::misc_off);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + C::bar_off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    S* const status = static_cast<S*>(a.status_cur);

    // clear the next pass's status rows (no reader in this launch)
    for (size_t i = (size_t)blockIdx.x * THREADS + tid; i < (size_t)a.num_tiles * R; i += (size_t)gridDim.x * THREADS)
        static_cast<S*>(a.status_next)[i] = 0;
    if (!ctrl->active[a.pass]) return;

    const int ss = ctrl->src_sel[a.pass], ds = ctrl->dst_sel[a.pass];
    const K* src = pick<const K>(ss, static_cast<const K*>(a.keys_in), static_cast<const K*>(a.keys_out),
                                 static_cast<const K*>(a.keys_alt));
    K* dst = pick<K>(ds, const_cast<K*>(static_cast<const K*>(a.keys_in)), static_cast<K*>(a.keys_out),
                     static_cast<K*>(a.keys_alt));
    const uint32_t* vsrc = nullptr;
    uint32_t* vdst = nullptr;
    if (HAS_VAL) {
        vsrc = pick<const uint32_t>(ss, a.vals_in, a.vals_out, a.vals_alt);
        vdst = pick<uint32_t>(ds, const_cast<uint32_t*>(a.vals_in), a.vals_out, a.vals_alt);
    }
    const int shift = a.shift;

    auto issue_load = [&](uint32_t t) {  // thread 0 only
        const size_t base = (size_t)t * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        const uint32_t kbytes = (valid * (uint32_t)sizeof(K)) & ~15u;
        if (LDGK) {  // L2 prefetch only; the threads load their keys (and values) themselves
            if (kbytes) bulk_prefetch_l2(src + base, kbytes);
            const uint32_t vb = HAS_VAL ? ((valid * 4u) & ~15u) : 0u;
            if (HAS_VAL && vb) bulk_prefetch_l2(vsrc + base, vb);
            return;
        }
        const uint32_t vbytes = HAS_VAL ? ((valid * 4u) & ~15u) : 0u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(s_bar, kbytes + vbytes);
        if (kbytes) bulk_g2s(s_in, src + base, kbytes, s_bar);
        if (HAS_VAL && vbytes) bulk_g2s(s_vin, vsrc + base, vbytes, s_bar);
    };

    if (tid == 0) {
        if (!LDGK) {
            mbar_init(s_bar, 1);
            fence_mbar_init();
        }
        const uint32_t t0 = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
        s_misc[0] = t0;
        if (t0 < a.num_tiles) issue_load(t0);
    }
    constexpr int WCW = W * R / (RS_AR_CT16 ? 2 : 1);  // counter words
    uint16_t* s_wc16 = reinterpret_cast<uint16_t*>(smem + C::wc_off);
    for (int i = tid; i < WCW; i += THREADS) s_wc[i] = 0;
    constexpr bool R2A = RANK2 == 1, RTM = RANK2 == 2;
    constexpr bool EARLY_NEXT = RS_AR_EARLY_NEXT && LDGK;  // TMA tiles need s_in free first
    constexpr int kRankCols = (W + 3) / 4 * (KPT / 2);  // TMEM columns per lane quarter
    static_assert(!RTM || kRankCols <= 512, "ranks must fit in 512 TMEM columns");
    constexpr uint32_t kTmemCols = kRankCols <= 32 ? 32u : kRankCols <= 64 ? 64u : kRankCols <= 128 ? 128u
                                                       : kRankCols <= 256 ? 256u : 512u;
    if (RTM && warp == 0) tmem_alloc(&s_misc[60], kTmemCols);
    if (RTM) tmem_fence_before_sync();
    __syncthreads();
    if (RTM) tmem_fence_after_sync();
    uint32_t tile = s_misc[0];
    uint32_t phase = 0;
    static_assert(KPT % 2 == 0 && WK <= 65536, "ranks are packed two per register");
#ifdef RS_AR_G
    constexpr int G = KPT % RS_AR_G == 0 ? RS_AR_G : (KPT % 8 == 0 ? 8 : (KPT % 6 == 0 ? 6 : (KPT % 4 == 0 ? 4 : 2)));
#else
    constexpr int G = KPT % 8 == 0 ? 8 : (KPT % 6 == 0 ? 6 : (KPT % 4 == 0 ? 4 : 2));  // batch of keys
#endif
    static_assert(G % 2 == 0 || R2A || RTM, "rank registers pack two 16-bit ranks");
    K kr[KREG ? KPT : 2];  // this thread's keys of the tile (rows j, lane)
    uint32_t rr[(R2A || RTM) ? 1 : KPT / 2];  // stable ranks within the warp's keys of their digit, 16 bits each
    // RTM: this thread's TMEM columns (lane quarter warp % 4; warps w and w + 4 side by side)
    uint32_t tcol = 0;
    if (RTM) tcol = s_misc[60] + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * (KPT / 2));

#if RS_AR_PROF
    unsigned long long prof_acc[5] = {0, 0, 0, 0, 0}, prof_t = clock64(), prof_tiles = 0;
#define RS_AR_PROF_MARK(i)                                  \
    do {                                                    \
        const unsigned long long t_ = clock64();            \
        prof_acc[i] += t_ - prof_t;                         \
        prof_t = t_;                                        \
    } while (0)
#else
#define RS_AR_PROF_MARK(i) \
    do {                   \
    } while (0)
#endif
    while (tile < a.num_tiles) {
        const size_t base = (size_t)tile * TILE;
#if RS_AR_PROF
        ++prof_tiles;
#endif
        // EARLY_NEXT: the next tile id (and its L2 prefetch) is taken as this tile
        // starts, so the id's global atomic round trip is off the [next] path
        if (EARLY_NEXT && tid == 0) {
            const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
            s_misc[2] = nt;
            if (nt < a.num_tiles) issue_load(nt);
        }
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);

        // ---- [load] wait for the tile; ragged tail by scalar loads, all-ones padding
        // (padding keys have digit 255 and come last, so they rank after every real key)
        const K* gk = src + base + warp * WK + lane;  // this thread's row-0 key (KSRC 1, 2)
        const uint32_t lim = valid - min(valid, (uint32_t)(warp * WK + lane));  // rows j*32 < lim are real
        if (KSRC == 1) {
            const K* g = gk;
            if (valid == (uint32_t)TILE) {
#pragma unroll
                for (int j = 0; j < KPT; ++j) kr[KREG ? j : 0] = __ldcs(g + j * 32);
            } else {
#pragma unroll
                for (int j = 0; j < KPT; ++j) kr[KREG ? j : 0] = (uint32_t)(j * 32) < lim ? g[j * 32] : ~K(0);
            }
        } else if (KSRC == 0 && valid < (uint32_t)TILE) {
            const uint32_t kdone = ((valid * (uint32_t)sizeof(K)) & ~15u) / sizeof(K);
            for (uint32_t i = kdone + tid; i < (uint32_t)TILE; i += THREADS)
                s_in[i] = i < valid ? src[base + i] : ~K(0);
            if (HAS_VAL) {
                const uint32_t vdone = ((valid * 4u) & ~15u) / 4;
                for (uint32_t i = vdone + tid; i < (uint32_t)TILE; i += THREADS)
                    s_vin[i] = i < valid ? vsrc[base + i] : 0u;
            }
        }
        if (!LDGK) {
            mbar_wait_parity(s_bar, phase);
            phase ^= 1u;
            __syncthreads();
        }

        // ---- [rank] one returning shared atomic per key: rank + per-warp histogram
        {
            const K* in = s_in + warp * WK + lane;
            uint32_t* wc = s_wc + warp * (WCW / W);
            // groups of G keys: G loads, then G atomics, then the packing of
            // their results, so G shared-memory round trips overlap (the compiler
            // keeps shared loads and atomics in program order)
#pragma unroll
            for (int g = 0; g < KPT; g += G) {
                K kk[G];
                uint32_t rg[G];
#pragma unroll
                for (int i = 0; i < G; ++i)
                    kk[i] = KSRC == 1   ? kr[KREG ? g + i : 0]
                            : KSRC == 2 ? ((uint32_t)((g + i) * 32) < lim ? (RS_AR_LDG & 1 ? __ldg(gk + (g + i) * 32) : gk[(g + i) * 32]) : ~K(0))
                                        : in[(g + i) * 32];
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    if (KREG && KSRC == 0) kr[KREG ? g + i : 0] = kk[i];
                    const uint32_t d = digit8<K>(kk[i], shift);
                    if (R2A) {
                        atomicAdd(&wc[RS_AR_CT16 ? d >> 1 : d], RS_AR_CT16 ? 1u << ((d & 1u) << 4) : 1u);
                        rg[i] = 0;
                    } else if (RS_AR_CT16) {
                        const uint32_t sh = (d & 1u) << 4;
                        rg[i] = atomicAdd(&wc[d >> 1], 1u << sh) >> sh;  // high bits cleared at packing
                    } else {
                        rg[i] = atomicAdd(&wc[d], 1u);
                    }
                }
                if (RTM) {
                    uint32_t rp[G / 2];
#pragma unroll
                    for (int i = 0; i < G; i += 2) rp[i / 2] = __byte_perm(rg[i], rg[i + 1], 0x5410);
                    if (G == 8) {
                        tmem_st4(tcol + g / 2, rp[0], rp[1 % (G / 2)], rp[2 % (G / 2)], rp[3 % (G / 2)]);
                    } else {
#pragma unroll
                        for (int i = 0; i < G / 2; ++i) tmem_st1(tcol + g / 2 + i, rp[i]);
                    }
                } else if (!R2A) {
#pragma unroll
                    for (int i = 0; i < G; i += 2)
                        rr[(R2A || RTM) ? 0 : (g + i) / 2] = __byte_perm(rg[i], rg[i + 1], 0x5410);
                }
            }
            if (RTM) tmem_wait_st();  // this thread reads its ranks back in [scatter]
        }
        __syncthreads();
        RS_AR_PROF_MARK(0);

        // ---- [offset] thread d: tile count, in-tile offset, warp start offsets; publish
        if (tid < R) {
            uint32_t c[W];
            uint32_t tcnt = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                c[w] = RS_AR_CT16 ? (uint32_t)s_wc16[w * R + tid] : s_wc[w * R + tid];
                tcnt += c[w];
            }
            uint32_t incl = tcnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_misc[8 + warp] = incl;
            const uint32_t pub = tcnt - (tid == R - 1 ? (uint32_t)TILE - valid : 0u);  // drop padding
            s_tcnt[tid] = pub;
            st_relaxed_gpu(status + (size_t)tile * R + tid, (tile == 0 ? ST::kFlagP : ST::kFlagA) | (S)pub);
            named_barrier_sync(1, R);
            uint32_t pre = 0;
#pragma unroll
            for (int w = 0; w < R / 32; ++w) pre += w < warp ? s_misc[8 + w] : 0u;
            uint32_t run = pre + incl - tcnt;  // in-tile offset of digit tid
            s_texcl[tid] = run;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (RS_AR_CT16) s_wc16[w * R + tid] = (uint16_t)run;
                else s_wc[w * R + tid] = run;
                run += c[w];
            }
        }
        __syncthreads();
        RS_AR_PROF_MARK(1);

        // ---- [scatter] each key to its stable slot of the tile sorted by digit
        {
            uint32_t* wc = s_wc + warp * R;
            uint32_t* wcp = s_wc + warp * (WCW / W);  // packed counters (RANK2 with CT16)
            const uint16_t* wc16 = s_wc16 + warp * R;
            const int ibase = warp * WK + lane;
            // groups of G keys: G key loads, G offset loads, then G stores
#pragma unroll
            for (int g = 0; g < ((RS_AR_ABLATE & 4) ? 0 : KPT); g += G) {
                K kk[G];
                uint32_t pos[G], vv[HAS_VAL ? G : 1];
                uint32_t rq[RTM ? G / 2 : 1];
                if (RTM) {
                    if (G == 8) {
                        tmem_ld4(tcol + g / 2, rq[0], rq[1 % (RTM ? G / 2 : 1)], rq[2 % (RTM ? G / 2 : 1)],
                                 rq[3 % (RTM ? G / 2 : 1)]);
                    } else {
#pragma unroll
                        for (int i = 0; i < (RTM ? G / 2 : 0); ++i) tmem_ld1(tcol + g / 2 + i, rq[i]);
                    }
                }
#pragma unroll
                for (int i = 0; i < G; ++i)
                    kk[i] = KREG        ? kr[KREG ? g + i : 0]
                            : KSRC == 2 ? ((uint32_t)((g + i) * 32) < lim ? (RS_AR_LDG & 2 ? __ldg(gk + (g + i) * 32) : __ldcs(gk + (g + i) * 32)) : ~K(0))
                                        : s_in[ibase + (g + i) * 32];
                if (RTM) tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    const int j = g + i;
                    const uint32_t d = digit8<K>(kk[i], shift);
                    if (R2A) {
                        if (RS_AR_CT16) {
                            const uint32_t sh = (d & 1u) << 4;
                            pos[i] = (atomicAdd(&wcp[d >> 1], 1u << sh) >> sh) & 0xFFFFu;
                        } else {
                            pos[i] = atomicAdd(&wc[d], 1u);
                        }
                    } else {
                        const uint32_t rw = RTM ? rq[RTM ? i / 2 : 0] : rr[(R2A || RTM) ? 0 : j / 2];
                        pos[i] = (RS_AR_CT16 ? (uint32_t)wc16[d] : wc[d]) + ((rw >> (16 * (j & 1))) & 0xFFFFu);
                    }
                    if (HAS_VAL)
                        vv[HAS_VAL ? i : 0] = KSRC == 2 ? ((uint32_t)(j * 32) < lim ? __ldcs(vsrc + base + ibase + j * 32) : 0u)
                                                        : s_vin[ibase + j * 32];
                }
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    RS_DCHECK(pos[i] < (uint32_t)TILE);
                    s_out[pos[i]] = kk[i];
                    if (HAS_VAL) s_vout[pos[i]] = vv[HAS_VAL ? i : 0];
                }
            }
        }

        // ---- [look-back] one digit per thread, windowed walk over earlier tiles
        RS_AR_PROF_MARK(2);
        if (tid < R) {
            S excl = 0;
            if (tile != 0 && (RS_AR_ABLATE & 1)) {
                st_relaxed_gpu(status + (size_t)tile * R + tid, ST::kFlagP | (S)s_tcnt[tid]);
            } else if (tile != 0) {
                const S* sp = status + (size_t)(tile - 1) * R + tid;
                int64_t left = (int64_t)tile;
                bool done = false;
                while (!done) {
                    S v[LB];
#pragma unroll
                    for (int i = 0; i < LB; ++i) v[i] = i < left ? ld_relaxed_gpu(sp - (size_t)i * R) : ST::kFlagP;
#pragma unroll
                    for (int i = 0; i < LB; ++i) {
                        if (done) break;
                        while ((v[i] & (ST::kFlagA | ST::kFlagP)) == 0) v[i] = ld_relaxed_gpu(sp - (size_t)i * R);
                        excl += ST::val(v[i]);
                        done = (v[i] & ST::kFlagP) != 0;
                    }
                    sp -= (size_t)LB * R;
                    left -= LB;
                }
                st_relaxed_gpu(status + (size_t)tile * R + tid, ST::kFlagP | (excl + (S)s_tcnt[tid]));
            }
            s_gofs[tid] = a.bases[a.pass * R + tid] + (uint32_t)excl - s_texcl[tid];
        }
        __syncthreads();
        RS_AR_PROF_MARK(3);

        // ---- [next] take the next tile and start its load; s_in and the counters are free
        if (tid == 0) {
            if (EARLY_NEXT) {
                s_misc[0] = s_misc[2];
            } else {
                const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
                s_misc[0] = nt;
                if (nt < a.num_tiles) issue_load(nt);
            }
        }
#pragma unroll
        for (int i = 0; i < (WCW + THREADS - 1) / THREADS; ++i)
            if (WCW % THREADS == 0 || i * THREADS + tid < WCW) s_wc[i * THREADS + tid] = 0;

        // ---- [store] bucket runs leave as coalesced bursts (full tiles in batches
        // of SG loads, SG offset lookups, SG stores)
        if (valid == (uint32_t)TILE && !(RS_AR_ABLATE & 2)) {
#ifdef RS_AR_SG
            constexpr int SG = KPT % RS_AR_SG == 0 ? RS_AR_SG : (KPT % 8 == 0 ? 8 : (KPT % 4 == 0 ? 4 : 2));
#else
            // 4 per batch: u32 2^27 pass 0.336 -> 0.326 ms, 2^31 and u64 / pairs unchanged;
            // 8 was the previous default, 22 / 44 cost 5.78 / 5.73 ms at 2^31 (more
            // stores in flight per thread make the scattered write stream slower)
            constexpr int SG = KPT % 4 == 0 ? 4 : 2;
#endif
#pragma unroll 1
            for (int b = 0; b < KPT; b += SG) {
                K k[SG];
                uint32_t g[SG], vv[HAS_VAL ? SG : 1];
#pragma unroll
                for (int i = 0; i < SG; ++i) k[i] = s_out[(b + i) * THREADS + tid];
#pragma unroll
                for (int i = 0; i < SG; ++i) {
                    g[i] = s_gofs[digit8<K>(k[i], shift)] + (uint32_t)((b + i) * THREADS + tid);
                    if (RS_AR_ABLATE & 8)  // timing only: the tile stored in place, aligned and coalesced
                        g[i] = (uint32_t)base + (uint32_t)((b + i) * THREADS + tid) + (g[i] & 0u);
                    if (HAS_VAL) vv[HAS_VAL ? i : 0] = s_vout[(b + i) * THREADS + tid];
                }
#pragma unroll
                for (int i = 0; i < SG; ++i) {
                    RS_DCHECK(g[i] < a.n);
                    if (RS_AR_STCS == 1 || (RS_AR_STCS < 0 && sizeof(K) == 4 && !HAS_VAL)) __stcs(&dst[g[i]], k[i]);
                    else dst[g[i]] = k[i];
                    if (HAS_VAL) vdst[g[i]] = vv[HAS_VAL ? i : 0];
                }
            }
        } else {
#pragma unroll 4
            for (uint32_t i = tid; i < valid; i += THREADS) {
                if (RS_AR_ABLATE & 2) break;
                const K k = s_out[i];
                const uint32_t g = s_gofs[digit8<K>(k, shift)] + i;
                RS_DCHECK(g < a.n);
                dst[g] = k;
                if (HAS_VAL) vdst[g] = s_vout[i];
            }
        }
        __syncthreads();
        RS_AR_PROF_MARK(4);
        tile = s_misc[0];
    }
#if RS_AR_PROF
    if (tid == 0 && blockIdx.x % 37 == 0)
        printf("PROF pass %d cta %d tiles %llu cycles/tile: rank %llu offset %llu scatter(t0) %llu lookback %llu store %llu\n",
               a.pass, blockIdx.x, prof_tiles, prof_acc[0] / max(prof_tiles, 1ull), prof_acc[1] / max(prof_tiles, 1ull),
               prof_acc[2] / max(prof_tiles, 1ull), prof_acc[3] / max(prof_tiles, 1ull), prof_acc[4] / max(prof_tiles, 1ull));
#endif
#undef RS_AR_PROF_MARK
    if (RTM) {  // every rank read back and waited for: release the columns
        tmem_fence_before_sync();
        __syncthreads();
        if (warp == 0) {
            tmem_fence_after_sync();
            tmem_dealloc(s_misc[60], kTmemCols);
        }
    }
}

// the pass as its own launch (the fused small-n sort runs the same body in a loop)
template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S, bool KREG_, int KSRC = 0,
          int RANK2 = 0, int LB = 8>
__global__ void __launch_bounds__(RT, MINB) k_onesweep_ar(PassArgs a) {
    onesweep_ar_body<K, HAS_VAL, RT, KPT, MINB, S, KREG_, KSRC, RANK2, LB>(a);
}

// Startup probe of the lane-order property design 5 relies on: every warp ranks
// `rows` rows of digits with returning shared atomics — on plain 32-bit counters
// and on 16-bit halves of shared words (digits 2w, 2w+1 in word w), the two
// forms the pass uses — and compares each result with the stable rank from the
// definition (count of equal digits in earlier rows + earlier lanes of the same
// row, via match.any).  Mismatches are added to *bad.
__global__ void __launch_bounds__(256) k_rank_probe(uint32_t seed, int rows, uint32_t* bad) {
    __shared__ uint32_t cnt[8][256];
    __shared__ uint32_t cnt2[8][128];
    __shared__ uint32_t ref[8][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
        (&cnt[0][0])[i] = 0;
        (&ref[0][0])[i] = 0;
    }
    for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) (&cnt2[0][0])[i] = 0;
    __syncthreads();
    // digit ranges 256, 16, 2, 1 (by block) so groups of every size occur
    const uint32_t mask = 0xFFu >> (2 * (blockIdx.x & 3));
    uint32_t miss = 0;
    for (int j = 0; j < rows; ++j) {
        uint32_t z = seed + (uint32_t)((blockIdx.x * 8 + warp) * rows + j) * 32u + lane;
        z ^= z >> 16; z *= 0x7feb352du; z ^= z >> 15; z *= 0x846ca68bu; z ^= z >> 16;
        const uint32_t d = (blockIdx.x & 3) == 3 ? 7u : (z & mask);
        const uint32_t r = atomicAdd(&cnt[warp][d], 1u);
        const uint32_t sh = (d & 1u) << 4;
        const uint32_t r2 = (atomicAdd(&cnt2[warp][d >> 1], 1u << sh) >> sh) & 0xFFFFu;
        // definition: earlier rows (ref) + earlier lanes of this row with digit d
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t want = ref[warp][d] + __popc(peers & lanemask_lt());
        miss += (r != want) + (r2 != want);
        __syncwarp();
        if ((peers & lanemask_gt()) == 0) ref[warp][d] += __popc(peers);
        __syncwarp();
    }
    if (miss) atomicAdd(bad, miss);
}

}  // namespace rs
