// K3 "atomic rank" (design 5, default when the startup probe passes) — one
// stable count-sort round of radix 256:
//
//   [load]    each warp reads its rows of the tile straight from global memory
//             (the tile was prefetched into L2 by the TMA engine at [next]);
//             keys-only large tiles keep them in registers until [scatter]
//   [rank]    warp w, row j (32 consecutive keys, lane order = input order).
//             Pairs (RANK2 = 0): one returning atomicAdd per key on the warp's
//             16-bit counter of its digit d; the returned old values ARE the
//             stable ranks of the keys among the warp's keys of digit d (earlier
//             rows were counted by earlier instructions, and within one
//             instruction the sm_100 shared-memory atomic unit returns the old
//             values of lanes that hit the same address in ascending lane order).
//             Keys only (RANK2 = 1, count-then-rank): this phase only counts —
//             on the large tiles into LANE-PRIVATE byte counters laid over the
//             (then unused) sorted-tile buffer, warp w / lane l / digit d at byte
//             d % 4 of word w·2048 + (d / 4)·32 + l, so every lane's RED hits its
//             own bank (one shared-memory wavefront per warp instruction instead
//             of ~3.8 for 32 random digits), after which each warp sums its 32
//             lanes' bytes into its 16-bit counters; on the small tiles by REDs on
//             the warp's 16-bit counters.  The lane order of the returning atomics
//             is a measured hardware property, not a PTX guarantee: the library
//             checks it with a probe kernel of this kernel's shape before it
//             selects this design (radix.cu) and otherwise runs design 2 (ballot
//             ranks, onesweep_ec.cuh).  The counters end as the warp's digit
//             histogram: the counting of PAPER.md:664-667.
//   [offset]  thread d: tile count, in-tile offset of digit d, per-warp start
//             offsets; publish the tile count to the look-back status (flag A,
//             or P for tile 0) — the tiles x 256 counter matrix of PR4,
//             PAPER.md:690-694
//   [scatter] key -> s_out[start_w[d] + r]  (the tile sorted by digit, stably);
//             RANK2 = 1 takes start + r from a returning atomic on the counters
//             [offset] turned into warp starts (no rank registers)
//   [lookback] thread d: windowed decoupled look-back over earlier tiles,
//             publishes the inclusive prefix (flag P)
//   [next]    thread 0 takes the next tile id and L2-prefetches it (TMA engine)
//   [store]   32 consecutive sorted slots per warp instruction: each bucket run
//             leaves as coalesced bursts at base[d] + prefix[d] + offset.  Keys
//             only: each warp walks a contiguous range of the tile and each lane
//             caches the bucket offset of its previous key's digit, so the offset
//             lookup is a rare predicated shared load (a lane's next key, 32
//             slots on, is mostly in the same run)
//
// What bounds the pass: the SM's L1 / shared-memory data pipe (ncu, u32 at 2^27:
// ~83 % of its wavefronts busy before the lane-private count, the register-
// resident keys and the cached offsets, which together cut its wavefronts per key
// by ~12 %).
#pragma once

#include "onesweep_ec.cuh"

namespace rs {

template <typename K, bool HAS_VAL, int RT, int KPT>
struct OnesweepArCfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;
    static constexpr int THREADS = RT;
    static constexpr int WK = 32 * KPT;
    static constexpr int TILE = RT * KPT;
    static constexpr size_t out_off = 0;
    static constexpr size_t vout_off = out_off + (size_t)TILE * sizeof(K);
    static constexpr size_t wc_off = vout_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t texcl_off = wc_off + (size_t)W * R * 2;  // 16-bit counters, two per word
    static constexpr size_t tcnt_off = texcl_off + R * 4;
    static constexpr size_t gofs_off = tcnt_off + R * 4;
    static constexpr size_t misc_off = gofs_off + R * 4;
    static constexpr size_t smem_bytes = misc_off + 64 * 4;
    // keys-only large tiles: lane-private count + keys in registers + cached offsets
    static constexpr bool kLpc =
        !HAS_VAL && KPT % 8 == 0 && KPT <= 127 && (size_t)W * 2048 * 4 <= (size_t)TILE * sizeof(K);
};

#ifdef RS_AR_TRACE
// (diagnostic build only) per tile: globaltimer at start, after [rank], after
// [scatter], after [look-back], at the end of [store]; SM id
__device__ unsigned long long g_rs_trace[1 << 17][6];
__device__ __forceinline__ unsigned long long rs_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RS_TRACE(tile, k)                                                      \
    do {                                                                        \
        if (tid == 0 && (tile) < (1u << 17)) g_rs_trace[tile][k] = rs_gtime(); \
    } while (0)
#else
#define RS_TRACE(tile, k) \
    do {                  \
    } while (0)
#endif
template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S, int RANK2, int LB>
__global__ void __launch_bounds__(RT, MINB) k_onesweep_ar(PassArgs a) {
    using ST = Status<S>;
    using C = OnesweepArCfg<K, HAS_VAL, RT, KPT>;
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE, THREADS = C::THREADS;
    static_assert(RT % R == 0, "threads 0..255: one per digit in the offset and look-back phases");
    static_assert(KPT % 2 == 0 && WK <= 65536, "16-bit counters; ranks are packed two per register");
    constexpr bool R2A = RANK2 == 1;
    constexpr bool LPC = R2A && C::kLpc;  // lane-private count, keys in registers, cached offsets
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_out = reinterpret_cast<K*>(smem + C::out_off);
    uint32_t* s_vout = reinterpret_cast<uint32_t*>(smem + C::vout_off);
    uint32_t* s_wc = reinterpret_cast<uint32_t*>(smem + C::wc_off);
    uint16_t* s_wc16 = reinterpret_cast<uint16_t*>(smem + C::wc_off);
    uint32_t* s_texcl = reinterpret_cast<uint32_t*>(smem + C::texcl_off);
    uint32_t* s_tcnt = reinterpret_cast<uint32_t*>(smem + C::tcnt_off);
    uint32_t* s_gofs = reinterpret_cast<uint32_t*>(smem + C::gofs_off);
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + C::misc_off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    S* const status = static_cast<S*>(a.status_cur);
    // PDL (common.cuh): every global access below (the tile counter, the plan, the
    // status rows the previous pass used, its output) comes after the wait; the
    // persistent grid is resident before any CTA triggers the next kernel
    pdl_wait();
    pdl_trigger();

    // small tiles (about one tile per CTA): the first tile id and the pass plan are
    // fetched together, two global round trips in flight at once (2^20 keys: 14.5 ->
    // 12.9 us per pass; an inactive pass just leaves its tile counter advanced).  The
    // large tiles keep the plan read after the status clearing (the early fetch
    // measured 1 % slower at 2^27).
    constexpr bool kEarlyTile = KPT <= 16;
    uint32_t t0 = 0;
    if (kEarlyTile && tid == 0) t0 = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
    int act = 1, ss = 0, ds = 0;
    if (kEarlyTile) {
        act = ctrl->active[a.pass];
        ss = ctrl->src_sel[a.pass];
        ds = ctrl->dst_sel[a.pass];
    }
    // clear the next pass's status rows (no reader in this launch)
    for (size_t i = (size_t)blockIdx.x * THREADS + tid; i < (size_t)a.num_tiles * R; i += (size_t)gridDim.x * THREADS)
        static_cast<S*>(a.status_next)[i] = 0;
    if (!kEarlyTile) {
        act = ctrl->active[a.pass];
        if (act) {
            ss = ctrl->src_sel[a.pass];
            ds = ctrl->dst_sel[a.pass];
        }
    }
    if (!act) return;

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

    auto prefetch = [&](uint32_t t) {  // thread 0 only: the tile into L2 by the TMA engine
        const size_t base = (size_t)t * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        const uint32_t kbytes = (valid * (uint32_t)sizeof(K)) & ~15u;
        if (kbytes) bulk_prefetch_l2(src + base, kbytes);
        const uint32_t vb = HAS_VAL ? ((valid * 4u) & ~15u) : 0u;
        if (HAS_VAL && vb) bulk_prefetch_l2(vsrc + base, vb);
    };

    if (tid == 0) {
        if (!kEarlyTile) t0 = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
        s_misc[0] = t0;
        if (t0 < a.num_tiles) prefetch(t0);
    }
    constexpr int WCW = W * R / 2;  // counter words
    for (int i = tid; i < WCW; i += THREADS) s_wc[i] = 0;
    __syncthreads();
    uint32_t tile = s_misc[0];
    // batches of G keys: G loads, then G atomics, so G shared-memory round trips overlap
    constexpr int G = KPT % 8 == 0 ? 8 : (KPT % 6 == 0 ? 6 : (KPT % 4 == 0 ? 4 : 2));
    uint32_t rr[R2A ? 1 : KPT / 2];  // pairs: stable ranks within the warp's keys of their digit, 16 bits each
    K kr[LPC ? KPT : 1];             // keys-only large tiles: this thread's keys of the tile

    while (tile < a.num_tiles) {
        const size_t base = (size_t)tile * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        // this thread's row-0 key; rows j*32 < lim are real, the rest are all-ones
        // padding (digit 255, ranked after every real key)
        const K* gk = src + base + warp * WK + lane;
        const uint32_t lim = valid - min(valid, (uint32_t)(warp * WK + lane));
        RS_TRACE(tile, 0);
#ifdef RS_AR_TRACE
        if (tid == 0 && tile < (1u << 17)) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_rs_trace[tile][5] = smid;
        }
#endif

        // ---- [rank]
        if (LPC) {
            uint32_t* lp = reinterpret_cast<uint32_t*>(smem + C::out_off) + warp * 2048;
#pragma unroll
            for (int q = 0; q < 16; ++q) reinterpret_cast<uint4*>(lp)[q * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
            // loads per batch (they all land in kr): half a row block in flight at once
            // (u32 2^31 pass: batches of 8 4.42 ms, 22 4.43, 44 4.29, 88 4.35)
            // (u64 keys: batches of 8, 0.936 ms per 2^28 pass against 0.952 with 20)
            constexpr int GR = sizeof(K) == 4 && (KPT / 2) % 2 == 0 ? KPT / 2 : G;
#pragma unroll
            for (int g = 0; g < KPT; g += GR) {
#pragma unroll
                for (int i = 0; i < GR; ++i)
                    kr[LPC ? g + i : 0] = (uint32_t)((g + i) * 32) < lim ? gk[(g + i) * 32] : ~K(0);
#pragma unroll
                for (int i = 0; i < GR; ++i) {
                    const uint32_t d = digit8<K>(kr[LPC ? g + i : 0], shift);
                    atomicAdd(&lp[(d >> 2) * 32 + lane], 1u << ((d & 3u) << 3));
                }
            }
            __syncwarp();
            // lane l sums rows l and l + 32 (digits 4·row .. 4·row + 3) over the 32 lanes
            uint32_t* wc = s_wc + warp * (WCW / W);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int row = lane + 32 * h;
                const uint4* rp = reinterpret_cast<const uint4*>(lp + row * 32);
                uint32_t lo = 0, hi = 0;  // 16-bit lanes: lo = digits 4r, 4r+2; hi = 4r+1, 4r+3
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 v = rp[(q + lane) & 7];  // staggered: 8 lanes cover the 32 banks
                    const uint32_t s0 = v.x + v.y, s1 = v.z + v.w;  // bytes <= 2·KPT < 256
                    lo += (s0 & 0x00FF00FFu) + (s1 & 0x00FF00FFu);
                    hi += ((s0 >> 8) & 0x00FF00FFu) + ((s1 >> 8) & 0x00FF00FFu);
                }
                wc[2 * row] = (lo & 0xFFFFu) | (hi << 16);
                wc[2 * row + 1] = (lo >> 16) | (hi & 0xFFFF0000u);
            }
        } else {
            uint32_t* wc = s_wc + warp * (WCW / W);
#ifdef RS_AR_GP
            constexpr int GK = HAS_VAL && KPT % RS_AR_GP == 0 ? RS_AR_GP : G;  // (tuning: pairs rank batch)
#else
            constexpr int GK = G;
#endif
#pragma unroll
            for (int g = 0; g < KPT; g += GK) {
                K kk[GK];
                uint32_t rg[GK];
#pragma unroll
                for (int i = 0; i < GK; ++i) kk[i] = (uint32_t)((g + i) * 32) < lim ? gk[(g + i) * 32] : ~K(0);
#pragma unroll
                for (int i = 0; i < GK; ++i) {
                    const uint32_t d = digit8<K>(kk[i], shift);
                    const uint32_t sh = (d & 1u) << 4;
                    if (R2A) {
                        atomicAdd(&wc[d >> 1], 1u << sh);
                        rg[i] = 0;
                    } else {
                        rg[i] = atomicAdd(&wc[d >> 1], 1u << sh) >> sh;  // high bits cleared at packing
                    }
                }
                if (!R2A) {
#pragma unroll
                    for (int i = 0; i < GK; i += 2) rr[R2A ? 0 : (g + i) / 2] = __byte_perm(rg[i], rg[i + 1], 0x5410);
                }
            }
        }
        __syncthreads();
        RS_TRACE(tile, 1);

        // ---- [offset] thread d: tile count, in-tile offset, warp start offsets; publish
        if (tid < R) {
            uint32_t c[W];
            uint32_t tcnt = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                c[w] = (uint32_t)s_wc16[w * R + tid];
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
                s_wc16[w * R + tid] = (uint16_t)run;
                run += c[w];
            }
        }
        __syncthreads();

        // ---- [scatter] each key to its stable slot of the tile sorted by digit
        {
            uint32_t* wcp = s_wc + warp * (WCW / W);
            const uint16_t* wc16 = s_wc16 + warp * R;
            const int ibase = warp * WK + lane;
#if defined(RS_AR_GS)
            constexpr int GS = LPC && KPT % RS_AR_GS == 0 ? RS_AR_GS : G;
#elif defined(RS_AR_GSP)
            constexpr int GS = HAS_VAL && KPT % RS_AR_GSP == 0 ? RS_AR_GSP : G;  // (tuning: pairs scatter batch)
#else
            constexpr int GS = G;
#endif
#pragma unroll
            for (int g = 0; g < KPT; g += GS) {
                K kk[GS];
                uint32_t pos[GS], vv[HAS_VAL ? GS : 1];
#pragma unroll
                for (int i = 0; i < GS; ++i)
                    kk[i] = LPC ? kr[LPC ? g + i : 0]
                                : ((uint32_t)((g + i) * 32) < lim ? __ldcs(gk + (g + i) * 32) : ~K(0));
#pragma unroll
                for (int i = 0; i < GS; ++i) {
                    const int j = g + i;
                    const uint32_t d = digit8<K>(kk[i], shift);
                    if (R2A) {
                        const uint32_t sh = (d & 1u) << 4;
                        pos[i] = (atomicAdd(&wcp[d >> 1], 1u << sh) >> sh) & 0xFFFFu;
                    } else {
                        const uint32_t rw = rr[R2A ? 0 : j / 2];
                        pos[i] = (uint32_t)wc16[d] + ((rw >> (16 * (j & 1))) & 0xFFFFu);
                    }
                    if (HAS_VAL)
                        vv[HAS_VAL ? i : 0] = (uint32_t)(j * 32) < lim ? __ldcs(vsrc + base + ibase + j * 32) : 0u;
                }
#pragma unroll
                for (int i = 0; i < GS; ++i) {
                    RS_DCHECK(pos[i] < (uint32_t)TILE);
                    s_out[pos[i]] = kk[i];
                    if (HAS_VAL) s_vout[pos[i]] = vv[HAS_VAL ? i : 0];
                }
            }
        }

        RS_TRACE(tile, 2);
        // ---- [look-back] one digit per thread, windowed walk over earlier tiles
        if (tid < R) {
            S excl = 0;
            if (tile != 0) {
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
        RS_TRACE(tile, 3);

        // ---- [next] take the next tile and prefetch it; the counters are free
        if (tid == 0) {
            const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
            s_misc[0] = nt;
            if (nt < a.num_tiles) prefetch(nt);
        }
        if (!LPC) {  // (the lane-private count rewrites every counter)
#pragma unroll
            for (int i = 0; i < (WCW + THREADS - 1) / THREADS; ++i)
                if (WCW % THREADS == 0 || i * THREADS + tid < WCW) s_wc[i * THREADS + tid] = 0;
        }

        // ---- [store] bucket runs leave as coalesced bursts (batches of 4 loads, 4
        // offset lookups, 4 stores: u32 2^27 pass 0.336 -> 0.326 ms against 8)
// pairs: 2 per batch (ms per pass at 2^26 / 2^28 / 2^30 pairs: 1 0.372 / 1.468 / 5.85, 2 0.371 /
// 1.446 / 5.84, 4 0.374 / 1.454 / 5.88, 6 0.377 / 1.472 / 5.92, 8 0.382 / 1.493 / 6.01)
#ifndef RS_AR_SGP
#define RS_AR_SGP 2
#endif
// keys: 4 (ms per pass at u32 2^26 / 2^27 / 2^31 and u64 2^28: 2 0.165 / 0.307 / 4.53 / 0.939,
// 4 0.156 / 0.290 / 4.29 / 0.935, 8 0.159 / 0.294 / 4.38 / 0.945)
#ifndef RS_AR_SGK
#define RS_AR_SGK 4
#endif
        constexpr int SG = HAS_VAL ? (KPT % RS_AR_SGP == 0 ? RS_AR_SGP : 2) : (KPT % RS_AR_SGK == 0 ? RS_AR_SGK : 2);
        if (LPC && valid == (uint32_t)TILE) {
            const int sb = warp * WK + lane;     // warp w: slots [w·WK, (w+1)·WK)
            uint32_t cd = 0xFFFFFFFFu, cg = 0;  // cached digit and its bucket offset
#pragma unroll 1
            for (int j = 0; j < KPT; j += SG) {
                K k[SG];
                uint32_t g[SG];
#pragma unroll
                for (int i = 0; i < SG; ++i) k[i] = s_out[sb + (j + i) * 32];
#pragma unroll
                for (int i = 0; i < SG; ++i) {
                    const uint32_t d = digit8<K>(k[i], shift);
                    g[i] = cg;  // predicated load: only lanes whose digit changed touch shared memory
                    asm volatile("{\n.reg .pred p;\nsetp.ne.u32 p, %1, %2;\n@p ld.shared.u32 %0, [%3];\n}"
                                 : "+r"(g[i])
                                 : "r"(d), "r"(cd), "r"(smem_addr(s_gofs + d)));
                    if (i == SG - 1) cd = d;
                }
                cg = g[SG - 1];
#pragma unroll
                for (int i = 0; i < SG; ++i) {
                    const uint32_t gi = g[i] + (uint32_t)(sb + (j + i) * 32);
                    RS_DCHECK(gi < a.n);
                    // evict-first stores for u32 keys (2^27 pass 0.335 -> 0.328 ms, DRAM bytes unchanged)
                    if (sizeof(K) == 4) __stcs(&dst[gi], k[i]);
                    else dst[gi] = k[i];
                }
            }
        } else if (valid == (uint32_t)TILE) {
#pragma unroll 1
            for (int b = 0; b < KPT; b += SG) {
                K k[SG];
                uint32_t g[SG], vv[HAS_VAL ? SG : 1];
#pragma unroll
                for (int i = 0; i < SG; ++i) k[i] = s_out[(b + i) * THREADS + tid];
#pragma unroll
                for (int i = 0; i < SG; ++i) {
                    g[i] = s_gofs[digit8<K>(k[i], shift)] + (uint32_t)((b + i) * THREADS + tid);
                    if (HAS_VAL) vv[HAS_VAL ? i : 0] = s_vout[(b + i) * THREADS + tid];
                }
#pragma unroll
                for (int i = 0; i < SG; ++i) {
                    RS_DCHECK(g[i] < a.n);
                    if (sizeof(K) == 4 && !HAS_VAL) __stcs(&dst[g[i]], k[i]);
                    else dst[g[i]] = k[i];
                    if (HAS_VAL) vdst[g[i]] = vv[HAS_VAL ? i : 0];
                }
            }
        } else {
#pragma unroll 4
            for (uint32_t i = tid; i < valid; i += THREADS) {
                const K k = s_out[i];
                const uint32_t g = s_gofs[digit8<K>(k, shift)] + i;
                RS_DCHECK(g < a.n);
                dst[g] = k;
                if (HAS_VAL) vdst[g] = s_vout[i];
            }
        }
        __syncthreads();
        RS_TRACE(tile, 4);
        tile = s_misc[0];
    }
}

// Probe of the lane-order property design 5 relies on, in the pass's own shape:
// the same block size, launch bounds and dynamic shared memory as the u32 pass
// (so the same occupancy and shared-memory contention), every warp ranking rows
// of digits in batches of G returning atomics on 16-bit halves of shared words
// (digits 2w, 2w+1 in word w) exactly as [rank] (RANK2 0) and [scatter] (RANK2 1)
// issue them, then once more on the counters turned into warp starts.  Each
// result is compared with the stable rank from the definition (count of equal
// digits in earlier rows + earlier lanes of the same row, via match.any);
// mismatches are added to *bad.  Digit ranges 256, 16, 2, 1 (by block) so
// same-address groups of every size occur.
template <int RT, int KPT, int MINB>
__global__ void __launch_bounds__(RT, MINB) k_rank_probe(uint32_t seed, uint32_t* bad) {
    constexpr int W = RT / 32, R = 256, G = KPT % 8 == 0 ? 8 : 2;
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);      // [W][128] packed 16-bit
    uint32_t* ref = cnt + W * R / 2;                          // [W][256]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < W * R / 2 + W * R; i += RT) cnt[i] = 0;
    __syncthreads();
    const uint32_t mask = 0xFFu >> (2 * (blockIdx.x & 3));
    uint32_t* wc = cnt + warp * (R / 2);
    uint32_t* wr = ref + warp * R;
    uint32_t miss = 0;
    auto dig = [&](int j) {
        uint32_t z = seed + (uint32_t)((blockIdx.x * W + warp) * KPT + j) * 32u + lane;
        z ^= z >> 16; z *= 0x7feb352du; z ^= z >> 15; z *= 0x846ca68bu; z ^= z >> 16;
        return (blockIdx.x & 3) == 3 ? 7u : (z & mask);
    };
    for (int round = 0; round < 2; ++round) {
        // round 0: counters from zero (RANK2 0 [rank]); round 1: counters at the
        // final counts of round 0, i.e. a nonzero start per digit (RANK2 1 [scatter])
        for (int g = 0; g < KPT; g += G) {
            uint32_t d[G], r[G];
#pragma unroll
            for (int i = 0; i < G; ++i) d[i] = dig(g + i);
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const uint32_t sh = (d[i] & 1u) << 4;
                r[i] = (atomicAdd(&wc[d[i] >> 1], 1u << sh) >> sh) & 0xFFFFu;
            }
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const uint32_t peers = __match_any_sync(0xffffffffu, d[i]);
                const uint32_t want = wr[d[i]] + __popc(peers & lanemask_lt());
                miss += r[i] != want;
                __syncwarp();
                if ((peers & lanemask_gt()) == 0) wr[d[i]] += __popc(peers);
                __syncwarp();
            }
        }
    }
    if (miss) atomicAdd(bad, miss);
}

}  // namespace rs
