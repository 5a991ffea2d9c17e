// K3 (early counts) — one stable count-sort round of radix 256,
// pipelined so that the cross-tile look-back and the next tile's load overlap
// the in-tile ranking.  Persistent CTAs of RT ranking threads + 1 look-back warp:
//
//   [load]   TMA bulk copy of tile k into s_in (issued during tile k-1's store)
//   [count]  ranking warps: per-warp digit histogram by shared-memory atomics
//   [offset] thread d: tile count, in-tile digit offset (scan over digits),
//            per-warp start offsets (scan over warps); publish the tile count to
//            the look-back status (flag A, or P for tile 0)  — PAPER.md:690-694
//   [rank]   ranking warps: stable warp rank from 8 ballots, key written straight
//            to its in-tile sorted slot in s_out
//            ‖ look-back warp: windowed decoupled look-back for all 256 digits,
//              publishes the inclusive prefix (flag P), computes store offsets
//   [next]   thread 0 takes the next tile id and starts its TMA load into s_in
//   [store]  consecutive threads store consecutive s_out slots: each bucket run
//            is a coalesced burst at base[d] + prefix[d] + offset
#pragma once
#include <type_traits>

#include "radix8.cuh"

namespace rs {

// COMPACT: 16-bit per-warp counters and no atomic-OR mask array (fits 4 CTAs/SM)
template <typename K, bool HAS_VAL, int RT, int KPT, bool LBW = true, bool COMPACT = false>
struct OnesweepEcCfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;                 // ranking warps
    static constexpr int THREADS = RT + (LBW ? 32 : 0);  // + one look-back warp (LBW)
    static constexpr int WK = 32 * KPT;
    static constexpr int TILE = RT * KPT;
    static constexpr size_t in_off = 0;
    static constexpr size_t out_off = in_off + (size_t)TILE * sizeof(K);
    static constexpr size_t vin_off = out_off + (size_t)TILE * sizeof(K);
    static constexpr size_t vout_off = vin_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t wc_off = vout_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t wm_off = wc_off + (size_t)W * R * (COMPACT ? 2 : 4);   // peer masks (RANKV 1, 2)
    static constexpr size_t texcl_off = wm_off + (COMPACT ? 0 : (size_t)W * R * 4);
    static constexpr size_t tcnt_off = texcl_off + R * 4;
    static constexpr size_t gofs_off = tcnt_off + R * 4;
    static constexpr size_t misc_off = gofs_off + R * 4;
    static constexpr size_t bar_off = misc_off + 64 * 4;
    static constexpr size_t smem_bytes = bar_off + 16;
};

template <typename K>
__device__ __forceinline__ uint32_t digit8(K k, int shift) {
    return static_cast<uint32_t>(k >> shift) & 0xFFu;
}
template <>
__device__ __forceinline__ uint32_t digit8<uint32_t>(uint32_t k, int shift) {
    return __byte_perm(k, 0u, 0x4440u + (uint32_t)(shift >> 3));  // byte shift/8, zero-extended
}

// ME > 0: every ME-th key (ME even) is ranked with match.any instead of ballots.
// RANKV 1: peer masks by shared-memory atomic OR of lane bits (order-independent,
// so stable by construction) instead of ballots.
// DBG: compile in the timing-ablation switches (a.debug_skip); off in normal builds.
template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S, bool LBW, int ME = 0, int RANKV = 0,
          bool DBG = false, bool COMPACT = false>
__global__ void __launch_bounds__(RT + (LBW ? 32 : 0), MINB) k_onesweep_ec(PassArgs a) {
    using ST = Status<S>;
    using C = OnesweepEcCfg<K, HAS_VAL, RT, KPT, LBW, COMPACT>;
    using CT = typename std::conditional<COMPACT, uint16_t, uint32_t>::type;  // per-warp counter type
    static_assert(!COMPACT || RANKV == 0, "the compact layout has no mask array");
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE, THREADS = C::THREADS;
    static_assert(RT >= R, "one ranking thread per digit in the offset phase");
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_in = reinterpret_cast<K*>(smem + C::in_off);
    K* s_out = reinterpret_cast<K*>(smem + C::out_off);
    uint32_t* s_vin = reinterpret_cast<uint32_t*>(smem + C::vin_off);
    uint32_t* s_vout = reinterpret_cast<uint32_t*>(smem + C::vout_off);
    CT* s_wc = reinterpret_cast<CT*>(smem + C::wc_off);
    uint32_t* s_wc32 = reinterpret_cast<uint32_t*>(smem + C::wc_off);
    constexpr int WCW = W * R * (int)sizeof(CT) / 4;  // counter words
    uint32_t* s_wm = reinterpret_cast<uint32_t*>(smem + C::wm_off);
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
    const uint32_t lt = lanemask_lt(), gt = lanemask_gt();

    // issue the bulk load of `t` into s_in (thread 0 only)
    auto issue_load = [&](uint32_t t) {
        const size_t base = (size_t)t * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        const uint32_t kbytes = (valid * (uint32_t)sizeof(K)) & ~15u;
        const uint32_t vbytes = HAS_VAL ? ((valid * 4u) & ~15u) : 0u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(s_bar, kbytes + vbytes);
        if (kbytes) bulk_g2s(s_in, src + base, kbytes, s_bar);
        if (HAS_VAL && vbytes) bulk_g2s(s_vin, vsrc + base, vbytes, s_bar);
    };

    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        const uint32_t t0 = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
        s_misc[0] = t0;
        if (t0 < a.num_tiles) issue_load(t0);
    }
    for (int i = tid; i < WCW; i += THREADS) s_wc32[i] = 0;
    if (RANKV != 0)
        for (int i = tid; i < W * R; i += THREADS) s_wm[i] = 0;  // kept zero by the group leaders
    __syncthreads();
    uint32_t tile = s_misc[0];
    uint32_t phase = 0;
    // KREG: the ranking warps keep their keys in registers from [count] to [rank]
    // (one shared-memory read of the tile instead of two)
    constexpr bool KREG = !DBG && !COMPACT && ME == 0 && (RANKV == 0 || RANKV == 2);
    K kr[KREG ? KPT : 1];

    while (tile < a.num_tiles) {
        const size_t base = (size_t)tile * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);

        // ---- [load] wait for the tile; ragged tail by scalar loads, all-ones padding
        if (valid < (uint32_t)TILE) {
            const uint32_t kdone = ((valid * (uint32_t)sizeof(K)) & ~15u) / sizeof(K);
            for (uint32_t i = kdone + tid; i < (uint32_t)TILE; i += THREADS)
                s_in[i] = i < valid ? src[base + i] : ~K(0);
            if (HAS_VAL) {
                const uint32_t vdone = ((valid * 4u) & ~15u) / 4;
                for (uint32_t i = vdone + tid; i < (uint32_t)TILE; i += THREADS)
                    s_vin[i] = i < valid ? vsrc[base + i] : 0u;
            }
        }
        mbar_wait_parity(s_bar, phase);
        phase ^= 1u;
        __syncthreads();

        // ---- [count] per-warp digit histograms
        if (warp < W && !(DBG && (a.debug_skip & 8))) {  // (bit 3: ablation, no counting)
            const K* in = s_in + warp * WK + lane;
            if (COMPACT) {
                uint32_t* wc = s_wc32 + warp * (R / 2);
#pragma unroll 8
                for (int j = 0; j < KPT; ++j) {
                    const uint32_t d = digit8<K>(in[j * 32], shift);
                    atomicAdd(&wc[d >> 1], 1u << ((d & 1) << 4));
                }
            } else if (KREG) {
                uint32_t* wc = s_wc32 + warp * R;
#pragma unroll
                for (int j = 0; j < KPT; ++j) {
                    kr[j] = in[j * 32];
                    atomicAdd(&wc[digit8<K>(kr[j], shift)], 1u);
                }
            } else {
                uint32_t* wc = s_wc32 + warp * R;
#pragma unroll 8
                for (int j = 0; j < KPT; ++j) atomicAdd(&wc[digit8<K>(in[j * 32], shift)], 1u);
            }
        }
        __syncthreads();

        // ---- [offset] thread d: tile count, in-tile offset, warp start offsets; publish
        if (tid < R) {
            uint32_t c[W];
            uint32_t tcnt = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                c[w] = COMPACT ? (s_wc32[w * (R / 2) + (tid >> 1)] >> ((tid & 1) << 4)) & 0xFFFFu
                               : s_wc32[w * R + tid];
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
            for (int w = 0; w < (tid >> 5); ++w) pre += s_misc[8 + w];
            uint32_t run = pre + incl - tcnt;  // in-tile offset of digit tid
            s_texcl[tid] = run;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                s_wc[w * R + tid] = (CT)run;
                run += c[w];
            }
        }
        __syncthreads();

        if (LBW && warp == W) {
            // ---- [look-back] one warp, 8 digits per lane (in G groups), windowed walk
            constexpr int DPL = R / 32, G = sizeof(S) == 4 ? 1 : 2, DG = DPL / G, LB = 4;
#pragma unroll 1
            for (int g = 0; g < G; ++g) {
                S excl[DG];
#pragma unroll
                for (int k = 0; k < DG; ++k) excl[k] = 0;
                const int d0 = lane + 32 * DG * g;  // digits d0 + 32k, k < DG
                if (tile != 0) {
                    uint32_t done = 0;  // bit k: digit d0 + 32k finished
                    int64_t off = 1;    // next predecessor distance to read
                    while (done != (1u << DG) - 1) {
                        S v[DG][LB];
#pragma unroll
                        for (int k = 0; k < DG; ++k)
#pragma unroll
                            for (int i = 0; i < LB; ++i)
                                v[k][i] = (!(done >> k & 1) && off + i <= (int64_t)tile)
                                              ? ld_relaxed_gpu(status + (size_t)(tile - off - i) * R + d0 + 32 * k)
                                              : ST::kFlagP;
#pragma unroll
                        for (int k = 0; k < DG; ++k) {
#pragma unroll
                            for (int i = 0; i < LB; ++i) {
                                if (done >> k & 1) break;
                                S s = v[k][i];
                                while ((s & (ST::kFlagA | ST::kFlagP)) == 0)
                                    s = ld_relaxed_gpu(status + (size_t)(tile - off - i) * R + d0 + 32 * k);
                                excl[k] += ST::val(s);
                                if (s & ST::kFlagP) done |= 1u << k;
                            }
                        }
                        off += LB;
                    }
#pragma unroll
                    for (int k = 0; k < DG; ++k)
                        st_relaxed_gpu(status + (size_t)tile * R + d0 + 32 * k,
                                       ST::kFlagP | (excl[k] + (S)s_tcnt[d0 + 32 * k]));
                }
#pragma unroll
                for (int k = 0; k < DG; ++k) {
                    const int d = d0 + 32 * k;
                    s_gofs[d] = a.bases[a.pass * R + d] + (uint32_t)excl[k] - s_texcl[d];
                }
            }
        } else {
            // ---- [rank] stable warp rank, straight to the sorted slot.  Keys are
            // taken in pairs: both peer masks are computed before either counter
            // update so their independent ALU chains interleave; every ME-th key
            // uses match.any instead (ADU pipe) to offload the ALU pipe.
            CT* wc = s_wc + warp * R;
            const int ibase = warp * WK + lane;
            auto place = [&](const K k, const uint32_t d, const uint32_t peers, const int idx) {
                const uint32_t cnt = wc[d];
                const uint32_t pos = cnt + __popc(peers & lt);
                RS_DCHECK(pos < (uint32_t)TILE);
                s_out[pos] = k;
                if (HAS_VAL) s_vout[pos] = s_vin[idx];
                __syncwarp();
                if ((peers & gt) == 0) wc[d] = (CT)(cnt + __popc(peers));
                __syncwarp();
            };
            static_assert(KPT % 2 == 0, "keys are ranked in pairs");
            if (DBG && (a.debug_skip & 2)) {  // ablation: no ranking, identity placement
                for (int j = 0; j < KPT; ++j) s_out[ibase + j * 32] = s_in[ibase + j * 32];
            } else if (RANKV == 1) {
                uint32_t* wm = s_wm + warp * R;
#pragma unroll 4
                for (int j = 0; j < KPT; ++j) {
                    const int idx = ibase + j * 32;
                    const K k = s_in[idx];
                    const uint32_t d = digit8<K>(k, shift);
                    atomicOr(&wm[d], 1u << lane);
                    __syncwarp();
                    const uint32_t peers = wm[d];
                    const uint32_t cnt = wc[d];
                    const uint32_t pos = cnt + __popc(peers & lt);
                    RS_DCHECK(pos < (uint32_t)TILE);
                    s_out[pos] = k;
                    if (HAS_VAL) s_vout[pos] = s_vin[idx];
                    __syncwarp();
                    if ((peers & gt) == 0) {
                        wc[d] = (CT)(cnt + __popc(peers));
                        wm[d] = 0;
                    }
                    __syncwarp();
                }
            } else if (RANKV == 3) {
                // ballot peers; the group's leader (highest lane) advances the warp
                // counter with one atomicAdd returning the old value, which the
                // group reads by shuffle: no load->store chain through shared memory
#pragma unroll 2
                for (int j = 0; j < KPT; j += 2) {
                    const int i0 = ibase + j * 32, i1 = i0 + 32;
                    const K k0 = s_in[i0], k1 = s_in[i1];
                    const uint32_t d0 = digit8<K>(k0, shift), d1 = digit8<K>(k1, shift);
                    const uint32_t p0 = peers8(d0), p1 = peers8(d1);
                    const int l0 = 31 - __clz(p0), l1 = 31 - __clz(p1);
                    uint32_t o0 = 0, o1 = 0;
                    if (lane == l0) o0 = atomicAdd(reinterpret_cast<uint32_t*>(&wc[d0]), (uint32_t)__popc(p0));
                    __syncwarp();
                    if (lane == l1) o1 = atomicAdd(reinterpret_cast<uint32_t*>(&wc[d1]), (uint32_t)__popc(p1));
                    o0 = __shfl_sync(0xffffffffu, o0, l0);
                    o1 = __shfl_sync(0xffffffffu, o1, l1);
                    const uint32_t pos0 = o0 + __popc(p0 & lt), pos1 = o1 + __popc(p1 & lt);
                    RS_DCHECK(pos0 < (uint32_t)TILE && pos1 < (uint32_t)TILE);
                    s_out[pos0] = k0;
                    s_out[pos1] = k1;
                    if (HAS_VAL) {
                        s_vout[pos0] = s_vin[i0];
                        s_vout[pos1] = s_vin[i1];
                    }
                    __syncwarp();
                }
            } else if (RANKV == 2) {
                // hybrid pairs: key j by ballots (ALU pipe), key j+1 by an atomic-OR
                // peer mask (shared-memory pipe) whose latency hides behind the ballots
                uint32_t* wm = s_wm + warp * R;
#pragma unroll
                for (int j = 0; j < KPT; j += 2) {
                    const int i0 = ibase + j * 32, i1 = i0 + 32;
                    const K k0 = KREG ? kr[KREG ? j : 0] : s_in[i0], k1 = KREG ? kr[KREG ? j + 1 : 0] : s_in[i1];
                    const uint32_t d0 = digit8<K>(k0, shift), d1 = digit8<K>(k1, shift);
                    atomicOr(&wm[d1], 1u << lane);
                    const uint32_t p0 = peers8(d0);
                    place(k0, d0, p0, i0);  // ends with __syncwarp: the ORs are complete
                    const uint32_t p1 = wm[d1];
                    const uint32_t cnt = wc[d1];
                    const uint32_t pos = cnt + __popc(p1 & lt);
                    RS_DCHECK(pos < (uint32_t)TILE);
                    s_out[pos] = k1;
                    if (HAS_VAL) s_vout[pos] = s_vin[i1];
                    __syncwarp();
                    if ((p1 & gt) == 0) {
                        wc[d1] = (CT)(cnt + __popc(p1));
                        wm[d1] = 0;
                    }
                    __syncwarp();
                }
            } else
#pragma unroll
            for (int j = 0; j < KPT; j += 2) {
                const int i0 = ibase + j * 32, i1 = i0 + 32;
                const K k0 = KREG ? kr[KREG ? j : 0] : s_in[i0], k1 = KREG ? kr[KREG ? j + 1 : 0] : s_in[i1];
                const uint32_t d0 = digit8<K>(k0, shift), d1 = digit8<K>(k1, shift);
                const uint32_t p0 = (ME > 0 && (j % ME) == 0) ? __match_any_sync(0xffffffffu, d0) : peers8(d0);
                const uint32_t p1 = peers8(d1);
                if (DBG && (a.debug_skip & 16)) {  // experiment: one extra random shared load per key
                    uint32_t x0, x1;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x0) : "r"(smem_addr(wc + ((d0 * 37u) & 255u))));
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x1) : "r"(smem_addr(wc + ((d1 * 37u) & 255u))));
                    if ((x0 ^ x1) == 0xDEADBEEFu) s_misc[63] = x0;
                }
                place(k0, d0, p0, i0);
                place(k1, d1, p1, i1);
            }
        }
        if (!LBW && tid < R) {
            // ---- [look-back] after ranking, one digit per thread, windowed walk
            S excl = 0;
            if (tile != 0 && DBG && (a.debug_skip & 1)) {
                st_relaxed_gpu(status + (size_t)tile * R + tid, ST::kFlagP | (S)s_tcnt[tid]);  // ablation
            } else if (tile != 0) {
                constexpr int LB = 8;
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

        // ---- [next] take the next tile and start its load; s_in is free now
        if (tid == 0) {
            const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
            s_misc[0] = nt;
            if (nt < a.num_tiles) issue_load(nt);
        }
        for (int i = tid; i < WCW; i += THREADS) s_wc32[i] = 0;

        // ---- [store] bucket runs leave as coalesced bursts
#pragma unroll 4
        for (uint32_t i = tid; i < valid; i += THREADS) {
            if (DBG && (a.debug_skip & 4)) break;  // ablation: no global store
            const K k = s_out[i];
            const uint32_t g = s_gofs[digit8<K>(k, shift)] + i;
            RS_DCHECK(g < a.n);
            dst[g] = k;
            if (HAS_VAL) vdst[g] = s_vout[i];
        }
        __syncthreads();
        tile = s_misc[0];
    }
}

}  // namespace rs
