// K3 design 2 (early counts, ballot ranks) — one stable count-sort round of radix
// 256.  It relies on no ordering property of the hardware, so it
// is the fallback whenever the design-5 lane-order probe fails (radix.cu), and the
// "safe mode" of the dev option pass_design = 2.  Persistent CTAs:
//
//   [load]   TMA bulk copy of tile k into s_in (issued during tile k-1's store)
//   [count]  per-warp digit histogram by shared-memory atomics (keys kept in registers)
//   [offset] thread d: tile count, in-tile digit offset (scan over digits),
//            per-warp start offsets (scan over warps); publish the tile count to
//            the look-back status (flag A, or P for tile 0)  — PAPER.md:690-694
//   [rank]   stable warp rank, key written straight to its in-tile sorted slot in
//            s_out; keys in pairs: key j's peer mask from 8 ballots (ALU pipe), key
//            j+1's from a shared-memory atomic-OR of lane bits (order-independent)
//   [lookback] thread d: windowed decoupled look-back, publishes the inclusive prefix
//   [next]   thread 0 takes the next tile id and starts its TMA load into s_in
//   [store]  consecutive threads store consecutive s_out slots: each bucket run
//            is a coalesced burst at base[d] + prefix[d] + offset
#pragma once

#include "radix8.cuh"

namespace rs {

template <typename K, bool HAS_VAL, int RT, int KPT>
struct OnesweepEcCfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;
    static constexpr int THREADS = RT;
    static constexpr int WK = 32 * KPT;
    static constexpr int TILE = RT * KPT;
    static constexpr size_t in_off = 0;
    static constexpr size_t out_off = in_off + (size_t)TILE * sizeof(K);
    static constexpr size_t vin_off = out_off + (size_t)TILE * sizeof(K);
    static constexpr size_t vout_off = vin_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t wc_off = vout_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t wm_off = wc_off + (size_t)W * R * 4;  // atomic-OR peer masks
    static constexpr size_t texcl_off = wm_off + (size_t)W * R * 4;
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

template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S>
__global__ void __launch_bounds__(RT, MINB) k_onesweep_ec(PassArgs a) {
    using ST = Status<S>;
    using C = OnesweepEcCfg<K, HAS_VAL, RT, KPT>;
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE, THREADS = C::THREADS;
    static_assert(RT >= R, "one thread per digit in the offset phase");
    static_assert(KPT % 2 == 0, "keys are ranked in pairs");
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_in = reinterpret_cast<K*>(smem + C::in_off);
    K* s_out = reinterpret_cast<K*>(smem + C::out_off);
    uint32_t* s_vin = reinterpret_cast<uint32_t*>(smem + C::vin_off);
    uint32_t* s_vout = reinterpret_cast<uint32_t*>(smem + C::vout_off);
    uint32_t* s_wc = reinterpret_cast<uint32_t*>(smem + C::wc_off);
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
    for (int i = tid; i < W * R; i += THREADS) {
        s_wc[i] = 0;
        s_wm[i] = 0;  // kept zero by the group leaders
    }
    __syncthreads();
    uint32_t tile = s_misc[0];
    uint32_t phase = 0;
    K kr[KPT];  // the warp's keys, from [count] to [rank]

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
        {
            const K* in = s_in + warp * WK + lane;
            uint32_t* wc = s_wc + warp * R;
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                kr[j] = in[j * 32];
                atomicAdd(&wc[digit8<K>(kr[j], shift)], 1u);
            }
        }
        __syncthreads();

        // ---- [offset] thread d: tile count, in-tile offset, warp start offsets; publish
        if (tid < R) {
            uint32_t c[W];
            uint32_t tcnt = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                c[w] = s_wc[w * R + tid];
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
                s_wc[w * R + tid] = run;
                run += c[w];
            }
        }
        __syncthreads();

        // ---- [rank] stable warp rank, straight to the sorted slot
        {
            uint32_t* wc = s_wc + warp * R;
            uint32_t* wm = s_wm + warp * R;
            const int ibase = warp * WK + lane;
#pragma unroll
            for (int j = 0; j < KPT; j += 2) {
                const int i0 = ibase + j * 32, i1 = i0 + 32;
                const K k0 = kr[j], k1 = kr[j + 1];
                const uint32_t d0 = digit8<K>(k0, shift), d1 = digit8<K>(k1, shift);
                atomicOr(&wm[d1], 1u << lane);
                const uint32_t p0 = peers8(d0);
                {
                    const uint32_t cnt = wc[d0];
                    const uint32_t pos = cnt + __popc(p0 & lt);
                    RS_DCHECK(pos < (uint32_t)TILE);
                    s_out[pos] = k0;
                    if (HAS_VAL) s_vout[pos] = s_vin[i0];
                    __syncwarp();
                    if ((p0 & gt) == 0) wc[d0] = cnt + __popc(p0);
                    __syncwarp();  // also completes the ORs of key j+1
                }
                const uint32_t p1 = wm[d1];
                const uint32_t cnt = wc[d1];
                const uint32_t pos = cnt + __popc(p1 & lt);
                RS_DCHECK(pos < (uint32_t)TILE);
                s_out[pos] = k1;
                if (HAS_VAL) s_vout[pos] = s_vin[i1];
                __syncwarp();
                if ((p1 & gt) == 0) {
                    wc[d1] = cnt + __popc(p1);
                    wm[d1] = 0;
                }
                __syncwarp();
            }
        }
        if (tid < R) {
            // ---- [look-back] after ranking, one digit per thread, windowed walk
            S excl = 0;
            if (tile != 0) {
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
        for (int i = tid; i < W * R; i += THREADS) s_wc[i] = 0;

        // ---- [store] bucket runs leave as coalesced bursts
#pragma unroll 4
        for (uint32_t i = tid; i < valid; i += THREADS) {
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
