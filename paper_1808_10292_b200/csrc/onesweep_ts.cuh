// K3 "TMA store" (design 6, keys only) — the atomic-rank pass of onesweep_ar.cuh
// (one stable count-sort round of radix 256) whose bucket
// runs leave shared memory through the TMA engine instead of per-key stores:
//
//   [load]      TMA bulk copy of tile k into s_in (issued during tile k-1's store)
//   [rank]      r = atomicAdd(&cnt_w[d], 1): stable ranks + per-warp histogram
//               (lane-ordered returns, checked by the startup probe)
//   [offset]    thread d: tile count of digit d; publish the aggregate (flag A)
//   [look-back] thread d: exclusive prefix over earlier tiles, publish the
//               inclusive prefix (flag P) — BEFORE the scatter, because the run's
//               global start G_d decides where the run is placed in s_out:
//   [place]     run d starts in s_out at P_d ∈ [B_d, B_d + 3] with P_d ≡ G_d (mod 4),
//               B_d = Σ_{d'<d} (count_d' + 3): a run and its destination share
//               their 16-byte alignment
//   [scatter]   key -> s_out[P_d + warp offset + r]
//   [store]     thread d: scalar head (< 16 B), one cp.async.bulk shared->global of
//               the aligned body, scalar tail; the warps issue ~7 instructions per
//               run instead of ~8 per key, and the copies run asynchronously
//               while the next tile is ranked (s_out is reused only after
//               cp.async.bulk.wait_group.read)
#pragma once
#include "onesweep_ar.cuh"

namespace rs {

template <typename K, int RT, int KPT>
struct OnesweepTsCfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;
    static constexpr int WK = 32 * KPT;
    static constexpr int TILE = RT * KPT;
    static constexpr int OUTN = (TILE + 3 * R + 3 + 3) & ~3;  // runs with up to 3 slack slots each
    static constexpr size_t in_off = 0;
    static constexpr size_t out_off = in_off + (size_t)TILE * sizeof(K);
    static constexpr size_t wc_off = out_off + (size_t)OUTN * sizeof(K);
    static constexpr size_t tcnt_off = wc_off + (size_t)W * R * 2;  // 16-bit per-warp counters
    static constexpr size_t gst_off = tcnt_off + R * 4;               // G_d: global start of run d
    static constexpr size_t pst_off = gst_off + R * 4;                // P_d: shared start of run d
    static constexpr size_t misc_off = pst_off + R * 4;
    static constexpr size_t bar_off = misc_off + 64 * 4;
    static constexpr size_t smem_bytes = bar_off + 16;
};

template <typename K, int RT, int KPT, int MINB, typename S>
__global__ void __launch_bounds__(RT, MINB) k_onesweep_ts(PassArgs a) {
    using ST = Status<S>;
    using C = OnesweepTsCfg<K, RT, KPT>;
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE, THREADS = RT;
    static_assert(RT == R, "one thread per digit");
    static_assert(KPT % 2 == 0 && C::OUTN <= 65536, "ranks and offsets are 16-bit");
    constexpr int G = KPT % 8 == 0 ? 8 : (KPT % 6 == 0 ? 6 : (KPT % 4 == 0 ? 4 : 2));
    constexpr int VE = 16 / sizeof(K);  // keys per 16 bytes
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_in = reinterpret_cast<K*>(smem + C::in_off);
    K* s_out = reinterpret_cast<K*>(smem + C::out_off);
    uint32_t* s_wc = reinterpret_cast<uint32_t*>(smem + C::wc_off);
    uint16_t* s_wc16 = reinterpret_cast<uint16_t*>(smem + C::wc_off);
    uint32_t* s_tcnt = reinterpret_cast<uint32_t*>(smem + C::tcnt_off);
    uint32_t* s_gst = reinterpret_cast<uint32_t*>(smem + C::gst_off);
    uint32_t* s_pst = reinterpret_cast<uint32_t*>(smem + C::pst_off);
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + C::misc_off);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + C::bar_off);
    constexpr int WCW = W * R / 2;  // counter words

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    S* const status = static_cast<S*>(a.status_cur);

    for (size_t i = (size_t)blockIdx.x * THREADS + tid; i < (size_t)a.num_tiles * R; i += (size_t)gridDim.x * THREADS)
        static_cast<S*>(a.status_next)[i] = 0;
    if (!ctrl->active[a.pass]) return;

    const int ss = ctrl->src_sel[a.pass], ds = ctrl->dst_sel[a.pass];
    const K* src = pick<const K>(ss, static_cast<const K*>(a.keys_in), static_cast<const K*>(a.keys_out),
                                 static_cast<const K*>(a.keys_alt));
    K* dst = pick<K>(ds, const_cast<K*>(static_cast<const K*>(a.keys_in)), static_cast<K*>(a.keys_out),
                     static_cast<K*>(a.keys_alt));
    const int shift = a.shift;

    auto issue_load = [&](uint32_t t) {  // thread 0 only
        const size_t base = (size_t)t * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        const uint32_t kbytes = (valid * (uint32_t)sizeof(K)) & ~15u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(s_bar, kbytes);
        if (kbytes) bulk_g2s(s_in, src + base, kbytes, s_bar);
    };
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        const uint32_t t0 = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
        s_misc[0] = t0;
        if (t0 < a.num_tiles) issue_load(t0);
    }
    for (int i = tid; i < WCW; i += THREADS) s_wc[i] = 0;
    __syncthreads();
    uint32_t tile = s_misc[0];
    uint32_t phase = 0;
    uint32_t rr[KPT / 2];  // stable ranks within the warp's keys of their digit, 16 bits each

    while (tile < a.num_tiles) {
        const size_t base = (size_t)tile * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);

        // ---- [load] (padding keys ~0: digit 255, last in the tile, never stored)
        if (valid < (uint32_t)TILE) {
            const uint32_t kdone = ((valid * (uint32_t)sizeof(K)) & ~15u) / sizeof(K);
            for (uint32_t i = kdone + tid; i < (uint32_t)TILE; i += THREADS) s_in[i] = i < valid ? src[base + i] : ~K(0);
        }
        mbar_wait_parity(s_bar, phase);
        phase ^= 1u;
        __syncthreads();

        // ---- [rank]
        {
            const K* in = s_in + warp * WK + lane;
            uint32_t* wc = s_wc + warp * (WCW / W);
#pragma unroll
            for (int g = 0; g < KPT; g += G) {
                K kk[G];
                uint32_t rg[G];
#pragma unroll
                for (int i = 0; i < G; ++i) kk[i] = in[(g + i) * 32];
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    const uint32_t d = digit8<K>(kk[i], shift);
                    const uint32_t sh = (d & 1u) << 4;
                    rg[i] = atomicAdd(&wc[d >> 1], 1u << sh) >> sh;
                }
#pragma unroll
                for (int i = 0; i < G; i += 2) rr[(g + i) / 2] = __byte_perm(rg[i], rg[i + 1], 0x5410);
            }
        }
        __syncthreads();

        // ---- [offset] + [look-back] + [place], thread d
        {
            uint32_t c[W];
            uint32_t tcnt = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                c[w] = s_wc16[w * R + tid];
                tcnt += c[w];
            }
            const uint32_t pub = tcnt - (tid == R - 1 ? (uint32_t)TILE - valid : 0u);  // drop padding
            st_relaxed_gpu(status + (size_t)tile * R + tid, (tile == 0 ? ST::kFlagP : ST::kFlagA) | (S)pub);
            s_tcnt[tid] = pub;
            // B_d = Σ_{d'<d} (count_d' + 3): scan of (tcnt + 3) over the digits
            uint32_t incl = tcnt + 3;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_misc[8 + warp] = incl;
            // look-back: exclusive prefix of digit d over the earlier tiles
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
                st_relaxed_gpu(status + (size_t)tile * R + tid, ST::kFlagP | (excl + (S)pub));
            }
            const uint32_t gd = a.bases[a.pass * R + tid] + (uint32_t)excl;  // global start of run d
            __syncthreads();  // s_misc scan totals; also: every thread's earlier bulk stores ...
            uint32_t pre = 0;
#pragma unroll
            for (int w = 0; w < R / 32; ++w) pre += w < warp ? s_misc[8 + w] : 0u;
            const uint32_t bd = pre + incl - (tcnt + 3);
            const uint32_t pd = bd + ((gd - bd) & 3u);  // ≡ gd (mod 4), within the run's slack
            s_gst[tid] = gd;
            s_pst[tid] = pd;
            uint32_t run = pd;
            bulk_wait_read();  // ... this thread's bulk stores of the previous tile have read s_out
#pragma unroll
            for (int w = 0; w < W; ++w) {
                s_wc16[w * R + tid] = (uint16_t)run;
                run += c[w];
            }
        }
        __syncthreads();

        // ---- [scatter]
        {
            const uint16_t* wc16 = s_wc16 + warp * R;
            const int ibase = warp * WK + lane;
#pragma unroll
            for (int g = 0; g < KPT; g += G) {
                K kk[G];
                uint32_t pos[G];
#pragma unroll
                for (int i = 0; i < G; ++i) kk[i] = s_in[ibase + (g + i) * 32];
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    const int j = g + i;
                    pos[i] = (uint32_t)wc16[digit8<K>(kk[i], shift)] + ((rr[j / 2] >> (16 * (j & 1))) & 0xFFFFu);
                }
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    RS_DCHECK(pos[i] < (uint32_t)C::OUTN);
                    s_out[pos[i]] = kk[i];
                }
            }
        }
        __syncthreads();

        // ---- [next] the next tile's load; s_in and the counters are free
        if (tid == 0) {
            const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
            s_misc[0] = nt;
            if (nt < a.num_tiles) issue_load(nt);
        }
        for (int i = tid; i < WCW; i += THREADS) s_wc[i] = 0;

        // ---- [store] thread d: run d = s_out[P_d, P_d + n_d) -> dst[G_d, G_d + n_d)
        {
            const uint32_t nd = s_tcnt[tid], gd = s_gst[tid], pd = s_pst[tid];
            if (nd) {
                const uint32_t head = min(nd, (uint32_t)((VE - (gd % VE)) % VE));
                const uint32_t body = (nd - head) / VE * VE;
                for (uint32_t i = 0; i < head; ++i) dst[gd + i] = s_out[pd + i];
                if (body) {
                    RS_DCHECK(gd + head + body <= a.n);
                    fence_proxy_async_smem();
                    bulk_s2g(dst + gd + head, s_out + pd + head, body * (uint32_t)sizeof(K));
                    bulk_commit();
                }
                for (uint32_t i = head + body; i < nd; ++i) dst[gd + i] = s_out[pd + i];
            }
        }
        __syncthreads();
        tile = s_misc[0];
    }
    bulk_wait_all();
}

}  // namespace rs
