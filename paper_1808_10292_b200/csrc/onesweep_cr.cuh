// K3 (counter ranking) — one stable count-sort round of radix 256
// with the in-tile stable sort done as two 4-bit counting sub-passes, i.e. the
// paper's count-sort round itself (count, exclusive prefix, stable scatter;
// PAPER.md:659-671) applied inside shared memory with per-thread counters.
//
// Persistent CTAs of RT threads; two tile buffers A/B whose roles alternate.
//   [load]   TMA bulk copy of tile k into A (issued during tile k-1's store)
//   [count]  per-warp digit histograms (shared atomics) -> tile count per digit,
//            in-tile digit offsets; publish the tile count (flag A / P)
//   [sub 1]  blocked keys (thread t owns keys t*KPT .. t*KPT+KPT-1, so (t, j)
//            order is input order): per-thread counters of the LOW nibble,
//            exclusive scan over (nibble, thread), scatter A -> B
//   [sub 2]  the same for the HIGH nibble, B -> A: A now holds the tile stably
//            sorted by the 8-bit digit
//   [look-back] one thread per digit, windowed decoupled look-back
//   [next]   next tile id; its TMA load goes into B (free now)
//   [store]  consecutive threads store consecutive slots of A (coalesced bursts
//            per bucket run); then A and B swap roles
#pragma once
#include "onesweep_ec.cuh"

namespace rs {

template <typename K, bool HAS_VAL, int RT, int KPT>
struct OnesweepCrCfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;
    static constexpr int TILE = RT * KPT;
    static constexpr int NB = 16;  // nibble bins
    static constexpr size_t buf_bytes = (size_t)TILE * sizeof(K);
    static constexpr size_t a_off = 0;
    static constexpr size_t b_off = a_off + buf_bytes;
    static constexpr size_t va_off = b_off + buf_bytes;
    static constexpr size_t vb_off = va_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t cnt_off = vb_off + (HAS_VAL ? (size_t)TILE * 4 : 0);  // u16 [NB][RT]
    static constexpr size_t wc_off = cnt_off + (size_t)NB * RT * 2;
    static constexpr size_t tcnt_off = wc_off + (size_t)W * R * 4;
    static constexpr size_t gofs_off = tcnt_off + R * 4;
    static constexpr size_t misc_off = gofs_off + R * 4;
    static constexpr size_t bar_off = misc_off + 64 * 4;
    static constexpr size_t smem_bytes = bar_off + 16;
    static_assert(KPT % 4 == 0, "blocked keys are read with 16-byte loads");
    static_assert(TILE < 65536, "16-bit counters");
    static_assert((NB * RT / 2) % RT == 0, "raking scan: whole words per thread");
};

// one 4-bit stable counting sub-pass over the tile: keys k[] (blocked, thread t
// holds tile positions t*KPT + j) -> dst at their stable rank by nibble
template <typename K, bool HAS_VAL, int RT, int KPT>
__device__ __forceinline__ void nibble_subpass(const K (&k)[KPT], const uint32_t (&v)[HAS_VAL ? KPT : 1], int nshift,
                                               uint16_t* s_cnt, K* dst, uint32_t* vdst, uint32_t* s_misc) {
    constexpr int NB = 16, WPT = NB * RT / 2 / RT;  // u32 counter words per thread in the raking scan
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* s_cnt32 = reinterpret_cast<uint32_t*>(s_cnt);
    for (int i = tid; i < NB * RT / 2; i += RT) s_cnt32[i] = 0;
    __syncthreads();
    // count: thread-private counters, earlier keys of this thread first
    uint32_t pre[(KPT + 1) / 2];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const uint32_t nb = static_cast<uint32_t>(k[j] >> nshift) & 0xFu;
        uint16_t* c = s_cnt + nb * RT + tid;
        const uint32_t p = *c;
        *c = (uint16_t)(p + 1);
        if (j & 1) pre[j >> 1] |= p << 16;
        else pre[j >> 1] = p;
    }
    __syncthreads();
    // exclusive scan over (nibble, thread): raking over WPT words per thread
    uint32_t w[WPT];
    uint32_t tot = 0;
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
        w[i] = s_cnt32[tid * WPT + i];
        tot += (w[i] & 0xFFFFu) + (w[i] >> 16);
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_misc[16 + warp] = incl;
    __syncthreads();
    uint32_t run = incl - tot;
    for (int i = 0; i < warp; ++i) run += s_misc[16 + i];
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
        const uint32_t lo = w[i] & 0xFFFFu, hi = w[i] >> 16;
        s_cnt32[tid * WPT + i] = run | ((run + lo) << 16);
        run += lo + hi;
    }
    __syncthreads();
    // rank = scanned counter + count among this thread's earlier keys; scatter
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const uint32_t nb = static_cast<uint32_t>(k[j] >> nshift) & 0xFu;
        const uint32_t r = (uint32_t)s_cnt[nb * RT + tid] + ((pre[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu);
        RS_DCHECK(r < (uint32_t)(RT * KPT));
        dst[r] = k[j];
        if (HAS_VAL) vdst[r] = v[j];
    }
}

template <typename K, bool HAS_VAL, int RT, int KPT>
__device__ __forceinline__ void load_blocked(const K* src, const uint32_t* vsrc, K (&k)[KPT],
                                             uint32_t (&v)[HAS_VAL ? KPT : 1]) {
    const int tid = threadIdx.x;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + (size_t)tid * KPT);
    constexpr int PER = 16 / sizeof(K);
#pragma unroll
    for (int q = 0; q < KPT / PER; ++q) {
        const uint4 x = s4[q];
        const K* xs = reinterpret_cast<const K*>(&x);
#pragma unroll
        for (int e = 0; e < PER; ++e) k[q * PER + e] = xs[e];
    }
    if (HAS_VAL) {
        const uint4* v4 = reinterpret_cast<const uint4*>(vsrc + (size_t)tid * KPT);
#pragma unroll
        for (int q = 0; q < KPT / 4; ++q) {
            const uint4 x = v4[q];
            v[q * 4 + 0] = x.x;
            v[q * 4 + 1] = x.y;
            v[q * 4 + 2] = x.z;
            v[q * 4 + 3] = x.w;
        }
    }
}

template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S>
__global__ void __launch_bounds__(RT, MINB) k_onesweep_cr(PassArgs a) {
    using ST = Status<S>;
    using C = OnesweepCrCfg<K, HAS_VAL, RT, KPT>;
    constexpr int R = C::R, W = C::W, TILE = C::TILE, THREADS = RT;
    static_assert(RT >= R, "one thread per digit in the offset / look-back phases");
    extern __shared__ __align__(128) unsigned char smem[];
    K* bufA = reinterpret_cast<K*>(smem + C::a_off);
    K* bufB = reinterpret_cast<K*>(smem + C::b_off);
    uint32_t* vbufA = reinterpret_cast<uint32_t*>(smem + C::va_off);
    uint32_t* vbufB = reinterpret_cast<uint32_t*>(smem + C::vb_off);
    uint16_t* s_cnt = reinterpret_cast<uint16_t*>(smem + C::cnt_off);
    uint32_t* s_wc = reinterpret_cast<uint32_t*>(smem + C::wc_off);
    uint32_t* s_tcnt = reinterpret_cast<uint32_t*>(smem + C::tcnt_off);
    uint32_t* s_gofs = reinterpret_cast<uint32_t*>(smem + C::gofs_off);
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + C::misc_off);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + C::bar_off);

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
    const uint32_t* vsrc = nullptr;
    uint32_t* vdst = nullptr;
    if (HAS_VAL) {
        vsrc = pick<const uint32_t>(ss, a.vals_in, a.vals_out, a.vals_alt);
        vdst = pick<uint32_t>(ds, const_cast<uint32_t*>(a.vals_in), a.vals_out, a.vals_alt);
    }
    const int shift = a.shift;

    auto issue_load = [&](uint32_t t, K* kb, uint32_t* vb) {
        const size_t base = (size_t)t * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        const uint32_t kbytes = (valid * (uint32_t)sizeof(K)) & ~15u;
        const uint32_t vbytes = HAS_VAL ? ((valid * 4u) & ~15u) : 0u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(s_bar, kbytes + vbytes);
        if (kbytes) bulk_g2s(kb, src + base, kbytes, s_bar);
        if (HAS_VAL && vbytes) bulk_g2s(vb, vsrc + base, vbytes, s_bar);
    };

    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        const uint32_t t0 = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
        s_misc[0] = t0;
        if (t0 < a.num_tiles) issue_load(t0, bufA, vbufA);
    }
    for (int i = tid; i < W * R; i += THREADS) s_wc[i] = 0;
    __syncthreads();
    uint32_t tile = s_misc[0];
    uint32_t phase = 0;

    while (tile < a.num_tiles) {
        const size_t base = (size_t)tile * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);

        // ---- [load]
        if (valid < (uint32_t)TILE) {
            const uint32_t kdone = ((valid * (uint32_t)sizeof(K)) & ~15u) / sizeof(K);
            for (uint32_t i = kdone + tid; i < (uint32_t)TILE; i += THREADS)
                bufA[i] = i < valid ? src[base + i] : ~K(0);
            if (HAS_VAL) {
                const uint32_t vdone = ((valid * 4u) & ~15u) / 4;
                for (uint32_t i = vdone + tid; i < (uint32_t)TILE; i += THREADS)
                    vbufA[i] = i < valid ? vsrc[base + i] : 0u;
            }
        }
        mbar_wait_parity(s_bar, phase);
        phase ^= 1u;
        __syncthreads();

        // ---- [count] per-warp histograms (warp-striped reads: conflict-free)
        {
            uint32_t* wc = s_wc + warp * R;
            const K* in = bufA + warp * (TILE / W) + lane;
#pragma unroll 8
            for (int j = 0; j < KPT; ++j) atomicAdd(&wc[digit8<K>(in[j * 32], shift)], 1u);
        }
        __syncthreads();

        // ---- [offset] tile count, in-tile offset; publish; reset warp histograms
        if (tid < R) {
            uint32_t tcnt = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                tcnt += s_wc[w * R + tid];
                s_wc[w * R + tid] = 0;
            }
            uint32_t incl = tcnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_misc[8 + warp] = incl;
            const uint32_t pub = tcnt - (tid == R - 1 ? (uint32_t)TILE - valid : 0u);
            s_tcnt[tid] = pub;
            st_relaxed_gpu(status + (size_t)tile * R + tid, (tile == 0 ? ST::kFlagP : ST::kFlagA) | (S)pub);
        }
        __syncthreads();

        // ---- [sub 1] low nibble, A -> B ; [sub 2] high nibble, B -> A
        {
            K k[KPT];
            uint32_t v[HAS_VAL ? KPT : 1];
            load_blocked<K, HAS_VAL, RT, KPT>(bufA, vbufA, k, v);
            nibble_subpass<K, HAS_VAL, RT, KPT>(k, v, shift, s_cnt, bufB, vbufB, s_misc);
            __syncthreads();
            load_blocked<K, HAS_VAL, RT, KPT>(bufB, vbufB, k, v);
            nibble_subpass<K, HAS_VAL, RT, KPT>(k, v, shift + 4, s_cnt, bufA, vbufA, s_misc);
        }

        // ---- [look-back] one digit per thread, windowed walk
        if (tid < R) {
            S excl = 0;
            if (tile != 0) {
                constexpr int LB = 8;
                const S* sp = status + (size_t)(tile - 1) * R + tid;
                int64_t left = (int64_t)tile;
                bool done = false;
                while (!done) {
                    S vv[LB];
#pragma unroll
                    for (int i = 0; i < LB; ++i) vv[i] = i < left ? ld_relaxed_gpu(sp - (size_t)i * R) : ST::kFlagP;
#pragma unroll
                    for (int i = 0; i < LB; ++i) {
                        if (done) break;
                        while ((vv[i] & (ST::kFlagA | ST::kFlagP)) == 0) {
                            __nanosleep(64);
                            vv[i] = ld_relaxed_gpu(sp - (size_t)i * R);
                        }
                        excl += ST::val(vv[i]);
                        done = (vv[i] & ST::kFlagP) != 0;
                    }
                    sp -= (size_t)LB * R;
                    left -= LB;
                }
                st_relaxed_gpu(status + (size_t)tile * R + tid, ST::kFlagP | (excl + (S)s_tcnt[tid]));
            }
            // in-tile offset of digit tid (exclusive scan of the tile counts)
            uint32_t texcl = 0;
            {
                uint32_t pre = 0;
                for (int w = 0; w < (tid >> 5); ++w) pre += s_misc[8 + w];
                // s_misc[8 + warp] holds the inclusive warp scan total; recover this
                // thread's exclusive value from the tile count
                uint32_t c = s_tcnt[tid] + (tid == R - 1 ? (uint32_t)TILE - valid : 0u);
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                texcl = pre + incl - c;
            }
            s_gofs[tid] = a.bases[a.pass * R + tid] + (uint32_t)excl - texcl;
        }
        __syncthreads();

        // ---- [next] the next tile's load goes into B (free now)
        if (tid == 0) {
            const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
            s_misc[0] = nt;
            if (nt < a.num_tiles) issue_load(nt, bufB, vbufB);
        }

        // ---- [store] from A (sorted by digit)
#pragma unroll 4
        for (uint32_t i = tid; i < valid; i += THREADS) {
            const K key = bufA[i];
            const uint32_t g = s_gofs[digit8<K>(key, shift)] + i;
            RS_DCHECK(g < a.n);
            dst[g] = key;
            if (HAS_VAL) vdst[g] = vbufA[i];
        }
        __syncthreads();
        tile = s_misc[0];
        // swap buffer roles: the next tile is in B
        K* t = bufA;
        bufA = bufB;
        bufB = t;
        uint32_t* tv = vbufA;
        vbufA = vbufB;
        vbufB = tv;
    }
}

}  // namespace rs
