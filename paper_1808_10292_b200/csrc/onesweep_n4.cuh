// K3 (design 4, "register nibble counters") — one stable count-sort round of
// radix 256.  Same tile pipeline as design 2 (TMA prefetch,
// early publication of the tile count, look-back after ranking, coalesced
// store), but the in-tile stable sort by the 8-bit digit is done as two 4-bit
// counting sub-passes whose per-warp bucket counters live in REGISTERS:
//
//   per warp-iteration (32 keys, warp-striped so (warp, j, lane) = input order):
//     4 ballots of the nibble bits; lanes that share my nibble = ~OR_b(m_b ^ s_b)
//     (s_b = my bit b as 0/-1 by PRMT sign-replication); warp rank =
//     shfl(counter, nibble) + popc(peers below me); lane v < 16 holds the count
//     of nibble v so far and adds popc of bucket v's mask (its own constant s_b)
//   then per-warp nibble totals -> offsets over (nibble, warp) -> scatter
//
// Design 2 touches shared memory at random addresses 4 times per key (histogram
// atomic, counter load, counter store, key scatter), each ~3.5-way bank
// conflicted, and was measured shared-memory-bound; here it is 3 (histogram
// atomic, two key scatters), the counters moving to registers and shuffles.
#pragma once
#include "onesweep_ec.cuh"

namespace rs {

template <typename K, bool HAS_VAL, int RT, int KPT>
struct OnesweepN4Cfg {
    static constexpr int R = 256;
    static constexpr int W = RT / 32;
    static constexpr int WK = 32 * KPT;
    static constexpr int TILE = RT * KPT;
    static constexpr size_t in_off = 0;                                   // TMA target, then sub-pass 1 output
    static constexpr size_t out_off = in_off + (size_t)TILE * sizeof(K);  // sub-pass 2 output (sorted tile)
    static constexpr size_t vin_off = out_off + (size_t)TILE * sizeof(K);
    static constexpr size_t vout_off = vin_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t hist_off = vout_off + (HAS_VAL ? (size_t)TILE * 4 : 0);  // [R] tile histogram
    static constexpr size_t nh_off = hist_off + R * 4;                   // [16][W] nibble counts / offsets
    static constexpr size_t texcl_off = nh_off + 16 * W * 4;
    static constexpr size_t tcnt_off = texcl_off + R * 4;
    static constexpr size_t gofs_off = tcnt_off + R * 4;
    static constexpr size_t misc_off = gofs_off + R * 4;
    static constexpr size_t bar_off = misc_off + 64 * 4;
    static constexpr size_t smem_bytes = bar_off + 16;
    static_assert(WK <= 65535, "16-bit packed ranks");
};

// Warp rank of each key by one nibble (bits [nshift, nshift+4)), stable in
// (j, lane) order; rk[] gets the 16-bit warp ranks, returns this lane's count of
// nibble `lane` (valid for lanes < 16).
template <typename K, int KPT>
__device__ __forceinline__ uint32_t nibble_rank(const K (&k)[KPT], int nshift, uint32_t (&rk)[(KPT + 1) / 2],
                                                uint32_t lt, uint32_t sown0, uint32_t sown1, uint32_t sown2,
                                                uint32_t sown3) {
    uint32_t ctr = 0;  // lane v < 16: keys with nibble v in earlier iterations
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const uint32_t nb = static_cast<uint32_t>(k[j] >> nshift) & 0xFu;
        uint32_t dis, bdis;
        asm("{\n"
            ".reg .pred p;\n"
            ".reg .b32 t, s, m, y;\n"
            "mul.lo.u32 y, %2, 0x10204080;\n"
            "mov.b32 %0, 0;\n"
            "mov.b32 %1, 0;\n"
#define RS_NIB_BIT(B, SEL, SOWN)                    \
    "and.b32 t, %2, " #B ";\n"                      \
    "setp.ne.u32 p, t, 0;\n"                        \
    "vote.sync.ballot.b32 m, p, 0xffffffff;\n"      \
    "prmt.b32 s, y, 0, " #SEL ";\n"                 \
    "xor.b32 t, m, s;\n"                            \
    "or.b32 %0, %0, t;\n"                           \
    "xor.b32 t, m, " SOWN ";\n"                     \
    "or.b32 %1, %1, t;\n"
            RS_NIB_BIT(1, 0x8888, "%3") RS_NIB_BIT(2, 0x9999, "%4") RS_NIB_BIT(4, 0xAAAA, "%5")
            RS_NIB_BIT(8, 0xBBBB, "%6")
#undef RS_NIB_BIT
            "}\n"
            : "=r"(dis), "=r"(bdis)
            : "r"(nb), "r"(sown0), "r"(sown1), "r"(sown2), "r"(sown3));
        const uint32_t r = __shfl_sync(0xffffffffu, ctr, nb) + __popc(~dis & lt);
        if (j & 1) rk[j >> 1] |= r << 16;
        else rk[j >> 1] = r;
        ctr += 32u - __popc(bdis);
    }
    return ctr;
}

template <typename K, bool HAS_VAL, int RT, int KPT, int MINB, typename S>
__global__ void __launch_bounds__(RT, MINB) k_onesweep_n4(PassArgs a) {
    using ST = Status<S>;
    using C = OnesweepN4Cfg<K, HAS_VAL, RT, KPT>;
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE, THREADS = RT;
    static_assert(RT >= R, "one thread per digit in the offset / look-back phases");
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_in = reinterpret_cast<K*>(smem + C::in_off);
    K* s_out = reinterpret_cast<K*>(smem + C::out_off);
    uint32_t* s_vin = reinterpret_cast<uint32_t*>(smem + C::vin_off);
    uint32_t* s_vout = reinterpret_cast<uint32_t*>(smem + C::vout_off);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + C::hist_off);
    uint32_t* s_nh = reinterpret_cast<uint32_t*>(smem + C::nh_off);
    uint32_t* s_texcl = reinterpret_cast<uint32_t*>(smem + C::texcl_off);
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
    const uint32_t lt = lanemask_lt();
    // constant masks of this lane's own bucket v = lane & 15 (bit b of v as 0 / -1)
    const uint32_t v = (uint32_t)lane & 15u;
    const uint32_t so0 = 0u - (v & 1u), so1 = 0u - ((v >> 1) & 1u), so2 = 0u - ((v >> 2) & 1u),
                   so3 = 0u - ((v >> 3) & 1u);

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
        if (t0 < a.num_tiles) issue_load(t0, s_in, s_vin);
    }
    if (tid < R) s_hist[tid] = 0;
    __syncthreads();
    uint32_t tile = s_misc[0];
    uint32_t phase = 0;

    // one 4-bit sub-pass: keys from `from` (warp-striped) -> `to` at their stable rank
    auto subpass = [&](const K* from, const uint32_t* vfrom, K* to, uint32_t* vto, int nshift) {
        K k[KPT];
        uint32_t rk[(KPT + 1) / 2];
        uint32_t vv[HAS_VAL ? KPT : 1];
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            k[j] = from[warp * WK + j * 32 + lane];
            if (HAS_VAL) vv[j] = vfrom[warp * WK + j * 32 + lane];
        }
        const uint32_t cnt = nibble_rank<K, KPT>(k, nshift, rk, lt, so0, so1, so2, so3);
        if (lane < 16) s_nh[lane * W + warp] = cnt;
        __syncthreads();  // all keys of `from` read; nibble counts visible
        if (warp == 0) {  // exclusive scan over (nibble, warp): 16*W values
            constexpr int PER = 16 * W / 32;
            uint32_t x[PER], tot = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                x[i] = s_nh[lane * PER + i];
                tot += x[i];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t run = incl - tot;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                s_nh[lane * PER + i] = run;
                run += x[i];
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const uint32_t nb = static_cast<uint32_t>(k[j] >> nshift) & 0xFu;
            const uint32_t pos = s_nh[nb * W + warp] + ((rk[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu);
            RS_DCHECK(pos < (uint32_t)TILE);
            to[pos] = k[j];
            if (HAS_VAL) vto[pos] = vv[j];
        }
        __syncthreads();
    };

    while (tile < a.num_tiles) {
        const size_t base = (size_t)tile * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);
        if (valid < (uint32_t)TILE) {
            const uint32_t kdone = ((valid * (uint32_t)sizeof(K)) & ~15u) / sizeof(K);
            for (uint32_t i = kdone + tid; i < (uint32_t)TILE; i += THREADS) s_in[i] = i < valid ? src[base + i] : ~K(0);
            if (HAS_VAL) {
                const uint32_t vdone = ((valid * 4u) & ~15u) / 4;
                for (uint32_t i = vdone + tid; i < (uint32_t)TILE; i += THREADS)
                    s_vin[i] = i < valid ? vsrc[base + i] : 0u;
            }
        }
        mbar_wait_parity(s_bar, phase);
        phase ^= 1u;
        __syncthreads();

        // ---- [count] tile histogram (for the early publication)
        {
            const K* in = s_in + warp * WK + lane;
#pragma unroll 8
            for (int j = 0; j < KPT; ++j) atomicAdd(&s_hist[digit8<K>(in[j * 32], shift)], 1u);
        }
        __syncthreads();
        // ---- [offset] in-tile digit offsets; publish the tile count
        if (tid < R) {
            const uint32_t tcnt = s_hist[tid];
            s_hist[tid] = 0;
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
            named_barrier_sync(1, R);
            uint32_t pre = 0;
            for (int w = 0; w < (tid >> 5); ++w) pre += s_misc[8 + w];
            s_texcl[tid] = pre + incl - tcnt;
        }
        // (no barrier needed here: the sub-passes below start and end with barriers)

        // ---- [sort] low nibble s_in -> s_out, high nibble s_out -> s_in
        subpass(s_in, s_vin, s_out, s_vout, shift);
        subpass(s_out, s_vout, s_in, s_vin, shift + 4);
        // the sorted tile is in s_in now

        // ---- [look-back]
        if (tid < R) {
            S excl = 0;
            if (tile != 0) {
                constexpr int LB = 8;
                const S* sp = status + (size_t)(tile - 1) * R + tid;
                int64_t left = (int64_t)tile;
                bool done = false;
                while (!done) {
                    S w8[LB];
#pragma unroll
                    for (int i = 0; i < LB; ++i) w8[i] = i < left ? ld_relaxed_gpu(sp - (size_t)i * R) : ST::kFlagP;
#pragma unroll
                    for (int i = 0; i < LB; ++i) {
                        if (done) break;
                        while ((w8[i] & (ST::kFlagA | ST::kFlagP)) == 0) w8[i] = ld_relaxed_gpu(sp - (size_t)i * R);
                        excl += ST::val(w8[i]);
                        done = (w8[i] & ST::kFlagP) != 0;
                    }
                    sp -= (size_t)LB * R;
                    left -= LB;
                }
                st_relaxed_gpu(status + (size_t)tile * R + tid, ST::kFlagP | (excl + (S)s_tcnt[tid]));
            }
            s_gofs[tid] = a.bases[a.pass * R + tid] + (uint32_t)excl - s_texcl[tid];
        }
        __syncthreads();

        // ---- [next] the sorted tile is in s_in; load the next tile into s_out
        if (tid == 0) {
            const uint32_t nt = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
            s_misc[0] = nt;
            if (nt < a.num_tiles) issue_load(nt, s_out, s_vout);
        }
        // ---- [store] from the sorted tile (s_in)
#pragma unroll 4
        for (uint32_t i = tid; i < valid; i += THREADS) {
            const K key = s_in[i];
            const uint32_t g = s_gofs[digit8<K>(key, shift)] + i;
            RS_DCHECK(g < a.n);
            dst[g] = key;
            if (HAS_VAL) vdst[g] = s_vin[i];
        }
        __syncthreads();
        tile = s_misc[0];
        // buffer roles for the next tile: it was loaded into s_out
        K* t = s_in;
        s_in = s_out;
        s_out = t;
        uint32_t* tv = s_vin;
        s_vin = s_vout;
        s_vout = tv;
    }
}

}  // namespace rs
