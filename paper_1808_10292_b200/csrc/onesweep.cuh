// K3 k_onesweep — one stable count-sort round of radix 256 (PAPER.md:659-663,
// the paper's SR4/PR4 round) as a single sweep over the keys on sm_100a.
//
// Persistent CTAs take tiles in order from an atomic counter (so every tile a
// CTA waits on belongs to a CTA that is already running).  Per tile:
//   a1 stage: one 1-D bulk copy per array (TMA engine, mbarrier completion)
//      into shared memory; ragged tail by scalar loads, padded with all-ones keys
//      (they sort last in the last bucket and are never stored)
//   a5 rank: keys warp-striped (warp w owns a contiguous 32·KPT slice, lane l
//      its j-th key at w·32·KPT + 32j + l, so (w, j, l) order = input order);
//      peers with the same digit from 8 ballots (or match.any), rank =
//      per-warp running count + popc(peers below me); the group's highest lane
//      advances the count: stable within the warp
//   a2/a3 tile histogram = Σ over warps; per-digit warp offsets (scan over
//      warps) and in-tile digit offsets (scan over digits)
//   a4 decoupled look-back, one thread per digit: publish the tile count
//      (flag A), walk back over predecessors adding aggregates until an
//      inclusive prefix (flag P) is found, publish own inclusive prefix.  This is
//      the single-GPU form of PR's p×r counter gather/scatter
//      and of SPEC.md:206's rank term Σ_{k'<k} count(k', d).
//   a5 reorder + store: keys (values) scattered to their in-tile sorted slot in
//      shared memory; then consecutive threads store consecutive slots, so each
//      bucket run leaves as a coalesced burst at base[d] + prefix[d] + offset.
#pragma once
#include "radix8.cuh"

namespace rs {

template <typename K, bool HAS_VAL, int THREADS, int KPT, int CS = 1>
struct OnesweepCfg {
    // CS: words per (warp, digit) counter slot — 1: count; 2: (peer mask, count)
    static constexpr int R = 256;
    static constexpr int W = THREADS / 32;
    static constexpr int WK = 32 * KPT;  // keys per warp
    static constexpr int TILE = THREADS * KPT;
    static constexpr size_t keys_off = 0;
    static constexpr size_t vals_off = (size_t)TILE * sizeof(K);
    static constexpr size_t wcnt_off = vals_off + (HAS_VAL ? (size_t)TILE * 4 : 0);
    static constexpr size_t texcl_off = wcnt_off + (size_t)W * R * 4 * CS;
    static constexpr size_t gofs_off = texcl_off + R * 4;
    static constexpr size_t misc_off = gofs_off + R * 4;
    static constexpr size_t bar_off = misc_off + 64 * 4;
    static constexpr size_t smem_bytes = bar_off + 16;
    static_assert(WK <= 65535, "packed 16-bit ranks");
};

// lanes of this warp whose 8-bit digit equals mine
template <int VARIANT>
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
    if (VARIANT == 1) return __match_any_sync(0xffffffffu, d);
    // per bit b: p = bit b of d; m = ballot(p); peers &= p ? m : ~m
    uint32_t peers;
    asm("{\n"
        ".reg .pred p;\n"
        ".reg .b32 t, m;\n"
        "mov.b32 %0, 0xffffffff;\n"
#define RS_PEER_BIT(B)                             \
    "and.b32 t, %1, " #B ";\n"                     \
    "setp.ne.u32 p, t, 0;\n"                       \
    "vote.sync.ballot.b32 m, p, 0xffffffff;\n"     \
    "@!p not.b32 m, m;\n"                          \
    "and.b32 %0, %0, m;\n"
        RS_PEER_BIT(1) RS_PEER_BIT(2) RS_PEER_BIT(4) RS_PEER_BIT(8)
        RS_PEER_BIT(16) RS_PEER_BIT(32) RS_PEER_BIT(64) RS_PEER_BIT(128)
#undef RS_PEER_BIT
        "}\n"
        : "=r"(peers)
        : "r"(d));
    return peers;
}

template <typename K, bool HAS_VAL, int THREADS, int KPT, int MINB, int VARIANT, typename S>
__global__ void __launch_bounds__(THREADS, MINB) k_onesweep(PassArgs a) {
    using ST = Status<S>;
    constexpr int CS = VARIANT == 2 ? 2 : 1;
    using C = OnesweepCfg<K, HAS_VAL, THREADS, KPT, CS>;
    constexpr int R = C::R, W = C::W, WK = C::WK, TILE = C::TILE;
    static_assert(THREADS >= R, "one thread per digit in the scan/look-back phase");
    extern __shared__ __align__(128) unsigned char smem[];
    K* s_keys = reinterpret_cast<K*>(smem + C::keys_off);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem + C::vals_off);
    uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(smem + C::wcnt_off);
    uint32_t* s_texcl = reinterpret_cast<uint32_t*>(smem + C::texcl_off);
    uint32_t* s_gofs = reinterpret_cast<uint32_t*>(smem + C::gofs_off);
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + C::misc_off);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + C::bar_off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;

    // Clear the next pass's status rows (stream order publishes them to the
    // next launch; nobody reads them in this one).
    S* const status_cur = static_cast<S*>(a.status_cur);
    if (tid < R)
        for (size_t row = blockIdx.x; row < a.num_tiles; row += gridDim.x)
            static_cast<S*>(a.status_next)[row * R + tid] = 0;
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
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
    }
    const uint32_t mask = R - 1;
    const int shift = a.shift;
    const uint32_t lt = lanemask_lt(), gt = lanemask_gt();
    uint32_t phase = 0;

    while (true) {
        if (tid == 0) s_misc[0] = atomicAdd(&ctrl->tile_ctr[a.pass], 1u);
        __syncthreads();  // tile id visible; previous tile's smem traffic complete
        const uint32_t tile = s_misc[0];
        if (tile >= a.num_tiles) break;
        const size_t base = (size_t)tile * TILE;
        const uint32_t valid = (uint32_t)min((size_t)TILE, (size_t)a.n - base);

        // ---- a1: stage the tile (bulk copies through the TMA engine)
        const uint32_t kbytes = (valid * (uint32_t)sizeof(K)) & ~15u;
        const uint32_t vbytes = HAS_VAL ? ((valid * 4u) & ~15u) : 0u;
        if (tid == 0) {
            fence_proxy_async_smem();  // generic smem accesses of the last tile before async writes
            mbar_arrive_expect_tx(s_bar, kbytes + vbytes);
            if (kbytes) bulk_g2s(s_keys, src + base, kbytes, s_bar);
            if (HAS_VAL && vbytes) bulk_g2s(s_vals, vsrc + base, vbytes, s_bar);
        }
        for (int i = tid; i < W * R * CS; i += THREADS) s_wcnt[i] = 0;
        if (valid < (uint32_t)TILE) {
            for (uint32_t i = kbytes / sizeof(K) + tid; i < (uint32_t)TILE; i += THREADS)
                s_keys[i] = i < valid ? src[base + i] : ~K(0);
            if (HAS_VAL)
                for (uint32_t i = vbytes / 4 + tid; i < (uint32_t)TILE; i += THREADS)
                    s_vals[i] = i < valid ? vsrc[base + i] : 0u;
        }
        mbar_wait_parity(s_bar, phase);
        phase ^= 1u;
        __syncthreads();

        // ---- a5 (rank)
        K key[KPT];
        uint32_t rk[(KPT + 1) / 2];  // packed 16-bit ranks
#pragma unroll
        for (int j = 0; j < KPT; ++j) key[j] = s_keys[warp * WK + j * 32 + lane];
        // running count of digit d in this warp lives at wc[d * CS + CS - 1]
        uint32_t* wc = s_wcnt + warp * R * CS + (CS - 1);
        if (a.debug_skip & 2) {  // ablation: no ranking
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                if (j & 1) rk[j >> 1] |= (uint32_t)(j * 32 + lane) << 16;
                else rk[j >> 1] = (uint32_t)(j * 32 + lane);
            }
        } else if (VARIANT == 2) {
            // peers by atomic OR of lane bits into a per-warp, per-digit mask word
            // that sits next to the digit's running count: (mask, count) pairs
            uint2* wmc = reinterpret_cast<uint2*>(s_wcnt) + warp * R;
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                const uint32_t d = digit_of<K>(key[j], shift, mask);
                atomicOr(&wmc[d].x, 1u << lane);
                __syncwarp();
                const uint2 mc = wmc[d];
                const uint32_t r = mc.y + __popc(mc.x & lt);
                if (j & 1) rk[j >> 1] |= r << 16;
                else rk[j >> 1] = r;
                __syncwarp();
                if ((mc.x & gt) == 0) wmc[d] = make_uint2(0u, mc.y + __popc(mc.x));
                __syncwarp();
            }
        } else {
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
                const uint32_t d = digit_of<K>(key[j], shift, mask);
                const uint32_t peers = digit_peers<VARIANT>(d);
                const uint32_t cnt = wc[d * CS];
                const uint32_t r = cnt + __popc(peers & lt);
                if (j & 1) rk[j >> 1] |= r << 16;
                else rk[j >> 1] = r;
                __syncwarp();
                if ((peers & gt) == 0) wc[d * CS] = cnt + __popc(peers);
                __syncwarp();
            }
        }
        uint32_t val[HAS_VAL ? KPT : 1];
        if (HAS_VAL) {
#pragma unroll
            for (int j = 0; j < KPT; ++j) val[j] = s_vals[warp * WK + j * 32 + lane];
        }
        __syncthreads();

        // ---- a2/a3: tile histogram, warp offsets, in-tile digit offsets
        uint32_t tcnt = 0, texcl = 0, incl = 0;
        if (tid < R) {
            uint32_t run = 0;
#pragma unroll 4
            for (int w = 0; w < W; ++w) {
                const uint32_t c = s_wcnt[(w * R + tid) * CS + CS - 1];
                s_wcnt[(w * R + tid) * CS + CS - 1] = run;
                run += c;
            }
            tcnt = run;
            incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_misc[8 + warp] = incl;
        }
        __syncthreads();
        uint32_t cnt_pub = 0;
        S* my_status = status_cur + (size_t)tile * R + tid;
        if (tid < R) {
            uint32_t pre = 0;
            for (int w = 0; w < (tid >> 5); ++w) pre += s_misc[8 + w];
            texcl = pre + incl - tcnt;
            s_texcl[tid] = texcl;
            cnt_pub = tcnt - (tid == R - 1 ? (uint32_t)TILE - valid : 0u);  // drop the padding
            st_relaxed_gpu(my_status, (tile == 0 ? ST::kFlagP : ST::kFlagA) | (S)cnt_pub);
        }
        __syncthreads();

        // ---- a5 (reorder into shared memory)
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            if (a.debug_skip & 8) break;  // ablation: no reorder
            const uint32_t d = digit_of<K>(key[j], shift, mask);
            const uint32_t r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
            const uint32_t pos = s_texcl[d] + wc[d * CS] + r;
            RS_DCHECK(pos < (uint32_t)TILE);
            s_keys[pos] = key[j];
            if (HAS_VAL) s_vals[pos] = val[j];
        }

        // ---- a4: decoupled look-back
        if (tid < R) {
            S excl = 0;
            if (tile != 0 && (a.debug_skip & 1)) {
                st_relaxed_gpu(my_status, ST::kFlagP | (S)cnt_pub);  // ablation: no look-back
            } else if (tile != 0) {
                // windowed walk: LB predecessors per L2 round trip (tile 0 always
                // holds an inclusive prefix, so the walk never passes it)
                constexpr int LB = 8;
                const S* sp = status_cur + (size_t)(tile - 1) * R + tid;
                int64_t left = (int64_t)tile;  // predecessors not yet visited
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
                st_relaxed_gpu(my_status, ST::kFlagP | (excl + cnt_pub));
            }
            s_gofs[tid] = a.bases[a.pass * R + tid] + (uint32_t)excl - texcl;
        }
        __syncthreads();

        // ---- a5 (store): bucket runs leave as coalesced bursts
#pragma unroll 4
        for (uint32_t i = tid; i < valid; i += THREADS) {
            if (a.debug_skip & 4) break;  // ablation: no global store
            const K k = s_keys[i];
            const uint32_t g = s_gofs[digit_of<K>(k, shift, mask)] + i;
            RS_DCHECK(g < a.n);
            dst[g] = k;
            if (HAS_VAL) vdst[g] = s_vals[i];
        }
    }
}

}  // namespace rs
