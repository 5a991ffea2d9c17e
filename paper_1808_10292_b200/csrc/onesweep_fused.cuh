// Small-input sort as ONE cooperative launch: K1 (all digit histograms, and the
// first pass's status region zeroed), K2 (bases and the ping-pong plan, CTA 0),
// every K3 pass (design 5, small tiles) and K4 (the final copy), separated by
// grid-wide barriers instead of kernel boundaries — the hypothesis being that
// below ~10 M keys a sort is bound by launch gaps rather than by HBM (c1: 2^20
// keys is 1.3 us per pass at the roofline); the same bodies run here as in the
// separate kernels, so results are identical.  Measured on B200 (option
// "small_fused", default off): 2^20 u32 70.8 us vs 73.4 us launched directly, but
// 69 us vs 55 us when the separate kernels are replayed from a CUDA graph: the
// passes themselves (one small tile per CTA, a chain of dependent phases) are the
// cost at this size, not the launches, and the in-kernel K1 (256 threads, 4 lane
// copies) and the grid barriers add to it.
//
// Memory visibility between phases: every phase's global writes (histogram
// atomics, plan, statuses, scattered keys) are ordered before the next phase's
// reads by cooperative_groups' grid.sync(), whose fence/atomic/acquire sequence
// makes them visible grid-wide (L1 lines of the ping-pong buffers included).
#pragma once
#include <cooperative_groups.h>

#include "onesweep_ar.cuh"

namespace rs {

struct FusedArgs {
    PassArgs a;           // buffers, n, num_tiles, ctrl, bases (pass, shift, statuses set per pass)
    uint32_t* hist;       // [P][256], zero on entry (as is ctrl)
    void* status;         // two status regions of status_bytes each
    size_t status_bytes;
    int inplace;
};

template <typename K, bool V, int RT, int KPT, int MINB, bool KREG_, int KSRC, int RANK2, int HC>
__global__ void __launch_bounds__(RT, MINB) k_sort_fused(FusedArgs f) {
    static_assert(RT == 256, "K2 runs one thread per digit on CTA 0");
    constexpr int P = sizeof(K);  // full sort: radix-256 passes
    extern __shared__ __align__(128) uint32_t f_smem[];
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const K* keys_in = static_cast<const K*>(f.a.keys_in);
    digit_hist_lp_body<K, RT, HC, P>(keys_in, f.a.n, f.hist, static_cast<uint32_t*>(f.status), f.status_bytes / 4, 0,
                                     f_smem);
    grid.sync();
    if (blockIdx.x == 0) plan_body(f.hist, f.a.n, P, const_cast<uint32_t*>(f.a.bases), f.a.ctrl, f.inplace, 0);
    grid.sync();
    PassArgs a = f.a;
    for (int t = 0; t < P; ++t) {
        a.pass = t;
        a.shift = 8 * t;
        a.status_cur = static_cast<char*>(f.status) + (size_t)(t & 1) * f.status_bytes;
        a.status_next = static_cast<char*>(f.status) + (size_t)((t + 1) & 1) * f.status_bytes;
        onesweep_ar_body<K, V, RT, KPT, MINB, uint32_t, KREG_, KSRC, RANK2, RS_AR_LB_SMALL>(a);
        grid.sync();
    }
    final_copy_body<K>(a.ctrl, keys_in, static_cast<const K*>(a.keys_alt), static_cast<K*>(a.keys_out), a.vals_in,
                       a.vals_alt, V ? a.vals_out : nullptr, a.n);
}

}  // namespace rs
