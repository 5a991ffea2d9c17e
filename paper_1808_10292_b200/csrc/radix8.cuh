// Radix-256 LSD pass machinery (the paper's PR4/SR4 count-sort round,
// PAPER.md:653-709) re-designed for sm_100a as a single-sweep pass:
//
//   K1 k_digit_hist_lp one HBM read of all keys -> every pass's 256-bin histogram
//                     ("initial counting process", all rounds at once)
//   K2 k_plan         exclusive prefix of the histograms -> bucket bases per pass
//                     and portion, plus the ping-pong plan
//                     (which passes are non-trivial, src/dst of each)
//   K3 k_onesweep_ar  one stable count-sort round: tile
//                     loads -> in-tile stable rank by shared atomics ->
//                     decoupled look-back across tiles for the per-digit tile
//                     offsets (the single-GPU form of PR's p×r counter matrix,
//                     PAPER.md:690-694) -> shared-memory reorder ->
//                     coalesced scatter of bucket runs.
//   K4 k_final_copy   only when the active-pass parity leaves the result in the
//                     scratch buffer (in-place call with an odd number of passes).
//
// Layout in HBM: keys SoA (u32 or u64) + optional u32 values; ping-pong between
// the caller's `out` and the workspace `alt`; look-back status [2][T][256]
// words, flags in the top bits: u32 words (31-bit prefixes) when n <= 2^31,
// u64 words (62-bit counts) otherwise.
#pragma once
#include "common.cuh"

namespace rs {

// look-back status word: 0 = not ready; [0 | 1 | tile count] = aggregate (A);
// [1 | inclusive prefix] = prefix (P).  A tile count is <= TILE; an inclusive
// prefix is <= the digit's total, which is <= n - 1 in every active pass (a
// digit holding all n keys makes the pass trivial and it is skipped), so u32
// words hold every P value for n <= 2^31 (31 value bits).
template <typename S>
struct Status {
    static constexpr S kFlagA = S(1) << (sizeof(S) * 8 - 2);  // tile aggregate available
    static constexpr S kFlagP = S(1) << (sizeof(S) * 8 - 1);  // inclusive prefix available
    static constexpr S kValMask = kFlagA - 1;                 // value bits of an A word
    static constexpr S kPMask = kFlagP - 1;                   // value bits of a P word
    __device__ __forceinline__ static S val(S s) { return s & ((s & kFlagP) ? kPMask : kValMask); }
};
constexpr uint64_t kNarrowStatusMaxN = 1ull << 31;  // u32 status words suffice up to here

enum BufSel : int32_t { kSelIn = 0, kSelOut = 1, kSelAlt = 2 };

struct Ctrl {
    uint32_t tile_ctr[kMaxPasses];  // dynamic tile ids (zeroed before K1)
    int32_t active[kMaxPasses];     // pass t is non-trivial
    int32_t src_sel[kMaxPasses];
    int32_t dst_sel[kMaxPasses];
    int32_t final_copy;             // 0 none, 1 in->out, 2 alt->out
    int32_t num_active;
    int32_t pad[14];
};

// ------------------------------------------------------------------ K1 ----
// K1, lane-private layout: the CTA keeps C copies of every pass's
// histogram and lane l adds to copy l % C, with copy c of digit d at word
// d*C + c, so the 32 lanes of an atomic touch 32/C words per bank at most:
// C = 32 (u32 keys, 4 passes: 128 KB) makes every warp-wide atomic a single
// conflict-free shared-memory wavefront (random digits in one 256-word array
// cost ~3.15 wavefronts); C = 16 (u64 keys, 8 passes: 128 KB) ~2.  One CTA of
// 1024 threads per SM, persistent; each thread loads 16-byte vectors.
template <typename K, int THREADS, int C, int P>
__device__ __forceinline__ void digit_hist_lp_body(const K* __restrict__ keys, size_t n, uint32_t* __restrict__ hist,
                                                   uint32_t* __restrict__ zero_ptr, size_t zero_words, int shift0,
                                                   uint32_t* s_h) {  // s_h: [P][256][C] shared
    const int tid = threadIdx.x, lane = tid & 31;
    const size_t gtid = (size_t)blockIdx.x * THREADS + tid;
    const size_t gstride = (size_t)gridDim.x * THREADS;
    for (size_t i = gtid; i < zero_words; i += gstride) zero_ptr[i] = 0;
    for (int i = tid; i < P * 256 * C; i += THREADS) s_h[i] = 0;
    __syncthreads();
    uint32_t* my = s_h + (lane % C);
    constexpr int VEC = 16 / sizeof(K);
    const size_t nvec = n / VEC;
    const uint4* vbase = reinterpret_cast<const uint4*>(keys);
    auto count = [&](K k) {
#pragma unroll
        for (int t = 0; t < P; ++t) atomicAdd(&my[(t * 256 + digit_of<K>(k, shift0 + 8 * t, 0xFFu)) * C], 1u);
    };
    size_t v = gtid;
    for (; v + 3 * gstride < nvec; v += 4 * gstride) {  // four 16-byte loads in flight
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = __ldg(vbase + v + u * gstride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const K* ks = reinterpret_cast<const K*>(&x[u]);
#pragma unroll
            for (int e = 0; e < VEC; ++e) count(ks[e]);
        }
    }
    for (; v < nvec; v += gstride) {
        uint4 x = __ldg(vbase + v);
        const K* ks = reinterpret_cast<const K*>(&x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) count(ks[e]);
    }
    for (size_t i = nvec * VEC + gtid; i < n; i += gstride) count(keys[i]);
    __syncthreads();
    for (int i = tid; i < P * 256; i += THREADS) {
        uint32_t s = 0;
#pragma unroll
        for (int c = 0; c < C; ++c) s += s_h[i * C + ((c + i) % C)];  // rotated: conflict-free
        if (s) atomicAdd(&hist[i], s);
    }
}

template <typename K, int THREADS, int C, int P>
__global__ void __launch_bounds__(THREADS, 1) k_digit_hist_lp(const K* __restrict__ keys, size_t n,
                                                             uint32_t* __restrict__ hist,
                                                             uint32_t* __restrict__ zero_ptr, size_t zero_words,
                                                             int shift0 = 0) {
    extern __shared__ __align__(16) uint32_t s_hist_lp[];
    pdl_trigger();  // one CTA per SM: K2's single CTA may wait beside it
    digit_hist_lp_body<K, THREADS, C, P>(keys, n, hist, zero_ptr, zero_words, shift0, s_hist_lp);
}

// ------------------------------------------------------------------ K2 ----
// One CTA of 256 threads.  bases[t][d] = Σ_{d'<d} hist[t][d'].
// Pass t is trivial (skipped: it would be the identity permutation) iff one
// bucket holds all n keys.  Then the ping-pong plan: the last active pass writes
// `out`, earlier ones alternate with `alt`, the first reads `in`; an in-place
// call with an odd count ends in `alt` and needs the final copy.
__device__ __forceinline__ void plan_body(const uint32_t* __restrict__ hist, uint32_t n, int P,
                                          uint32_t* __restrict__ bases, Ctrl* __restrict__ ctrl, int inplace,
                                          int first) {  // threads 0..255 of one CTA
    __shared__ uint32_t s_warp[8];
    __shared__ int s_active[kMaxPasses];
    const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
    for (int t = 0; t < P; ++t) {
        const uint32_t tot = hist[t * 256 + d];
        const int full = __syncthreads_or(tot == n);
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        uint32_t pre = 0;
        for (int w = 0; w < warp; ++w) pre += s_warp[w];
        bases[t * 256 + d] = pre + x - tot;  // exclusive over digits
        if (d == 0) s_active[t] = !full && t >= first;  // passes below `first` are not run
        __syncthreads();
    }
    if (d == 0) {
        int k = 0;
        for (int t = 0; t < P; ++t) k += s_active[t];
        // dst of the i-th active pass: OUT if (k-1-i) even else ALT; flipped when
        // in-place with odd k (the first pass must not write its own source).
        const bool flip = inplace && (k % 2 == 1);
        int i = 0, prev = kSelIn;
        for (int t = 0; t < kMaxPasses; ++t) {
            ctrl->active[t] = 0;
            ctrl->src_sel[t] = kSelIn;
            ctrl->dst_sel[t] = kSelIn;
        }
        for (int t = 0; t < P; ++t) {
            ctrl->active[t] = s_active[t];
            if (!s_active[t]) continue;
            bool to_out = ((k - 1 - i) % 2 == 0) != flip;
            int dst = to_out ? kSelOut : kSelAlt;
            ctrl->src_sel[t] = prev;
            ctrl->dst_sel[t] = dst;
            prev = dst;
            ++i;
        }
        ctrl->num_active = k;
        if (k == 0) ctrl->final_copy = inplace ? 0 : 1;
        else ctrl->final_copy = flip ? 2 : 0;
    }
}

__global__ void __launch_bounds__(256) k_plan(const uint32_t* __restrict__ hist, uint32_t n, int P,
                                              uint32_t* __restrict__ bases, Ctrl* __restrict__ ctrl,
                                              int inplace, int first = 0) {
    pdl_wait();
    pdl_trigger();
    plan_body(hist, n, P, bases, ctrl, inplace, first);
}

template <typename T>
__device__ __forceinline__ T* pick(int sel, T* in, T* out, T* alt) {
    return sel == kSelIn ? in : (sel == kSelOut ? out : alt);
}

// ------------------------------------------------------------------ K3 ----
struct PassArgs {
    const void* keys_in;
    void* keys_out;
    void* keys_alt;
    const uint32_t* vals_in;
    uint32_t* vals_out;
    uint32_t* vals_alt;
    uint32_t n;
    uint32_t num_tiles;
    int pass;
    int shift;
    int P;
    Ctrl* ctrl;
    const uint32_t* bases;  // [P][256]
    void* status_cur;       // [T][256] status words, zero on entry
    void* status_next;      // [T][256], cleared here for the next pass
};

// ------------------------------------------------------------------ K4 ----
template <typename K>
__device__ __forceinline__ void final_copy_body(const Ctrl* __restrict__ ctrl, const K* in, const K* alt, K* out,
                                                const uint32_t* vin, const uint32_t* valt, uint32_t* vout,
                                                size_t n) {
    const int fc = ctrl->final_copy;
    if (fc == 0) return;
    const K* s = fc == 1 ? in : alt;
    const uint32_t* vs = fc == 1 ? vin : valt;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int VEC = 16 / sizeof(K);
    const size_t nv = n / VEC;
    for (size_t i = g; i < nv; i += stride)
        reinterpret_cast<uint4*>(out)[i] = reinterpret_cast<const uint4*>(s)[i];
    for (size_t i = nv * VEC + g; i < n; i += stride) out[i] = s[i];
    if (vout) {
        const size_t nv4 = n / 4;
        for (size_t i = g; i < nv4; i += stride)
            reinterpret_cast<uint4*>(vout)[i] = reinterpret_cast<const uint4*>(vs)[i];
        for (size_t i = nv4 * 4 + g; i < n; i += stride) vout[i] = vs[i];
    }
}

template <typename K>
__global__ void k_final_copy(const Ctrl* __restrict__ ctrl, const K* in, const K* alt, K* out,
                             const uint32_t* vin, const uint32_t* valt, uint32_t* vout, size_t n) {
    pdl_wait();
    final_copy_body<K>(ctrl, in, alt, out, vin, valt, vout, n);
}

}  // namespace rs
