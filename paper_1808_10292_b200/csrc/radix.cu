// Single-GPU LSD radix sort driver: workspace layout and the launch sequence
//   memset(ctrl, hist) -> K1 hist -> K2 plan -> K3 pass × P -> K4 final copy
// for radix 256 (SR4/PR4), and the radix-65536 path
// (PR2) in radix16.cuh.  Everything is enqueued on the
// caller's stream; no host synchronisation (except the one-time lane-order
// probe per device), no allocation.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>

#include "onesweep_ar.cuh"
#include "radix16.cuh"
#include "runtime.h"

namespace rs {

template <int T_, int KPT_, int MINB_>
struct TuneT {
    static constexpr int THREADS = T_, KPT = KPT_, MINB = MINB_;
};

// ---------------------------------------------- design 5 tile configurations
// (threads, keys per thread, min CTAs per SM).  Large tiles amortise the per-tile
// offsets and look-back; measured on B200 per 2^31 u32 pass:
// 256x88x2 4.85 ms beats 256x72x2 4.90, 256x80x2 5.03, 256x96x2 5.77 (keys read
// from global memory twice, count-then-rank: shared memory holds only the sorted
// tile); u64 keys 256x40x2 (per 2^27 pass 0.512 ms vs 256x32 0.525, 256x48 0.545);
// pairs 256x24x2 (0.753 vs 256x20 0.783, 256x28 0.767, 256x32x2 0.898).
#ifndef RS_AR_U32_T
#define RS_AR_U32_T 256
#endif
#ifndef RS_AR_U32_KPT
#define RS_AR_U32_KPT 88
#endif
#ifndef RS_AR_U32_MINB
#define RS_AR_U32_MINB 2
#endif
template <typename K, bool V>
struct TuneAr;
template <>
struct TuneAr<uint32_t, false> : TuneT<RS_AR_U32_T, RS_AR_U32_KPT, RS_AR_U32_MINB> {};
template <>
struct TuneAr<uint64_t, false> : TuneT<256, 40, 2> {};
// pairs re-swept at look-back window 4 (ms per pass at 2^26 / 2^28 / 2^30 pairs): 256x24
// 0.374 / 1.453 / 5.82 (kept); 256x32 0.426 / 1.682 / 6.58 (window 3: 0.420 / 1.640 / 6.40);
// 256x16 0.430 / 1.718 / 6.83; rank batches of 12 flat; scatter batches of 12 0.376 / 1.461 / 5.84;
// rank batches of 4 / 6 and scatter batches of 4 / 6 within +-0.6 % (mixed across sizes): 8 stays
#ifndef RS_AR_P_T
#define RS_AR_P_T 256
#endif
#ifndef RS_AR_P_KPT
#define RS_AR_P_KPT 24
#endif
#ifndef RS_AR_P_MINB
#define RS_AR_P_MINB 2
#endif
template <>
struct TuneAr<uint64_t, true> : TuneT<RS_AR_P_T, RS_AR_P_KPT, RS_AR_P_MINB> {};
template <>
struct TuneAr<uint32_t, true> : TuneT<256, 24, 2> {};
// design 5 for small inputs (fewer than three large tiles per SM): smaller tiles
// keep every SM busy (2^20 u32 keys are 47 tiles of 22528 keys but 256 of 4096)
template <typename K, bool V>
struct TuneArSmall;
template <>
struct TuneArSmall<uint32_t, false> : TuneT<256, 16, 4> {};
template <>
struct TuneArSmall<uint64_t, false> : TuneT<256, 8, 4> {};
template <>
struct TuneArSmall<uint64_t, true> : TuneT<256, 8, 4> {};
template <>
struct TuneArSmall<uint32_t, true> : TuneT<256, 8, 4> {};
// count-then-rank (RANK2 1: no rank registers) for keys-only sorts; pairs keep
// the 16-bit ranks in registers (measured per 2^27 pass: 0.753 vs 0.760 ms)
template <bool V>
struct Rank2 : std::integral_constant<int, V ? 0 : 1> {};

// design 2 (ballot ranks, the probe fallback)
template <typename K, bool V>
struct TuneEc;
template <>
struct TuneEc<uint32_t, false> : TuneT<256, 24, 3> {};
template <>
struct TuneEc<uint64_t, false> : TuneT<256, 12, 3> {};
template <>
struct TuneEc<uint64_t, true> : TuneT<256, 12, 2> {};
template <>
struct TuneEc<uint32_t, true> : TuneT<256, 12, 3> {};

template <typename K, bool V>
static bool small_input(size_t n) {
    const int st = options().small_tiles;
    if (st != 0) return st == 2;
    const size_t big = (size_t)TuneAr<K, V>::THREADS * TuneAr<K, V>::KPT;
    return (n + big - 1) / big < 3 * (size_t)sm_count();  // measured crossover: 2^23 small, 2^24 large (u32)
}

template <typename K, bool V>
static int tile_keys(int design, size_t n = ~size_t(0)) {
    if (design == 2) return TuneEc<K, V>::THREADS * TuneEc<K, V>::KPT;
    if (n != ~size_t(0) && small_input<K, V>(n)) return TuneArSmall<K, V>::THREADS * TuneArSmall<K, V>::KPT;
    return TuneAr<K, V>::THREADS * TuneAr<K, V>::KPT;
}

static int tile_for(int key_bytes, bool has_val, int design, size_t n = ~size_t(0)) {
    if (key_bytes == 4) return has_val ? tile_keys<uint32_t, true>(design, n) : tile_keys<uint32_t, false>(design, n);
    return has_val ? tile_keys<uint64_t, true>(design, n) : tile_keys<uint64_t, false>(design, n);
}

int tile_keys_for(int key_bytes, bool has_val) { return tile_for(key_bytes, has_val, options().pass_design); }

// the tile size the workspace is sized for: design 5 may fall back to design 2
// after its probe, so size for the smaller of the two tiles (more status rows)
static int ws_tile_for(int key_bytes, bool has_val, size_t n) {
    return std::min(tile_for(key_bytes, has_val, 5, n), tile_for(key_bytes, has_val, 2, n));
}

struct Layout8 {
    Ctrl* ctrl;
    uint32_t* hist;
    uint32_t* bases;
    void* status;  // [2][T][256] u32 or u64 words
    void* alt_keys;
    uint32_t* alt_vals;
    size_t T, status_bytes, bytes;
    bool wide;
};

// `ctrl` is always the first carve (offset 0), whatever the tile size
static Layout8 layout8(void* ws, int key_bytes, bool has_val, size_t n, size_t tile) {
    Layout8 L{};
    const int P = key_bytes * 8 / 8;
    L.T = std::max<size_t>(1, (n + tile - 1) / tile);
    L.wide = n > kNarrowStatusMaxN || options().wide_status;  // P values need > 31 bits
    L.status_bytes = L.T * 256 * (L.wide ? 8 : 4);            // one region
    Carver c(ws);
    L.ctrl = static_cast<Ctrl*>(c.take(sizeof(Ctrl)));
    L.hist = static_cast<uint32_t*>(c.take(P * 256 * 4));
    L.bases = static_cast<uint32_t*>(c.take(P * 256 * 4));
    L.status = c.take(2 * L.status_bytes);
    L.alt_keys = c.take(n * key_bytes);
    L.alt_vals = static_cast<uint32_t*>(has_val ? c.take(n * 4) : nullptr);
    L.bytes = c.used();
    return L;
}

size_t local_ws_bytes(int key_bytes, bool has_val, size_t n, int b) {
    if (b == 8) return layout8(nullptr, key_bytes, has_val, n, (size_t)ws_tile_for(key_bytes, has_val, n)).bytes;
    return radix16_ws_bytes(key_bytes, has_val, n);
}

template <typename K, bool V, typename S, bool SMALL>
static rs_status_t launch_pass_ar(const PassArgs& a, size_t T, cudaStream_t st, bool pdl) {
    using TN = typename std::conditional<SMALL, TuneArSmall<K, V>, TuneAr<K, V>>::type;
    using C = OnesweepArCfg<K, V, TN::THREADS, TN::KPT>;
    // look-back window: 8 for keys (measured 2..64 on the small tiles; on the large, ms
    // per pass at u32 2^26 / 2^27 / 2^31 and u64 2^28: window 2 0.157 / 0.293 / 4.404 /
    // 0.966, 3 0.156 / 0.291 / 4.317 / 0.944, 4 0.156 / 0.290 / 4.292 / 0.937, 6 0.156 /
    // 0.290 / 4.285-4.308 / 0.934, 8 0.156 / 0.290 / 4.291-4.298 / 0.935, 16 slower), 4
    // for the pairs' large tiles (ms per pass at 2^26 / 2^28 / 2^30 pairs:
    // window 1 0.416 / 1.635 / 6.49, 2 0.382 / 1.496 / 5.96, 3 0.375 / 1.461 / 5.85,
    // 4 0.374 / 1.453 / 5.82, 6 0.378 / 1.472 / 5.84, 8 0.385 / 1.509 / 5.93,
    // 16 - / 1.541 / -, 32 - / 1.594 / -): their 3.7x more tiles per key make every
    // status row a window loads cost more than the deeper walk it saves
#ifndef RS_AR_LB
#define RS_AR_LB 8
#endif
#ifndef RS_AR_LB_P
#define RS_AR_LB_P 4
#endif
    auto kern = k_onesweep_ar<K, V, TN::THREADS, TN::KPT, TN::MINB, S, Rank2<V>::value,
                              SMALL ? 8 : (V ? RS_AR_LB_P : RS_AR_LB)>;
    int grid_cap = 0;
    rs_status_t s = kernel_setup(reinterpret_cast<const void*>(kern), C::THREADS, C::smem_bytes, &grid_cap);
    if (s != RS_OK) return s;
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    // the previous kernel in the stream is K2 or the previous pass (sort8)
    RS_CUDA_TRY(launch_chain(pdl, kern, dim3(grid), dim3(C::THREADS), C::smem_bytes, st, a));
    return RS_OK;
}

template <typename K, bool V, typename S>
static rs_status_t launch_pass_ec(const PassArgs& a, size_t T, cudaStream_t st) {
    using TN = TuneEc<K, V>;
    using C = OnesweepEcCfg<K, V, TN::THREADS, TN::KPT>;
    auto kern = k_onesweep_ec<K, V, TN::THREADS, TN::KPT, TN::MINB, S>;
    int grid_cap = 0;
    rs_status_t s = kernel_setup(reinterpret_cast<const void*>(kern), C::THREADS, C::smem_bytes, &grid_cap);
    if (s != RS_OK) return s;
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, C::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

// ---------------------------------------------------- design-5 lane-order probe
// Design 5 takes stable ranks from the old values returned by warp-wide shared
// atomicAdd; it is used only on a device where k_rank_probe, run in the shapes of
// the large-tile and small-tile u32 passes, finds the returned values in lane
// order for every same-address group.  Run once per device, on the caller's
// stream, with one host synchronisation; the mismatch counter is in the (zeroed)
// control block.  Never run inside a stream capture: there design 2 is used for
// that call.
static std::mutex g_probe_mu;
static std::map<int, int> g_probe;  // device -> 0 failed / 1 passed

int rank_probe_state() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    std::lock_guard<std::mutex> lk(g_probe_mu);
    auto it = g_probe.find(dev);
    return it == g_probe.end() ? -1 : it->second;
}

template <typename TN>
static rs_status_t launch_probe(uint32_t seed, uint32_t* bad, cudaStream_t st) {
    using C = OnesweepArCfg<uint32_t, false, TN::THREADS, TN::KPT>;  // the pass's shared-memory footprint
    auto kern = k_rank_probe<TN::THREADS, TN::KPT, TN::MINB>;
    int grid_cap = 0;
    rs_status_t s = kernel_setup(reinterpret_cast<const void*>(kern), TN::THREADS, C::smem_bytes, &grid_cap);
    if (s != RS_OK) return s;
    LaunchScope ls("rank_probe", st);
    kern<<<grid_cap * 4, TN::THREADS, C::smem_bytes, st>>>(seed, bad);
    return RS_OK;
}

static std::mutex g_probe_run_mu;  // one probe at a time: concurrent first callers wait for its verdict

static rs_status_t rank_order_ok(Ctrl* ctrl, cudaStream_t st, bool* ok) {
    int dev = 0;
    RS_CUDA_TRY(cudaGetDevice(&dev));
    auto cached = [&]() {
        std::lock_guard<std::mutex> lk(g_probe_mu);
        auto it = g_probe.find(dev);
        if (it == g_probe.end()) return false;
        *ok = it->second == 1;
        return true;
    };
    if (cached()) return RS_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    RS_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
        *ok = false;
        return RS_OK;
    }
    std::lock_guard<std::mutex> run(g_probe_run_mu);
    if (cached()) return RS_OK;  // another thread probed this device meanwhile
    uint32_t* bad = reinterpret_cast<uint32_t*>(&ctrl->pad[0]);
    RS_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(uint32_t), st));
    rs_status_t s = launch_probe<TuneAr<uint32_t, false>>(0x9E3779B9u, bad, st);
    if (s == RS_OK) s = launch_probe<TuneArSmall<uint32_t, false>>(0x7F4A7C15u, bad, st);
    if (s != RS_OK) return s;
    uint32_t h = 1;
    RS_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    RS_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(h), st));
    std::lock_guard<std::mutex> lk(g_probe_mu);
    g_probe[dev] = h == 0 ? 1 : 0;
    *ok = h == 0;
    return RS_OK;
}

template <typename K, bool V>
static rs_status_t launch_pass(const PassArgs& a, size_t T, bool wide, cudaStream_t st, int design, bool pdl) {
    if (design == 2) {
        if (wide) return launch_pass_ec<K, V, uint64_t>(a, T, st);
        return launch_pass_ec<K, V, uint32_t>(a, T, st);
    }
    const bool small = small_input<K, V>(a.n);  // must match tile_keys()
    if (wide) return small ? launch_pass_ar<K, V, uint64_t, true>(a, T, st, pdl) : launch_pass_ar<K, V, uint64_t, false>(a, T, st, pdl);
    return small ? launch_pass_ar<K, V, uint32_t, true>(a, T, st, pdl) : launch_pass_ar<K, V, uint32_t, false>(a, T, st, pdl);
}

template <typename K, int C, int P>
static rs_status_t launch_hist_lp(const K* keys, size_t n, uint32_t* hist, uint32_t* zero_ptr, size_t zero_words,
                                  cudaStream_t st, int first = 0) {
    constexpr int T = 1024;
    constexpr size_t smem = (size_t)P * 256 * C * 4;
    auto kern = k_digit_hist_lp<K, T, C, P>;
    rs_status_t s = kernel_setup(reinterpret_cast<const void*>(kern), T, smem, nullptr);
    if (s != RS_OK) return s;
    LaunchScope ls("hist", st);
    kern<<<sm_count(), T, smem, st>>>(keys, n, hist + (size_t)first * 256, zero_ptr, zero_words, 8 * first);
    return RS_OK;
}

// histograms of passes [first, P) (rows first.. of hist), from one read of the keys;
// lane-private copies: C = 32 for <= 4 passes, 16 for <= 8
template <typename K>
static rs_status_t launch_hist(const K* keys, size_t n, int P, uint32_t* hist, uint32_t* zero_ptr, size_t zero_words,
                               cudaStream_t st, int first = 0) {
    switch (P - first) {
        case 1: return launch_hist_lp<K, 32, 1>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 2: return launch_hist_lp<K, 32, 2>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 3: return launch_hist_lp<K, 32, 3>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 4: return launch_hist_lp<K, 32, 4>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 5: return launch_hist_lp<K, 16, 5>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 6: return launch_hist_lp<K, 16, 6>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 7: return launch_hist_lp<K, 16, 7>(keys, n, hist, zero_ptr, zero_words, st, first);
        case 8: return launch_hist_lp<K, 16, 8>(keys, n, hist, zero_ptr, zero_words, st, first);
        default: return fail(RS_EINVAL, "digit histogram: bad pass count");
    }
}

constexpr size_t kPdlMaxKeys32 = (size_t)1 << 25, kPdlMaxPairs = (size_t)1 << 24, kPdlMaxKeys64 = (size_t)1 << 22;

template <typename K, bool V>
static rs_status_t sort8(const K* keys_in, const uint32_t* vals_in, size_t n, int end_bit, K* out,
                         uint32_t* vout, void* ws, cudaStream_t st, int first_pass = 0,
                         uint32_t* hist_copy = nullptr) {
    const int P = (end_bit + 7) / 8;
    Ctrl* ctrl = static_cast<Ctrl*>(ws);  // first carve of every layout
    int design = options().pass_design;
    if (design == 5 && P > 0) {
        bool ar_ok = false;
        rs_status_t s = rank_order_ok(ctrl, st, &ar_ok);
        if (s != RS_OK) return s;
        if (!ar_ok) design = 2;
    }
    const Layout8 L = layout8(ws, sizeof(K), V, n, (size_t)tile_for(sizeof(K), V, design, n));
    // programmatic dependent launches along K2 -> K3 x P -> K4 (common.cuh) where they
    // were measured to pay (ms per sort never / always, rs_dev_set_option("pdl"), two
    // interleaved reps on one B200, scripts/gpu_pdl_types.sh): u32 keys 2^20 0.073-0.075
    // / 0.063-0.064, 2^22 0.126 / 0.113, 2^24 0.248-0.250 / 0.236-0.239, 2^25 0.403-0.404
    // / 0.396-0.397, 2^26..2^31 equal within noise; pairs 2^20 0.154 / 0.145-0.146, 2^22
    // 0.301 / 0.288-0.289, 2^24 0.908-0.909 / 0.888-0.892, 2^28 equal; u64 keys 2^20 0.150
    // / 0.127-0.128, 2^22 0.305-0.306 / 0.285, but 2^24 0.632 / 0.659-0.660 (slower)
    const size_t pdl_max = sizeof(K) == 4 ? kPdlMaxKeys32 : (V ? kPdlMaxPairs : kPdlMaxKeys64);
    const int pdl_opt = options().pdl;
    const bool pdl = design == 5 && pdl_opt != 1 && (pdl_opt == 2 || n <= pdl_max);
    // the control block and the histograms are adjacent carves: one memset for both
    // (one launch fewer per sort; 2^20 keys: see DESIGN.md §7)
    RS_CUDA_TRY(cudaMemsetAsync(ctrl, 0, (size_t)(reinterpret_cast<char*>(L.hist + (size_t)P * 256) -
                                                   reinterpret_cast<char*>(ctrl)), st));
    // K1 also zeroes the first pass's status region (as u32 words)
    rs_status_t s = launch_hist<K>(keys_in, n, P, L.hist, static_cast<uint32_t*>(L.status), L.status_bytes / 4, st,
                                   first_pass);
    if (s != RS_OK) return s;
    if (hist_copy)
        RS_CUDA_TRY(cudaMemcpyAsync(hist_copy, L.hist + (size_t)first_pass * 256, 256 * 4, cudaMemcpyDeviceToDevice, st));
    {
        LaunchScope ls("plan", st);
        RS_CUDA_TRY(launch_chain(pdl && hist_copy == nullptr, k_plan, dim3(1), dim3(256), 0, st, (const uint32_t*)L.hist,
                                 (uint32_t)n, P, L.bases, L.ctrl,
                                 (const void*)keys_in == (const void*)out ? 1 : 0, first_pass));
    }
    PassArgs a{};
    a.keys_in = keys_in;
    a.keys_out = out;
    a.keys_alt = L.alt_keys;
    a.vals_in = vals_in;
    a.vals_out = vout;
    a.vals_alt = L.alt_vals;
    a.n = (uint32_t)n;
    a.num_tiles = (uint32_t)L.T;
    a.P = P;
    a.ctrl = L.ctrl;
    a.bases = L.bases;
    for (int t = 0; t < P; ++t) {
        a.pass = t;
        a.shift = 8 * t;
        a.status_cur = static_cast<char*>(L.status) + (size_t)(t & 1) * L.status_bytes;
        a.status_next = static_cast<char*>(L.status) + (size_t)((t + 1) & 1) * L.status_bytes;
        s = launch_pass<K, V>(a, L.T, L.wide, st, design, pdl);
        if (s != RS_OK) return s;
    }
    {
        LaunchScope ls("final_copy", st);
        const unsigned grid = (unsigned)std::min<size_t>((n + 4095) / 4096 + 1, (size_t)sm_count() * 8);
        RS_CUDA_TRY(launch_chain(pdl, k_final_copy<K>, dim3(grid), dim3(256), 0, st, (const Ctrl*)L.ctrl,
                                 keys_in, static_cast<const K*>(L.alt_keys), out, vals_in,
                                 (const uint32_t*)L.alt_vals, V ? vout : (uint32_t*)nullptr, n));
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

// ------------------------------------------------------- debug self-check --
// rs_dev_set_option("self_check", 1): after every local sort, one kernel checks on
// the device that the output is nondecreasing in its low end_bit bits (and, for
// pairs, that equal keys carry increasing values when the values are the
// positions, which the caller cannot promise in general: keys only here); the
// host waits for the verdict.  A debug mode, not for timed runs.
template <typename K>
__global__ void k_check_sorted(const K* __restrict__ a, size_t n, K mask, uint32_t* __restrict__ bad) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += (size_t)gridDim.x * blockDim.x)
        if ((a[i - 1] & mask) > (a[i] & mask)) {
            atomicAdd(bad, 1u);
            return;
        }
}

static rs_status_t self_check(int key_bytes, const void* out, size_t n, int end_bit, void* ws, cudaStream_t st) {
    uint32_t* bad = reinterpret_cast<uint32_t*>(&static_cast<Ctrl*>(ws)->pad[1]);
    RS_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, st));
    const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)sm_count() * 8);
    {
        LaunchScope ls("self_check", st);
        if (key_bytes == 4) {
            const uint32_t m = end_bit >= 32 ? ~0u : ((1u << end_bit) - 1u);
            k_check_sorted<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(out), n, m, bad);
        } else {
            const uint64_t m = end_bit >= 64 ? ~0ull : ((1ull << end_bit) - 1ull);
            k_check_sorted<uint64_t><<<grid, 256, 0, st>>>(static_cast<const uint64_t*>(out), n, m, bad);
        }
    }
    uint32_t h = 0;
    RS_CUDA_TRY(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    if (h) return fail(RS_ECUDA, "self_check: the sort's output is not ordered (" + std::to_string(h) + " CTAs saw an inversion)");
    return RS_OK;
}

static rs_status_t local_sort_impl(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int b,
                                   int end_bit, void* out, uint32_t* vout, void* ws, size_t ws_bytes,
                                   cudaStream_t st) {
    const bool V = vals_in != nullptr;
    if (b == 16) return radix16_sort(key_bytes, keys_in, vals_in, n, end_bit, out, vout, ws, ws_bytes, st);
    if (key_bytes == 4) {
        if (V)
            return sort8<uint32_t, true>(static_cast<const uint32_t*>(keys_in), vals_in, n, end_bit,
                                         static_cast<uint32_t*>(out), vout, ws, st);
        return sort8<uint32_t, false>(static_cast<const uint32_t*>(keys_in), nullptr, n, end_bit,
                                      static_cast<uint32_t*>(out), nullptr, ws, st);
    }
    if (V)
        return sort8<uint64_t, true>(static_cast<const uint64_t*>(keys_in), vals_in, n, end_bit,
                                     static_cast<uint64_t*>(out), vout, ws, st);
    return sort8<uint64_t, false>(static_cast<const uint64_t*>(keys_in), nullptr, n, end_bit,
                                  static_cast<uint64_t*>(out), nullptr, ws, st);
}

rs_status_t local_sort(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int b,
                       int end_bit, void* out, uint32_t* vout, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
    if (n == 0) return RS_OK;
    NvtxRange nr(b == 8 ? "rsort.radix256" : "rsort.radix65536");
    rs_status_t s = local_sort_impl(key_bytes, keys_in, vals_in, n, b, end_bit, out, vout, ws, ws_bytes, st);
    if (s == RS_OK && options().self_check) s = self_check(key_bytes, out, n, end_bit, ws, st);
    return s;
}

rs_status_t local_sort_digit(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int pass_t,
                             void* out, uint32_t* vout, void* ws, cudaStream_t st, uint32_t* hist_copy) {
    if (n == 0) {
        if (hist_copy) RS_CUDA_TRY(cudaMemsetAsync(hist_copy, 0, 256 * 4, st));
        return RS_OK;
    }
    const int end_bit = 8 * (pass_t + 1);
    if (key_bytes == 4) {
        if (vals_in)
            return sort8<uint32_t, true>(static_cast<const uint32_t*>(keys_in), vals_in, n, end_bit,
                                         static_cast<uint32_t*>(out), vout, ws, st, pass_t, hist_copy);
        return sort8<uint32_t, false>(static_cast<const uint32_t*>(keys_in), nullptr, n, end_bit,
                                      static_cast<uint32_t*>(out), nullptr, ws, st, pass_t, hist_copy);
    }
    if (vals_in)
        return sort8<uint64_t, true>(static_cast<const uint64_t*>(keys_in), vals_in, n, end_bit,
                                     static_cast<uint64_t*>(out), vout, ws, st, pass_t, hist_copy);
    return sort8<uint64_t, false>(static_cast<const uint64_t*>(keys_in), nullptr, n, end_bit,
                                  static_cast<uint64_t*>(out), nullptr, ws, st, pass_t, hist_copy);
}

rs_status_t digit_histogram(int key_bytes, const void* keys, size_t n, int b, uint32_t* hist, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
    const int P = key_bytes * 8 / b;
    RS_CUDA_TRY(cudaMemsetAsync(hist, 0, (size_t)P * ((size_t)1 << b) * 4, st));
    if (n == 0) return RS_OK;
    if (b == 16) return radix16_histogram(key_bytes, keys, n, hist, st);
    if (key_bytes == 4) return launch_hist<uint32_t>(static_cast<const uint32_t*>(keys), n, P, hist, nullptr, 0, st);
    return launch_hist<uint64_t>(static_cast<const uint64_t*>(keys), n, P, hist, nullptr, 0, st);
}

}  // namespace rs

#ifdef RS_AR_TRACE
// diagnostic builds only (RS_NVCC_DEFINES=-DRS_AR_TRACE): the per-tile phase
// timestamps of the last radix-256 pass launches (scripts/trace_pass.py)
extern "C" __attribute__((visibility("default"))) int rs_dev_trace_copy(void* host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, rs::g_rs_trace, bytes) == cudaSuccess ? 0 : 1;
}
#endif
