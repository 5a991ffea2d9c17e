// Single-GPU LSD radix sort driver: workspace layout and the launch sequence
//   memset(ctrl, hist) -> K1 hist -> K2 plan -> K3 pass × P -> K4 final copy
// for radix 256 (SR4/PR4), and the radix-65536 path
// (PR2) in radix16.cuh.  Everything is enqueued on the
// caller's stream; no host synchronisation, no allocation.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>

#include "onesweep.cuh"
#include "onesweep_ec.cuh"
#include "onesweep_ar.cuh"
#include "onesweep_fused.cuh"
#include "onesweep_ts.cuh"
#include "onesweep_cr.cuh"
#include "onesweep_n4.cuh"
#include "radix16.cuh"
#include "runtime.h"

namespace rs {

// ------------------------------------------------------- tile configurations
// (THREADS, keys per thread, min CTAs per SM); overridable with -D for tuning runs
#ifndef RS_U32_T
#define RS_U32_T 512
#define RS_U32_KPT 12
#define RS_U32_MINB 2
#endif
#define RS_TUNE_U32 RS_U32_T, RS_U32_KPT, RS_U32_MINB
// early-counts design: (ranking threads, keys per thread, min CTAs per SM)
#ifndef RS_EC_U32_T
#define RS_EC_U32_T 256
#define RS_EC_U32_KPT 24
#define RS_EC_U32_MINB 3
#endif
#define RS_EC_U32 RS_EC_U32_T, RS_EC_U32_KPT, RS_EC_U32_MINB
#ifndef RS_EC_U64_T
#define RS_EC_U64_T 256
#define RS_EC_U64_KPT 12
#define RS_EC_U64_MINB 3
#endif
#define RS_EC_U64 RS_EC_U64_T, RS_EC_U64_KPT, RS_EC_U64_MINB
#ifndef RS_EC_PAIRS_T
#define RS_EC_PAIRS_T 256
#define RS_EC_PAIRS_KPT 12
#define RS_EC_PAIRS_MINB 2
#endif
#define RS_EC_PAIRS RS_EC_PAIRS_T, RS_EC_PAIRS_KPT, RS_EC_PAIRS_MINB
#define RS_EC_U32V 256, 12, 3
#define RS_TUNE_U64 512, 8, 2
#define RS_TUNE_PAIRS 512, 8, 2
#define RS_TUNE_U32V 512, 8, 2
template <int T_, int KPT_, int MINB_>
struct TuneT {
    static constexpr int THREADS = T_, KPT = KPT_, MINB = MINB_;
};
template <typename K, bool V>
struct Tune;
template <>
struct Tune<uint32_t, false> : TuneT<RS_TUNE_U32> {};
template <>
struct Tune<uint64_t, false> : TuneT<RS_TUNE_U64> {};
template <>
struct Tune<uint64_t, true> : TuneT<RS_TUNE_PAIRS> {};
template <>
struct Tune<uint32_t, true> : TuneT<RS_TUNE_U32V> {};

constexpr int kHistThreads = 512;

template <typename K, bool V>
struct TuneEc;
template <>
struct TuneEc<uint32_t, false> : TuneT<RS_EC_U32> {};
template <>
struct TuneEc<uint64_t, false> : TuneT<RS_EC_U64> {};
template <>
struct TuneEc<uint64_t, true> : TuneT<RS_EC_PAIRS> {};
template <>
struct TuneEc<uint32_t, true> : TuneT<RS_EC_U32V> {};

// counter-ranking design (3): (threads, keys per thread, min CTAs per SM)
#ifndef RS_CR_U32_T
#define RS_CR_U32_T 256
#define RS_CR_U32_KPT 24
#define RS_CR_U32_MINB 3
#endif
#ifndef RS_CR_U64_T
#define RS_CR_U64_T 256
#define RS_CR_U64_KPT 12
#define RS_CR_U64_MINB 3
#endif
#ifndef RS_CR_PAIRS_T
#define RS_CR_PAIRS_T 256
#define RS_CR_PAIRS_KPT 12
#define RS_CR_PAIRS_MINB 2
#endif
template <typename K, bool V>
struct TuneCr;
template <>
struct TuneCr<uint32_t, false> : TuneT<RS_CR_U32_T, RS_CR_U32_KPT, RS_CR_U32_MINB> {};
template <>
struct TuneCr<uint64_t, false> : TuneT<RS_CR_U64_T, RS_CR_U64_KPT, RS_CR_U64_MINB> {};
template <>
struct TuneCr<uint64_t, true> : TuneT<RS_CR_PAIRS_T, RS_CR_PAIRS_KPT, RS_CR_PAIRS_MINB> {};
template <>
struct TuneCr<uint32_t, true> : TuneT<256, 12, 3> {};

// register-nibble-counter design (4)
#ifndef RS_N4_U32_T
#define RS_N4_U32_T 256
#define RS_N4_U32_KPT 24
#define RS_N4_U32_MINB 3
#endif
template <typename K, bool V>
struct TuneN4;
template <>
struct TuneN4<uint32_t, false> : TuneT<RS_N4_U32_T, RS_N4_U32_KPT, RS_N4_U32_MINB> {};
template <>
struct TuneN4<uint64_t, false> : TuneT<256, 12, 3> {};
template <>
struct TuneN4<uint64_t, true> : TuneT<256, 12, 2> {};
template <>
struct TuneN4<uint32_t, true> : TuneT<256, 12, 3> {};

// atomic-rank design (5): (threads, keys per thread, min CTAs per SM).  Large
// tiles amortise the per-tile offsets and look-back (measured on B200, 2^27 and
// 2^31 keys).  u32, input tile by TMA: 256x48 with 2 CTAs/SM beats 256x24x3,
// 256x30x3, 256x40x2, 256x64x1, 256x96x1, 512x20x2, 512x24x1, 512x32x1; u32 with
// the keys read from global memory twice and count-then-rank (no s_in, no rank
// registers): 256x88x2 (4.85 ms per 2^31 pass) beats 256x48x2 with TMA (5.14),
// 256x72x2 (4.90), 256x80x2 (5.03), 256x96x2 (5.77); pairs 256x32x1 beats
// 256x12x2, 256x16x2, 256x24x1; u64 keys 256x24x2 beats 256x12x3, 512x12x1)
template <typename K, bool V>
struct TuneAr;
#ifndef RS_AR_U32_MINB
#define RS_AR_U32_MINB 2
#endif
// where keys-only passes take their keys (onesweep_ar.cuh KSRC): 0 TMA tile in
// shared memory, 1 registers, 2 global memory twice.  Measured per 2^27 pass:
// u64 KSRC 0 -> 1 0.576 -> 0.533 ms; u32 at 256x48 KSRC 1 no gain (register-bound)
#ifndef RS_AR_KSRC_U32
#define RS_AR_KSRC_U32 2  // u32 keys: from global memory twice (no input tile in shared memory)
#endif
#ifndef RS_AR_KSRC_PAIRS
#define RS_AR_KSRC_PAIRS 2  // pairs: keys and values from global memory (TMA tile 256x32x1: 0.801 ms per
                            // 2^27 pass; global 256x24x2: 0.753; with RANK2 0.760; 256x28x2 0.767; 256x32x2 0.898)
#endif
#ifndef RS_AR_RANK2_PAIRS
#define RS_AR_RANK2_PAIRS 0
#endif
#ifndef RS_AR_RANK2_U64
#define RS_AR_RANK2_U64 1
#endif
#ifndef RS_AR_RANK2_U32
#define RS_AR_RANK2_U32 1  // u32 keys: count-then-rank scatter (onesweep_ar.cuh RANK2): no rank registers
#endif
#ifndef RS_AR_KSRC_U64
#define RS_AR_KSRC_U64 2  // measured per 2^27 pass: KSRC 1 at 256x24 0.534 ms; KSRC 2 + RANK2 at 256x40 0.516
#endif
#ifndef RS_AR_KREG
#define RS_AR_KREG 2  // 0 never, 1 always, 2 with values (pairs: 2 CTAs/SM leave room)
#endif
#ifndef RS_AR_U32_KPT
#define RS_AR_U32_KPT 88  // with KSRC 2 + RANK2: shared memory holds only s_out, so the tile can grow
#endif
#ifndef RS_AR_U32_T
#define RS_AR_U32_T 256
#endif
template <>
struct TuneAr<uint32_t, false> : TuneT<RS_AR_U32_T, RS_AR_U32_KPT, RS_AR_U32_MINB> {};
#ifndef RS_AR_U64_T
#define RS_AR_U64_T 256
#define RS_AR_U64_KPT 40
#define RS_AR_U64_MINB 2
#endif
template <>
struct TuneAr<uint64_t, false> : TuneT<RS_AR_U64_T, RS_AR_U64_KPT, RS_AR_U64_MINB> {};
#ifndef RS_AR_PAIRS_T
#define RS_AR_PAIRS_T 256
#define RS_AR_PAIRS_KPT 24
#define RS_AR_PAIRS_MINB 2
#endif
template <>
struct TuneAr<uint64_t, true> : TuneT<RS_AR_PAIRS_T, RS_AR_PAIRS_KPT, RS_AR_PAIRS_MINB> {};
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

template <typename K, bool V>
static bool small_input(size_t n) {
    if (options().small_tiles != 0) return options().small_tiles == 2;
    const size_t big = (size_t)TuneAr<K, V>::THREADS * TuneAr<K, V>::KPT;
    return (n + big - 1) / big < 3 * (size_t)sm_count();  // measured crossover: 2^23 small, 2^24 large (u32)
}

template <typename K, bool V>
static int tile_keys(int design, size_t n = ~size_t(0)) {
    if (design == 5 && n != ~size_t(0) && small_input<K, V>(n))
        return TuneArSmall<K, V>::THREADS * TuneArSmall<K, V>::KPT;
    if (design == 5 || design == 6) return TuneAr<K, V>::THREADS * TuneAr<K, V>::KPT;
    if (design == 4) return TuneN4<K, V>::THREADS * TuneN4<K, V>::KPT;
    if (design == 3) return TuneCr<K, V>::THREADS * TuneCr<K, V>::KPT;
    if (design >= 1) return TuneEc<K, V>::THREADS * TuneEc<K, V>::KPT;  // 1, 2
    return Tune<K, V>::THREADS * Tune<K, V>::KPT;
}

static int tile_for(int key_bytes, bool has_val, int design, size_t n = ~size_t(0)) {
    if (key_bytes == 4) return has_val ? tile_keys<uint32_t, true>(design, n) : tile_keys<uint32_t, false>(design, n);
    return has_val ? tile_keys<uint64_t, true>(design, n) : tile_keys<uint64_t, false>(design, n);
}

int tile_keys_for(int key_bytes, bool has_val) { return tile_for(key_bytes, has_val, options().pass_design); }

// the tile size the workspace is sized for: design 5 may fall back to design 2
// after its probe, so size for the smaller of the two tiles (more status rows)
static int ws_tile_for(int key_bytes, bool has_val, size_t n) {
    const int d = options().pass_design;
    const int t = tile_for(key_bytes, has_val, d, n);
    return (d == 5 || d == 6) ? std::min(t, tile_for(key_bytes, has_val, 2)) : t;
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

template <typename K, bool V, int VARIANT, typename S>
static rs_status_t launch_pass_v(const PassArgs& a, size_t T, cudaStream_t st) {
    using TN = Tune<K, V>;
    using C = OnesweepCfg<K, V, TN::THREADS, TN::KPT, VARIANT == 2 ? 2 : 1>;
    auto kern = k_onesweep<K, V, TN::THREADS, TN::KPT, TN::MINB, VARIANT, S>;
    static int grid_cap = 0;
    if (!grid_cap) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        int per_sm = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TN::THREADS, C::smem_bytes));
        grid_cap = std::max(1, per_sm) * sm_count();
    }
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, TN::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

template <typename K, bool V, typename S, bool LBW, int ME, int RANKV = 0, bool DBG = false, bool COMPACT = false>
static rs_status_t launch_pass_ec(const PassArgs& a, size_t T, cudaStream_t st) {
    using TN = TuneEc<K, V>;
    using C = OnesweepEcCfg<K, V, TN::THREADS, TN::KPT, LBW, COMPACT>;
    auto kern = k_onesweep_ec<K, V, TN::THREADS, TN::KPT, TN::MINB, S, LBW, ME, RANKV, DBG, COMPACT>;
    static int grid_cap = 0;
    if (!grid_cap) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        int per_sm = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::smem_bytes));
        grid_cap = std::max(1, per_sm) * sm_count();
    }
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, C::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

// match-every variants are instantiated for u32 keys only (the tuned case)
template <typename K, bool V, typename S, bool LBW>
static rs_status_t launch_pass_ec_me(const PassArgs& a, size_t T, cudaStream_t st) {
    if (options().debug_skip) return launch_pass_ec<K, V, S, LBW, 0, 0, true>(a, T, st);
    if (options().compact) return launch_pass_ec<K, V, S, LBW, 0, 0, false, true>(a, T, st);
    if (options().rank_variant == 2) return launch_pass_ec<K, V, S, LBW, 0, 1>(a, T, st);
    if (options().rank_variant == 3) return launch_pass_ec<K, V, S, LBW, 0, 2>(a, T, st);
    if (options().rank_variant == 4) return launch_pass_ec<K, V, S, LBW, 0, 3>(a, T, st);
    if (std::is_same<K, uint32_t>::value && !V) {
        switch (options().match_every) {
            case 4: return launch_pass_ec<K, V, S, LBW, 4>(a, T, st);
            case 6: return launch_pass_ec<K, V, S, LBW, 6>(a, T, st);
            case 8: return launch_pass_ec<K, V, S, LBW, 8>(a, T, st);
            default: break;
        }
    }
    return launch_pass_ec<K, V, S, LBW, 0>(a, T, st);
}

template <typename K, typename S>
static rs_status_t launch_pass_ts(const PassArgs& a, size_t T, cudaStream_t st) {
    using TA = TuneAr<K, false>;
    using TN = TuneT<256, TA::THREADS * TA::KPT / 256, TA::MINB>;  // one thread per digit; same tile
    using C = OnesweepTsCfg<K, TN::THREADS, TN::KPT>;
    auto kern = k_onesweep_ts<K, TN::THREADS, TN::KPT, TN::MINB, S>;
    static int grid_cap = 0;
    if (!grid_cap) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        int per_sm = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TN::THREADS, C::smem_bytes));
        grid_cap = std::max(1, per_sm) * sm_count();
    }
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, TN::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

// the whole small-tile sort as one cooperative launch (onesweep_fused.cuh);
// *done = false when the device cannot co-schedule the grid (then the caller
// runs the separate kernels)
template <typename K, bool V>
static rs_status_t launch_sort_fused(const FusedArgs& f, cudaStream_t st, bool* done) {
    using TN = TuneArSmall<K, V>;
    constexpr int KSRC = V ? RS_AR_KSRC_PAIRS : (sizeof(K) == 8 ? RS_AR_KSRC_U64 : RS_AR_KSRC_U32);
    constexpr int RANK2 = V ? RS_AR_RANK2_PAIRS : (sizeof(K) == 4 ? RS_AR_RANK2_U32 : RS_AR_RANK2_U64);
    constexpr int HC = 4;  // K1 lane copies inside the fused kernel (P·256·HC words of shared memory)
    using C = OnesweepArCfg<K, V, TN::THREADS, TN::KPT, KSRC>;
    auto kern = k_sort_fused<K, V, TN::THREADS, TN::KPT, TN::MINB, (RS_AR_KREG == 1 || (RS_AR_KREG == 2 && V)), KSRC,
                             RANK2, HC>;
    constexpr size_t hist_smem = sizeof(K) * 256 * HC * 4;
    constexpr size_t smem = C::smem_bytes > hist_smem ? C::smem_bytes : hist_smem;
    static int grid = -1;
    if (grid < 0) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0, coop = 0, dev = 0;
        RS_CUDA_TRY(cudaGetDevice(&dev));
        RS_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TN::THREADS, smem));
        grid = coop ? per_sm * sm_count() : 0;
    }
    *done = false;
    if (grid <= 0) return RS_OK;
    FusedArgs fa = f;
    void* params[] = {&fa};
    LaunchScope ls("sort_fused", st);
    RS_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3((unsigned)grid),
                                            dim3(TN::THREADS), params, smem, st));
    *done = true;
    return RS_OK;
}

template <typename K, bool V, typename S, bool SMALL>
static rs_status_t launch_pass_ar(const PassArgs& a, size_t T, cudaStream_t st) {
    using TN = typename std::conditional<SMALL, TuneArSmall<K, V>, TuneAr<K, V>>::type;
    constexpr int KSRC = V ? RS_AR_KSRC_PAIRS : (sizeof(K) == 8 ? RS_AR_KSRC_U64 : RS_AR_KSRC_U32);
    constexpr int RANK2 = V ? RS_AR_RANK2_PAIRS : (sizeof(K) == 4 ? RS_AR_RANK2_U32 : RS_AR_RANK2_U64);
    using C = OnesweepArCfg<K, V, TN::THREADS, TN::KPT, KSRC>;
    // look-back window: small inputs run all tiles at once, so a tile's walk
    // crosses many predecessors that have only published aggregates
    constexpr int LB = SMALL ? RS_AR_LB_SMALL : 8;
    auto kern = k_onesweep_ar<K, V, TN::THREADS, TN::KPT, TN::MINB, S, (RS_AR_KREG == 1 || (RS_AR_KREG == 2 && V)), KSRC,
                              RANK2, LB>;
    static int grid_cap = 0;
    if (!grid_cap) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        int per_sm = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::smem_bytes));
        grid_cap = std::max(1, per_sm) * sm_count();
    }
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, C::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

// ---------------------------------------------------- design-5 lane-order probe
// Design 5 takes stable ranks from the old values returned by warp-wide shared
// atomicAdd; it is used only on a device where k_rank_probe finds the returned
// values in lane order for every same-address group (onesweep_ar.cuh).  Run
// once per device, on the caller's stream, with one host synchronisation; the
// counter word is in the (zeroed) control block.  Never run inside a stream
// capture: there design 2 is used for that call.
static std::mutex g_probe_mu;
static std::map<int, int> g_probe;  // device -> 0 failed / 1 passed

int rank_probe_state() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    std::lock_guard<std::mutex> lk(g_probe_mu);
    auto it = g_probe.find(dev);
    return it == g_probe.end() ? -1 : it->second;
}

static rs_status_t rank_order_ok(Ctrl* ctrl, cudaStream_t st, bool* ok) {
    int dev = 0;
    RS_CUDA_TRY(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_probe_mu);
        auto it = g_probe.find(dev);
        if (it != g_probe.end()) {
            *ok = it->second == 1;
            return RS_OK;
        }
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    RS_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
        *ok = false;
        return RS_OK;
    }
    uint32_t* bad = reinterpret_cast<uint32_t*>(&ctrl->pad[0]);  // zeroed with the control block
    {
        LaunchScope ls("rank_probe", st);
        k_rank_probe<<<sm_count() * 4, 256, 0, st>>>(0x9E3779B9u, 64, bad);
    }
    uint32_t h = 1;
    RS_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    std::lock_guard<std::mutex> lk(g_probe_mu);
    g_probe[dev] = h == 0 ? 1 : 0;
    *ok = h == 0;
    return RS_OK;
}

template <typename K, bool V, typename S>
static rs_status_t launch_pass_cr(const PassArgs& a, size_t T, cudaStream_t st) {
    using TN = TuneCr<K, V>;
    using C = OnesweepCrCfg<K, V, TN::THREADS, TN::KPT>;
    auto kern = k_onesweep_cr<K, V, TN::THREADS, TN::KPT, TN::MINB, S>;
    static int grid_cap = 0;
    if (!grid_cap) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        int per_sm = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TN::THREADS, C::smem_bytes));
        grid_cap = std::max(1, per_sm) * sm_count();
    }
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, TN::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

template <typename K, bool V, typename S>
static rs_status_t launch_pass_n4(const PassArgs& a, size_t T, cudaStream_t st) {
    using TN = TuneN4<K, V>;
    using C = OnesweepN4Cfg<K, V, TN::THREADS, TN::KPT>;
    auto kern = k_onesweep_n4<K, V, TN::THREADS, TN::KPT, TN::MINB, S>;
    static int grid_cap = 0;
    if (!grid_cap) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        int per_sm = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TN::THREADS, C::smem_bytes));
        grid_cap = std::max(1, per_sm) * sm_count();
    }
    const unsigned grid = (unsigned)std::min<size_t>(T, (size_t)grid_cap);  // persistent CTAs
    LaunchScope ls("onesweep", st);
    kern<<<grid, TN::THREADS, C::smem_bytes, st>>>(a);
    return RS_OK;
}

template <typename K, bool V>
static rs_status_t launch_pass(const PassArgs& a, size_t T, bool wide, cudaStream_t st, int design) {
    if (design == 6 && !V) {
        if (wide) return launch_pass_ts<K, uint64_t>(a, T, st);
        return launch_pass_ts<K, uint32_t>(a, T, st);
    }
    if (design == 5 || design == 6) {
        const bool small = design == 5 && small_input<K, V>(a.n);  // must match tile_keys()
        if (wide) return small ? launch_pass_ar<K, V, uint64_t, true>(a, T, st) : launch_pass_ar<K, V, uint64_t, false>(a, T, st);
        return small ? launch_pass_ar<K, V, uint32_t, true>(a, T, st) : launch_pass_ar<K, V, uint32_t, false>(a, T, st);
    }
    if (design == 4) {
        if (wide) return launch_pass_n4<K, V, uint64_t>(a, T, st);
        return launch_pass_n4<K, V, uint32_t>(a, T, st);
    }
    if (design == 3) {
        if (wide) return launch_pass_cr<K, V, uint64_t>(a, T, st);
        return launch_pass_cr<K, V, uint32_t>(a, T, st);
    }
    if (design == 1) {
        if (wide) return launch_pass_ec<K, V, uint64_t, true, 0>(a, T, st);
        return launch_pass_ec<K, V, uint32_t, true, 0>(a, T, st);
    }
    if (design == 2) {
        if (wide) return launch_pass_ec_me<K, V, uint64_t, false>(a, T, st);
        return launch_pass_ec_me<K, V, uint32_t, false>(a, T, st);
    }
    const int rv = options().rank_variant;
    if (wide) {
        if (rv == 1) return launch_pass_v<K, V, 1, uint64_t>(a, T, st);
        if (rv == 2) return launch_pass_v<K, V, 2, uint64_t>(a, T, st);
        return launch_pass_v<K, V, 0, uint64_t>(a, T, st);
    }
    if (rv == 1) return launch_pass_v<K, V, 1, uint32_t>(a, T, st);
    if (rv == 2) return launch_pass_v<K, V, 2, uint32_t>(a, T, st);
    return launch_pass_v<K, V, 0, uint32_t>(a, T, st);
}

template <typename K, int C, int P>
static rs_status_t launch_hist_lp(const K* keys, size_t n, uint32_t* hist, uint32_t* zero_ptr, size_t zero_words,
                                  cudaStream_t st, int first = 0) {
    constexpr int T = 1024;
    constexpr size_t smem = (size_t)P * 256 * C * 4;
    auto kern = k_digit_hist_lp<K, T, C, P>;
    static bool attr = false;
    if (!attr) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    LaunchScope ls("hist", st);
    kern<<<sm_count(), T, smem, st>>>(keys, n, hist + (size_t)first * 256, zero_ptr, zero_words, 8 * first);
    return RS_OK;
}

// histograms of passes [first, P) (rows first.. of hist); first > 0 only with
// the lane-private kernel (single-digit rounds of PR4 across GPUs)
template <typename K>
static rs_status_t launch_hist(const K* keys, size_t n, int P, uint32_t* hist,
                               uint32_t* zero_ptr, size_t zero_words, cudaStream_t st, int first = 0) {
    if (first > 0 && !options().hist_shared) {
        const int np = P - first;
        switch (np) {
            case 1: return launch_hist_lp<K, 32, 1>(keys, n, hist, zero_ptr, zero_words, st, first);
            case 2: return launch_hist_lp<K, 32, 2>(keys, n, hist, zero_ptr, zero_words, st, first);
            case 3: return launch_hist_lp<K, 32, 3>(keys, n, hist, zero_ptr, zero_words, st, first);
            case 4: return launch_hist_lp<K, 32, 4>(keys, n, hist, zero_ptr, zero_words, st, first);
            default: break;  // more passes: count from 0 below
        }
    }
    if (!options().hist_shared) {
        // lane-private copies (default): C = 32 for <= 4 passes, 16 for <= 8
        switch (P) {
            case 1: return launch_hist_lp<K, 32, 1>(keys, n, hist, zero_ptr, zero_words, st);
            case 2: return launch_hist_lp<K, 32, 2>(keys, n, hist, zero_ptr, zero_words, st);
            case 3: return launch_hist_lp<K, 32, 3>(keys, n, hist, zero_ptr, zero_words, st);
            case 4: return launch_hist_lp<K, 32, 4>(keys, n, hist, zero_ptr, zero_words, st);
            case 5: return launch_hist_lp<K, 16, 5>(keys, n, hist, zero_ptr, zero_words, st);
            case 6: return launch_hist_lp<K, 16, 6>(keys, n, hist, zero_ptr, zero_words, st);
            case 7: return launch_hist_lp<K, 16, 7>(keys, n, hist, zero_ptr, zero_words, st);
            case 8: return launch_hist_lp<K, 16, 8>(keys, n, hist, zero_ptr, zero_words, st);
            default: return fail(RS_EINVAL, "digit histogram: bad pass count");
        }
    }
    constexpr int COPIES = kHistThreads / 128;
    const size_t smem = (size_t)COPIES * P * 256 * 4;
    auto kern = k_digit_hist<K, kHistThreads>;
    static bool attr_set = false;
    if (!attr_set) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        attr_set = true;
    }
    const size_t want = (n + kHistThreads * 16 - 1) / (kHistThreads * 16);
    const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>(want, (size_t)sm_count() * 4));
    LaunchScope ls("hist", st);
    kern<<<grid, kHistThreads, smem, st>>>(keys, n, P, 8, hist, zero_ptr, zero_words);
    return RS_OK;
}

template <typename K, bool V>
static rs_status_t sort8(const K* keys_in, const uint32_t* vals_in, size_t n, int end_bit, K* out,
                         uint32_t* vout, void* ws, cudaStream_t st, int first_pass = 0,
                         uint32_t* hist_copy = nullptr) {
    const int P = (end_bit + 7) / 8;
    Ctrl* ctrl = static_cast<Ctrl*>(ws);  // first carve of every layout
    RS_CUDA_TRY(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), st));
    int design = options().pass_design;
    if ((design == 5 || design == 6) && P > 0) {
        bool ar_ok = false;
        rs_status_t s = rank_order_ok(ctrl, st, &ar_ok);
        if (s != RS_OK) return s;
        if (!ar_ok) design = 2;
    }
    const Layout8 L = layout8(ws, sizeof(K), V, n, (size_t)tile_for(sizeof(K), V, design, n));
    if (options().small_fused && design == 5 && P == (int)sizeof(K) && first_pass == 0 && !hist_copy && !L.wide &&
        small_input<K, V>(n)) {
        RS_CUDA_TRY(cudaMemsetAsync(L.hist, 0, (size_t)P * 256 * 4, st));
        FusedArgs f{};
        f.a.keys_in = keys_in;
        f.a.keys_out = out;
        f.a.keys_alt = L.alt_keys;
        f.a.vals_in = vals_in;
        f.a.vals_out = vout;
        f.a.vals_alt = L.alt_vals;
        f.a.n = (uint32_t)n;
        f.a.num_tiles = (uint32_t)L.T;
        f.a.P = P;
        f.a.ctrl = L.ctrl;
        f.a.bases = L.bases;
        f.a.debug_skip = options().debug_skip;
        f.hist = L.hist;
        f.status = L.status;
        f.status_bytes = L.status_bytes;
        f.inplace = (const void*)keys_in == (const void*)out ? 1 : 0;
        bool done = false;
        rs_status_t s = launch_sort_fused<K, V>(f, st, &done);
        if (s != RS_OK || done) return s;
    }
    RS_CUDA_TRY(cudaMemsetAsync(L.hist, 0, (size_t)P * 256 * 4, st));
    // K1 also zeroes the first pass's status region (as u32 words)
    rs_status_t s = launch_hist<K>(keys_in, n, P, L.hist, static_cast<uint32_t*>(L.status), L.status_bytes / 4, st,
                                   first_pass);
    if (s != RS_OK) return s;
    if (hist_copy)
        RS_CUDA_TRY(cudaMemcpyAsync(hist_copy, L.hist + (size_t)first_pass * 256, 256 * 4, cudaMemcpyDeviceToDevice, st));
    {
        LaunchScope ls("plan", st);
        k_plan<<<1, 256, 0, st>>>(L.hist, (uint32_t)n, P, L.bases, L.ctrl,
                                  (const void*)keys_in == (const void*)out ? 1 : 0, first_pass);
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
    a.debug_skip = options().debug_skip;
    for (int t = 0; t < P; ++t) {
        a.pass = t;
        a.shift = 8 * t;
        a.status_cur = static_cast<char*>(L.status) + (size_t)(t & 1) * L.status_bytes;
        a.status_next = static_cast<char*>(L.status) + (size_t)((t + 1) & 1) * L.status_bytes;
        s = launch_pass<K, V>(a, L.T, L.wide, st, design);
        if (s != RS_OK) return s;
    }
    {
        LaunchScope ls("final_copy", st);
        const unsigned grid = (unsigned)std::min<size_t>((n + 4095) / 4096 + 1, (size_t)sm_count() * 8);
        k_final_copy<K><<<grid, 256, 0, st>>>(L.ctrl, keys_in, static_cast<const K*>(L.alt_keys), out, vals_in,
                                              L.alt_vals, V ? vout : nullptr, n);
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

rs_status_t local_sort(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int b,
                       int end_bit, void* out, uint32_t* vout, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
    if (n == 0) return RS_OK;
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
