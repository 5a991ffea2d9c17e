// Radix-65536 pass kernels and driver (see radix16.cuh for the design).
#include <algorithm>
#include <type_traits>

#include "radix16.cuh"

namespace rs {

constexpr int kC16Threads = 1024;  // count kernel
constexpr int kS16Threads = 512;   // scatter kernel
constexpr int kS16KPT = 8;
constexpr int kS16Chunk = kS16Threads * kS16KPT;

// ------------------------------------------------------------------ C1 ----
// smem: 32768 u32 words, each holding two 16-bit counters (digit d in word d>>1,
// half d&1).  A round covers at most 65535 keys so no half overflows.
template <typename K>
__global__ void __launch_bounds__(kC16Threads) k16_count(const K* __restrict__ keys, size_t n, int shift,
                                                         size_t part_keys, uint32_t* __restrict__ H) {
    extern __shared__ uint32_t s_cnt[];  // [32768]
    const int tid = threadIdx.x;
    const size_t g = blockIdx.x;
    const size_t lo = g * part_keys;
    const size_t hi = min(n, lo + part_keys);
    uint32_t* Hg = H + g * kR16;
    int round = 0;
    for (size_t r0 = lo; r0 < hi || round == 0; r0 += 65535, ++round) {
        for (int i = tid; i < kR16 / 2; i += kC16Threads) s_cnt[i] = 0;
        __syncthreads();
        const size_t r1 = min(hi, r0 + 65535);
        for (size_t i = r0 + tid; i < r1; i += kC16Threads) {
            const uint32_t d = static_cast<uint32_t>(keys[i] >> shift) & 0xFFFFu;
            atomicAdd(&s_cnt[d >> 1], 1u << ((d & 1) * 16));
        }
        __syncthreads();
        for (int w = tid; w < kR16 / 2; w += kC16Threads) {
            const uint32_t v = s_cnt[w];
            const uint32_t c0 = v & 0xFFFFu, c1 = v >> 16;
            if (round == 0) {
                Hg[2 * w] = c0;
                Hg[2 * w + 1] = c1;
            } else if (v) {
                Hg[2 * w] += c0;
                Hg[2 * w + 1] += c1;
            }
        }
        __syncthreads();
        if (r1 >= hi) break;
    }
}

// ------------------------------------------------------------------ C2 ----
__global__ void __launch_bounds__(256) k16_total(const uint32_t* __restrict__ H, int G, uint32_t* __restrict__ tot) {
    const int d = blockIdx.x * 256 + threadIdx.x;
    uint32_t s = 0;
    for (int g = 0; g < G; ++g) s += H[(size_t)g * kR16 + d];
    tot[d] = s;
}

// ------------------------------------------------------------------ C3 ----
// One CTA: warp w owns digits [2048w, 2048w + 2048); pass 1 sums them with
// coalesced loads (32 consecutive digits per instruction), the 32 warp totals are
// scanned, pass 2 rescans the segment 32 digits at a time (warp inclusive scan +
// running carry) and writes base coalesced.  (Was: thread t scanned digits
// 64t..64t+63 serially, every load instruction touching 32 different lines: 77 us.)
__global__ void __launch_bounds__(1024) k16_scan(const uint32_t* __restrict__ tot, uint32_t* __restrict__ base) {
    __shared__ uint32_t s_w[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int SEG = kR16 / 32, ROUNDS = SEG / 32;
    const uint32_t* t = tot + warp * SEG;
    uint32_t sum = 0;
#pragma unroll 16
    for (int i = 0; i < ROUNDS; ++i) sum += t[32 * i + lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_w[warp] = sum;
    __syncthreads();
    uint32_t carry = 0;
    for (int w = 0; w < warp; ++w) carry += s_w[w];
    uint32_t* bo = base + warp * SEG;
#pragma unroll 8
    for (int i = 0; i < ROUNDS; ++i) {
        const uint32_t v = t[32 * i + lane];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        bo[32 * i + lane] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

// ------------------------------------------------------------------ C4 ----
// also flags partitions with a digit count >= 2^16 (they cannot use 16-bit
// shared-memory running counts in k16_scatter_fast); big[] zeroed beforehand
__global__ void __launch_bounds__(256) k16_offsets(uint32_t* __restrict__ H, int G, const uint32_t* __restrict__ base,
                                                   uint32_t* __restrict__ big) {
    const int d = blockIdx.x * 256 + threadIdx.x;
    uint32_t run = base[d];
    constexpr int B = 8;  // loads in flight per thread (the G-loop is latency-bound)
    for (int g0 = 0; g0 < G; g0 += B) {
        uint32_t h[B];
#pragma unroll
        for (int j = 0; j < B; ++j) h[j] = g0 + j < G ? H[(size_t)(g0 + j) * kR16 + d] : 0u;
#pragma unroll
        for (int j = 0; j < B; ++j) {
            if (g0 + j >= G) break;
            H[(size_t)(g0 + j) * kR16 + d] = run;
            run += h[j];
            if (h[j] >= 65536u) atomicOr(&big[g0 + j], 1u);
        }
    }
}

// ------------------------------------------------------------------ C5 ----
// Block-level stable 8-bit reorder of a chunk held in shared memory
// (A -> B), keys warp-striped, rank by warp ballots, per-digit scan over warps
// and an exclusive scan over the 256 digits.
template <typename K, bool V>
__device__ __forceinline__ void smem_pass8(const K* A, K* B, const uint32_t* VA, uint32_t* VB, int shift,
                                           uint32_t* s_wcnt, uint32_t* s_aux) {
    constexpr int T = kS16Threads, KPT = kS16KPT, W = T / 32, WK = 32 * KPT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < W * 256; i += T) s_wcnt[i] = 0;
    __syncthreads();
    K key[KPT];
    uint32_t rk[KPT];
    uint32_t* wc = s_wcnt + warp * 256;
    const uint32_t lt = lanemask_lt(), gt = lanemask_gt();
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        key[j] = A[warp * WK + j * 32 + lane];
        const uint32_t d = static_cast<uint32_t>(key[j] >> shift) & 0xFFu;
        const uint32_t peers = peers8(d);
        const uint32_t c = wc[d];
        rk[j] = c + __popc(peers & lt);
        __syncwarp();
        if ((peers & gt) == 0) wc[d] = c + __popc(peers);
        __syncwarp();
    }
    uint32_t val[V ? KPT : 1];
    if (V) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) val[j] = VA[warp * WK + j * 32 + lane];
    }
    __syncthreads();
    uint32_t tcnt = 0, incl = 0;
    if (tid < 256) {
        uint32_t run = 0;
        for (int w = 0; w < W; ++w) {
            const uint32_t c = s_wcnt[w * 256 + tid];
            s_wcnt[w * 256 + tid] = run;
            run += c;
        }
        tcnt = incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_aux[warp] = incl;
    }
    __syncthreads();
    if (tid < 256) {
        uint32_t pre = 0;
        for (int w = 0; w < (tid >> 5); ++w) pre += s_aux[w];
        s_aux[32 + tid] = pre + incl - tcnt;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const uint32_t d = static_cast<uint32_t>(key[j] >> shift) & 0xFFu;
        const uint32_t pos = s_aux[32 + d] + wc[d] + rk[j];
        RS_DCHECK(pos < (uint32_t)kS16Chunk);
        B[pos] = key[j];
        if (V) VB[pos] = val[j];
    }
    __syncthreads();
}

template <typename K, bool V>
struct Scatter16Smem {
    static constexpr size_t keysA = 0;
    static constexpr size_t keysB = keysA + (size_t)kS16Chunk * sizeof(K);
    static constexpr size_t valsA = keysB + (size_t)kS16Chunk * sizeof(K);
    static constexpr size_t valsB = valsA + (V ? (size_t)kS16Chunk * 4 : 0);
    static constexpr size_t wcnt = valsB + (V ? (size_t)kS16Chunk * 4 : 0);
    static constexpr size_t aux = wcnt + (size_t)(kS16Threads / 32) * 256 * 4;
    static constexpr size_t goff = aux + (32 + 256) * 4;
    static constexpr size_t segs = goff + (size_t)kS16Chunk * 4;
    static constexpr size_t bytes = segs + 64 * 4;
};

// partitions per SM (> 1: the generic scatter, RS_R16_MINB CTAs per SM).  Measured (ms per
// sort, u32 2^24 / u32 2^27 / pairs 2^24, b = 16): 1 partition per SM (fast path) 1.28 / 17.2
// / 6.54; 2 per SM at 2 CTAs 1.95 / 18.5 / 6.01; 3 at 3 CTAs 2.69 / 20.7 / 6.41; 4 at 2 CTAs
// 2.04 / 18.5 / 5.80 — the G x 65536 offset matrix grows with G (offsets kernel 17 -> 267 us
// at G = 592) and the global running offsets cost more than the concurrency gains: the
// paper's PR2 trade-off once more
#ifndef RS_R16_GX
#define RS_R16_GX 1
#endif
#ifndef RS_R16_MINB
#define RS_R16_MINB 1
#endif
template <typename K, bool V>
__global__ void __launch_bounds__(kS16Threads, RS_R16_MINB)
    k16_scatter(const K* __restrict__ src, K* __restrict__ dst, const uint32_t* __restrict__ vsrc,
                uint32_t* __restrict__ vdst, size_t n, int shift, size_t part_keys, uint32_t* __restrict__ O) {
    using S = Scatter16Smem<K, V>;
    constexpr int T = kS16Threads, KPT = kS16KPT, CH = kS16Chunk;
    extern __shared__ __align__(16) unsigned char smem[];
    K* kA = reinterpret_cast<K*>(smem + S::keysA);
    K* kB = reinterpret_cast<K*>(smem + S::keysB);
    uint32_t* vA = reinterpret_cast<uint32_t*>(smem + S::valsA);
    uint32_t* vB = reinterpret_cast<uint32_t*>(smem + S::valsB);
    uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(smem + S::wcnt);
    uint32_t* s_aux = reinterpret_cast<uint32_t*>(smem + S::aux);
    uint32_t* s_goff = reinterpret_cast<uint32_t*>(smem + S::goff);
    uint32_t* s_seg = reinterpret_cast<uint32_t*>(smem + S::segs);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t g = blockIdx.x;
    const size_t lo = g * part_keys;
    const size_t hi = min(n, lo + part_keys);
    uint32_t* Og = O + g * kR16;

    for (size_t c0 = lo; c0 < hi; c0 += CH) {
        const uint32_t valid = (uint32_t)min((size_t)CH, hi - c0);
        for (uint32_t i = tid; i < (uint32_t)CH; i += T) {
            kA[i] = i < valid ? src[c0 + i] : ~K(0);
            if (V) vA[i] = i < valid ? vsrc[c0 + i] : 0u;
        }
        __syncthreads();
        // stable sort of the chunk by the 16-bit digit: low byte, then high byte
        smem_pass8<K, V>(kA, kB, vA, vB, shift, s_wcnt, s_aux);
        smem_pass8<K, V>(kB, kA, vB, vA, shift + 8, s_wcnt, s_aux);

        // segment starts: blocked arrangement, max-scan of head positions
        const int i0 = tid * KPT;
        uint32_t d[KPT], st[KPT];
        uint32_t prevd = i0 > 0 ? static_cast<uint32_t>(kA[i0 - 1] >> shift) & 0xFFFFu : 0xFFFFFFFFu;
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            d[j] = static_cast<uint32_t>(kA[i0 + j] >> shift) & 0xFFFFu;
            if (d[j] != prevd) run = (uint32_t)(i0 + j) + 1;  // head position + 1 (0 = none yet)
            st[j] = run;
            prevd = d[j];
        }
        uint32_t x = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = max(x, y);
        }
        if (lane == 31) s_seg[warp] = x;
        __syncthreads();
        uint32_t carry = 0;
        for (int w = 0; w < warp; ++w) carry = max(carry, s_seg[w]);
        const uint32_t prev_lane = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane > 0) carry = max(carry, prev_lane);
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            st[j] = (st[j] ? st[j] : carry) - 1;  // segment start of position i0+j
            if ((uint32_t)(i0 + j) == st[j] && (uint32_t)(i0 + j) < valid) s_goff[i0 + j] = Og[d[j]];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const uint32_t i = (uint32_t)(i0 + j);
            if (i >= valid) continue;
            const uint32_t o = s_goff[st[j]] + (i - st[j]);
            RS_DCHECK(o < n);
            dst[o] = kA[i];
            if (V) vdst[o] = vA[i];
            const uint32_t dnext = j + 1 < KPT ? d[j + 1] : (i + 1 < valid ? static_cast<uint32_t>(kA[i + 1] >> shift) & 0xFFFFu : d[j]);
            const bool last = (i + 1 == valid) || dnext != d[j];
            if (last) Og[d[j]] = o + 1;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ C5 (fast) ---
// u32 keys without values: the partition's running count per digit lives in
// shared memory (16-bit; partitions whose count matrix row has an entry
// >= 65536 — skewed data — take the global read-modify-write path), so the
// offset matrix is read-only; chunks are loaded by the TMA engine into a third
// buffer while the current chunk is sorted and written.
struct Scatter16FastSmem {
    static constexpr int CH = kS16Chunk;
    static constexpr size_t cnt16 = 0;                                   // u16[65536]
    static constexpr size_t buf0 = cnt16 + (size_t)kR16 * 2;             // 3 chunk buffers
    static constexpr size_t wcnt = buf0 + 3 * (size_t)CH * 4;
    static constexpr size_t aux = wcnt + (size_t)(kS16Threads / 32) * 256 * 4;
    static constexpr size_t goff = aux + (32 + 256) * 4;
    static constexpr size_t segs = goff + (size_t)CH * 4;
    static constexpr size_t bar = segs + 64 * 4;
    static constexpr size_t bytes = bar + 16;
};

__global__ void __launch_bounds__(kS16Threads, 1)
    k16_scatter_fast(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, size_t n, int shift,
                     size_t part_keys, uint32_t* __restrict__ O, const uint32_t* __restrict__ big) {
    using S = Scatter16FastSmem;
    constexpr int T = kS16Threads, KPT = kS16KPT, CH = S::CH;
    extern __shared__ __align__(128) unsigned char smem[];
    uint16_t* s_cnt = reinterpret_cast<uint16_t*>(smem + S::cnt16);
    uint32_t* bufA = reinterpret_cast<uint32_t*>(smem + S::buf0);
    uint32_t* bufB = bufA + CH;
    uint32_t* bufC = bufB + CH;
    uint32_t* s_wcnt = reinterpret_cast<uint32_t*>(smem + S::wcnt);
    uint32_t* s_aux = reinterpret_cast<uint32_t*>(smem + S::aux);
    uint32_t* s_goff = reinterpret_cast<uint32_t*>(smem + S::goff);
    uint32_t* s_seg = reinterpret_cast<uint32_t*>(smem + S::segs);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + S::bar);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t g = blockIdx.x;
    const size_t lo = g * part_keys;
    const size_t hi = min(n, lo + part_keys);
    uint32_t* Og = O + g * kR16;
    const bool gpath = big[g] != 0;  // some digit count of this partition needs > 16 bits
    if (!gpath)
        for (int i = tid; i < kR16 / 2; i += T) reinterpret_cast<uint32_t*>(s_cnt)[i] = 0;
    auto issue = [&](size_t c0, uint32_t* buf) {
        const uint32_t valid = (uint32_t)min((size_t)CH, hi - c0);
        const uint32_t bytes = (valid * 4u) & ~15u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(s_bar, bytes);
        if (bytes) bulk_g2s(buf, src + c0, bytes, s_bar);
    };
    if (tid == 0) {
        mbar_init(s_bar, 1);
        fence_mbar_init();
        if (lo < hi) issue(lo, bufA);
    }
    __syncthreads();
    uint32_t phase = 0;
    for (size_t c0 = lo; c0 < hi; c0 += CH) {
        const uint32_t valid = (uint32_t)min((size_t)CH, hi - c0);
        if (valid < (uint32_t)CH)
            for (uint32_t i = ((valid * 4u) & ~15u) / 4 + tid; i < (uint32_t)CH; i += T)
                bufA[i] = i < valid ? src[c0 + i] : ~0u;
        mbar_wait_parity(s_bar, phase);
        phase ^= 1u;
        __syncthreads();
        if (tid == 0 && c0 + CH < hi) issue(c0 + CH, bufC);  // prefetch the next chunk
        smem_pass8<uint32_t, false>(bufA, bufB, nullptr, nullptr, shift, s_wcnt, s_aux);
        smem_pass8<uint32_t, false>(bufB, bufA, nullptr, nullptr, shift + 8, s_wcnt, s_aux);

        const int i0 = tid * KPT;
        uint32_t d[KPT], st[KPT];
        uint32_t prevd = i0 > 0 ? (bufA[i0 - 1] >> shift) & 0xFFFFu : 0xFFFFFFFFu;
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            d[j] = (bufA[i0 + j] >> shift) & 0xFFFFu;
            if (d[j] != prevd) run = (uint32_t)(i0 + j) + 1;
            st[j] = run;
            prevd = d[j];
        }
        uint32_t x = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = max(x, y);
        }
        if (lane == 31) s_seg[warp] = x;
        __syncthreads();
        uint32_t carry = 0;
        for (int w = 0; w < warp; ++w) carry = max(carry, s_seg[w]);
        const uint32_t prev_lane = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane > 0) carry = max(carry, prev_lane);
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            st[j] = (st[j] ? st[j] : carry) - 1;
            if ((uint32_t)(i0 + j) == st[j] && (uint32_t)(i0 + j) < valid)
                s_goff[i0 + j] = Og[d[j]] + (gpath ? 0u : (uint32_t)s_cnt[d[j]]);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            const uint32_t i = (uint32_t)(i0 + j);
            if (i >= valid) continue;
            const uint32_t o = s_goff[st[j]] + (i - st[j]);
            RS_DCHECK(o < n);
            dst[o] = bufA[i];
            const uint32_t dnext = j + 1 < KPT ? d[j + 1] : (i + 1 < valid ? (bufA[i + 1] >> shift) & 0xFFFFu : d[j]);
            if ((i + 1 == valid) || dnext != d[j]) {
                if (gpath) Og[d[j]] = o + 1;
                else s_cnt[d[j]] = (uint16_t)(s_cnt[d[j]] + (i - st[j] + 1));
            }
        }
        __syncthreads();
        uint32_t* t = bufA;  // the next chunk is in C
        bufA = bufC;
        bufC = t;
    }
}

// ------------------------------------------------------------ histogram ---
template <typename K>
__global__ void k16_hist_all(const K* __restrict__ keys, size_t n, int P, uint32_t* __restrict__ hist) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const K k = keys[i];
        for (int t = 0; t < P; ++t) atomicAdd(&hist[(size_t)t * kR16 + (static_cast<uint32_t>(k >> (16 * t)) & 0xFFFFu)], 1u);
    }
}

// -------------------------------------------------------------- driver ----
struct Layout16 {
    uint32_t* H;  // [G][65536]
    uint32_t* tot;
    uint32_t* base;
    uint32_t* big;  // [G]
    void* alt_keys;
    uint32_t* alt_vals;
    size_t G, part, bytes;
};

static Layout16 layout16(void* ws, int key_bytes, bool has_val, size_t n) {
    Layout16 L{};
#ifdef RS_R16_G
    L.G = std::min<size_t>((size_t)RS_R16_G, (size_t)sm_count());  // bounded-frontier experiment
#else
    L.G = (size_t)sm_count() * RS_R16_GX;
#endif
    L.part = (n + L.G - 1) / L.G;
    L.part = std::max<size_t>(1, (L.part + kS16Chunk - 1) / kS16Chunk * kS16Chunk);
    L.G = std::max<size_t>(1, (n + L.part - 1) / L.part);
    Carver c(ws);
    L.H = static_cast<uint32_t*>(c.take(L.G * kR16 * 4));
    L.tot = static_cast<uint32_t*>(c.take(kR16 * 4));
    L.base = static_cast<uint32_t*>(c.take(kR16 * 4));
    L.big = static_cast<uint32_t*>(c.take(L.G * 4));
    L.alt_keys = c.take(n * key_bytes);
    L.alt_vals = static_cast<uint32_t*>(has_val ? c.take(n * 4) : nullptr);
    L.bytes = c.used();
    return L;
}

size_t radix16_ws_bytes(int key_bytes, bool has_val, size_t n) { return layout16(nullptr, key_bytes, has_val, n).bytes; }

template <typename K, bool V>
static rs_status_t sort16(const K* in, const uint32_t* vin, size_t n, int end_bit, K* out, uint32_t* vout, void* ws,
                          cudaStream_t st) {
    const Layout16 L = layout16(ws, sizeof(K), V, n);
    const int P = (end_bit + 15) / 16;
    using S = Scatter16Smem<K, V>;
    {
        rs_status_t s = kernel_setup(reinterpret_cast<const void*>(k16_count<K>), kC16Threads, kR16 / 2 * 4, nullptr);
        if (s == RS_OK) s = kernel_setup(reinterpret_cast<const void*>(k16_scatter<K, V>), kS16Threads, S::bytes, nullptr);
        if (s == RS_OK)
            s = kernel_setup(reinterpret_cast<const void*>(k16_scatter_fast), kS16Threads, Scatter16FastSmem::bytes, nullptr);
        if (s != RS_OK) return s;
    }
    K* alt = static_cast<K*>(L.alt_keys);
    // static ping-pong: the last pass writes `out`; an in-place odd count ends in alt + copy
    const bool inplace = (const void*)in == (const void*)out;
    const bool flip = inplace && (P % 2 == 1);
    const K* src = in;
    const uint32_t* vsrc = vin;
    for (int t = 0; t < P; ++t) {
        const bool to_out = ((P - 1 - t) % 2 == 0) != flip;
        K* dst = to_out ? out : alt;
        uint32_t* vdst = V ? (to_out ? vout : L.alt_vals) : nullptr;
        const int shift = 16 * t;
        {
            LaunchScope ls("r16_count", st);
            k16_count<K><<<(unsigned)L.G, kC16Threads, kR16 / 2 * 4, st>>>(src, n, shift, L.part, L.H);
        }
        {
            LaunchScope ls("r16_total", st);
            k16_total<<<kR16 / 256, 256, 0, st>>>(L.H, (int)L.G, L.tot);
        }
        {
            LaunchScope ls("r16_scan", st);
            k16_scan<<<1, 1024, 0, st>>>(L.tot, L.base);
        }
        {
            LaunchScope ls("r16_offsets", st);
            RS_CUDA_TRY(cudaMemsetAsync(L.big, 0, L.G * 4, st));
            k16_offsets<<<kR16 / 256, 256, 0, st>>>(L.H, (int)L.G, L.base, L.big);
        }
        {
            LaunchScope ls("r16_scatter", st);
            if (std::is_same<K, uint32_t>::value && !V && RS_R16_GX == 1)
                k16_scatter_fast<<<(unsigned)L.G, kS16Threads, Scatter16FastSmem::bytes, st>>>(
                    reinterpret_cast<const uint32_t*>(src), reinterpret_cast<uint32_t*>(dst), n, shift, L.part, L.H,
                    L.big);
            else
                k16_scatter<K, V><<<(unsigned)L.G, kS16Threads, S::bytes, st>>>(src, dst, vsrc, vdst, n, shift,
                                                                                 L.part, L.H);
        }
        src = dst;
        vsrc = vdst;
    }
    if (flip) {
        RS_CUDA_TRY(cudaMemcpyAsync(out, alt, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
        if (V) RS_CUDA_TRY(cudaMemcpyAsync(vout, L.alt_vals, n * 4, cudaMemcpyDeviceToDevice, st));
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

rs_status_t radix16_sort(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int end_bit,
                         void* out, uint32_t* vout, void* ws, size_t, cudaStream_t st) {
    if (key_bytes == 4) {
        if (vals_in)
            return sort16<uint32_t, true>(static_cast<const uint32_t*>(keys_in), vals_in, n, end_bit,
                                          static_cast<uint32_t*>(out), vout, ws, st);
        return sort16<uint32_t, false>(static_cast<const uint32_t*>(keys_in), nullptr, n, end_bit,
                                       static_cast<uint32_t*>(out), nullptr, ws, st);
    }
    if (vals_in)
        return sort16<uint64_t, true>(static_cast<const uint64_t*>(keys_in), vals_in, n, end_bit,
                                      static_cast<uint64_t*>(out), vout, ws, st);
    return sort16<uint64_t, false>(static_cast<const uint64_t*>(keys_in), nullptr, n, end_bit,
                                   static_cast<uint64_t*>(out), nullptr, ws, st);
}

rs_status_t radix16_histogram(int key_bytes, const void* keys, size_t n, uint32_t* hist, cudaStream_t st) {
    const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)sm_count() * 8);
    LaunchScope ls("r16_hist", st);
    if (key_bytes == 4)
        k16_hist_all<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(keys), n, 2, hist);
    else
        k16_hist_all<uint64_t><<<grid, 256, 0, st>>>(static_cast<const uint64_t*>(keys), n, 4, hist);
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

}  // namespace rs
