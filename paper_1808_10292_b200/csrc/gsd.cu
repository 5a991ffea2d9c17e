// GSD (Algorithm 1) across GPUs: one host orchestration over a
// Transport (gsd.h) — NCCL + CUDA IPC between processes, or p threads of one
// process on one GPU — the radix sort for step 1, and these kernels:
//
//   step 1 LocalSorting    local radix sort of the rank's block in place  (radix.cu)
//   step 2 SampleSelection K5 k_gsd_sample: s = r·p composites of X_k at ⌈N·i/s⌉−1,
//                          i = 1..s−1, plus N−1 (reading R10), written behind this
//                          call's header into the rank's sample record; C1: the
//                          records are all-gathered
//   step 3 SplitterSelect  K6 k_gsd_splitters: bitonic sort of the r·p² sample in one
//                          CTA, S_i = T[i·s−1] (R11, R12) — identical on every rank,
//                          so the paper's "Broadcast splitters" is implicit
//   step 4 Split           K7 k_gsd_split: binary search of the composite splitters
//                          (R14) -> |X_{k,j}|, written into the rank's count record
//                          with its peer-buffer records; C2: the count records are
//                          all-gathered, then the call's ONLY host synchronisation
//                          reads every rank's header, counts and peer records
//   step 5 Merging         Y_j from the p runs, ties to the lower source rank (R16):
//                          default: the one-pass p-way merge reads every peer's
//                          X_{k,j} in place (NVLink through the peer mappings) and
//                          writes Y_j once (pwmerge.cu); fallback: an all-to-all of
//                          the zero-copy slices into a receive buffer, then the merge
//                          tree or a stable radix re-sort (the same result, R17).
//
// Every rank runs every exchange whatever its arguments: a rank that failed its
// own validation contributes an empty block (comm-owned buffers), and every rank
// decides the outcome from the same all-gathered headers — argument, setting and
// capacity errors come back identically on every rank, never as a hang.
//
// GER replaces steps 2-3 (Comm::sampling = 1): s·p − 1 keys drawn
// uniformly at random from the concatenation of the sorted blocks (readings R28-R30:
// SplitMix64 counter draws, position ⌊z·n/2^64⌋, with replacement).  Each rank fills
// the draws that fall in its block (k_ger_draw), a max all-reduce assembles the
// sample everywhere, and two stable radix sorts of the (position, draw) and then
// (key, draw) pairs order it by composite (key, rank, pos); S_i is the (i·s)-th
// smallest (k_ger_pick).  GVR (Comm::sampling = 2) splits before
// it sorts: the same random sample drawn from the unsorted blocks, each key's
// destination by a binary search of the composite splitters (k_gvr_dest), a stable
// count-sort by destination, the exchange, then a local radix sort of Y_j (SR4).
// GER and GVR need n over all ranks before their draws, so they exchange the
// headers first (two host synchronisations per call).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "gsd.h"
#include "merge.h"

namespace rs {

// ------------------------------------------------------------------ K5 ----
template <typename K>
__global__ void k_gsd_sample(const K* __restrict__ X, size_t N, uint32_t rank, int s, Comp* __restrict__ out) {
    for (int i = 1 + threadIdx.x + blockIdx.x * blockDim.x; i <= s; i += blockDim.x * gridDim.x) {
        Comp c;
        c.rank = rank;
        if (N == 0) {
            c.key = ~0ull;
            c.pos = kPosInf;
        } else {
            const size_t pos = i < s ? (N * (size_t)i + (size_t)s - 1) / (size_t)s - 1 : N - 1;
            c.key = static_cast<uint64_t>(X[pos]);
            c.pos = (uint32_t)pos;
        }
        out[i - 1] = c;
    }
}

__device__ __forceinline__ bool comp_less(const Comp& a, const Comp& b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.rank != b.rank) return a.rank < b.rank;
    return a.pos < b.pos;
}

// ------------------------------------------------------------------ K6 ----
// the p records of s composites each (record k at recs + k·stride + hdr) sorted in
// shared memory by a bitonic network; S_i = T[i·s − 1]
__global__ void __launch_bounds__(1024) k_gsd_splitters(const unsigned char* __restrict__ recs, size_t stride, int hdr,
                                                        int p, int s, Comp* __restrict__ S) {
    extern __shared__ Comp sT[];
    const int M = p * s;
    int L = 1;
    while (L < M) L <<= 1;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        if (i < M) sT[i] = *reinterpret_cast<const Comp*>(recs + (size_t)(i / s) * stride + hdr + (size_t)(i % s) * 16);
        else sT[i] = Comp{~0ull, 0xFFFFFFFFu, 0xFFFFFFFFu};
    }
    __syncthreads();
    for (int k = 2; k <= L; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    Comp a = sT[i], b = sT[ixj];
                    if (comp_less(b, a) == up) {
                        sT[i] = b;
                        sT[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = 1 + threadIdx.x; i < p; i += blockDim.x) S[i - 1] = sT[(size_t)i * s - 1];
}

// ------------------------------------------------------------------ K7 ----
template <typename K>
__device__ size_t bound(const K* X, size_t N, uint64_t v, bool upper) {
    size_t lo = 0, hi = N;
    while (lo < hi) {
        const size_t mid = (lo + hi) >> 1;
        const uint64_t x = static_cast<uint64_t>(X[mid]);
        if (upper ? (x <= v) : (x < v)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// cut(j) = #{e in X_k : e <=_c S_j}; for S_j = (v, r, q): k < r -> upper_bound(v),
// k > r -> lower_bound(v), k == r -> min(q + 1, N)   (reading R14)
template <typename K>
__global__ void k_gsd_split(const K* __restrict__ X, size_t N, uint32_t rank, int p, const Comp* __restrict__ S,
                            uint64_t* __restrict__ counts) {
    for (int j = threadIdx.x; j < p; j += blockDim.x) {
        auto cut = [&](int jj) -> size_t {
            if (jj <= 0) return 0;
            if (jj >= p) return N;
            const Comp sp = S[jj - 1];
            if (rank < sp.rank) return bound<K>(X, N, sp.key, true);
            if (rank > sp.rank) return bound<K>(X, N, sp.key, false);
            const uint64_t q1 = (uint64_t)sp.pos + 1;
            return (size_t)(q1 < (uint64_t)N ? q1 : (uint64_t)N);
        };
        counts[j] = (uint64_t)(cut(j + 1) - cut(j));
    }
}

// ------------------------------------------------------------------ GER ---
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// draws i < M that land in this rank's block [off, off + N): key and position
// (the other entries are left as they are: zero, for the max all-reduce)
template <typename K>
__global__ void k_ger_draw(const K* __restrict__ X, uint64_t off, size_t N, uint64_t n_total, uint64_t seed, size_t M,
                           uint64_t* __restrict__ key, uint64_t* __restrict__ q) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (size_t)gridDim.x * blockDim.x) {
        const uint64_t qi = __umul64hi(splitmix64_at(seed, i), n_total);
        if (qi >= off && qi - off < N) {
            key[i] = static_cast<uint64_t>(X[qi - off]);
            q[i] = qi;
        }
    }
}

__global__ void k_iota_u32(uint32_t* __restrict__ a, size_t M) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (size_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

__global__ void k_ger_gather(const uint64_t* __restrict__ key, const uint32_t* __restrict__ idx, size_t M,
                             uint64_t* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (size_t)gridDim.x * blockDim.x)
        out[i] = key[idx[i]];
}

// S_j = composite of the (j·s)-th smallest draw: rank = owner of its position
__global__ void k_ger_pick(const uint64_t* __restrict__ key, const uint64_t* __restrict__ q,
                           const uint32_t* __restrict__ order, size_t s, int p, const uint64_t* __restrict__ off,
                           Comp* __restrict__ S) {
    for (int j = 1 + threadIdx.x; j < p; j += blockDim.x) {
        const uint32_t e = order[(size_t)j * s - 1];
        const uint64_t qe = q[e];
        int k = 0;
        while (k + 1 < p && off[k + 1] <= qe) ++k;  // last block starting at or before qe: non-empty, owns qe
        S[j - 1] = Comp{key[e], (uint32_t)k, (uint32_t)(qe - off[k])};
    }
}

// GVR step 3: destination of every key of the unsorted block, j = #{i : S_i <_c (x, rank, q)}
// (p <= 256, checked when the sampling mode is set)
template <typename K>
__global__ void __launch_bounds__(256) k_gvr_dest(const K* __restrict__ X, size_t N, uint32_t rank,
                                                  const Comp* __restrict__ S, int p, uint32_t* __restrict__ dest,
                                                  uint32_t* __restrict__ idx, uint64_t* __restrict__ counts) {
    __shared__ Comp sS[256];
    __shared__ uint64_t sT[256];
    __shared__ uint32_t sc[256];
    // u32 keys: for this rank, S_i <_c (x, rank, q) iff T_i <= (x << 32 | q) with
    // T_i = key_i << 32 + (0 if rank_i < rank, pos_i + 1 if rank_i == rank, 2^32 if
    // rank_i > rank), saturated — one 64-bit threshold per splitter, nondecreasing in i
    constexpr bool kT = sizeof(K) == 4;
    for (int i = threadIdx.x; i < p - 1; i += blockDim.x) {
        const Comp c = S[i];
        sS[i] = c;
        if (kT) {
            const uint64_t thr = c.rank < rank ? 0ull : (c.rank == rank ? (uint64_t)c.pos + 1 : (1ull << 32));
            const uint64_t hi = c.key << 32;
            sT[i] = (c.key >= (1ull << 32) || hi > ~0ull - thr) ? ~0ull : hi + thr;
        }
    }
    for (int i = threadIdx.x; i < p; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    auto dest_of = [&](K x, size_t q) {
        int lo = 0, hi = p - 1;  // count of splitters <_c e (they are sorted)
        if (kT) {
            const uint64_t E = (static_cast<uint64_t>(x) << 32) | (uint32_t)q;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sT[mid] <= E) lo = mid + 1;
                else hi = mid;
            }
        } else {
            const Comp e{static_cast<uint64_t>(x), rank, (uint32_t)q};
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (comp_less(sS[mid], e)) lo = mid + 1;
                else hi = mid;
            }
        }
        atomicAdd(&sc[lo], 1u);
        return (uint32_t)lo;
    };
    // 16-byte vectors of keys (X, dest and idx are 16-byte aligned): VEC keys per load and
    // independent searches per iteration (one key per iteration ran at 2.5 TB/s, latency-bound)
    constexpr int VEC = 16 / sizeof(K);
    const size_t nv = N / VEC, gstride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 2
    for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gstride) {
        const uint4 w = reinterpret_cast<const uint4*>(X)[v];
        const K* ks = reinterpret_cast<const K*>(&w);
        uint32_t dd[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) dd[e] = dest_of(ks[e], v * VEC + e);
        const uint32_t q0 = (uint32_t)(v * VEC);
        if (VEC == 4) {
            reinterpret_cast<uint4*>(dest)[v] = make_uint4(dd[0], dd[VEC > 1 ? 1 : 0], dd[VEC > 2 ? 2 : 0], dd[VEC > 3 ? 3 : 0]);
            if (idx) reinterpret_cast<uint4*>(idx)[v] = make_uint4(q0, q0 + 1, q0 + 2, q0 + 3);
        } else {
            reinterpret_cast<uint2*>(dest)[v] = make_uint2(dd[0], dd[VEC > 1 ? 1 : 0]);
            if (idx) reinterpret_cast<uint2*>(idx)[v] = make_uint2(q0, q0 + 1);
        }
    }
    for (size_t q = nv * VEC + (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += gstride) {
        dest[q] = dest_of(X[q], q);
        if (idx) idx[q] = (uint32_t)q;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < p; i += blockDim.x)
        if (sc[i]) atomicAdd(reinterpret_cast<unsigned long long*>(&counts[i]), (unsigned long long)sc[i]);
}

template <typename K>
__global__ void k_gvr_gather(const K* __restrict__ X, const uint32_t* __restrict__ V, const uint32_t* __restrict__ idx,
                             size_t N, K* __restrict__ outK, uint32_t* __restrict__ outV) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t j = idx[i];
        outK[i] = X[j];
        if (V) outV[i] = V[j];
    }
}

size_t ger_default_s(uint64_t n_total) {
    // s = 2⌈ω⌉²⌈lg n⌉, ω = lg lg n  (reading R30)
    const double lg = n_total > 1 ? std::log2((double)n_total) : 1.0;
    const double w = std::max(1.0, std::ceil(lg > 1.0 ? std::log2(lg) : 1.0));
    return (size_t)(2.0 * w * w * std::ceil(lg));
}

// ------------------------------------------------------------------ host --
struct GsdLayout {
    void* local_ws;
    size_t local_ws_bytes;
    void* recv_keys;         // cap keys: the all-to-all fallback's receive buffer
    uint32_t* recv_vals;
    // GER: M = s·p − 1 draws
    uint64_t* ger_key;   // M
    uint64_t* ger_q;     // M
    uint64_t* ger_k2;    // M (positions in order, then gathered keys)
    uint64_t* ger_k3;    // M (keys in composite order)
    uint32_t* ger_idx;   // M
    uint32_t* ger_ia;    // M
    uint32_t* ger_ib;    // M
    uint64_t* ger_off;   // p + 1 block offsets
    void* ger_ws;        // radix workspace for M (u64, u32) pairs
    size_t ger_ws_bytes, ger_M;
    // GVR: N = local keys
    uint32_t *gv_dest, *gv_idx, *gv_sdest, *gv_sidx;  // N each
    void* gv_keys;                                     // N keys partitioned by destination
    uint32_t* gv_vals;                                 // N
    void* gv_ws;                                       // radix workspace for N (u32, u32) pairs
    size_t gv_ws_bytes;
    void* merge_keys;        // merge scratch: cap keys (+ values); the p-way pass's sample and tables
    uint32_t* merge_vals;
    size_t* merge_split;
    size_t bytes;
};

static GsdLayout gsd_layout(void* ws, int key_bytes, bool has_val, size_t n, size_t cap, int b, int p,
                            size_t ger_M = 0, bool gvr = false) {
    GsdLayout L{};
    Carver c(ws);
    L.local_ws_bytes = local_ws_bytes(key_bytes, has_val, std::max(n, cap), b);
    L.local_ws = c.take(L.local_ws_bytes);
    L.recv_keys = c.take(cap * key_bytes);
    L.recv_vals = static_cast<uint32_t*>(has_val ? c.take(cap * 4) : nullptr);
    L.merge_keys = c.take(cap * key_bytes);
    L.merge_vals = static_cast<uint32_t*>(has_val ? c.take(cap * 4) : nullptr);
    L.merge_split = static_cast<size_t*>(c.take(merge_scratch_bytes(cap)));
    L.ger_M = ger_M;
    if (ger_M) {
        L.ger_key = static_cast<uint64_t*>(c.take(ger_M * 8));
        L.ger_q = static_cast<uint64_t*>(c.take(ger_M * 8));
        L.ger_k2 = static_cast<uint64_t*>(c.take(ger_M * 8));
        L.ger_k3 = static_cast<uint64_t*>(c.take(ger_M * 8));
        L.ger_idx = static_cast<uint32_t*>(c.take(ger_M * 4));
        L.ger_ia = static_cast<uint32_t*>(c.take(ger_M * 4));
        L.ger_ib = static_cast<uint32_t*>(c.take(ger_M * 4));
        L.ger_off = static_cast<uint64_t*>(c.take(((size_t)p + 1) * 8));
        L.ger_ws_bytes = local_ws_bytes(8, true, ger_M, 8);
        L.ger_ws = c.take(L.ger_ws_bytes);
    }
    if (gvr) {
        L.gv_dest = static_cast<uint32_t*>(c.take(std::max<size_t>(n, 1) * 4));
        L.gv_idx = static_cast<uint32_t*>(c.take(std::max<size_t>(n, 1) * 4));
        L.gv_sdest = static_cast<uint32_t*>(c.take(std::max<size_t>(n, 1) * 4));
        L.gv_sidx = static_cast<uint32_t*>(c.take(std::max<size_t>(n, 1) * 4));
        L.gv_keys = c.take(std::max<size_t>(n, 1) * key_bytes);
        L.gv_vals = static_cast<uint32_t*>(has_val ? c.take(std::max<size_t>(n, 1) * 4) : nullptr);
        L.gv_ws_bytes = local_ws_bytes(4, true, n, 8);
        L.gv_ws = c.take(L.gv_ws_bytes);
    }
    L.bytes = c.used();
    return L;
}

// GER draws for n_total keys over p ranks (0 for GSD)
static size_t ger_draws(size_t s, int p) { return p > 1 ? s * (size_t)p - 1 : 0; }

static size_t capacity_for(size_t n_local_max, int r, int p) {
    // ⌊(1 + 1/r)·N_max⌋ + p   (reading R18)
    return n_local_max + n_local_max / (size_t)r + (size_t)p;
}

// GER: Lemma `Sampling1` with ρ = 1 bounds every bucket of the
// non-sample keys by ⌈(1+ε)(n−p+1)/p⌉ with probability ≥ 1 − 1/n, for the smallest
// ε with s ≥ (1+ε)/ε²·(2 ln n + ln(2π p²(ps−1) e^{1/(3(ps−1))})); a bucket also
// holds at most s sample keys.  Capacity = ⌈(1+ε)·N_max⌉ + s + p (n ≤ p·N_max).
static size_t ger_capacity_for(size_t n_local_max, int p, size_t s) {
    const double n = std::max(2.0, (double)n_local_max * p), ps1 = std::max(1.0, (double)s * p - 1);
    const double A = 2.0 * std::log(n) + std::log(2.0 * 3.141592653589793 * p * p * ps1) + 1.0 / (3.0 * ps1);
    const double eps = (A + std::sqrt(A * A + 4.0 * (double)s * A)) / (2.0 * (double)s);  // s·ε² − A·ε − A = 0
    return (size_t)std::ceil((1.0 + eps) * (double)n_local_max) + s + (size_t)p;
}

static size_t ger_s_for(Comm* c, uint64_t n_total) { return c->ger_s ? c->ger_s : ger_default_s(n_total); }

size_t gsd_capacity(Comm* c, size_t n_local_max) {
    if (c->sampling >= 3) return n_local_max;  // PR4 / BTN / OET: rank j ends with exactly its input size
    if (c->sampling >= 1) return ger_capacity_for(n_local_max, c->nranks, ger_s_for(c, (uint64_t)n_local_max * c->nranks));
    return capacity_for(n_local_max, c->r, c->nranks);
}

static size_t ws_need(Comm* c, int key_bytes, bool hv, size_t n, size_t cap, int b, uint64_t n_total) {
    if (c->sampling == 3) return pr_ws_bytes(key_bytes, hv, n, c->nranks);
    if (c->sampling >= 4) return net_ws_bytes(key_bytes, hv, n, b);
    const size_t M = c->sampling >= 1 ? ger_draws(ger_s_for(c, n_total), c->nranks) : 0;
    return gsd_layout(nullptr, key_bytes, hv, n, cap, b, c->nranks, M, c->sampling == 2).bytes;
}

size_t gsd_ws_bytes(Comm* c, int key_bytes, bool has_val, size_t n_local_max, int b) {
    return ws_need(c, key_bytes, has_val, n_local_max, gsd_capacity(c, n_local_max), b,
                   (uint64_t)n_local_max * c->nranks);
}

// GER steps 2b-3 on the assembled draws (L.ger_key, L.ger_q, M entries; offsets in
// L.ger_off): order the draws by composite with two stable radix sorts, pick S_j
static rs_status_t ger_splitters(const GsdLayout& L, size_t M, size_t s, int p, uint64_t n_total, Comp* S,
                                 cudaStream_t st) {
    const int threads = 256;
    const int grid = (int)std::min<size_t>((M + threads - 1) / threads, 1024);
    {
        LaunchScope ls("ger_sample", st);
        k_iota_u32<<<grid, threads, 0, st>>>(L.ger_idx, M);
    }
    // (position, draw) -> draws in position order; positions need ⌈log2 n⌉ bits
    int qbits = 8;
    while (qbits < 64 && (n_total >> qbits) != 0) qbits += 8;
    rs_status_t sst = local_sort(8, L.ger_q, L.ger_idx, M, 8, qbits, L.ger_k2, L.ger_ia, L.ger_ws, L.ger_ws_bytes, st);
    if (sst != RS_OK) return sst;
    {
        LaunchScope ls("ger_sample", st);
        k_ger_gather<<<grid, threads, 0, st>>>(L.ger_key, L.ger_ia, M, L.ger_k2);
    }
    // stable by key: ties keep position order, i.e. (key, rank, pos) order
    sst = local_sort(8, L.ger_k2, L.ger_ia, M, 8, 64, L.ger_k3, L.ger_ib, L.ger_ws, L.ger_ws_bytes, st);
    if (sst != RS_OK) return sst;
    LaunchScope ls("ger_sample", st);
    k_ger_pick<<<1, 256, 0, st>>>(L.ger_key, L.ger_q, L.ger_ib, s, p, L.ger_off, S);
    return RS_OK;
}

// GVR step 3 on one rank's unsorted block: destinations, counts (added to
// counts[0..p)), and the block partitioned by destination into L.gv_keys/gv_vals
static rs_status_t gvr_partition(const GsdLayout& L, int key_bytes, const void* X, const uint32_t* V, size_t N,
                                 int rank, int p, const Comp* S, uint64_t* counts, cudaStream_t st) {
    if (!N) return RS_OK;
    const int grid = (int)std::min<size_t>((N + 255) / 256, (size_t)sm_count() * 8);
    if (key_bytes == 4 && !V) {
        // u32 keys: the keys themselves ride as the values of one stable radix pass
        // over the destinations — X_{k,j} in source order, no index gather
        {
            LaunchScope ls("gvr_split", st);
            k_gvr_dest<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(X), N, (uint32_t)rank, S, p,
                                                       L.gv_dest, nullptr, counts);
        }
        return local_sort(4, L.gv_dest, static_cast<const uint32_t*>(X), N, 8, 8, L.gv_sdest,
                          static_cast<uint32_t*>(L.gv_keys), L.gv_ws, L.gv_ws_bytes, st);
    }
    {
        LaunchScope ls("gvr_split", st);
        if (key_bytes == 4)
            k_gvr_dest<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(X), N, (uint32_t)rank, S, p,
                                                       L.gv_dest, L.gv_idx, counts);
        else
            k_gvr_dest<uint64_t><<<grid, 256, 0, st>>>(static_cast<const uint64_t*>(X), N, (uint32_t)rank, S, p,
                                                       L.gv_dest, L.gv_idx, counts);
    }
    // stable count-sort by destination: one radix-256 pass (p <= 256)
    rs_status_t sst = local_sort(4, L.gv_dest, L.gv_idx, N, 8, 8, L.gv_sdest, L.gv_sidx, L.gv_ws, L.gv_ws_bytes, st);
    if (sst != RS_OK) return sst;
    LaunchScope ls("gvr_split", st);
    if (key_bytes == 4)
        k_gvr_gather<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(X), V, L.gv_sidx, N,
                                                     static_cast<uint32_t*>(L.gv_keys), L.gv_vals);
    else
        k_gvr_gather<uint64_t><<<grid, 256, 0, st>>>(static_cast<const uint64_t*>(X), V, L.gv_sidx, N,
                                                     static_cast<uint64_t*>(L.gv_keys), L.gv_vals);
    return RS_OK;
}

static rs_status_t launch_ger_draw(int key_bytes, const void* X, uint64_t off, size_t N, uint64_t n_total,
                                   uint64_t seed, size_t M, uint64_t* key, uint64_t* q, cudaStream_t st) {
    if (!N || !M) return RS_OK;
    LaunchScope ls("ger_sample", st);
    const int grid = (int)std::min<size_t>((M + 255) / 256, 1024);
    if (key_bytes == 4)
        k_ger_draw<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(X), off, N, n_total, seed, M, key, q);
    else
        k_ger_draw<uint64_t><<<grid, 256, 0, st>>>(static_cast<const uint64_t*>(X), off, N, n_total, seed, M, key, q);
    return RS_OK;
}

static rs_status_t launch_sample(int key_bytes, const void* X, size_t N, int rank, int s, Comp* out,
                                 cudaStream_t st) {
    LaunchScope ls("gsd_sample", st);
    const int threads = std::min(256, std::max(32, s));
    const int grid = (s + threads - 1) / threads;
    if (key_bytes == 4)
        k_gsd_sample<uint32_t><<<grid, threads, 0, st>>>(static_cast<const uint32_t*>(X), N, rank, s, out);
    else
        k_gsd_sample<uint64_t><<<grid, threads, 0, st>>>(static_cast<const uint64_t*>(X), N, rank, s, out);
    return RS_OK;
}

static rs_status_t launch_splitters(const unsigned char* recs, size_t stride, int p, int s, Comp* S, cudaStream_t st) {
    int L = 1;
    while (L < p * s) L <<= 1;
    rs_status_t r = kernel_setup(reinterpret_cast<const void*>(k_gsd_splitters), 1024, kMaxSample * sizeof(Comp),
                                 nullptr);
    if (r != RS_OK) return r;
    LaunchScope ls("gsd_splitters", st);
    k_gsd_splitters<<<1, 1024, (size_t)L * sizeof(Comp), st>>>(recs, stride, 128, p, s, S);
    return RS_OK;
}

static rs_status_t launch_split(int key_bytes, const void* X, size_t N, int rank, int p, const Comp* S,
                                uint64_t* counts, cudaStream_t st) {
    LaunchScope ls("gsd_split", st);
    const int threads = std::min(1024, ((p + 31) / 32) * 32);
    if (key_bytes == 4)
        k_gsd_split<uint32_t><<<1, threads, 0, st>>>(static_cast<const uint32_t*>(X), N, rank, p, S, counts);
    else
        k_gsd_split<uint64_t><<<1, threads, 0, st>>>(static_cast<const uint64_t*>(X), N, rank, p, S, counts);
    return RS_OK;
}

// step 5 on received runs (source-rank order): the p-way pass (gsd_merge 3), the
// merge tree (0, 2) or a stable radix re-sort of the concatenation (1); all give
// the identical result (reading R17)
static rs_status_t merge_runs(int key_bytes, void* runs, uint32_t* vruns, const std::vector<uint64_t>& roff, int b,
                              void* out, uint32_t* vout, const GsdLayout& L, size_t cap, int merge, cudaStream_t st) {
    const size_t total = roff.back();
    if (total == 0) return RS_OK;
    if (merge == 1)
        return local_sort(key_bytes, runs, vruns, total, b, key_bytes * 8, out, vout, L.local_ws, L.local_ws_bytes, st);
    const int p = (int)roff.size() - 1;
    std::vector<uint64_t> len(p);
    for (int k = 0; k < p; ++k) len[k] = roff[k + 1] - roff[k];
    if (merge == 3 && pway_applicable(p, len) && pway_scratch_bytes(key_bytes, total, p) <= cap * (size_t)key_bytes) {
        std::vector<const void*> rk(p);
        std::vector<const uint32_t*> rv(vruns ? p : 0);
        for (int k = 0; k < p; ++k) {
            rk[k] = static_cast<const char*>(runs) + roff[k] * key_bytes;
            if (vruns) rv[k] = vruns + roff[k];
        }
        return merge_pway(key_bytes, rk, rv, len, L.merge_keys, cap * (size_t)key_bytes, out, vout, st);
    }
    return merge_runs_tree(key_bytes, runs, vruns, roff, L.merge_keys, L.merge_vals, out, vout, L.merge_split, st);
}

// step 5 over runs read in place (pull merge): the one-pass p-way merge (gsd_merge 3)
// when it applies and its scratch fits, else the 2-way tree
static rs_status_t pull_merge(int key_bytes, const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                              const std::vector<uint64_t>& len, const GsdLayout& L, size_t cap, int merge, void* out,
                              uint32_t* vout, cudaStream_t st) {
    uint64_t total = 0;
    for (uint64_t l : len) total += l;
    if (merge == 3 && pway_applicable((int)len.size(), len) &&
        pway_scratch_bytes(key_bytes, total, (int)len.size()) <= cap * (size_t)key_bytes)
        return merge_pway(key_bytes, rk, rv, len, L.merge_keys, cap * (size_t)key_bytes, out, vout, st);
    return merge_runs_ptrs(key_bytes, rk, rv, len, L.merge_keys, L.merge_vals, out, vout, L.merge_split, st);
}

// ------------------------------------------------------------ headers ----
enum HdrField {
    kHMagic = 0, kHKeyBytes, kHHasVal, kHBits, kHSampling, kHR, kHP, kHGerS, kHGerSeed, kHMerge,
    kHAgreed,  // fields [0, kHAgreed) must be equal on every rank
    kHOutCap = kHAgreed, kHN, kHWs, kHErr
};
constexpr uint64_t kMagic = 0x52534F5254ull;  // "RSORT"

struct CallArgs {
    int key_bytes;
    void* keys;
    uint32_t* vals;   // NULL for keys-only; may be NULL with n = 0 in a pair sort (hv says which)
    bool hv;          // a pair sort (rs_sort_pairs_*), whatever this rank's n
    size_t n;
    int b;
    void* out;
    uint32_t* vout;
    size_t out_cap;
    void* ws;
    size_t ws_bytes;
    int merge;  // gsd_merge: 0 tree, 1 radix re-sort, 2 tree / 3 p-way pass (pull merge when `pull`)
    bool pull;  // gsd_pull: read the peers' blocks in place instead of an all-to-all
};

static void fill_header(const Comm* c, const CallArgs& a, bool local_err, uint64_t* h) {
    std::memset(h, 0, kHdrWords * 8);
    h[kHMagic] = kMagic;
    h[kHKeyBytes] = (uint64_t)a.key_bytes;
    h[kHHasVal] = a.hv;
    h[kHBits] = (uint64_t)a.b;
    h[kHSampling] = (uint64_t)c->sampling;
    h[kHR] = (uint64_t)c->r;
    h[kHP] = (uint64_t)c->nranks;
    h[kHGerS] = (uint64_t)c->ger_s;
    h[kHGerSeed] = c->ger_seed;
    h[kHMerge] = (uint64_t)a.merge | ((uint64_t)a.pull << 8);
    h[kHOutCap] = (uint64_t)a.out_cap;
    h[kHN] = (uint64_t)a.n;
    h[kHWs] = (uint64_t)a.ws_bytes;
    h[kHErr] = local_err ? 1 : 0;
}

// every rank reaches the same verdict from the same all-gathered headers
static rs_status_t check_headers(const Comm* c, const uint64_t* all, const uint64_t* mine, std::vector<uint64_t>* n_all,
                                 std::vector<uint64_t>* caps) {
    const int p = c->nranks;
    n_all->assign(p, 0);
    caps->assign(p, 0);
    for (int k = 0; k < p; ++k) {
        const uint64_t* hk = all + (size_t)k * kHdrWords;
        for (int f = 0; f < kHAgreed; ++f)
            if (hk[f] != mine[f])
                return fail(RS_EINVAL, "collective sort: arguments / settings differ on rank " + std::to_string(k) +
                                           " (header field " + std::to_string(f) + ")");
    }
    for (int k = 0; k < p; ++k) {
        const uint64_t* hk = all + (size_t)k * kHdrWords;
        if (hk[kHErr]) return fail(RS_EINVAL, "rank " + std::to_string(k) + " failed argument validation");
        (*n_all)[k] = hk[kHN];
        (*caps)[k] = hk[kHOutCap];
    }
    return RS_OK;
}

// this rank's own argument checks, before anything is enqueued
static std::string validate_local(Comm* c, const CallArgs& a, rs_status_t local_status) {
    if (local_status != RS_OK) return rs_last_error();
    const bool hv = a.hv;
    if (a.out_cap && (!a.out || (hv && !a.vout))) return "NULL output with out_cap > 0";
    if (!a.ws || !aligned16(a.ws)) return "collective workspace NULL or misaligned";
    if (c->nranks > 1 && c->sampling <= 2 && a.n && a.out_cap) {
        // the pull merge reads the peers' sorted blocks while this rank writes Y_j:
        // `out` must not overlap `keys` (nor vout `vals`)
        auto overlap = [](const void* x, size_t xb, const void* y, size_t yb) {
            const uintptr_t a0 = reinterpret_cast<uintptr_t>(x), b0 = reinterpret_cast<uintptr_t>(y);
            return a0 < b0 + yb && b0 < a0 + xb;
        };
        if (overlap(a.out, a.out_cap * a.key_bytes, a.keys, a.n * a.key_bytes) ||
            (hv && overlap(a.vout, a.out_cap * 4, a.vals, a.n * 4)))
            return "with a comm (p > 1), out must not overlap keys (nor out_vals vals)";
    }
    return "";
}

// ------------------------------------------------- exchange + merge (step 4-5)
// After the count sync: plan, then pull merge or all-to-all + merge.  X / XV: the
// rank's sorted block (GVR: the block partitioned by destination); recs: every
// rank's count record (p counts, key peer record, value peer record, export flag).
static rs_status_t exchange_and_merge(Comm* c, const CallArgs& a, const GsdLayout& L, void* X, uint32_t* XV,
                                      const uint64_t* recs, size_t wc, bool gvr, uint64_t* total_out,
                                      cudaStream_t st) {
    const int p = c->nranks, rank = c->rank, kb = a.key_bytes;
    const bool hv = a.hv;
    std::vector<uint64_t> cnt((size_t)p * p);
    bool all_exported = true;
    for (int k = 0; k < p; ++k) {
        for (int j = 0; j < p; ++j) cnt[(size_t)k * p + j] = recs[(size_t)k * wc + j];
        all_exported = all_exported && recs[(size_t)k * wc + p + 2 * kPeerRecWords] == 1;
    }
    c->last_counts = cnt;
    std::vector<uint64_t> soff(p + 1, 0), roff(p + 1, 0);
    for (int j = 0; j < p; ++j) soff[j + 1] = soff[j] + cnt[(size_t)rank * p + j];
    for (int k = 0; k < p; ++k) roff[k + 1] = roff[k] + cnt[(size_t)k * p + rank];
    const uint64_t total = roff[p];
    *total_out = total;
    rs_status_t s = RS_OK;
    if (p == 1) {  // Y_0 = X_0 (GVR: its one local sort)
        if (gvr)
            return total ? local_sort(kb, X, XV, total, a.b, kb * 8, a.out, a.vout, L.local_ws, L.local_ws_bytes, st)
                         : RS_OK;
        if (total && X != a.out) {
            RS_CUDA_TRY(cudaMemcpyAsync(a.out, X, total * kb, cudaMemcpyDeviceToDevice, st));
            if (hv) RS_CUDA_TRY(cudaMemcpyAsync(a.vout, XV, total * 4, cudaMemcpyDeviceToDevice, st));
        }
        return RS_OK;
    }
    if (!gvr && a.merge >= 2 && a.pull && all_exported) {
        // pull merge: no all-to-all; the p-way pass reads every
        // peer's X_{k,j} in place — over NVLink between GPUs — and writes Y_j once
        std::vector<const void*> rk(p);
        std::vector<const uint32_t*> rv(hv ? p : 0);
        std::vector<uint64_t> len(p);
        bool opened = true;
        for (int k = 0; k < p && opened; ++k) {
            uint64_t so = 0;  // start of X_{k,rank} in rank k's sorted block
            for (int jj = 0; jj < rank; ++jj) so += cnt[(size_t)k * p + jj];
            len[k] = cnt[(size_t)k * p + rank];
            void* kbp = X;
            void* vbp = XV;
            if (k != rank) {
                const uint64_t* rec = recs + (size_t)k * wc + p;
                opened = c->tr->open_peer(k, rec, &kbp) == RS_OK;
                if (opened && hv) opened = c->tr->open_peer(k, rec + kPeerRecWords, &vbp) == RS_OK;
            }
            rk[k] = static_cast<const char*>(kbp) + so * kb;
            if (hv) rv[k] = static_cast<const uint32_t*>(vbp) + so;
        }
        if (opened) {
            LaunchScope ls("gsd_pull_merge", st, false);
            s = pull_merge(kb, rk, rv, len, L, a.out_cap, a.merge, a.out, a.vout, st);
        } else {
            s = RS_ECUDA;  // rs_last_error() names the mapping failure
        }
        // every rank waits here (also one that failed above): no rank may reuse its
        // block before every peer has read its slices
        const rs_status_t bs = c->tr->barrier(st);
        c->tr->release_unused();
        return s != RS_OK ? s : bs;
    }
    // all-to-all of the zero-copy slices X_{k,j} into the receive buffer
    {
        LaunchScope ls("gsd_exchange", st, false);
        if ((s = c->tr->alltoallv(X, soff, L.recv_keys, roff, kb, st)) != RS_OK) return s;
        if (hv && (s = c->tr->alltoallv(XV, soff, L.recv_vals, roff, 4, st)) != RS_OK) return s;
    }
    c->tr->release_unused();
    if (gvr)  // GVR step 4: local sort of the received concatenation
        return total ? local_sort(kb, L.recv_keys, L.recv_vals, total, a.b, kb * 8, a.out, a.vout, L.local_ws,
                                  L.local_ws_bytes, st)
                     : RS_OK;
    return merge_runs(kb, L.recv_keys, L.recv_vals, roff, a.b, a.out, a.vout, L, a.out_cap, a.merge, st);
}

// count record of this rank: counts (written by a kernel) + key / value peer
// records + export flag (host, staged through pinned memory)
static rs_status_t stage_peer_records(Comm* c, const CallArgs& a, const void* X, const uint32_t* XV, bool want,
                                      uint64_t* cnt_send, cudaStream_t st) {
    const int p = c->nranks;
    uint64_t* rec = c->h + 16;  // staging words [16, 16 + 2·kPeerRecWords + 2)
    std::memset(rec, 0, (2 * kPeerRecWords + 2) * 8);
    bool ok = want && c->tr->export_buffer(X, rec);
    if (ok && a.hv) ok = c->tr->export_buffer(XV, rec + kPeerRecWords);
    rec[2 * kPeerRecWords] = ok ? 1 : 0;
    RS_CUDA_TRY(cudaMemcpyAsync(cnt_send + p, rec, (2 * kPeerRecWords + 2) * 8, cudaMemcpyHostToDevice, st));
    return RS_OK;
}

// GSD with regular oversampling: ONE host synchronisation per call
static rs_status_t gsd_regular(Comm* c, const CallArgs& a, const std::string& local_err, size_t* n_out,
                               cudaStream_t st) {
    const int p = c->nranks, rank = c->rank, kb = a.key_bytes;
    const int s = c->r * p;
    const bool valid = local_err.empty();
    const bool hv = a.hv;
    const CommRegions R = comm_regions(c);
    const size_t Bs = 128 + 16 * (size_t)s;  // record: header + s composites
    unsigned char* samp_send = R.samp;
    unsigned char* samp_all = R.samp + R.bs_max;
    uint64_t* cnt_send = R.cnt;
    uint64_t* cnt_all = R.cnt + R.wc;
    uint64_t* hdr = c->h;  // staging words [0, 16)
    fill_header(c, a, !valid, hdr);
    RS_CUDA_TRY(cudaMemcpyAsync(samp_send, hdr, 128, cudaMemcpyHostToDevice, st));
    GsdLayout L{};
    if (valid) L = gsd_layout(a.ws, kb, hv, a.n, a.out_cap, a.b, p);
    const size_t N = valid ? a.n : 0;  // an invalid rank takes part with an empty block
    rs_status_t sst = RS_OK;
    // step 1: local sort in place -> X_k
    {
        NvtxRange nr("rsort.gsd.local_sort");
        if (N && (sst = local_sort(kb, a.keys, a.vals, N, a.b, kb * 8, a.keys, a.vals, L.local_ws, L.local_ws_bytes,
                                   st)) != RS_OK)
            return sst;
    }
    NvtxRange nr_split("rsort.gsd.sample_split_sync");
    // step 2: sample into this rank's record; C1 all-gather of the records
    if ((sst = launch_sample(kb, a.keys, N, rank, s, reinterpret_cast<Comp*>(samp_send + 128), st)) != RS_OK) return sst;
    if ((sst = c->tr->allgather(samp_send, samp_all, Bs, st)) != RS_OK) return sst;
    // step 3: splitters, identical on every rank
    if ((sst = launch_splitters(samp_all, Bs, p, s, R.spl, st)) != RS_OK) return sst;
    // step 4: split -> counts; peer records; C2 all-gather of the count records
    if ((sst = launch_split(kb, a.keys, N, rank, p, R.spl, cnt_send, st)) != RS_OK) return sst;
    if ((sst = stage_peer_records(c, a, a.keys, a.vals, valid && p > 1 && a.merge >= 2 && a.pull, cnt_send, st)) !=
        RS_OK)
        return sst;
    if ((sst = c->tr->allgather(cnt_send, cnt_all, R.wc * 8, st)) != RS_OK) return sst;
    // the one host synchronisation: every rank's header, count record, and the splitters
    uint64_t* in = c->h + comm_hin_offset();
    uint64_t* in_hdr = in;
    uint64_t* in_cnt = in + (size_t)p * kHdrWords;
    uint64_t* in_spl = in_cnt + (size_t)p * R.wc;
    RS_CUDA_TRY(cudaMemcpy2DAsync(in_hdr, kHdrWords * 8, samp_all, Bs, kHdrWords * 8, p, cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaMemcpyAsync(in_cnt, cnt_all, (size_t)p * R.wc * 8, cudaMemcpyDeviceToHost, st));
    if (p > 1) RS_CUDA_TRY(cudaMemcpyAsync(in_spl, R.spl, (size_t)(p - 1) * sizeof(Comp), cudaMemcpyDeviceToHost, st));
    if ((sst = c->wait(st)) != RS_OK) return sst;
    std::vector<uint64_t> n_all, caps;
    if ((sst = check_headers(c, in_hdr, hdr, &n_all, &caps)) != RS_OK) return valid ? sst : fail(RS_EINVAL, local_err);
    c->last_splitters.assign((size_t)3 * (p - 1), 0);
    for (int i = 0; i + 1 < p; ++i) {
        const Comp* sp = reinterpret_cast<const Comp*>(in_spl) + i;
        c->last_splitters[3 * i] = sp->key;
        c->last_splitters[3 * i + 1] = sp->rank;
        c->last_splitters[3 * i + 2] = sp->pos == kPosInf ? ~0ull : sp->pos;
    }
    // every rank checks every rank's capacity: all fail together
    for (int j = 0; j < p; ++j) {
        uint64_t tot = 0;
        for (int k = 0; k < p; ++k) tot += in_cnt[(size_t)k * R.wc + j];
        if (tot > caps[j])
            return fail(RS_ECAPACITY, "rank " + std::to_string(j) + " receives " + std::to_string(tot) +
                                          " keys > out_cap " + std::to_string(caps[j]));
    }
    uint64_t total = 0;
    NvtxRange nr_x("rsort.gsd.exchange_merge");
    sst = exchange_and_merge(c, a, L, a.keys, a.vals, in_cnt, R.wc, false, &total, st);
    if (sst != RS_OK) return sst;
    if (n_out) *n_out = total;
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

// GER / GVR (random oversampling): header exchange first (n over all ranks fixes
// s and the draws), then the same split / exchange / merge
static rs_status_t gsd_random(Comm* c, const CallArgs& a, const std::vector<uint64_t>& n_all,
                              const std::vector<uint64_t>& caps, size_t* n_out, cudaStream_t st) {
    const int p = c->nranks, rank = c->rank, kb = a.key_bytes;
    const bool hv = a.hv, gvr = c->sampling == 2;
    const CommRegions R = comm_regions(c);
    uint64_t* cnt_send = R.cnt;
    uint64_t* cnt_all = R.cnt + R.wc;
    std::vector<uint64_t> noff(p + 1, 0);
    for (int k = 0; k < p; ++k) noff[k + 1] = noff[k] + n_all[k];
    const uint64_t n_total = noff[p];
    const size_t gs = ger_s_for(c, n_total), M = ger_draws(gs, p);
    const GsdLayout L = gsd_layout(a.ws, kb, hv, a.n, a.out_cap, a.b, p, M, gvr);
    rs_status_t sst = RS_OK;
    // step 1 (GVR sorts last)
    if (a.n && !gvr &&
        (sst = local_sort(kb, a.keys, a.vals, a.n, a.b, kb * 8, a.keys, a.vals, L.local_ws, L.local_ws_bytes, st)) !=
            RS_OK)
        return sst;
    if (M) {
        // steps 2-3: random sample assembled on every rank by a max all-reduce
        uint64_t* offs = c->h + 64;  // staging words [64, 64 + p + 1)
        std::memcpy(offs, noff.data(), (p + 1) * 8);
        RS_CUDA_TRY(cudaMemcpyAsync(L.ger_off, offs, (p + 1) * 8, cudaMemcpyHostToDevice, st));
        RS_CUDA_TRY(cudaMemsetAsync(L.ger_key, 0, M * 8, st));
        RS_CUDA_TRY(cudaMemsetAsync(L.ger_q, 0, M * 8, st));
        if ((sst = launch_ger_draw(kb, a.keys, noff[rank], a.n, n_total, c->ger_seed, M, L.ger_key, L.ger_q, st)) !=
            RS_OK)
            return sst;
        if ((sst = c->tr->allreduce_max_u64(L.ger_key, M, st)) != RS_OK) return sst;
        if ((sst = c->tr->allreduce_max_u64(L.ger_q, M, st)) != RS_OK) return sst;
        if ((sst = ger_splitters(L, M, gs, p, n_total, R.spl, st)) != RS_OK) return sst;
    }
    // step 4: split + count records
    void* X = a.keys;
    uint32_t* XV = a.vals;
    if (gvr) {
        RS_CUDA_TRY(cudaMemsetAsync(cnt_send, 0, (size_t)p * 8, st));
        if (p > 1) {
            if ((sst = gvr_partition(L, kb, a.keys, a.vals, a.n, rank, p, R.spl, cnt_send, st)) != RS_OK) return sst;
            X = L.gv_keys;
            XV = L.gv_vals;
        } else {
            c->h[80] = a.n;
            RS_CUDA_TRY(cudaMemcpyAsync(cnt_send, c->h + 80, 8, cudaMemcpyHostToDevice, st));
        }
    } else if ((sst = launch_split(kb, a.keys, a.n, rank, p, R.spl, cnt_send, st)) != RS_OK) {
        return sst;
    }
    if ((sst = stage_peer_records(c, a, X, XV, !gvr && p > 1 && a.merge >= 2 && a.pull, cnt_send, st)) != RS_OK)
        return sst;
    if ((sst = c->tr->allgather(cnt_send, cnt_all, R.wc * 8, st)) != RS_OK) return sst;
    uint64_t* in_cnt = c->h + comm_hin_offset();
    uint64_t* in_spl = in_cnt + (size_t)p * R.wc;
    RS_CUDA_TRY(cudaMemcpyAsync(in_cnt, cnt_all, (size_t)p * R.wc * 8, cudaMemcpyDeviceToHost, st));
    if (p > 1 && M) RS_CUDA_TRY(cudaMemcpyAsync(in_spl, R.spl, (size_t)(p - 1) * sizeof(Comp), cudaMemcpyDeviceToHost, st));
    if ((sst = c->wait(st)) != RS_OK) return sst;
    c->last_splitters.assign((size_t)3 * (p - 1), 0);
    for (int i = 0; i + 1 < p && M; ++i) {
        const Comp* sp = reinterpret_cast<const Comp*>(in_spl) + i;
        c->last_splitters[3 * i] = sp->key;
        c->last_splitters[3 * i + 1] = sp->rank;
        c->last_splitters[3 * i + 2] = sp->pos == kPosInf ? ~0ull : sp->pos;
    }
    for (int j = 0; j < p; ++j) {  // capacities came with the headers: every rank checks every rank
        uint64_t tot = 0;
        for (int k = 0; k < p; ++k) tot += in_cnt[(size_t)k * R.wc + j];
        if (tot > caps[j])
            return fail(RS_ECAPACITY, "rank " + std::to_string(j) + " receives " + std::to_string(tot) +
                                          " keys > out_cap " + std::to_string(caps[j]));
    }
    uint64_t total = 0;
    sst = exchange_and_merge(c, a, L, X, XV, in_cnt, R.wc, gvr, &total, st);
    if (sst != RS_OK) return sst;
    if (n_out) *n_out = total;
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

rs_status_t gsd_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, bool has_val, size_t n, int b, void* out,
                     uint32_t* vout, size_t out_cap, size_t* n_out, void* ws, size_t ws_bytes, cudaStream_t st,
                     rs_status_t local_status) {
    c->last_host_syncs = 0;
    if (c->broken) return fail(RS_ENCCL, "communicator is broken by an earlier failure; destroy it");
    const int p = c->nranks;
    CallArgs a{key_bytes, keys, vals, has_val, n, b, out, vout, out_cap, ws, ws_bytes, options().gsd_merge,
               options().gsd_pull != 0};
    std::string local_err = validate_local(c, a, local_status);
    if (local_err.empty() && c->sampling == 0 && (size_t)c->r * p * p > (size_t)kMaxSample)
        local_err = "r·p² exceeds the one-CTA sample sort limit of 8192";
    if (local_err.empty()) {
        const size_t need = ws_need(c, key_bytes, has_val, n, out_cap, b, 0);
        if (c->sampling != 1 && c->sampling != 2 && ws_bytes < need)
            local_err = "collective workspace too small: need " + std::to_string(need) + " bytes";
    }
    if (c->sampling == 0) return gsd_regular(c, a, local_err, n_out, st);

    // the other modes agree on the call first (one host synchronisation)
    uint64_t hdr[kHdrWords];
    fill_header(c, a, !local_err.empty(), hdr);
    std::vector<uint64_t> all((size_t)p * kHdrWords), n_all, caps;
    rs_status_t s = c->host_allgather(hdr, kHdrWords, all.data(), st);
    if (s != RS_OK) return s;
    if ((s = check_headers(c, all.data(), hdr, &n_all, &caps)) != RS_OK)
        return local_err.empty() ? s : fail(RS_EINVAL, local_err);
    if (c->sampling == 3) {  // PR4 across GPUs: sizes, digit width and capacity agreed here
        if (b != 8) return fail(RS_EINVAL, "PR4 routing across GPUs is radix 256 (digit_bits 8)");
        for (int k = 0; k < p; ++k) {
            if (all[(size_t)k * kHdrWords + kHWs] < pr_ws_bytes(key_bytes, has_val, n_all[k], p))
                return fail(RS_EINVAL, "PR workspace of rank " + std::to_string(k) + " too small");
            if (caps[k] < n_all[k]) return fail(RS_ECAPACITY, "PR: out_cap < n on rank " + std::to_string(k));
        }
        return pr_sort(c, key_bytes, keys, vals, has_val, n, out, vout, n_out, ws, n_all, st);
    }
    if (c->sampling >= 4) {  // BTN / OET: equal blocks (reading R34), agreed here
        if (c->sampling == 4 && (p & (p - 1))) return fail(RS_EINVAL, "BTN needs a power-of-two number of ranks");
        for (int k = 0; k < p; ++k) {
            if (n_all[k] != n)
                return fail(RS_EINVAL, "BTN/OET need the same n on every rank (rank " + std::to_string(k) + ")");
            if (caps[k] < n_all[k]) return fail(RS_ECAPACITY, "BTN/OET: out_cap < n on rank " + std::to_string(k));
        }
        return net_sort(c, key_bytes, keys, vals, has_val, n, b, out, vout, n_out, ws, st);
    }
    // GER / GVR: every rank checks every rank's workspace (sizes from the headers)
    uint64_t n_total = 0;
    for (int k = 0; k < p; ++k) n_total += n_all[k];
    for (int k = 0; k < p; ++k) {
        const size_t need = ws_need(c, key_bytes, has_val, n_all[k], caps[k], b, n_total);
        if (all[(size_t)k * kHdrWords + kHWs] < need)
            return fail(RS_EINVAL, "workspace of rank " + std::to_string(k) + " too small: need " +
                                       std::to_string(need) + " (size it with the largest local n)");
    }
    // capacity is checked after the split, identically on every rank
    return gsd_random(c, a, n_all, caps, n_out, st);
}

}  // namespace rs

using namespace rs;

extern "C" {

rs_status_t rs_gsd_exchange_plan(int p, int rank, const uint64_t* counts, const uint64_t* caps,
                                 uint64_t* send_off, uint64_t* recv_off, uint64_t* total) {
    if (p < 1 || rank < 0 || rank >= p || !counts || !send_off || !recv_off)
        return fail(RS_EINVAL, "rs_gsd_exchange_plan: bad arguments");
    // every rank checks every rank's capacity, so all ranks fail together
    if (caps)
        for (int j = 0; j < p; ++j) {
            uint64_t tot = 0;
            for (int k = 0; k < p; ++k) tot += counts[(size_t)k * p + j];
            if (tot > caps[j])
                return fail(RS_ECAPACITY, "rank " + std::to_string(j) + " receives " + std::to_string(tot) +
                                              " keys > out_cap " + std::to_string(caps[j]));
        }
    send_off[0] = recv_off[0] = 0;
    for (int j = 0; j < p; ++j) send_off[j + 1] = send_off[j] + counts[(size_t)rank * p + j];
    for (int k = 0; k < p; ++k) recv_off[k + 1] = recv_off[k] + counts[(size_t)k * p + rank];
    if (total) *total = recv_off[p];
    return RS_OK;
}

size_t rs_ger_capacity(size_t n_local_max, int p, size_t s) {
    if (p < 1) return 0;
    return ger_capacity_for(n_local_max, p, s ? s : ger_default_s((uint64_t)n_local_max * p));
}

size_t rs_ger_default_s(uint64_t n_total) { return ger_default_s(n_total); }

}  // extern "C"
