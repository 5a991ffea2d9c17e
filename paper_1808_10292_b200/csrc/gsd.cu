// GSD (Algorithm 1) on B200s: one process per GPU, NCCL
// over NVLink/NVSwitch for the three exchanges, the radix sort for step 1.
//
//   step 1 LocalSorting    local radix sort of the rank's block in place  (radix.cu)
//   step 2 SampleSelection K5 k_gsd_sample: s = r·p composites of X_k at ⌈N·i/s⌉−1,
//                          i = 1..s−1, plus N−1 (reading R10); C1 ncclAllGather
//   step 3 SplitterSelect  K6 k_gsd_splitters: bitonic sort of the r·p² sample in one
//                          CTA, S_i = T[i·s−1] (R11, R12) — identical on every rank,
//                          so the paper's "Broadcast splitters" is implicit
//   step 4 Split           K7 k_gsd_split: binary search of the composite splitters
//                          (R14) -> |X_{k,j}|; C2 ncclAllGather of the p counts, one
//                          D2H copy + host sync (NCCL send/recv take host counts);
//                          C3 grouped ncclSend/ncclRecv of the X_{k,j} slices (the
//                          sorted block is already grouped by destination: zero-copy)
//   step 5 Merging         Y_j from the p received runs, ties to the lower source rank
//                          (R16): a tree of stable 2-way merge-path merges (merge.cu),
//                          or optionally a stable radix re-sort of the concatenation,
//                          which gives the identical result (R17).
//
// GER replaces step 2-3 (Comm::sampling = 1): s·p − 1 keys drawn
// uniformly at random from the concatenation of the sorted blocks (readings R28-R30:
// SplitMix64 counter draws, position ⌊z·n/2^64⌋, with replacement).  Each rank fills
// the draws that fall in its block (k_ger_draw), ncclAllReduce(max) assembles the
// sample everywhere, and two stable radix sorts of the (position, draw) and then
// (key, draw) pairs order it by composite (key, rank, pos) — too large for the
// one-CTA bitonic sort; S_i is the (i·s)-th smallest (k_ger_pick).
//
// GVR (Comm::sampling = 2) splits before it sorts: the same
// random sample, drawn from the unsorted blocks; each key's destination by a
// binary search of the composite splitters (k_gvr_dest); a stable count-sort by
// destination (one radix-256 pass of (destination, index) pairs + a gather) gives
// the X_{k,j}; after the exchange, Y_j is sorted by the local radix sort (SR4).
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
__global__ void __launch_bounds__(1024) k_gsd_splitters(const Comp* __restrict__ T_all, int M, int s, int p,
                                                        Comp* __restrict__ S) {
    extern __shared__ Comp sT[];
    int L = 1;
    while (L < M) L <<= 1;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        if (i < M) sT[i] = T_all[i];
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
    const int j = threadIdx.x;
    if (j >= p) return;
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
    const int j = 1 + threadIdx.x;
    if (j >= p) return;
    const uint32_t e = order[(size_t)j * s - 1];
    const uint64_t qe = q[e];
    int k = 0;
    while (k + 1 < p && off[k + 1] <= qe) ++k;  // last block starting at or before qe: non-empty, owns qe
    S[j - 1] = Comp{key[e], (uint32_t)k, (uint32_t)(qe - off[k])};
}

// GVR step 3: destination of every key of the unsorted block, j = #{i : S_i <_c (x, rank, q)}
template <typename K>
__global__ void __launch_bounds__(256) k_gvr_dest(const K* __restrict__ X, size_t N, uint32_t rank,
                                                  const Comp* __restrict__ S, int p, uint32_t* __restrict__ dest,
                                                  uint32_t* __restrict__ idx, uint64_t* __restrict__ counts) {
    __shared__ Comp sS[256];
    __shared__ uint32_t sc[257];
    for (int i = threadIdx.x; i < p - 1; i += blockDim.x) sS[i] = S[i];
    for (int i = threadIdx.x; i < p; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (size_t)gridDim.x * blockDim.x) {
        const Comp e{static_cast<uint64_t>(X[q]), rank, (uint32_t)q};
        int lo = 0, hi = p - 1;  // count of splitters <_c e (they are sorted)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (comp_less(sS[mid], e)) lo = mid + 1;
            else hi = mid;
        }
        dest[q] = (uint32_t)lo;
        if (idx) idx[q] = (uint32_t)q;
        atomicAdd(&sc[lo], 1u);
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
    void* recv_keys;
    uint32_t* recv_vals;
    Comp* samp_local;     // s
    Comp* samp_all;       // p*s
    Comp* splitters;      // p-1
    uint64_t* counts_local;  // p
    uint64_t* counts_all;    // p*p (or p slots of p for the emulation)
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
    void* merge_keys;        // merge-tree scratch: cap keys (+ values)
    uint32_t* merge_vals;
    size_t* merge_split;
    size_t bytes;
};

static GsdLayout gsd_layout(void* ws, int key_bytes, bool has_val, size_t n, size_t cap, int b, int p, int r,
                            size_t recv_slots, size_t ger_M = 0, bool gvr = false) {
    GsdLayout L{};
    Carver c(ws);
    const size_t s = (size_t)r * p;
    L.local_ws_bytes = local_ws_bytes(key_bytes, has_val, std::max(n, cap), b);
    L.local_ws = c.take(L.local_ws_bytes);
    L.recv_keys = c.take(recv_slots * cap * key_bytes);
    L.recv_vals = static_cast<uint32_t*>(has_val ? c.take(recv_slots * cap * 4) : nullptr);
    L.samp_local = static_cast<Comp*>(c.take(s * sizeof(Comp)));
    L.samp_all = static_cast<Comp*>(c.take((size_t)p * s * sizeof(Comp)));
    L.splitters = static_cast<Comp*>(c.take((size_t)p * sizeof(Comp)));
    L.counts_local = static_cast<uint64_t*>(c.take((size_t)p * 8));
    L.counts_all = static_cast<uint64_t*>(c.take((size_t)p * p * 8));
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

size_t gsd_ws_bytes(Comm* c, int key_bytes, bool has_val, size_t n_local_max, int b) {
    if (c->sampling == 3) return pr_ws_bytes(key_bytes, has_val, n_local_max, c->nranks);
    if (c->sampling >= 4) return net_ws_bytes(key_bytes, has_val, n_local_max, b);
    const size_t cap = gsd_capacity(c, n_local_max);
    const size_t M = c->sampling >= 1 ? ger_draws(ger_s_for(c, (uint64_t)n_local_max * c->nranks), c->nranks) : 0;
    return gsd_layout(nullptr, key_bytes, has_val, n_local_max, cap, b, c->nranks, c->r, 1, M, c->sampling == 2).bytes;
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
    k_ger_pick<<<1, ((p + 31) / 32) * 32, 0, st>>>(L.ger_key, L.ger_q, L.ger_ib, s, p, L.ger_off, S);
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
        return local_sort(4, L.gv_dest, static_cast<const uint32_t*>(X), N, 8, p <= 256 ? 8 : 16, L.gv_sdest,
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
    // stable count-sort by destination: one radix-256 pass (two for p > 256)
    rs_status_t sst = local_sort(4, L.gv_dest, L.gv_idx, N, 8, p <= 256 ? 8 : 16, L.gv_sdest, L.gv_sidx, L.gv_ws,
                                 L.gv_ws_bytes, st);
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

static rs_status_t launch_splitters(const Comp* T_all, int M, int s, int p, Comp* S, cudaStream_t st) {
    int L = 1;
    while (L < M) L <<= 1;
    const size_t smem = (size_t)L * sizeof(Comp);
    static bool attr = false;
    if (!attr) {
        RS_CUDA_TRY(cudaFuncSetAttribute(k_gsd_splitters, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kMaxSample * sizeof(Comp))));
        attr = true;
    }
    LaunchScope ls("gsd_splitters", st);
    k_gsd_splitters<<<1, 1024, smem, st>>>(T_all, M, s, p, S);
    return RS_OK;
}

static rs_status_t launch_split(int key_bytes, const void* X, size_t N, int rank, int p, const Comp* S,
                                uint64_t* counts, cudaStream_t st) {
    LaunchScope ls("gsd_split", st);
    const int threads = ((p + 31) / 32) * 32;
    if (key_bytes == 4)
        k_gsd_split<uint32_t><<<1, threads, 0, st>>>(static_cast<const uint32_t*>(X), N, rank, p, S, counts);
    else
        k_gsd_split<uint64_t><<<1, threads, 0, st>>>(static_cast<const uint64_t*>(X), N, rank, p, S, counts);
    return RS_OK;
}

// step 5: Y_j from the p received runs (source-rank order): the merge tree
// (default) or a stable radix re-sort of the concatenation (option gsd_merge=1);
// both give the identical result (reading R17)
static rs_status_t merge_runs(int key_bytes, void* runs, uint32_t* vruns, const std::vector<uint64_t>& roff, int b,
                              void* out, uint32_t* vout, const GsdLayout& L, size_t cap, cudaStream_t st) {
    const size_t total = roff.back();
    if (total == 0) return RS_OK;
    if (options().gsd_merge == 1)
        return local_sort(key_bytes, runs, vruns, total, b, key_bytes * 8, out, vout, L.local_ws, L.local_ws_bytes, st);
    const int p = (int)roff.size() - 1;
    std::vector<uint64_t> len(p);
    for (int k = 0; k < p; ++k) len[k] = roff[k + 1] - roff[k];
    if (options().gsd_merge == 3 && pway_applicable(p, len) &&
        pway_scratch_bytes(key_bytes, total, p) <= cap * (size_t)key_bytes) {
        // the received runs merged in one p-way pass (the all-to-all fallback of the pull merge)
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

#define RS_NCCL_TRY(expr)                                                                     \
    do {                                                                                      \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(RS_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));        \
    } while (0)

// step 5 over runs read in place (pull merge): one-pass p-way merge (gsd_merge 3)
// when it applies and its scratch fits in the tree's, else the 2-way tree
static rs_status_t pull_merge(int key_bytes, const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                              const std::vector<uint64_t>& len, const GsdLayout& L, size_t cap, void* out,
                              uint32_t* vout, cudaStream_t st) {
    uint64_t total = 0;
    for (uint64_t l : len) total += l;
    if (options().gsd_merge == 3 && pway_applicable((int)len.size(), len) &&
        pway_scratch_bytes(key_bytes, total, (int)len.size()) <= cap * (size_t)key_bytes)
        return merge_pway(key_bytes, rk, rv, len, L.merge_keys, cap * (size_t)key_bytes, out, vout, st);
    return merge_runs_ptrs(key_bytes, rk, rv, len, L.merge_keys, L.merge_vals, out, vout, L.merge_split, st);
}

rs_status_t gsd_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, size_t n, int b, void* out, uint32_t* vout,
                     size_t out_cap, size_t* n_out, void* ws, size_t ws_bytes, cudaStream_t st,
                     rs_status_t local_status) {
    const int p = c->nranks, rank = c->rank, r = c->r;
    const size_t s = (size_t)r * p;
    const bool hv = vals != nullptr;
    const bool ger = c->sampling == 1 || c->sampling == 2;  // random sample (GER or GVR)
    const bool gvr = c->sampling == 2;          // split before sorting
    std::string local_err = local_status != RS_OK ? rs_last_error() : "";
    if (local_err.empty() && out_cap && (!out || (hv && !vout))) local_err = "NULL output with out_cap > 0";
    if (local_err.empty() && (!ws || !aligned16(ws))) local_err = "GSD workspace NULL or misaligned";

    // header all-gather on comm-owned buffers, before anything else: a mismatch or a
    // failed local validation on any rank is RS_EINVAL on every rank, not a hang
    uint64_t* h = c->h_pinned;
    const uint64_t samp_id =
        ger ? ((0x4745520000000000ull + (uint64_t)c->sampling) ^ (uint64_t)c->ger_s ^ (c->ger_seed * 0x9E3779B97F4A7C15ull))
            : ((uint64_t)r | ((uint64_t)c->sampling << 56));
    const uint64_t hdr[kHdrWords] = {0x52534F5254ull, (uint64_t)key_bytes, (uint64_t)hv, (uint64_t)b, samp_id,
                                     (uint64_t)p, (uint64_t)out_cap, (uint64_t)n, (uint64_t)ws_bytes,
                                     local_err.empty() ? 0ull : 1ull, 0, 0};
    std::memcpy(h, hdr, sizeof(hdr));
    RS_CUDA_TRY(cudaMemcpyAsync(c->d_hdr, h, sizeof(hdr), cudaMemcpyHostToDevice, st));
    RS_NCCL_TRY(ncclAllGather(c->d_hdr, c->d_hdr + kHdrWords, kHdrWords, ncclUint64, c->nccl, st));
    RS_CUDA_TRY(cudaMemcpyAsync(h, c->d_hdr + kHdrWords, (size_t)p * kHdrWords * 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    if (!local_err.empty()) return fail(RS_EINVAL, local_err);
    std::vector<uint64_t> caps(p), noff(p + 1, 0);
    for (int k = 0; k < p; ++k) {
        const uint64_t* hk = h + (size_t)k * kHdrWords;
        for (int f = 0; f < 6; ++f)
            if (hk[f] != hdr[f])
                return fail(RS_EINVAL, "GSD header mismatch with rank " + std::to_string(k) + " (field " +
                                           std::to_string(f) + ")");
        if (hk[9]) return fail(RS_EINVAL, "rank " + std::to_string(k) + " failed argument validation");
        caps[k] = hk[6];
        if (hk[7] >= (1ull << 32)) return fail(RS_EINVAL, "n >= 2^32 on rank " + std::to_string(k));
        noff[k + 1] = noff[k] + hk[7];
    }
    if (c->sampling == 3) {  // PR4 across GPUs: sizes, digit width and capacity agreed here
        if (b != 8) return fail(RS_EINVAL, "PR4 routing across GPUs is radix 256 (digit_bits 8)");
        std::vector<uint64_t> n_all(p);
        for (int k = 0; k < p; ++k) {
            const uint64_t* hk = h + (size_t)k * kHdrWords;
            n_all[k] = hk[7];
            if (hk[8] < pr_ws_bytes(key_bytes, hv, hk[7], p))
                return fail(RS_EINVAL, "PR workspace of rank " + std::to_string(k) + " too small");
            if (hk[6] < hk[7]) return fail(RS_ECAPACITY, "PR: out_cap < n on rank " + std::to_string(k));
        }
        return pr_sort(c, key_bytes, keys, vals, n, out, vout, n_out, ws, n_all, st);
    }
    if (c->sampling >= 4) {  // BTN / OET: equal blocks (reading R34), agreed here
        if (c->sampling == 4 && (p & (p - 1))) return fail(RS_EINVAL, "BTN needs a power-of-two number of ranks");
        for (int k = 0; k < p; ++k) {
            const uint64_t* hk = h + (size_t)k * kHdrWords;
            if (hk[7] != n) return fail(RS_EINVAL, "BTN/OET need the same n on every rank (rank " +
                                                       std::to_string(k) + ")");
            if (hk[8] < net_ws_bytes(key_bytes, hv, hk[7], b))
                return fail(RS_EINVAL, "BTN/OET workspace of rank " + std::to_string(k) + " too small");
            if (hk[6] < hk[7]) return fail(RS_ECAPACITY, "BTN/OET: out_cap < n on rank " + std::to_string(k));
        }
        return net_sort(c, key_bytes, keys, vals, n, b, out, vout, n_out, ws, st);
    }
    if (!ger && (size_t)p * s > (size_t)kMaxSample)
        return fail(RS_EINVAL, "r*p^2 exceeds the one-CTA sample sort limit of 8192");
    const uint64_t n_total = noff[p];
    const size_t ger_s = ger ? ger_s_for(c, n_total) : 0;
    const size_t M = ger ? ger_draws(ger_s, p) : 0;
    // every rank checks every rank's workspace (sizes from the headers): all agree
    for (int k = 0; k < p; ++k) {
        const uint64_t* hk = h + (size_t)k * kHdrWords;
        const size_t need = gsd_layout(nullptr, key_bytes, hv, hk[7], hk[6], b, p, r, 1, M, gvr).bytes;
        if (hk[8] < need)
            return fail(RS_EINVAL, "GSD workspace of rank " + std::to_string(k) + " too small: need " +
                                       std::to_string(need) + " (size it with the largest local n)");
    }
    const GsdLayout L = gsd_layout(ws, key_bytes, hv, n, out_cap, b, p, r, 1, M, gvr);

    // step 1: local sort in place -> X_k  (GVR sorts last)
    rs_status_t sst = (n && !gvr) ? local_sort(key_bytes, keys, vals, n, b, key_bytes * 8, keys, vals, L.local_ws,
                                               L.local_ws_bytes, st)
                                  : RS_OK;
    if (sst != RS_OK) return sst;
    if (ger && M) {
        // GER step 2: random sample assembled on every rank by a max all-reduce
        std::memcpy(h, noff.data(), (p + 1) * 8);
        RS_CUDA_TRY(cudaMemcpyAsync(L.ger_off, h, (p + 1) * 8, cudaMemcpyHostToDevice, st));
        RS_CUDA_TRY(cudaMemsetAsync(L.ger_key, 0, M * 8, st));
        RS_CUDA_TRY(cudaMemsetAsync(L.ger_q, 0, M * 8, st));
        if ((sst = launch_ger_draw(key_bytes, keys, noff[rank], n, n_total, c->ger_seed, M, L.ger_key, L.ger_q,
                                   st)) != RS_OK)
            return sst;
        RS_NCCL_TRY(ncclAllReduce(L.ger_key, L.ger_key, M, ncclUint64, ncclMax, c->nccl, st));
        RS_NCCL_TRY(ncclAllReduce(L.ger_q, L.ger_q, M, ncclUint64, ncclMax, c->nccl, st));
        // GER step 3: S_i = (i·s)-th smallest, identical on every rank
        if ((sst = ger_splitters(L, M, ger_s, p, n_total, L.splitters, st)) != RS_OK) return sst;
    } else if (!ger) {
        // step 2: regular sample + all-gather
        if ((sst = launch_sample(key_bytes, keys, n, rank, (int)s, L.samp_local, st)) != RS_OK) return sst;
        RS_NCCL_TRY(ncclAllGather(L.samp_local, L.samp_all, s * sizeof(Comp), ncclUint8, c->nccl, st));
        // step 3: splitters, identical on every rank
        if ((sst = launch_splitters(L.samp_all, (int)(p * s), (int)s, p, L.splitters, st)) != RS_OK) return sst;
    }
    // step 4: split + count exchange
    if (gvr) {
        RS_CUDA_TRY(cudaMemsetAsync(L.counts_local, 0, (size_t)p * 8, st));
        if (p > 1) {
            if ((sst = gvr_partition(L, key_bytes, keys, vals, n, rank, p, L.splitters, L.counts_local, st)) != RS_OK)
                return sst;
        } else {
            h[0] = n;
            RS_CUDA_TRY(cudaMemcpyAsync(L.counts_local, h, 8, cudaMemcpyHostToDevice, st));
        }
    } else if ((sst = launch_split(key_bytes, keys, n, rank, p, L.splitters, L.counts_local, st)) != RS_OK) {
        return sst;
    }
    RS_NCCL_TRY(ncclAllGather(L.counts_local, L.counts_all, p, ncclUint64, c->nccl, st));
    RS_CUDA_TRY(cudaMemcpyAsync(h, L.counts_all, (size_t)p * p * 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<uint64_t> cnt(h, h + (size_t)p * p);
    c->last_counts = cnt;
    std::vector<uint64_t> soff(p + 1, 0), roff(p + 1, 0);
    uint64_t total = 0;
    if ((sst = rs_gsd_exchange_plan(p, rank, cnt.data(), caps.data(), soff.data(), roff.data(), &total)) != RS_OK)
        return sst;
    // pull merge (gsd_merge = 2): no all-to-all; the merge
    // tree's first level reads the peers' X_{k,j} in place over NVLink through
    // CUDA IPC mappings exchanged now (falls back to the all-to-all on every
    // rank if any rank cannot export its block, e.g. VMM memory)
    if (options().gsd_merge >= 2 && options().gsd_pull && !gvr && p > 1) {
        uint64_t* rec = h;
        std::memset(rec, 0, kIpcWords * 8);
        bool ok = ipc_export(keys, rec, &rec[8]) == RS_OK;
        if (ok && hv) ok = ipc_export(vals, &rec[9], &rec[17]) == RS_OK;
        rec[18] = ok ? 1 : 0;
        RS_CUDA_TRY(cudaMemcpyAsync(c->d_ipc, rec, kIpcWords * 8, cudaMemcpyHostToDevice, st));
        RS_NCCL_TRY(ncclAllGather(c->d_ipc, c->d_ipc + kIpcWords, kIpcWords, ncclUint64, c->nccl, st));
        RS_CUDA_TRY(cudaMemcpyAsync(h, c->d_ipc + kIpcWords, (size_t)p * kIpcWords * 8, cudaMemcpyDeviceToHost, st));
        RS_CUDA_TRY(cudaStreamSynchronize(st));
        bool all_ok = true;
        for (int k = 0; k < p; ++k) all_ok = all_ok && h[(size_t)k * kIpcWords + 18] == 1;
        std::vector<const void*> rk(p);
        std::vector<const uint32_t*> rv(hv ? p : 0);
        std::vector<uint64_t> len(p);
        if (all_ok) {
            // map the peers' blocks; whether every rank could is agreed on collectively
            bool opened = true;
            for (int k = 0; k < p && opened; ++k) {
                uint64_t so = 0;  // start of X_{k,rank} in rank k's sorted block
                for (int jj = 0; jj < rank; ++jj) so += cnt[(size_t)k * p + jj];
                len[k] = cnt[(size_t)k * p + rank];
                const uint64_t* rk_rec = h + (size_t)k * kIpcWords;
                void* kb = keys;
                void* vb = vals;
                if (k != rank) {
                    opened = ipc_open(rk_rec, rk_rec[8], &kb) == RS_OK;
                    if (opened && hv) opened = ipc_open(&rk_rec[9], rk_rec[17], &vb) == RS_OK;
                }
                rk[k] = static_cast<const char*>(kb) + so * key_bytes;
                if (hv) rv[k] = static_cast<const uint32_t*>(vb) + so;
            }
            h[0] = opened ? 0 : 1;
            RS_CUDA_TRY(cudaMemcpyAsync(c->d_ipc, h, 8, cudaMemcpyHostToDevice, st));
            RS_NCCL_TRY(ncclAllReduce(c->d_ipc, c->d_ipc, 1, ncclUint64, ncclMax, c->nccl, st));
            RS_CUDA_TRY(cudaMemcpyAsync(h, c->d_ipc, 8, cudaMemcpyDeviceToHost, st));
            RS_CUDA_TRY(cudaStreamSynchronize(st));
            all_ok = h[0] == 0;
        }
        if (all_ok) {
            {
                LaunchScope ls("gsd_pull_merge", st, false);
                if ((sst = pull_merge(key_bytes, rk, rv, len, L, out_cap, out, vout, st)) != RS_OK)
                    return sst;
            }
            // no rank may reuse its block before every peer has read its slices
            RS_NCCL_TRY(ncclAllReduce(c->d_ipc, c->d_ipc, 1, ncclUint64, ncclMax, c->nccl, st));
            if (n_out) *n_out = total;
            RS_CUDA_TRY(cudaGetLastError());
            return RS_OK;
        }
    }
    // exchange X_{k,j}: grouped send/recv; the self slice is a device copy
    char* kx = static_cast<char*>(gvr && p > 1 ? L.gv_keys : keys);
    if (gvr && p > 1) vals = L.gv_vals;
    char* rk = static_cast<char*>(L.recv_keys);
    {
        LaunchScope ls("gsd_exchange", st, false);
        RS_NCCL_TRY(ncclGroupStart());
        for (int j = 0; j < p; ++j) {
            if (j == rank) continue;
            const uint64_t sc = cnt[(size_t)rank * p + j], rc = cnt[(size_t)j * p + rank];
            if (sc) {
                RS_NCCL_TRY(ncclSend(kx + soff[j] * key_bytes, sc * key_bytes, ncclUint8, j, c->nccl, st));
                if (hv) RS_NCCL_TRY(ncclSend(vals + soff[j], sc, ncclUint32, j, c->nccl, st));
            }
            if (rc) {
                RS_NCCL_TRY(ncclRecv(rk + roff[j] * key_bytes, rc * key_bytes, ncclUint8, j, c->nccl, st));
                if (hv) RS_NCCL_TRY(ncclRecv(L.recv_vals + roff[j], rc, ncclUint32, j, c->nccl, st));
            }
        }
        RS_NCCL_TRY(ncclGroupEnd());
        const uint64_t self = cnt[(size_t)rank * p + rank];
        if (self) {
            RS_CUDA_TRY(cudaMemcpyAsync(rk + roff[rank] * key_bytes, kx + soff[rank] * key_bytes, self * key_bytes,
                                        cudaMemcpyDeviceToDevice, st));
            if (hv)
                RS_CUDA_TRY(cudaMemcpyAsync(L.recv_vals + roff[rank], vals + soff[rank], self * 4,
                                            cudaMemcpyDeviceToDevice, st));
        }
    }
    // step 5: merge (GVR: local sort of the received concatenation)
    if (gvr) {
        if (total && (sst = local_sort(key_bytes, L.recv_keys, L.recv_vals, total, b, key_bytes * 8, out, vout,
                                       L.local_ws, L.local_ws_bytes, st)) != RS_OK)
            return sst;
    } else if ((sst = merge_runs(key_bytes, L.recv_keys, L.recv_vals, roff, b, out, vout, L, out_cap, st)) != RS_OK) {
        return sst;
    }
    if (n_out) *n_out = total;
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
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

rs_status_t rs_get_unique_id(void* uid128) {
    if (!uid128) return fail(RS_EINVAL, "NULL uid");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    RS_NCCL_TRY(ncclGetUniqueId(&id));
    std::memcpy(uid128, &id, sizeof(id));
    return RS_OK;
}

rs_status_t rs_comm_create(const void* uid128, int nranks, int rank, int cuda_device, void** out) {
    if (!uid128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(RS_EINVAL, "bad comm arguments");
    Comm* c = new (std::nothrow) Comm();
    if (!c) return fail(RS_ENOMEM, "comm allocation");
    c->rank = rank;
    c->nranks = nranks;
    c->device = cuda_device;
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaSetDevice");
    }
    c->h_pinned_words = std::max<size_t>(std::max<size_t>((size_t)nranks * nranks, (size_t)nranks * kIpcWords),
                                          ((size_t)nranks * 256 + 1) * 4) + 64;  // + PR4's piece list
    e = cudaMallocHost(&c->h_pinned, c->h_pinned_words * 8);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaMallocHost");
    }
    e = cudaMalloc(&c->d_hdr, ((size_t)nranks + 1) * kHdrWords * 8);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_ipc, ((size_t)nranks + 1) * kIpcWords * 8);
    if (e != cudaSuccess) {
        if (c->d_hdr) cudaFree(c->d_hdr);
        cudaFreeHost(c->h_pinned);
        delete c;
        return cuda_fail(e, "cudaMalloc (comm header buffer)");
    }
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        cudaFreeHost(c->h_pinned);
        cudaFree(c->d_hdr);
        cudaFree(c->d_ipc);
        delete c;
        return fail(RS_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    *out = c;
    return RS_OK;
}

rs_status_t rs_comm_destroy(void* comm) {
    if (!comm) return RS_OK;
    Comm* c = static_cast<Comm*>(comm);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->d_hdr) cudaFree(c->d_hdr);
    if (c->d_ipc) cudaFree(c->d_ipc);
    delete c;
    return RS_OK;
}

rs_status_t rs_comm_set_oversampling(void* comm, int r) {
    if (!comm || r < 1) return fail(RS_EINVAL, "bad comm / r");
    static_cast<Comm*>(comm)->r = r;
    return RS_OK;
}

rs_status_t rs_comm_last_counts(void* comm, uint64_t* counts) {
    if (!comm || !counts) return fail(RS_EINVAL, "NULL comm / counts");
    const Comm* c = static_cast<Comm*>(comm);
    if (c->last_counts.empty()) return fail(RS_EINVAL, "no sample sort has run on this communicator");
    std::memcpy(counts, c->last_counts.data(), c->last_counts.size() * 8);
    return RS_OK;
}

int rs_comm_rank(void* comm) { return comm ? static_cast<Comm*>(comm)->rank : 0; }
int rs_comm_size(void* comm) { return comm ? static_cast<Comm*>(comm)->nranks : 1; }

// ---------------------------------------------------------- emulation ----
}  // extern "C"

namespace rs {
// GSD (mode 0, oversampling r) or GER (mode 1, s draws per rank, seed) over p
// ranks held on this GPU: every rank's steps, device copies in place of NCCL
static rs_status_t emulate(int mode, int key_bytes, int p, int r, size_t ger_s, uint64_t seed, int digit_bits,
                           void* const* keys, uint32_t* const* vals, const size_t* n, void* const* out_keys,
                           uint32_t* const* out_vals, size_t out_cap, size_t* n_out, uint64_t* splitters,
                           uint64_t* counts, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (p < 1 || r < 1 || !keys || !n || !out_keys || !n_out) return fail(RS_EINVAL, "bad emulate arguments");
    if (digit_bits != 8 && digit_bits != 16) return fail(RS_EINVAL, "digit_bits must be 8 or 16");
    if (key_bytes != 4 && key_bytes != 8) return fail(RS_EINVAL, "key_bytes must be 4 or 8");
    const bool hv = vals != nullptr;
    const size_t s = (size_t)r * p;
    if (mode == 0 && (size_t)p * s > (size_t)kMaxSample) return fail(RS_EINVAL, "r*p^2 exceeds 8192");
    size_t n_max = 0;
    std::vector<uint64_t> noff(p + 1, 0);
    for (int k = 0; k < p; ++k) {
        if (n[k] >= (1ull << 32)) return fail(RS_EINVAL, "n >= 2^32");
        if (n[k] && (!keys[k] || !aligned16(keys[k]) || (hv && (!vals[k] || !aligned16(vals[k])))))
            return fail(RS_EINVAL, "NULL / misaligned block");
        n_max = std::max(n_max, n[k]);
        noff[k + 1] = noff[k] + n[k];
    }
    const uint64_t n_total = noff[p];
    const size_t gs = mode >= 1 ? (ger_s ? ger_s : ger_default_s(n_total)) : 0;
    const size_t M = mode >= 1 ? ger_draws(gs, p) : 0;
    const GsdLayout L = gsd_layout(ws, key_bytes, hv, n_max, out_cap, digit_bits, p, r, 1, M, mode == 2);
    if (!ws || ws_bytes < L.bytes) return fail(RS_EINVAL, "emulate workspace too small: need " + std::to_string(L.bytes));
    rs_status_t sst;
    for (int k = 0; k < p && mode != 2; ++k)  // step 1 (GVR sorts last)
        if (n[k] && (sst = local_sort(key_bytes, keys[k], hv ? vals[k] : nullptr, n[k], digit_bits, key_bytes * 8,
                                      keys[k], hv ? vals[k] : nullptr, L.local_ws, L.local_ws_bytes, st)) != RS_OK)
            return sst;
    if (mode >= 1) {  // GER/GVR steps 2-3: the draws of every rank into one array (= the all-reduce)
        if (M) {
            RS_CUDA_TRY(cudaMemcpyAsync(L.ger_off, noff.data(), (p + 1) * 8, cudaMemcpyHostToDevice, st));
            RS_CUDA_TRY(cudaMemsetAsync(L.ger_key, 0, M * 8, st));
            RS_CUDA_TRY(cudaMemsetAsync(L.ger_q, 0, M * 8, st));
            for (int k = 0; k < p; ++k)
                if ((sst = launch_ger_draw(key_bytes, keys[k], noff[k], n[k], n_total, seed, M, L.ger_key, L.ger_q,
                                           st)) != RS_OK)
                    return sst;
            if ((sst = ger_splitters(L, M, gs, p, n_total, L.splitters, st)) != RS_OK) return sst;
        }
    } else {
    for (int k = 0; k < p; ++k)  // step 2 (the all-gather is the slot layout)
        if ((sst = launch_sample(key_bytes, keys[k], n[k], k, (int)s, L.samp_all + (size_t)k * s, st)) != RS_OK)
            return sst;
    if ((sst = launch_splitters(L.samp_all, (int)(p * s), (int)s, p, L.splitters, st)) != RS_OK) return sst;
    }
    if (mode == 2) {  // GVR step 3: partition each block by destination (in place: the blocks are scratch)
        RS_CUDA_TRY(cudaMemsetAsync(L.counts_all, 0, (size_t)p * p * 8, st));
        for (int k = 0; k < p; ++k) {
            if (p == 1) {
                std::vector<uint64_t> one(1, n[k]);
                RS_CUDA_TRY(cudaMemcpyAsync(L.counts_all, one.data(), 8, cudaMemcpyHostToDevice, st));
                RS_CUDA_TRY(cudaStreamSynchronize(st));
                break;
            }
            if ((sst = gvr_partition(L, key_bytes, keys[k], hv ? vals[k] : nullptr, n[k], k, p, L.splitters,
                                     L.counts_all + (size_t)k * p, st)) != RS_OK)
                return sst;
            if (n[k]) {
                RS_CUDA_TRY(cudaMemcpyAsync(keys[k], L.gv_keys, n[k] * key_bytes, cudaMemcpyDeviceToDevice, st));
                if (hv) RS_CUDA_TRY(cudaMemcpyAsync(vals[k], L.gv_vals, n[k] * 4, cudaMemcpyDeviceToDevice, st));
            }
        }
    } else {
        for (int k = 0; k < p; ++k)  // step 4
            if ((sst = launch_split(key_bytes, keys[k], n[k], k, p, L.splitters, L.counts_all + (size_t)k * p,
                                    st)) != RS_OK)
                return sst;
    }
    std::vector<uint64_t> cnt((size_t)p * p);
    std::vector<Comp> spl(std::max(1, p - 1));
    RS_CUDA_TRY(cudaMemcpyAsync(cnt.data(), L.counts_all, cnt.size() * 8, cudaMemcpyDeviceToHost, st));
    if (p > 1)
        RS_CUDA_TRY(cudaMemcpyAsync(spl.data(), L.splitters, (p - 1) * sizeof(Comp), cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    if (counts) std::memcpy(counts, cnt.data(), cnt.size() * 8);
    if (splitters)
        for (int i = 0; i + 1 < p; ++i) {
            splitters[3 * i] = spl[i].key;
            splitters[3 * i + 1] = spl[i].rank;
            splitters[3 * i + 2] = spl[i].pos == kPosInf ? ~0ull : spl[i].pos;
        }
    std::vector<uint64_t> cut((size_t)p * (p + 1));
    for (int k = 0; k < p; ++k) {
        cut[(size_t)k * (p + 1)] = 0;
        for (int j = 0; j < p; ++j) cut[(size_t)k * (p + 1) + j + 1] = cut[(size_t)k * (p + 1) + j] + cnt[(size_t)k * p + j];
    }
    {
        const std::vector<uint64_t> caps(p, out_cap);
        std::vector<uint64_t> so(p + 1), ro(p + 1);
        for (int j = 0; j < p; ++j) {
            uint64_t tot = 0;
            if ((sst = rs_gsd_exchange_plan(p, j, cnt.data(), caps.data(), so.data(), ro.data(), &tot)) != RS_OK)
                return sst;
            n_out[j] = tot;
        }
    }
    if (mode != 2 && options().gsd_merge >= 2 && options().gsd_pull && p > 1) {  // pull merge: blocks read in place
        for (int j = 0; j < p; ++j) {
            std::vector<const void*> rk(p);
            std::vector<const uint32_t*> rv(hv ? p : 0);
            std::vector<uint64_t> len(p);
            for (int k = 0; k < p; ++k) {
                const uint64_t so = cut[(size_t)k * (p + 1) + j];
                len[k] = cnt[(size_t)k * p + j];
                rk[k] = static_cast<const char*>(keys[k]) + so * key_bytes;
                if (hv) rv[k] = vals[k] + so;
            }
            LaunchScope ls("gsd_pull_merge", st, false);
            if ((sst = pull_merge(key_bytes, rk, rv, len, L, out_cap, out_keys[j], hv ? out_vals[j] : nullptr,
                                  st)) != RS_OK)
                return sst;
        }
        RS_CUDA_TRY(cudaGetLastError());
        return RS_OK;
    }
    for (int j = 0; j < p; ++j) {  // step 4 exchange + step 5 merge, rank by rank
        char* rk = static_cast<char*>(L.recv_keys);
        uint64_t off = 0;
        std::vector<uint64_t> roff(1, 0);
        {
            LaunchScope ls("gsd_exchange", st, false);
            for (int k = 0; k < p; ++k) {
                const uint64_t c = cnt[(size_t)k * p + j];
                if (c) {
                    const uint64_t so = cut[(size_t)k * (p + 1) + j];
                    RS_CUDA_TRY(cudaMemcpyAsync(rk + off * key_bytes, static_cast<char*>(keys[k]) + so * key_bytes,
                                                c * key_bytes, cudaMemcpyDeviceToDevice, st));
                    if (hv)
                        RS_CUDA_TRY(cudaMemcpyAsync(L.recv_vals + off, vals[k] + so, c * 4, cudaMemcpyDeviceToDevice, st));
                    off += c;
                }
                roff.push_back(off);
            }
        }
        if (mode == 2) {  // GVR step 4: local sort of the received concatenation
            if (off && (sst = local_sort(key_bytes, L.recv_keys, L.recv_vals, off, digit_bits, key_bytes * 8,
                                         out_keys[j], hv ? out_vals[j] : nullptr, L.local_ws, L.local_ws_bytes,
                                         st)) != RS_OK)
                return sst;
        } else if ((sst = merge_runs(key_bytes, L.recv_keys, L.recv_vals, roff, digit_bits, out_keys[j],
                                     hv ? out_vals[j] : nullptr, L, out_cap, st)) != RS_OK) {
            return sst;
        }
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}
}  // namespace rs

extern "C" {

size_t rs_gsd_emulate_ws_bytes(int key_bytes, int val_bytes, int p, int r, int digit_bits, size_t n_max,
                               size_t out_cap) {
    if (p < 1 || r < 1) return 0;
    return gsd_layout(nullptr, key_bytes, val_bytes != 0, n_max, out_cap, digit_bits, p, r, 1).bytes;
}

rs_status_t rs_gsd_emulate(int key_bytes, int p, int r, int digit_bits, void* const* keys, uint32_t* const* vals,
                           const size_t* n, void* const* out_keys, uint32_t* const* out_vals, size_t out_cap,
                           size_t* n_out, uint64_t* splitters, uint64_t* counts, void* ws, size_t ws_bytes,
                           void* stream) {
    return emulate(0, key_bytes, p, r, 0, 0, digit_bits, keys, vals, n, out_keys, out_vals, out_cap, n_out,
                   splitters, counts, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

size_t rs_ger_emulate_ws_bytes(int key_bytes, int val_bytes, int p, size_t s, int digit_bits, size_t n_max,
                               size_t out_cap) {
    if (p < 1) return 0;
    const size_t gs = s ? s : ger_default_s((uint64_t)n_max * p);
    return gsd_layout(nullptr, key_bytes, val_bytes != 0, n_max, out_cap, digit_bits, p, 1, 1, ger_draws(gs, p)).bytes;
}

rs_status_t rs_ger_emulate(int key_bytes, int p, size_t s, uint64_t seed, int digit_bits, void* const* keys,
                           uint32_t* const* vals, const size_t* n, void* const* out_keys, uint32_t* const* out_vals,
                           size_t out_cap, size_t* n_out, uint64_t* splitters, uint64_t* counts, void* ws,
                           size_t ws_bytes, void* stream) {
    return emulate(1, key_bytes, p, 1, s, seed, digit_bits, keys, vals, n, out_keys, out_vals, out_cap, n_out,
                   splitters, counts, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

size_t rs_gvr_emulate_ws_bytes(int key_bytes, int val_bytes, int p, size_t s, int digit_bits, size_t n_max,
                               size_t out_cap) {
    if (p < 1) return 0;
    const size_t gs = s ? s : ger_default_s((uint64_t)n_max * p);
    return gsd_layout(nullptr, key_bytes, val_bytes != 0, n_max, out_cap, digit_bits, p, 1, 1, ger_draws(gs, p), true)
        .bytes;
}

rs_status_t rs_gvr_emulate(int key_bytes, int p, size_t s, uint64_t seed, int digit_bits, void* const* keys,
                           uint32_t* const* vals, const size_t* n, void* const* out_keys, uint32_t* const* out_vals,
                           size_t out_cap, size_t* n_out, uint64_t* splitters, uint64_t* counts, void* ws,
                           size_t ws_bytes, void* stream) {
    return emulate(2, key_bytes, p, 1, s, seed, digit_bits, keys, vals, n, out_keys, out_vals, out_cap, n_out,
                   splitters, counts, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

size_t rs_ger_capacity(size_t n_local_max, int p, size_t s) {
    if (p < 1) return 0;
    return ger_capacity_for(n_local_max, p, s ? s : ger_default_s((uint64_t)n_local_max * p));
}

size_t rs_ger_default_s(uint64_t n_total) { return ger_default_s(n_total); }

rs_status_t rs_comm_set_sampling(void* comm, int mode, size_t s, uint64_t seed) {
    if (!comm || mode < 0 || mode > 5) return fail(RS_EINVAL, "bad comm / sampling mode");
    Comm* c = static_cast<Comm*>(comm);
    c->sampling = mode;
    c->ger_s = s;
    c->ger_seed = seed;
    return RS_OK;
}

}  // extern "C"
