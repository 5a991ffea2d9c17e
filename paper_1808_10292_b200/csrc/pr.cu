// PR4 across GPUs — the paper's parallel radix-256 sort (PAPER.md:685-709,
// SPEC.md:206) with its key routing done as NVLink pulls.
//
// For each 8-bit digit t, least significant first:
//   1 every rank sorts its block stably by digit t alone (one local count-sort
//     round, radix.cu local_sort_digit) into S_k and keeps the round's 256 counts;
//   2 the p×256 counts are all-gathered (the paper's 2rpg counter exchange) and the
//     global start of rank k's run of digit d is
//         G[k][d] = Σ_{d'<d} total[d'] + Σ_{k'<k} count[k'][d];
//   3 rank j owns global positions [off_j, off_j + n_j) — the same sizes as its
//     input, so the output is balanced — and copies the overlapping piece of every
//     rank's run from that rank's S_k (peer memory through CUDA IPC, read over
//     NVLink; the paper's 4Ng key routing) into its next-round block.
// After the last round rank j holds positions [off_j, off_j + n_j) of the stable
// sorted order.  Every round moves the keys through HBM twice (local round + pull)
// and across NVLink once: the comparison point of the paper's Observation 4/5
// discussion (GSD moves the data across NVLink once in all).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "gsd.h"

namespace rs {
namespace {

struct Piece {  // one destination-contiguous copy
    uint64_t dst;  // element offset in the destination block
    uint64_t len;
    const void* src_k;
    const uint32_t* src_v;
};

constexpr int kPullChunk = 8192;  // destination elements per CTA

// destination [u·chunk, (u+1)·chunk) of a block fully tiled by `pieces` (sorted by dst)
template <typename K>
__global__ void __launch_bounds__(256) k_pull_pieces(const Piece* __restrict__ pieces, int np, uint64_t n,
                                                     K* __restrict__ dk, uint32_t* __restrict__ dv) {
    const uint64_t b0 = (uint64_t)blockIdx.x * kPullChunk, b1 = min(b0 + kPullChunk, n);
    int lo = 0, hi = np - 1;  // last piece with dst <= b0
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pieces[mid].dst <= b0) lo = mid;
        else hi = mid - 1;
    }
    for (int pi = lo; pi < np; ++pi) {
        const Piece pc = pieces[pi];
        if (pc.dst >= b1) break;
        const uint64_t s0 = max(pc.dst, b0), s1 = min(pc.dst + pc.len, b1);
        const K* sk = static_cast<const K*>(pc.src_k);
        // 4 independent loads in flight per thread (one per iteration was latency-bound)
        constexpr int U = 4;
        for (uint64_t i = s0 + threadIdx.x; i < s1; i += (uint64_t)U * blockDim.x) {
            K r[U];
            uint32_t rv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t j = i + (uint64_t)u * blockDim.x;
                if (j < s1) {
                    r[u] = sk[j - pc.dst];
                    if (dv) rv[u] = pc.src_v[j - pc.dst];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t j = i + (uint64_t)u * blockDim.x;
                if (j < s1) {
                    dk[j] = r[u];
                    if (dv) dv[j] = rv[u];
                }
            }
        }
    }
}

struct PrLayout {
    void* local_ws;
    size_t local_ws_bytes;
    void* s_keys;      // S: the locally sorted block (read by the peers)
    uint32_t* s_vals;
    void* b_keys;      // the next round's block
    uint32_t* b_vals;
    uint32_t* hist_local;  // 256
    uint32_t* hist_all;    // p*256
    Piece* pieces;         // <= p*256 + 1
    size_t bytes;
};

PrLayout pr_layout(void* ws, int key_bytes, bool hv, size_t n, int p) {
    PrLayout L{};
    Carver c(ws);
    L.local_ws_bytes = local_ws_bytes(key_bytes, hv, std::max<size_t>(n, 1), 8);
    L.local_ws = c.take(L.local_ws_bytes);
    L.s_keys = c.take(std::max<size_t>(n, 1) * key_bytes);
    L.s_vals = static_cast<uint32_t*>(hv ? c.take(std::max<size_t>(n, 1) * 4) : nullptr);
    L.b_keys = c.take(std::max<size_t>(n, 1) * key_bytes);
    L.b_vals = static_cast<uint32_t*>(hv ? c.take(std::max<size_t>(n, 1) * 4) : nullptr);
    L.hist_local = static_cast<uint32_t*>(c.take(256 * 4));
    L.hist_all = static_cast<uint32_t*>(c.take((size_t)p * 256 * 4));
    L.pieces = static_cast<Piece*>(c.take(((size_t)p * 256 + 1) * sizeof(Piece)));
    L.bytes = c.used();
    return L;
}

// host: the pieces of rank j's destination range, from the p×256 counts of this
// round (cnt[k*256 + d]), block sizes n[k] and each rank's S pointers
std::vector<Piece> plan_pieces(int p, int j, const std::vector<uint64_t>& cnt, const std::vector<uint64_t>& n,
                               const std::vector<const void*>& sk, const std::vector<const uint32_t*>& sv,
                               int key_bytes) {
    std::vector<uint64_t> off(p + 1, 0);
    for (int k = 0; k < p; ++k) off[k + 1] = off[k] + n[k];
    const uint64_t lo_j = off[j], hi_j = off[j + 1];
    std::vector<Piece> out;
    uint64_t G = 0;  // running global start, digit-major then rank
    for (int d = 0; d < 256; ++d) {
        for (int k = 0; k < p; ++k) {
            const uint64_t c = cnt[(size_t)k * 256 + d];
            if (c) {
                const uint64_t a = std::max(G, lo_j), b = std::min(G + c, hi_j);
                if (a < b) {
                    uint64_t ls = 0;  // local start of run d in S_k
                    for (int dd = 0; dd < d; ++dd) ls += cnt[(size_t)k * 256 + dd];
                    const uint64_t so = ls + (a - G);
                    out.push_back(Piece{a - lo_j, b - a, static_cast<const char*>(sk[k]) + so * key_bytes,
                                        sv.empty() ? nullptr : sv[k] + so});
                }
            }
            G += c;
        }
    }
    return out;
}

rs_status_t launch_pull(int key_bytes, const Piece* d_pieces, int np, uint64_t n, void* dk, uint32_t* dv,
                        cudaStream_t st) {
    if (!n || !np) return RS_OK;
    LaunchScope ls("pr_pull", st);
    const unsigned grid = (unsigned)((n + kPullChunk - 1) / kPullChunk);
    if (key_bytes == 4)
        k_pull_pieces<uint32_t><<<grid, 256, 0, st>>>(d_pieces, np, n, static_cast<uint32_t*>(dk), dv);
    else
        k_pull_pieces<uint64_t><<<grid, 256, 0, st>>>(d_pieces, np, n, static_cast<uint64_t*>(dk), dv);
    return RS_OK;
}

}  // namespace

size_t pr_ws_bytes(int key_bytes, bool hv, size_t n_local_max, int p) {
    return pr_layout(nullptr, key_bytes, hv, n_local_max, p).bytes;
}

// the multi-GPU call (Comm::sampling = 3): header / validation exchanged by the
// caller (gsd_sort), sizes n_all (per rank) known; every rank must be able to map
// every peer's S block (agreed collectively, else RS_ECUDA on every rank)
rs_status_t pr_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, bool hv, size_t n, void* out, uint32_t* vout,
                    size_t* n_out, void* ws, const std::vector<uint64_t>& n_all, cudaStream_t st) {
    NvtxRange nr("rsort.pr4_across_gpus");
    const int p = c->nranks, rank = c->rank;
    const PrLayout L = pr_layout(ws, key_bytes, hv, n, p);
    const int P = key_bytes;  // radix-256 rounds
    // map the peers' S blocks once per call
    const void* mine[2] = {L.s_keys, L.s_vals};
    const int nb = hv ? 2 : 1;
    std::vector<void*> peers;
    rs_status_t s = map_peer_buffers(c, mine, nb, &peers, st);
    if (s != RS_OK) return s;
    std::vector<const void*> sk(p);
    std::vector<const uint32_t*> sv(hv ? p : 0);
    for (int k = 0; k < p; ++k) {
        sk[k] = peers[(size_t)k * nb];
        if (hv) sv[k] = static_cast<const uint32_t*>(peers[(size_t)k * nb + 1]);
    }
    uint64_t* h_hist = c->h + comm_hin_offset();           // p·256 u32 counts
    Piece* h_pieces = reinterpret_cast<Piece*>(h_hist + (size_t)p * 128);  // staged piece list
    void* A = keys;
    uint32_t* Av = vals;
    void* B = L.b_keys;
    uint32_t* Bv = L.b_vals;
    std::vector<uint64_t> cnt((size_t)p * 256);
    for (int t = 0; t < P && s == RS_OK; ++t) {
        if ((s = local_sort_digit(key_bytes, A, Av, n, t, L.s_keys, L.s_vals, L.local_ws, st, L.hist_local)) != RS_OK)
            break;
        // the counter exchange; it also orders every rank's S before any pull
        if ((s = c->tr->allgather(L.hist_local, L.hist_all, 256 * 4, st)) != RS_OK) break;
        RS_CUDA_TRY(cudaMemcpyAsync(h_hist, L.hist_all, (size_t)p * 256 * 4, cudaMemcpyDeviceToHost, st));
        // (this wait also retires the previous round's pull, so the staged piece list is free)
        if ((s = c->wait(st)) != RS_OK) break;
        const uint32_t* h32 = reinterpret_cast<const uint32_t*>(h_hist);
        for (size_t i = 0; i < cnt.size(); ++i) cnt[i] = h32[i];
        const std::vector<Piece> pcs = plan_pieces(p, rank, cnt, n_all, sk, sv, key_bytes);
        if (!pcs.empty()) {
            std::memcpy(h_pieces, pcs.data(), pcs.size() * sizeof(Piece));
            RS_CUDA_TRY(cudaMemcpyAsync(L.pieces, h_pieces, pcs.size() * sizeof(Piece), cudaMemcpyHostToDevice, st));
        }
        if ((s = launch_pull(key_bytes, L.pieces, (int)pcs.size(), n, B, Bv, st)) != RS_OK) break;
        // nobody rewrites its S (next round) before every peer has pulled from it
        if ((s = c->tr->barrier(st)) != RS_OK) break;
        std::swap(A, B);
        std::swap(Av, Bv);
    }
    c->tr->release_unused();
    if (s != RS_OK) return s;
    if (A != out && n) {
        RS_CUDA_TRY(cudaMemcpyAsync(out, A, n * key_bytes, cudaMemcpyDeviceToDevice, st));
        if (hv) RS_CUDA_TRY(cudaMemcpyAsync(vout, Av, n * 4, cudaMemcpyDeviceToDevice, st));
    }
    if (n_out) *n_out = n;
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

}  // namespace rs
