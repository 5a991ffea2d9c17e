// BTN and OET across GPUs — the paper's network sorts over p sorted blocks of
// N = n/p keys (§2, costs PAPER.md:717-763 §3.2; SURVEY §8(f)
// NEXT 4), Comm::sampling 4 (BTN) and 5 (OET).
//
//   1 every rank sorts its block locally (radix.cu local_sort: the paper's SR4)
//     into X[0] of its workspace;
//   2 the workspaces are mapped into every peer (CUDA IPC, one handle each);
//   3 per stage of the network (net_schedule, readings R32/R33) a rank and its
//     partner each compute ONE half of the merge-split of their two blocks: the
//     merge reads the partner's current block in place over NVLink and writes only
//     the rank's own N outputs (merge.cu merge_range: positions [0, N) for the
//     rank that keeps the smaller keys, [N, 2N) for the other) into its other
//     buffer — no copy of the partner's block is ever staged; a rank reads only the
//     part of the partner's block its half needs (about N/2 keys on random data,
//     up to N), against the paper's whole-block exchange (4Ng per round: two inputs
//     and one output through HBM, one block over the link);
//   4 a stage barrier of the transport orders the stages (nobody overwrites a block a peer
//     may still be reading); the last stage writes the caller's output directly.
//
// Readings (R32-R34): standard bitonic network, OET round parity, equal
// block sizes, ties to the lower-indexed block (OET stable, BTN not).
#include <cstring>
#include <string>
#include <vector>

#include "gsd.h"
#include "merge.h"

namespace rs {
namespace {

struct NetLayout {
    void* local_ws;
    size_t local_ws_bytes;
    void* X[2];       // the rank's current / next block (read by the partner)
    uint32_t* V[2];
    size_t* split;
    size_t bytes;
};

NetLayout net_layout(void* ws, int key_bytes, bool hv, size_t n, int b) {
    NetLayout L{};
    Carver c(ws);
    const size_t n1 = std::max<size_t>(n, 1);
    L.local_ws_bytes = local_ws_bytes(key_bytes, hv, n1, b);
    L.local_ws = c.take(L.local_ws_bytes);
    for (int i = 0; i < 2; ++i) {
        L.X[i] = c.take(n1 * key_bytes);
        L.V[i] = static_cast<uint32_t*>(hv ? c.take(n1 * 4) : nullptr);
    }
    L.split = static_cast<size_t*>(c.take(merge_scratch_bytes(n1)));
    L.bytes = c.used();
    return L;
}

}  // namespace

struct NetExchange {  // one rank's role in one stage
    int partner;      // -1: idle this stage
    bool keep_low;    // this rank receives the smaller N keys
};

// stage-by-stage schedule, [stage][rank]; mode 4 BTN (p a power of 2), 5 OET
std::vector<std::vector<NetExchange>> net_schedule(int mode, int p) {
    std::vector<std::vector<NetExchange>> S;
    if (mode == 4) {
        int m = 0;
        while ((1 << m) < p) ++m;
        for (int k = 1; k <= m; ++k)
            for (int j = k; j >= 1; --j) {
                std::vector<NetExchange> st(p);
                for (int i = 0; i < p; ++i) {
                    const int q = i ^ (1 << (j - 1));
                    const bool asc = ((i >> k) & 1) == 0;  // same bit for i and q (j - 1 < k)
                    st[i] = NetExchange{q, (i < q) == asc};
                }
                S.push_back(st);
            }
    } else {
        for (int t = 0; t < p; ++t) {
            std::vector<NetExchange> st(p, NetExchange{-1, false});
            for (int i = t % 2; i + 1 < p; i += 2) {
                st[i] = NetExchange{i + 1, true};
                st[i + 1] = NetExchange{i, false};
            }
            S.push_back(st);
        }
    }
    return S;
}

int net_stage_count(int mode, int p) { return (int)net_schedule(mode, p).size(); }

size_t net_ws_bytes(int key_bytes, bool hv, size_t n_local, int b) {
    return net_layout(nullptr, key_bytes, hv, n_local, b).bytes;
}

// one rank's merge-split half: blocks of the lower / higher index of the pair
static rs_status_t merge_split_half(int key_bytes, size_t N, int self, int partner, bool keep_low, const void* Xs,
                                    const uint32_t* Vs, const void* Xq, const uint32_t* Vq, void* dst, uint32_t* vdst,
                                    size_t* split, cudaStream_t st) {
    const bool self_low = self < partner;
    const void* A = self_low ? Xs : Xq;
    const uint32_t* VA = self_low ? Vs : Vq;
    const void* B = self_low ? Xq : Xs;
    const uint32_t* VB = self_low ? Vq : Vs;
    const size_t lo = keep_low ? 0 : N;
    return merge_range(key_bytes, A, VA, N, B, VB, N, lo, lo + N, dst, vdst, split, st);
}

// the multi-GPU call: header / validation done by gsd_sort (equal n on every rank,
// out_cap >= n, workspaces sized, BTN p a power of 2)
rs_status_t net_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, bool hv, size_t n, int b, void* out,
                     uint32_t* vout, size_t* n_out, void* ws, cudaStream_t st) {
    NvtxRange nr(c->sampling == 4 ? "rsort.btn" : "rsort.oet");
    const int p = c->nranks, rank = c->rank;
    if (n_out) *n_out = n;
    if (p == 1 || n == 0) {
        rs_status_t s = RS_OK;
        if (n) {
            const NetLayout L = net_layout(ws, key_bytes, hv, n, b);
            s = local_sort(key_bytes, keys, vals, n, b, key_bytes * 8, out, vout, L.local_ws, L.local_ws_bytes, st);
        }
        // every rank takes the same branch (n agreed in the header): no collective here
        return s;
    }
    const NetLayout L = net_layout(ws, key_bytes, hv, n, b);
    rs_status_t s = local_sort(key_bytes, keys, vals, n, b, key_bytes * 8, L.X[0], L.V[0], L.local_ws,
                               L.local_ws_bytes, st);
    if (s != RS_OK) return s;
    // map every peer's workspace; the exchange also orders all local sorts before any read
    const void* mine[1] = {ws};
    std::vector<void*> peer_ws;
    if ((s = map_peer_buffers(c, mine, 1, &peer_ws, st)) != RS_OK) return s;
    // the peer's copy of a layout pointer: same layout (equal n, b) at the peer's base
    auto at_peer = [&](int k, const void* local) -> const void* {
        if (!local) return nullptr;
        return static_cast<char*>(peer_ws[k]) + (static_cast<const char*>(local) - static_cast<const char*>(ws));
    };
    const auto S = net_schedule(c->sampling, p);
    std::vector<int> cur(p, 0);
    bool in_out = false;
    {
        LaunchScope ls("net_stages", st, false);
        for (size_t t = 0; t < S.size() && s == RS_OK; ++t) {
            const NetExchange e = S[t][rank];
            const bool last = t + 1 == S.size();
            if (e.partner >= 0) {
                const int q = e.partner;
                void* dst = last ? out : L.X[cur[rank] ^ 1];
                uint32_t* vdst = hv ? (last ? vout : L.V[cur[rank] ^ 1]) : nullptr;
                const void* Xq = at_peer(q, L.X[cur[q]]);
                const uint32_t* Vq = hv ? static_cast<const uint32_t*>(at_peer(q, L.V[cur[q]])) : nullptr;
                s = merge_split_half(key_bytes, n, rank, q, e.keep_low, L.X[cur[rank]], hv ? L.V[cur[rank]] : nullptr,
                                     Xq, Vq, dst, vdst, L.split, st);
                in_out = last;
            }
            for (int k = 0; k < p; ++k)
                if (S[t][k].partner >= 0) cur[k] ^= 1;
            // stage barrier: no rank overwrites a block before its partner has read it
            const rs_status_t bs = c->tr->barrier(st);
            if (s == RS_OK) s = bs;
        }
    }
    c->tr->release_unused();
    if (s != RS_OK) return s;
    if (!in_out) {  // idle in the last stage (OET end ranks)
        RS_CUDA_TRY(cudaMemcpyAsync(out, L.X[cur[rank]], n * key_bytes, cudaMemcpyDeviceToDevice, st));
        if (hv) RS_CUDA_TRY(cudaMemcpyAsync(vout, L.V[cur[rank]], n * 4, cudaMemcpyDeviceToDevice, st));
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

}  // namespace rs

extern "C" {

int rs_net_stages(int mode, int p) {
    if ((mode != 4 && mode != 5) || p < 1 || (mode == 4 && (p & (p - 1)))) return -1;
    return rs::net_stage_count(mode, p);
}

int rs_net_schedule(int mode, int p, int stage, int rank, int* partner, int* keep_low) {
    if (!partner || !keep_low || rs_net_stages(mode, p) < 0 || rank < 0 || rank >= p) return -1;
    const auto S = rs::net_schedule(mode, p);
    if (stage < 0 || stage >= (int)S.size()) return -1;
    *partner = S[stage][rank].partner;
    *keep_low = S[stage][rank].keep_low ? 1 : 0;
    return 0;
}

}  // extern "C"
