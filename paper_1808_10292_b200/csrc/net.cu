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
//   4 a one-word all-reduce orders the stages (nobody overwrites a block a peer
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

#define RS_NCCL_TRY3(expr)                                                             \
    do {                                                                               \
        ncclResult_t r_ = (expr);                                                      \
        if (r_ != ncclSuccess)                                                         \
            return fail(RS_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
    } while (0)

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
rs_status_t net_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, size_t n, int b, void* out, uint32_t* vout,
                     size_t* n_out, void* ws, cudaStream_t st) {
    const int p = c->nranks, rank = c->rank;
    const bool hv = vals != nullptr;
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
    // map every peer's workspace; the all-gather also orders all local sorts before any read
    uint64_t* h = c->h_pinned;
    std::memset(h, 0, kIpcWords * 8);
    h[18] = ipc_export(ws, h, &h[8]) == RS_OK ? 1 : 0;
    RS_CUDA_TRY(cudaMemcpyAsync(c->d_ipc, h, kIpcWords * 8, cudaMemcpyHostToDevice, st));
    RS_NCCL_TRY3(ncclAllGather(c->d_ipc, c->d_ipc + kIpcWords, kIpcWords, ncclUint64, c->nccl, st));
    RS_CUDA_TRY(cudaMemcpyAsync(h, c->d_ipc + kIpcWords, (size_t)p * kIpcWords * 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<char*> peer_ws(p, nullptr);
    bool ok = true;
    for (int k = 0; k < p; ++k) ok = ok && h[(size_t)k * kIpcWords + 18] == 1;
    for (int k = 0; k < p && ok; ++k) {
        void* base = ws;
        if (k != rank) ok = ipc_open(h + (size_t)k * kIpcWords, h[(size_t)k * kIpcWords + 8], &base) == RS_OK;
        peer_ws[k] = static_cast<char*>(base);
    }
    h[0] = ok ? 0 : 1;
    RS_CUDA_TRY(cudaMemcpyAsync(c->d_ipc, h, 8, cudaMemcpyHostToDevice, st));
    RS_NCCL_TRY3(ncclAllReduce(c->d_ipc, c->d_ipc, 1, ncclUint64, ncclMax, c->nccl, st));
    RS_CUDA_TRY(cudaMemcpyAsync(h, c->d_ipc, 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    if (h[0]) return fail(RS_ECUDA, "BTN/OET across GPUs needs every rank to map every peer's workspace (CUDA IPC)");
    // the peer's copy of a layout pointer: same layout (equal n, b) at the peer's base
    auto at_peer = [&](int k, const void* local) -> const void* {
        if (!local) return nullptr;
        return peer_ws[k] + (static_cast<const char*>(local) - static_cast<const char*>(ws));
    };
    const auto S = net_schedule(c->sampling, p);
    std::vector<int> cur(p, 0);
    bool in_out = false;
    {
        LaunchScope ls("net_stages", st, false);
        for (size_t t = 0; t < S.size(); ++t) {
            const NetExchange e = S[t][rank];
            const bool last = t + 1 == S.size();
            if (e.partner >= 0) {
                const int q = e.partner;
                void* dst = last ? out : L.X[cur[rank] ^ 1];
                uint32_t* vdst = hv ? (last ? vout : L.V[cur[rank] ^ 1]) : nullptr;
                const void* Xq = at_peer(q, L.X[cur[q]]);
                const uint32_t* Vq = hv ? static_cast<const uint32_t*>(at_peer(q, L.V[cur[q]])) : nullptr;
                if ((s = merge_split_half(key_bytes, n, rank, q, e.keep_low, L.X[cur[rank]], hv ? L.V[cur[rank]] : nullptr,
                                          Xq, Vq, dst, vdst, L.split, st)) != RS_OK)
                    return s;
                in_out = last;
            }
            for (int k = 0; k < p; ++k)
                if (S[t][k].partner >= 0) cur[k] ^= 1;
            // stage barrier: no rank overwrites a block before its partner has read it
            RS_NCCL_TRY3(ncclAllReduce(c->d_ipc, c->d_ipc, 1, ncclUint64, ncclMax, c->nccl, st));
        }
    }
    if (!in_out) {  // idle in the last stage (OET end ranks)
        RS_CUDA_TRY(cudaMemcpyAsync(out, L.X[cur[rank]], n * key_bytes, cudaMemcpyDeviceToDevice, st));
        if (hv) RS_CUDA_TRY(cudaMemcpyAsync(vout, L.V[cur[rank]], n * 4, cudaMemcpyDeviceToDevice, st));
    }
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
}

// all p ranks on this GPU: keys[k] (N each, read) -> out_keys[j] (N each)
rs_status_t net_emulate(int mode, int key_bytes, int p, int b, void* const* keys, const uint32_t* const* vals, size_t N,
                        void* const* out_keys, uint32_t* const* out_vals, void* ws, size_t ws_bytes, cudaStream_t st) {
    const bool hv = vals != nullptr;
    const size_t per = net_layout(nullptr, key_bytes, hv, N, b).bytes;
    if (!ws || ws_bytes < per * (size_t)p)
        return fail(RS_EINVAL, "net emulate workspace too small: need " + std::to_string(per * p));
    std::vector<NetLayout> L(p);
    for (int k = 0; k < p; ++k) L[k] = net_layout(static_cast<char*>(ws) + per * k, key_bytes, hv, N, b);
    if (N == 0) return RS_OK;
    const auto S = net_schedule(mode, p);
    for (int k = 0; k < p; ++k) {
        void* dst = S.empty() ? out_keys[k] : L[k].X[0];
        uint32_t* vdst = hv ? (S.empty() ? out_vals[k] : L[k].V[0]) : nullptr;
        rs_status_t s = local_sort(key_bytes, keys[k], hv ? vals[k] : nullptr, N, b, key_bytes * 8, dst, vdst,
                                   L[k].local_ws, L[k].local_ws_bytes, st);
        if (s != RS_OK) return s;
    }
    if (S.empty()) return RS_OK;
    std::vector<int> cur(p, 0);
    std::vector<bool> in_out(p, false);
    for (size_t t = 0; t < S.size(); ++t) {
        const bool last = t + 1 == S.size();
        for (int k = 0; k < p; ++k) {
            const NetExchange e = S[t][k];
            if (e.partner < 0) continue;
            const int q = e.partner;
            void* dst = last ? out_keys[k] : L[k].X[cur[k] ^ 1];
            uint32_t* vdst = hv ? (last ? out_vals[k] : L[k].V[cur[k] ^ 1]) : nullptr;
            rs_status_t s = merge_split_half(key_bytes, N, k, q, e.keep_low, L[k].X[cur[k]], hv ? L[k].V[cur[k]] : nullptr,
                                             L[q].X[cur[q]], hv ? L[q].V[cur[q]] : nullptr, dst, vdst, L[k].split, st);
            if (s != RS_OK) return s;
            in_out[k] = last;
        }
        for (int k = 0; k < p; ++k)
            if (S[t][k].partner >= 0) cur[k] ^= 1;
    }
    for (int k = 0; k < p; ++k)
        if (!in_out[k]) {
            RS_CUDA_TRY(cudaMemcpyAsync(out_keys[k], L[k].X[cur[k]], N * key_bytes, cudaMemcpyDeviceToDevice, st));
            if (hv) RS_CUDA_TRY(cudaMemcpyAsync(out_vals[k], L[k].V[cur[k]], N * 4, cudaMemcpyDeviceToDevice, st));
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

size_t rs_net_emulate_ws_bytes(int key_bytes, int val_bytes, int p, int digit_bits, size_t N) {
    if (p < 1 || (key_bytes != 4 && key_bytes != 8) || (digit_bits != 8 && digit_bits != 16)) return 0;
    return rs::net_ws_bytes(key_bytes, val_bytes != 0, N, digit_bits) * (size_t)p;
}

rs_status_t rs_net_emulate(int mode, int key_bytes, int p, int digit_bits, void* const* keys, const uint32_t* const* vals,
                           size_t N, void* const* out_keys, uint32_t* const* out_vals, void* ws, size_t ws_bytes,
                           void* stream) {
    if ((mode != 4 && mode != 5) || p < 1 || !keys || !out_keys || (key_bytes != 4 && key_bytes != 8) ||
        (digit_bits != 8 && digit_bits != 16))
        return rs::fail(RS_EINVAL, "bad BTN/OET emulate arguments");
    if (mode == 4 && (p & (p - 1))) return rs::fail(RS_EINVAL, "BTN needs p a power of two");
    if (N >= (1ull << 32)) return rs::fail(RS_EINVAL, "N >= 2^32");
    for (int k = 0; k < p; ++k)
        if (N && (!keys[k] || !out_keys[k] || (vals && (!vals[k] || !out_vals[k]))))
            return rs::fail(RS_EINVAL, "NULL block");
    return rs::net_emulate(mode, key_bytes, p, digit_bits, keys, vals, N, out_keys, out_vals, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

}  // extern "C"
