// GSD — deterministic regular oversampling sample sort across GPUs
// (Algorithm 1), host side.
#pragma once
#include <nccl.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "runtime.h"

namespace rs {

struct Comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1, device = 0;
    int r = 8;                     // oversampling factor, s = r·p
    int sampling = 0;              // 0 GSD (regular), 1 GER (random),
                                   // 2 GVR, 3 PR4 routing,
                                   // 4 BTN, 5 OET
    size_t ger_s = 0;              // GER: samples per rank (s·p − 1 in all); 0 = 2⌈ω⌉²⌈lg n⌉, ω = lg lg n
    uint64_t ger_seed = 0;         // GER: SplitMix64 seed of the sample draws
    uint64_t* h_pinned = nullptr;  // p*p counts + headers (pinned host)
    uint64_t* d_hdr = nullptr;     // device: this rank's header + all ranks' headers (kHdrWords each)
    uint64_t* d_ipc = nullptr;     // device: IPC handle exchange of the pull merge (kIpcWords per rank)
    size_t h_pinned_words = 0;
    std::vector<uint64_t> last_counts;  // p×p count matrix of the last sort (rs_comm_last_counts)
};

// composite key (key, rank, pos): the unique total order used for sampling
// and splitting (readings R10, R14-R16)
struct Comp {
    uint64_t key;
    uint32_t rank;
    uint32_t pos;
};
constexpr uint32_t kPosInf = 0xFFFFFFFFu;
constexpr int kMaxSample = 8192;  // r·p² composites sorted in one CTA
constexpr int kHdrWords = 12;     // per-rank header of a collective sort call
constexpr int kIpcWords = 20;     // per-rank IPC record: key handle + offset, value handle + offset, ok

// GER's s for n keys in all when the caller did not fix it (reading R30)
size_t ger_default_s(uint64_t n_total);

// PR4 across GPUs (pr.cu; Comm::sampling = 3)
size_t pr_ws_bytes(int key_bytes, bool hv, size_t n_local_max, int p);
rs_status_t pr_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, size_t n, void* out, uint32_t* vout,
                    size_t* n_out, void* ws, const std::vector<uint64_t>& n_all, cudaStream_t st);

// BTN / OET across GPUs (net.cu; Comm::sampling = 4 / 5)
size_t net_ws_bytes(int key_bytes, bool hv, size_t n_local, int b);
rs_status_t net_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, size_t n, int b, void* out, uint32_t* vout,
                     size_t* n_out, void* ws, cudaStream_t st);

size_t gsd_capacity(Comm* c, size_t n_local_max);
size_t gsd_ws_bytes(Comm* c, int key_bytes, bool has_val, size_t n_local_max, int b);
// local_status: the caller's validation of this rank's arguments; a failure on
// any rank makes every rank return RS_EINVAL after the header exchange (no hang)
rs_status_t gsd_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, size_t n, int b, void* out,
                     uint32_t* vout, size_t out_cap, size_t* n_out, void* ws, size_t ws_bytes, cudaStream_t st,
                     rs_status_t local_status = RS_OK);

}  // namespace rs
