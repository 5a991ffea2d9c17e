// GSD — deterministic regular oversampling sample sort across GPUs
// (Algorithm 1), host side: the communicator, the transport
// it talks through, and the collective sort entry points.
//
// One host orchestration (gsd.cu, pr.cu, net.cu) runs over a Transport:
//   NcclTransport  (transport_nccl.cu) one process per GPU: NCCL collectives over
//                  NVLink/NVSwitch for the small exchanges, CUDA IPC mappings of
//                  the peers' buffers for the data (the pull merge reads them in
//                  place), grouped ncclSend/ncclRecv as the all-to-all fallback;
//   LocalTransport (transport_local.cu) p ranks as p host threads of one process
//                  on one GPU: host barriers and device copies.  Nothing on the
//                  device ever waits for another rank (every cross-rank
//                  dependency is a host barrier after a stream synchronisation),
//                  so the ranks may share one GPU; it runs the same orchestration
//                  and kernels as the multi-GPU path, bit for bit.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "runtime.h"

namespace rs {

constexpr int kPeerRecWords = 9;  // a shareable buffer: CUDA IPC handle (8 words) + offset, or a raw pointer

class Transport {
public:
    virtual ~Transport() = default;
    virtual const char* kind() const = 0;
    // stream-ordered: recv[k·bytes, (k+1)·bytes) = rank k's send[0, bytes), every rank
    virtual rs_status_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
    // stream-ordered: buf[i] = max over ranks of buf[i] (in place), count u64 words
    virtual rs_status_t allreduce_max_u64(uint64_t* buf, size_t count, cudaStream_t st) = 0;
    // stream-ordered all-to-all of elements of `elt` bytes with host-known offsets
    // (p + 1 entries each): rank j gets send[soff[j], soff[j+1]) of every rank k at
    // its recv[roff[k], roff[k+1]); every rank's soff/roff must agree
    virtual rs_status_t alltoallv(const void* send, const std::vector<uint64_t>& soff, void* recv,
                                  const std::vector<uint64_t>& roff, size_t elt, cudaStream_t st) = 0;
    // stream-ordered: work enqueued on st after the barrier runs only once every
    // rank's work enqueued before it has completed
    virtual rs_status_t barrier(cudaStream_t st) = 0;
    // host wait for st with failure detection (NCCL asynchronous errors, timeout)
    virtual rs_status_t wait(cudaStream_t st, int timeout_ms) = 0;
    // peer memory: a record (kPeerRecWords) by which every peer can open `p`;
    // false if this buffer cannot be shared (e.g. VMM memory for CUDA IPC)
    virtual bool export_buffer(const void* p, uint64_t* rec) = 0;
    // rank k's exported buffer, mapped here (cached for the life of the transport
    // while it keeps being used; see release_unused)
    virtual rs_status_t open_peer(int k, const uint64_t* rec, void** p) = 0;
    // end of a collective call: unmap the peer buffers this call did not open
    virtual void release_unused() {}
    virtual void set_timeout(int /*ms*/) {}
};

struct Comm {
    Transport* tr = nullptr;       // owned
    int rank = 0, nranks = 1, device = 0;
    int r = 8;                     // oversampling factor, s = r·p (agreed at rs_comm_set_oversampling)
    int sampling = 0;              // 0 GSD (regular), 1 GER (random),
                                   // 2 GVR, 3 PR4 routing,
                                   // 4 BTN, 5 OET
    size_t ger_s = 0;              // GER: samples per rank (s·p − 1 in all); 0 = 2⌈ω⌉²⌈lg n⌉, ω = lg lg n
    uint64_t ger_seed = 0;         // GER: SplitMix64 seed of the sample draws
    int timeout_ms = 600000;       // blocking waits give up (and abort the comm) after this
    // comm-owned scratch (allocated at creation, so a rank whose own arguments are
    // invalid still takes part in every exchange): pinned host words and device bytes
    uint64_t* h = nullptr;
    size_t h_words = 0;
    unsigned char* d = nullptr;
    size_t d_bytes = 0;
    // introspection of the last collective call (rsort_dev.h)
    std::vector<uint64_t> last_counts;     // p×p |X_{k,j}|
    std::vector<uint64_t> last_splitters;  // (p−1)×3 (key, rank, pos)
    int last_host_syncs = 0;
    bool broken = false;                   // a wait failed: the comm must be destroyed

    // host wait for st (counted in last_host_syncs); failure marks the comm broken
    rs_status_t wait(cudaStream_t st);
    // blocking all-gather of `words` host words per rank through the device scratch
    rs_status_t host_allgather(const uint64_t* mine, size_t words, uint64_t* all, cudaStream_t st);
};

// creation of the comm-owned buffers for p ranks (both transports)
rs_status_t comm_init_buffers(Comm* c);
void comm_free_buffers(Comm* c);
Transport* make_nccl_transport(const void* uid128, int nranks, int rank, rs_status_t* st);
Transport* make_local_transport(void* group, int rank, rs_status_t* st);
int local_group_size(void* group);
size_t comm_hin_offset();  // Comm::h words [0, off) stage outgoing copies, [off, h_words) receive

// composite key (key, rank, pos): the unique total order used for sampling
// and splitting (readings R10, R14-R16)
struct Comp {
    uint64_t key;
    uint32_t rank;
    uint32_t pos;
};
constexpr uint32_t kPosInf = 0xFFFFFFFFu;
constexpr int kMaxSample = 8192;  // r·p² composites sorted in one CTA
constexpr int kHdrWords = 16;     // per-rank header of a collective sort call
constexpr int kMaxLocalRanks = 64;

// the comm's device scratch (Comm::d), per rank of the gathered arrays:
//   xg   host all-gathers (send row + p rows of kXWords words)
//   samp GSD sample records: 128-byte header + s composites (send + p rows of bs_max bytes)
//   cnt  count records: p counts, key / value peer records, flags (send + p rows of wc words)
//   spl  the p − 1 splitters
struct CommRegions {
    uint64_t* xg;
    unsigned char* samp;
    size_t bs_max;
    uint64_t* cnt;
    size_t wc;
    Comp* spl;
    size_t bytes;
};
CommRegions comm_regions(const Comm* c);

// GER's s for n keys in all when the caller did not fix it (reading R30)
size_t ger_default_s(uint64_t n_total);

// PR4 across GPUs (pr.cu; Comm::sampling = 3)
size_t pr_ws_bytes(int key_bytes, bool hv, size_t n_local_max, int p);
rs_status_t pr_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, bool hv, size_t n, void* out, uint32_t* vout,
                    size_t* n_out, void* ws, const std::vector<uint64_t>& n_all, cudaStream_t st);

// BTN / OET across GPUs (net.cu; Comm::sampling = 4 / 5)
size_t net_ws_bytes(int key_bytes, bool hv, size_t n_local, int b);
rs_status_t net_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, bool hv, size_t n, int b, void* out,
                     uint32_t* vout, size_t* n_out, void* ws, cudaStream_t st);
int net_stage_count(int mode, int p);

// map every peer's buffers (nb per rank): peers[k·nb + i] = rank k's ptrs[i]
// (rank's own entries are its own pointers); agreed collectively: RS_ECUDA on
// every rank if any rank cannot share or map
rs_status_t map_peer_buffers(Comm* c, const void* const* ptrs, int nb, std::vector<void*>* peers, cudaStream_t st);

size_t gsd_capacity(Comm* c, size_t n_local_max);
size_t gsd_ws_bytes(Comm* c, int key_bytes, bool has_val, size_t n_local_max, int b);
// local_status: the caller's validation of this rank's arguments; a failure on
// any rank makes every rank return RS_EINVAL (no hang)
// has_val: a pair sort (vals may be NULL on a rank with n = 0)
rs_status_t gsd_sort(Comm* c, int key_bytes, void* keys, uint32_t* vals, bool has_val, size_t n, int b, void* out,
                     uint32_t* vout, size_t out_cap, size_t* n_out, void* ws, size_t ws_bytes, cudaStream_t st,
                     rs_status_t local_status = RS_OK);

}  // namespace rs
