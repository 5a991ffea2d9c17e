// Communicator lifecycle and the blocking helpers every collective path shares:
// comm-owned scratch, the host wait with failure detection, host all-gathers of a
// few words, and the collective mapping of peer buffers.  The transports are in
// transport_nccl.cu (one process per GPU) and transport_local.cu (p host threads
// on one GPU).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "gsd.h"

namespace rs {

namespace {
constexpr size_t kXWords = 64;  // per-rank words of a host all-gather
}

size_t comm_hin_offset() { return 1024; }  // h[0, 1024): outgoing staging; h[1024, ...): incoming

// device scratch: [xg: (p+1) x kXWords words][samp: (p+1) x bs_max bytes]
//                 [cnt: (p+1) x wc words][spl: p composites]
CommRegions comm_regions(const Comm* c) {
    const size_t p = (size_t)c->nranks;
    CommRegions R{};
    R.bs_max = 128 + 16 * (size_t)(kMaxSample / c->nranks);  // header + s <= 8192/p composites (r·p² <= 8192)
    R.wc = p + 2 * kPeerRecWords + 2;
    size_t off = 0;
    R.xg = reinterpret_cast<uint64_t*>(c->d + off);
    off += (p + 1) * kXWords * 8;
    R.samp = c->d + off;
    off += (p + 1) * R.bs_max;
    off = align_up(off, 256);
    R.cnt = reinterpret_cast<uint64_t*>(c->d + off);
    off += (p + 1) * R.wc * 8;
    off = align_up(off, 256);
    R.spl = reinterpret_cast<Comp*>(c->d + off);
    off += p * sizeof(Comp);
    R.bytes = align_up(off, 256);
    return R;
}

rs_status_t comm_init_buffers(Comm* c) {
    const size_t p = (size_t)c->nranks;
    const CommRegions R = comm_regions(c);  // sizes only (c->d is still NULL)
    c->d_bytes = R.bytes;
    // incoming: p rows of the largest all-gathered record (PR4: 256 u32 counts = 128 words),
    // then PR4's staged piece list (<= p·256 + 1 pieces of 4 words)
    c->h_words = comm_hin_offset() + p * (kXWords + kHdrWords + R.wc + 128) + (p * 256 + 1) * 4 + 1024;
    cudaError_t e = cudaMalloc(&c->d, c->d_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc (comm scratch)");
    e = cudaMallocHost(&c->h, c->h_words * 8);
    if (e != cudaSuccess) {
        cudaFree(c->d);
        c->d = nullptr;
        return cuda_fail(e, "cudaMallocHost (comm scratch)");
    }
    return RS_OK;
}

void comm_free_buffers(Comm* c) {
    if (c->d) cudaFree(c->d);
    if (c->h) cudaFreeHost(c->h);
    c->d = nullptr;
    c->h = nullptr;
}

rs_status_t Comm::wait(cudaStream_t st) {
    ++last_host_syncs;
    if (broken) return fail(RS_ENCCL, "communicator is broken by an earlier failure; destroy it");
    rs_status_t s = tr->wait(st, timeout_ms);
    if (s != RS_OK) broken = true;
    return s;
}


rs_status_t Comm::host_allgather(const uint64_t* mine, size_t words, uint64_t* all, cudaStream_t st) {
    if (words > kXWords) return fail(RS_EINVAL, "host_allgather: record too long");
    uint64_t* out = h;                       // staging (outgoing)
    uint64_t* in = h + comm_hin_offset();    // incoming
    std::memcpy(out, mine, words * 8);
    uint64_t* d_send = comm_regions(this).xg;
    uint64_t* d_all = d_send + kXWords;
    RS_CUDA_TRY(cudaMemcpyAsync(d_send, out, words * 8, cudaMemcpyHostToDevice, st));
    rs_status_t s = tr->allgather(d_send, d_all, words * 8, st);
    if (s != RS_OK) return s;
    RS_CUDA_TRY(cudaMemcpyAsync(in, d_all, (size_t)nranks * words * 8, cudaMemcpyDeviceToHost, st));
    if ((s = wait(st)) != RS_OK) return s;
    std::memcpy(all, in, (size_t)nranks * words * 8);
    return RS_OK;
}

rs_status_t map_peer_buffers(Comm* c, const void* const* ptrs, int nb, std::vector<void*>* peers, cudaStream_t st) {
    const int p = c->nranks, words = 1 + nb * kPeerRecWords;
    std::vector<uint64_t> mine(words, 0), all((size_t)p * words);
    bool ok = true;
    for (int i = 0; i < nb && ok; ++i) ok = c->tr->export_buffer(ptrs[i], &mine[1 + i * kPeerRecWords]);
    mine[0] = ok ? 1 : 0;
    rs_status_t s = c->host_allgather(mine.data(), words, all.data(), st);
    if (s != RS_OK) return s;
    for (int k = 0; k < p; ++k)
        if (all[(size_t)k * words] != 1)
            return fail(RS_ECUDA, "rank " + std::to_string(k) + " cannot share its buffers with its peers");
    peers->assign((size_t)p * nb, nullptr);
    bool opened = true;
    for (int k = 0; k < p; ++k)
        for (int i = 0; i < nb; ++i) {
            void* q = const_cast<void*>(ptrs[i]);
            if (k != c->rank && opened)
                opened = c->tr->open_peer(k, &all[(size_t)k * words + 1 + i * kPeerRecWords], &q) == RS_OK;
            (*peers)[(size_t)k * nb + i] = q;
        }
    uint64_t f = opened ? 0 : 1;
    std::vector<uint64_t> fl(p);
    if ((s = c->host_allgather(&f, 1, fl.data(), st)) != RS_OK) return s;
    for (int k = 0; k < p; ++k)
        if (fl[k]) return fail(RS_ECUDA, "rank " + std::to_string(k) + " could not map its peers' buffers");
    return RS_OK;
}

// a comm-owned stream for the configuration collectives (never the caller's)
static rs_status_t config_allgather(Comm* c, const uint64_t* mine, size_t words, uint64_t* all) {
    cudaStream_t st = nullptr;
    RS_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    rs_status_t s = c->host_allgather(mine, words, all, st);
    cudaStreamDestroy(st);
    return s;
}

static rs_status_t finish_create(Comm* c, Transport* t, rs_status_t ts, void** out) {
    if (!t) {
        delete c;
        return ts;
    }
    c->tr = t;
    c->r = std::max(1, std::min(8, kMaxSample / (c->nranks * c->nranks)));  // r = 8 (BASELINE c4) while r·p² fits
    rs_status_t s = comm_init_buffers(c);
    if (s != RS_OK) {
        delete c->tr;
        delete c;
        return s;
    }
    *out = c;
    return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" {

rs_status_t rs_comm_create(const void* uid128, int nranks, int rank, int cuda_device, void** out) {
    if (!uid128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(RS_EINVAL, "bad comm arguments");
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    Comm* c = new (std::nothrow) Comm();
    if (!c) return fail(RS_ENOMEM, "comm allocation");
    c->rank = rank;
    c->nranks = nranks;
    c->device = cuda_device;
    rs_status_t ts = RS_OK;
    Transport* t = make_nccl_transport(uid128, nranks, rank, &ts);
    return finish_create(c, t, ts, out);
}

rs_status_t rs_comm_create_local(void* group, int rank, void** out) {
    if (!group || !out) return fail(RS_EINVAL, "rs_comm_create_local: NULL argument");
    Comm* c = new (std::nothrow) Comm();
    if (!c) return fail(RS_ENOMEM, "comm allocation");
    int dev = 0;
    cudaGetDevice(&dev);
    rs_status_t ts = RS_OK;
    Transport* t = make_local_transport(group, rank, &ts);
    if (t) {
        c->rank = rank;
        c->nranks = local_group_size(group);
        c->device = dev;
    }
    return finish_create(c, t, ts, out);
}

rs_status_t rs_comm_destroy(void* comm) {
    if (!comm) return RS_OK;
    Comm* c = static_cast<Comm*>(comm);
    delete c->tr;  // NCCL: destroys the communicator and unmaps every peer buffer it opened
    comm_free_buffers(c);
    delete c;
    return RS_OK;
}

rs_status_t rs_comm_set_oversampling(void* comm, int r) {
    if (!comm) return fail(RS_EINVAL, "NULL comm");
    Comm* c = static_cast<Comm*>(comm);
    const uint64_t p = (uint64_t)c->nranks;
    const uint64_t bad = (r < 1 || (uint64_t)r * p * p > (uint64_t)kMaxSample) ? 1 : 0;
    const uint64_t mine[2] = {(uint64_t)(r < 0 ? 0 : r), bad};
    std::vector<uint64_t> all(2 * p);
    rs_status_t s = config_allgather(c, mine, 2, all.data());
    if (s != RS_OK) return s;
    for (uint64_t k = 0; k < p; ++k) {
        if (all[2 * k + 1]) return fail(RS_EINVAL, "oversampling r must satisfy 1 <= r and r·p² <= 8192 (rank " +
                                                       std::to_string(k) + ")");
        if (all[2 * k] != mine[0]) return fail(RS_EINVAL, "oversampling factor differs on rank " + std::to_string(k));
    }
    c->r = r;
    return RS_OK;
}

rs_status_t rs_comm_set_sampling(void* comm, int mode, size_t s, uint64_t seed) {
    if (!comm) return fail(RS_EINVAL, "NULL comm");
    Comm* c = static_cast<Comm*>(comm);
    const uint64_t p = (uint64_t)c->nranks;
    uint64_t bad = (mode < 0 || mode > 5) ? 1 : 0;
    if ((mode == 1 || mode == 2) && p > 256) bad = 1;  // k_gvr_dest / k_ger_pick keep p splitters in one CTA
    const uint64_t mine[4] = {(uint64_t)mode, (uint64_t)s, seed, bad};
    std::vector<uint64_t> all(4 * p);
    rs_status_t st = config_allgather(c, mine, 4, all.data());
    if (st != RS_OK) return st;
    for (uint64_t k = 0; k < p; ++k) {
        if (all[4 * k + 3]) return fail(RS_EINVAL, "bad sampling mode on rank " + std::to_string(k) +
                                                       " (0..5; GER/GVR need p <= 256)");
        for (int f = 0; f < 3; ++f)
            if (all[4 * k + f] != mine[f])
                return fail(RS_EINVAL, "sampling mode / s / seed differ on rank " + std::to_string(k));
    }
    c->sampling = mode;
    c->ger_s = s;
    c->ger_seed = seed;
    return RS_OK;
}

rs_status_t rs_comm_set_timeout(void* comm, int timeout_ms) {
    if (!comm || timeout_ms < 1) return fail(RS_EINVAL, "bad comm / timeout");
    Comm* c = static_cast<Comm*>(comm);
    c->timeout_ms = timeout_ms;
    c->tr->set_timeout(timeout_ms);
    return RS_OK;
}

rs_status_t rs_comm_last_counts(void* comm, uint64_t* counts) {
    if (!comm || !counts) return fail(RS_EINVAL, "NULL comm / counts");
    const Comm* c = static_cast<Comm*>(comm);
    if (c->last_counts.empty()) return fail(RS_EINVAL, "no sample sort has run on this communicator");
    std::memcpy(counts, c->last_counts.data(), c->last_counts.size() * 8);
    return RS_OK;
}

rs_status_t rs_comm_last_splitters(void* comm, uint64_t* splitters) {
    if (!comm || !splitters) return fail(RS_EINVAL, "NULL comm / splitters");
    const Comm* c = static_cast<Comm*>(comm);
    if (c->last_counts.empty()) return fail(RS_EINVAL, "no sample sort has run on this communicator");
    if (!c->last_splitters.empty())
        std::memcpy(splitters, c->last_splitters.data(), c->last_splitters.size() * 8);
    return RS_OK;
}

int rs_comm_last_host_syncs(void* comm) { return comm ? static_cast<Comm*>(comm)->last_host_syncs : -1; }

int rs_comm_rank(void* comm) { return comm ? static_cast<Comm*>(comm)->rank : 0; }
int rs_comm_size(void* comm) { return comm ? static_cast<Comm*>(comm)->nranks : 1; }

}  // extern "C"
