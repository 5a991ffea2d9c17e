// In-process transport: p ranks = p host threads of one process sharing one GPU
// (rs_local_group_create / rs_comm_create_local, include/rsort_dev.h).
//
// Every collective synchronises the calling rank's stream, then meets the other
// ranks at a host barrier, then moves data with device copies from the peers'
// buffers (all on this GPU, so a peer pointer is directly usable) — no kernel
// ever waits on another rank's kernel, so the ranks may run on one GPU in any
// order.  The orchestration above (gsd.cu, pr.cu, net.cu) is the multi-GPU one,
// unchanged: this transport is how a single B200 runs rs_sort_* with a comm at
// p = 2..64.  The host barrier times out (Comm::timeout_ms) instead of hanging
// when a rank never arrives, and the group then stays broken.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "gsd.h"

namespace rs {
namespace {

struct LocalGroup {
    int p = 0, device = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    struct Slot {
        const void* ptr = nullptr;
        const uint64_t* soff = nullptr;
    };
    std::vector<Slot> slot;
    std::vector<bool> joined;

    rs_status_t barrier(int timeout_ms) {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return fail(RS_ECUDA, "local group broken by an earlier barrier timeout");
        const uint64_t g = gen;
        if (++arrived == p) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return RS_OK;
        }
        if (!cv.wait_for(lk, std::chrono::milliseconds(timeout_ms), [&] { return gen != g || broken; })) {
            broken = true;
            cv.notify_all();
            return fail(RS_ECUDA, "local group barrier timed out (a rank did not reach the collective)");
        }
        if (broken && gen == g) return fail(RS_ECUDA, "local group broken by another rank's barrier timeout");
        return RS_OK;
    }
};

__global__ void k_max_rows(const uint64_t* __restrict__ rows, int p, size_t count, uint64_t* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t m = rows[i];
        for (int k = 1; k < p; ++k) m = max(m, rows[(size_t)k * count + i]);
        out[i] = m;
    }
}

class LocalTransport final : public Transport {
public:
    LocalTransport(LocalGroup* g, int rank) : g_(g), rank_(rank) {}
    ~LocalTransport() override {
        if (tmp_) cudaFree(tmp_);
    }
    const char* kind() const override { return "local"; }
    void set_timeout(int ms) override { timeout_ms = ms; }
    int timeout_ms = 600000;

    rs_status_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        RS_CUDA_TRY(cudaStreamSynchronize(st));  // my send buffer is complete
        g_->slot[rank_].ptr = send;
        rs_status_t s = g_->barrier(timeout_ms);
        if (s != RS_OK) return s;
        for (int k = 0; k < g_->p && bytes; ++k)
            RS_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)k * bytes, g_->slot[k].ptr, bytes,
                                        cudaMemcpyDeviceToDevice, st));
        RS_CUDA_TRY(cudaStreamSynchronize(st));
        return g_->barrier(timeout_ms);  // nobody reuses its send buffer before every copy is done
    }

    rs_status_t allreduce_max_u64(uint64_t* buf, size_t count, cudaStream_t st) override {
        const size_t need = (size_t)g_->p * count * 8;
        if (need > tmp_bytes_) {
            if (tmp_) cudaFree(tmp_);
            tmp_ = nullptr;
            tmp_bytes_ = 0;
            RS_CUDA_TRY(cudaMalloc(&tmp_, need));  // test transport: grows once, owned by the comm
            tmp_bytes_ = need;
        }
        rs_status_t s = allgather(buf, tmp_, count * 8, st);
        if (s != RS_OK || !count) return s;
        LaunchScope ls("local_allreduce", st);
        k_max_rows<<<(unsigned)std::min<size_t>((count + 255) / 256, 1024), 256, 0, st>>>(
            static_cast<const uint64_t*>(tmp_), g_->p, count, buf);
        RS_CUDA_TRY(cudaGetLastError());
        return RS_OK;
    }

    rs_status_t alltoallv(const void* send, const std::vector<uint64_t>& soff, void* recv,
                          const std::vector<uint64_t>& roff, size_t elt, cudaStream_t st) override {
        RS_CUDA_TRY(cudaStreamSynchronize(st));
        g_->slot[rank_].ptr = send;
        g_->slot[rank_].soff = soff.data();
        rs_status_t s = g_->barrier(timeout_ms);
        if (s != RS_OK) return s;
        for (int k = 0; k < g_->p; ++k) {
            const uint64_t* so = g_->slot[k].soff;
            const uint64_t len = so[rank_ + 1] - so[rank_];
            if (len != roff[k + 1] - roff[k]) {
                g_->barrier(timeout_ms);
                return fail(RS_EINVAL, "local alltoallv: send/receive counts disagree with rank " + std::to_string(k));
            }
            if (len)
                RS_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + roff[k] * elt,
                                            static_cast<const char*>(g_->slot[k].ptr) + so[rank_] * elt, len * elt,
                                            cudaMemcpyDeviceToDevice, st));
        }
        RS_CUDA_TRY(cudaStreamSynchronize(st));
        return g_->barrier(timeout_ms);
    }

    rs_status_t barrier(cudaStream_t st) override {
        RS_CUDA_TRY(cudaStreamSynchronize(st));
        return g_->barrier(timeout_ms);
    }

    rs_status_t wait(cudaStream_t st, int) override {
        RS_CUDA_TRY(cudaStreamSynchronize(st));
        return RS_OK;
    }

    bool export_buffer(const void* p, uint64_t* rec) override {
        for (int i = 0; i < kPeerRecWords; ++i) rec[i] = 0;
        rec[0] = reinterpret_cast<uintptr_t>(p);
        return true;
    }
    rs_status_t open_peer(int, const uint64_t* rec, void** p) override {
        *p = reinterpret_cast<void*>(static_cast<uintptr_t>(rec[0]));
        return RS_OK;
    }


private:
    LocalGroup* g_;
    int rank_;
    void* tmp_ = nullptr;
    size_t tmp_bytes_ = 0;
};

}  // namespace

Transport* make_local_transport(void* group, int rank, rs_status_t* st) {
    LocalGroup* g = static_cast<LocalGroup*>(group);
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (rank < 0 || rank >= g->p || g->joined[rank]) {
            *st = fail(RS_EINVAL, "rs_comm_create_local: bad or duplicate rank");
            return nullptr;
        }
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev != g->device) {
            *st = fail(RS_EINVAL, "rs_comm_create_local: every rank of a local group must use the group's device");
            return nullptr;
        }
        g->joined[rank] = true;
    }
    *st = RS_OK;
    return new LocalTransport(g, rank);
}

int local_group_size(void* group) { return static_cast<LocalGroup*>(group)->p; }

}  // namespace rs

extern "C" {

rs_status_t rs_local_group_create(int p, void** group) {
    if (!group || p < 1 || p > rs::kMaxLocalRanks) return rs::fail(RS_EINVAL, "rs_local_group_create: 1 <= p <= 64");
    auto* g = new (std::nothrow) rs::LocalGroup();
    if (!g) return rs::fail(RS_ENOMEM, "local group allocation");
    g->p = p;
    cudaGetDevice(&g->device);
    g->slot.resize(p);
    g->joined.assign(p, false);
    *group = g;
    return RS_OK;
}

rs_status_t rs_local_group_destroy(void* group) {
    delete static_cast<rs::LocalGroup*>(group);
    return RS_OK;
}

}  // extern "C"
