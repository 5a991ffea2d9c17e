// NCCL + CUDA IPC transport: one process per GPU (rs_get_unique_id /
// rs_comm_create).  The small exchanges (sample records, count records, GER's
// draws, stage barriers) are NCCL collectives over NVLink/NVSwitch on the sort's
// stream; the data moves either by the pull merge reading the peers' blocks in
// place through CUDA IPC mappings (default), or by a grouped ncclSend/ncclRecv
// all-to-all (fallback).  Blocking waits poll the stream together with
// ncclCommGetAsyncError and give up after the comm's timeout, aborting the NCCL
// communicator, so a dead or failing peer turns into RS_ENCCL instead of a hang.
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "gsd.h"

namespace rs {

rs_status_t ipc_export(const void* ptr, void* handle64, uint64_t* offset);
rs_status_t ipc_open_ref(const void* handle64, void** base);
void ipc_release(void* base);

namespace {

#define RS_NCCL_T(expr)                                                                                \
    do {                                                                                               \
        if (!nccl_) return fail(RS_ENCCL, "NCCL communicator aborted by an earlier failure");          \
        ncclResult_t r_ = (expr);                                                                      \
        if (r_ != ncclSuccess) return fail(RS_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
    } while (0)

class NcclTransport final : public Transport {
public:
    NcclTransport(ncclComm_t c, int rank, int p, uint64_t* d_word) : nccl_(c), rank_(rank), p_(p), d_word_(d_word) {}
    ~NcclTransport() override {
        for (auto& kv : maps_) ipc_release(kv.second.base);
        if (nccl_) ncclCommDestroy(nccl_);
        if (d_word_) cudaFree(d_word_);
    }
    const char* kind() const override { return "nccl"; }

    rs_status_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        RS_NCCL_T(ncclAllGather(send, recv, bytes, ncclUint8, nccl_, st));
        return RS_OK;
    }
    rs_status_t allreduce_max_u64(uint64_t* buf, size_t count, cudaStream_t st) override {
        RS_NCCL_T(ncclAllReduce(buf, buf, count, ncclUint64, ncclMax, nccl_, st));
        return RS_OK;
    }
    rs_status_t alltoallv(const void* send, const std::vector<uint64_t>& soff, void* recv,
                          const std::vector<uint64_t>& roff, size_t elt, cudaStream_t st) override {
        const char* s = static_cast<const char*>(send);
        char* r = static_cast<char*>(recv);
        RS_NCCL_T(ncclGroupStart());
        for (int j = 0; j < p_; ++j) {
            if (j == rank_) continue;
            const uint64_t sc = soff[j + 1] - soff[j], rc = roff[j + 1] - roff[j];
            if (sc) RS_NCCL_T(ncclSend(s + soff[j] * elt, sc * elt, ncclUint8, j, nccl_, st));
            if (rc) RS_NCCL_T(ncclRecv(r + roff[j] * elt, rc * elt, ncclUint8, j, nccl_, st));
        }
        RS_NCCL_T(ncclGroupEnd());
        const uint64_t self = soff[rank_ + 1] - soff[rank_];
        if (self)
            RS_CUDA_TRY(cudaMemcpyAsync(r + roff[rank_] * elt, s + soff[rank_] * elt, self * elt,
                                        cudaMemcpyDeviceToDevice, st));
        return RS_OK;
    }
    rs_status_t barrier(cudaStream_t st) override {
        RS_NCCL_T(ncclAllReduce(d_word_, d_word_, 1, ncclUint64, ncclMax, nccl_, st));
        return RS_OK;
    }
    rs_status_t wait(cudaStream_t st, int timeout_ms) override {
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0;; ++spin) {
            const cudaError_t e = cudaStreamQuery(st);
            if (e == cudaSuccess) return RS_OK;
            if (e != cudaErrorNotReady) return cuda_fail(e, "cudaStreamQuery");
            if (!nccl_) return fail(RS_ENCCL, "NCCL communicator aborted by an earlier failure");
            ncclResult_t ar = ncclSuccess;
            if (ncclCommGetAsyncError(nccl_, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
                ncclCommAbort(nccl_);
                nccl_ = nullptr;
                return fail(RS_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
            }
            const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
            if (ms.count() > timeout_ms) {
                ncclCommAbort(nccl_);
                nccl_ = nullptr;
                return fail(RS_ENCCL, "collective wait timed out after " + std::to_string(timeout_ms) +
                                          " ms (a peer is dead or did not enter the call); comm aborted");
            }
            if (spin > 2000) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    // a NULL buffer (a rank with n = 0) travels as the all-zero record: never read
    bool export_buffer(const void* p, uint64_t* rec) override {
        std::memset(rec, 0, kPeerRecWords * 8);
        return !p || ipc_export(p, rec, &rec[8]) == RS_OK;
    }
    rs_status_t open_peer(int k, const uint64_t* rec, void** p) override {
        bool null_rec = true;
        for (int i = 0; i < kPeerRecWords; ++i) null_rec = null_rec && rec[i] == 0;
        if (null_rec) {
            *p = nullptr;
            return RS_OK;
        }
        const std::pair<int, std::string> key(k, std::string(reinterpret_cast<const char*>(rec), 64));
        auto it = maps_.find(key);
        if (it == maps_.end()) {
            void* base = nullptr;
            rs_status_t s = ipc_open_ref(rec, &base);
            if (s != RS_OK) return s;
            it = maps_.emplace(key, Map{base, gen_}).first;
        }
        it->second.used = gen_;
        *p = static_cast<char*>(it->second.base) + rec[8];
        return RS_OK;
    }
    void release_unused() override {
        for (auto it = maps_.begin(); it != maps_.end();) {
            if (it->second.used != gen_) {
                ipc_release(it->second.base);
                it = maps_.erase(it);
            } else {
                ++it;
            }
        }
        ++gen_;
    }

private:
    struct Map {
        void* base;
        uint64_t used;
    };
    ncclComm_t nccl_;
    int rank_, p_;
    uint64_t* d_word_;
    std::map<std::pair<int, std::string>, Map> maps_;  // (peer, handle) -> mapping
    uint64_t gen_ = 1;
};

}  // namespace

Transport* make_nccl_transport(const void* uid128, int nranks, int rank, rs_status_t* st) {
    uint64_t* d_word = nullptr;
    cudaError_t e = cudaMalloc(&d_word, 8);
    if (e != cudaSuccess) {
        *st = cuda_fail(e, "cudaMalloc (barrier word)");
        return nullptr;
    }
    cudaMemset(d_word, 0, 8);
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    ncclComm_t c = nullptr;
    const ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) {
        cudaFree(d_word);
        *st = fail(RS_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        return nullptr;
    }
    *st = RS_OK;
    return new NcclTransport(c, rank, nranks, d_word);
}

}  // namespace rs

extern "C" rs_status_t rs_get_unique_id(void* uid128) {
    if (!uid128) return rs::fail(RS_EINVAL, "NULL uid");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return rs::fail(RS_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(uid128, &id, sizeof(id));
    return RS_OK;
}
