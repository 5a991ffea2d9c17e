// CUDA IPC mappings of peers' device buffers (the GSD pull merge reads the
// peers' sorted blocks X_{k,j} straight over NVLink).
//
// A buffer is exported as the IPC handle of its cudaMalloc allocation plus the
// byte offset of the pointer inside it (torch tensors are sub-allocations of
// larger segments).  Opening is reference counted per (device, handle): a handle
// is mapped once however many communicators use it, and unmapped when the last
// user releases it (the NCCL transport releases a mapping as soon as a collective
// call no longer uses it, and all of them when the comm is destroyed).
#include <cuda.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "runtime.h"

namespace rs {
namespace {

using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRange get_range_fn() {
    static GetRange fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<GetRange>(p);
    });
    return fn;
}

struct Mapping {
    void* base;
    int refs;
};
std::mutex g_mu;
std::map<std::pair<int, std::string>, Mapping> g_open;  // (device, handle bytes) -> mapping

}  // namespace

rs_status_t ipc_export(const void* ptr, void* handle64, uint64_t* offset) {
    GetRange fn = get_range_fn();
    if (!fn) return fail(RS_ECUDA, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(RS_EINVAL, "ipc export: pointer is not device memory");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle (VMM / non-cudaMalloc memory?)");
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
    *offset = reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base);
    return RS_OK;
}

// map (or reference again) the allocation of handle64; *base = its mapped start
rs_status_t ipc_open_ref(const void* handle64, void** base) {
    int dev = 0;
    RS_CUDA_TRY(cudaGetDevice(&dev));
    const std::pair<int, std::string> key(dev, std::string(static_cast<const char*>(handle64), 64));
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_open.find(key);
    if (it == g_open.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        void* b = nullptr;
        RS_CUDA_TRY(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
        it = g_open.emplace(key, Mapping{b, 0}).first;
    }
    ++it->second.refs;
    *base = it->second.base;
    return RS_OK;
}

// drop one reference to the mapping at `base`; unmapped at zero
void ipc_release(void* base) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_open.begin(); it != g_open.end(); ++it)
        if (it->second.base == base) {
            if (--it->second.refs <= 0) {
                int cur = 0;
                cudaGetDevice(&cur);
                cudaSetDevice(it->first.first);
                cudaIpcCloseMemHandle(base);
                cudaSetDevice(cur);
                g_open.erase(it);
            }
            return;
        }
}

rs_status_t ipc_open(const void* handle64, uint64_t offset, void** ptr) {
    void* base = nullptr;
    rs_status_t s = ipc_open_ref(handle64, &base);
    if (s == RS_OK) *ptr = static_cast<char*>(base) + offset;
    return s;
}

rs_status_t ipc_close_all() {
    std::lock_guard<std::mutex> lk(g_mu);
    rs_status_t s = RS_OK;
    for (auto& kv : g_open) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first.first);
        if (cudaIpcCloseMemHandle(kv.second.base) != cudaSuccess) s = RS_ECUDA;
        cudaSetDevice(cur);
    }
    g_open.clear();
    return s;
}

}  // namespace rs

extern "C" {

rs_status_t rs_ipc_export(const void* ptr, void* handle64, uint64_t* offset) {
    if (!ptr || !handle64 || !offset) return rs::fail(RS_EINVAL, "rs_ipc_export: NULL argument");
    return rs::ipc_export(ptr, handle64, offset);
}

rs_status_t rs_ipc_open(const void* handle64, uint64_t offset, void** ptr) {
    if (!handle64 || !ptr) return rs::fail(RS_EINVAL, "rs_ipc_open: NULL argument");
    return rs::ipc_open(handle64, offset, ptr);
}

rs_status_t rs_ipc_close_all(void) { return rs::ipc_close_all(); }

}  // extern "C"
