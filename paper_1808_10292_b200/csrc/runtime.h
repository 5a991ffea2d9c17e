// Host-side runtime shared by the rsort translation units: error state,
// per-kernel timing registry, device properties, workspace carving.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rsort.h"
#include "../../include/rsort_dev.h"

namespace rs {

// thread-local last-error message; returns `s` for tail calls
rs_status_t fail(rs_status_t s, const std::string& msg);
rs_status_t cuda_fail(cudaError_t e, const char* what);
#define RS_CUDA_TRY(expr)                                        \
    do {                                                         \
        cudaError_t e_ = (expr);                                 \
        if (e_ != cudaSuccess) return ::rs::cuda_fail(e_, #expr); \
    } while (0)

// Kernel launch bookkeeping: counts every launch; when timing is enabled,
// brackets it with events on `stream` under `name`.
void timing_before(const char* name, cudaStream_t stream, int* slot, bool is_kernel);
void timing_after(int slot, cudaStream_t stream);
struct LaunchScope {
    int slot = -1;
    cudaStream_t st;
    LaunchScope(const char* name, cudaStream_t s, bool is_kernel = true) : st(s) {
        timing_before(name, s, &slot, is_kernel);
    }
    ~LaunchScope() { timing_after(slot, st); }
};

int sm_count();

// NVTX range over a host-side phase of a call (header-only NVTX 3: a no-op unless a
// profiler injects itself), e.g. "rsort.gsd.exchange"
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// process-wide test / tuning knobs (include/rsort_dev.h rs_dev_set_option); read
// once per call, written only between calls
struct Options {
    std::atomic<int> wide_status{0};   // force 64-bit look-back status words (tests)
    std::atomic<int> gsd_merge{3};     // GSD step 5: 0 all-to-all + merge tree, 1 all-to-all + stable radix
                                       // re-sort, 2 pull merge (tree), 3 pull merge as one p-way pass
    std::atomic<int> gsd_pull{1};      // 0: exchange by all-to-all even with gsd_merge 2/3 (the fallback)
    std::atomic<int> small_tiles{0};   // design 5 small-input tiles: 0 auto, 1 never, 2 always
    std::atomic<int> pass_design{5};   // 5 atomic ranks (if the lane-order probe passes, else 2); 2 ballots
    std::atomic<int> self_check{0};    // 1: verify every local sort's output on the device (debug)
    std::atomic<int> pdl{0};           // programmatic dependent launches: 0 auto (radix.cu kPdlMax*), 1 never, 2 always
};
// per (kernel, device): set the kernel's dynamic shared-memory limit to `smem` once
// and return its persistent grid (resident CTAs per SM at `threads` x SMs)
rs_status_t kernel_setup(const void* kern, int threads, size_t smem, int* grid_cap);
// design 5 precondition (radix.cu): -1 not probed yet on this device, 0 failed, 1 passed
int rank_probe_state();
// CUDA IPC mappings (ipc.cu)
rs_status_t ipc_export(const void* ptr, void* handle64, uint64_t* offset);
rs_status_t ipc_open(const void* handle64, uint64_t offset, void** ptr);
// radix-256 tile (keys) of the selected pass design (radix.cu)
int tile_keys_for(int key_bytes, bool has_val);
Options& options();

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// bump allocator over the caller's workspace
struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base(static_cast<char*>(b)) {}
    void* take(size_t bytes) {
        off = align_up(off, 256);
        void* p = base ? base + off : nullptr;
        off += bytes;
        return p;
    }
    size_t used() const { return align_up(off, 256); }
};

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// single-GPU sort core (radix.cu): key_bytes 4/8, vals optional, b 8/16
size_t local_ws_bytes(int key_bytes, bool has_val, size_t n, int b);
rs_status_t local_sort(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int b,
                       int end_bit, void* out, uint32_t* vout, void* ws, size_t ws_bytes,
                       cudaStream_t stream);
// one stable radix-256 count-sort round on digit `pass_t` only (PR4 across GPUs):
// keys_in -> out (out-of-place), the round's 256-bin histogram copied to hist_copy
// (device); ws sized by local_ws_bytes(key_bytes, vals, n, 8)
rs_status_t local_sort_digit(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int pass_t,
                             void* out, uint32_t* vout, void* ws, cudaStream_t st, uint32_t* hist_copy);
rs_status_t digit_histogram(int key_bytes, const void* keys, size_t n, int b, uint32_t* hist, void* ws,
                            size_t ws_bytes, cudaStream_t stream);

}  // namespace rs
