// Host runtime: error strings, launch counting / event timing, device queries.
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <atomic>

#include "runtime.h"

namespace rs {

static thread_local std::string t_last_error;

rs_status_t fail(rs_status_t s, const std::string& msg) {
    t_last_error = msg;
    return s;
}

rs_status_t cuda_fail(cudaError_t e, const char* what) {
    return fail(RS_ECUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

// ------------------------------------------------------------------ timing --
struct Timed {
    std::string name;
    cudaEvent_t e0, e1;
};
static std::mutex g_mu;
static std::vector<Timed> g_timed;
static std::vector<cudaEvent_t> g_pool;
static bool g_timing = false;
static std::atomic<long long> g_launches{0};

static cudaEvent_t pool_get() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void timing_before(const char* name, cudaStream_t stream, int* slot, bool is_kernel) {
    if (is_kernel) g_launches.fetch_add(1, std::memory_order_relaxed);
    *slot = -1;
    if (!g_timing) return;
    std::lock_guard<std::mutex> lk(g_mu);
    Timed t{name, pool_get(), pool_get()};
    cudaEventRecord(t.e0, stream);
    g_timed.push_back(t);
    *slot = static_cast<int>(g_timed.size()) - 1;
}

void timing_after(int slot, cudaStream_t stream) {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(g_timed[slot].e1, stream);
}

Options& options() {
    static Options o;
    return o;
}

static std::mutex g_kmu;
static std::map<std::pair<const void*, int>, int> g_kgrid;  // (kernel, device) -> persistent grid

rs_status_t kernel_setup(const void* kern, int threads, size_t smem, int* grid_cap) {
    int dev = 0;
    RS_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_kmu);
    auto it = g_kgrid.find({kern, dev});
    if (it == g_kgrid.end()) {
        RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0, sms = 0;
        RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
        RS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        it = g_kgrid.emplace(std::make_pair(kern, dev), std::max(1, per_sm) * std::max(1, sms)).first;
    }
    if (grid_cap) *grid_cap = it->second;
    return RS_OK;
}

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

}  // namespace rs

using namespace rs;

extern "C" {

const char* rs_status_string(rs_status_t s) {
    switch (s) {
        case RS_OK: return "RS_OK";
        case RS_EINVAL: return "RS_EINVAL";
        case RS_ECUDA: return "RS_ECUDA";
        case RS_ENCCL: return "RS_ENCCL";
        case RS_ENOMEM: return "RS_ENOMEM";
        case RS_ECAPACITY: return "RS_ECAPACITY";
    }
    return "RS_UNKNOWN";
}

const char* rs_last_error(void) { return t_last_error.c_str(); }

const char* rs_version(void) { return "rsort-b200 0.1 sm_100a"; }

void rs_timing_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_timing = on != 0;
}

void rs_timing_reset(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& t : g_timed) {
        g_pool.push_back(t.e0);
        g_pool.push_back(t.e1);
    }
    g_timed.clear();
    g_launches.store(0);
}

rs_status_t rs_timing_query(const char* prefix, double* total_ms, int* launches) {
    std::lock_guard<std::mutex> lk(g_mu);
    const std::string pre = prefix ? prefix : "";
    double tot = 0;
    int cnt = 0;
    for (auto& t : g_timed) {
        if (t.name.compare(0, pre.size(), pre) != 0) continue;
        cudaError_t e = cudaEventSynchronize(t.e1);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float ms = 0;
        e = cudaEventElapsedTime(&ms, t.e0, t.e1);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
        tot += ms;
        ++cnt;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = cnt;
    return RS_OK;
}

long long rs_launch_count(void) { return g_launches.load(); }

rs_status_t rs_dev_set_option(const char* name, long long value) {
    if (!name || value < 0) return fail(RS_EINVAL, "rs_dev_set_option: bad name / negative value");
    const std::string n(name);
    Options& o = options();
    if (n == "wide_status" && value <= 1) o.wide_status = (int)value;
    else if (n == "gsd_merge" && value <= 3) o.gsd_merge = (int)value;
    else if (n == "gsd_pull" && value <= 1) o.gsd_pull = (int)value;
    else if (n == "small_tiles" && value <= 2) o.small_tiles = (int)value;
    else if (n == "pass_design" && (value == 2 || value == 5)) o.pass_design = (int)value;
    else if (n == "self_check" && value <= 1) o.self_check = (int)value;
    else if (n == "pdl" && value <= 2) o.pdl = (int)value;
    else return fail(RS_EINVAL, "rs_dev_set_option: unknown option or value: " + n);
    return RS_OK;
}

rs_status_t rs_dev_get_option(const char* name, long long* value) {
    if (!name || !value) return fail(RS_EINVAL, "rs_dev_get_option: null argument");
    const std::string n(name);
    const Options& o = options();
    if (n == "wide_status") *value = o.wide_status;
    else if (n == "gsd_merge") *value = o.gsd_merge;
    else if (n == "gsd_pull") *value = o.gsd_pull;
    else if (n == "small_tiles") *value = o.small_tiles;
    else if (n == "pass_design") *value = o.pass_design;
    else if (n == "self_check") *value = o.self_check;
    else if (n == "pdl") *value = o.pdl;
    else if (n == "rank_probe") *value = rank_probe_state();
    else if (n == "tile_u32") *value = tile_keys_for(4, false);
    else if (n == "tile_u64") *value = tile_keys_for(8, false);
    else if (n == "tile_pairs") *value = tile_keys_for(8, true);
    else return fail(RS_EINVAL, "rs_dev_get_option: unknown option: " + n);
    return RS_OK;
}

}  // extern "C"
