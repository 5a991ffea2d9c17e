// extern "C" entry points of librsort.so (declared and documented in
// include/rsort.h).  Validation happens here, before anything is enqueued.
#include <string>

#include "gsd.h"
#include "runtime.h"

using namespace rs;

namespace {

rs_status_t check_common(int key_bytes, const void* keys, const void* vals, bool want_vals, size_t n, int b,
                         const void* out, const void* vout) {
    if (b != 8 && b != 16) return fail(RS_EINVAL, "digit_bits must be 8 or 16 (got " + std::to_string(b) + ")");
    if (key_bytes != 4 && key_bytes != 8) return fail(RS_EINVAL, "key_bytes must be 4 or 8");
    if (n >= (1ull << 32)) return fail(RS_EINVAL, "n must be < 2^32 per GPU");
    if (n == 0) return RS_OK;
    if (!keys || !out) return fail(RS_EINVAL, "NULL key pointer with n > 0");
    if (want_vals && (!vals || !vout)) return fail(RS_EINVAL, "NULL value pointer with n > 0");
    if (!aligned16(keys) || !aligned16(out)) return fail(RS_EINVAL, "key pointers must be 16-byte aligned");
    if (want_vals && (!aligned16(vals) || !aligned16(vout)))
        return fail(RS_EINVAL, "value pointers must be 16-byte aligned");
    return RS_OK;
}

rs_status_t sort_entry(int key_bytes, void* keys, uint32_t* vals, bool want_vals, size_t n, int b, void* comm,
                       void* out, uint32_t* vout, size_t out_cap, size_t* n_out, void* ws, size_t ws_bytes,
                       void* stream) {
    NvtxRange nr(comm ? "rsort.sort.collective" : "rsort.sort");
    rs_status_t s = check_common(key_bytes, keys, vals, want_vals, n, b, out, vout);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // collective: a rank whose arguments fail still takes part in the header
    // exchange, so every rank returns RS_EINVAL instead of the others hanging
    if (comm)
        return gsd_sort(static_cast<Comm*>(comm), key_bytes, keys, want_vals ? vals : nullptr, want_vals, n, b, out,
                        want_vals ? vout : nullptr, out_cap, n_out, ws, ws_bytes, st, s);
    if (s != RS_OK) return s;
    if (out_cap < n) return fail(RS_ECAPACITY, "out_cap < n");
    const size_t need = local_ws_bytes(key_bytes, want_vals, n, b);
    if (n && (!ws || ws_bytes < need))
        return fail(RS_EINVAL, "workspace too small: need " + std::to_string(need) + " bytes");
    if (n && !aligned16(ws)) return fail(RS_EINVAL, "workspace must be 16-byte aligned");
    if (n_out) *n_out = n;
    return local_sort(key_bytes, keys, want_vals ? vals : nullptr, n, b, key_bytes * 8, out,
                      want_vals ? vout : nullptr, ws, ws_bytes, st);
}

}  // namespace

extern "C" {

size_t rs_workspace_bytes(int key_bytes, int val_bytes, size_t n, int digit_bits, void* comm) {
    if ((key_bytes != 4 && key_bytes != 8) || (val_bytes != 0 && val_bytes != 4) ||
        (digit_bits != 8 && digit_bits != 16))
        return 0;
    if (comm) return gsd_ws_bytes(static_cast<Comm*>(comm), key_bytes, val_bytes != 0, n, digit_bits);
    return local_ws_bytes(key_bytes, val_bytes != 0, n, digit_bits);
}

size_t rs_output_capacity(size_t n_local_max, void* comm) {
    if (!comm) return n_local_max;
    return gsd_capacity(static_cast<Comm*>(comm), n_local_max);
}

rs_status_t rs_sort_u32(uint32_t* keys, size_t n, int digit_bits, void* comm, uint32_t* out, size_t out_cap,
                        size_t* n_out, void* ws, size_t ws_bytes, void* stream) {
    return sort_entry(4, keys, nullptr, false, n, digit_bits, comm, out, nullptr, out_cap, n_out, ws, ws_bytes,
                      stream);
}

rs_status_t rs_sort_u64(uint64_t* keys, size_t n, int digit_bits, void* comm, uint64_t* out, size_t out_cap,
                        size_t* n_out, void* ws, size_t ws_bytes, void* stream) {
    return sort_entry(8, keys, nullptr, false, n, digit_bits, comm, out, nullptr, out_cap, n_out, ws, ws_bytes,
                      stream);
}

rs_status_t rs_sort_pairs_u64_u32(uint64_t* keys, uint32_t* vals, size_t n, int digit_bits, void* comm,
                                  uint64_t* out_keys, uint32_t* out_vals, size_t out_cap, size_t* n_out, void* ws,
                                  size_t ws_bytes, void* stream) {
    return sort_entry(8, keys, vals, true, n, digit_bits, comm, out_keys, out_vals, out_cap, n_out, ws, ws_bytes,
                      stream);
}

rs_status_t rs_sort_bits(int key_bytes, void* keys, uint32_t* vals, size_t n, int digit_bits, int end_bit,
                         void* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes, void* stream) {
    rs_status_t s = check_common(key_bytes, keys, vals, vals != nullptr, n, digit_bits, out_keys, out_vals);
    if (s != RS_OK) return s;
    if (end_bit < 1 || end_bit > key_bytes * 8) return fail(RS_EINVAL, "end_bit out of range");
    if (n == 0) return RS_OK;
    const size_t need = local_ws_bytes(key_bytes, vals != nullptr, n, digit_bits);
    if (!ws || ws_bytes < need) return fail(RS_EINVAL, "workspace too small: need " + std::to_string(need));
    if (!aligned16(ws)) return fail(RS_EINVAL, "workspace must be 16-byte aligned");
    return local_sort(key_bytes, keys, vals, n, digit_bits, end_bit, out_keys, out_vals, ws, ws_bytes,
                      static_cast<cudaStream_t>(stream));
}

rs_status_t rs_digit_histogram(int key_bytes, const void* keys, size_t n, int digit_bits, uint32_t* hist, void* ws,
                               size_t ws_bytes, void* stream) {
    rs_status_t s = check_common(key_bytes, keys, nullptr, false, n, digit_bits, keys, nullptr);
    if (s != RS_OK) return s;
    if (!hist) return fail(RS_EINVAL, "NULL hist");
    return digit_histogram(key_bytes, keys, n, digit_bits, hist, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
