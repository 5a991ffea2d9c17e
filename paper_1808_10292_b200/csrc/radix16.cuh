// Radix-65536 LSD pass (the paper's PR2) for sm_100a.
//
// A 65536-bin per-tile state does not fit a decoupled look-back (a tiles×65536
// status array would outweigh the data), so the pass follows the paper's PR
// structure with G "processors" = G partitions of the array (one CTA each):
//
//   C1 k16_count    H[g][d] = #{keys of partition g with digit d}
//                   (packed 16-bit shared-memory counters, flushed per ≤65535 keys)
//   C2 k16_total    tot[d] = Σ_g H[g][d]
//   C3 k16_scan     base[d] = Σ_{d'<d} tot[d'] (single CTA)
//   C4 k16_offsets  H[g][d] <- base[d] + Σ_{g'<g} H[g'][d]   (the p×r counter matrix
//                   scanned digit-major: SPEC.md:206's rank formula)
//   C5 k16_scatter  each partition streams its keys in chunks: stable in-smem sort
//                   of the chunk by the 16-bit digit (two 8-bit sub-passes with warp
//                   match ranking), then every run of equal digits is written at the
//                   partition's running offset for that digit, which is advanced.
//
// The G×65536 counter matrix is the paper's 2·p·r·g term:
// it is why PR2 trails PR4 (Observation 4), here as on CPUs.
#pragma once
#include "common.cuh"
#include "runtime.h"

namespace rs {

constexpr int kR16 = 65536;

size_t radix16_ws_bytes(int key_bytes, bool has_val, size_t n);
rs_status_t radix16_sort(int key_bytes, const void* keys_in, const uint32_t* vals_in, size_t n, int end_bit,
                         void* out, uint32_t* vout, void* ws, size_t ws_bytes, cudaStream_t st);
rs_status_t radix16_histogram(int key_bytes, const void* keys, size_t n, uint32_t* hist, cudaStream_t st);

}  // namespace rs
