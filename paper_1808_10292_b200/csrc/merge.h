// GSD step 5: stable p-way merge of the received runs (merge.cu).
#pragma once
#include <cstdint>
#include <vector>

#include "runtime.h"

namespace rs {

// scratch (device) bytes for the co-rank table of one 2-way merge of `total` keys
size_t merge_scratch_bytes(size_t total);
// runs: p sorted runs at [roff[k], roff[k+1]) (source-rank order), clobbered;
// tmp: scratch of roff[p] keys (+ values); out: Y_j.  Ties go to the lower run.
rs_status_t merge_runs_tree(int key_bytes, void* runs, uint32_t* vruns, const std::vector<uint64_t>& roff, void* tmp,
                            uint32_t* vtmp, void* out, uint32_t* vout, size_t* split, cudaStream_t st);

// runs at arbitrary addresses rk[k] (+ rv[k]) of len[k] keys, read but not written
// (peers' blocks over NVLink in the pull merge); tmp and out: total keys each.
rs_status_t merge_runs_ptrs(int key_bytes, const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                            const std::vector<uint64_t>& len, void* tmp, uint32_t* vtmp, void* out, uint32_t* vout,
                            size_t* split, cudaStream_t st);

// merged positions [lo, hi) (0 <= lo <= hi <= na + nb) of the stable 2-way merge of
// sorted A and B (ties to A) -> out[0, hi - lo): one half of a merge-split (BTN/OET).
// A and B may be peer memory; split: merge_scratch_bytes(hi - lo).
rs_status_t merge_range(int key_bytes, const void* A, const uint32_t* VA, size_t na, const void* B, const uint32_t* VB,
                        size_t nb, size_t lo, size_t hi, void* out, uint32_t* vout, size_t* split, cudaStream_t st);

// one-pass stable p-way merge (pwmerge.cu): runs at rk[k] (+ rv[k]) of len[k],
// read only (peer memory allowed) -> out (+ vout); 2 <= p <= 32, each run < 2^31.
bool pway_applicable(int p, const std::vector<uint64_t>& len);
size_t pway_scratch_bytes(int key_bytes, uint64_t total, int p);
rs_status_t merge_pway(int key_bytes, const std::vector<const void*>& rk, const std::vector<const uint32_t*>& rv,
                       const std::vector<uint64_t>& len, void* scratch, size_t scratch_bytes, void* out,
                       uint32_t* vout, cudaStream_t st);

}  // namespace rs
