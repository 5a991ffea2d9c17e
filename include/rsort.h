/*
 * rsort.h — C ABI of the B200-native radix sort / GSD sample sort library
 * (paper_1808_10292_b200/librsort.so).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, Gerbessiotis,
 * "A study of integer sorting on multicores", arXiv 1808.10292):
 *
 *   single GPU (comm == NULL): LSD radix sort of unsigned keys as a sequence of
 *     stable count-sort passes — digit histogram, exclusive prefix of bucket
 *     offsets, stable scatter (SR4; PAPER.md:685-714 PR4/PR2).
 *     digit_bits = 8 is the paper's radix-256 (PR4: 4 passes on u32, 8 on u64);
 *     digit_bits = 16 is radix-65536 (PR2: 2 passes on u32, 4 on u64).
 *   multi GPU (comm != NULL): GSD, deterministic regular oversampling sample sort
 *     (Algorithm 1): local radix sort, regular sample of
 *     s = r·p composite keys per rank, splitters S_i = T[i·s−1], binary-search
 *     split, NCCL all-to-all over NVLink, final p-way merge on each rank.
 *
 * Result order: ascending unsigned.  Sorts are STABLE: equal keys keep input
 * order (pairs: the payload travels with its key).  Across ranks a rank's keys
 * precede equal keys of higher ranks (readings R14-R16).
 *
 * Conventions for every entry point:
 *   - extern "C", plain pointers and sizes; no torch / CUDA types (a `stream`
 *     is a cudaStream_t passed as void*, NULL = legacy default stream).
 *   - Pointers named keys/vals/out/ws are DEVICE pointers (cudaMalloc or torch
 *     CUDA tensors) on the current CUDA device, 16-byte aligned.
 *   - The caller owns all buffers.  The library never allocates device memory
 *     on a sort call: scratch comes from `ws` (size from rs_workspace_bytes).
 *   - Calls are asynchronous on `stream` unless stated; they never abort or
 *     throw.  Exception: the first radix-256 sort on a device runs the
 *     design-5 lane-order probe (about 60 us) on `stream` and waits for it once
 *     (rs_get_option "rank_probe"); inside a stream capture the probe is skipped
 *     and that call uses the ballot design instead.  Arguments are validated before anything is enqueued, so on
 *     RS_EINVAL the inputs are untouched (single GPU: also on RS_ECAPACITY; the
 *     GSD collective detects RS_ECAPACITY after its local sort, so `keys` then
 *     holds the rank's sorted block).  On RS_ECUDA / RS_ENCCL buffer contents
 *     are undefined (and a comm must be destroyed).
 *   - rs_last_error() returns a thread-local message for the last failure.
 *   - n = 0 is a no-op returning RS_OK (a rank with n = 0 still participates
 *     in a collective call).  n must be < 2^32 per GPU.
 */
#ifndef RSORT_H
#define RSORT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* only the declarations below are exported */
#endif

typedef enum {
    RS_OK = 0,
    RS_EINVAL = 1,      /* bad argument: digit_bits ∉ {8,16}, NULL with n>0, misaligned,
                           n >= 2^32, ws too small, collective header mismatch */
    RS_ECUDA = 2,       /* a CUDA launch / runtime call failed */
    RS_ENCCL = 3,       /* an NCCL call failed */
    RS_ENOMEM = 4,      /* host allocation failed (comm creation only) */
    RS_ECAPACITY = 5    /* multi-GPU: out_cap smaller than |Y_j| */
} rs_status_t;

const char* rs_status_string(rs_status_t s);
const char* rs_last_error(void);
/* library version string, e.g. "rsort-b200 0.1 sm_100a" */
const char* rs_version(void);

/* ---------------------------------------------------------------- sizing -- */

/* Bytes of device scratch needed by rs_sort_* for this (key, value) width,
 * local n, digit width and communicator (NULL = single GPU).
 * key_bytes ∈ {4, 8}; val_bytes ∈ {0, 4}.  Returns 0 on an invalid combination. */
size_t rs_workspace_bytes(int key_bytes, int val_bytes, size_t n, int digit_bits, void* comm);

/* Multi-GPU: capacity each rank's `out` must have when every rank holds at most
 * n_local_max keys: ⌊(1 + 1/r)·n_local_max⌋ + p (R18, the Lemma
 * `balance` bound PAPER.md:891-955 for this reading).  comm NULL → n_local_max. */
size_t rs_output_capacity(size_t n_local_max, void* comm);

/* ------------------------------------------------------------ single GPU -- */
/* (comm == NULL in rs_sort_*) — keys/out may alias (in-place).  *n_out = n.     */

/* rs_sort_u32: sort n u32 keys.  keys: input (read; clobbered only if out==keys).
 * out: n u32 result.  digit_bits ∈ {8, 16}. */
rs_status_t rs_sort_u32(uint32_t* keys, size_t n, int digit_bits, void* comm,
                        uint32_t* out, size_t out_cap, size_t* n_out,
                        void* ws, size_t ws_bytes, void* stream);

/* rs_sort_u64: sort n u64 keys (8 passes at digit_bits 8, 4 at 16). */
rs_status_t rs_sort_u64(uint64_t* keys, size_t n, int digit_bits, void* comm,
                        uint64_t* out, size_t out_cap, size_t* n_out,
                        void* ws, size_t ws_bytes, void* stream);

/* rs_sort_pairs_u64_u32: stable sort of (u64 key, u32 value) pairs stored as
 * two arrays (SoA).  Values are permuted with their keys; equal keys keep input
 * order.  out_keys/out_vals may alias keys/vals. */
rs_status_t rs_sort_pairs_u64_u32(uint64_t* keys, uint32_t* vals, size_t n, int digit_bits,
                                  void* comm, uint64_t* out_keys, uint32_t* out_vals,
                                  size_t out_cap, size_t* n_out,
                                  void* ws, size_t ws_bytes, void* stream);

/* rs_sort_bits: single-GPU core with an explicit bit range: stable sort by
 * the low `end_bit` bits of the key (digits t = 0 .. ⌈end_bit/b⌉−1, LSD first;
 * end_bit = keybits is the full sort).  After t+1 passes of radix 2^b the array
 * is exactly the paper's array after round t — the hook the
 * per-pass parity tests use.  key_bytes ∈ {4, 8}; vals/out_vals NULL or u32. */
rs_status_t rs_sort_bits(int key_bytes, void* keys, uint32_t* vals, size_t n, int digit_bits,
                         int end_bit, void* out_keys, uint32_t* out_vals,
                         void* ws, size_t ws_bytes, void* stream);

/* rs_digit_histogram: counting step of every pass in ONE read of the keys
 * ("initial counting process", all rounds at once):
 * hist[t*2^b + d] = #{i : (key_i >> t·b) & (2^b − 1) = d}, t < keybits/b.
 * hist: device u32 array of (keybits/b)·2^b entries, overwritten.  Needs
 * ws of rs_workspace_bytes(key_bytes, 0, n, b, NULL). */
rs_status_t rs_digit_histogram(int key_bytes, const void* keys, size_t n, int digit_bits,
                               uint32_t* hist, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------- multi GPU -- */

/* NCCL bootstrap: rank 0 calls rs_get_unique_id, the caller broadcasts the
 * 128 bytes (e.g. torch.distributed.broadcast_object_list), then every rank
 * calls rs_comm_create on its own device.  The comm owns an NCCL communicator,
 * a small pinned host buffer and ~200 KB of device scratch, and the CUDA IPC
 * mappings of peer buffers it opens (a mapping is released as soon as a call no
 * longer uses it; all of them at rs_comm_destroy).  Blocking, collective.
 * (One GPU, several ranks as threads: rs_comm_create_local, rsort_dev.h.) */
rs_status_t rs_get_unique_id(void* uid128);
rs_status_t rs_comm_create(const void* uid128, int nranks, int rank, int cuda_device, void** comm);
rs_status_t rs_comm_destroy(void* comm);
/* GSD oversampling factor r (s = r·p samples per rank; default 8, BASELINE
 * config 4 "oversampling factor 8·p", or the largest r with r·p² <= 8192 below
 * 8).  COLLECTIVE and blocking: every rank calls it with the same r (checked:
 * RS_EINVAL on every rank otherwise, or if r·p² > 8192). */
rs_status_t rs_comm_set_oversampling(void* comm, int r);
/* Sample selection of the sample sort (§3.3): mode 0 = GSD's regular
 * oversampling (default; r from rs_comm_set_oversampling); mode 1 = GER
 * (Algorithm GER): s·p − 1 keys drawn uniformly at random,
 * with replacement, from the concatenation of the locally sorted blocks, by
 * SplitMix64(seed) in counter form — draw i at global position
 * ⌊z_i·n/2^64⌋, z_i = mix(seed + (i+1)·0x9E3779B97F4A7C15); S_i = (i·s)-th
 * smallest composite (key, rank, position).  s = 0 selects the paper's
 * s = 2⌈ω⌉²⌈lg n⌉, ω = lg lg n (n = keys on all ranks).  Everything after the
 * splitters is GSD's.  mode 2 = GVR (Algorithm GVR): the
 * same draws taken from the UNSORTED blocks (positions in the unsorted block),
 * each key sent to the rank of its splitter interval (binary search, then a
 * stable count-sort by destination), and Y_j sorted locally after the exchange
 * (same result, no merge).  Mode, s and seed must match on every rank (checked).
 * The output capacity (rs_output_capacity) then follows Lemma Sampling1 with
 * ρ = 1: exceeding it has probability ≤ 1/n and returns RS_ECAPACITY. */
rs_status_t rs_comm_set_sampling(void* comm, int mode, size_t s, uint64_t seed);
/* (rs_comm_set_sampling is COLLECTIVE and blocking like rs_comm_set_oversampling;
 * GER / GVR need p <= 256.) */
/* mode 3 (not a sample sort) = the paper's PR4 across GPUs:
 * per 8-bit digit, a local count-sort round, an all-gather of the p×256 counts,
 * and each rank pulling from every peer (CUDA IPC over NVLink) the keys whose
 * global rank (SPEC.md:206 formula) falls in its range; rank j ends with exactly
 * its input count of the sorted order (balanced).  digit_bits 8 only; every rank
 * must be able to map its peers' memory (else RS_ECUDA on every rank).
 * modes 4 and 5 (network sorts; costs PAPER.md:717-763):
 * every rank sorts its block locally (the SR-b above), then the ranks run the
 * p-processor merge-split network over their sorted blocks — mode 4 BTN, the
 * lg p (lg p + 1)/2-stage bitonic network (p must be a power of two), mode 5
 * OET, p rounds of odd-even transposition (round t pairs (0,1),(2,3),… for even
 * t, (1,2),(3,4),… for odd t).  In a BTN stage k (1-based), substage j, rank i
 * pairs with i XOR 2^(j−1) and the pair is ascending iff bit k of i is 0; an
 * ascending pair gives the smaller n keys to the lower rank, a descending pair to
 * the higher (R32-R34).  Each rank computes only its own half of the
 * merge, reading its partner's current block in place over NVLink (CUDA IPC;
 * every rank must be able to map its peers' workspace, else RS_ECUDA on every
 * rank).  Every rank must pass the same n (else RS_EINVAL on every rank); rank j
 * ends with positions [j·n, (j+1)·n) of the sorted order, so out_cap ≥ n.  Ties
 * merge the lower-indexed block first: OET keeps pairs stable, BTN only moves
 * each value with its key.  The workspace must be one cudaMalloc'd allocation
 * region (it is exported whole). */
int rs_comm_rank(void* comm);
int rs_comm_size(void* comm);

/* With comm != NULL, rs_sort_* is the GSD collective: every rank calls it with
 * the same key/value types and digit_bits (checked: RS_EINVAL on all ranks on a
 * mismatch).  n may differ per rank.  Rank j receives Y_j, the j-th contiguous
 * slice of the global sorted order, in out[0 .. *n_out).  `keys` (and vals) are
 * used as scratch: they hold X_j, the locally sorted block, on return, also when
 * the call fails because of ANOTHER rank's arguments.  `out` must not overlap
 * `keys` (nor out_vals vals) when p > 1.  GSD (mode 0) blocks the host ONCE per
 * call, on the all-gather of every rank's header and count record; GER / GVR
 * exchange the headers first (twice); *n_out is valid on return.  Receive
 * capacity: out_cap < |Y_j| on any rank → RS_ECAPACITY on every rank.  Argument
 * errors on any rank (bad pointers, digit width, workspace too small, mismatched
 * types or settings) are agreed on from the all-gathered headers: every rank
 * returns RS_EINVAL, none hangs (a rank that fails its own checks still takes
 * part in every exchange with an empty block).  A peer that dies, or an NCCL
 * asynchronous error, turns a blocking wait into RS_ENCCL after the comm's
 * timeout (rsort_dev.h rs_comm_set_timeout, default 600 s); the comm is then
 * unusable and must be destroyed. */

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RSORT_H */
