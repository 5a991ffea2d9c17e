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
 * calls rs_comm_create on its own device.  The comm owns an NCCL communicator
 * and a small pinned host buffer.  Blocking, collective. */
rs_status_t rs_get_unique_id(void* uid128);
rs_status_t rs_comm_create(const void* uid128, int nranks, int rank, int cuda_device, void** comm);
rs_status_t rs_comm_destroy(void* comm);
/* GSD oversampling factor r (s = r·p samples per rank; default 8, BASELINE
 * config 4 "oversampling factor 8·p").  Must match on every rank. */
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
/* mode 3 (not a sample sort) = the paper's PR4 across GPUs:
 * per 8-bit digit, a local count-sort round, an all-gather of the p×256 counts,
 * and each rank pulling from every peer (CUDA IPC over NVLink) the keys whose
 * global rank (SPEC.md:206 formula) falls in its range; rank j ends with exactly
 * its input count of the sorted order (balanced).  digit_bits 8 only; every rank
 * must be able to map its peers' memory (else RS_ECUDA on every rank).
 * rs_pr_emulate runs all ranks on one GPU (ws: rs_pr_emulate_ws_bytes). */
size_t rs_pr_emulate_ws_bytes(int key_bytes, int val_bytes, int p, size_t n_max);
rs_status_t rs_pr_emulate(int key_bytes, int p, void* const* keys, uint32_t* const* vals, const size_t* n,
                          void* const* out_keys, uint32_t* const* out_vals, void* ws, size_t ws_bytes,
                          void* stream);
/* modes 4 and 5 (network sorts; costs PAPER.md:717-763):
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
 * region (it is exported whole); rs_ws_bytes sizes it.
 * rs_net_stages: the number of stages (BTN) / rounds (OET) for p ranks, −1 if
 * p is invalid for the mode.  rs_net_emulate runs all p ranks on this GPU:
 * keys[k] / vals[k] (N each, vals NULL or u32 values of every block; read only),
 * out_keys[j] / out_vals[j] (N each), ws of rs_net_emulate_ws_bytes (device,
 * 16-byte aligned), stream-ordered, no sync. */
int rs_net_stages(int mode, int p);
/* The exchange of `rank` in stage `stage` (0-based) of the mode's network, host
 * only: *partner = the other rank of its merge-split (−1: idle this stage),
 * *keep_low = 1 if it keeps the smaller half.  Returns 0, or −1 on a bad argument. */
int rs_net_schedule(int mode, int p, int stage, int rank, int* partner, int* keep_low);
size_t rs_net_emulate_ws_bytes(int key_bytes, int val_bytes, int p, int digit_bits, size_t N);
rs_status_t rs_net_emulate(int mode, int key_bytes, int p, int digit_bits, void* const* keys,
                           const uint32_t* const* vals, size_t N, void* const* out_keys,
                           uint32_t* const* out_vals, void* ws, size_t ws_bytes, void* stream);
/* GER's default s for n keys in all, and the Lemma-Sampling1 capacity for a
 * largest block of n_local_max keys over p ranks (s = 0: the default s). */
size_t rs_ger_default_s(uint64_t n_total);
size_t rs_ger_capacity(size_t n_local_max, int p, size_t s);
/* The p×p count matrix |X_{k,j}| (row k = sender) of the last sample sort on
 * this communicator, into host u64[p*p]; RS_EINVAL before the first sort.
 * (bench.py derives the all-to-all bytes from it.) */
rs_status_t rs_comm_last_counts(void* comm, uint64_t* counts);
int rs_comm_rank(void* comm);
int rs_comm_size(void* comm);

/* With comm != NULL, rs_sort_* is the GSD collective: every rank calls it with
 * the same key/value types, digit_bits and r (checked: RS_EINVAL on all ranks
 * on a mismatch).  n may differ per rank.  Rank j receives Y_j, the j-th
 * contiguous slice of the global sorted order, in out[0 .. *n_out).  `keys`
 * (and vals) are used as scratch (they hold X_j, the locally sorted block, on
 * return).  The call blocks the host twice (the header exchange and the p×p
 * count exchange); *n_out is valid on return.  Receive capacity: out_cap <
 * |Y_j| on any rank → RS_ECAPACITY on every rank.  Argument errors on any rank
 * (bad pointers, digit width, workspace too small, mismatched settings) are
 * agreed on in the header exchange: every rank returns RS_EINVAL, none hangs. */

/* rs_gsd_exchange_plan: the host-side plan of GSD's all-to-all (PAPER.md:797-803,
 * "Processor k sends to processor j sequence X_{k,j}") from the all-gathered
 * count matrix counts[k*p + j] = |X_{k,j}| (host, p×p).  For `rank`:
 *   send_off[0..p]: X_{rank,j} = sorted block [send_off[j], send_off[j+1])
 *   recv_off[0..p]: X_{k,rank} lands at [recv_off[k], recv_off[k+1]) of the
 *                   receive buffer, runs in source-rank order (reading R16)
 *   *total = |Y_rank|.
 * caps (host, p entries, may be NULL): every rank's output capacity; any
 * |Y_j| > caps[j] returns RS_ECAPACITY, identically on every rank.
 * Pure host function (no device access); used by the GSD call itself. */
rs_status_t rs_gsd_exchange_plan(int p, int rank, const uint64_t* counts, const uint64_t* caps,
                                 uint64_t* send_off, uint64_t* recv_off, uint64_t* total);

/* ---------------------------------------------------------- GSD emulation -- */
/* rs_gsd_emulate: GSD over p ranks whose blocks all live on THIS GPU, run rank
 * by rank in one stream (no NCCL, nothing waits on another rank): the same
 * kernels and host plan as the multi-GPU path, with device copies standing in
 * for the all-gathers and the all-to-all.  Used to test the multi-GPU path's
 * kernels on one GPU.
 *   keys[k], vals[k] (vals NULL for keys-only), n[k]: the p blocks (scratch).
 *   out_keys[j], out_vals[j], out_cap: per-rank outputs; n_out[j] = |Y_j|.
 *   splitters: NULL or host u64[3*(p-1)] receiving (key, rank, pos) of S_i.
 *   counts:    NULL or host u64[p*p] receiving |X_{k,j}| at [k*p + j].
 *   ws: rs_gsd_emulate_ws_bytes(key_bytes, val_bytes, p, r, digit_bits,
 *       max_k n[k], out_cap) bytes.
 * Blocks the host once (the count exchange), like the multi-GPU call. */
size_t rs_gsd_emulate_ws_bytes(int key_bytes, int val_bytes, int p, int r, int digit_bits, size_t n_max,
                               size_t out_cap);
rs_status_t rs_gsd_emulate(int key_bytes, int p, int r, int digit_bits,
                           void* const* keys, uint32_t* const* vals, const size_t* n,
                           void* const* out_keys, uint32_t* const* out_vals, size_t out_cap,
                           size_t* n_out, uint64_t* splitters, uint64_t* counts,
                           void* ws, size_t ws_bytes, void* stream);

/* rs_ger_emulate: GER (see rs_comm_set_sampling) over p ranks on this GPU, with
 * the same arguments as rs_gsd_emulate except s and seed in place of r
 * (the draws of every rank go into one array, standing in for the all-reduce).
 *   ws: rs_ger_emulate_ws_bytes(key_bytes, val_bytes, p, s, digit_bits,
 *       max_k n[k], out_cap) bytes (s = 0: sized for n = p·max_k n[k]). */
size_t rs_ger_emulate_ws_bytes(int key_bytes, int val_bytes, int p, size_t s, int digit_bits, size_t n_max,
                               size_t out_cap);
rs_status_t rs_ger_emulate(int key_bytes, int p, size_t s, uint64_t seed, int digit_bits,
                           void* const* keys, uint32_t* const* vals, const size_t* n,
                           void* const* out_keys, uint32_t* const* out_vals, size_t out_cap,
                           size_t* n_out, uint64_t* splitters, uint64_t* counts,
                           void* ws, size_t ws_bytes, void* stream);

/* rs_gvr_emulate: GVR over p ranks on this GPU, arguments as rs_ger_emulate
 * (the blocks are partitioned by destination in place). */
size_t rs_gvr_emulate_ws_bytes(int key_bytes, int val_bytes, int p, size_t s, int digit_bits, size_t n_max,
                               size_t out_cap);
rs_status_t rs_gvr_emulate(int key_bytes, int p, size_t s, uint64_t seed, int digit_bits,
                           void* const* keys, uint32_t* const* vals, const size_t* n,
                           void* const* out_keys, uint32_t* const* out_vals, size_t out_cap,
                           size_t* n_out, uint64_t* splitters, uint64_t* counts,
                           void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ CUDA IPC -- */
/* Device-buffer mappings used by the GSD pull merge (gsd_merge = 2, 3): export
 * the IPC handle (64 bytes) of the cudaMalloc allocation containing `ptr` and
 * ptr's byte offset in it; open a peer's (handle, offset) as a local pointer
 * (each handle is opened once per device and cached; rs_ipc_close_all unmaps).
 * Export fails with RS_ECUDA for memory that has no IPC handle (VMM / cuMem
 * allocations); the pull merge then falls back to the all-to-all. */
rs_status_t rs_ipc_export(const void* ptr, void* handle64, uint64_t* offset);
rs_status_t rs_ipc_open(const void* handle64, uint64_t offset, void** ptr);
rs_status_t rs_ipc_close_all(void);

/* --------------------------------------------------------------- options -- */
/* Process-wide tuning / test knobs (not needed for normal use):
 *   "wide_status"    1 = use 64-bit look-back status words at any n (they are
 *                    used automatically when n > 2^31, where a 31-bit
 *                    inclusive prefix could overflow); lets the tests run that
 *                    path on small n.
 *   "rank_variant"   in-tile ranking: 3 = pairs of keys, one by 8 ballots and one
 *                    by a shared-memory atomic-OR peer mask (default); 0 = ballots;
 *                    2 = atomic-OR masks; 1 = match.any (classic design only).
 *   "pass_design"    radix-256 pass kernel: 5 = atomic ranks (default; used when
 *                    the lane-order probe passes on this device, otherwise 2);
 *                    2 = early counts + tile prefetch, ballot ranks,
 *                    look-back after ranking; 1 = early counts + tile
 *                    prefetch with a dedicated look-back warp; 0 = classic single
 *                    sweep (rank, look-back, reorder, store).
 *   "match_every"    0, 4, 6 or 8: in the default pass (u32 keys) every k-th key is
 *                    ranked with match.any (ADU pipe) instead of ballots (ALU pipe).
 *   "gsd_merge"      GSD step 5 (all give the same Y_j): 3 = pull merge in one
 *                    p-way pass (default): no all-to-all; every peer's X_{k,j}
 *                    is read in place over NVLink through CUDA IPC mappings
 *                    (see below; emulation: the blocks in place), cut into
 *                    chunks by a regular sample of the runs and merged chunk by
 *                    chunk in shared memory, Y_j written once (2 ≤ p ≤ 32, else
 *                    as 2); 2 = pull merge as a tree of 2-way merges whose first
 *                    level reads the peers' blocks; if any rank cannot export or
 *                    map a block, every rank falls back to 0 for that call.
 *                    0 = NCCL all-to-all into a receive buffer, then the tree of
 *                    stable 2-way merge-path merges; 1 = all-to-all, then a
 *                    stable radix re-sort.
 *   "gsd_pull"       1 (default) = modes 2 and 3 pull over NVLink; 0 = they take
 *                    the all-to-all path (the fallback taken when a mapping
 *                    fails), merging the received runs the same way.
 *   "compact"        1 = default pass with 16-bit per-warp counters (smaller
 *                    shared-memory footprint; ballots only).
 *   "small_tiles"    design-5 tiles: 0 = small tiles when the input makes fewer
 *                    than three large tiles per SM (default), 1 = always large,
 *                    2 = always small.
 *   "small_fused"    1 = small-tile full sorts as one cooperative launch (all
 *                    phases separated by grid barriers); 0 = separate kernels
 *                    (default: the fused form measured no faster).
 *   "hist_shared"    1 = digit-histogram kernel with one shared histogram per
 *                    4 warps (0, default: lane-private copies, conflict-free).
 *   "debug_skip"     timing ablations, OUTPUT INVALID: bit 0 no look-back,
 *                    bit 1 no ranking, bit 2 no global store, bit 3 no reorder.
 * Returns RS_EINVAL for an unknown name or a negative value. */
rs_status_t rs_set_option(const char* name, long long value);
/* Current value of an rs_set_option knob, or a read-only value: "rank_probe",
 * the result of the design-5 lane-order probe on the current device (-1 not run
 * yet, 0 failed -> design 2 is used, 1 passed); "tile_u32", "tile_u64",
 * "tile_pairs", the radix-256 tile (keys per look-back row) of the selected
 * pass design.  RS_EINVAL for unknown names. */
rs_status_t rs_get_option(const char* name, long long* value);

/* ---------------------------------------------------------------- timing -- */
/* Per-kernel device timing for measurement (bench.py): when enabled, every
 * kernel the library launches is bracketed by CUDA events on its own stream.
 * rs_timing_query sums the elapsed ms and launch count of kernels whose name
 * starts with `prefix` (e.g. "onesweep", "hist", "" = all) since the last
 * rs_timing_reset; it synchronises the recorded events. */
void rs_timing_enable(int on);
void rs_timing_reset(void);
rs_status_t rs_timing_query(const char* prefix, double* total_ms, int* launches);
/* kernel launches issued by the library since the last rs_timing_reset
 * (counted whether or not timing is enabled) */
long long rs_launch_count(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RSORT_H */
