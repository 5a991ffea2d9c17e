/*
 * rsort_dev.h — development / test surface of librsort.so, kept apart from the
 * product ABI in rsort.h (which is all a user needs).  Everything here is
 * extern "C", plain pointers and sizes, never aborts; errors as in rsort.h.
 *
 *   - in-process ranks: p threads of one process on ONE GPU run the multi-GPU
 *     collective (rs_sort_* with a comm) through host barriers and device copies
 *     instead of NCCL; nothing on the device waits for another rank.  This is how
 *     the GSD / GER / GVR / PR4 / BTN / OET orchestration is tested bit-exactly on
 *     a single B200;
 *   - introspection of a comm's last collective call (count matrix, splitters,
 *     host synchronisations), the blocking-wait timeout;
 *   - host-only helpers (exchange plan, network schedules, GER sizing);
 *   - CUDA IPC export / open (the NCCL transport's peer mappings);
 *   - process-wide test knobs and per-kernel event timing (bench.py).
 */
#ifndef RSORT_DEV_H
#define RSORT_DEV_H
#include "rsort.h"

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ------------------------------------------------------ in-process ranks -- */
/* A group of p ranks (1 <= p <= 64) living as threads of this process on the
 * current CUDA device.  Each rank's thread then calls rs_comm_create_local with
 * its rank (on that device) and uses the comm exactly like an NCCL one — every
 * collective call must be made by all p threads concurrently, each on its own
 * stream.  Destroy the group after all its comms.  A rank that never reaches a
 * collective makes the others fail with RS_ECUDA after the comm's timeout (the
 * group is then broken). */
rs_status_t rs_local_group_create(int p, void** group);
rs_status_t rs_local_group_destroy(void* group);
rs_status_t rs_comm_create_local(void* group, int rank, void** comm);

/* --------------------------------------------------- comm introspection -- */
/* The p×p count matrix |X_{k,j}| (row k = sender) of the last sample sort on
 * this communicator, into host u64[p*p]; RS_EINVAL before the first sort. */
rs_status_t rs_comm_last_counts(void* comm, uint64_t* counts);
/* The p−1 splitters of the last sample sort as (key, rank, pos) triples into
 * host u64[3*(p−1)] (pos = 2^64−1 for the +∞ composite of an empty block). */
rs_status_t rs_comm_last_splitters(void* comm, uint64_t* splitters);
/* Host synchronisations (blocking waits) the last collective call made on this
 * comm: 1 for GSD (mode 0); -1 for a NULL comm. */
int rs_comm_last_host_syncs(void* comm);
/* Blocking waits of this comm give up after timeout_ms (default 600000): NCCL
 * comms are aborted (RS_ENCCL), local groups are broken (RS_ECUDA). */
rs_status_t rs_comm_set_timeout(void* comm, int timeout_ms);

/* ------------------------------------------------------------ host only -- */
/* The host-side plan of GSD's all-to-all ("Processor k sends
 * to processor j sequence X_{k,j}") from the all-gathered count matrix
 * counts[k*p + j] = |X_{k,j}| (host, p×p).  For `rank`:
 *   send_off[0..p]: X_{rank,j} = sorted block [send_off[j], send_off[j+1])
 *   recv_off[0..p]: X_{k,rank} lands at [recv_off[k], recv_off[k+1]) of the
 *                   receive buffer, runs in source-rank order (reading R16)
 *   *total = |Y_rank|.
 * caps (host, p entries, may be NULL): every rank's output capacity; any
 * |Y_j| > caps[j] returns RS_ECAPACITY, identically on every rank. */
rs_status_t rs_gsd_exchange_plan(int p, int rank, const uint64_t* counts, const uint64_t* caps,
                                 uint64_t* send_off, uint64_t* recv_off, uint64_t* total);
/* BTN (mode 4) / OET (mode 5) networks: the number of stages / rounds for p
 * ranks (−1 if p is invalid for the mode), and the exchange of `rank` in
 * `stage` (0-based): *partner (−1: idle), *keep_low (1: it keeps the smaller
 * half).  Returns 0, or −1 on a bad argument. */
int rs_net_stages(int mode, int p);
int rs_net_schedule(int mode, int p, int stage, int rank, int* partner, int* keep_low);
/* GER's default s for n keys in all, and the Lemma-Sampling1 capacity for a
 * largest block of n_local_max keys over p ranks (s = 0: the default s). */
size_t rs_ger_default_s(uint64_t n_total);
size_t rs_ger_capacity(size_t n_local_max, int p, size_t s);

/* ------------------------------------------------------------- CUDA IPC -- */
/* Export the IPC handle (64 bytes) of the cudaMalloc allocation containing ptr
 * and ptr's byte offset in it; open a peer's (handle, offset) as a local
 * pointer (reference counted per device and handle); rs_ipc_close_all unmaps
 * every mapping opened through rs_ipc_open.  Export fails with RS_ECUDA for
 * memory without an IPC handle (VMM / cuMem allocations). */
rs_status_t rs_ipc_export(const void* ptr, void* handle64, uint64_t* offset);
rs_status_t rs_ipc_open(const void* handle64, uint64_t offset, void** ptr);
rs_status_t rs_ipc_close_all(void);

/* -------------------------------------------------------------- options -- */
/* Process-wide knobs, set between calls (not while a sort runs):
 *   "pass_design"  5 = atomic-rank pass (default; used when the lane-order probe
 *                  passes on this device, otherwise 2); 2 = ballot ranks ("safe
 *                  mode": relies on no ordering property of the hardware).
 *   "self_check"   1 = after every local sort one kernel checks on the device
 *                  that the output is ordered; the host waits for the verdict
 *                  and the call fails with RS_ECUDA on a violation (debug).
 *   "wide_status"  1 = 64-bit look-back status words at any n (tests that path).
 *   "small_tiles"  design-5 tiles: 0 auto, 1 always large, 2 always small.
 *   "pdl"          programmatic dependent launches along the radix-256 kernel chain:
 *                  0 auto (n <= 2^25 u32 keys, 2^24 pairs, 2^22 u64 keys), 1 never, 2 always.
 *   "gsd_merge"    GSD step 5 (all give the same Y_j): 3 = one p-way pass
 *                  (default), 2 = tree of 2-way merges, 1 = stable radix
 *                  re-sort (after an all-to-all), 0 = tree after an all-to-all.
 *   "gsd_pull"     1 (default) = modes 2 and 3 read the peers' blocks in place
 *                  (CUDA IPC over NVLink) instead of an all-to-all; 0 = they take
 *                  the all-to-all (the fallback used when a block cannot be
 *                  shared).  gsd_merge and gsd_pull must match on every rank
 *                  (checked with the call's header).
 * Read-only: "rank_probe" (-1 not run on this device yet, 0 failed, 1 passed),
 * "tile_u32" / "tile_u64" / "tile_pairs" (keys per look-back tile of the
 * selected pass design).  RS_EINVAL for an unknown name or value. */
rs_status_t rs_dev_set_option(const char* name, long long value);
rs_status_t rs_dev_get_option(const char* name, long long* value);

/* --------------------------------------------------------------- timing -- */
/* Per-kernel device timing (bench.py): when enabled, every kernel the library
 * launches is bracketed by CUDA events on its own stream.  rs_timing_query sums
 * the elapsed ms and launch count of kernels whose name starts with `prefix`
 * (e.g. "onesweep", "hist", "" = all) since the last rs_timing_reset; it
 * synchronises the recorded events.  rs_launch_count: kernel launches issued by
 * the library since the last rs_timing_reset (counted whether or not timing is
 * enabled). */
void rs_timing_enable(int on);
void rs_timing_reset(void);
rs_status_t rs_timing_query(const char* prefix, double* total_ms, int* launches);
long long rs_launch_count(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RSORT_DEV_H */
