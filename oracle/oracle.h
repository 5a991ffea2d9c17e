/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, serial C implementation of what the GPU path computes,
 * written from the paper (Gerbessiotis, "A study of integer sorting on
 * multicores", arXiv 1808.10292 = /root/reference/PAPER.md).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or constant with
 * paper_1808_10292_b200/ (the CUDA path), and the product path never calls it.
 *
 *   sr.c      SR-b: serial LSD radix sort by count-sort rounds
 *             (§3.2 "Serial radix-r radix-sort: SR4").
 *   gsd.c     GSD: deterministic regular oversampling sort, simulated for p
 *             processors in one process (Algorithm 1), and
 *             GER, its random-oversampling variant.
 *   net.c     BTN and OET: bitonic / odd-even transposition merge-split
 *             networks over p sorted blocks.
 *   verify.c  invariants: nondecreasing order, multiset hash, pair stability.
 *
 * Pins (tests/test_oracle.py, tests/test_oracle_gsd.py): library sort
 * (numpy/qsort), brute force over all short sequences on a 4-letter alphabet,
 * the stable-sort-by-masked-key identity for every intermediate round, bincount
 * for the histograms, the SPEC.md:290 GSD hand trace, a hand-derived p = 3,
 * r = 2 GSD trace with duplicates (tests/golden/gsd_hand_trace_p3_r2.json), and
 * the balance bound ⌊(1+1/r)·N_max⌋ (reading R18) by brute force.
 * The paper prints no partition: beyond those traces GSD's per-rank partition
 * rests on DESIGN.md readings R10/R12/R14.
 */
#ifndef RS_ORACLE_H
#define RS_ORACLE_H
#include <stddef.h>
#include <stdint.h>

/* ---- sr.c ---------------------------------------------------------------- */
/* Run `rounds` count-sort rounds (rounds < 0: all keybits/b rounds) of radix
 * r = 2^b, b in {8, 16}, least-significant digit first.  Result in a[] (and
 * v[]).  Returns 0, or -1 on a bad argument / allocation failure. */
int or_sr_u32(uint32_t* a, size_t n, int b, int rounds);
int or_sr_u64(uint64_t* a, size_t n, int b, int rounds);
int or_sr_pairs_u64_u32(uint64_t* a, uint32_t* v, size_t n, int b, int rounds);

/* Digit counts of every round in one read: out[t*R + d] = #{i : digit_t(a_i) = d}. */
int or_hist_u32(const uint32_t* a, size_t n, int b, uint64_t* out);
int or_hist_u64(const uint64_t* a, size_t n, int b, uint64_t* out);

/* ---- gsd.c --------------------------------------------------------------- */
/* One GSD(X, n, p) run over p shards held in one process.
 *   keys[k], vals[k] (vals may be NULL), N[k]  — the p input blocks (read-only)
 *   r, b                                        — oversampling r (s = r·p), digit bits
 *   Y_keys[j], Y_vals[j], Ycap                  — output blocks (capacity Ycap each)
 *   Ylen[j]                                     — |Y_j|
 *   splitters[3*(p-1)]                          — (key, rank, pos) of S_1..S_{p-1}
 *   counts[p*p]                                 — counts[k*p + j] = |X_{k,j}|
 * Returns 0, -1 bad argument, -2 capacity exceeded. */
int or_gsd_u64(int p, int r, int b,
               const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
               uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts);
int or_gsd_u32(int p, int r, int b,
               const uint32_t* const* keys, const size_t* N,
               uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts);

/* GER(X, n, p): as GSD but the sample is s·p − 1 keys drawn
 * uniformly at random (with replacement, SplitMix64 `seed`, readings R28-R30)
 * from the concatenation of the sorted blocks; S_i = T[i·s − 1]. */
int or_ger_u64(int p, size_t s, uint64_t seed, int b,
               const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
               uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts);
int or_ger_u32(int p, size_t s, uint64_t seed, int b,
               const uint32_t* const* keys, const size_t* N,
               uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts);
/* GVR(X, n, p): random sample of the unsorted blocks (the GER
 * draws), split by destination, exchange, then SR-b of each Y_j. */
int or_gvr_u64(int p, size_t s, uint64_t seed, int b,
               const uint64_t* const* keys, const uint32_t* const* vals, const size_t* N,
               uint64_t* const* Y_keys, uint32_t* const* Y_vals, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts);
int or_gvr_u32(int p, size_t s, uint64_t seed, int b,
               const uint32_t* const* keys, const size_t* N,
               uint32_t* const* Y_keys, size_t Ycap, size_t* Ylen,
               uint64_t* splitters, uint64_t* counts);
/* the i-th output of SplitMix64 seeded `seed` (the generator GER draws with) */
uint64_t or_splitmix64_at(uint64_t seed, uint64_t i);

/* ---- net.c ---------------------------------------------------------------- */
/* BTN and OET over p blocks of N keys held
 * contiguously in keys[] (block k at k·N), in place: SR-b of every block, then
 * the merge-split network (readings R32-R34).  max_stages >= 0 stops after that
 * many stages (BTN) / rounds (OET); *stages = the number executed.  vals (u64
 * only) may be NULL.  Returns 0, or -1 (bad argument; BTN: p not a power of 2). */
int or_btn_u32(int p, int b, uint32_t* keys, size_t N, int max_stages, int* stages);
int or_btn_u64(int p, int b, uint64_t* keys, uint32_t* vals, size_t N, int max_stages, int* stages);
int or_oet_u32(int p, int b, uint32_t* keys, size_t N, int max_stages, int* stages);
int or_oet_u64(int p, int b, uint64_t* keys, uint32_t* vals, size_t N, int max_stages, int* stages);

/* ---- verify.c ------------------------------------------------------------ */
int or_is_nondecreasing_u32(const uint32_t* a, size_t n);
int or_is_nondecreasing_u64(const uint64_t* a, size_t n);
/* (count, Σ h(x) mod 2^64, ⊕ h(x)); h = SplitMix64 finaliser; out[3] */
void or_multiset_hash_u32(const uint32_t* a, size_t n, uint64_t* out);
void or_multiset_hash_u64(const uint64_t* a, size_t n, uint64_t* out);
/* pairs (k_i, v_i): out[3] = multiset hash of h(k) * 0x100000001B3 ^ h(v) combos */
void or_multiset_hash_pairs_u64_u32(const uint64_t* k, const uint32_t* v, size_t n, uint64_t* out);
/* 1 iff keys nondecreasing and, within every run of equal keys, v strictly increasing */
int or_pairs_stable_u64_u32(const uint64_t* k, const uint32_t* v, size_t n);
/* sampled order statistics: for each m, checks #{x < val[m]} <= pos[m] < #{x <= val[m]}
 * over the unsorted input a[0..n).  Returns the number of failing samples. */
size_t or_check_order_stats_u32(const uint32_t* a, size_t n, const uint64_t* pos,
                                const uint32_t* val, size_t m);
#endif
