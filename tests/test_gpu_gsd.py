"""GPU parity of the collective sort itself — rs_sort_u32 / rs_sort_u64 /
rs_sort_pairs_u64_u32 with a comm, one call per rank, the ranks being p threads
on this GPU (LocalGroup, include/rsort_dev.h: the multi-GPU orchestration over
the in-process transport) — against the CPU simulators (oracle/gsd.c,
PAPER.md:775-805 GSD, 965-986 GER, 988-1016 GVR, 685-709 PR4): splitters, the
p×p count matrix and every Y_j bit-exact, on the pull merge and on the
all-to-all fallback; errors come back identically on every rank."""
import numpy as np
import pytest

import inputs
import oracle
import paper_1808_10292_b200 as rs
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


def _check(blocks_np, r, b, vals_np=None):
    p = len(blocks_np)
    dt = blocks_np[0].dtype
    want = oracle.gsd(blocks_np, r=r, b=b, vals=vals_np)
    got = rs.sort_ranks([dev(x) for x in blocks_np], "gsd", r=r, digit_bits=b,
                        vals=[dev(v) for v in vals_np] if vals_np is not None else None)
    assert got["counts"].tolist() == want["counts"].tolist()
    assert got["splitters"].tolist() == want["splitters"].tolist()
    for j in range(p):
        assert (host(got["Y"][j], dt) == want["Y"][j]).all(), j
        if vals_np is not None:
            assert (host(got["Yv"][j], np.uint32) == want["Yv"][j]).all(), j
    nmax = max(x.size for x in blocks_np)
    if min(x.size for x in blocks_np) >= r * p:
        assert max(got["n_out"]) <= nmax + nmax // r          # balance bound (R18)
    assert got["host_syncs"] == [1] * p                       # one blocking wait per call, every rank
    return got


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "sorted"])
def test_gsd_u32_matches_simulator(p, dist):
    total = 40000 + p
    a = inputs.gen_u32(total, 40 + p, dist)
    cuts = np.linspace(0, total, p + 1).astype(int)
    _check([a[cuts[k]:cuts[k + 1]] for k in range(p)], r=8, b=8)


def test_gsd_hand_trace_spec290():
    blocks = [np.arange(1, 16, 2, dtype=np.uint32), np.arange(2, 17, 2, dtype=np.uint32)]
    got = _check(blocks, r=1, b=8)
    assert [host(y, np.uint32).tolist() for y in got["Y"]] == [list(range(1, 9)), list(range(9, 17))]


def test_gsd_hand_trace_p3_r2():
    """The hand-derived p = 3, r = 2 trace (tests/golden/gsd_hand_trace_p3_r2.json)
    through rs_sort_u32 with a comm on three in-process ranks: the literal
    splitters, count matrix and Y_j."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "gsd_hand_trace_p3_r2.json")))
    blocks = [np.array(b, dtype=np.uint32) for b in g["blocks"]]
    got = _check(blocks, r=g["r"], b=8)
    assert got["splitters"].tolist() == g["splitters"]
    assert got["counts"].tolist() == g["counts"]
    assert [host(y, np.uint32).tolist() for y in got["Y"]] == g["Y"]


def test_ger_gvr_hand_trace_p2_s2():
    """The hand-derived GER / GVR traces (tests/golden/ger_gvr_hand_trace_p2_s2.json)
    through rs_sort_u32 with a comm on two in-process ranks: literal splitters,
    count matrix and Y_j."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ger_gvr_hand_trace_p2_s2.json")))
    for mode in ("ger", "gvr"):
        got = rs.sort_ranks([dev(np.array(b, dtype=np.uint32)) for b in g["blocks"]], mode, s=g["s"], seed=g["seed"])
        assert got["splitters"].tolist() == g[mode]["splitters"], mode
        assert got["counts"].tolist() == g[mode]["counts"], mode
        assert [host(y, np.uint32).tolist() for y in got["Y"]] == g[mode]["Y"], mode


@pytest.mark.parametrize("b", [8, 16])
def test_gsd_pairs_global_stability(b):
    p, N = 4, 30000
    k = inputs.gen_u64(p * N, 5, "mod1024")
    v = inputs.iota_u32(p * N)
    got = _check([k[i * N:(i + 1) * N] for i in range(p)], r=8, b=b, vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)


def test_gsd_uneven_and_empty_blocks():
    blocks = [inputs.gen_u32(n, 50 + n) for n in (0, 5, 12345, 0, 70000, 3)]
    _check(blocks, r=8, b=8)


def test_gsd_u64_radix16():
    p = 4
    k = inputs.gen_u64(4 * 25000, 60)
    _check([k[i * 25000:(i + 1) * 25000] for i in range(p)], r=8, b=16)


def test_gsd_config4_shape_reduced():
    """configs[3] shape (uniform u32, r=8, p=8) at 2^24 total keys."""
    p, n = 8, 1 << 24
    a = inputs.gen_u32(n, 4)
    N = n // p
    blocks = [a[k * N:(k + 1) * N] for k in range(p)]
    got = rs.sort_ranks([dev(x) for x in blocks], "gsd", r=8, digit_bits=8)
    Y = np.concatenate([host(y, np.uint32) for y in got["Y"]])
    assert (Y == oracle.sr(a, 8)).all()
    assert max(got["n_out"]) <= N + N // 8


@pytest.fixture
def option():
    saved = {}

    def _set(name, value):
        saved.setdefault(name, rs.get_option(name))
        rs.set_option(name, value)
    yield _set
    for name, value in saved.items():
        rs.set_option(name, value)


@pytest.mark.parametrize("merge", [0, 1, 2, 3])
@pytest.mark.parametrize("p", [2, 3, 5, 6, 7, 8])
def test_gsd_merge_tree_and_resort(option, merge, p):
    """Step 5 as the merge tree (0), as a stable re-sort (1), as the pull merge
    (2: no exchange copies, the tree's first level reads every rank's block in
    place) and as the one-pass p-way pull merge (3): identical Y_j, for odd run
    counts too; narrow pair keys check the tie rule (lower rank first)."""
    option("gsd_merge", merge)
    N = 9000 + 37 * p
    k = inputs.gen_u64(p * N, 70 + p, "mod1024")
    v = inputs.iota_u32(p * N)
    got = _check([k[i * N:(i + 1) * N] for i in range(p)], r=8, b=8, vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)
    a = inputs.gen_u32(p * N, 80 + p)
    _check([a[i * N:(i + 1) * N] for i in range(p)], r=8, b=8)


def test_merge_tree_large_runs(option):
    """Merge tree over big uneven runs (several merge tiles per pair)."""
    option("gsd_merge", 0)
    blocks = [inputs.gen_u32(n, 90 + i, "sorted" if i % 2 else "uniform") for i, n in
              enumerate((300000, 17, 250001, 0, 123457))]
    _check(blocks, r=8, b=8)


# ---------------------------------------------------------------- GER ----
def _check_ger(blocks_np, s, seed, b=8, vals_np=None):
    p = len(blocks_np)
    dt = blocks_np[0].dtype
    want = oracle.ger(blocks_np, s=s if s else _default_s(sum(x.size for x in blocks_np)), seed=seed, b=b,
                      vals=vals_np)
    got = rs.sort_ranks([dev(x) for x in blocks_np], "ger", s=s, seed=seed, digit_bits=b,
                        vals=[dev(v) for v in vals_np] if vals_np is not None else None)
    assert got["counts"].tolist() == want["counts"].tolist()
    assert got["splitters"].tolist() == want["splitters"].tolist()
    for j in range(p):
        assert (host(got["Y"][j], dt) == want["Y"][j]).all(), j
        if vals_np is not None:
            assert (host(got["Yv"][j], np.uint32) == want["Yv"][j]).all(), j
    return got


def _default_s(n):
    return int(rs.lib().rs_ger_default_s(n))


@pytest.mark.parametrize("p", [2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "reversed"])
def test_ger_u32_matches_simulator(p, dist):
    """GER: random sample drawn on the GPU (SplitMix64 counter
    draws), ordered by two stable radix sorts, S_i = (i·s)-th: splitters, count
    matrix and every Y_j bit-exact against the CPU simulator."""
    total = 50000 + 3 * p
    a = inputs.gen_u32(total, 80 + p, dist)
    cuts = np.linspace(0, total, p + 1).astype(int)
    _check_ger([a[cuts[k]:cuts[k + 1]] for k in range(p)], s=0, seed=11 + p)   # the paper's s
    _check_ger([a[cuts[k]:cuts[k + 1]] for k in range(p)], s=13, seed=7)


@pytest.mark.parametrize("b", [8, 16])
def test_ger_pairs_global_stability(b):
    p, N = 4, 20000
    k = inputs.gen_u64(p * N, 6, "mod1024")
    v = inputs.iota_u32(p * N)
    got = _check_ger([k[i * N:(i + 1) * N] for i in range(p)], s=0, seed=2, b=b,
                     vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)


def test_ger_uneven_empty_blocks_and_u64():
    a = inputs.gen_u32(9000, 91)
    _check_ger([a[:0], a[:5000], a[5000:5003], a[5003:]], s=6, seed=4)
    k = inputs.gen_u64(30001, 92)
    _check_ger([k[:12000], k[12000:12001], k[12001:]], s=0, seed=5)


# ---------------------------------------------------------------- GVR ----
def _check_gvr(blocks_np, s, seed, b=8, vals_np=None):
    p = len(blocks_np)
    dt = blocks_np[0].dtype
    want = oracle.gvr(blocks_np, s=s if s else _default_s(sum(x.size for x in blocks_np)), seed=seed, b=b,
                      vals=vals_np)
    got = rs.sort_ranks([dev(x) for x in blocks_np], "gvr", s=s, seed=seed, digit_bits=b,
                        vals=[dev(v) for v in vals_np] if vals_np is not None else None)
    assert got["counts"].tolist() == want["counts"].tolist()
    assert got["splitters"].tolist() == want["splitters"].tolist()
    for j in range(p):
        assert (host(got["Y"][j], dt) == want["Y"][j]).all(), j
        if vals_np is not None:
            assert (host(got["Yv"][j], np.uint32) == want["Yv"][j]).all(), j
    return got


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "sorted"])
def test_gvr_u32_matches_simulator(p, dist):
    """GVR: sample of the unsorted blocks, destinations by
    binary search of the composite splitters, stable count-sort by destination,
    exchange, local radix sort: bit-exact against the CPU simulator."""
    total = 50000 + 5 * p
    a = inputs.gen_u32(total, 100 + p, dist)
    cuts = np.linspace(0, total, p + 1).astype(int)
    _check_gvr([a[cuts[k]:cuts[k + 1]] for k in range(p)], s=0, seed=21 + p)
    _check_gvr([a[cuts[k]:cuts[k + 1]] for k in range(p)], s=9, seed=8)


@pytest.mark.parametrize("b", [8, 16])
def test_gvr_pairs_global_stability_and_u64(b):
    p, N = 4, 20000
    k = inputs.gen_u64(p * N, 7, "mod1024")
    v = inputs.iota_u32(p * N)
    got = _check_gvr([k[i * N:(i + 1) * N] for i in range(p)], s=0, seed=3, b=b,
                     vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)
    u = inputs.gen_u64(30001, 93)
    _check_gvr([u[:12000], u[12000:12001], u[12001:]], s=0, seed=6, b=b)


def test_gvr_uneven_and_empty_blocks():
    a = inputs.gen_u32(9000, 94)
    _check_gvr([a[:0], a[:5000], a[5000:5003], a[5003:]], s=6, seed=4)


@pytest.mark.parametrize("merge", [2, 3])
def test_pull_merge_ger_and_large(option, merge):
    """The pull merge (tree and p-way) under GER sampling and over large uneven runs."""
    option("gsd_merge", merge)
    a = inputs.gen_u32(600000, 95)
    cuts = [0, 100000, 350001, 350002, 600000]
    _check_ger([a[cuts[k]:cuts[k + 1]] for k in range(4)], s=0, seed=9)
    _check([a[cuts[k]:cuts[k + 1]] for k in range(4)], r=8, b=8)


@pytest.mark.parametrize("p", [2, 4, 16, 32])
@pytest.mark.parametrize("dist", ["uniform", "equal", "mod16", "sorted"])
def test_pway_merge_many_runs(option, p, dist):
    """The one-pass p-way merge (pwmerge.cu) against the GSD simulator: many runs
    (p up to 32, r = 8 keeps r·p² ≤ 8192), all-equal keys (every chunk boundary
    decided by the (run, position) tie rule), sizes spanning many chunks, ragged."""
    option("gsd_merge", 3)
    N = 40000 + 77 * p
    a = inputs.gen_u32(p * N, 400 + p, dist)
    _check([a[i * N:(i + 1) * N] for i in range(p)], r=8, b=8)


@pytest.mark.parametrize("merge", [2, 3])
def test_exchange_fallback_with_pull_merges(option, merge):
    """With pulling disabled (the path taken when a peer block cannot be mapped)
    the all-to-all runs and the received runs are merged by the tree (2) or the
    one-pass p-way merge (3): identical Y_j, pairs stable."""
    option("gsd_merge", merge)
    option("gsd_pull", 0)
    p, N = 8, 30011
    k = inputs.gen_u64(p * N, 430, "mod1024")
    v = inputs.iota_u32(p * N)
    got = _check([k[i * N:(i + 1) * N] for i in range(p)], r=8, b=8, vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)
    a = inputs.gen_u32(5 * 40000, 431, "gauss")
    _check([a[i * 40000:(i + 1) * 40000] for i in range(5)], r=8, b=8)


@pytest.mark.parametrize("span", [1, 3, 6])
def test_pway_merge_partially_overlapping_runs(option, span):
    """p-way merge with runs that overlap only in part (block k holds keys in
    [k·D, (k + span)·D)): inside a merged pair one run is spent long before the
    pair ends, so the unchecked forward slots, the copy of the surviving run, the
    bound-checked slots and the backwards pair-end slots all run; u32 keys against
    the simulator, (u64, u32) pairs with many ties also stable."""
    option("gsd_merge", 3)
    p, N, D = 8, 50021, 1 << 26
    base = inputs.gen_u32(p * N, 470 + span)
    blocks = [(base[i * N:(i + 1) * N] % np.uint32(span * D)) + np.uint32(i * D) for i in range(p)]
    _check(blocks, r=8, b=8)
    k = inputs.gen_u64(p * N, 480 + span, "mod1024")
    kb = [(k[i * N:(i + 1) * N] % np.uint64(64 * span)) + np.uint64(64 * i) for i in range(p)]
    v = inputs.iota_u32(p * N)
    got = _check(kb, r=8, b=8, vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)


def test_pway_merge_pairs_uneven_tiny_and_empty_blocks(option):
    """p-way merge: stable pairs over uneven blocks, including blocks shorter than
    one sample stride and empty ones (runs with no samples)."""
    option("gsd_merge", 3)
    k = inputs.gen_u64(300000, 411, "mod1024")
    v = inputs.iota_u32(k.size)
    cuts = [0, 0, 50, 100000, 100001, 230000, 300000]
    got = _check([k[cuts[i]:cuts[i + 1]] for i in range(6)], r=8, b=8,
                 vals_np=[v[cuts[i]:cuts[i + 1]] for i in range(6)])
    K = np.concatenate([host(y, np.uint64) for y in got["Y"]])
    V = np.concatenate([host(y, np.uint32) for y in got["Yv"]])
    assert oracle.pairs_stable(K, V)
    small = inputs.gen_u32(700, 412)
    _check([small[:100], small[100:300], small[300:301], small[301:]], r=8, b=8)


# ---------------------------------------------------------- PR4 across GPUs ----
@pytest.mark.parametrize("p", [1, 2, 3, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "sorted"])
def test_pr4_across_ranks_matches_the_sort(p, dist):
    """PR4 routing (PAPER.md:685-709, SPEC.md:206 rank formula), rank by rank:
    after the four rounds rank j holds exactly positions [off_j, off_j + n_j) of
    the stable sorted order — the oracle's SR4 result sliced by the input sizes."""
    sizes = [7000 + 1311 * k for k in range(p)]
    a = inputs.gen_u32(sum(sizes), 150 + p, dist)
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    blocks = [a[cuts[k]:cuts[k + 1]] for k in range(p)]
    got = rs.sort_ranks([dev(x) for x in blocks], "pr4")
    want = oracle.sr(a, 8)
    for j in range(p):
        assert (host(got["Y"][j], np.uint32) == want[cuts[j]:cuts[j + 1]]).all(), j


def test_pr4_pairs_stability_u64_uneven_and_empty_blocks():
    sizes = [0, 20000, 3, 0, 15001]
    k = inputs.gen_u64(sum(sizes), 151, "mod1024")
    v = inputs.iota_u32(k.size)
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    got = rs.sort_ranks([dev(k[cuts[i]:cuts[i + 1]]) for i in range(5)], "pr4",
                        vals=[dev(v[cuts[i]:cuts[i + 1]]) for i in range(5)])
    wk, wv = oracle.sr(k, 8, vals=v)
    for j in range(5):
        assert (host(got["Y"][j], np.uint64) == wk[cuts[j]:cuts[j + 1]]).all(), j
        assert (host(got["Yv"][j], np.uint32) == wv[cuts[j]:cuts[j + 1]]).all(), j


# ------------------------------------------------- collective error agreement ----
def _statuses(p, fn):
    """run fn(comm) on p in-process ranks; each rank's RSortError status (0 = ok)"""
    g = rs.LocalGroup(p)

    def body(c):
        try:
            fn(c)
            return 0
        except rs.RSortError as e:
            return e.status
    try:
        return g.run(body, timeout_ms=60000)
    finally:
        g.close()


def test_capacity_error_identical_on_every_rank():
    """One rank's out_cap below its |Y_j| -> RS_ECAPACITY on EVERY rank (the
    capacities travel with the headers; every rank checks every rank)."""
    p, N = 4, 20000
    a = inputs.gen_u32(p * N, 501)
    blocks = [dev(a[k * N:(k + 1) * N]) for k in range(p)]

    def fn(c):
        cap = c.capacity(N)  # (collective: every rank takes part in the size agreement)
        rs.sort(blocks[c.rank], comm=c, out_cap=N // 2 if c.rank == 2 else cap)
    assert _statuses(p, fn) == [5] * p  # RS_ECAPACITY


def test_header_mismatch_identical_on_every_rank():
    """Rank 1 sorts u64 keys while the others sort u32: RS_EINVAL on every rank,
    no hang (the header rides on the sample all-gather)."""
    p, N = 3, 5000
    a32 = inputs.gen_u32(p * N, 502)
    a64 = inputs.gen_u64(N, 503)

    def fn(c):
        x = dev(a64) if c.rank == 1 else dev(a32[c.rank * N:(c.rank + 1) * N])
        rs.sort(x, comm=c, out_cap=4 * N)
    assert _statuses(p, fn) == [1] * p  # RS_EINVAL


def test_local_argument_error_identical_on_every_rank():
    """Rank 0 passes a workspace that is too small: it never touches its buffers,
    takes part in both all-gathers with an empty block, and every rank returns
    RS_EINVAL; then the same group sorts correctly."""
    import torch
    p, N = 4, 8000
    a = inputs.gen_u32(p * N, 504)

    def fn(c):
        x = dev(a[c.rank * N:(c.rank + 1) * N])
        ws = torch.empty(1024 if c.rank == 0 else
                         rs.workspace_bytes(4, 0, 2 * N, 8, c), dtype=torch.uint8, device="cuda")
        rs.sort(x, comm=c, ws=ws, out_cap=2 * N)
    assert _statuses(p, fn) == [1] * p


def test_out_aliasing_keys_rejected_with_comm():
    """out overlapping keys is rejected (the pull merge reads every peer's block
    while each rank writes Y_j): RS_EINVAL on every rank."""
    p, N = 2, 4000
    a = inputs.gen_u32(p * N, 505)

    def fn(c):
        x = dev(np.concatenate([a[c.rank * N:(c.rank + 1) * N], np.zeros(N, np.uint32)]))
        rs.sort(x[:N], comm=c, out=x, out_cap=2 * N)
    assert _statuses(p, fn) == [1] * p


@pytest.mark.parametrize("pull", [1, 0])
@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_gsd_pull_and_alltoall_paths(option, pull, p):
    """rs_sort_pairs_u64_u32 / rs_sort_u32 with a comm at p = 2, 3, 4, 8 on one
    GPU, both data paths — the pull merge (peers' blocks read in place) and the
    all-to-all fallback — bit-exact against oracle.gsd: counts, splitters, Y_j."""
    option("gsd_pull", pull)
    N = 12000 + 101 * p
    k = inputs.gen_u64(p * N, 510 + p, "mod1024")
    v = inputs.iota_u32(p * N)
    _check([k[i * N:(i + 1) * N] for i in range(p)], r=8, b=8, vals_np=[v[i * N:(i + 1) * N] for i in range(p)])
    a = inputs.gen_u32(p * N + 7, 520 + p)
    cuts = np.linspace(0, a.size, p + 1).astype(int)
    _check([a[cuts[i]:cuts[i + 1]] for i in range(p)], r=8, b=8)


def test_repeated_calls_same_comm():
    """Several collective calls on the same comms (mapping cache, header reuse)."""
    p, N = 4, 10000
    g = rs.LocalGroup(p)
    arrays = [inputs.gen_u32(p * N, 530 + t) for t in range(3)]

    def fn(c):
        outs = []
        for a in arrays:
            y = rs.sort(dev(a[c.rank * N:(c.rank + 1) * N]), comm=c)
            outs.append(host(y, np.uint32))
        return outs
    try:
        res = g.run(fn)
    finally:
        g.close()
    for t, a in enumerate(arrays):
        assert (np.concatenate([res[k][t] for k in range(p)]) == np.sort(a)).all()
