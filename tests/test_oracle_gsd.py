"""Pins of the GSD simulator (oracle/gsd.c, Algorithm 1):
the SPEC.md:290 hand trace, concatenation == library sort (unique result),
global pair stability, the balance bound (Lemma `balance`, PAPER.md:891-955,
in the DESIGN.md reading R18), and brute force of the split rule."""
import json
import os

import numpy as np
import pytest

import inputs
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_trace_spec290():
    g = json.load(open(os.path.join(GOLD, "gsd_hand_trace_spec290.json")))
    shards = [np.array(b, dtype=np.uint32) for b in g["blocks"]]
    res = oracle.gsd(shards, r=g["r"])
    assert [int(s[0]) for s in res["splitters"]] == g["splitters"]
    assert [y.tolist() for y in res["Y"]] == g["Y"]
    assert res["counts"].tolist() == [[4, 4], [4, 4]]


def test_hand_trace_p3_r2_duplicates():
    """A hand-derived trace beyond SPEC.md:290 (tests/golden/gsd_hand_trace_p3_r2.json):
    p = 3, r = 2, duplicates within and across ranks, every intermediate written
    out by hand (X_k, T_k, T, S_i with their rank and position, the composite cuts,
    X_{k,j}, Y_j).  A wrong sample index (R10), splitter index (R12) or tie
    direction at a splitter (R14) changes the counts or the splitters."""
    g = json.load(open(os.path.join(GOLD, "gsd_hand_trace_p3_r2.json")))
    shards = [np.array(b, dtype=np.uint32) for b in g["blocks"]]
    res = oracle.gsd(shards, r=g["r"])
    assert res["splitters"].tolist() == g["splitters"]
    assert res["counts"].tolist() == g["counts"]
    assert [y.tolist() for y in res["Y"]] == g["Y"]
    assert max(len(y) for y in g["Y"]) <= g["balance_bound"]
    # the hand-written intermediates agree with each other (slices of X_k by counts)
    for k in range(g["p"]):
        assert sum(g["X_kj"][k], []) == g["X_k"][k] == sorted(g["blocks"][k])
        assert [len(x) for x in g["X_kj"][k]] == g["counts"][k]
    for j in range(g["p"]):
        assert sorted(sum((g["X_kj"][k][j] for k in range(g["p"])), [])) == g["Y"][j]


def _shards(total, p, seed, dist="uniform"):
    a = inputs.gen_u32(total, seed, dist)
    N = total // p
    return a, [a[k * N:(k + 1) * N] if k < p - 1 else a[k * N:] for k in range(p)]


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "sorted", "reversed"])
def test_concatenation_is_the_sort(p, dist):
    a, shards = _shards(4000, p, 21, dist)
    res = oracle.gsd(shards, r=8)
    assert (np.concatenate(res["Y"]) == np.sort(a)).all()
    assert res["counts"].sum() == a.size
    assert (res["counts"].sum(axis=0) == res["Ylen"]).all()
    assert (res["counts"].sum(axis=1) == [s.size for s in shards]).all()


def test_pairs_globally_stable_narrow_keys():
    p, N = 4, 1500
    k = inputs.gen_u64(p * N, 5, "mod1024") & np.uint64(31)
    v = inputs.iota_u32(p * N)
    res = oracle.gsd([k[i * N:(i + 1) * N] for i in range(p)], r=8,
                     vals=[v[i * N:(i + 1) * N] for i in range(p)])
    K = np.concatenate(res["Y"])
    V = np.concatenate(res["Yv"])
    order = np.lexsort((v, k))
    assert (K == k[order]).all() and (V == v[order]).all()


def test_split_rule_brute_force():
    """Bucket j = {(x, k, q) : S_{j-1} <_c (x,k,q) <=_c S_j} (reading R14), checked
    element by element against the counts the simulator reports."""
    p, r = 4, 2
    a, shards = _shards(400, p, 23, "mod16")
    res = oracle.gsd(shards, r=r)
    S = [tuple(int(v) for v in s) for s in res["splitters"]]
    for k, sh in enumerate(shards):
        xs = np.sort(sh)
        bucket_sizes = [0] * p
        for q, x in enumerate(xs.tolist()):
            e = (x, k, q)
            j = sum(1 for s in S if s < e)      # number of splitters strictly below e
            bucket_sizes[j] += 1
        assert bucket_sizes == res["counts"][k].tolist()


def test_sample_positions_reading_r10():
    """T_k = keys at ceil(N*i/s)-1, i=1..s-1, plus the max (R10): with p=1 the
    single splitter list is empty and with p=2, r=1 the splitter is T[s-1]."""
    x = np.arange(100, 200, dtype=np.uint32)
    y = np.arange(0, 100, dtype=np.uint32)
    res = oracle.gsd([x, y], r=1)            # s = 2: T_0 = [149, 199], T_1 = [49, 99]
    assert res["splitters"][0].tolist() == [99, 1, 99]     # T = [49, 99, 149, 199], S_1 = T[1]
    assert [v.tolist() for v in res["Y"]] == [list(range(0, 100)), list(range(100, 200))]


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("r", [1, 2, 3, 8])
def test_balance_bound_bruteforce(p, r):
    """|Y_j| <= floor((1+1/r) * N_max) whenever every N_k >= s = r*p
    (R18: the Lemma `balance` bound, for this
    reading, tighter than the printed (1+1/r)(n/p) + rp)."""
    rng = np.random.default_rng(1000 * p + r)
    s = r * p
    worst = 0.0
    for trial in range(12):
        even = trial % 2 == 0
        N = [int(rng.integers(s, s + 300))] * p if even else [int(rng.integers(s, s + 300)) for _ in range(p)]
        kind = trial % 6
        shards = []
        for k in range(p):
            if kind == 0:
                sh = rng.integers(0, 1 << 32, N[k], dtype=np.uint64).astype(np.uint32)
            elif kind == 1:
                sh = rng.integers(0, 4, N[k]).astype(np.uint32)
            elif kind == 2:
                sh = np.full(N[k], 7, dtype=np.uint32)
            elif kind == 3:
                sh = np.arange(N[k], dtype=np.uint32) + np.uint32(k * 1000)   # disjoint ranges
            elif kind == 4:
                sh = (np.arange(N[k], dtype=np.uint32) * np.uint32(p) + np.uint32(k))  # interleaved
            else:
                sh = np.where(rng.random(N[k]) < 0.9, 5, rng.integers(0, 100, N[k])).astype(np.uint32)
            shards.append(sh)
        res = oracle.gsd(shards, r=r)
        bound = int(np.floor((1 + 1 / r) * max(N)))
        assert int(res["Ylen"].max()) <= bound, (N, res["Ylen"].tolist(), bound)
        worst = max(worst, float(res["Ylen"].max()) / bound)
        if even:   # the Lemma assumes blocks of n/p keys
            n = sum(N)
            printed = (1 + 1 / r) * (n / p) + r * p     # Lemma `balance` as printed
            assert res["Ylen"].max() <= printed
    assert worst <= 1.0


def test_empty_shards_and_small_shards():
    shards = [np.array([], dtype=np.uint32), np.array([3, 1, 2], dtype=np.uint32),
              np.array([], dtype=np.uint32), np.array([9, 0], dtype=np.uint32)]
    res = oracle.gsd(shards, r=8)
    assert np.concatenate(res["Y"]).tolist() == [0, 1, 2, 3, 9]


def test_deterministic():
    a, shards = _shards(3000, 4, 29)
    r1 = oracle.gsd(shards, r=8)
    r2 = oracle.gsd(shards, r=8)
    assert r1["splitters"].tolist() == r2["splitters"].tolist()
    assert r1["counts"].tolist() == r2["counts"].tolist()
