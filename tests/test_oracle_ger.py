"""Pins of the GER simulator (oracle/gsd.c or_ger_*, Algorithm
GER: GSD's skeleton with a random sample of s·p − 1 keys of all X_k, readings
R28-R30): its SplitMix64 against the published vector, the splitters re-derived
here in plain Python from the definition (draws -> composites -> sorted ->
(i·s)-th), the split rule by brute force, concatenation == library sort, global
pair stability, and the bucket-size bound of Lemma `Sampling1`."""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
M64 = (1 << 64) - 1


def _splitmix_py(seed, i):
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_oracle_splitmix64_is_the_published_generator():
    g = json.load(open(os.path.join(GOLD, "splitmix64_seed1234567.json")))
    want = [int(x) for x in g["outputs"]]
    assert [oracle.splitmix64_at(g["seed"], i) for i in range(len(want))] == want
    assert [_splitmix_py(g["seed"], i) for i in range(len(want))] == want


def _blocks(sizes, seed, dist="uniform"):
    a = inputs.gen_u32(sum(sizes), seed, dist)
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    return a, [a[cuts[k]:cuts[k + 1]] for k in range(len(sizes))]


def _definition(blocks, s, seed):
    """Steps 1-3 of Algorithm GER from their definition, in Python."""
    X = [np.sort(b) for b in blocks]
    off = np.concatenate([[0], np.cumsum([x.size for x in X])]).astype(object)
    n = int(off[-1])
    p = len(X)
    T = []
    for i in range(s * p - 1):
        q = (_splitmix_py(seed, i) * n) >> 64
        k = max(kk for kk in range(p) if off[kk] <= q and X[kk].size > 0 and q < off[kk] + X[kk].size)
        T.append((int(X[k][q - off[k]]), k, int(q - off[k])))
    T.sort()
    return X, [T[i * s - 1] for i in range(1, p)]


@pytest.mark.parametrize("p,sizes_seed", [(2, 1), (3, 2), (4, 3), (8, 4)])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal"])
def test_splitters_and_split_from_the_definition(p, sizes_seed, dist):
    rng = np.random.default_rng(sizes_seed)
    sizes = [int(x) for x in rng.integers(50, 400, p)]
    s, seed = 7, 1000 + sizes_seed
    a, blocks = _blocks(sizes, 60 + p, dist)
    res = oracle.ger(blocks, s=s, seed=seed)
    X, S = _definition(blocks, s, seed)
    assert [tuple(int(v) for v in row) for row in res["splitters"]] == S
    # bucket j = {(x, k, q) : S_{j-1} < (x, k, q) <= S_j}, element by element
    for k in range(p):
        for j in range(p):
            lo = S[j - 1] if j > 0 else None
            hi = S[j] if j < p - 1 else None
            c = sum(1 for q in range(X[k].size)
                    if (lo is None or (int(X[k][q]), k, q) > lo) and (hi is None or (int(X[k][q]), k, q) <= hi))
            assert res["counts"][k][j] == c, (k, j)
    assert (np.concatenate(res["Y"]) == np.sort(a)).all()


@pytest.mark.parametrize("p", [1, 2, 5, 8])
@pytest.mark.parametrize("dist", ["uniform", "sorted", "reversed", "gauss"])
def test_concatenation_is_the_sort(p, dist):
    a, blocks = _blocks([3000 + 7 * k for k in range(p)], 70 + p, dist)
    res = oracle.ger(blocks, s=16, seed=5)
    assert (np.concatenate(res["Y"]) == np.sort(a)).all()
    assert (res["counts"].sum(axis=0) == res["Ylen"]).all()


def test_empty_blocks_and_empty_input():
    a, blocks = _blocks([0, 500, 0, 300], 77)
    res = oracle.ger(blocks, s=5, seed=9)
    assert (np.concatenate(res["Y"]) == np.sort(a)).all()
    res = oracle.ger([np.zeros(0, np.uint32)] * 3, s=4, seed=1)
    assert all(y.size == 0 for y in res["Y"])


def test_pairs_globally_stable_narrow_keys():
    p, N = 4, 1200
    k = inputs.gen_u64(p * N, 8, "mod1024") & np.uint64(15)
    v = inputs.iota_u32(p * N)
    res = oracle.ger([k[i * N:(i + 1) * N] for i in range(p)], s=9, seed=3,
                     vals=[v[i * N:(i + 1) * N] for i in range(p)])
    order = np.lexsort((v, k))
    assert (np.concatenate(res["Y"]) == k[order]).all()
    assert (np.concatenate(res["Yv"]) == v[order]).all()


def _lemma_eps(n, p, s, rho=1.0):
    """Smallest ε of Lemma Sampling1 (natural logarithms): s ≥ (1+ε)/ε²·A."""
    ps1 = p * s - 1
    A = 2 * rho * math.log(n) + math.log(2 * math.pi * p * p * ps1 * math.exp(1 / (3 * ps1)))
    return (A + math.sqrt(A * A + 4 * s * A)) / (2 * s)


def test_sampling_lemma_bound_over_seeds():
    """Lemma Sampling1 (ρ = 1): P(some bucket of non-sample keys > ⌈(1+ε)(n−p+1)/p⌉)
    ≤ 1/n.  A bucket holds at most s sample keys (the splitters are every s-th
    sample), so |Y_j| − s must stay within the bound; 40 seeds on distinct keys."""
    p, n = 8, 40000
    s = oracle_default_s(n)
    eps = _lemma_eps(n, p, s)
    bound = math.ceil((1 + eps) * (n - p + 1) / p)
    a = np.random.default_rng(0).permutation(n).astype(np.uint32)  # distinct keys (the lemma's setting)
    blocks = [a[k * n // p:(k + 1) * n // p] for k in range(p)]
    worst = 0
    for seed in range(40):
        res = oracle.ger(blocks, s=s, seed=seed)
        worst = max(worst, int(res["Ylen"].max()) - s)
    assert worst <= bound, (worst, bound)


def oracle_default_s(n):
    # reading R30: s = 2⌈ω⌉²⌈lg n⌉ with ω = lg lg n
    lg = math.log2(n)
    w = max(1, math.ceil(math.log2(lg)))
    return int(2 * w * w * math.ceil(lg))


# ---------------------------------------------------------------- GVR ----
def _gvr_definition(blocks, s, seed):
    """Steps 1-2 of Algorithm GVR from the definition: draws over the UNSORTED blocks."""
    off = np.concatenate([[0], np.cumsum([b.size for b in blocks])]).astype(object)
    n = int(off[-1])
    p = len(blocks)
    T = []
    for i in range(s * p - 1):
        q = (_splitmix_py(seed, i) * n) >> 64
        k = max(kk for kk in range(p) if blocks[kk].size > 0 and off[kk] <= q < off[kk] + blocks[kk].size)
        T.append((int(blocks[k][q - off[k]]), k, int(q - off[k])))
    T.sort()
    return [T[i * s - 1] for i in range(1, p)]


@pytest.mark.parametrize("p", [2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "sorted"])
def test_gvr_splitters_destinations_and_result(p, dist):
    """GVR: splitters from the definition over the unsorted
    blocks; X_{k,j} = keys of X_k whose composite (x, k, q) lies in (S_{j-1}, S_j],
    counted element by element; Y = sorted input."""
    rng = np.random.default_rng(p)
    sizes = [int(x) for x in rng.integers(40, 300, p)]
    s, seed = 6, 500 + p
    a, blocks = _blocks(sizes, 90 + p, dist)
    res = oracle.gvr(blocks, s=s, seed=seed)
    S = _gvr_definition(blocks, s, seed)
    assert [tuple(int(v) for v in row) for row in res["splitters"]] == S
    for k in range(p):
        dest = [sum(1 for sp in S if sp < (int(x), k, q)) for q, x in enumerate(blocks[k])]
        assert [dest.count(j) for j in range(p)] == res["counts"][k].tolist(), k
    assert (np.concatenate(res["Y"]) == np.sort(a)).all()


def test_gvr_pairs_globally_stable_and_same_result_as_gsd():
    p, N = 4, 1000
    k = inputs.gen_u64(p * N, 12, "mod1024") & np.uint64(7)
    v = inputs.iota_u32(p * N)
    sh = [k[i * N:(i + 1) * N] for i in range(p)]
    vs = [v[i * N:(i + 1) * N] for i in range(p)]
    r1 = oracle.gvr(sh, s=11, seed=2, vals=vs)
    r0 = oracle.gsd(sh, r=8, vals=vs)
    order = np.lexsort((v, k))
    assert (np.concatenate(r1["Y"]) == k[order]).all() and (np.concatenate(r1["Yv"]) == v[order]).all()
    assert (np.concatenate(r1["Yv"]) == np.concatenate(r0["Yv"])).all()   # the sort is unique


def test_gvr_sampling_lemma_bound_over_seeds():
    p, n = 8, 40000
    s = oracle_default_s(n)
    eps = _lemma_eps(n, p, s)
    bound = math.ceil((1 + eps) * (n - p + 1) / p)
    a = np.random.default_rng(1).permutation(n).astype(np.uint32)
    blocks = [a[k * n // p:(k + 1) * n // p] for k in range(p)]
    worst = max(int(oracle.gvr(blocks, s=s, seed=seed)["Ylen"].max()) - s for seed in range(40))
    assert worst <= bound, (worst, bound)


def test_hand_trace_ger_gvr_p2_s2():
    """GER and GVR traces derived by hand (tests/golden/ger_gvr_hand_trace_p2_s2.json)
    from the PUBLISHED SplitMix64 outputs for seed 1234567: the draw positions, the
    composite sample, the splitter with its rank and position, the cuts / destinations,
    and Y_j — an outside pin of readings R28-R30 (a draw taken from the wrong block
    order, position formula or composite tie rule changes the splitter or the counts)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ger_gvr_hand_trace_p2_s2.json")))
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "splitmix64_seed1234567.json")))
    for i, q in enumerate(g["draw_positions"]):  # floor(z_i * n / 2^64) of the published vector
        assert int(ref["outputs"][i]) * g["n"] >> 64 == q
        assert oracle.splitmix64_at(g["seed"], i) == int(ref["outputs"][i])
    blocks = [np.array(b, dtype=np.uint32) for b in g["blocks"]]
    for mode in ("ger", "gvr"):
        res = getattr(oracle, mode)(blocks, s=g["s"], seed=g["seed"])
        assert res["splitters"].tolist() == g[mode]["splitters"], mode
        assert res["counts"].tolist() == g[mode]["counts"], mode
        assert [y.tolist() for y in res["Y"]] == g[mode]["Y"], mode
