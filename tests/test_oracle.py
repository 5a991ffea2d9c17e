"""Pins of the SR-b oracle (oracle/sr.c) to things other than itself:
library sorts, brute force over every short sequence on a 4-letter alphabet,
the masked-stable-sort identity for intermediate rounds, and
np.bincount for the counting step.  PAPER.md:653-681 (SR4 count-sort rounds)."""
import itertools
import json
import os

import numpy as np
import pytest

import inputs
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cases_u32(n, seed):
    u = inputs.gen_u32(n, seed)
    return {
        "uniform": u,
        "ascending": np.sort(u),
        "descending": np.sort(u)[::-1].copy(),
        "constant": np.full(n, 0xDEADBEEF, dtype=np.uint32),
        "mod16": u & np.uint32(15),
        "all_distinct_bytes": (np.arange(n, dtype=np.uint32) * np.uint32(0x01010101)),
        "extremes": np.where(u & np.uint32(1), np.uint32(0xFFFFFFFF), np.uint32(0)).astype(np.uint32),
    }


@pytest.mark.parametrize("b", [8, 16])
def test_sr_u32_equals_library_sort(b):
    for name, a in _cases_u32(3001, 11).items():
        assert (oracle.sr(a, b) == np.sort(a, kind="stable")).all(), name


@pytest.mark.parametrize("b", [8, 16])
def test_sr_u64_equals_library_sort(b):
    a = inputs.gen_u64(2777, 12)
    assert (oracle.sr(a, b) == np.sort(a)).all()
    a2 = a & np.uint64(0xFF00FF)
    assert (oracle.sr(a2, b) == np.sort(a2)).all()


@pytest.mark.parametrize("b", [8, 16])
@pytest.mark.parametrize("dist", ["uniform", "mod1024"])
def test_sr_pairs_stable_equals_lexsort(b, dist):
    k = inputs.gen_u64(4099, 5, dist)
    v = inputs.iota_u32(4099)
    ks, vs = oracle.sr(k, b, vals=v)
    order = np.lexsort((v, k))              # primary key k, ties by original index
    assert (ks == k[order]).all() and (vs == v[order]).all()
    assert oracle.pairs_stable(ks, vs)


def test_sr_pairs_stable_with_arbitrary_payload():
    k = inputs.gen_u64(3000, 9, "mod1024") & np.uint64(7)
    v = inputs.gen_u32(3000, 10)            # payload not the index: stability = input order
    ks, vs = oracle.sr(k, 8, vals=v)
    order = np.argsort(k, kind="stable")
    assert (ks == k[order]).all() and (vs == v[order]).all()


@pytest.mark.parametrize("b", [8, 16])
def test_intermediate_rounds_are_masked_stable_sorts(b):
    """After t rounds the array is the stable sort by the low t·b bits
    (SPEC.md:208-209 'masking oracle'); this is what GPU pass t must equal."""
    a = inputs.gen_u32(5000, 13)
    for t in range(0, 32 // b + 1):
        mask = np.uint32((1 << (t * b)) - 1) if t * b < 32 else np.uint32(0xFFFFFFFF)
        want = a[np.argsort(a & mask, kind="stable")]
        assert (oracle.sr(a, b, rounds=t) == want).all(), t
    k = inputs.gen_u64(3000, 14)
    for t in range(0, 64 // b + 1):
        mask = np.uint64((1 << (t * b)) - 1) if t * b < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
        want = k[np.argsort(k & mask, kind="stable")]
        assert (oracle.sr(k, b, rounds=t) == want).all(), t


def _insertion_sort(seq):
    out = list(seq)
    for i in range(1, len(out)):
        x = out[i]
        j = i - 1
        while j >= 0 and out[j] > x:
            out[j + 1] = out[j]
            j -= 1
        out[j + 1] = x
    return out


def test_brute_force_all_short_sequences():
    alphabet = [0, 1, 1 << 31, (1 << 32) - 1]
    for length in range(0, 7):
        for seq in itertools.product(alphabet, repeat=length):
            a = np.array(seq, dtype=np.uint32)
            want = _insertion_sort(seq)
            assert oracle.sr(a, 8).tolist() == want, seq
            if length <= 4:
                assert oracle.sr(a, 16).tolist() == want, seq


def test_hist_equals_bincount():
    a = inputs.gen_u32(4096, 15)
    for b in (8, 16):
        h = oracle.hist(a, b)
        for t in range(32 // b):
            d = (a >> np.uint32(t * b)) & np.uint32((1 << b) - 1)
            assert (h[t] == np.bincount(d, minlength=1 << b)).all()
        assert (h.sum(axis=1) == a.size).all()   # histogram conservation
    k = inputs.gen_u64(1000, 16)
    h = oracle.hist(k, 8)
    for t in range(8):
        d = (k >> np.uint64(8 * t)) & np.uint64(255)
        assert (h[t] == np.bincount(d.astype(np.int64), minlength=256)).all()


def test_spec_tiny_cases():
    g = json.load(open(os.path.join(GOLD, "spec_tiny_cases.json")))
    c = g["countsort_digit0"]
    got = oracle.sr(np.array(c["input"], dtype=np.uint32), c["b"], rounds=c["rounds"])
    assert got.tolist() == c["output"]
    for case in g["sr4"]:
        assert oracle.sr(np.array(case["input"], dtype=np.uint32), 8).tolist() == case["output"]
    blocks = [np.array(b, dtype=np.uint32) for b in g["pr_p2"]["blocks"]]
    assert oracle.sr(np.concatenate(blocks), 8).tolist() == g["pr_p2"]["output"]


def test_radix256_and_radix65536_identical():
    """PR4 and PR2 produce bitwise identical output."""
    a = inputs.gen_u32(20000, 2, "half")
    assert (oracle.sr(a, 8) == oracle.sr(a, 16)).all()


def test_bad_digit_width_rejected():
    with pytest.raises(ValueError):
        oracle.sr(np.arange(4, dtype=np.uint32), 4)


def test_invariant_checkers_detect_errors():
    a = inputs.gen_u32(1000, 17)
    s = np.sort(a)
    assert oracle.is_nondecreasing(s) and not oracle.is_nondecreasing(a)
    assert oracle.multiset_hash(a) == oracle.multiset_hash(s)
    t = s.copy()
    t[5] += np.uint32(1)
    assert oracle.multiset_hash(t) != oracle.multiset_hash(s)
    pos = np.array([0, 1, 500, 999], dtype=np.uint64)
    assert oracle.check_order_stats_u32(a, pos, s[pos.astype(np.int64)]) == 0
    bad = s[pos.astype(np.int64)].copy()
    bad[2] = s[600] if s[600] != s[500] else s[900]
    assert oracle.check_order_stats_u32(a, pos, bad) == 1
    k = inputs.gen_u64(500, 3, "mod1024") & np.uint64(3)
    v = inputs.iota_u32(500)
    ks, vs = oracle.sr(k, 8, vals=v)
    assert oracle.pairs_stable(ks, vs)
    vs2 = vs.copy()
    i = int(np.nonzero(ks[1:] == ks[:-1])[0][0])
    vs2[i], vs2[i + 1] = vs2[i + 1], vs2[i]
    assert not oracle.pairs_stable(ks, vs2)
    assert oracle.multiset_hash(ks, vs) == oracle.multiset_hash(k, v)
    vs3 = vs.copy()
    j = int(np.nonzero(ks[1:] != ks[:-1])[0][0])       # swap payloads across different keys
    vs3[j], vs3[j + 1] = vs3[j + 1], vs3[j]
    assert oracle.multiset_hash(ks, vs3) != oracle.multiset_hash(k, v)
