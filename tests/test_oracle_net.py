"""Pins of the BTN / OET oracle (oracle/net.c) against what the paper and the
mathematics fix, not against the oracle itself.

  * stage counts: lg p (lg p + 1)/2 for BTN, p rounds for OET
    (PAPER.md:518-521);
  * the 0-1 principle: with one key per block BTN is Batcher's bitonic sorting
    network and OET the odd-even transposition network; a comparator network sorts
    every input iff it sorts every 0/1 input (Knuth, TAOCP 5.3.4) — exhaustive over
    all 0/1 inputs for p = 8 and 16;
  * brute force over every input on a 3-letter alphabet for p = 4 blocks of 2;
  * hand traces: SPEC.md:246 (OET p = 2) and the bitonic p = 4 network stage by
    stage (derived by hand from reading R32);
  * the final distribution equals the library sort of the concatenation (numpy);
  * OET with values is the stable sort (merge-split of adjacent blocks with ties to
    the lower index preserves the order of equal keys); BTN permutes pairs.
"""
import itertools

import numpy as np
import pytest

import oracle


def _cat(o):
    return np.concatenate(o["Y"]) if o["Y"] else np.empty(0)


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16, 32])
def test_stage_counts(p):
    m = p.bit_length() - 1
    bl = [np.arange(3, dtype=np.uint32)[::-1].copy() for _ in range(p)]
    assert oracle.btn(bl)["stages"] == m * (m + 1) // 2
    assert oracle.oet(bl)["stages"] == p


def test_btn_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        oracle.btn([np.zeros(2, np.uint32)] * 3)
    o = oracle.oet([np.array([5, 4], np.uint32), np.array([3, 2], np.uint32), np.array([1, 0], np.uint32)])
    assert _cat(o).tolist() == [0, 1, 2, 3, 4, 5]


def test_unequal_blocks_rejected():
    with pytest.raises(ValueError):
        oracle.oet([np.zeros(2, np.uint32), np.zeros(3, np.uint32)])


def test_oet_spec_hand_trace():
    # blocks [9,10] and [1,2]; round 1 (pair (0,1)) -> [1,2],[9,10]
    bl = [np.array([9, 10], np.uint32), np.array([1, 2], np.uint32)]
    o = oracle.oet(bl, max_stages=1)
    assert [y.tolist() for y in o["Y"]] == [[1, 2], [9, 10]] and o["stages"] == 1
    o = oracle.oet(bl)
    assert [y.tolist() for y in o["Y"]] == [[1, 2], [9, 10]] and o["stages"] == 2


def test_btn_p4_hand_trace():
    # stage 1 (k=1, j=1): (0,1) ascending, (2,3) descending (bit 1 of 2 is set)
    #   [3] [1] [2] [4] -> [1] [3] [4] [2]   (a bitonic sequence)
    # stage 2 (k=2, j=2): 0<->2, 1<->3 ascending -> [1] [2] [4] [3]
    # stage 3 (k=2, j=1): 0<->1, 2<->3 ascending -> [1] [2] [3] [4]
    bl = [np.array([x], np.uint32) for x in (3, 1, 2, 4)]
    want = [[1, 3, 4, 2], [1, 2, 4, 3], [1, 2, 3, 4]]
    for s, w in enumerate(want, start=1):
        assert _cat(oracle.btn(bl, max_stages=s)).tolist() == w
    # with blocks of two the halves move the same way
    bl2 = [np.array([5, 6], np.uint32), np.array([1, 2], np.uint32), np.array([3, 4], np.uint32),
           np.array([7, 8], np.uint32)]
    assert [y.tolist() for y in oracle.btn(bl2, max_stages=1)["Y"]] == [[1, 2], [5, 6], [7, 8], [3, 4]]


@pytest.mark.parametrize("p", [8, 16])
def test_zero_one_principle_btn(p):
    for bits in range(1 << p):
        bl = [np.array([(bits >> i) & 1], np.uint32) for i in range(p)]
        got = _cat(oracle.btn(bl))
        assert got.tolist() == sorted(got.tolist()), bits


def test_zero_one_principle_oet():
    p = 8
    for bits in range(1 << p):
        bl = [np.array([(bits >> i) & 1], np.uint32) for i in range(p)]
        got = _cat(oracle.oet(bl))
        assert got.tolist() == sorted(got.tolist()), bits
    # p - 1 rounds are not enough in general for OET (the reversed 0/1 input needs p)
    bl = [np.array([1], np.uint32)] * 4 + [np.array([0], np.uint32)] * 4
    assert _cat(oracle.oet(bl, max_stages=p - 2)).tolist() != sorted([0] * 4 + [1] * 4)


@pytest.mark.parametrize("fn", ["btn", "oet"])
def test_brute_force_alphabet3(fn):
    f = getattr(oracle, fn)
    for seq in itertools.product(range(3), repeat=8):
        a = np.array(seq, np.uint32)
        got = _cat(f([a[0:2], a[2:4], a[4:6], a[6:8]]))
        assert got.tolist() == sorted(seq), seq


@pytest.mark.parametrize("fn", ["btn", "oet"])
@pytest.mark.parametrize("dt,b", [(np.uint32, 8), (np.uint32, 16), (np.uint64, 8), (np.uint64, 16)])
def test_library_sort(fn, dt, b):
    rng = np.random.default_rng(7)
    p, N = 8, 1000
    hi = np.iinfo(dt).max
    bl = [rng.integers(0, hi, N, dtype=dt, endpoint=True) for _ in range(p)]
    bl[3][:500] = bl[5][0]  # duplicates across blocks
    o = getattr(oracle, fn)(bl, b=b)
    assert np.array_equal(_cat(o), np.sort(np.concatenate(bl)))
    assert all(y.size == N for y in o["Y"])


def test_oet_pairs_stable_btn_pairs_permuted():
    rng = np.random.default_rng(3)
    p, N = 8, 300
    bl = [rng.integers(0, 40, N, dtype=np.uint64) for _ in range(p)]
    vals = [np.arange(k * N, (k + 1) * N, dtype=np.uint32) for k in range(p)]
    keys = np.concatenate(bl)
    order = np.argsort(keys, kind="stable")
    o = oracle.oet(bl, vals=vals)
    assert np.array_equal(_cat(o), keys[order])
    assert np.array_equal(np.concatenate(o["Yv"]), order.astype(np.uint32))
    o = oracle.btn(bl, vals=vals)
    k2, v2 = _cat(o), np.concatenate(o["Yv"])
    assert np.array_equal(k2, keys[order])
    assert np.array_equal(keys[v2], k2)  # every value still rides with its key
    assert sorted(v2.tolist()) == list(range(p * N))
