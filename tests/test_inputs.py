"""Seeded input generator: pinned to the published SplitMix64 vector and to the
distribution shapes of BASELINE.json configs."""
import json
import os

import numpy as np
import pytest

import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_published_vector():
    g = json.load(open(os.path.join(GOLD, "splitmix64_seed1234567.json")))
    got = [inputs.splitmix64_at(g["seed"], i) for i in range(len(g["outputs"]))]
    assert got == [int(x) for x in g["outputs"]]


def _np_splitmix(seed, idx):
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def test_counter_form_matches_numpy_and_shards():
    idx = np.arange(5000, dtype=np.uint64)
    z = _np_splitmix(4, idx)
    assert (inputs.gen_u64(5000, 4) == z).all()
    assert (inputs.gen_u32(5000, 4) == (z >> np.uint64(32)).astype(np.uint32)).all()
    # sharding: [start, start+count) of the global stream
    full = inputs.gen_u32(4096, 7)
    parts = [inputs.gen_u32(1024, 7, start=k * 1024) for k in range(4)]
    assert (np.concatenate(parts) == full).all()


def test_distribution_shapes():
    n = 1 << 16
    u = inputs.gen_u32(n, 3, "uniform")
    assert u.max() > (1 << 31) and u.min() < (1 << 20)
    m = inputs.gen_u32(n, 3, "mod16")
    assert set(np.unique(m).tolist()) == set(range(16))
    h = inputs.gen_u32(n, 2, "half")
    assert h.max() < (1 << 31)
    s = inputs.gen_u32(n, 3, "sorted")
    assert (np.diff(s.astype(np.int64)) >= 0).all() and s[-1] > (1 << 31)
    r = inputs.gen_u32(n, 3, "reversed")
    assert (r == s[::-1]).all()
    e = inputs.gen_u32(n, 3, "equal")
    assert (e == e[0]).all() and e[0] == (inputs.splitmix64_at(3, 0) >> 32)
    g = inputs.gen_u32(n, 3, "gauss").astype(np.float64)
    assert abs(g.mean() - 2 ** 31) < 0.02 * 2 ** 28
    assert abs(g.std() - 2 ** 28) < 0.02 * 2 ** 28
    k = inputs.gen_u64(n, 5, "mod1024")
    assert k.max() < 1024


def test_sorted_shards_agree_with_global():
    n = 10000
    full = inputs.gen_u32(n, 3, "sorted")
    part = inputs.gen_u32(2500, 3, "sorted", start=5000, n_total=n)
    assert (part == full[5000:7500]).all()


def test_frozen_prefixes():
    g = json.load(open(os.path.join(GOLD, "inputs_frozen.json")))
    for name, rec in g["u32"].items():
        dist, seed, n_total = rec["dist"], rec["seed"], rec["n_total"]
        got = inputs.gen_u32(16, seed, dist, n_total=n_total)
        assert got.tolist() == rec["first16"], name
    for name, rec in g["u64"].items():
        got = inputs.gen_u64(16, rec["seed"], rec["dist"])
        assert [str(x) for x in got.tolist()] == rec["first16"], name


def test_bad_args():
    with pytest.raises(KeyError):
        inputs.gen_u32(4, 1, "nope")
    with pytest.raises(ValueError):
        inputs.gen_u32(4, 1, "sorted", start=2, n_total=4)
