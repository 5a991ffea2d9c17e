"""BASELINE configs[3] and [4] at their full sizes on the multi-GPU path: p = 8
ranks as threads on this GPU, each calling rs_sort_u32 / rs_sort_pairs_u64_u32
with its comm (LocalGroup: the multi-GPU orchestration — local sort, sample,
splitters, split, the one host sync, and the default one-pass p-way pull merge
reading the peers' blocks in place — over the in-process transport).  Too large
for the serial GSD simulator in a test: the concatenation Y_0‖…‖Y_7 is compared
element by element with the serial SR-8 oracle's sort of the whole input (keys,
and payloads for pairs), checked for order, multiset (hash + count) and 64 sampled
order statistics, and every |Y_j| against the balance bound ⌊(1 + 1/r)·N⌋ + p
(R18); pairs also for global stability (payload = global index)."""
import numpy as np
import pytest
import torch

import inputs
import oracle
import paper_1808_10292_b200 as rs
from tests.gpu_util import free_dev_gb, free_host_gb, host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config4_gsd_p8_full_size():
    n, p, r = 1 << 31, 8, 8
    N = n // p
    if free_host_gb() < 48 or free_dev_gb() < 40:
        pytest.skip("needs ~48 GB host, ~40 GB device")
    a = inputs.gen_u32(n, 4)
    h_in = oracle.multiset_hash(a)
    blocks = [torch.from_numpy(a[k * N:(k + 1) * N].view(np.int32)).cuda() for k in range(p)]
    got = rs.sort_ranks(blocks, "gsd", r=r, digit_bits=8)
    del blocks
    ys = [host(y, np.uint32) for y in got["Y"]]
    del got["Y"]
    torch.cuda.empty_cache()
    assert max(y.size for y in ys) <= N + N // r + p
    y = np.concatenate(ys)
    del ys
    assert y.size == n
    assert oracle.is_nondecreasing(y)
    assert oracle.multiset_hash(y) == h_in
    pos = np.unique(np.linspace(0, n - 1, 64).astype(np.uint64))
    assert oracle.check_order_stats_u32(a, pos, y[pos.astype(np.int64)]) == 0
    assert np.array_equal(y, oracle.sr(a, 8))  # the serial oracle, element by element (~40 s)


def test_config5_gsd_p8_full_size():
    n, p, r = 1 << 30, 8, 8
    N = n // p
    if free_host_gb() < 80 or free_dev_gb() < 60:
        pytest.skip("needs ~80 GB host, ~60 GB device")
    k = inputs.gen_u64(n, 5)
    v = inputs.iota_u32(n)
    h_in = oracle.multiset_hash(k, v)
    kb = [torch.from_numpy(k[i * N:(i + 1) * N].view(np.int64)).cuda() for i in range(p)]
    vb = [torch.from_numpy(v[i * N:(i + 1) * N].view(np.int32)).cuda() for i in range(p)]
    got = rs.sort_ranks(kb, "gsd", r=r, digit_bits=8, vals=vb)
    del kb, vb
    yk = [host(t, np.uint64) for t in got["Y"]]
    yv = [host(t, np.uint32) for t in got["Yv"]]
    del got
    torch.cuda.empty_cache()
    assert max(y.size for y in yk) <= N + N // r + p
    gk, gv = np.concatenate(yk), np.concatenate(yv)
    del yk, yv
    assert gk.size == n
    assert oracle.pairs_stable(gk, gv)
    assert oracle.multiset_hash(gk, gv) == h_in
    wk, wv = oracle.sr(k, 8, vals=v)  # the serial oracle, element by element
    del k, v
    assert np.array_equal(gk, wk) and np.array_equal(gv, wv)


def test_config4_every_collective_mode_p8_full_size():
    """configs[3] at full size through every collective path at p = 8 — GER, GVR
    (random oversampling), PR4 across ranks, BTN and OET — each concatenation
    compared element by element with the serial oracle's sort (computed once)."""
    n, p = 1 << 31, 8
    N = n // p
    if free_host_gb() < 48 or free_dev_gb() < 40:
        pytest.skip("needs ~48 GB host, ~40 GB device")
    a = inputs.gen_u32(n, 4)
    want = oracle.sr(a, 8)
    for mode in ("ger", "gvr", "pr4", "btn", "oet"):
        blocks = [torch.from_numpy(a[k * N:(k + 1) * N].view(np.int32)).cuda() for k in range(p)]
        got = rs.sort_ranks(blocks, mode, digit_bits=8, seed=11)
        del blocks
        ys = [host(y, np.uint32) for y in got["Y"]]
        del got
        torch.cuda.empty_cache()
        y = np.concatenate(ys)
        del ys
        assert y.size == n, mode
        assert np.array_equal(y, want), mode
        del y
