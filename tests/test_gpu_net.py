"""GPU parity of BTN and OET: rs_sort_* with a comm in BTN / OET
mode (rs_comm_set_sampling 4 / 5), one call per rank, the ranks being threads on
this GPU (LocalGroup: the multi-GPU orchestration over the in-process transport;
each rank computes its merge-split half reading its partner's block in place)
against the CPU oracle (oracle/net.c): every block bit-exact, values included
(both sides merge ties lower-indexed block first, so BTN's non-stable value order
is also determined)."""
import numpy as np
import pytest
import torch

import inputs
import oracle
import paper_1808_10292_b200 as rs
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


def _check(mode, blocks_np, b=8, vals_np=None):
    dt = blocks_np[0].dtype
    want = getattr(oracle, mode)(blocks_np, b=b, vals=vals_np)
    got = rs.sort_ranks([dev(x) for x in blocks_np], mode, digit_bits=b,
                        vals=[dev(v) for v in vals_np] if vals_np is not None else None)
    for j in range(len(blocks_np)):
        assert (host(got["Y"][j], dt) == want["Y"][j]).all(), j
        if vals_np is not None:
            assert (host(got["Yv"][j], np.uint32) == want["Yv"][j]).all(), j
    assert rs.net_stages(mode, len(blocks_np)) == want["stages"]


def _blocks_u32(p, N, seed, dist):
    a = inputs.gen_u32(p * N, seed, dist)
    return [a[k * N:(k + 1) * N].copy() for k in range(p)]


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "equal", "reversed"])
def test_btn_u32(p, dist):
    # N spans several merge tiles with a ragged tail
    _check("btn", _blocks_u32(p, 20011, 100 + p, dist))


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["uniform", "mod16", "sorted", "gauss"])
def test_oet_u32(p, dist):
    _check("oet", _blocks_u32(p, 20011, 200 + p, dist))


@pytest.mark.parametrize("mode,p", [("btn", 8), ("oet", 6)])
@pytest.mark.parametrize("b", [8, 16])
def test_pairs_u64(mode, p, b):
    N = 12345
    k = inputs.gen_u64(p * N, 300 + p + b, "mod1024")
    v = inputs.iota_u32(k.size)
    _check(mode, [k[i * N:(i + 1) * N].copy() for i in range(p)], b=b,
           vals_np=[v[i * N:(i + 1) * N].copy() for i in range(p)])


@pytest.mark.parametrize("mode", ["btn", "oet"])
def test_u64_keys_radix16(mode):
    N = 7777
    k = inputs.gen_u64(4 * N, 77, "uniform")
    _check(mode, [k[i * N:(i + 1) * N].copy() for i in range(4)], b=16)


@pytest.mark.parametrize("mode", ["btn", "oet"])
@pytest.mark.parametrize("N", [0, 1, 2, 5])
def test_tiny_and_empty_blocks(mode, N):
    _check(mode, _blocks_u32(4, N, 9, "uniform"))


def test_stage_counts_and_errors():
    assert [rs.net_stages("btn", 1 << m) for m in range(6)] == [0, 1, 3, 6, 10, 15]
    assert [rs.net_stages("oet", p) for p in (1, 2, 3, 7)] == [1, 2, 3, 7]
    with pytest.raises(ValueError):
        rs.net_stages("btn", 6)
    with pytest.raises(rs.RSortError):  # BTN over 3 ranks: RS_EINVAL on every rank
        rs.sort_ranks([dev(np.zeros(4, np.uint32)) for _ in range(3)], "btn")
    with pytest.raises(rs.RSortError):  # unequal blocks
        rs.sort_ranks([dev(np.zeros(4, np.uint32)), dev(np.zeros(5, np.uint32))], "oet")


@pytest.mark.parametrize("mode", ["btn", "oet"])
def test_large_blocks_property(mode):
    """p = 8 blocks of 2^22 keys: the concatenation equals the library sort (a
    property that holds at any size; the oracle runs the element-wise cases)."""
    p, N = 8, 1 << 22
    a = torch.randint(0, 1 << 32, (p * N,), dtype=torch.int64, device="cuda").to(torch.int32)
    got = rs.sort_ranks([a[k * N:(k + 1) * N].clone() for k in range(p)], mode)
    y = torch.cat(got["Y"]).to(torch.int64) & 0xFFFFFFFF
    want = torch.sort(a.to(torch.int64) & 0xFFFFFFFF).values
    assert torch.equal(y, want)
