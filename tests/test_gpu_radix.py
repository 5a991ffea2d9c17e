"""GPU parity of the single-GPU radix sort (through the C ABI) against the
serial oracle: bit-exact after every pass, for every key type, digit width,
size edge case and BASELINE distribution (configs 1-3 at full size; configs
4-5 at p = 1 by invariants and sampled order statistics)."""
import ctypes

import numpy as np
import pytest
import torch

import inputs
import oracle
import paper_1808_10292_b200 as rs
from tests.gpu_util import dev, free_dev_gb, free_host_gb, host

pytestmark = pytest.mark.gpu


def _tile(kind):
    return rs.get_option(f"tile_{kind}")


# tiles (keys per look-back row) of the default pass design, for ragged sizes
TILE32 = _tile("u32")     # u32 keys
TILE64 = _tile("u64")     # u64 keys
TILEP = _tile("pairs")    # (u64, u32) pairs


def _sort_u32(a, b, inplace=True):
    t = dev(a)
    if inplace:
        rs.sort(t, digit_bits=b)
        return host(t, np.uint32)
    out = torch.empty_like(t)
    rs.sort(t, digit_bits=b, out=out)
    assert (host(t, np.uint32) == a).all(), "input clobbered by an out-of-place sort"
    return host(out, np.uint32)


def test_native_library_runs():
    a = inputs.gen_u32(5000, 1)
    rs.lib().rs_timing_reset()
    got = _sort_u32(a, 8)
    torch.cuda.synchronize()
    assert rs.lib().rs_launch_count() >= 6
    assert (got == oracle.sr(a, 8)).all()


@pytest.mark.parametrize("b", [8, 16])
def test_histogram_parity(b):
    a = inputs.gen_u32(3 * TILE32 + 1234, 21)
    h = rs.digit_histogram(dev(a), b).cpu().numpy().view(np.uint32)
    assert (h.astype(np.uint64) == oracle.hist(a, b)).all()
    k = inputs.gen_u64(2 * TILE64 + 77, 22)
    h = rs.digit_histogram(dev(k), b).cpu().numpy().view(np.uint32)
    assert (h.astype(np.uint64) == oracle.hist(k, b)).all()


def test_histogram_u64_large_counts():
    """K1 for u64 keys (8 passes, 16 lane-private 32-bit copies, radix8.cuh) at
    2^29 + 3 keys: a constant top byte (pass 7: one bin holds every key, ~113 K
    counts per copy per CTA), half the keys sharing byte 3, an odd tail; every
    count against the oracle."""
    n = (1 << 29) + 3
    if free_host_gb() < 16 or free_dev_gb() < 16:
        pytest.skip("needs ~16 GB host/device")
    k = inputs.gen_u64(n, 25)
    k &= np.uint64(0x00FFFFFFFFFFFFFF)
    k[: n // 2] = (k[: n // 2] & np.uint64(0xFFFFFFFF00FFFFFF)) | np.uint64(0x5A000000)
    h = rs.digit_histogram(dev(k), 8).cpu().numpy().view(np.uint32)
    want = oracle.hist(k, 8)
    assert want[7, 0] == n and want[3, 0x5A] > n // 2
    assert (h.reshape(want.shape).astype(np.uint64) == want).all()


@pytest.mark.parametrize("n", [3 * TILE32 + 1234, (1 << 20) + 7])
@pytest.mark.parametrize("b", [8, 16])
def test_every_pass_u32(n, b):
    """After pass t the array equals the oracle's array after round t (bit-exact)."""
    a = inputs.gen_u32(n, 23)
    for t in range(1, 32 // b + 1):
        got = host(rs.sort_bits(dev(a), end_bit=b * t, digit_bits=b), np.uint32)
        assert (got == oracle.sr(a, b, rounds=t)).all(), f"pass {t}"


@pytest.mark.parametrize("b", [8, 16])
def test_every_pass_u64_and_pairs(b):
    n = 5 * TILE64 + 999
    k = inputs.gen_u64(n, 24)
    v = inputs.iota_u32(n)
    for t in range(1, 64 // b + 1):
        got = host(rs.sort_bits(dev(k), end_bit=b * t, digit_bits=b), np.uint64)
        assert (got == oracle.sr(k, b, rounds=t)).all(), f"u64 pass {t}"
        gk, gv = rs.sort_bits(dev(k), end_bit=b * t, digit_bits=b, vals=dev(v))
        wk, wv = oracle.sr(k, b, rounds=t, vals=v)
        assert (host(gk, np.uint64) == wk).all() and (host(gv, np.uint32) == wv).all(), f"pairs pass {t}"


EDGE_N = sorted({1, 2, 3, 31, 32, 33, 1000, TILE64 - 1, TILE64, TILE64 + 1, TILEP - 1, TILEP, TILEP + 1,
                 TILE32 - 1, TILE32, TILE32 + 1, 2 * TILE32 + 3, 7 * TILE32 + 4095})


@pytest.mark.parametrize("tiles", [1, 2])
def test_edge_sizes_large_and_small_tiles(option, tiles):
    """Both design-5 tile sizes (large: the size-dependent default above ~6.7 M
    u32 keys; small: below) at every edge size, u32 keys, u64 keys and pairs."""
    option("small_tiles", tiles)
    for n in EDGE_N:
        a = inputs.gen_u32(n, 125 + n)
        assert (_sort_u32(a, 8) == oracle.sr(a, 8)).all(), n
        k = inputs.gen_u64(n, 126 + n, "mod1024")
        v = inputs.iota_u32(n)
        tk, tv = dev(k), dev(v)
        rs.sort_pairs(tk, tv)
        wk, wv = oracle.sr(k, 8, vals=v)
        assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all(), n
        t = dev(k)
        rs.sort(t)
        assert (host(t, np.uint64) == wk).all(), n
    a = inputs.gen_u32((1 << 21) + 77, 127)
    for t in range(1, 5):
        got = host(rs.sort_bits(dev(a), end_bit=8 * t, digit_bits=8), np.uint32)
        assert (got == oracle.sr(a, 8, rounds=t)).all(), t


@pytest.mark.parametrize("b", [8, 16])
@pytest.mark.parametrize("inplace", [True, False])
def test_edge_sizes_u32(b, inplace):
    for n in EDGE_N:
        a = inputs.gen_u32(n, 25 + n)
        assert (_sort_u32(a, b, inplace) == oracle.sr(a, b)).all(), n


@pytest.mark.parametrize("b", [8, 16])
def test_edge_sizes_u64_and_pairs(b):
    for n in EDGE_N:
        k = inputs.gen_u64(n, 26 + n, "mod1024" if n % 2 else "uniform")
        v = inputs.iota_u32(n)
        t = dev(k)
        rs.sort(t, digit_bits=b)
        assert (host(t, np.uint64) == oracle.sr(k, b)).all(), n
        tk, tv = dev(k), dev(v)
        ok_, ov_ = torch.empty_like(tk), torch.empty_like(tv)
        rs.sort_pairs(tk, tv, digit_bits=b, out_keys=ok_, out_vals=ov_)
        wk, wv = oracle.sr(k, b, vals=v)
        assert (host(ok_, np.uint64) == wk).all() and (host(ov_, np.uint32) == wv).all(), n
        assert oracle.pairs_stable(host(ok_, np.uint64), host(ov_, np.uint32))


def test_empty_input():
    t = torch.empty(0, dtype=torch.int32, device="cuda")
    rs.sort(t)
    k = torch.empty(0, dtype=torch.int64, device="cuda")
    v = torch.empty(0, dtype=torch.int32, device="cuda")
    rs.sort_pairs(k, v)


@pytest.mark.parametrize("dist", ["uniform", "mod16", "gauss", "sorted", "reversed", "equal", "half"])
@pytest.mark.parametrize("b", [8, 16])
def test_distributions(dist, b):
    a = inputs.gen_u32((1 << 20) + 3, 3, dist)
    want = oracle.sr(a, b)
    assert (_sort_u32(a, b, True) == want).all()
    assert (_sort_u32(a, b, False) == want).all()


def test_extreme_keys():
    a = inputs.gen_u32(100003, 9)
    a = np.where(a & np.uint32(1), np.uint32(0xFFFFFFFF), np.uint32(0)).astype(np.uint32)
    for b in (8, 16):
        assert (_sort_u32(a, b) == np.sort(a)).all()
    k = inputs.gen_u64(50001, 9)
    k = np.where(k & np.uint64(1), np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64(0)).astype(np.uint64)
    t = dev(k)
    rs.sort(t)
    assert (host(t, np.uint64) == np.sort(k)).all()


def test_config1():
    """BASELINE configs[0]: n=2^20 uniform u32 seed 1, radix-256, bit-exact."""
    a = inputs.gen_u32(1 << 20, 1, "uniform")
    assert (_sort_u32(a, 8) == oracle.sr(a, 8)).all()


def test_config2_radix256_vs_radix65536():
    """BASELINE configs[1]: 2^24 keys in [0,2^31) seed 2; PR4 and PR2 both bit-exact."""
    a = inputs.gen_u32(1 << 24, 2, "half")
    want = oracle.sr(a, 8)
    g8 = _sort_u32(a, 8)
    g16 = _sort_u32(a, 16)
    assert (g8 == want).all() and (g16 == want).all()


@pytest.mark.slow
@pytest.mark.parametrize("dist", ["uniform", "mod16", "gauss", "sorted", "reversed", "equal"])
def test_config3_full_size(dist):
    """BASELINE configs[2]: 2^27 u32 keys, six distributions, seed 3, bit-exact."""
    a = inputs.gen_u32(1 << 27, 3, dist)
    want = oracle.sr(a, 8)
    assert (_sort_u32(a, 8) == want).all()


@pytest.mark.slow
def test_config4_single_gpu_full_size():
    """BASELINE configs[3] at p=1 (the bench.py N=1 workload): 2^31 u32 keys,
    seed 4.  Too large for the serial oracle in a test: sortedness, multiset hash
    against the input, and 64 sampled order statistics checked one by one."""
    n = 1 << 31
    if free_host_gb() < 20 or free_dev_gb() < 20:
        pytest.skip(f"needs ~20 GB host/device (host {free_host_gb():.0f}, dev {free_dev_gb():.0f})")
    a = inputs.gen_u32(n, 4)
    h_in = oracle.multiset_hash(a)
    t = dev(a)
    rs.sort(t, digit_bits=8)
    got = host(t, np.uint32)
    del t
    torch.cuda.empty_cache()
    assert oracle.is_nondecreasing(got)
    assert oracle.multiset_hash(got) == h_in
    pos = np.unique(np.linspace(0, n - 1, 64).astype(np.uint64))
    assert oracle.check_order_stats_u32(a, pos, got[pos.astype(np.int64)]) == 0


@pytest.mark.slow
def test_config4_single_gpu_full_memcmp():
    """configs[3] at p = 1 compared element by element with the serial SR4 oracle
    (one full memcmp of 2^31 keys; the oracle takes ~40 s on one core)."""
    n = 1 << 31
    if free_host_gb() < 44 or free_dev_gb() < 20:
        pytest.skip(f"needs ~44 GB host (have {free_host_gb():.0f})")
    a = inputs.gen_u32(n, 4)
    t = dev(a)
    rs.sort(t, digit_bits=8)
    got = host(t, np.uint32)
    del t
    torch.cuda.empty_cache()
    want = oracle.sr(a, 8)
    del a
    assert np.array_equal(got, want)


@pytest.mark.slow
def test_31bit_lookback_prefixes():
    """2^31 - 1001 u32 keys whose low byte is zeroed for the first 3/4: in pass 0
    digit 0 holds > 2^30 keys, so its inclusive look-back prefixes need the 31st
    value bit of the narrow (u32) status words (radix8.cuh Status).  Checked by
    sortedness, multiset hash and sampled order statistics (full size)."""
    n = (1 << 31) - 1001
    if free_host_gb() < 20 or free_dev_gb() < 20:
        pytest.skip("needs ~20 GB host/device")
    a = inputs.gen_u32(n, 7)
    a[: 3 * n // 4] &= np.uint32(0xFFFFFF00)
    h_in = oracle.multiset_hash(a)
    t = dev(a)
    rs.sort(t, digit_bits=8)
    got = host(t, np.uint32)
    del t
    torch.cuda.empty_cache()
    assert oracle.is_nondecreasing(got)
    assert oracle.multiset_hash(got) == h_in
    pos = np.unique(np.linspace(0, n - 1, 64).astype(np.uint64))
    assert oracle.check_order_stats_u32(a, pos, got[pos.astype(np.int64)]) == 0


@pytest.mark.slow
def test_maximum_n_wide_status():
    """n = 2^32 - 1 u32 keys, the per-GPU maximum of the ABI (rsort.h: n < 2^32):
    above 2^31 the look-back status words are u64 (radix8.cuh kNarrowStatusMaxN),
    and the low byte of the first 5/8 of the keys is zeroed so pass 0's digit 0
    holds > 2^31 keys — its inclusive prefixes need the 32nd bit, and every
    32-bit position computation in the pass runs at its limit.  Checked by
    sortedness, multiset hash and 64 sampled order statistics (full size)."""
    n = (1 << 32) - 1
    if free_host_gb() < 48 or free_dev_gb() < 40:
        pytest.skip(f"needs ~48 GB host / 40 GB device (host {free_host_gb():.0f}, dev {free_dev_gb():.0f})")
    a = inputs.gen_u32(n, 9)
    a[: 5 * (n // 8)] &= np.uint32(0xFFFFFF00)
    h_in = oracle.multiset_hash(a)
    t = dev(a)
    rs.sort(t, digit_bits=8)
    got = host(t, np.uint32)
    del t
    torch.cuda.empty_cache()
    assert oracle.is_nondecreasing(got)
    assert oracle.multiset_hash(got) == h_in
    pos = np.unique(np.linspace(0, n - 1, 64).astype(np.uint64))
    assert oracle.check_order_stats_u32(a, pos, got[pos.astype(np.int64)]) == 0


@pytest.mark.slow
def test_config5_single_gpu_full_size():
    """BASELINE configs[4] at p=1: 2^30 (u64 key, u32 payload = index) pairs,
    seed 5, 8 radix-256 passes; stability via payload order."""
    n = 1 << 30
    if free_host_gb() < 30 or free_dev_gb() < 30:
        pytest.skip("needs ~30 GB host/device")
    k = inputs.gen_u64(n, 5)
    v = inputs.iota_u32(n)
    h_in = oracle.multiset_hash(k, v)
    tk, tv = dev(k), dev(v)
    del k, v
    rs.sort_pairs(tk, tv, digit_bits=8)
    gk, gv = host(tk, np.uint64), host(tv, np.uint32)
    del tk, tv
    torch.cuda.empty_cache()
    assert oracle.pairs_stable(gk, gv)
    assert oracle.multiset_hash(gk, gv) == h_in


@pytest.mark.slow
def test_pairs_above_2p31_wide_status():
    """(u64 key, u32 index) pairs with n = 2^31 + 7: the pairs pass with u64
    look-back status words (n > 2^31), the top byte of 5/8 of the keys cleared so
    pass 7's digit 0 holds > 2^31 pairs (inclusive prefixes past 31 bits).  The
    payload is the input index, so nondecreasing keys + increasing payloads among
    equal keys + the pair multiset hash pin the unique stable output."""
    n = (1 << 31) + 7
    if free_host_gb() < 64 or free_dev_gb() < 60:
        pytest.skip(f"needs ~64 GB host / 60 GB device (host {free_host_gb():.0f}, dev {free_dev_gb():.0f})")
    k = inputs.gen_u64(n, 27)
    k[: 5 * (n // 8)] &= np.uint64(0x00FFFFFFFFFFFFFF)
    v = inputs.iota_u32(n)
    h_in = oracle.multiset_hash(k, v)
    tk, tv = dev(k), dev(v)
    del k, v
    rs.sort_pairs(tk, tv, digit_bits=8)
    gk, gv = host(tk, np.uint64), host(tv, np.uint32)
    del tk, tv
    torch.cuda.empty_cache()
    assert oracle.pairs_stable(gk, gv)
    assert oracle.multiset_hash(gk, gv) == h_in


@pytest.mark.slow
def test_config5_single_gpu_full_memcmp():
    """configs[4] at p = 1 compared element by element with the serial SR-8 oracle:
    2^30 (u64 key, u32 index) pairs, all 8 passes, keys and payloads."""
    n = 1 << 30
    if free_host_gb() < 64 or free_dev_gb() < 30:
        pytest.skip(f"needs ~64 GB host (have {free_host_gb():.0f})")
    k = inputs.gen_u64(n, 5)
    v = inputs.iota_u32(n)
    tk, tv = dev(k), dev(v)
    rs.sort_pairs(tk, tv, digit_bits=8)
    gk, gv = host(tk, np.uint64), host(tv, np.uint32)
    del tk, tv
    torch.cuda.empty_cache()
    wk, wv = oracle.sr(k, 8, vals=v)
    del k, v
    assert np.array_equal(gk, wk)
    assert np.array_equal(gv, wv)


def test_narrow_pairs_stability_at_scale():
    """configs[4] narrow-range variant: key = z mod 1024, many equal keys."""
    n = (1 << 22) + 5
    k = inputs.gen_u64(n, 5, "mod1024")
    v = inputs.iota_u32(n)
    for b in (8, 16):
        tk, tv = dev(k), dev(v)
        rs.sort_pairs(tk, tv, digit_bits=b)
        wk, wv = oracle.sr(k, b, vals=v)
        assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all()


get_option = rs.get_option


@pytest.fixture
def option():
    saved = {}

    def _set(name, value):
        saved.setdefault(name, get_option(name))
        rs.set_option(name, value)
    yield _set
    for name, value in saved.items():
        rs.set_option(name, value)


def test_atomic_rank_probe_passes():
    """Design 5 (the default pass) ranks keys by the old values of warp-wide
    shared atomicAdd; the library enables it only after its probe kernel found
    those values in lane order for every same-address group on this device.
    On a B200 the probe must pass, so the parity tests run design 5."""
    a = inputs.gen_u32(3 * TILE32 + 11, 50)
    assert (_sort_u32(a, 8) == oracle.sr(a, 8)).all()
    assert get_option("pass_design") == 5
    assert get_option("rank_probe") == 1


@pytest.mark.parametrize("kind", ["u32", "u64", "pairs"])
def test_wide_status_lookback(option, kind):
    """64-bit look-back status words (used when n >= 2^30, configs 4/5 at p = 1)
    forced at small n, every pass checked, ragged tail."""
    option("wide_status", 1)
    tile = TILE32 if kind == "u32" else TILE64
    n = 11 * tile + 517
    if kind == "u32":
        a = inputs.gen_u32(n, 31)
        for t in range(1, 5):
            got = host(rs.sort_bits(dev(a), end_bit=8 * t, digit_bits=8), np.uint32)
            assert (got == oracle.sr(a, 8, rounds=t)).all(), t
        assert (_sort_u32(a, 8) == oracle.sr(a, 8)).all()
    else:
        k = inputs.gen_u64(n, 32, "mod1024" if kind == "pairs" else "uniform")
        v = inputs.iota_u32(n)
        if kind == "u64":
            t = dev(k)
            rs.sort(t)
            assert (host(t, np.uint64) == oracle.sr(k, 8)).all()
        else:
            tk, tv = dev(k), dev(v)
            rs.sort_pairs(tk, tv)
            wk, wv = oracle.sr(k, 8, vals=v)
            assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all()


@pytest.mark.parametrize("design", [2, 5])
@pytest.mark.parametrize("wide", [0, 1])
def test_pass_designs(option, design, wide):
    """The default atomic-rank pass (5) and the ballot-rank fallback / safe mode
    (2) are bit-exact after every pass, for u32 keys and (u64, u32) pairs, narrow
    and wide status words."""
    option("pass_design", design)
    option("wide_status", wide)
    n = 9 * TILE32 + 4321
    a = inputs.gen_u32(n, 41)
    for t in range(1, 5):
        got = host(rs.sort_bits(dev(a), end_bit=8 * t, digit_bits=8), np.uint32)
        assert (got == oracle.sr(a, 8, rounds=t)).all(), t
    for dist in ("mod16", "sorted"):
        b = inputs.gen_u32(n, 42, dist)
        assert (_sort_u32(b, 8) == oracle.sr(b, 8)).all(), dist
    k = inputs.gen_u64(5 * TILE64 + 77, 43, "mod1024")
    v = inputs.iota_u32(k.size)
    tk, tv = dev(k), dev(v)
    rs.sort_pairs(tk, tv)
    wk, wv = oracle.sr(k, 8, vals=v)
    assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all()


def test_self_check_mode(option):
    """Debug self-check: every local sort verified on the device (the host waits
    for the verdict); a correct sort passes, at full tiles and ragged sizes."""
    option("self_check", 1)
    for n in (1, 5000, 3 * TILE32 + 7):
        a = inputs.gen_u32(n, 47 + n)
        assert (_sort_u32(a, 8) == oracle.sr(a, 8)).all(), n
    k = inputs.gen_u64(2 * TILEP + 3, 48)
    v = inputs.iota_u32(k.size)
    tk, tv = dev(k), dev(v)
    rs.sort_pairs(tk, tv)
    wk, wv = oracle.sr(k, 8, vals=v)
    assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all()


def test_cuda_graph_capture_and_replay():
    """The single-GPU sort is stream-ordered with no host synchronisation (after
    the one-time probe), so it can be captured in a CUDA graph and replayed:
    launch overhead disappears for small inputs (config 1)."""
    n = 1 << 20
    a = inputs.gen_u32(n, 1)
    want = oracle.sr(a, 8)
    src = dev(a)
    work = torch.empty_like(src)
    ws = torch.empty(rs.workspace_bytes(4, 0, n, 8), dtype=torch.uint8, device="cuda")
    work.copy_(src)
    rs.sort(work, ws=ws)  # warm-up: probe + kernel attributes outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            work.copy_(src)
            rs.sort(work, ws=ws, stream=s)
    for _ in range(3):
        work.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert (host(work, np.uint32) == want).all()


def test_sort_graph_u32_and_pairs():
    """rs.SortGraph: capture once, replay on new contents of the same buffers;
    every replay matches the oracle (u32 at config 1's size, pairs ragged)."""
    n = 1 << 20
    g0 = None
    for seed in (3, 4):
        a = inputs.gen_u32(n, seed)
        if g0 is None:
            buf = dev(a)
            g0 = rs.SortGraph(buf)
            assert g0.launches >= 2
        else:
            buf.copy_(dev(a))
            g0.replay()
        torch.cuda.synchronize()
        assert (host(buf, np.uint32) == oracle.sr(a, 8)).all(), seed
    m = 3 * TILEP + 11
    k1, k2 = inputs.gen_u64(m, 5), inputs.gen_u64(m, 6, "mod1024")
    v = inputs.iota_u32(m)
    tk, tv = dev(k1), dev(v)
    gp = rs.SortGraph(tk, tv)
    tk.copy_(dev(k2))
    tv.copy_(dev(v))
    gp.replay()
    torch.cuda.synchronize()
    wk, wv = oracle.sr(k2, 8, vals=v)
    assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all()


@pytest.mark.parametrize("pdl", [1, 2])
@pytest.mark.parametrize("tiles", [1, 2])
def test_programmatic_dependent_launch_on_and_off(option, pdl, tiles):
    """The radix-256 kernel chain K2 -> K3 x P -> K4 with programmatic dependent
    launches forced on for every key type (pdl 2; by default only u32 keys up to
    2^24) and forced off (pdl 1): bit-exact against the oracle at ragged
    multi-tile sizes, with skipped passes (mod16, equal keys: the active-pass
    parity decides whether K4 copies) and in place / out of place."""
    option("pdl", pdl)
    option("small_tiles", tiles)
    for n in (1, TILE32 - 1, 3 * TILE32 + 5, (1 << 20) + 3, (1 << 22) + 7):
        for dist in ("uniform", "mod16", "equal"):
            a = inputs.gen_u32(n, 211 + n, dist)
            want = oracle.sr(a, 8)
            assert (_sort_u32(a, 8) == want).all(), (n, dist)
            assert (_sort_u32(a, 8, inplace=False) == want).all(), (n, dist)
    for n in (TILEP + 1, (1 << 20) + 5):
        k = inputs.gen_u64(n, 212 + n, "mod1024")
        v = inputs.iota_u32(n)
        tk, tv = dev(k), dev(v)
        rs.sort_pairs(tk, tv)
        wk, wv = oracle.sr(k, 8, vals=v)
        assert (host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all(), n
        t = dev(k)
        rs.sort(t)
        assert (host(t, np.uint64) == wk).all(), n
