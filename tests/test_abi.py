"""C-ABI boundary checks that need no GPU: librsort.so loads, exports every
symbol include/rsort.h and include/rsort_dev.h declare (and nothing else), and
rejects bad arguments before touching the device."""
import ctypes
import subprocess

import pytest

from paper_1808_10292_b200 import _abi
from paper_1808_10292_b200.build import LIB, build

RS_OK, RS_EINVAL, RS_ECAPACITY = 0, 1, 5


@pytest.fixture(scope="module")
def L():
    build()
    return _abi.lib()


def test_exports_every_declared_symbol(L):
    declared = _abi.header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(L, name), name
        assert name in _abi.SIGNATURES, f"binding lacks {name}"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared) <= exported
    assert {s for s in exported if s.startswith("rs_")} == set(declared)


def test_version_and_status_strings(L):
    assert b"sm_100a" in L.rs_version()
    assert L.rs_status_string(RS_EINVAL) == b"RS_EINVAL"
    assert L.rs_status_string(RS_ECAPACITY) == b"RS_ECAPACITY"


def test_workspace_sizing(L):
    assert L.rs_workspace_bytes(4, 0, 0, 8, None) > 0
    w8 = L.rs_workspace_bytes(4, 0, 1 << 20, 8, None)
    assert w8 >= (1 << 20) * 4          # at least the ping-pong buffer
    assert L.rs_workspace_bytes(8, 4, 1 << 20, 8, None) >= (1 << 20) * 12
    assert L.rs_workspace_bytes(4, 0, 1 << 20, 16, None) >= (1 << 20) * 4
    assert L.rs_workspace_bytes(4, 0, 100, 7, None) == 0
    assert L.rs_workspace_bytes(3, 0, 100, 8, None) == 0
    assert L.rs_workspace_bytes(4, 2, 100, 8, None) == 0
    assert L.rs_output_capacity(12345, None) == 12345


def _sort_u32(L, keys, n, b, out, cap, ws, wsb):
    n_out = ctypes.c_size_t(0)
    return L.rs_sort_u32(keys, n, b, None, out, cap, ctypes.byref(n_out), ws, wsb, None)


def test_validation_before_any_launch(L):
    fake = 0x10000  # never dereferenced: validation fails first
    wsb = L.rs_workspace_bytes(4, 0, 1000, 8, None)
    assert _sort_u32(L, fake, 1000, 7, fake, 1000, fake, wsb) == RS_EINVAL
    assert b"digit_bits" in L.rs_last_error()
    assert _sort_u32(L, None, 1000, 8, fake, 1000, fake, wsb) == RS_EINVAL
    assert _sort_u32(L, fake + 4, 1000, 8, fake, 1000, fake, wsb) == RS_EINVAL      # misaligned
    assert b"aligned" in L.rs_last_error()
    assert _sort_u32(L, fake, 1000, 8, fake, 1000, fake, wsb - 1) == RS_EINVAL      # ws too small
    assert _sort_u32(L, fake, 1 << 32, 8, fake, 1 << 32, fake, 1 << 40) == RS_EINVAL
    assert _sort_u32(L, fake, 1000, 8, fake, 999, fake, wsb) == RS_ECAPACITY
    assert _sort_u32(L, None, 0, 8, None, 0, None, 0) == RS_OK                       # n = 0 no-op
    n_out = ctypes.c_size_t(0)
    assert L.rs_sort_pairs_u64_u32(fake, None, 10, 8, None, fake, fake, 10, ctypes.byref(n_out), fake,
                                   1 << 30, None) == RS_EINVAL
    assert L.rs_sort_bits(4, fake, None, 10, 8, 33, fake, None, fake, 1 << 30, None) == RS_EINVAL
    assert L.rs_sort_bits(4, fake, None, 10, 8, 0, fake, None, fake, 1 << 30, None) == RS_EINVAL


def test_comm_argument_validation(L):
    h = ctypes.c_void_p()
    assert L.rs_comm_create(None, 2, 0, 0, ctypes.byref(h)) == RS_EINVAL
    uid = (ctypes.c_char * 128)()
    assert L.rs_comm_create(uid, 2, 2, 0, ctypes.byref(h)) == RS_EINVAL
    assert L.rs_comm_destroy(None) == RS_OK
    assert L.rs_comm_rank(None) == 0 and L.rs_comm_size(None) == 1
    assert L.rs_comm_set_oversampling(None, 8) == RS_EINVAL


def test_product_header_is_the_scope_table(L):
    """include/rsort.h carries exactly SURVEY §8(b)'s calls and the comm helpers;
    test / tuning surface lives in include/rsort_dev.h."""
    prod = set(_abi.header_symbols("rsort.h"))
    assert prod == {"rs_status_string", "rs_last_error", "rs_version", "rs_workspace_bytes", "rs_output_capacity",
                    "rs_sort_u32", "rs_sort_u64", "rs_sort_pairs_u64_u32", "rs_sort_bits", "rs_digit_histogram",
                    "rs_get_unique_id", "rs_comm_create", "rs_comm_destroy", "rs_comm_set_oversampling",
                    "rs_comm_set_sampling", "rs_comm_rank", "rs_comm_size"}
    dev = set(_abi.header_symbols("rsort_dev.h"))
    assert not prod & dev
    assert {"rs_local_group_create", "rs_comm_create_local", "rs_dev_set_option", "rs_ipc_open"} <= dev


def test_local_group_validation(L):
    g = ctypes.c_void_p()
    assert L.rs_local_group_create(0, ctypes.byref(g)) == RS_EINVAL
    assert L.rs_local_group_create(65, ctypes.byref(g)) == RS_EINVAL
    assert L.rs_local_group_create(2, None) == RS_EINVAL
    assert L.rs_local_group_create(2, ctypes.byref(g)) == RS_OK
    c = ctypes.c_void_p()
    assert L.rs_comm_create_local(g, 2, ctypes.byref(c)) == RS_EINVAL      # rank out of range
    assert L.rs_comm_create_local(g, -1, ctypes.byref(c)) == RS_EINVAL
    assert L.rs_comm_create_local(None, 0, ctypes.byref(c)) == RS_EINVAL
    assert L.rs_local_group_destroy(g) == RS_OK
    assert L.rs_comm_last_host_syncs(None) == -1
    assert L.rs_comm_set_timeout(None, 10) == RS_EINVAL


def test_dev_options_validation(L):
    v = ctypes.c_longlong()
    assert L.rs_dev_get_option(b"pass_design", ctypes.byref(v)) == RS_OK and v.value == 5
    assert L.rs_dev_set_option(b"pass_design", 3) == RS_EINVAL               # designs 5 and 2 only
    assert L.rs_dev_set_option(b"rank_variant", 1) == RS_EINVAL              # removed knobs
    assert L.rs_dev_set_option(b"gsd_merge", 4) == RS_EINVAL
    assert L.rs_dev_set_option(b"self_check", 1) == RS_OK
    assert L.rs_dev_set_option(b"self_check", 0) == RS_OK
    assert L.rs_dev_get_option(b"nope", ctypes.byref(v)) == RS_EINVAL


def test_net_host_logic(L):
    """BTN / OET stage counts (lg p (lg p + 1)/2; OET p rounds)
    and argument validation, all before any device work."""
    for m in range(7):
        assert L.rs_net_stages(4, 1 << m) == m * (m + 1) // 2
    assert L.rs_net_stages(4, 12) == -1 and L.rs_net_stages(6, 4) == -1
    assert [L.rs_net_stages(5, p) for p in (1, 2, 9)] == [1, 2, 9]
    q, kl = ctypes.c_int(), ctypes.c_int()
    assert L.rs_net_schedule(4, 3, 0, 0, ctypes.byref(q), ctypes.byref(kl)) == -1   # BTN needs a power of 2
    assert L.rs_net_schedule(5, 3, 0, 3, ctypes.byref(q), ctypes.byref(kl)) == -1   # rank out of range


def test_timing_api_without_gpu(L):
    L.rs_timing_reset()
    ms = ctypes.c_double(-1)
    cnt = ctypes.c_int(-1)
    assert L.rs_timing_query(b"", ctypes.byref(ms), ctypes.byref(cnt)) == RS_OK
    assert cnt.value == 0 and ms.value == 0.0
    assert L.rs_launch_count() == 0


@pytest.mark.parametrize("mode,name,ps", [(4, "btn", [1, 2, 4, 8, 16]), (5, "oet", [1, 2, 3, 5, 8])])
def test_net_schedule_drives_the_oracle_network(L, mode, name, ps):
    """The library's BTN / OET schedule (host logic of net.cu, the one the GPU
    stages follow) replayed on tiny blocks in Python reproduces the independent C
    oracle (oracle/net.c) stage by stage, and pairs are symmetric."""
    import numpy as np
    import oracle
    rng = np.random.default_rng(mode)
    for p in ps:
        blocks = [np.sort(rng.integers(0, 20, 3).astype(np.uint32)) for _ in range(p)]
        cur = [b.copy() for b in blocks]
        stages = L.rs_net_stages(mode, p)
        for t in range(stages):
            nxt = [None] * p
            for r in range(p):
                q, kl = ctypes.c_int(), ctypes.c_int()
                assert L.rs_net_schedule(mode, p, t, r, ctypes.byref(q), ctypes.byref(kl)) == 0
                if q.value < 0:
                    nxt[r] = cur[r]
                    continue
                q2, kl2 = ctypes.c_int(), ctypes.c_int()
                assert L.rs_net_schedule(mode, p, t, q.value, ctypes.byref(q2), ctypes.byref(kl2)) == 0
                assert q2.value == r and kl2.value == 1 - kl.value
                lo, hi = (r, q.value) if r < q.value else (q.value, r)
                merged = np.concatenate([cur[lo], cur[hi]])
                merged = merged[np.argsort(merged, kind="stable")]
                nxt[r] = merged[:3] if kl.value else merged[3:]
            cur = nxt
            want = getattr(oracle, name)(blocks, max_stages=t + 1)
            assert [c.tolist() for c in cur] == [w.tolist() for w in want["Y"]], (p, t)
        q, kl = ctypes.c_int(), ctypes.c_int()
        assert L.rs_net_schedule(mode, p, stages, 0, ctypes.byref(q), ctypes.byref(kl)) == -1
