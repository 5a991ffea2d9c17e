"""The NCCL GSD path (rs_sort_* with a communicator) on one GPU with a 1-rank
NCCL communicator bootstrapped over a torch.distributed process group: header
all-gather, local sort, sample/splitters/split, count all-gather, the
(self-)exchange and the merge all run through the multi-GPU code."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import inputs
import oracle
import paper_1808_10292_b200 as rs
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    c = rs.Comm(oversampling=8)
    yield c
    c.close()
    dist.destroy_process_group()


def test_comm_bootstrap(comm):
    assert rs.lib().rs_comm_rank(comm.handle) == 0 and rs.lib().rs_comm_size(comm.handle) == 1
    assert comm.capacity(1000) == 1000 + 1000 // 8 + 1


@pytest.mark.parametrize("n", [0, 1, 4097, 100003])
def test_gsd_p1_u32(comm, n):
    a = inputs.gen_u32(n, 50 + n)
    t = dev(a) if n else torch.empty(0, dtype=torch.int32, device="cuda")
    y = rs.sort(t, comm=comm)
    assert y.numel() == n
    if n:
        assert (host(y, np.uint32) == oracle.sr(a, 8)).all()


@pytest.mark.parametrize("b", [8, 16])
def test_gsd_p1_pairs_and_u64(comm, b):
    n = 50001
    k = inputs.gen_u64(n, 60, "mod1024")
    v = inputs.iota_u32(n)
    yk, yv = rs.sort_pairs(dev(k), dev(v), digit_bits=b, comm=comm)
    wk, wv = oracle.sr(k, b, vals=v)
    assert (host(yk, np.uint64) == wk).all() and (host(yv, np.uint32) == wv).all()
    y = rs.sort(dev(k), digit_bits=b, comm=comm)
    assert (host(y, np.uint64) == np.sort(k)).all()


def test_gsd_capacity_error(comm):
    a = inputs.gen_u32(1000, 61)
    with pytest.raises(rs.RSortError) as e:
        rs.sort(dev(a), comm=comm, out_cap=999)
    assert e.value.status == 5


def test_ger_p1_through_nccl(comm):
    """GER sampling selected on the communicator (header-checked); at p = 1 there
    are no splitters, so the call is the local sort through the NCCL path."""
    comm.set_sampling("ger", s=0, seed=3)
    try:
        a = inputs.gen_u32(70001, 62)
        y = rs.sort(dev(a), comm=comm)
        assert (host(y, np.uint32) == oracle.sr(a, 8)).all()
    finally:
        comm.set_sampling("gsd")


def test_gvr_p1_through_nccl(comm):
    comm.set_sampling("gvr", s=0, seed=4)
    try:
        k = inputs.gen_u64(40001, 63, "mod1024")
        v = inputs.iota_u32(k.size)
        yk, yv = rs.sort_pairs(dev(k), dev(v), comm=comm)
        wk, wv = oracle.sr(k, 8, vals=v)
        assert (host(yk, np.uint64) == wk).all() and (host(yv, np.uint32) == wv).all()
    finally:
        comm.set_sampling("gsd")


def test_last_counts_after_a_sort(comm):
    a = inputs.gen_u32(12345, 64)
    rs.sort(dev(a), comm=comm)
    assert comm.last_counts().tolist() == [[12345]]


def test_collective_validation_errors(comm):
    """Bad arguments on a collective call are agreed on in the header exchange
    (every rank returns RS_EINVAL; a rank never returns early and leaves the
    others waiting): too-small workspace, bad digit width, NULL keys."""
    L = rs.lib()
    a = dev(inputs.gen_u32(5000, 65))
    out = torch.empty(6000, dtype=torch.int32, device="cuda")
    ws = torch.empty(4096, dtype=torch.uint8, device="cuda")
    n_out = ctypes.c_size_t()
    s = torch.cuda.current_stream().cuda_stream
    assert L.rs_sort_u32(a.data_ptr(), a.numel(), 8, comm.handle, out.data_ptr(), 6000, ctypes.byref(n_out),
                         ws.data_ptr(), ws.numel(), s) == 1
    assert b"too small" in L.rs_last_error()
    big = torch.empty(L.rs_workspace_bytes(4, 0, 5000, 8, comm.handle), dtype=torch.uint8, device="cuda")
    assert L.rs_sort_u32(a.data_ptr(), a.numel(), 7, comm.handle, out.data_ptr(), 6000, ctypes.byref(n_out),
                         big.data_ptr(), big.numel(), s) == 1
    assert L.rs_sort_u32(None, 5000, 8, comm.handle, out.data_ptr(), 6000, ctypes.byref(n_out),
                         big.data_ptr(), big.numel(), s) == 1
    # the communicator still works afterwards
    y = rs.sort(a, comm=comm)
    assert (host(y, np.uint32) == np.sort(host(a, np.uint32))).all()


def test_pr4_p1_through_nccl(comm):
    """PR4 routing selected on the communicator: at p = 1 every round pulls the
    whole locally sorted block from itself (no IPC mapping needed)."""
    comm.set_sampling("pr4")
    try:
        k = inputs.gen_u64(30001, 66, "mod1024")
        v = inputs.iota_u32(k.size)
        yk, yv = rs.sort_pairs(dev(k), dev(v), comm=comm)
        wk, wv = oracle.sr(k, 8, vals=v)
        assert (host(yk, np.uint64) == wk).all() and (host(yv, np.uint32) == wv).all()
        a = inputs.gen_u32(50001, 67)
        y = rs.sort(dev(a), comm=comm)
        assert (host(y, np.uint32) == oracle.sr(a, 8)).all()
    finally:
        comm.set_sampling("gsd")


@pytest.mark.parametrize("mode", ["btn", "oet"])
def test_net_sorts_p1_through_nccl(comm, mode):
    """BTN / OET selected on the communicator (header validation, workspace and
    capacity sizing through the collective path); at p = 1 the network has no
    exchange and the result is the local sort."""
    comm.set_sampling(mode)
    try:
        k = inputs.gen_u64(30001, 68, "mod1024")
        v = inputs.iota_u32(k.size)
        yk, yv = rs.sort_pairs(dev(k), dev(v), comm=comm)
        wk, wv = oracle.sr(k, 8, vals=v)
        assert (host(yk, np.uint64) == wk).all() and (host(yv, np.uint32) == wv).all()
        a = inputs.gen_u32(50001, 69)
        y = rs.sort(dev(a), comm=comm, digit_bits=16)
        assert (host(y, np.uint32) == oracle.sr(a, 16)).all()
    finally:
        comm.set_sampling("gsd")
