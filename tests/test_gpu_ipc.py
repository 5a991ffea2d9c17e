"""CUDA IPC plumbing of the GSD pull merge (rs_ipc_export / rs_ipc_open,
ipc.cu): a child process maps a buffer of this process — a torch sub-allocation
at a non-zero offset, as the GSD blocks are — and reads it back exactly.  The
merge itself over mapped peer blocks is checked by the pull-merge emulation
(test_gpu_gsd.py, gsd_merge = 2)."""
import ctypes
import multiprocessing as mp

import numpy as np
import pytest
import torch

import inputs
import paper_1808_10292_b200 as rs

pytestmark = pytest.mark.gpu


def _child(handle: bytes, offset: int, n: int, q):
    try:
        import torch as t
        t.cuda.set_device(0)
        t.cuda.init()
        L = rs.lib()
        h = (ctypes.c_char * 64).from_buffer_copy(handle)
        ptr = ctypes.c_void_p()
        st = L.rs_ipc_open(h, offset, ctypes.byref(ptr))
        if st != 0:
            q.put(("open failed", L.rs_last_error().decode()))
            return
        host = np.empty(n, dtype=np.uint32)
        cudart = ctypes.CDLL("libcudart.so.12")
        cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        e = cudart.cudaMemcpy(host.ctypes.data, ptr, n * 4, 2)  # device -> host
        q.put(("ok", host.tobytes()) if e == 0 else ("memcpy failed", e))
        L.rs_ipc_close_all()
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put(("exception", repr(ex)))


def test_ipc_export_open_roundtrip_with_offset():
    n = 100003
    want = inputs.gen_u32(n, 77)
    big = torch.zeros(3 * n + 1000, dtype=torch.int32, device="cuda")
    view = big[777:777 + n]                       # sub-allocation at an offset
    view.copy_(torch.from_numpy(want.view(np.int32)))
    torch.cuda.synchronize()
    L = rs.lib()
    h = (ctypes.c_char * 64)()
    off = ctypes.c_uint64()
    assert L.rs_ipc_export(ctypes.c_void_p(view.data_ptr()), h, ctypes.byref(off)) == 0
    assert off.value >= 777 * 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_child, args=(bytes(h), off.value, n, q))
    p.start()
    status, payload = q.get(timeout=240)
    p.join(timeout=60)
    assert status == "ok", payload
    assert (np.frombuffer(payload, dtype=np.uint32) == want).all()
