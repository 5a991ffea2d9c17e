"""B200-native LSD radix sort (the paper's PR4/PR2 count-sort passes) and GSD
regular-oversampling sample sort across GPUs — Gerbessiotis, "A study of
integer sorting on multicores" (arXiv 1808.10292).

The work happens in librsort.so (hand-written sm_100a CUDA + NCCL) behind the C
ABI of include/rsort.h.  This module only marshals torch tensors (device memory,
the current stream, process groups) into those calls; it never computes on the
CPU and has no fallback.
"""
from __future__ import annotations

import ctypes

import torch

from . import _abi
from ._abi import RSortError, check, lib

__all__ = ["sort", "sort_pairs", "sort_bits", "digit_histogram", "workspace_bytes", "Comm", "gsd_emulate",
           "ger_emulate", "gvr_emulate", "pr_emulate", "net_emulate", "net_stages",
           "RSortError", "lib", "rs_sort_u32", "rs_sort_u64", "rs_sort_pairs_u64_u32"]

_KEY_BYTES = {torch.uint32: 4, torch.int32: 4, torch.uint64: 8, torch.int64: 8}


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _check_tensor(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def workspace_bytes(key_bytes: int, val_bytes: int, n: int, digit_bits: int = 8, comm: "Comm | None" = None) -> int:
    return lib().rs_workspace_bytes(key_bytes, val_bytes, n, digit_bits, comm.handle if comm else None)


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)


# ---- C-ABI names, re-exported -------------------------------------------------
def rs_sort_u32(*a):
    return lib().rs_sort_u32(*a)


def rs_sort_u64(*a):
    return lib().rs_sort_u64(*a)


def rs_sort_pairs_u64_u32(*a):
    return lib().rs_sort_pairs_u64_u32(*a)


# ---- tensor API -----------------------------------------------------------------
def sort(keys: torch.Tensor, digit_bits: int = 8, comm: "Comm | None" = None, out: torch.Tensor | None = None,
         ws: torch.Tensor | None = None, out_cap: int | None = None, stream=None) -> torch.Tensor:
    """Sort a 1-D CUDA tensor of uint32/uint64 keys (unsigned order).

    Single GPU: returns `out` (default: in place in `keys`).  With `comm`, runs
    GSD across ranks and returns this rank's slice Y_j (keys is scratch)."""
    _check_tensor(keys, "keys")
    kb = _KEY_BYTES[keys.dtype]
    n = keys.numel()
    h = comm.handle if comm else None
    if comm is not None:
        cap = out_cap if out_cap is not None else comm.capacity(n)
        if out is None:
            out = torch.empty(max(cap, 1), dtype=keys.dtype, device=keys.device)
        cap = min(cap, out.numel())
    else:
        if out is None:
            out = keys
        cap = out.numel()
    if ws is None:
        ws = _workspace(lib().rs_workspace_bytes(kb, 0, comm.ws_n(n) if comm else n, digit_bits, h), keys.device)
    n_out = ctypes.c_size_t(0)
    fn = lib().rs_sort_u32 if kb == 4 else lib().rs_sort_u64
    check(fn(keys.data_ptr(), n, digit_bits, h, out.data_ptr(), cap, ctypes.byref(n_out), ws.data_ptr(), ws.numel(),
             _stream(stream)), "rs_sort")
    return out[: n_out.value] if comm is not None else out


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor, digit_bits: int = 8, comm: "Comm | None" = None,
               out_keys: torch.Tensor | None = None, out_vals: torch.Tensor | None = None,
               ws: torch.Tensor | None = None, out_cap: int | None = None, stream=None):
    """Stable sort of (uint64 key, uint32 value) pairs; returns (keys, vals)."""
    _check_tensor(keys, "keys")
    _check_tensor(vals, "vals")
    if _KEY_BYTES[keys.dtype] != 8 or vals.element_size() != 4 or vals.numel() != keys.numel():
        raise ValueError("sort_pairs expects uint64 keys and 32-bit values of equal length")
    n = keys.numel()
    h = comm.handle if comm else None
    if comm is not None:
        cap = out_cap if out_cap is not None else comm.capacity(n)
        out_keys = out_keys if out_keys is not None else torch.empty(max(cap, 1), dtype=keys.dtype, device=keys.device)
        out_vals = out_vals if out_vals is not None else torch.empty(max(cap, 1), dtype=vals.dtype, device=vals.device)
        cap = min(cap, out_keys.numel(), out_vals.numel())
    else:
        out_keys = keys if out_keys is None else out_keys
        out_vals = vals if out_vals is None else out_vals
        cap = out_keys.numel()
    if ws is None:
        ws = _workspace(lib().rs_workspace_bytes(8, 4, comm.ws_n(n) if comm else n, digit_bits, h), keys.device)
    n_out = ctypes.c_size_t(0)
    check(lib().rs_sort_pairs_u64_u32(keys.data_ptr(), vals.data_ptr(), n, digit_bits, h, out_keys.data_ptr(),
                                      out_vals.data_ptr(), cap, ctypes.byref(n_out), ws.data_ptr(), ws.numel(),
                                      _stream(stream)), "rs_sort_pairs_u64_u32")
    if comm is not None:
        return out_keys[: n_out.value], out_vals[: n_out.value]
    return out_keys, out_vals


def sort_bits(keys: torch.Tensor, end_bit: int, digit_bits: int = 8, vals: torch.Tensor | None = None,
              out_keys: torch.Tensor | None = None, out_vals: torch.Tensor | None = None,
              ws: torch.Tensor | None = None, stream=None):
    """Stable sort by the low `end_bit` bits (passes 0..ceil(end_bit/b)-1)."""
    _check_tensor(keys, "keys")
    kb = _KEY_BYTES[keys.dtype]
    n = keys.numel()
    out_keys = torch.empty_like(keys) if out_keys is None else out_keys
    if vals is not None and out_vals is None:
        out_vals = torch.empty_like(vals)
    if ws is None:
        ws = _workspace(lib().rs_workspace_bytes(kb, 4 if vals is not None else 0, n, digit_bits, None), keys.device)
    check(lib().rs_sort_bits(kb, keys.data_ptr(), _ptr(vals), n, digit_bits, end_bit, out_keys.data_ptr(),
                             _ptr(out_vals), ws.data_ptr(), ws.numel(), _stream(stream)), "rs_sort_bits")
    return (out_keys, out_vals) if vals is not None else out_keys


def digit_histogram(keys: torch.Tensor, digit_bits: int = 8, stream=None) -> torch.Tensor:
    """All passes' digit counts from one read: int64-viewable (P, 2^b) uint32 tensor."""
    _check_tensor(keys, "keys")
    kb = _KEY_BYTES[keys.dtype]
    P = kb * 8 // digit_bits
    hist = torch.empty(P * (1 << digit_bits), dtype=torch.int32, device=keys.device)
    ws = _workspace(16, keys.device)
    check(lib().rs_digit_histogram(kb, keys.data_ptr(), keys.numel(), digit_bits, hist.data_ptr(), ws.data_ptr(),
                                   ws.numel(), _stream(stream)), "rs_digit_histogram")
    return hist.view(P, 1 << digit_bits)


def max_over_ranks(n_local: int, group=None) -> int:
    """Largest local n over the process group (sizes the GSD workspace and
    receive capacity; every rank must agree on them)."""
    import torch.distributed as dist
    t = torch.tensor([n_local], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def exchange_plan(counts, rank: int, caps=None):
    """rs_gsd_exchange_plan on a (p, p) count matrix: (send_off, recv_off, total)."""
    import numpy as np
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    p = c.shape[0]
    so = np.zeros(p + 1, dtype=np.uint64)
    ro = np.zeros(p + 1, dtype=np.uint64)
    tot = np.zeros(1, dtype=np.uint64)
    cp = None
    if caps is not None:
        caps = np.ascontiguousarray(caps, dtype=np.uint64)
        cp = caps.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    u = ctypes.POINTER(ctypes.c_uint64)
    check(lib().rs_gsd_exchange_plan(p, rank, c.ctypes.data_as(u), cp, so.ctypes.data_as(u), ro.ctypes.data_as(u),
                                     tot.ctypes.data_as(u)), "rs_gsd_exchange_plan")
    return so, ro, int(tot[0])


class Comm:
    """GSD communicator: an NCCL comm owned by librsort, bootstrapped over a
    torch.distributed process group (only the 128-byte unique id travels)."""

    def __init__(self, group=None, device: int | None = None, oversampling: int = 8):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else device
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            check(lib().rs_get_unique_id(uid), "rs_get_unique_id")
        obj = [bytes(uid)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        check(lib().rs_comm_create(uid, self.size, self.rank, self.device, ctypes.byref(h)), "rs_comm_create")
        self.handle = h
        self.set_oversampling(oversampling)
        # largest local n over ranks, for workspace / capacity sizing
        self._group = group

    def set_oversampling(self, r: int):
        check(lib().rs_comm_set_oversampling(self.handle, r), "rs_comm_set_oversampling")
        self.r = r

    def set_sampling(self, mode: str = "gsd", s: int = 0, seed: int = 0):
        """"gsd" (regular oversampling, default), "ger" (random oversampling
        with s samples per rank, s = 0 the paper's choice, SplitMix64 seed),
        "gvr" (the same sample, split before sorting), "pr4" (PR4 routing across
        GPUs), "btn" / "oet" (the bitonic / odd-even transposition merge-split
        networks over equal sorted blocks)."""
        m = {"gsd": 0, "ger": 1, "gvr": 2, "pr4": 3, "btn": 4, "oet": 5}[mode]
        check(lib().rs_comm_set_sampling(self.handle, m, s, seed), "rs_comm_set_sampling")
        self.sampling = mode

    def last_counts(self):
        """(p, p) uint64 count matrix |X_{k,j}| of the last sort on this communicator."""
        import numpy as np
        c = np.zeros((self.size, self.size), dtype=np.uint64)
        check(lib().rs_comm_last_counts(self.handle, c.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))),
              "rs_comm_last_counts")
        return c

    def capacity(self, n_local: int) -> int:
        return lib().rs_output_capacity(self.ws_n(n_local), self.handle)

    def ws_n(self, n_local: int) -> int:
        return max_over_ranks(n_local, self._group)

    def close(self):
        if self.handle:
            lib().rs_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gsd_emulate(blocks: list[torch.Tensor], r: int = 8, digit_bits: int = 8, vals: list[torch.Tensor] | None = None,
                out_cap: int | None = None, stream=None):
    """GSD over p = len(blocks) ranks held on this GPU (see include/rsort.h):
    returns dict(Y, Yv, n_out, splitters (p-1,3) uint64, counts (p,p) uint64)."""
    return _emulate(0, blocks, r, 0, 0, digit_bits, vals, out_cap, stream)


def ger_emulate(blocks: list[torch.Tensor], s: int = 0, seed: int = 0, digit_bits: int = 8,
                vals: list[torch.Tensor] | None = None, out_cap: int | None = None, stream=None):
    """GER (random oversampling) over p = len(blocks) ranks on
    this GPU; s = 0 selects the paper's s.  Same result dict as gsd_emulate."""
    return _emulate(1, blocks, 1, s, seed, digit_bits, vals, out_cap, stream)


def pr_emulate(blocks: list[torch.Tensor], vals: list[torch.Tensor] | None = None, stream=None):
    """PR4 across p = len(blocks) ranks held on this GPU (per-digit local round,
    count exchange, pull of each rank's global-rank range): returns dict(Y, Yv)
    with |Y_j| = |blocks[j]|.  The blocks are scratch."""
    p = len(blocks)
    kb = _KEY_BYTES[blocks[0].dtype]
    n = [b.numel() for b in blocks]
    dev = blocks[0].device
    outs = [torch.empty(max(x, 1), dtype=blocks[0].dtype, device=dev) for x in n]
    vouts = [torch.empty(max(x, 1), dtype=torch.int32, device=dev) for x in n] if vals is not None else None
    ws = _workspace(lib().rs_pr_emulate_ws_bytes(kb, 4 if vals is not None else 0, p, max(n) if n else 0), dev)
    arr = ctypes.c_void_p * p
    check(lib().rs_pr_emulate(kb, p, arr(*[b.data_ptr() for b in blocks]),
                              arr(*[v.data_ptr() for v in vals]) if vals is not None else None,
                              (ctypes.c_size_t * p)(*n), arr(*[o.data_ptr() for o in outs]),
                              arr(*[o.data_ptr() for o in vouts]) if vals is not None else None,
                              ws.data_ptr(), ws.numel(), _stream(stream)), "rs_pr_emulate")
    return dict(Y=[outs[j][: n[j]] for j in range(p)],
                Yv=[vouts[j][: n[j]] for j in range(p)] if vals is not None else None)


def net_stages(mode: str, p: int) -> int:
    """Stages of BTN (lg p (lg p + 1)/2) or rounds of OET (p) for p ranks."""
    st = lib().rs_net_stages({"btn": 4, "oet": 5}[mode], p)
    if st < 0:
        raise ValueError(f"{mode} is not defined for p = {p}")
    return st


def net_emulate(mode: str, blocks: list[torch.Tensor], digit_bits: int = 8,
                vals: list[torch.Tensor] | None = None, stream=None):
    """BTN ("btn") or OET ("oet") over p = len(blocks) ranks held on this GPU:
    local radix sort of every block, then the merge-split network.
    Blocks must have equal sizes; they are read only.  Returns dict(Y, Yv)."""
    p = len(blocks)
    kb = _KEY_BYTES[blocks[0].dtype]
    N = blocks[0].numel()
    if any(b.numel() != N for b in blocks):
        raise ValueError("BTN/OET need equal block sizes")
    dev = blocks[0].device
    outs = [torch.empty(max(N, 1), dtype=blocks[0].dtype, device=dev) for _ in range(p)]
    vouts = [torch.empty(max(N, 1), dtype=torch.int32, device=dev) for _ in range(p)] if vals is not None else None
    vb = 4 if vals is not None else 0
    ws = _workspace(lib().rs_net_emulate_ws_bytes(kb, vb, p, digit_bits, N), dev)
    arr = ctypes.c_void_p * p
    check(lib().rs_net_emulate({"btn": 4, "oet": 5}[mode], kb, p, digit_bits, arr(*[b.data_ptr() for b in blocks]),
                               arr(*[v.data_ptr() for v in vals]) if vals is not None else None, N,
                               arr(*[o.data_ptr() for o in outs]),
                               arr(*[o.data_ptr() for o in vouts]) if vals is not None else None,
                               ws.data_ptr(), ws.numel(), _stream(stream)), "rs_net_emulate")
    return dict(Y=[o[:N] for o in outs], Yv=[o[:N] for o in vouts] if vals is not None else None)


def gvr_emulate(blocks: list[torch.Tensor], s: int = 0, seed: int = 0, digit_bits: int = 8,
                vals: list[torch.Tensor] | None = None, out_cap: int | None = None, stream=None):
    """GVR (split, exchange, then sort) over p = len(blocks)
    ranks on this GPU; the blocks are used as scratch.  Same result dict."""
    return _emulate(2, blocks, 1, s, seed, digit_bits, vals, out_cap, stream)


def _emulate(mode, blocks, r, s, seed, digit_bits, vals, out_cap, stream):
    import numpy as np
    p = len(blocks)
    kb = _KEY_BYTES[blocks[0].dtype]
    n = [b.numel() for b in blocks]
    nmax = max(n) if n else 0
    if out_cap is not None:
        cap = out_cap
    elif mode == 0:
        cap = nmax + nmax // r + p
    else:
        cap = lib().rs_ger_capacity(nmax, p, s)
    dev = blocks[0].device
    outs = [torch.empty(max(cap, 1), dtype=blocks[0].dtype, device=dev) for _ in range(p)]
    vouts = [torch.empty(max(cap, 1), dtype=torch.int32, device=dev) for _ in range(p)] if vals is not None else None
    vb = 4 if vals is not None else 0
    wsb = (lib().rs_gsd_emulate_ws_bytes(kb, vb, p, r, digit_bits, nmax, cap) if mode == 0
           else (lib().rs_ger_emulate_ws_bytes if mode == 1 else lib().rs_gvr_emulate_ws_bytes)(
               kb, vb, p, s, digit_bits, nmax, cap))
    ws = _workspace(wsb, dev)
    arr = ctypes.c_void_p * p
    n_arr = (ctypes.c_size_t * p)(*n)
    n_out = (ctypes.c_size_t * p)()
    spl = np.zeros((max(p - 1, 1), 3), dtype=np.uint64)
    counts = np.zeros((p, p), dtype=np.uint64)
    head = (kb, p, r) if mode == 0 else (kb, p, s, seed)
    fn = [lib().rs_gsd_emulate, lib().rs_ger_emulate, lib().rs_gvr_emulate][mode]
    check(fn(*head, digit_bits, arr(*[b.data_ptr() for b in blocks]),
             arr(*[v.data_ptr() for v in vals]) if vals is not None else None, n_arr,
             arr(*[o.data_ptr() for o in outs]),
             arr(*[o.data_ptr() for o in vouts]) if vals is not None else None, cap, n_out,
             spl.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
             counts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ws.data_ptr(), ws.numel(),
             _stream(stream)), ["rs_gsd_emulate", "rs_ger_emulate", "rs_gvr_emulate"][mode])
    return dict(Y=[outs[j][: n_out[j]] for j in range(p)],
                Yv=[vouts[j][: n_out[j]] for j in range(p)] if vals is not None else None,
                n_out=list(n_out), splitters=spl[: p - 1], counts=counts)
