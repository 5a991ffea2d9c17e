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

__all__ = ["sort", "sort_pairs", "sort_bits", "digit_histogram", "workspace_bytes", "Comm", "LocalGroup",
           "sort_ranks", "net_stages", "set_option", "get_option",
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
        # with a comm: sized for the largest block, and for out_cap if the caller's is larger
        wn = max(comm.ws_n(n), cap) if comm else n
        ws = _workspace(lib().rs_workspace_bytes(kb, 0, wn, digit_bits, h), keys.device)
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
        wn = max(comm.ws_n(n), cap) if comm else n
        ws = _workspace(lib().rs_workspace_bytes(8, 4, wn, digit_bits, h), keys.device)
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


class SortGraph:
    """One single-GPU sort of fixed buffers, captured once in a CUDA graph and
    replayed: for small inputs (config 1) the host launch cost of the ~6 kernels
    per sort disappears.  The sort is stream-ordered with no host synchronisation
    (after the one-time per-device probe), which is what makes it capturable.

    The constructor sorts `keys` (and `vals`) once outside the capture — kernel
    attributes and the device probe are set up there — then captures the same
    call; replay() re-sorts whatever the buffers hold, on the current stream."""

    def __init__(self, keys: torch.Tensor, vals: torch.Tensor | None = None, digit_bits: int = 8):
        self.keys, self.vals, self.digit_bits = keys, vals, digit_bits
        kb = _KEY_BYTES[keys.dtype]
        self.ws = _workspace(lib().rs_workspace_bytes(kb, 4 if vals is not None else 0, keys.numel(), digit_bits,
                                                      None), keys.device)
        self._call(torch.cuda.current_stream(keys.device))
        torch.cuda.synchronize(keys.device)
        c0 = lib().rs_launch_count()
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=keys.device)
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                self._call(s)
        self.launches = lib().rs_launch_count() - c0  # kernels per replay

    def _call(self, stream):
        if self.vals is None:
            sort(self.keys, self.digit_bits, ws=self.ws, stream=stream)
        else:
            sort_pairs(self.keys, self.vals, self.digit_bits, ws=self.ws, stream=stream)

    def replay(self):
        self.graph.replay()


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
    """Collective-sort communicator.  Default: an NCCL comm owned by librsort,
    bootstrapped over a torch.distributed process group (only the 128-byte
    unique id travels).  Comm.local(group, rank) instead joins an in-process
    LocalGroup (p threads on one GPU, include/rsort_dev.h)."""

    def __init__(self, group=None, device: int | None = None, oversampling: int = 8, *, _handle=None,
                 _rank=None, _size=None, _local=None):
        if _handle is not None:  # Comm.local
            self.handle, self.rank, self.size, self._local, self._group = _handle, _rank, _size, _local, None
            self.device = torch.cuda.current_device()
        else:
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
            self._group = group
            self._local = None
        self.sampling = "gsd"
        if oversampling is not None:
            self.set_oversampling(min(oversampling, max(1, 8192 // (self.size * self.size))))

    @classmethod
    def local(cls, group: "LocalGroup", rank: int, oversampling: int = 8) -> "Comm":
        """Rank `rank` of an in-process group; call from that rank's thread (collective)."""
        h = ctypes.c_void_p()
        check(lib().rs_comm_create_local(group.handle, rank, ctypes.byref(h)), "rs_comm_create_local")
        return cls(oversampling=oversampling, _handle=h, _rank=rank, _size=group.p, _local=group)

    def set_oversampling(self, r: int):
        """Collective: every rank with the same r."""
        check(lib().rs_comm_set_oversampling(self.handle, r), "rs_comm_set_oversampling")
        self.r = r

    def set_sampling(self, mode: str = "gsd", s: int = 0, seed: int = 0):
        """Collective.  "gsd" (regular oversampling, default), "ger" (random
        oversampling with s samples per rank, s = 0 the paper's choice, SplitMix64
        seed), "gvr" (the same sample, split before sorting), "pr4" (PR4 routing
        across GPUs), "btn" / "oet" (the bitonic / odd-even transposition
        merge-split networks over equal sorted blocks)."""
        m = {"gsd": 0, "ger": 1, "gvr": 2, "pr4": 3, "btn": 4, "oet": 5}[mode]
        check(lib().rs_comm_set_sampling(self.handle, m, s, seed), "rs_comm_set_sampling")
        self.sampling = mode

    def set_timeout(self, ms: int):
        check(lib().rs_comm_set_timeout(self.handle, ms), "rs_comm_set_timeout")

    def last_counts(self):
        """(p, p) uint64 count matrix |X_{k,j}| of the last sort on this communicator."""
        import numpy as np
        c = np.zeros((self.size, self.size), dtype=np.uint64)
        check(lib().rs_comm_last_counts(self.handle, c.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))),
              "rs_comm_last_counts")
        return c

    def last_splitters(self):
        """(p-1, 3) uint64 (key, rank, pos) splitters of the last sample sort."""
        import numpy as np
        sp = np.zeros((max(self.size - 1, 1), 3), dtype=np.uint64)
        check(lib().rs_comm_last_splitters(self.handle, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))),
              "rs_comm_last_splitters")
        return sp[: self.size - 1]

    def last_host_syncs(self) -> int:
        return lib().rs_comm_last_host_syncs(self.handle)

    def capacity(self, n_local: int) -> int:
        return lib().rs_output_capacity(self.ws_n(n_local), self.handle)

    def ws_n(self, n_local: int) -> int:
        if self._local is not None:
            return self._local.allreduce_max(self.rank, n_local)
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


class LocalGroup:
    """p ranks as p threads of this process on the current GPU: the multi-GPU
    collective (rs_sort_* with a comm) run through host barriers and device
    copies (include/rsort_dev.h).  run(fn) calls fn(comm) on p threads, each with
    its own CUDA stream and Comm.local, and returns the p results."""

    def __init__(self, p: int):
        import threading
        self.p = p
        h = ctypes.c_void_p()
        check(lib().rs_local_group_create(p, ctypes.byref(h)), "rs_local_group_create")
        self.handle = h
        self._bar = threading.Barrier(p)
        self._vals = [0] * p

    def allreduce_max(self, rank: int, value: int) -> int:
        self._vals[rank] = value
        self._bar.wait()
        m = max(self._vals)
        self._bar.wait()
        return m

    def run(self, fn, oversampling: int = 8, timeout_ms: int | None = None):
        import threading
        torch.cuda.synchronize()
        dev = torch.cuda.current_device()
        res, err = [None] * self.p, [None] * self.p

        def body(k):
            try:
                torch.cuda.set_device(dev)
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    c = Comm.local(self, k, oversampling)
                    if timeout_ms is not None:
                        c.set_timeout(timeout_ms)
                    try:
                        res[k] = fn(c)
                    finally:
                        st.synchronize()
                        c.close()
            except BaseException as e:  # re-raised on the caller's thread
                err[k] = e
                try:
                    self._bar.abort()
                except Exception:
                    pass

        th = [threading.Thread(target=body, args=(k,)) for k in range(self.p)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return res

    def close(self):
        if self.handle:
            lib().rs_local_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_MODES = ("gsd", "ger", "gvr", "pr4", "btn", "oet")


def sort_ranks(blocks: list[torch.Tensor], mode: str = "gsd", digit_bits: int = 8,
               vals: list[torch.Tensor] | None = None, r: int = 8, s: int = 0, seed: int = 0,
               out_cap: int | None = None, out_caps: list[int] | None = None):
    """The collective sort over p = len(blocks) in-process ranks on this GPU
    (LocalGroup): rank k calls rs_sort_* with block k (used as scratch) through
    its own Comm.  Returns dict(Y, Yv, n_out, counts (p,p), splitters (p-1,3),
    host_syncs, capacity) — the same call a multi-GPU job makes on each rank."""
    import numpy as np
    p = len(blocks)
    g = LocalGroup(p)
    kb = _KEY_BYTES[blocks[0].dtype]

    def rank_fn(c: Comm):
        k = c.rank
        if mode != "gsd":
            c.set_sampling(mode, s, seed)
        x = blocks[k]
        v = vals[k] if vals is not None else None
        cap = out_caps[k] if out_caps is not None else (out_cap if out_cap is not None else c.capacity(x.numel()))
        if v is None:
            y = sort(x, digit_bits, comm=c, out_cap=cap)
            yv = None
        else:
            y, yv = sort_pairs(x, v, digit_bits, comm=c, out_cap=cap)
        torch.cuda.current_stream().synchronize()
        info = dict(Y=y, Yv=yv, host_syncs=c.last_host_syncs(), capacity=cap)
        if mode in ("gsd", "ger", "gvr"):
            info["counts"] = c.last_counts()
            info["splitters"] = c.last_splitters()
        return info

    try:
        out = g.run(rank_fn, oversampling=min(r, max(1, 8192 // (p * p))))
    finally:
        g.close()
    res = dict(Y=[o["Y"] for o in out], Yv=[o["Yv"] for o in out] if vals is not None else None,
               n_out=[int(o["Y"].numel()) for o in out], host_syncs=[o["host_syncs"] for o in out],
               capacity=[o["capacity"] for o in out])
    if mode in ("gsd", "ger", "gvr"):
        res["counts"] = out[0]["counts"]
        res["splitters"] = out[0]["splitters"]
    del kb
    return res


def net_stages(mode: str, p: int) -> int:
    """Stages of BTN (lg p (lg p + 1)/2) or rounds of OET (p) for p ranks."""
    st = lib().rs_net_stages({"btn": 4, "oet": 5}[mode], p)
    if st < 0:
        raise ValueError(f"{mode} is not defined for p = {p}")
    return st


def set_option(name: str, value: int):
    check(lib().rs_dev_set_option(name.encode(), value), "rs_dev_set_option")


def get_option(name: str) -> int:
    v = ctypes.c_longlong()
    check(lib().rs_dev_get_option(name.encode(), ctypes.byref(v)), "rs_dev_get_option")
    return int(v.value)
