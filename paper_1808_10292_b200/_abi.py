"""ctypes binding of librsort.so: the C-ABI entry points of include/rsort.h under
the same names.  Argument marshalling only — every step of the sort runs in the
library's CUDA kernels.  Loading fails loudly if the library is missing."""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RS_LIB_PATH", os.path.join(HERE, "librsort.so"))
HEADERS = [os.path.join(os.path.dirname(HERE), "include", h) for h in ("rsort.h", "rsort_dev.h")]

RS_OK, RS_EINVAL, RS_ECUDA, RS_ENCCL, RS_ENOMEM, RS_ECAPACITY = range(6)

_vp, _sz, _i32, _u64p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)
_szp = ctypes.POINTER(ctypes.c_size_t)
_vpp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes)
SIGNATURES = {
    # include/rsort.h
    "rs_status_string": (ctypes.c_char_p, [_i32]),
    "rs_last_error": (ctypes.c_char_p, []),
    "rs_version": (ctypes.c_char_p, []),
    "rs_workspace_bytes": (_sz, [_i32, _i32, _sz, _i32, _vp]),
    "rs_output_capacity": (_sz, [_sz, _vp]),
    "rs_sort_u32": (_i32, [_vp, _sz, _i32, _vp, _vp, _sz, _szp, _vp, _sz, _vp]),
    "rs_sort_u64": (_i32, [_vp, _sz, _i32, _vp, _vp, _sz, _szp, _vp, _sz, _vp]),
    "rs_sort_pairs_u64_u32": (_i32, [_vp, _vp, _sz, _i32, _vp, _vp, _vp, _sz, _szp, _vp, _sz, _vp]),
    "rs_sort_bits": (_i32, [_i32, _vp, _vp, _sz, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "rs_digit_histogram": (_i32, [_i32, _vp, _sz, _i32, _vp, _vp, _sz, _vp]),
    "rs_get_unique_id": (_i32, [_vp]),
    "rs_comm_create": (_i32, [_vp, _i32, _i32, _i32, _vpp]),
    "rs_comm_destroy": (_i32, [_vp]),
    "rs_comm_set_oversampling": (_i32, [_vp, _i32]),
    "rs_comm_set_sampling": (_i32, [_vp, _i32, _sz, ctypes.c_uint64]),
    "rs_comm_rank": (_i32, [_vp]),
    "rs_comm_size": (_i32, [_vp]),
    # include/rsort_dev.h
    "rs_local_group_create": (_i32, [_i32, _vpp]),
    "rs_local_group_destroy": (_i32, [_vp]),
    "rs_comm_create_local": (_i32, [_vp, _i32, _vpp]),
    "rs_comm_last_counts": (_i32, [_vp, _u64p]),
    "rs_comm_last_splitters": (_i32, [_vp, _u64p]),
    "rs_comm_last_host_syncs": (_i32, [_vp]),
    "rs_comm_set_timeout": (_i32, [_vp, _i32]),
    "rs_gsd_exchange_plan": (_i32, [_i32, _i32, _u64p, _u64p, _u64p, _u64p, _u64p]),
    "rs_net_stages": (_i32, [_i32, _i32]),
    "rs_net_schedule": (_i32, [_i32, _i32, _i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "rs_ger_default_s": (_sz, [ctypes.c_uint64]),
    "rs_ger_capacity": (_sz, [_sz, _i32, _sz]),
    "rs_ipc_export": (_i32, [_vp, _vp, _u64p]),
    "rs_ipc_open": (_i32, [_vp, ctypes.c_uint64, _vpp]),
    "rs_ipc_close_all": (_i32, []),
    "rs_dev_set_option": (_i32, [ctypes.c_char_p, ctypes.c_longlong]),
    "rs_dev_get_option": (_i32, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_longlong)]),
    "rs_timing_enable": (None, [_i32]),
    "rs_timing_reset": (None, []),
    "rs_timing_query": (_i32, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32)]),
    "rs_launch_count": (ctypes.c_longlong, []),
}

_lib = None


def header_symbols(which: str | None = None) -> list[str]:
    """Every function name include/rsort.h and include/rsort_dev.h declare (or one of them)."""
    names = set()
    for path in HEADERS:
        if which is not None and os.path.basename(path) != which:
            continue
        src = re.sub(r"/\*.*?\*/", "", open(path).read(), flags=re.S)
        names |= set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1808_10292_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def __getattr__(name):
    if name in SIGNATURES:
        return getattr(lib(), name)
    raise AttributeError(name)


class RSortError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib().rs_last_error().decode()
        super().__init__(f"{where}: {lib().rs_status_string(status).decode()}: {msg}")


def check(status: int, where: str) -> None:
    if status != RS_OK:
        raise RSortError(status, where)
