"""Seeded synthetic inputs (SplitMix64 counter stream) shared by oracle and GPU path.

Holds none of the sorting method's arithmetic; see inputs/gen.c for the recipe
and DESIGN.md "Input recipe" for how each BASELINE.json config maps onto it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB_PATH = os.path.join(_HERE, "libinputs.so")
_lib = None

# distribution names -> codes of inputs/gen.c
U32_DISTS = {
    "uniform": 0,    # (u32)(z>>32)                cfg 1, 3(i), 4
    "mod16": 1,      # (z>>32) & 15                cfg 3(ii)
    "gauss": 2,      # rounded |N(2^31, 2^28^2)|   cfg 3(iii)
    "sorted": 3,     # stratified ascending        cfg 3(iv)
    "reversed": 4,   # stratified descending       cfg 3(v)
    "equal": 5,      # all = (u32)(z_0>>32)        cfg 3(vi)
    "half": 6,       # (u32)(z>>33) in [0,2^31)    cfg 2
}
U64_DISTS = {"uniform": 0, "mod1024": 1}


def build(force: bool = False) -> str:
    """Compile inputs/gen.c into inputs/libinputs.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.inp_splitmix64_at.argtypes = [u64, u64]
        L.inp_splitmix64_at.restype = u64
        L.inp_splitmix64_mix.argtypes = [u64]
        L.inp_splitmix64_mix.restype = u64
        L.inp_gen_u32.argtypes = [vp, u64, u64, u64, i32, u64]
        L.inp_gen_u32.restype = i32
        L.inp_gen_u64.argtypes = [vp, u64, u64, u64, i32]
        L.inp_gen_u64.restype = i32
        L.inp_iota_u32.argtypes = [vp, u64, u64]
        L.inp_iota_u32.restype = i32
        _lib = L
    return _lib


def _ptr(out, dtype, count):
    if isinstance(out, np.ndarray):
        assert out.dtype == dtype and out.flags.c_contiguous and out.size >= count
        return out.ctypes.data
    return int(out)  # raw host pointer (e.g. pinned torch tensor .data_ptr())


def splitmix64_at(seed: int, i: int) -> int:
    return lib().inp_splitmix64_at(seed, i)


def gen_u32(n: int, seed: int, dist: str = "uniform", start: int = 0,
            n_total: int | None = None, out=None) -> np.ndarray | None:
    """Keys of global indices [start, start+n) of the (seed, dist) stream."""
    if n_total is None:
        n_total = start + n
    arr = np.empty(n, dtype=np.uint32) if out is None else None
    p = _ptr(arr if out is None else out, np.uint32, n)
    if n and lib().inp_gen_u32(p, start, n, seed, U32_DISTS[dist], n_total) != 0:
        raise ValueError(f"inp_gen_u32 rejected dist={dist} n={n} start={start} n_total={n_total}")
    return arr


def gen_u64(n: int, seed: int, dist: str = "uniform", start: int = 0, out=None) -> np.ndarray | None:
    arr = np.empty(n, dtype=np.uint64) if out is None else None
    p = _ptr(arr if out is None else out, np.uint64, n)
    if n and lib().inp_gen_u64(p, start, n, seed, U64_DISTS[dist]) != 0:
        raise ValueError(f"inp_gen_u64 rejected dist={dist}")
    return arr


def iota_u32(n: int, start: int = 0, out=None) -> np.ndarray | None:
    arr = np.empty(n, dtype=np.uint32) if out is None else None
    p = _ptr(arr if out is None else out, np.uint32, n)
    if n:
        lib().inp_iota_u32(p, start, n)
    return arr


# BASELINE.json configs -> (key kind, n, seed, dist); see DESIGN.md "Input recipe"
CONFIGS = {
    "c1": dict(kind="u32", n=1 << 20, seed=1, dist="uniform", bits=(8,)),
    "c2": dict(kind="u32", n=1 << 24, seed=2, dist="half", bits=(8, 16)),
    "c3": dict(kind="u32", n=1 << 27, seed=3,
               dists=("uniform", "mod16", "gauss", "sorted", "reversed", "equal"), bits=(8,)),
    "c4": dict(kind="u32", n=1 << 31, seed=4, dist="uniform", bits=(8,)),
    "c5": dict(kind="pairs_u64_u32", n=1 << 30, seed=5, dist="uniform", bits=(8,)),
}
