"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of the plain serial C oracle (oracle/*.c), written from the paper
(PAPER.md:653-681 SR4 count-sort rounds; Algorithm 1 GSD;
PAPER.md:471-535 BTN and OET).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product path
(paper_1808_10292_b200/) never does, and shares no code with it.

Parity status: SR-b, histograms and the GSD concatenated
output are pinned (library sort, brute force, masked stable sort, bincount);
GSD's per-rank partition is pinned by two hand-derived traces (SPEC.md:290,
p = 2; tests/golden/gsd_hand_trace_p3_r2.json, p = 3, r = 2 with duplicates
within and across ranks) and the balance bound; the paper prints no partition,
so beyond those traces it rests on DESIGN.md readings R10/R12/R14.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, f) for f in ("sr.c", "gsd.c", "net.c", "verify.c")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# bench.py's CPU baseline: the same sources built on the timing host with
# -O3 -march=native; tests use the generic build
_NATIVE_PATH = os.path.join("/tmp", f"liboracle_native_{os.getuid()}_{os.getpid()}.so")
_FLAGS = {"generic": ["-O2"], "native": ["-O3", "-march=native"]}
_lib = None
_flavor = "generic"


def build(force: bool = False, flavor: str = "generic") -> str:
    """gcc -O2 generic x86-64 (the test build, also runs on the GPU box's host), or
    flavor "native": gcc -O3 -march=native for this host (bench CPU baseline)."""
    path = _LIB_PATH if flavor == "generic" else _NATIVE_PATH
    newest = max(os.path.getmtime(p) for p in _SRCS + [os.path.join(_HERE, "oracle.h")])
    if force or not os.path.exists(path) or os.path.getmtime(path) < newest:
        tmp = path + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc"] + _FLAGS[flavor] + ["-std=c99", "-fPIC", "-shared", "-o", tmp] + _SRCS)
        os.replace(tmp, path)
    return path


def use_native() -> str:
    """Load the -O3 -march=native build instead (before the first oracle call of
    the process); returns the compiler flags used."""
    global _flavor
    if _lib is not None and _flavor != "native":
        raise RuntimeError("oracle already loaded with the generic build")
    _flavor = "native"
    return " ".join(_FLAGS["native"])


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build(flavor=_flavor))
        vp, sz, i32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
        for name in ("or_sr_u32", "or_sr_u64"):
            getattr(L, name).argtypes = [vp, sz, i32, i32]
            getattr(L, name).restype = i32
        L.or_sr_pairs_u64_u32.argtypes = [vp, vp, sz, i32, i32]
        L.or_sr_pairs_u64_u32.restype = i32
        for name in ("or_hist_u32", "or_hist_u64"):
            getattr(L, name).argtypes = [vp, sz, i32, vp]
            getattr(L, name).restype = i32
        L.or_gsd_u64.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, sz, vp, vp, vp]
        L.or_gsd_u64.restype = i32
        L.or_gsd_u32.argtypes = [i32, i32, i32, vp, vp, vp, sz, vp, vp, vp]
        L.or_gsd_u32.restype = i32
        u64 = ctypes.c_uint64
        L.or_ger_u64.argtypes = [i32, sz, u64, i32, vp, vp, vp, vp, vp, sz, vp, vp, vp]
        L.or_ger_u64.restype = i32
        L.or_ger_u32.argtypes = [i32, sz, u64, i32, vp, vp, vp, sz, vp, vp, vp]
        L.or_ger_u32.restype = i32
        L.or_gvr_u64.argtypes = [i32, sz, u64, i32, vp, vp, vp, vp, vp, sz, vp, vp, vp]
        L.or_gvr_u64.restype = i32
        L.or_gvr_u32.argtypes = [i32, sz, u64, i32, vp, vp, vp, sz, vp, vp, vp]
        L.or_gvr_u32.restype = i32
        for name in ("or_btn_u32", "or_oet_u32"):
            getattr(L, name).argtypes = [i32, i32, vp, sz, i32, vp]
            getattr(L, name).restype = i32
        for name in ("or_btn_u64", "or_oet_u64"):
            getattr(L, name).argtypes = [i32, i32, vp, vp, sz, i32, vp]
            getattr(L, name).restype = i32
        L.or_splitmix64_at.argtypes = [u64, u64]
        L.or_splitmix64_at.restype = u64
        for name in ("or_is_nondecreasing_u32", "or_is_nondecreasing_u64"):
            getattr(L, name).argtypes = [vp, sz]
            getattr(L, name).restype = i32
        for name in ("or_multiset_hash_u32", "or_multiset_hash_u64"):
            getattr(L, name).argtypes = [vp, sz, vp]
            getattr(L, name).restype = None
        L.or_multiset_hash_pairs_u64_u32.argtypes = [vp, vp, sz, vp]
        L.or_multiset_hash_pairs_u64_u32.restype = None
        L.or_pairs_stable_u64_u32.argtypes = [vp, vp, sz]
        L.or_pairs_stable_u64_u32.restype = i32
        L.or_check_order_stats_u32.argtypes = [vp, sz, vp, vp, sz]
        L.or_check_order_stats_u32.restype = sz
        _lib = L
    return _lib


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


# ---- SR-b ------------------------------------------------

def sr(keys: np.ndarray, b: int = 8, rounds: int = -1, vals: np.ndarray | None = None):
    """Serial LSD radix sort by count-sort rounds; returns a sorted copy (and vals).

    `rounds` >= 0 stops after that many rounds (the intermediate array after
    round t is what a GPU pass t must produce)."""
    k = np.array(keys, copy=True)
    L = lib()
    if vals is not None:
        assert k.dtype == np.uint64
        v = np.array(vals, dtype=np.uint32, copy=True)
        rc = L.or_sr_pairs_u64_u32(k.ctypes.data, v.ctypes.data, k.size, b, rounds)
        if rc:
            raise ValueError("or_sr_pairs_u64_u32 failed")
        return k, v
    if k.dtype == np.uint32:
        rc = L.or_sr_u32(k.ctypes.data, k.size, b, rounds)
    elif k.dtype == np.uint64:
        rc = L.or_sr_u64(k.ctypes.data, k.size, b, rounds)
    else:
        raise TypeError(k.dtype)
    if rc:
        raise ValueError(f"or_sr failed (b={b})")
    return k


def hist(keys: np.ndarray, b: int = 8) -> np.ndarray:
    """All rounds' digit counts: shape (keybits/b, 2^b)."""
    k = np.ascontiguousarray(keys)
    P = k.dtype.itemsize * 8 // b
    out = np.zeros((P, 1 << b), dtype=np.uint64)
    fn = lib().or_hist_u32 if k.dtype == np.uint32 else lib().or_hist_u64
    if fn(k.ctypes.data, k.size, b, out.ctypes.data):
        raise ValueError("or_hist failed")
    return out


# ---- GSD ---------------------------------------------------

def gsd(shards, r: int, b: int = 8, vals=None, cap: int | None = None):
    """Simulate GSD over p = len(shards) blocks.

    Returns dict(Y=[...], Yv=[...] or None, splitters=(p-1,3) array, counts=(p,p))."""
    return _sample_sort(shards, 0, r, 0, b, vals, cap)


def ger(shards, s: int, seed: int, b: int = 8, vals=None, cap: int | None = None):
    """Simulate GER over p = len(shards) blocks: s·p − 1 random
    samples drawn with SplitMix64(seed) (readings R28-R30); same result dict as gsd()."""
    return _sample_sort(shards, 1, s, seed, b, vals, cap)


def gvr(shards, s: int, seed: int, b: int = 8, vals=None, cap: int | None = None):
    """Simulate GVR over p = len(shards) blocks: random sample
    of the unsorted blocks, split by destination, local sort of each Y_j."""
    return _sample_sort(shards, 2, s, seed, b, vals, cap)


def splitmix64_at(seed: int, i: int) -> int:
    return int(lib().or_splitmix64_at(seed, i))


def _net(mode, blocks, b, vals, max_stages):
    p = len(blocks)
    N = blocks[0].size if p else 0
    if any(x.size != N for x in blocks):
        raise ValueError("BTN/OET need equal block sizes (reading R34)")
    is32 = blocks[0].dtype == np.uint32
    dt = np.uint32 if is32 else np.uint64
    K = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=dt) for x in blocks]) if p else
                             np.empty(0, dt))
    Vv = None
    if vals is not None:
        assert not is32, "values ride with u64 keys"
        Vv = np.ascontiguousarray(np.concatenate([np.asarray(v, dtype=np.uint32) for v in vals]))
    st = ctypes.c_int(0)
    L = lib()
    if is32:
        assert vals is None
        fn = L.or_btn_u32 if mode == 0 else L.or_oet_u32
        rc = fn(p, b, K.ctypes.data, N, max_stages, ctypes.byref(st))
    else:
        fn = L.or_btn_u64 if mode == 0 else L.or_oet_u64
        rc = fn(p, b, K.ctypes.data, None if Vv is None else Vv.ctypes.data, N, max_stages, ctypes.byref(st))
    if rc:
        raise ValueError("BTN needs p a power of two" if mode == 0 else "bad OET arguments")
    out = dict(Y=[K[k * N:(k + 1) * N] for k in range(p)], stages=st.value)
    out["Yv"] = None if Vv is None else [Vv[k * N:(k + 1) * N] for k in range(p)]
    return out


def btn(blocks, b: int = 8, vals=None, max_stages: int = -1):
    """BTN: local SR-b of each equal-size block, then the
    lg p (lg p + 1)/2-stage bitonic merge-split network.  Returns dict(Y, Yv, stages)."""
    return _net(0, blocks, b, vals, max_stages)


def oet(blocks, b: int = 8, vals=None, max_stages: int = -1):
    """OET: local SR-b, then p rounds of odd-even transposition
    merge-splits.  Returns dict(Y, Yv, stages)."""
    return _net(1, blocks, b, vals, max_stages)


def _sample_sort(shards, mode, r_or_s, seed, b, vals, cap):
    p = len(shards)
    is32 = shards[0].dtype == np.uint32
    dt = np.uint32 if is32 else np.uint64
    ks = [np.ascontiguousarray(s, dtype=dt) for s in shards]
    N = np.array([s.size for s in ks], dtype=np.uint64)
    if cap is None:
        cap = int(N.sum())
    Y = [np.empty(max(cap, 1), dtype=dt) for _ in range(p)]
    kp = (ctypes.c_void_p * p)(*[s.ctypes.data for s in ks])
    yp = (ctypes.c_void_p * p)(*[y.ctypes.data for y in Y])
    ylen = np.zeros(p, dtype=np.uint64)
    spl = np.zeros((max(p - 1, 1), 3), dtype=np.uint64)
    counts = np.zeros((p, p), dtype=np.uint64)
    L = lib()
    Yv = None
    if is32:
        assert vals is None
        if mode == 0:
            rc = L.or_gsd_u32(p, r_or_s, b, kp, N.ctypes.data, yp, cap, ylen.ctypes.data,
                              spl.ctypes.data, counts.ctypes.data)
        else:
            fn = L.or_ger_u32 if mode == 1 else L.or_gvr_u32
            rc = fn(p, r_or_s, seed, b, kp, N.ctypes.data, yp, cap, ylen.ctypes.data,
                    spl.ctypes.data, counts.ctypes.data)
    else:
        vp_ = None
        if vals is not None:
            vs = [np.ascontiguousarray(v, dtype=np.uint32) for v in vals]
            Yv = [np.empty(max(cap, 1), dtype=np.uint32) for _ in range(p)]
            vp_ = (ctypes.c_void_p * p)(*[v.ctypes.data for v in vs])
            yvp = (ctypes.c_void_p * p)(*[y.ctypes.data for y in Yv])
        fn = [L.or_gsd_u64, L.or_ger_u64, L.or_gvr_u64][mode]
        args = (p, r_or_s) if mode == 0 else (p, r_or_s, seed)
        rc = fn(*args, b, kp, vp_, N.ctypes.data, yp,
                yvp if vals is not None else None, cap, ylen.ctypes.data,
                spl.ctypes.data, counts.ctypes.data)
    if rc == -2:
        raise OverflowError("GSD output exceeds capacity")
    if rc:
        raise ValueError("or_gsd failed")
    out = dict(Y=[Y[j][: int(ylen[j])] for j in range(p)], splitters=spl[: p - 1], counts=counts,
               Ylen=ylen)
    out["Yv"] = None if Yv is None else [Yv[j][: int(ylen[j])] for j in range(p)]
    return out


# ---- invariants -------------------------------------------------------------

def is_nondecreasing(a: np.ndarray) -> bool:
    a = np.ascontiguousarray(a)
    fn = lib().or_is_nondecreasing_u32 if a.dtype == np.uint32 else lib().or_is_nondecreasing_u64
    return bool(fn(a.ctypes.data, a.size))


def multiset_hash(a: np.ndarray, vals: np.ndarray | None = None) -> tuple:
    a = np.ascontiguousarray(a)
    out = np.zeros(3, dtype=np.uint64)
    if vals is not None:
        v = np.ascontiguousarray(vals, dtype=np.uint32)
        lib().or_multiset_hash_pairs_u64_u32(a.ctypes.data, v.ctypes.data, a.size, out.ctypes.data)
    elif a.dtype == np.uint32:
        lib().or_multiset_hash_u32(a.ctypes.data, a.size, out.ctypes.data)
    else:
        lib().or_multiset_hash_u64(a.ctypes.data, a.size, out.ctypes.data)
    return tuple(int(x) for x in out)


def pairs_stable(k: np.ndarray, v: np.ndarray) -> bool:
    k = np.ascontiguousarray(k, dtype=np.uint64)
    v = np.ascontiguousarray(v, dtype=np.uint32)
    return bool(lib().or_pairs_stable_u64_u32(k.ctypes.data, v.ctypes.data, k.size))


def check_order_stats_u32(a: np.ndarray, pos: np.ndarray, val: np.ndarray) -> int:
    """Number of sampled (pos, val) that are NOT the pos-th smallest of a[]."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    pos = np.ascontiguousarray(pos, dtype=np.uint64)
    val = np.ascontiguousarray(val, dtype=np.uint32)
    return int(lib().or_check_order_stats_u32(a.ctypes.data, a.size, pos.ctypes.data,
                                               val.ctypes.data, pos.size))
