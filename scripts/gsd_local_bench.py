"""Per-phase device times of the collective sort run by p in-process ranks on one
GPU (LocalGroup; the multi-GPU orchestration over the in-process transport).  The
host barriers of the in-process transport serialise the ranks' exchanges, so the
wall time is not a multi-GPU number; the per-kernel event times are (each rank's
kernels are its own).  Usage: python scripts/gsd_local_bench.py [log2_total] [p] [mode] [u32|pairs]
(pairs: config 5's (u64 key, u32 index) pairs)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_10292_b200 as rs  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mode = sys.argv[3] if len(sys.argv) > 3 else "gsd"
kind = sys.argv[4] if len(sys.argv) > 4 else "u32"
n = 1 << lg
N = n // p
L = rs.lib()
g = torch.Generator(device="cuda").manual_seed(4)
if kind == "pairs":
    src = torch.randint(-2 ** 63, 2 ** 63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
    idx = torch.arange(n, dtype=torch.int32, device="cuda")
else:
    src = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    idx = None


def q(prefix):
    ms, cnt = ctypes.c_double(), ctypes.c_int()
    L.rs_timing_query(prefix.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value


for rep in range(3):
    blocks = [src[k * N:(k + 1) * N].clone() for k in range(p)]
    vblocks = [idx[k * N:(k + 1) * N].clone() for k in range(p)] if idx is not None else None
    torch.cuda.synchronize()
    L.rs_timing_reset()
    L.rs_timing_enable(1)
    got = rs.sort_ranks(blocks, mode, vals=vblocks)
    torch.cuda.synchronize()
    L.rs_timing_enable(0)
    if rep < 2:
        continue
    import bench  # device-side order + multiset checks
    y = torch.cat(got["Y"])
    yv = torch.cat(got["Yv"]) if idx is not None else None
    ok = bench.order_violations(y, yv) == 0 and bench.multiset_hash(y, yv) == bench.multiset_hash(src, idx)
    print(f"{mode} {kind} n=2^{lg} p={p}: correct={ok} max|Y_j|={max(got['n_out'])} (N={N})")
    for name in ("hist", "onesweep", "gsd_sample", "gsd_splitters", "gsd_split", "pw_sample", "pw_pos", "pw_bounds",
                 "pw_merge", "merge_", "gsd_pull_merge", "gsd_exchange"):
        ms, cnt = q(name)
        if cnt:
            print(f"   {name:16s} {cnt:4d} launches  total {ms:8.3f} ms  per rank {ms / p:7.3f} ms")
    ms, cnt = q("pw_merge")
    if cnt:
        out_bytes = 2 * n * (4 if idx is None else 12)
        print(f"   k_pw_merge: {out_bytes / (ms / p * 1e-3) / p / 1e12:.2f} TB/s per rank "
              f"(read + write of Y_j, {out_bytes / p / 1e9:.2f} GB per rank)")
