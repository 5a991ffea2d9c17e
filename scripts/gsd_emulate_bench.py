"""Time GSD's device phases through rs_gsd_emulate (all p ranks on one GPU, run
rank by rank): per-rank local sort, sample/splitters/split kernels and step-5
merge, as averages per rank.  Development aid for projecting the multi-GPU step.
Usage: python scripts/gsd_emulate_bench.py [log2_total] [p] [merge(0 tree|1 resort|2 pull|3 pull p-way)] [gsd|ger|gvr|pr4|btn|oet]
(pr4: "sample/split kernels" is the per-round pull of the routed keys; btn/oet:
"merge-tree" is the merge-split stages, each rank's half per stage)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 27
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
merge = int(sys.argv[3]) if len(sys.argv) > 3 else 0
mode = sys.argv[4] if len(sys.argv) > 4 else "gsd"
L = rs.lib()
L.rs_set_option(b"gsd_merge", merge)
n = 1 << log2n
N = n // p
host = torch.empty(n, dtype=torch.int32, pin_memory=True)
inputs.gen_u32(n, 4, "uniform", out=host.data_ptr())
pristine = host.cuda()
blocks = [torch.empty(N, dtype=torch.int32, device="cuda") for _ in range(p)]


def q(prefix):
    ms, cnt = ctypes.c_double(), ctypes.c_int()
    L.rs_timing_query(prefix.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value


for it in range(3):
    for k in range(p):
        blocks[k].copy_(pristine[k * N:(k + 1) * N])
    torch.cuda.synchronize()
    if it == 2:
        L.rs_timing_reset()
        L.rs_timing_enable(1)
    if mode == "gsd":
        got = rs.gsd_emulate(blocks, r=8, digit_bits=8)
    elif mode == "ger":
        got = rs.ger_emulate(blocks, s=0, seed=1, digit_bits=8)
    elif mode == "gvr":
        got = rs.gvr_emulate(blocks, s=0, seed=1, digit_bits=8)
    elif mode in ("btn", "oet"):
        got = rs.net_emulate(mode, blocks)
        got.update(counts=np.zeros((p, p), dtype=np.uint64), n_out=[N] * p)
    else:
        got = rs.pr_emulate(blocks)
        got.update(counts=np.zeros((p, p), dtype=np.uint64), n_out=[N] * p)
    torch.cuda.synchronize()
L.rs_timing_enable(0)
sort_ms = sum(q(x)[0] for x in ("hist", "plan", "onesweep", "final_copy"))
merge_ms = sum(q(x)[0] for x in ("merge_split", "merge_tile", "pw_sample", "pw_pos", "pw_bounds", "pw_merge"))
gsd_ms = sum(q(x)[0] for x in ("gsd_sample", "gsd_splitters", "gsd_split", "ger_sample", "gvr_split", "pr_pull"))
all_ms = q("")[0] - q("gsd_pull_merge")[0]  # the pull scope wraps kernels timed on their own
ex_ms = q("gsd_exchange")[0]
counts = got["counts"].astype(np.int64)
off_rank = max(int(counts[k].sum() - counts[k, k]) for k in range(p))
print(f"{mode.upper()} emulation n=2^{log2n} p={p} merge={['tree', 're-sort', 'pull', 'pull p-way'][merge]}")
print(f"  per rank: all device time {all_ms / p:.3f} ms")
print(f"  per rank: local sort {sort_ms / p:.3f} ms (incl. re-sort if merge=1), sample/split kernels {gsd_ms / p:.3f} ms,"
      f" merge-tree {merge_ms / p:.3f} ms, device-copy exchange {ex_ms / p:.3f} ms")
print(f"  max off-rank keys sent by a rank: {off_rank} ({off_rank * 4 / 2**20:.1f} MiB) -> at 770 GB/s "
      f"{off_rank * 4 / 770e9 * 1e3:.3f} ms")
print(f"  p-way: sample {q('pw_sample')[0] / p:.3f}, bounds {q('pw_bounds')[0] / p:.3f}, merge {q('pw_merge')[0] / p:.3f} ms per rank")
print(f"  merge_split {q('merge_split')[0] / p:.3f} ms ({q('merge_split')[1]} launches), merge_tile {q('merge_tile')[0] / p:.3f} ms per rank")
print(f"  max |Y_j| = {max(got['n_out'])}, N = {N}, GSD bound = {N + N // 8}, "
      f"GER/GVR capacity = {L.rs_ger_capacity(N, p, 0)}")
