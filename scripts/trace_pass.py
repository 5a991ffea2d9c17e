"""Phase timeline of one radix-256 pass (diagnostic build: RS_NVCC_DEFINES=-DRS_AR_TRACE,
library path in RS_LIB_PATH).  Sorts n u32 keys; the trace holds the last pass's
per-tile globaltimer stamps: start, after [rank], after [scatter], after
[look-back], end of [store].  Prints where the pass's time goes: the first wave,
the steady state and the tail.  Usage: python scripts/trace_pass.py [log2n]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
n = 1 << lg
L = rs.lib()
L.rs_dev_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
a = inputs.gen_u32(n, 3)
src = torch.from_numpy(a.view(np.int32)).cuda()
x = torch.empty_like(src)
ws = torch.empty(rs.workspace_bytes(4, 0, n, 8), dtype=torch.uint8, device="cuda")
for _ in range(3):
    x.copy_(src)
    torch.cuda.synchronize()
    rs.sort(x, ws=ws)
    torch.cuda.synchronize()
TILE = rs.get_option("tile_u32")
T = (n + TILE - 1) // TILE
buf = np.zeros((1 << 17, 6), dtype=np.uint64)
assert L.rs_dev_trace_copy(buf.ctypes.data, buf.nbytes) == 0
tr = buf[:T].astype(np.int64)
t0 = tr[:, 0].min()
st, rk, sc, lb, en = [(tr[:, k] - t0) / 1e3 for k in range(5)]  # us
sm = tr[:, 5]
span = en.max()
print(f"n=2^{lg}: {T} tiles of {TILE}; pass span {span:.1f} us (first tile start -> last tile end)")
d = np.stack([rk - st, sc - rk, lb - sc, en - lb], 1)
names = ["rank", "offset+scatter", "look-back", "next+store"]
W = 296
for lo, hi, lab in ((0, W, "first wave"), (W, max(W, T - W), "steady"), (max(W, T - W), T, "last wave")):
    if hi > lo:
        m = d[lo:hi].mean(0)
        print(f"  {lab:10s} tiles {lo:6d}-{hi:6d}: " + ", ".join(f"{nm} {v:6.2f}" for nm, v in zip(names, m)) +
              f"  (tile {m.sum():.2f} us)")
# CTA occupancy over time: how many tiles are in flight at each moment
ts = np.linspace(0, span, 400)
busy = np.array([((st <= t) & (en > t)).sum() for t in ts])
full = np.median(busy[len(ts) // 4: 3 * len(ts) // 4])
ramp = ts[np.argmax(busy >= 0.9 * full)]
tail = span - ts[len(ts) - 1 - np.argmax(busy[::-1] >= 0.9 * full)]
lost = ((full - np.minimum(busy, full)) * (ts[1] - ts[0])).sum() / full
print(f"  tiles in flight: steady {full:.0f}; ramp to 90 % after {ramp:.1f} us; below 90 % for the last {tail:.1f} us;"
      f" in-flight deficit = {lost:.1f} us of full-occupancy time")
first_end = np.sort(en[:W])
print(f"  first wave: tiles start within {st[:W].max():.1f} us; end between {first_end[0]:.1f} and {first_end[-1]:.1f} us")
last = np.argsort(en)[-W:]
print(f"  last {W} tiles to finish end between {en[last].min():.1f} and {span:.1f} us; the last tile started at "
      f"{st[np.argmax(en)]:.1f} us")
