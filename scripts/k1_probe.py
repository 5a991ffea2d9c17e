"""K1 (digit histogram) timing: back-to-back calls timed with one event pair, per
size (development aid).  python scripts/k1_probe.py 27 28:u64 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1808_10292_b200 as rs  # noqa: E402

for arg in (sys.argv[1:] or ["20", "24", "26", "27", "28", "30"]):
    lg, _, kind = arg.partition(":")
    lg, kind = int(lg), kind or "u32"
    n = 1 << lg
    dt, kb = (torch.int32, 4) if kind == "u32" else (torch.int64, 8)
    keys = torch.randint(-2**31, 2**31 - 1, (n,), dtype=dt, device="cuda")
    if kind == "u64":
        keys = keys * 0x9E3779B97F4A7C15 + 12345
    for _ in range(3):
        rs.digit_histogram(keys)
    torch.cuda.synchronize()
    reps = 50 if lg <= 28 else 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rs.digit_histogram(keys)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{kind} n=2^{lg}: {ms * 1000:.1f} us per call  {kb * n / ms / 1e6:.0f} GB/s", flush=True)
    del keys
