"""K1 (digit histogram) fixed cost: back-to-back launches timed with one event pair,
per size (development aid).  python scripts/k1_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1808_10292_b200 as rs  # noqa: E402

for lg in [int(x) for x in (sys.argv[1:] or [20, 22, 24, 26, 27, 28, 30])]:
    n = 1 << lg
    keys = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
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
    print(f"n=2^{lg}: {ms * 1000:.1f} us per call  {4 * n / ms / 1e6:.0f} GB/s", flush=True)
    del keys
