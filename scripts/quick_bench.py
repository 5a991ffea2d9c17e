"""Quick per-kernel timing of the single-GPU sort (development aid; bench.py is
the contract).  Usage: python scripts/quick_bench.py [log2n ...]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

L = rs.lib()
PEAK = 6545.6
ONE_PASS = os.environ.get("RS_ONE_PASS") == "1"
for _opt in ("wide_status", "pass_design", "small_tiles", "pdl"):
    if os.environ.get("RS_" + _opt.upper()):
        L.rs_dev_set_option(_opt.encode(), int(os.environ["RS_" + _opt.upper()]))


def q(prefix):
    ms, cnt = ctypes.c_double(), ctypes.c_int()
    L.rs_timing_query(prefix.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value


def run(log2n, kind="u32", b=8, dist="uniform", reps=5):
    n = 1 << log2n if isinstance(log2n, int) else int(log2n[1:])  # "n133365760": an explicit size
    if kind == "u32":
        a = inputs.gen_u32(n, 4, dist)
        src = torch.from_numpy(a.view(np.int32)).cuda()
        kb, vb = 4, 0
    else:
        a = inputs.gen_u64(n, 5)
        src = torch.from_numpy(a.view(np.int64)).cuda()
        kb = 8
        vb = 4 if kind == "pairs" else 0
    vals0 = torch.arange(n, dtype=torch.int32, device="cuda") if vb else None
    work = torch.empty_like(src)
    vwork = torch.empty_like(vals0) if vb else None
    ws = torch.empty(rs.workspace_bytes(kb, vb, n, b), dtype=torch.uint8, device="cuda")
    obuf = torch.empty_like(src) if ONE_PASS else None
    ovbuf = torch.empty_like(vals0) if (ONE_PASS and vb) else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for i in range(reps + 2):
        work.copy_(src)
        if vb:
            vwork.copy_(vals0)
        torch.cuda.synchronize()
        if i == 2 and os.environ.get("RS_NO_KTIMING") != "1":  # whole-sort time only (no events between kernels)
            L.rs_timing_reset()
            L.rs_timing_enable(1)
        e0.record()
        if ONE_PASS:  # pass 0 only (ablations: later passes would see corrupted digits)
            rs.sort_bits(work, end_bit=b, digit_bits=b, vals=vwork if vb else None, out_keys=obuf,
                         out_vals=ovbuf, ws=ws)
        elif vb:
            rs.sort_pairs(work, vwork, digit_bits=b, ws=ws)
        else:
            rs.sort(work, digit_bits=b, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            times.append(e0.elapsed_time(e1))
    L.rs_timing_enable(0)
    t = float(np.median(times))
    per_key = {("u32", 8): 36, ("u32", 16): 20, ("u64", 8): 72, ("pairs", 8): 200, ("u64", 16): 40,
               ("pairs", 16): 104}[(kind, b)]
    gk = n / t / 1e6
    print(f"{kind} b={b} {dist} n={n}: {t:.3f} ms  {gk:.1f} Gkeys/s  "
          f"{per_key * n / t / 1e6:.0f} GB/s ({per_key * n / t / 1e6 / PEAK * 100:.1f}% of {PEAK})")
    for name in ["hist", "plan", "onesweep", "final_copy", "r16_count", "r16_total", "r16_scan", "r16_offsets",
                 "r16_scatter"]:
        ms, cnt = q(name)
        if cnt:
            avg = ms / cnt
            extra = ""
            if name == "onesweep":
                bpk = {4: 8, 8: 16}[kb] + (8 if vb else 0)
                extra = f"  pass {avg:.3f} ms -> {bpk * n / avg / 1e6:.0f} GB/s ({bpk * n / avg / 1e6 / PEAK * 100:.1f}%)"
            if name == "hist":
                extra = f"  -> {kb * n / avg / 1e6:.0f} GB/s"
            print(f"   {name:12s} {cnt:4d} launches  avg {avg:.4f} ms{extra}")
    del ws, work, src


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["20", "24", "27", "30"]
    for c in cfgs:
        parts = c.split(":")
        log2n = int(parts[0]) if not parts[0].startswith("n") else parts[0]
        kind = parts[1] if len(parts) > 1 else "u32"
        b = int(parts[2]) if len(parts) > 2 else 8
        dist = parts[3] if len(parts) > 3 else "uniform"
        run(log2n, kind, b, dist)
