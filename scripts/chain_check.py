"""Quick device-side check of the sort against torch.sort (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

L = rs.lib()
if os.environ.get("RS_CHAIN"):
    L.rs_dev_set_option(b"chain", int(os.environ["RS_CHAIN"]))
g = torch.Generator(device="cuda").manual_seed(1)
for n in [1000, 6144 * 3 + 5, 1 << 20, (1 << 24) + 77, 1 << 27]:
    x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    ref = torch.sort(x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
    y = x.clone()
    rs.sort(y, digit_bits=8)
    ok = torch.equal(y.to(torch.int64) & 0xFFFFFFFF, ref)
    k = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64, device="cuda", generator=g) & 0xFFFF
    v = torch.arange(n, dtype=torch.int32, device="cuda")
    rk, ri = torch.sort(k, stable=True)
    rs.sort_pairs(k, v, digit_bits=8)
    okp = torch.equal(k, rk) and torch.equal(v.to(torch.int64), ri)
    print(f"n={n}: u32 {'ok' if ok else 'MISMATCH'}  pairs {'ok' if okp else 'MISMATCH'}", flush=True)
