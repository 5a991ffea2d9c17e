"""Small run of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): radix-256 and radix-65536 sorts of u32 / u64 / pairs with ragged
tails, the wide-status and alternative pass designs, histogram, GSD emulation
with the merge tree.  Exits non-zero on any mismatch against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

L = rs.lib()


def dev(a):
    return torch.from_numpy(a.view(np.int32 if a.dtype == np.uint32 else np.int64)).cuda()


def host(t, dt):
    return t.cpu().numpy().view(dt)


def check(ok, what):
    if not ok:
        print("MISMATCH", what)
        sys.exit(1)


n = 3 * 6144 + 777
a = inputs.gen_u32(n, 1)
for design in (2, 0, 1, 3):
    L.rs_set_option(b"pass_design", design)
    for wide in (0, 1):
        L.rs_set_option(b"wide_status", wide)
        t = dev(a)
        rs.sort(t, digit_bits=8)
        check((host(t, np.uint32) == oracle.sr(a, 8)).all(), f"u32 design {design} wide {wide}")
L.rs_set_option(b"pass_design", 2)
L.rs_set_option(b"wide_status", 0)
t = dev(a)
rs.sort(t, digit_bits=16)
check((host(t, np.uint32) == oracle.sr(a, 16)).all(), "u32 b16")
k = inputs.gen_u64(n, 2, "mod1024")
v = inputs.iota_u32(n)
for b in (8, 16):
    tk, tv = dev(k), dev(v)
    rs.sort_pairs(tk, tv, digit_bits=b)
    wk, wv = oracle.sr(k, b, vals=v)
    check((host(tk, np.uint64) == wk).all() and (host(tv, np.uint32) == wv).all(), f"pairs b{b}")
h = rs.digit_histogram(dev(a), 8).cpu().numpy().view(np.uint32)
check((h.astype(np.uint64) == oracle.hist(a, 8)).all(), "hist")
blocks = [inputs.gen_u32(m, 10 + m) for m in (5000, 0, 7001, 333)]
got = rs.gsd_emulate([dev(x) for x in blocks], r=8, digit_bits=8)
want = oracle.gsd(blocks, r=8)
check(all((host(got["Y"][j], np.uint32) == want["Y"][j]).all() for j in range(4)), "gsd")
torch.cuda.synchronize()
print("sanitize workload ok")
