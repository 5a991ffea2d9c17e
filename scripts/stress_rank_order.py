"""Stress evidence for design 5's one hardware assumption (same-address shared
atomics return their old values in lane order): many sorts of
fresh seeded inputs at the pass's real shapes and occupancy, every output checked
on the device — u32 keys for order and multiset (an unstable early pass leaves
the final keys out of order), (u64 key, u32 index) pairs with many equal keys for
stability directly (values of equal keys must ascend).  Prints one summary line.
Usage: python scripts/stress_rank_order.py [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (device-side order / stability / multiset checks)
import inputs  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
L = rs.lib()
assert rs.get_option("rank_probe") in (-1, 1)
SIZES_U32 = [(1 << 20) + 17, 1 << 24, (1 << 27) + 12345, 1 << 29]
DISTS_U32 = ["uniform", "mod16", "gauss", "half"]
SIZES_P = [(1 << 20) + 5, (1 << 24) + 3, 1 << 27]
t0 = time.time()
sorts = keys = bad = 0
seed = 1000
while time.time() - t0 < budget:
    for n in SIZES_U32:
        for d in DISTS_U32:
            seed += 1
            host = torch.empty(n, dtype=torch.int32, pin_memory=True)
            inputs.gen_u32(n, seed, d, out=host.data_ptr())
            x = host.cuda()
            h0 = bench.multiset_hash(x)
            rs.sort(x)
            viol = bench.order_violations(x)
            ok = viol == 0 and bench.multiset_hash(x) == h0
            sorts += 1
            keys += n
            bad += 0 if ok else 1
            del x, host
    for n in SIZES_P:
        seed += 1
        k = torch.from_numpy(inputs.gen_u64(n, seed, "mod1024").view(np.int64)).cuda()
        v = torch.arange(n, dtype=torch.int32, device="cuda")
        h0 = bench.multiset_hash(k, v)
        rs.sort_pairs(k, v)
        ok = bench.order_violations(k, v) == 0 and bench.multiset_hash(k, v) == h0
        sorts += 1
        keys += n
        bad += 0 if ok else 1
        del k, v
    torch.cuda.synchronize()
print(f"stress: {sorts} sorts, {keys / 1e9:.2f} G keys, {bad} failed (order / stability / multiset), "
      f"design {rs.get_option('pass_design')}, rank probe {rs.get_option('rank_probe')}, "
      f"{torch.cuda.get_device_name()}, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
