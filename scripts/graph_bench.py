"""Single-GPU sort launched directly vs replayed from a CUDA graph (small
inputs are launch-bound: BASELINE config 1).  Usage: python scripts/graph_bench.py [log2n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1808_10292_b200 as rs  # noqa: E402

if os.environ.get("RS_SMALL_FUSED"):
    rs.lib().rs_set_option(b"small_fused", int(os.environ["RS_SMALL_FUSED"]))
for log2n in [int(x) for x in sys.argv[1:]] or [20, 22, 24]:
    n = 1 << log2n
    src = torch.from_numpy(inputs.gen_u32(n, 1).view(np.int32)).cuda()
    work = torch.empty_like(src)
    ws = torch.empty(rs.workspace_bytes(4, 0, n, 8), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        work.copy_(src)
        rs.sort(work, ws=ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            rs.sort(work, ws=ws, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for mode in ("direct", "graph"):
        ts = []
        for i in range(25):
            with torch.cuda.stream(s):
                work.copy_(src)
                e0.record(s)
                if mode == "graph":
                    g.replay()
                else:
                    rs.sort(work, ws=ws, stream=s)
                e1.record(s)
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1))
        res[mode] = float(np.median(ts))
    print(f"n=2^{log2n}: direct {res['direct']:.4f} ms ({n / res['direct'] / 1e6:.1f} Gkeys/s), "
          f"graph replay {res['graph']:.4f} ms ({n / res['graph'] / 1e6:.1f} Gkeys/s)")
