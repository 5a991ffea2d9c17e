"""Time one 2-way merge level through rs_gsd_emulate with p=2 (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs, paper_1808_10292_b200 as rs
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
a = inputs.gen_u32(n, 4)
blocks = [torch.from_numpy(a[k * (n // 2):(k + 1) * (n // 2)].view("int32")).cuda() for k in range(2)]
for _ in range(2):
    rs.gsd_emulate([b.clone() for b in blocks], r=8, digit_bits=8)
torch.cuda.synchronize()
