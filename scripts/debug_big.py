"""Debug aid: sort large u32 inputs, report descents / CUDA errors per size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, paper_1808_10292_b200 as rs
for spec in sys.argv[1:]:
    n = eval(spec)
    a = inputs.gen_u32(n, 4)
    try:
        t = torch.from_numpy(a.view(np.int32)).cuda()
        for end_bit in (8, 32):
            out = rs.sort_bits(t, end_bit=end_bit, digit_bits=8)
            torch.cuda.synchronize()
            g = out.cpu().numpy().view(np.uint32)
            m = np.uint32((1 << end_bit) - 1) if end_bit < 32 else np.uint32(0xFFFFFFFF)
            gm = g & m
            bad = np.nonzero(gm[1:] < gm[:-1])[0]
            print(f"n={spec} end_bit={end_bit}: {bad.size} descents {bad[:6]}", flush=True)
            del out
        del t
        torch.cuda.empty_cache()
    except Exception as e:
        print(f"n={spec}: EXCEPTION {type(e).__name__}: {str(e)[:300]}", flush=True)
        break
