"""Write tests/golden/inputs_frozen.json: the first 16 keys of every config's
(dist, seed) stream (SPEC.md:467 asks for frozen generator vectors).  Calls only
inputs/ (no oracle, no CUDA path)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402

out = {"citation": "regression vectors of inputs/gen.c (SplitMix64 counter stream; SPEC.md:316, 467); "
                   "written by scripts/freeze_inputs.py", "u32": {}, "u64": {}}
for name, dist, seed, n_total in [("c1_uniform", "uniform", 1, 1 << 20), ("c2_half", "half", 2, 1 << 24),
                                  ("c3_uniform", "uniform", 3, 1 << 27), ("c3_mod16", "mod16", 3, 1 << 27),
                                  ("c3_gauss", "gauss", 3, 1 << 27), ("c3_sorted", "sorted", 3, 1 << 27),
                                  ("c3_reversed", "reversed", 3, 1 << 27), ("c3_equal", "equal", 3, 1 << 27),
                                  ("c4_uniform", "uniform", 4, 1 << 31)]:
    out["u32"][name] = dict(dist=dist, seed=seed, n_total=n_total,
                            first16=inputs.gen_u32(16, seed, dist, n_total=n_total).tolist())
for name, dist, seed in [("c5_uniform", "uniform", 5), ("c5_mod1024", "mod1024", 5)]:
    out["u64"][name] = dict(dist=dist, seed=seed, first16=[str(x) for x in inputs.gen_u64(16, seed, dist).tolist()])
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "inputs_frozen.json")
json.dump(out, open(p, "w"), indent=1)
print("wrote", p)
