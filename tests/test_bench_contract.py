"""bench.py's contract on a host without a GPU: the reference arm (the serial
oracle on one host core) prints one well-formed JSON line, other ranks of a
torchrun launch print nothing, and our arm fails loudly instead of falling back
to the CPU."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=e, cwd=ROOT)


def test_reference_arm_json_line():
    r = _bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "sorted keys/sec" and d["unit"] == "Gkeys/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["value"] == d["value"] and "sample" in d["cpu_baseline"]
    assert d["e2e"] == {"value": d["value"], "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "c1"


def test_reference_arm_other_ranks_silent():
    r = _bench("--impl", "reference", "--config", "c1", "--steps", "1", env={"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure")
def test_our_arm_fails_loudly_without_gpu():
    r = _bench("--config", "c1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "0")
    assert r.returncode != 0
    assert not any(ln.startswith("{") for ln in r.stdout.splitlines())


def test_rank_boundary_violations_unsigned():
    """the cross-rank order check of bench.py's verification (N > 1): unsigned
    order over int64 bit patterns, empty ranks skipped"""
    sys.path.insert(0, ROOT)
    import bench
    top = -(1 << 63)  # the bit pattern of 2^63
    ok = [(0, 5), (None, None), (7, (1 << 63) - 1), (top, top + 3), (-2, -1)]  # ..., 2^63, 2^64-2
    assert bench.rank_boundary_violations(ok) == 0
    assert bench.rank_boundary_violations([(0, 9), (8, 10)]) == 1
    assert bench.rank_boundary_violations([(top, top), (5, 6)]) == 1  # 5 < 2^63 unsigned
    assert bench.rank_boundary_violations([(None, None), (3, 4), (None, None), (4, 4)]) == 0


def test_multiset_hash_and_order_on_host_tensors():
    """bench.py's device checks are plain torch ops: on host tensors a sorted
    permutation has the input's hash and no violations; a changed key or an
    inversion is caught (u32 as int32 bit patterns, pairs with stability)"""
    sys.path.insert(0, ROOT)
    import bench
    g = torch.Generator().manual_seed(1)
    x = torch.randint(-2 ** 31, 2 ** 31 - 1, (5000,), dtype=torch.int32, generator=g)
    s = torch.from_numpy(np.sort(x.numpy().view(np.uint32)).view(np.int32))  # unsigned order
    assert bench.multiset_hash(s) == bench.multiset_hash(x)
    assert bench.order_violations(s) == 0
    t = s.clone()
    t[10] += 1
    assert bench.multiset_hash(t) != bench.multiset_hash(x)
    t = s.clone()
    t[[3, 4]] = t[[4, 3]]
    assert bench.order_violations(t) == (1 if int(s[3]) != int(s[4]) else 0)
    k = torch.tensor([5, 5, -1, -1], dtype=torch.int64)  # -1 = 2^64-1: last in unsigned order
    v = torch.tensor([0, 1, 2, 3], dtype=torch.int32)
    assert bench.order_violations(k, v) == 0
    assert bench.order_violations(k, torch.tensor([1, 0, 2, 3], dtype=torch.int32)) == 1
