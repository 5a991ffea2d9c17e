"""Benchmark of the B200 radix sort / GSD sample sort (arXiv 1808.10292 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Workload (default, BASELINE.json configs[3]): n = 2^31 uint32 keys, uniform over
[0, 2^32) from seed 4 (SplitMix64 counter stream, inputs/), radix-256.  N = 1:
single-GPU LSD radix sort of all 2^31 keys; N > 1 (torchrun, one rank per GPU):
rank k holds keys [k·n/N, (k+1)·n/N) and the ranks run GSD with oversampling
r = 8 (s = 8N samples per rank) over NCCL.  A step = one full sort of the
workload (K1 histogram, K2 plan, 4 radix passes [, GSD sample / splitters /
split / all-to-all / merge]).  Inputs are larger than L2, so no flush is needed.

Prints ONE JSON line (rank 0).  `--impl reference` times the serial C oracle
(oracle/, the paper's SR4) on the host instead, on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (kind, n_total, seed, dist, digit_bits, description)
    "c4": ("u32", 1 << 31, 4, "uniform", 8, "BASELINE configs[3]: 2^31 u32 uniform seed 4, radix-256, GSD r=8 over N GPUs"),
    "c3": ("u32", 1 << 27, 3, "uniform", 8, "BASELINE configs[2] (uniform): 2^27 u32 seed 3, radix-256"),
    "c2": ("u32", 1 << 24, 2, "half", 8, "BASELINE configs[1]: 2^24 u32 in [0,2^31) seed 2, radix-256"),
    "c1": ("u32", 1 << 20, 1, "uniform", 8, "BASELINE configs[0]: 2^20 u32 uniform seed 1, radix-256"),
    "c2b16": ("u32", 1 << 24, 2, "half", 16, "BASELINE configs[1]: 2^24 u32 in [0,2^31) seed 2, radix-65536"),
    "c5": ("pairs", 1 << 30, 5, "uniform", 8, "BASELINE configs[4]: 2^30 (u64 key, u32 index) pairs seed 5, radix-256"),
}
BYTES_PER_KEY_PASS = {"u32": 8, "pairs": 24}      # algorithmic bytes of one pass (read + write)
KEY_BYTES = {"u32": 4, "pairs": 8}
PASSES = {("u32", 8): 4, ("u32", 16): 2, ("pairs", 8): 8}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 5 ms during the
    timed region through NVML (the data nvidia-smi's clocks query reports)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples = []
        self.smax = None
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                         pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except Exception:
                    pass
                self._stop.wait(0.005)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": [], "samples": 0, "source": "nvml"}
        sm = [s for s, _ in self.samples]
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r & bit for _, r in self.samples))
        loaded = [x for x in sm if x > 0.5 * (self.smax or max(sm))] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.smax, "sm_min_mhz": min(sm),
                "reasons": reasons, "samples": len(sm), "source": "nvml, 5 ms"}


def host_info():
    info = {"cores": os.cpu_count()}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu"] = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                info["mem_gb"] = round(int(ln.split()[1]) / 2 ** 20, 1)
    except Exception:
        pass
    return info


def bind_gpu_local_cpus(device_index: int):
    """Run on the host CPUs of the GPU's NUMA node (sysfs local_cpulist of its PCI
    device), so pinned host buffers are first-touched on that node and the e2e
    copies do not cross the socket interconnect.  Best effort; returns the CPU list."""
    try:
        import pynvml
        pynvml.nvmlInit()
        bus = pynvml.nvmlDeviceGetPciInfo(pynvml.nvmlDeviceGetHandleByIndex(device_index)).busId
        bus = (bus.decode() if isinstance(bus, bytes) else bus).lower()
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/local_cpulist"
        cpus = set()
        for part in open(path).read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return sorted(cpus)
    except Exception:
        pass
    return None


# ------------------------------------------------------- device-side verification
_GOLD = 0x9E3779B97F4A7C15


def _s64(c):  # unsigned 64-bit constant as a signed int64 (torch wraps on overflow)
    return c - (1 << 64) if c >= 1 << 63 else c


def _mix(x):
    """SplitMix64 finaliser on an int64 tensor (wrapping arithmetic, logical shifts)."""
    import torch
    def shr(v, k):
        return (v >> k) & ((1 << (64 - k)) - 1)
    x = x ^ shr(x, 30)
    x = x * _s64(0xBF58476D1CE4E5B9)
    x = x ^ shr(x, 27)
    x = x * _s64(0x94D049BB133111EB)
    return x ^ shr(x, 31)


def _as_u64(t):
    """keys as int64 carrying the unsigned value's bits (u32 zero-extended)"""
    import torch
    return t.to(torch.int64) & 0xFFFFFFFF if t.dtype == torch.int32 else t


def multiset_hash(keys, vals=None, chunk=1 << 26):
    """(count, Σ mix(x), Σ mix(x + φ)) mod 2^64 over the (key[, value]) multiset."""
    import torch
    h1 = torch.zeros((), dtype=torch.int64, device=keys.device)
    h2 = torch.zeros_like(h1)
    for i in range(0, keys.numel(), chunk):
        x = _as_u64(keys[i:i + chunk])
        if vals is not None:
            x = x ^ _mix(vals[i:i + chunk].to(torch.int64) & 0xFFFFFFFF)
        h1 += _mix(x).sum()
        h2 += _mix(x + _s64(_GOLD)).sum()
    return [keys.numel(), int(h1), int(h2)]


def order_violations(keys, vals=None, chunk=1 << 26):
    """# adjacent inversions (unsigned order); with vals (= global index), also
    # equal-key pairs whose values do not increase (stability)"""
    import torch
    bad = 0
    n = keys.numel()
    for i in range(0, max(n - 1, 0), chunk):
        x = _as_u64(keys[i:min(i + chunk + 1, n)])
        if keys.dtype == torch.int64:
            x = x ^ _s64(1 << 63)  # unsigned order as signed order
        bad += int((x[1:] < x[:-1]).sum())
        if vals is not None:
            v = vals[i:min(i + chunk + 1, n)].to(torch.int64) & 0xFFFFFFFF
            bad += int(((x[1:] == x[:-1]) & (v[1:] <= v[:-1])).sum())
    return bad


def rank_boundary_violations(edges):
    """edges[j] = (first, last) key of Y_j as int64 bit patterns, or (None, None)
    for an empty Y_j; counts ranks whose first key is below the last key of the
    nearest nonempty rank before it, in unsigned order"""
    bad, last = 0, None
    for fe, le in edges:
        if fe is None:
            continue
        if last is not None and (fe & ((1 << 64) - 1)) < last:
            bad += 1
        last = le & ((1 << 64) - 1)
    return bad


def verify_output(out, vout, comm, n_out, pristine, vals_pristine, kind, p, n_total, dist, dev):
    """the last timed step's output, checked on the device against the pristine
    input: nondecreasing (pairs: stable), same multiset (count + two SplitMix64
    sums), and across ranks the boundary last(Y_j) <= first(Y_{j+1})"""
    import torch
    res_k = out if comm is None else out[: n_out]
    res_v = (vout if comm is None else vout[: n_out]) if kind == "pairs" else None
    torch.cuda.synchronize()
    h_in = multiset_hash(pristine, vals_pristine)
    h_out = multiset_hash(res_k, res_v)
    viol = order_violations(res_k, res_v)
    edges = [None, None]
    if res_k.numel():
        edges = [int(_as_u64(res_k[:1])[0]), int(_as_u64(res_k[-1:])[0])]
    if p > 1:
        t = torch.tensor([h_in[1], h_in[2], h_out[1], h_out[2], h_out[0], viol], dtype=torch.int64, device=dev)
        dist.all_reduce(t)  # wrapping sums of the per-rank hashes and counts
        h_in = [n_total, int(t[0]), int(t[1])]
        h_out = [int(t[4]), int(t[2]), int(t[3])]
        viol = int(t[5])
        allg = [None] * p
        dist.all_gather_object(allg, edges)
        viol += rank_boundary_violations(allg)
    verified = viol == 0 and h_in == h_out
    verify = {"method": "device: adjacent order" + (" + stability (value = global index)" if kind == "pairs" else "") +
                        (" + rank boundaries" if p > 1 else "") + "; multiset (count, two SplitMix64 sums) vs the "
                        "pristine input", "violations": viol, "multiset_equal": h_in == h_out}
    return verified, verify


def oracle_baseline(kind, seed, dist, b, target_s=10.0):
    """The serial C oracle (SR-b) as it stands, built with gcc
    -O3 -march=native on this host, on a bounded sample of the workload's stream,
    one host core, until >= target_s elapsed."""
    import inputs
    import oracle
    flags = oracle.use_native()
    n = 1 << 25
    if kind == "u32":
        a = inputs.gen_u32(n, seed, dist)
        vals = None
    else:
        a = inputs.gen_u64(n, seed, dist)
        vals = inputs.iota_u32(n)
    done, t_total = 0, 0.0
    prev = os.sched_getaffinity(0)
    core = min(prev)
    os.sched_setaffinity(0, {core})  # the serial oracle pinned to one host core
    try:
        while t_total < target_s:
            t0 = time.perf_counter()
            if vals is None:
                oracle.sr(a, b)
            else:
                oracle.sr(a, b, vals=vals)
            t_total += time.perf_counter() - t0
            done += n
    finally:
        os.sched_setaffinity(0, prev)
    return {"value": done / t_total / 1e9, "unit": "Gkeys/s", "cores": 1, "kind": "oracle", "core": core,
            "flags": f"gcc {flags}",
            "sample": f"first 2^25 keys of the workload stream (seed {seed}, {dist}), serial SR-{b} oracle "
                      f"(oracle/sr.c, gcc {flags}), pinned to core {core}, {done // n} repetition(s), {t_total:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle on the host (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind, n_total, seed, dist, b, desc = CONFIGS[args.config]
    import inputs
    import oracle
    flags = oracle.use_native()
    n = 1 << 25 if kind == "u32" else 1 << 24
    a = inputs.gen_u32(n, seed, dist) if kind == "u32" else inputs.gen_u64(n, seed, dist)
    vals = inputs.iota_u32(n) if kind == "pairs" else None
    core = min(os.sched_getaffinity(0))
    os.sched_setaffinity(0, {core})  # one host core, as the "cores" field says
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.sr(a, b) if vals is None else oracle.sr(a, b, vals=vals)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    v = n / t / 1e9
    sample = (f"first 2^{n.bit_length() - 1} keys of the workload stream per step, serial SR-{b} oracle "
              f"(gcc {flags}), pinned to core {core}")
    print(json.dumps({
        "impl": "reference", "metric": "sorted keys/sec", "value": round(v, 6), "unit": "Gkeys/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32" if kind == "u32" else "u64+u32",
        "data": "synthetic", "config": {"workload": args.config, "description": desc, "sample_keys": n},
        "cpu_baseline": {"value": round(v, 6), "unit": "Gkeys/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "flags": f"gcc {flags}"},
        "e2e": {"value": round(v, 6), "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": host_info()}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--e2e-slots", type=int, default=3,
                    help="single GPU e2e: device buffer sets pipelined on their own streams (H2D of later "
                         "steps overlaps the sort and D2H of earlier ones)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="single GPU: also time the sort replayed from a CUDA graph (rs.SortGraph)")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the device-side check of the output (profiling runs: keeps the launch list to the sort)")
    ap.add_argument("--sampling", default="gsd", choices=["gsd", "ger", "gvr", "pr4", "btn", "oet"],
                    help="N > 1: sample sort of the paper's §3.3 (GSD regular oversampling r=8, default; "
                         "GER / GVR random oversampling with the paper's s), or the comparison paths "
                         "PR4 across GPUs / BTN / OET (PAPER.md:471-535, 685-709)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import inputs
    import paper_1808_10292_b200 as rs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    local_cpus = bind_gpu_local_cpus(torch.cuda.current_device())
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    kind, n_total, seed, dist_name, b, desc = CONFIGS[args.config]
    p = world
    lo, hi = rank * n_total // p, (rank + 1) * n_total // p
    n = hi - lo
    L = rs.lib()

    # ---- inputs resident in HBM: pristine copy + working buffer
    host_keys = torch.empty(n, dtype=torch.int32 if kind == "u32" else torch.int64, pin_memory=True)
    if kind == "u32":
        inputs.gen_u32(n, seed, dist_name, start=lo, n_total=n_total, out=host_keys.data_ptr())
    else:
        inputs.gen_u64(n, seed, dist_name, start=lo, out=host_keys.data_ptr())
    pristine = host_keys.to(dev, non_blocking=False)
    work = torch.empty_like(pristine)
    vals_pristine = vals_work = None
    if kind == "pairs":
        hv = torch.empty(n, dtype=torch.int32, pin_memory=True)
        inputs.iota_u32(n, start=lo, out=hv.data_ptr())
        vals_pristine = hv.to(dev)
        vals_work = torch.empty_like(vals_pristine)
    comm = rs.Comm() if p > 1 else None
    if comm is not None:
        comm.set_oversampling(8)
        comm.set_sampling(args.sampling, s=0, seed=seed)
        cap = comm.capacity(n)
        out = torch.empty(cap, dtype=work.dtype, device=dev)
        vout = torch.empty(cap, dtype=torch.int32, device=dev) if kind == "pairs" else None
        ws = torch.empty(rs.workspace_bytes(KEY_BYTES[kind], 4 if kind == "pairs" else 0, comm.ws_n(n), b, comm),
                         dtype=torch.uint8, device=dev)
    else:
        out = work
        vout = vals_work
        ws = torch.empty(rs.workspace_bytes(KEY_BYTES[kind], 4 if kind == "pairs" else 0, n, b),
                         dtype=torch.uint8, device=dev)

    out_cap = out.numel()

    comm_n_out = [n]

    def one_sort():
        if kind == "u32":
            r = rs.sort(work, digit_bits=b, comm=comm, out=out, ws=ws, out_cap=out_cap)
            comm_n_out[0] = r.numel()
            return r
        r = rs.sort_pairs(work, vals_work, digit_bits=b, comm=comm, out_keys=out, out_vals=vout, ws=ws,
                          out_cap=out_cap)
        comm_n_out[0] = r[0].numel()
        return r

    def barrier():
        if p > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # inputs smaller than L2 (c1-c3 single GPU): flush L2 after every reset by
    # writing a buffer twice its size, outside the timed region
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    in_bytes = n * (KEY_BYTES[kind] + (4 if kind == "pairs" else 0))
    flush = torch.empty(2 * l2_bytes, dtype=torch.uint8, device=dev) if 2 * in_bytes < 4 * l2_bytes else None

    def reset():
        work.copy_(pristine)
        if vals_work is not None:
            vals_work.copy_(vals_pristine)
        if flush is not None:
            flush.fill_(1)

    # ---- warm-up (includes a full GSD exchange when p > 1: NCCL connects lazily)
    for _ in range(args.warmup):
        reset()
        barrier()
        one_sort()
    barrier()

    # ---- timed steps: inputs reset outside the timed region (between the step events).
    # One GPU: the K steps issued back to back inside one barrier + synchronize bracket,
    # each step's reset (input restore, L2 flush) before its start event, so the device
    # does not idle on the host's per-call launch latency.  GSD (p > 1) synchronises
    # the host once per call: each step bracketed on its own.  No per-kernel timing
    # events here (they put a bubble at every kernel boundary); the kernel times for
    # the roofline come from a second, separately timed set of K steps below.
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run_steps(k):
        ms, nl = [], 0
        if p == 1:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
            barrier()
            c0 = L.rs_launch_count()
            for a, z in ev:
                reset()
                a.record()
                one_sort()
                z.record()
            barrier()
            return [a.elapsed_time(z) for a, z in ev], L.rs_launch_count() - c0
        for _ in range(k):
            reset()
            barrier()
            c0 = L.rs_launch_count()
            e0.record()
            one_sort()
            e1.record()
            barrier()
            nl += L.rs_launch_count() - c0
            ms.append(e0.elapsed_time(e1))
        return ms, nl

    with ClockSampler(torch.cuda.current_device()) as clk:
        step_ms, launches = run_steps(args.steps)
    clocks = clk.summary()

    # ---- the last timed step's output, checked on the device against the pristine
    # input: nondecreasing (pairs: stable), same multiset (count + two SplitMix64
    # sums), and across ranks the boundary last(Y_j) <= first(Y_{j+1})
    verified, verify = None, {"method": "skipped (--no-verify)"}
    if not args.no_verify:
        verified, verify = verify_output(out, vout, comm, comm_n_out[0], pristine, vals_pristine, kind, p, n_total,
                                         dist, dev)
    # ---- per-kernel device times (K3's average launch for the roofline, the exchange
    # for nvlink_roofline): K more steps with an event pair around every launch
    L.rs_timing_reset()
    L.rs_timing_enable(1)
    run_steps(args.steps)
    L.rs_timing_enable(0)
    # ---- optional (--graph, single GPU): the same sort captured once in a CUDA graph
    # (rs.SortGraph) and replayed, same reset / flush / bracketing; its output is
    # verified like the direct one's
    graph = None
    if args.graph and p == 1:
        try:
            reset()
            sg = rs.SortGraph(work, vals_work, digit_bits=b)
            g_ms = []
            for _ in range(args.warmup):
                reset()
                sg.replay()
            for _ in range(args.steps):
                reset()
                barrier()
                e0.record()
                sg.replay()
                e1.record()
                barrier()
                g_ms.append(e0.elapsed_time(e1))
            gms = sum(g_ms) / len(g_ms)
            graph = {"value": round(n_total / (gms / 1e3) / 1e9, 4), "unit": "Gkeys/s", "ms_per_step": round(gms, 4),
                     "kernels_per_replay": sg.launches,
                     "note": "rs.SortGraph: the sort captured once in a CUDA graph, replayed per step"}
            if not args.no_verify:
                graph["verified"], graph["verify"] = verify_output(out, vout, comm, n, pristine, vals_pristine, kind,
                                                                   p, n_total, dist, dev)
        except Exception as e:  # reported, not fatal: the direct numbers stand
            graph = {"error": f"{type(e).__name__}: {e}"}
    ms_q, cnt_q = ctypes.c_double(), ctypes.c_int()
    # the dominant kernel: the radix-256 pass, or the radix-65536 scatter (its count,
    # total, scan and offsets kernels are timed separately and are not in launch_ms)
    L.rs_timing_query(b"r16_scatter" if b == 16 else b"onesweep", ctypes.byref(ms_q), ctypes.byref(cnt_q))
    pass_ms = ms_q.value / max(cnt_q.value, 1)
    L.rs_timing_query(b"", ctypes.byref(ms_q), ctypes.byref(cnt_q))
    all_kernels_ms = ms_q.value
    # GSD all-to-all (N > 1): bytes that cross NVLink from the count matrix, time of
    # the grouped send/recv from events on the sort stream (max over ranks below)
    xchg = None
    if p > 1 and args.sampling in ("gsd", "ger", "gvr"):
        L.rs_timing_query(b"gsd_exchange", ctypes.byref(ms_q), ctypes.byref(cnt_q))
        pulled = cnt_q.value == 0  # pull merge: the transfer is the first merge level's NVLink reads
        if pulled:
            L.rs_timing_query(b"gsd_pull_merge", ctypes.byref(ms_q), ctypes.byref(cnt_q))
        x_ms = ms_q.value / max(cnt_q.value, 1)
        cm = comm.last_counts().astype(np.float64)
        w = KEY_BYTES[kind] + (4 if kind == "pairs" else 0)
        sent = (cm[rank].sum() - cm[rank, rank]) * w
        recv = (cm[:, rank].sum() - cm[rank, rank]) * w
        t = torch.tensor([x_ms, max(sent, recv)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        x_ms, x_bytes = float(t[0]), float(t[1])
        nvl_peak = 770.0
        ach = x_bytes / (x_ms / 1e3) / 1e9 if x_ms > 0 else None
        xchg = {"kernel": ("pull merge: merge tree whose first level reads the peers' blocks over NVLink "
                           "(CUDA IPC); time = the whole merge" if pulled
                           else "grouped ncclSend/ncclRecv all-to-all (GSD step 4)"), "bound": "nvlink",
                "bytes_max_rank": int(x_bytes), "ms": round(x_ms, 4),
                "achieved": round(ach, 1) if ach else None, "peak": nvl_peak, "unit": "GB/s",
                "frac": round(ach / nvl_peak, 4) if ach else None,
                "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 GB/s nominal)"}
    total_ms = sum(step_ms)
    if p > 1:
        t = torch.tensor([total_ms, pass_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, pass_ms = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    value = n_total / (ms_per_step / 1e3) / 1e9

    # ---- e2e through the public API: pinned host keys -> device -> sort -> host.
    # Single GPU: several slots on their own streams, so later steps' uploads overlap
    # step i's sort and download (PCIe is full duplex).  GSD (p > 1): one slot (one NCCL
    # communicator, collectives issued in one order).
    e2e = None
    if args.e2e_steps > 0:
        nslot = args.e2e_slots if p == 1 else 1
        streams = [torch.cuda.Stream(device=dev) for _ in range(nslot)]
        slots = [dict(work=work, vals=vals_work, out=out, vout=vout, ws=ws)]
        for _ in range(nslot - 1):
            slots.append(dict(work=torch.empty_like(work),
                              vals=torch.empty_like(vals_work) if vals_work is not None else None,
                              ws=torch.empty_like(ws)))
            slots[-1]["out"], slots[-1]["vout"] = slots[-1]["work"], slots[-1]["vals"]
        res_hosts = [torch.empty_like(host_keys, pin_memory=True) for _ in range(nslot)]

        def e2e_step(i):
            sl, st = slots[i % nslot], streams[i % nslot]
            with torch.cuda.stream(st):
                sl["work"].copy_(host_keys, non_blocking=True)
                if sl["vals"] is not None:
                    sl["vals"].copy_(hv, non_blocking=True)
                if kind == "u32":
                    res = rs.sort(sl["work"], digit_bits=b, comm=comm, out=sl["out"], ws=sl["ws"],
                                  out_cap=sl["out"].numel(), stream=st)
                else:
                    res, _ = rs.sort_pairs(sl["work"], sl["vals"], digit_bits=b, comm=comm, out_keys=sl["out"],
                                           out_vals=sl["vout"], ws=sl["ws"], out_cap=sl["out"].numel(), stream=st)
                res_hosts[i % nslot][: res.numel()].copy_(res, non_blocking=True)
                done = torch.cuda.Event()
                done.record(st)
            return done

        for i in range(nslot):  # warm every slot (first-touch, NCCL / probe setup)
            e2e_step(i)
        barrier()
        if p == 1:
            # steady-state throughput: W = nslot priming steps, then K timed steps, all
            # issued back to back; the clock starts when priming step W-1 has come
            # back to the host and stops when the last timed step has
            evs = [e2e_step(i) for i in range(nslot + args.e2e_steps)]
            evs[nslot - 1].synchronize()
            t0 = time.perf_counter()
            evs[-1].synchronize()
            torch.cuda.synchronize()
            e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        else:
            t0 = time.perf_counter()
            for i in range(args.e2e_steps):
                e2e_step(i)
            barrier()
            e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        if p > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        kb = KEY_BYTES[kind]
        e2e = {"value": round(n_total / (e_ms / 1e3) / 1e9, 4), "unit": "Gkeys/s",
               "h2d_bytes_per_step": n * (kb + (4 if kind == "pairs" else 0)), "d2h_bytes_per_step": n * kb,
               "ms_per_step": round(e_ms, 3), "steps": args.e2e_steps, "slots": nslot,
               "host_cpus": f"{len(local_cpus)} GPU-local CPUs" if local_cpus else "unbound",
               "note": "host clock over the steps: pinned H2D of the inputs + sort + D2H of the sorted keys "
                       f"every step; steps pipelined over {nslot} streams on one GPU; single GPU: clock from "
                       "the completion of the last priming step to that of the last timed step (max over ranks)"}

    if rank != 0:
        if p > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    bpk = BYTES_PER_KEY_PASS[kind]
    n_local = n
    achieved = bpk * n_local / (pass_ms / 1e3) / 1e9 if kind in BYTES_PER_KEY_PASS and pass_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{args.config}:p{p}")
    design, probe = ctypes.c_longlong(), ctypes.c_longlong()
    L.rs_dev_get_option(b"pass_design", ctypes.byref(design))
    L.rs_dev_get_option(b"rank_probe", ctypes.byref(probe))
    kname = ("k_onesweep_ar (design 5: atomic ranks)" if design.value == 5 and probe.value == 1
             else f"k_onesweep_* (design {design.value if design.value != 5 else 2})")
    if b == 16:
        kname = "k16_scatter (radix-65536 pass: the scatter kernel"
    roofline = {"kernel": kname + (", one count-sort pass" if b == 8 else "; reads and writes every key)"),
                "bound": "hbm",
                "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None, "traffic": traffic,
                "algorithmic_bytes_per_launch": bpk * n_local, "launch_ms": round(pass_ms, 4),
                "peak_source": peak_src,
                "pass_share_of_step": round(pass_ms * PASSES.get((kind, b), 4) / ms_per_step, 4)}
    cpu = None
    if not args.no_cpu_baseline:
        cpu = oracle_baseline(kind, seed, dist_name, b)
        cpu["host"] = host_info()
    line = {
        "metric": "sorted keys/sec", "value": round(value, 4), "unit": "Gkeys/s", "n_gpus": p,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32" if kind == "u32" else "u64+u32", "data": "synthetic",
        "config": {"workload": args.config, "description": desc, "n": n_total, "keys_per_gpu": n,
                   "digit_bits": b, "seed": seed, "dist": dist_name,
                   "parallelism": (f"gsd-p{p} (r=8)" if args.sampling == "gsd" else
                                   f"{args.sampling}-p{p} (paper's s)" if args.sampling in ("ger", "gvr") else
                                   f"{args.sampling}-p{p}")
                   if p > 1 else "single GPU",
                   "l2": ("L2 flushed before every step (2x L2 write)" if flush is not None
                          else "inputs larger than L2 (no flush)"), "l2_bytes": l2_bytes,
                   "inputs": "resident in HBM, reset outside timed region",
                   "timing": ("CUDA events around each sort; the K steps issued back to back inside one "
                              "barrier + synchronize bracket, resets between the event pairs" if p == 1 else
                              "CUDA events around each sort, each step bracketed by barrier + synchronize, "
                              "max over ranks")},
        "verified": verified, "verify": verify,
        **({"graph_replay": graph} if graph is not None else {}),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        **({"nvlink_roofline": xchg} if xchg else {}),
        "clocks": clocks, "kernel_ms_per_step": round(all_kernels_ms / args.steps, 4),
        "step_ms_rank0": {"mean": round(statistics.mean(step_ms), 4), "median": round(statistics.median(step_ms), 4),
                          "min": round(min(step_ms), 4), "max": round(max(step_ms), 4)},
    }
    print(json.dumps(line))
    if p > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
