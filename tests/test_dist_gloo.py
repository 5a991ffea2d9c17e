"""Multi-process (gloo, CPU) coverage of GSD's N > 1 host logic: the exchange
plan from the all-gathered p×p count matrix (rs_gsd_exchange_plan, the same
function the NCCL path calls), the all-to-all it drives, capacity errors raised
identically on every rank, and the max-over-ranks sizing helper.  Local sorting
and counting are done with the oracle (the device kernels are covered by
tests/test_gpu_gsd.py); the exchange itself runs over gloo send/recv."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cut_counts(xs, rank, splitters):
    """|X_{k,j}| for sorted block xs of rank k under composite splitters (R14)."""
    n = xs.size
    cuts = [0]
    for (v, r, q) in splitters:
        if rank < r:
            cuts.append(int(np.searchsorted(xs, v, side="right")))
        elif rank > r:
            cuts.append(int(np.searchsorted(xs, v, side="left")))
        else:
            cuts.append(min(q + 1, n))
    cuts.append(n)
    return np.diff(np.array(cuts, dtype=np.int64)).astype(np.uint64)


def _worker(rank, world, port, total, r, result_q, cap_shrink):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import inputs
        import oracle
        import paper_1808_10292_b200 as rs
        lo, hi = rank * total // world, (rank + 1) * total // world
        keys = inputs.gen_u32(hi - lo, 7, "mod16" if total % 2 else "uniform", start=lo)
        # step 1: local sort (oracle stands in for the device sort here)
        xs = oracle.sr(keys, 8)
        N = xs.size
        # step 2: regular sample (R10) and all-gather
        s = r * world
        pos = [(N * i + s - 1) // s - 1 for i in range(1, s)] + [N - 1]
        samples = [(int(xs[q]), rank, q) for q in pos]
        gathered = [None] * world
        dist.all_gather_object(gathered, samples)
        T = sorted(c for part in gathered for c in part)
        splitters = [T[i * s - 1] for i in range(1, world)]
        # step 4: counts row + all-gather -> p×p matrix
        row = torch.from_numpy(_cut_counts(xs, rank, splitters).astype(np.int64))
        rows = [torch.zeros_like(row) for _ in range(world)]
        dist.all_gather(rows, row)
        counts = torch.stack(rows).numpy().astype(np.uint64)
        n_max = rs.max_over_ranks(N)
        cap = n_max + n_max // r + world if not cap_shrink else n_max - cap_shrink
        caps = np.full(world, cap, dtype=np.uint64)
        try:
            so, ro, tot = rs.exchange_plan(counts, rank, caps)
        except rs.RSortError as e:
            result_q.put((rank, "ECAPACITY" if e.status == 5 else str(e), None, None))
            return
        # the all-to-all the plan drives (gloo p2p in place of NCCL)
        recv = np.empty(tot, dtype=np.int32)
        reqs = []
        for j in range(world):
            seg = torch.from_numpy(xs[int(so[j]):int(so[j + 1])].view(np.int32).copy())
            if j == rank:
                recv[int(ro[j]):int(ro[j + 1])] = seg.numpy()
            elif seg.numel():
                reqs.append(dist.isend(seg, dst=j))
        bufs = {}
        for k in range(world):
            c = int(ro[k + 1] - ro[k])
            if k != rank and c:
                bufs[k] = torch.empty(c, dtype=torch.int32)
                reqs.append(dist.irecv(bufs[k], src=k))
        for q in reqs:
            q.wait()
        for k, b in bufs.items():
            recv[int(ro[k]):int(ro[k + 1])] = b.numpy()
        # step 5: merge (stable sort of the source-ordered runs)
        Y = oracle.sr(recv.view(np.uint32), 8)
        result_q.put((rank, "ok", Y, counts))
    finally:
        dist.destroy_process_group()


def _run(world, total, r, cap_shrink=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, total, r, q, cap_shrink)) for k in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("world,total", [(2, 30001), (2, 40000), (4, 50000)])
def test_gsd_exchange_over_gloo_matches_simulator(world, total):
    import inputs
    import oracle
    res = _run(world, total, r=8)
    assert all(st == "ok" for _, st, _, _ in res)
    Y = np.concatenate([y for _, _, y, _ in res])
    full = inputs.gen_u32(total, 7, "mod16" if total % 2 else "uniform")
    assert (Y == np.sort(full)).all()
    shards = [full[k * total // world:(k + 1) * total // world] for k in range(world)]
    sim = oracle.gsd(shards, r=8)
    for _, _, y, counts in res:
        assert counts.tolist() == sim["counts"].tolist()
    for j in range(world):
        assert (res[j][2] == sim["Y"][j]).all()


def test_capacity_error_on_every_rank():
    # capacity below n/p: some rank must overflow; all ranks must fail alike
    res = _run(2, 40000, r=8, cap_shrink=100)
    assert [st for _, st, _, _ in res] == ["ECAPACITY", "ECAPACITY"]
