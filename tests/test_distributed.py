"""Multi-rank merge over torch.distributed (gloo, world_size 2, CPU).

Each rank takes half of the streams of a synthetic trace, computes its local
tally rows (with the CPU oracle standing in for the GPU engine's dense
output), and the ranks merge them with the same code the GPU path uses over
NCCL (paper_2504_03683_b200.distributed.merge_dense).  The merged rows must
equal the single-process tally of the whole trace; the global-last-timestamp
all-reduce that truncation needs is checked the same way."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2504_03683_b200 import synth
        from paper_2504_03683_b200.distributed import merge_dense, torch_all_reduce

        wl = synth.config("c2", 0.0003)
        raws = synth.generate(wl)
        mine = raws[rank::world]
        local = oracle.run(mine, wl.registry, [r.info for r in mine])
        rows = {k: (r.count, r.error_count, r.time_ns, r.min_ns, r.max_ns) for k, r in local.report.rows.items()}
        gathered = [None] * world
        dist.all_gather_object(gathered, sorted(rows))
        keys = sorted({k for g in gathered for k in g})
        merged = merge_dense(rows, keys, torch_all_reduce())
        t = torch.tensor([local.last_ts - (1 << 63)], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            full = oracle.run(raws, wl.registry, [r.info for r in raws])
            want = {k: (r.count, r.error_count, r.time_ns, r.min_ns, r.max_ns) for k, r in full.report.rows.items()}
            q.put((merged == want, t.item() + (1 << 63) == full.last_ts, len(want)))
    finally:
        dist.destroy_process_group()


def test_two_rank_merge_equals_single_pass():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    rows_equal, last_equal, n = q.get(timeout=10)
    assert rows_equal and last_equal and n > 10


def test_limbs_round_trip():
    from paper_2504_03683_b200.distributed import limbs, unlimbs

    for v in (0, 1, -1, 2**64 - 1, 2**64, -(2**70) + 12345, 2**100 + 7):
        assert unlimbs(*limbs(v)) == v
