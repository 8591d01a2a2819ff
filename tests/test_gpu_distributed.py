"""Two ranks on one B200 (gloo carries the collectives; the engine path is the real one).

Each rank owns half of the streams, runs phase 1 on the GPU, all-reduces the
last timestamp (truncated spans end at the GLOBAL last ts, pipeline.py:152),
finishes, and merges its dense tally rows with the other rank's through
ShardedRun.report -- the code bench.py --gpus N runs over NCCL.  The merged
report must equal the single-process oracle of the whole trace."""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _workload():
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec(f"n{i % 2}", P + 100 * (i % 3), P + 100 * (i % 3) + i, 4000 + 1301 * i, 8800 + i)
               for i in range(10)]
    # unclosed calls (truncation at the global last ts), orphans and device records with per-rank names
    return synth.Workload("dist", synth.ze_registry(), streams,
                          dict(close_at_end=0, orphan_p=0.01, prof_p=0.3, max_depth=6),
                          kernel_names=synth.kernel_pool(40))


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_03683_b200 import synth
        from paper_2504_03683_b200.distributed import ShardedRun
        from paper_2504_03683_b200.engine import Engine

        wl = _workload()
        raws = synth.generate(wl)
        mine = raws[rank::world]
        eng = Engine(device=0)
        eng.set_registry(wl.registry)
        eng.set_streams(mine)
        eng.stage()
        run = ShardedRun(eng, wl.registry, world_size=world, rank=rank)
        info = run.step()
        rep = run.report([r.info for r in mine])
        if rank == 0:
            from oracle import oracle

            want = oracle.run(raws, wl.registry, [r.info for r in raws])
            q.put((rep == want.report, info["rc"], run.global_last_ts == want.last_ts, len(want.report.rows),
                   eng.last_path()[0]))
        eng.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_gpu_merge_equals_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs)
    same, rc, last_ok, n_rows, path = q.get(timeout=10)
    assert rc == 0 and last_ok and n_rows > 10 and path == 1
    assert same
