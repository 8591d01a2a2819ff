"""Multi-rank host logic over torch.distributed (gloo, world_size 2, CPU).

`run_pipeline(..., distributed=True)` on every rank, with tests/fake_engine.FakeEngine (the CPU
oracle over the rank's streams + a numpy restatement of csrc/merge.cu's buffer layout) in place of
the GPU engine: the partitioner, the last-ts / status exchange, the device-name agreement, the
SUM/MAX merge, the orphan gathering and the first-error reconciliation all run for real.  Every
rank's result must equal the single-process oracle of the whole trace."""

import os
import socket
import tempfile

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _workload(orphan_p=0.01):
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec(f"n{i % 3}", P + 100 * (i % 4), P + 100 * (i % 4) + i, 300 + 97 * i, 700 + i)
               for i in range(9)]
    # unclosed calls (truncation at the GLOBAL last ts), orphans, device names that differ per rank
    return synth.Workload("dist", synth.ze_registry(), streams,
                          dict(close_at_end=0, orphan_p=orphan_p, prof_p=0.3, max_depth=6),
                          kernel_names=synth.kernel_pool(30))


def _generate():
    """The workload with the last records of every third stream cut off: open calls are flushed as
    truncated spans at the GLOBAL last timestamp (pipeline.py:152, :235)."""
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.pipeline import _walk
    from paper_2504_03683_b200.tracefile import RawStream, StreamInfo

    wl = _workload()
    raws = synth.generate(wl)
    for i in range(0, len(raws), 3):
        r = raws[i]
        offs = _walk(r)[0]
        keep = len(offs) - 3
        info = StreamInfo(r.hostname, r.pid, r.tid, keep, 0)
        raws[i] = RawStream(r.hostname, r.pid, r.tid, r.name, r.data[:offs[keep]], info)
    return wl, raws


def _corrupt(raws, which, k):
    """Record k of stream `which` gets an unknown schema id (UnknownSchemaError mid-stream)."""
    from paper_2504_03683_b200.pipeline import _walk
    from paper_2504_03683_b200.tracefile import RawStream

    r = raws[which]
    at = _walk(r)[0][k]
    data = bytearray(r.data)
    data[at:at + 4] = b"\xff\xff\xff\x7f"  # an unknown schema id in a record header
    raws[which] = RawStream(r.hostname, r.pid, r.tid, r.name, bytes(data), r.info)
    return raws


def _worker(rank, world, port, q, case, tmp):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world == 1:
        os.environ["HAPIGPU_COLLECTIVES"] = "1"  # the multi-rank protocol at world size 1
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from fake_engine import FakeEngine
        from paper_2504_03683_b200 import run_pipeline, synth
        from paper_2504_03683_b200.distributed import pack_exception
        from paper_2504_03683_b200.pipeline import Sink, TallySink
        from paper_2504_03683_b200.tracefile import open_trace_reader

        class Diag(Sink):
            name = "diag"

            def on_diagnostics(self, orphans):
                self.orphans = orphans

        wl, raws = _generate()
        if case == "corrupt":
            raws = _corrupt(raws, 5, 40)
        if case == "few":  # more ranks than streams: some ranks own nothing
            raws = raws[:2]
        d = os.path.join(tmp, "trace")
        if rank == 0:
            synth.write(wl, raws, d)
        dist.barrier()
        if case == "header" and rank == 0:
            f = os.path.join(d, raws[6].name)
            b = bytearray(open(f, "rb").read())
            b[0] ^= 1
            open(f, "wb").write(bytes(b))
        dist.barrier()
        eng = FakeEngine(fail_run=(case == "engine" and rank == 1))
        diag = Diag()
        try:
            res = run_pipeline(open_trace_reader(d), [TallySink(), diag], engine=eng, distributed=True)
            out = ("ok", res["tally"], vars(res.stats), res.orphans, diag.orphans)
        except Exception as e:  # noqa: BLE001
            out = ("raised", pack_exception(e), getattr(diag, "orphans", None))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    with tempfile.TemporaryDirectory() as tmp:
        procs = [ctx.Process(target=_worker, args=(r, world, port, q, case, tmp)) for r in range(world)]
        for p in procs:
            p.start()
        outs = dict(q.get(timeout=300) for _ in procs)
        for p in procs:
            p.join(timeout=60)
        assert all(p.exitcode == 0 for p in procs)
    return outs


def _oracle(case):
    from oracle import oracle
    from paper_2504_03683_b200 import synth

    wl, raws = _generate()
    if case == "corrupt":
        raws = _corrupt(raws, 5, 40)
    if case == "few":
        raws = raws[:2]
    return oracle.run(raws, wl.registry, [r.info for r in raws])


def test_two_ranks_tally_stats_orphans_equal_single_process():
    outs = _run("clean")
    want = _oracle("clean")
    assert want.error is None and want.stats["truncated_spans"] > 0 and want.stats["orphan_exits"] > 0
    for rank in (0, 1):
        kind, rep, stats, orphans, diag = outs[rank]
        assert kind == "ok"
        assert rep == want.report
        assert stats == want.stats
        assert orphans == want.orphans == diag


def test_two_ranks_raise_the_reference_first_error():
    outs = _run("corrupt")
    want = _oracle("corrupt")
    assert want.error is not None
    from paper_2504_03683_b200.distributed import unpack_exception

    for rank in (0, 1):
        kind, packed, diag = outs[rank]
        assert kind == "raised"
        e = unpack_exception(packed)
        assert type(e).__name__ == type(want.error).__name__ and str(e) == str(want.error)
        assert diag == want.orphans


def test_two_ranks_file_header_error_reaches_every_rank():
    outs = _run("header")
    from paper_2504_03683_b200.distributed import unpack_exception

    texts = set()
    for rank in (0, 1):
        kind, packed, _ = outs[rank]
        assert kind == "raised"
        e = unpack_exception(packed)
        assert type(e).__name__ == "CorruptRecordError" and "bad magic" in str(e)
        texts.add(str(e))
    assert len(texts) == 1


def test_engine_failure_on_one_rank_stops_both():
    outs = _run("engine")
    from paper_2504_03683_b200.distributed import unpack_exception

    for rank in (0, 1):
        kind, packed, _ = outs[rank]
        assert kind == "raised"
        assert "injected engine failure" in str(unpack_exception(packed))


def test_four_ranks_two_streams_idle_ranks_still_agree():
    """World size 4 over a 2-stream trace: two ranks own no stream, all four return the whole result."""
    outs = _run("few", world=4)
    want = _oracle("few")
    for rank in range(4):
        kind, rep, stats, orphans, diag = outs[rank]
        assert kind == "ok" and rep == want.report and stats == want.stats and orphans == want.orphans


@pytest.mark.parametrize("case", ["clean", "corrupt"])
def test_one_rank_through_the_collectives(case):
    """World size 1 with the multi-rank protocol forced (split run, merge buffer, error exchange)."""
    outs = _run(case, world=1)
    want = _oracle(case)
    if case == "corrupt":
        from paper_2504_03683_b200.distributed import unpack_exception

        kind, packed, diag = outs[0]
        e = unpack_exception(packed)
        assert kind == "raised" and type(e).__name__ == type(want.error).__name__ and str(e) == str(want.error)
        assert diag == want.orphans
        return
    kind, rep, stats, orphans, diag = outs[0]
    assert kind == "ok" and rep == want.report and stats == want.stats and orphans == want.orphans == diag


def test_partition_lpt_balances_and_keeps_identities_together():
    from paper_2504_03683_b200.distributed import partition_streams

    sizes = [100, 90, 80, 70, 60, 50, 40, 30, 20, 10]
    parts = partition_streams(sizes, 3)
    assert sorted(i for p in parts for i in p) == list(range(10))
    loads = [sum(sizes[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(sizes) and all(p == sorted(p) for p in parts)
    keys = ["a", "a", "b", "c", "c", "c", "d", "e", "f", "g"]
    parts = partition_streams(sizes, 4, keys)
    owner = {i: r for r, p in enumerate(parts) for i in p}
    assert owner[0] == owner[1] and owner[3] == owner[4] == owner[5]
    assert partition_streams([], 2) == [[], []]


def test_exception_packing_round_trip():
    from paper_2504_03683_b200.distributed import pack_exception, unpack_exception
    from paper_2504_03683_b200.errors import CorruptRecordError, MuxOrderingError

    for e in (CorruptRecordError("truncated record header", "s.bin", 48), MuxOrderingError("s.bin", 7)):
        u = unpack_exception(pack_exception(e))
        assert type(u) is type(e) and str(u) == str(e) and vars(u) == vars(e)
