"""Two ranks on one B200 (gloo carries the collectives; the engine path is the real one).

Every rank calls run_pipeline(reader, ..., distributed=True): it reads only the stream files the LPT
partitioner gives it, runs phase 1 on the GPU, all-reduces [last ts, status] (truncated spans end at
the GLOBAL last ts, pipeline.py:152), composes, and merges its device-resident tally rows through
hg_merge_export / two all-reduces / hg_merge_import (csrc/merge.cu) -- the code bench.py --gpus N
runs over NCCL.  Every rank's report, IntervalStats and orphan list must equal the single-process
oracle of the whole trace; a corrupt record must raise the same exception on both ranks."""

import os
import socket
import tempfile

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _c5():
    from paper_2504_03683_b200 import synth

    wl = synth.config("c5", 0.0004)  # 256 call streams + the telemetry sampler stream
    return wl, synth.generate(wl)


def _worker(rank, world, port, q, case, tmp, backend="gloo"):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(0)
        os.environ["HAPIGPU_COLLECTIVES"] = "1"  # the multi-rank protocol at world size 1
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        from test_distributed import _corrupt, _generate
        from paper_2504_03683_b200 import run_pipeline, synth
        from paper_2504_03683_b200.distributed import pack_exception
        from paper_2504_03683_b200.engine import Engine
        from paper_2504_03683_b200.pipeline import Sink, TallySink
        from paper_2504_03683_b200.tracefile import open_trace_reader

        class Diag(Sink):
            name = "diag"

            def on_diagnostics(self, orphans):
                self.orphans = orphans

        wl, raws = _generate() if case != "c5" else _c5()
        if case == "corrupt":
            raws = _corrupt(raws, 5, 40)
        if case == "few":  # more ranks than streams: one rank owns nothing
            raws = raws[:2]
        d = os.path.join(tmp, "trace")
        if rank == 0:
            synth.write(wl, raws, d)
        dist.barrier()
        eng = Engine(device=0)
        diag = Diag()
        try:
            if case == "c5":  # the timeline merged across ranks (device spans, samples, metadata objects)
                from paper_2504_03683_b200 import TimelineSink

                res = run_pipeline(open_trace_reader(d), [TallySink(), TimelineSink(device_index=3)], engine=eng,
                                   distributed=True)
                eng.close()
                q.put((rank, ("ok", res["tally"], res["timeline"])))
                return
            if case == "ordered":  # timeline / pretty / validation: rank 0 serves them from the whole trace
                import json as _json

                from paper_2504_03683_b200 import PrettyPrintSink, TimelineSink, ValidationRules, ValidationSink
                from golden_util import GOLDEN

                rules = ValidationRules.from_dict(_json.loads((GOLDEN / "expected" / "validation_rules.json").read_text()))
                res = run_pipeline(open_trace_reader(d), [TallySink(), TimelineSink(), PrettyPrintSink(),
                                                          ValidationSink(rules=rules)], engine=eng, distributed=True)
                out = ("ok", res["tally"], res["timeline"], res["pretty"],
                       None if res["validate"] is None else [tuple(vars(f).values()) for f in res["validate"]])
                eng.close()
                q.put((rank, out))
                return
            res = run_pipeline(open_trace_reader(d), [TallySink(), diag], engine=eng, distributed=True)
            out = ("ok", res["tally"], vars(res.stats), res.orphans, diag.orphans, eng.last_path()[0])
        except Exception as e:  # noqa: BLE001
            out = ("raised", pack_exception(e), getattr(diag, "orphans", None))
        eng.close()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(case, world=2, backend="gloo"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    with tempfile.TemporaryDirectory() as tmp:
        procs = [ctx.Process(target=_worker, args=(r, world, port, q, case, tmp, backend)) for r in range(world)]
        for p in procs:
            p.start()
        outs = dict(q.get(timeout=600) for _ in procs)
        for p in procs:
            p.join(timeout=120)
        assert all(p.exitcode == 0 for p in procs)
    return outs


def _oracle(case):
    from oracle import oracle
    from test_distributed import _corrupt, _generate

    wl, raws = _generate()
    if case == "corrupt":
        raws = _corrupt(raws, 5, 40)
    if case == "few":
        raws = raws[:2]
    return oracle.run(raws, wl.registry, [r.info for r in raws])


def test_two_ranks_one_gpu_equal_single_process_oracle():
    outs = _run("clean")
    want = _oracle("clean")
    assert want.stats["truncated_spans"] > 0 and want.stats["orphan_exits"] > 0
    for rank in (0, 1):
        kind, rep, stats, orphans, diag, path = outs[rank]
        assert kind == "ok" and path == 1
        assert rep == want.report
        assert stats == want.stats
        assert orphans == want.orphans == diag


def test_three_ranks_two_streams_idle_rank():
    """A rank with no stream runs an empty engine pass and still returns the whole trace's result."""
    outs = _run("few", world=3)
    want = _oracle("few")
    for rank in range(3):
        kind, rep, stats, orphans, diag, _path = outs[rank]
        assert kind == "ok" and rep == want.report and stats == want.stats and orphans == want.orphans


def test_two_ranks_one_gpu_raise_the_reference_first_error():
    from paper_2504_03683_b200.distributed import unpack_exception

    outs = _run("corrupt")
    want = _oracle("corrupt")
    assert want.error is not None
    for rank in (0, 1):
        kind, packed, diag = outs[rank]
        assert kind == "raised"
        e = unpack_exception(packed)
        assert type(e).__name__ == type(want.error).__name__ and str(e) == str(want.error)
        assert diag == want.orphans


def test_two_ranks_ordered_sinks_served_by_rank0():
    """TimelineSink / PrettyPrintSink / ValidationSink in a distributed run: rank 0 returns what one GPU
    over the whole trace returns, the other ranks None; the tally is still the merged one."""
    import json

    from oracle import oracle
    from test_distributed import _generate

    from paper_2504_03683_b200 import ValidationRules
    from golden_util import GOLDEN

    outs = _run("ordered")
    wl, raws = _generate()
    want = oracle.run(raws, wl.registry, [r.info for r in raws], want_timeline=True)
    rules = ValidationRules.from_dict(json.loads((GOLDEN / "expected" / "validation_rules.json").read_text()))
    findings = oracle.validate(raws, wl.registry, rules, want.orphans)
    kind, rep, tl, pretty, val = outs[0]
    assert kind == "ok" and rep == want.report
    assert tl == json.loads(want.timeline) and pretty == oracle.pretty(raws, wl.registry)
    assert val == [tuple(f) for f in findings]
    kind, rep, tl, pretty, val = outs[1]
    assert kind == "ok" and rep == want.report and tl is None and pretty is None and val is None


def test_three_ranks_timeline_merged_across_ranks():
    """Collective (6): each rank's timeline messages (global stream keys, record payloads attached)
    merged and formatted by rank 0 -- equal to the single-process timeline of the whole trace."""
    import json

    from oracle import oracle

    outs = _run("c5", world=3)
    wl, raws = _c5()
    want = oracle.run(raws, wl.registry, [r.info for r in raws], want_timeline=True, device_index=3)
    kind, rep, tl = outs[0]
    assert kind == "ok" and rep == want.report and tl == json.loads(want.timeline)
    for rank in (1, 2):
        kind, rep, tl = outs[rank]
        assert kind == "ok" and rep == want.report and tl is None


@pytest.mark.parametrize("case", ["clean", "corrupt", "c5"])
def test_nccl_one_rank(case):
    """The NCCL flavour of the collectives (CUDA tensors, the merge buffer all-reduced in HBM, the
    timeline runs gathered on the device) at world size 1 -- the only NCCL world one GPU allows."""
    import json

    from oracle import oracle
    from paper_2504_03683_b200.distributed import unpack_exception

    outs = _run(case, world=1, backend="nccl")
    if case == "c5":
        wl, raws = _c5()
        want = oracle.run(raws, wl.registry, [r.info for r in raws], want_timeline=True, device_index=3)
        kind, rep, tl = outs[0]
        assert kind == "ok" and rep == want.report and tl == json.loads(want.timeline)
        return
    want = _oracle(case)
    if case == "corrupt":
        kind, packed, diag = outs[0]
        e = unpack_exception(packed)
        assert kind == "raised" and type(e).__name__ == type(want.error).__name__ and str(e) == str(want.error)
        return
    kind, rep, stats, orphans, diag, path = outs[0]
    assert kind == "ok" and rep == want.report and stats == want.stats and orphans == want.orphans == diag
