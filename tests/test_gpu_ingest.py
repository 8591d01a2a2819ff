"""Ingest: the same streams staged from every source kind must give the
oracle's results bit-exactly -- stream files read by the engine (hg_add_stream_file, pinned
double-buffered chunks), pageable host bytes (the same pipeline), pinned host memory (direct DMA)
and CUDA tensors on the engine's GPU (hg_add_stream_device, HBM->HBM)."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


@pytest.fixture(scope="module")
def trace(tmp_path_factory):
    from paper_2504_03683_b200 import synth

    wl = synth.config("c1", 0.3)  # one ~10 MB stream (two staging chunks) ...
    small = synth.config("c2", 0.001)  # ... plus 256 small ones
    wl.streams[0].file = "stream_c1.bin"  # small's first stream has the same (pid, tid)
    for sp in small.streams:
        sp.hostname = "small"
    wl.streams = wl.streams + small.streams
    raws = synth.generate(wl)
    d = tmp_path_factory.mktemp("ingest") / "trace"
    synth.write(wl, raws, d)
    return wl, raws, d


def _want(wl, raws):
    from oracle import oracle

    return oracle.run(raws, wl.registry, [r.info for r in raws])


def _got(engine, wl, raws):
    r = engine.run(raws, wl.registry, [x.info for x in raws], reuse_streams=True)
    assert r.error is None
    return r


def test_file_streams_through_run_pipeline(engine, trace):
    from paper_2504_03683_b200 import TallySink, open_trace_reader, run_pipeline

    wl, raws, d = trace
    want = _want(wl, raws)
    res = run_pipeline(open_trace_reader(d), [TallySink()], engine=engine)
    assert res["tally"] == want.report and vars(res.stats) == want.stats and res.orphans == want.orphans
    st = engine.ingest_stats()
    assert st["file_bytes"] == sum(len(r.data) for r in raws) and st["pinned_bytes"] == 0


def test_pageable_pinned_and_device_sources_agree(engine, trace):
    import torch

    wl, raws, _ = trace
    want = _want(wl, raws)
    total = sum(len(r.data) for r in raws)
    idents = [(r.hostname, r.pid, r.tid) for r in raws]

    engine.set_registry(wl.registry)
    engine.set_streams(raws)  # Python bytes: pageable
    got = _got(engine, wl, raws)
    assert got.report == want.report and got.stats == want.stats
    assert engine.ingest_stats()["pageable_bytes"] == total

    pinned = []
    for r in raws:
        t = torch.empty(len(r.data), dtype=torch.uint8, pin_memory=True)
        t.copy_(torch.frombuffer(bytearray(r.data), dtype=torch.uint8))
        pinned.append(t)
    engine.set_streams_pinned(idents, pinned)
    got = _got(engine, wl, raws)
    assert got.report == want.report and got.stats == want.stats
    assert engine.ingest_stats()["pinned_bytes"] == total

    dev = [t.to("cuda:0") for t in pinned]
    engine.set_streams_device(idents, dev)
    got = _got(engine, wl, raws)
    assert got.report == want.report and got.stats == want.stats
    st = engine.ingest_stats()
    assert st["device_bytes"] == total and st["pinned_bytes"] == st["pageable_bytes"] == 0


def test_device_stream_from_another_gpu_is_refused(engine):
    import torch

    from paper_2504_03683_b200.errors import EngineError

    host = torch.zeros(64, dtype=torch.uint8)
    with pytest.raises(EngineError):
        engine.add_stream_device("h", 1, 1, host)  # host memory is not device memory
