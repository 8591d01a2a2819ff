"""A trace written by the native C writer binding (csrc/ztrc_writer.c, §8(f) row 4) from several
threads, analysed on the GPU through run_pipeline: equal to the oracle."""

import threading

import pytest

pytestmark = pytest.mark.gpu


def test_c_writer_trace_through_gpu_pipeline(tmp_path):
    from test_writer import _records

    from oracle import oracle
    from paper_2504_03683_b200 import PrettyPrintSink, TallySink, open_trace_reader, run_pipeline, synth
    from paper_2504_03683_b200.engine import Engine
    from paper_2504_03683_b200.writer import CWriter, export_metadata

    ze = synth.ze_registry()
    meta = tmp_path / "meta.json"
    export_metadata(ze, meta)
    d = tmp_path / "trace"
    w = CWriter()
    assert w.open(d, meta, 1 << 14) == 0

    def work(k):
        s = w.acquire()
        for sc, ts, p in _records(ze, 5000, 100 + k):
            w.emit(s, sc, ts, p)

    th = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert w.close() == 0
    reader = open_trace_reader(d)
    raws = reader.raw_streams()
    want = oracle.run(raws, reader.registry, reader.stream_infos())
    eng = Engine(device=0)
    res = run_pipeline(open_trace_reader(d), [TallySink(), PrettyPrintSink()], engine=eng)
    assert res["tally"] == want.report and vars(res.stats) == want.stats and res.orphans == want.orphans
    assert res["pretty"] == oracle.pretty(raws, reader.registry)
    eng.close()
