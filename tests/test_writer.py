"""The native C writer binding (include/ztrc_writer.h, csrc/ztrc_writer.c)
against the reference's writer contract (writer-binding.md, TraceWriter tracefile.py:222-441):
per-thread streams, drop-newest overflow counted in records, streams.json in json.dumps(indent=1)
layout, metadata flipped to complete, and the trace it writes analysed exactly like any other."""

import json
import threading
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")


def _records(registry, n, seed):
    import random

    rnd = random.Random(seed)
    ids = [s for s in registry.schemas if s.event_class in ("host_entry", "host_exit")]
    out = []
    ts = 1000
    for _ in range(n):
        sc = rnd.choice(ids)
        payload = {}
        for f in sc.fields:
            payload[f.name] = {"string": "k" * rnd.randint(0, 40), "blob": bytes(rnd.randint(0, 60)),
                               "f64": 0.5}.get(f.kind, rnd.randint(0, 1 << 40))
        ts += rnd.randint(1, 500)
        out.append((sc, ts, payload))
    return out


@pytest.fixture
def writer():
    from paper_2504_03683_b200.writer import CWriter

    return CWriter()


def test_threads_write_a_trace_the_reader_and_oracle_accept(tmp_path, writer):
    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.tracefile import encode_record, open_trace_reader
    from paper_2504_03683_b200.writer import export_metadata

    ze = synth.ze_registry()
    meta = tmp_path / "meta.json"
    export_metadata(ze, meta)
    d = tmp_path / "trace"
    assert writer.open(d, meta, 1 << 12) == 0
    per_thread = {}

    def work(k):
        s = writer.acquire()
        recs = _records(ze, 3000, k)
        codes = [writer.emit(s, sc, ts, p) for sc, ts, p in recs]
        per_thread[k] = (recs, codes)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert writer.close() == 0
    reader = open_trace_reader(d)
    assert reader.metadata["complete"] is True
    index = json.loads((d / "streams.json").read_text())
    assert (d / "streams.json").read_text() == json.dumps(index, indent=1)  # the writer's layout
    entries = index["streams"]
    assert len(entries) == 4 and entries == sorted(entries, key=lambda e: (e["hostname"], e["pid"], e["tid"]))
    raws = reader.raw_streams()
    written = sorted(sum(1 for c in codes if c == 0) for _, codes in per_thread.values())
    assert sorted(e["event_count"] for e in entries) == written
    assert sum(e["event_count"] + e["dropped_count"] for e in entries) == 4 * 3000
    # every stream's bytes: the header, then exactly the records that were not dropped, in order
    bodies = sorted(r.data for r in raws)
    want = sorted(b"".join([b"IPHT", (1).to_bytes(4, "little"), bytes(8)] +
                           [encode_record(sc, ts, p) for (sc, ts, p), c in zip(recs, codes) if c == 0])
                  for recs, codes in per_thread.values())
    assert bodies == want
    res = oracle.run(raws, reader.registry, reader.stream_infos())
    assert res.error is None and res.stats["events_in"] == sum(written)


def test_drop_newest_overflow_is_counted(tmp_path, writer):
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.tracefile import open_trace_reader
    from paper_2504_03683_b200.writer import export_metadata

    ze = synth.ze_registry()
    meta = tmp_path / "meta.json"
    export_metadata(ze, meta)
    d = tmp_path / "trace"
    assert writer.open(d, meta, 4) == 0
    writer.pause_drainer(True)
    s = writer.acquire()
    recs = _records(ze, 10, 7)
    codes = [writer.emit(s, sc, ts, p) for sc, ts, p in recs]
    assert codes == [0] * 4 + [1] * 6  # drop-newest (tracefile.py:231-236)
    assert writer.close() == 0
    (e,) = json.loads((d / "streams.json").read_text())["streams"]
    assert (e["event_count"], e["dropped_count"]) == (4, 6)
    reader = open_trace_reader(d)
    assert [r.info for r in reader.raw_streams()][0].event_count == 4
    assert writer.emit(s, recs[0][0], 1, recs[0][2]) == -1  # after close


def test_open_refusals_and_stale_handles(tmp_path, writer):
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.writer import export_metadata

    ze = synth.ze_registry()
    meta = tmp_path / "meta.json"
    export_metadata(ze, meta)
    busy = tmp_path / "busy"
    busy.mkdir()
    (busy / "x").write_text("x")
    assert writer.open(busy, meta, 8) == -1  # not an empty directory
    done = tmp_path / "done.json"
    done.write_text(meta.read_text().replace('"complete": false', '"complete": true'))
    assert writer.open(tmp_path / "t1", done, 8) == -1  # metadata must carry complete: false
    assert writer.acquire() is None  # not open
    assert writer.open(tmp_path / "t2", meta, 8) == 0
    s = writer.acquire()
    assert writer.close() == 0
    assert writer.open(tmp_path / "t3", meta, 8) == 0
    sc = ze.schemas[0]
    assert writer.emit(s, sc, 1, {f.name: 0 for f in sc.fields}) == -1  # a handle of the closed trace
    s2 = writer.acquire()
    assert s2 and writer.emit(s2, sc, 1, {f.name: 0 if f.kind not in ("string", "blob") else
                                          ("" if f.kind == "string" else b"") for f in sc.fields}) == 0
    assert writer.close() == 0
    # an acquired-but-silent stream is not listed
    assert json.loads((tmp_path / "t2" / "streams.json").read_text()) == {"streams": []}


@pytest.mark.skipif(not REF.exists(), reason="the reference is importable only in the build container")
def test_reference_reads_the_c_writer_trace(tmp_path, writer):
    """The reference's own reader and tally over a trace the C binding wrote (and the oracle agrees)."""
    import subprocess
    import sys

    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.tracefile import open_trace_reader
    from paper_2504_03683_b200.writer import export_metadata

    ze = synth.ze_registry()
    meta = tmp_path / "meta.json"
    export_metadata(ze, meta)
    d = tmp_path / "trace"
    assert writer.open(d, meta, 1 << 10) == 0
    s = writer.acquire()
    for sc, ts, p in _records(ze, 500, 3):
        writer.emit(s, sc, ts, p)
    assert writer.close() == 0
    code = ("import sys, json; sys.path.insert(0, %r); from hapitrace.harness import tally_trace; "
            "print(tally_trace(%r).to_json())" % (str(REF), str(d)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True,
                         env={"PYTHONDONTWRITEBYTECODE": "1", "PATH": "/usr/bin:/bin"}).stdout
    reader = open_trace_reader(d)
    mine = oracle.run(reader.raw_streams(), reader.registry, reader.stream_infos())
    assert json.loads(out) == json.loads(mine.report.to_json())
