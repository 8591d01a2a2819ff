"""PrettyPrintSink on the GPU: every record in mux order, rendered by
csrc/events.cu, byte-identical to the reference (golden traces) and to the oracle restatement
(synthetic traces); error traces raise what the reference raises."""

import hashlib
import json

import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

INDEX = json.loads((GOLDEN / "expected" / "pretty_index.json").read_text())


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


@pytest.mark.parametrize("name", sorted(INDEX))
def test_pretty_matches_reference_golden(engine, name):
    from paper_2504_03683_b200 import PrettyPrintSink, open_trace_reader, run_pipeline

    want = INDEX[name]
    reader = open_trace_reader(GOLDEN / "traces" / name)
    if "raises" in want:
        with pytest.raises(Exception) as ei:
            run_pipeline(reader, [PrettyPrintSink()], engine=engine)
        assert type(ei.value).__name__ == want["raises"] and str(ei.value) == want["str"]
        return
    text = run_pipeline(reader, [PrettyPrintSink()], engine=engine)["pretty"].encode("utf-8")
    assert len(text) == want["bytes"] and hashlib.sha256(text).hexdigest() == want["sha256"]


def _check_synthetic(engine, wl):
    from oracle import oracle
    from paper_2504_03683_b200 import PrettyPrintSink, TallySink, run_pipeline, synth

    raws = synth.generate(wl)

    class Src:
        registry = wl.registry

        def raw_streams(self):
            return raws

        def stream_infos(self):
            return [r.info for r in raws]

    lines = []
    p1, p2 = PrettyPrintSink(), PrettyPrintSink(write=lines.append)
    p2.name = "pretty2"
    res = run_pipeline(Src(), [p1, TallySink(), p2], engine=engine)
    want_text = oracle.pretty(raws, wl.registry)
    want = oracle.run(raws, wl.registry, [r.info for r in raws])
    assert res["pretty"] == want_text
    assert res["pretty2"] == "" and lines == want_text.split("\n")[:-1]
    assert res["tally"] == want.report and vars(res.stats) == want.stats
    order = engine.event_order()
    assert len(order) == want.stats["events_in"] and len(set(order)) == len(order)
    return want_text


@pytest.mark.parametrize("name,scale", [("c2", 0.0004), ("c5", 0.0005), ("c4", 0.0005), ("c1", 0.01)])
def test_pretty_synthetic_configs(engine, name, scale):
    from paper_2504_03683_b200 import synth

    text = _check_synthetic(engine, synth.config(name, scale))
    assert text.count("\n") > 1000


def test_pretty_wide_values_and_ties(engine):
    """Timestamps near 2^60 (fmt_timestamp modulo a day), ties broken by identity, f64 results."""
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec(f"h{i % 2}", P + i, P + i, 2000, 900 + i) for i in range(6)]
    wl = synth.Workload("wide", synth.ze_registry(), streams,
                        dict(gap_lo=0, gap_hi=3, ts0_hi=1 << 60, prof_p=0.4, orphan_p=0.02, close_at_end=0,
                             dev_lo=-(1 << 40), dev_hi=1 << 40),
                        kernel_names=synth.kernel_pool(20))
    _check_synthetic(engine, wl)


def test_pretty_memcpy_fixture_through_record_source(engine):
    """The reference's pretty_memcpy.txt golden (test_acceptance.py:311-336) from a record list."""
    from paper_2504_03683_b200 import PrettyPrintSink, run_pipeline, synth
    from paper_2504_03683_b200.tracefile import EventRecord

    ze = synth.ze_registry()
    sc = ze.schema("ze:zeMockCommandListAppendMemoryCopy_entry")
    ts = (21 * 3600 + 41 * 60 + 26) * 10**9 + 240059291
    rec = EventRecord(sc.id, ts, {"hCommandList": 0x0508AEA8, "dstptr": 0xFF007FFFFFF90000,
                                  "srcptr": 0x00007FFFEDCEAB98, "size": 472, "hSignalEvent": 0x05165898,
                                  "numWaitEvents": 0, "phWaitEvents": 0, "phWaitEvents_vals": b""},
                      hostname="x4204c0s1b0n0", pid=124765, tid=124765)
    res = run_pipeline([[rec]], [PrettyPrintSink()], registry=ze, engine=engine)
    assert res["pretty"] == (GOLDEN / "pretty_memcpy.txt").read_text()


def test_pretty_none_identity(engine):
    """Records without identity print "None" for hostname, vpid and vtid (f-string of None)."""
    from paper_2504_03683_b200 import PrettyPrintSink, run_pipeline, synth
    from paper_2504_03683_b200.tracefile import EventRecord

    ze = synth.ze_registry()
    sc = ze.schema("ze:zeMockInit_entry")
    payload = {f.name: 0 for f in sc.fields}
    res = run_pipeline([[EventRecord(sc.id, 5, payload)]], [PrettyPrintSink()], registry=ze, engine=engine)
    assert " - None - vpid: None, vtid: None - ze:zeMockInit_entry: " in res["pretty"]
