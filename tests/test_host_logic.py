"""CPU tests of the host-side logic around the GPU engine (no CUDA device needed).

Covers the registry flattening (roles, unsupported layouts), the choice of the
first trace error in the reference's muxer order and its exception text, the
tally report's wire/text forms and the monoid merge (aggregator.py:35-76),
and the synthetic generator's byte format."""

import json
import random
import struct

import pytest

from golden_util import GOLDEN
from paper_2504_03683_b200 import errors
from paper_2504_03683_b200.abi import (
    FEED_ALWAYS, FEED_TIMELINE, HG_ERR_FEED, HG_ERR_ORDER, HG_ERR_TELEMETRY, HG_ERR_TRUNC_PAYLOAD,
    HG_ERR_UNKNOWN_SCHEMA, HG_ERR_UTF8, HgTraceError, ROLE_NAME, ROLE_RESULT, ROLE_START, flatten_registry,
)
from paper_2504_03683_b200.registry import SchemaRegistry
from paper_2504_03683_b200.results import error_key, first_error, make_exception
from paper_2504_03683_b200.synth import config, count_records, generate, ze_registry
from paper_2504_03683_b200.tally import TallyReport, TallyRow, empty_report, fmt_duration, merge_tallies, render_tally
from paper_2504_03683_b200.tracefile import RawStream, encode_record, stream_bytes


def _reg(schemas):
    return SchemaRegistry.from_dict({"api_name": "t", "fingerprint": "0" * 16, "schemas": schemas})


def _s(sid, name, cls, fields, fn=None):
    return {"id": sid, "name": name, "class": cls, "function": fn, "mode_mask": ["full"],
            "fields": [{"name": n, "kind": k, "origin": "x"} for n, k in fields]}


def test_flatten_bundled_registry_roles():
    flat = flatten_registry(ze_registry())
    assert flat.n_schemas == 38
    assert len(flat.function_names) == 13
    by = {s.id: s for s in flat.schemas}
    reg = ze_registry()
    exit_ = reg.schema("ze:zeMockInit_exit")
    assert by[exit_.id].role[ROLE_RESULT] == 0
    prof = reg.schema("ze:zeMockCommandListAppendLaunchKernel_profiling")
    assert by[prof.id].role[ROLE_START] == 0 and by[prof.id].role[ROLE_NAME] == 3
    tel = reg.schema("ze:telemetry_copy_tile_1")
    assert by[tel.id].counter_kind == 3 and by[tel.id].counter_domain == 1 and by[tel.id].feed_error == 0


def test_flatten_feed_errors_and_unsupported():
    reg = _reg([
        _s(0, "t:telemetry_bogus_1", "telemetry_sample", [("device", "u64"), ("value", "f64")]),
        _s(1, "t:telemetry_power_domain_7", "telemetry_sample", [("device", "u64"), ("value", "f64")]),
        _s(2, "t:k_profiling", "device_profiling", [("device_start_ns", "u64"), ("device_end_ns", "u64")]),
    ])
    flat = flatten_registry(reg)
    by = {s.id: s for s in flat.schemas}
    assert by[0].feed_error == FEED_ALWAYS
    assert str(flat.feed_errors[0]()) == "not a telemetry schema: 't:telemetry_bogus_1'"
    assert by[1].feed_error == FEED_TIMELINE
    assert str(flat.feed_errors[1]()) == "no timeline track for counter power|7"
    assert by[2].feed_error == FEED_ALWAYS and isinstance(flat.feed_errors[2](), KeyError)
    with pytest.raises(errors.UnsupportedTraceError):
        flatten_registry(_reg([_s(0, "t:f_exit", "host_exit", [("result", "string")], "f")]))


def _err(code, stream, seq, ts=0, prev=0, off=0, aux=0):
    e = HgTraceError()
    e.code, e.stream, e.seq, e.ts, e.prev_ts, e.offset, e.aux = code, stream, seq, ts, prev, off, aux
    return e


def test_first_error_follows_pull_order():
    # priming failures beat everything, in stream order
    a = _err(HG_ERR_ORDER, 1, 0)
    b = _err(HG_ERR_UNKNOWN_SCHEMA, 0, 5, prev=1)
    assert first_error([b, a]) is a
    # a later pull surfaces after the previous record of its stream was delivered
    c = _err(HG_ERR_ORDER, 0, 10, ts=3, prev=50)
    d = _err(HG_ERR_TRUNC_PAYLOAD, 1, 4, prev=40)
    assert first_error([c, d]) is d
    # an interval-stage failure at record r beats a pull failure after r
    e = _err(HG_ERR_TELEMETRY, 2, 7, ts=40)
    assert error_key(e) < error_key(_err(HG_ERR_ORDER, 2, 8, prev=40))
    # ... but not one beyond the stream's first decode failure
    f = _err(HG_ERR_FEED, 0, 12, ts=1)
    assert first_error([c, f]) is c


def test_make_exception_texts():
    reg = ze_registry()
    flat = flatten_registry(reg)
    sch = reg.schema("ze:zeMockCommandListAppendLaunchKernel_entry")
    payload = struct.pack("<Q", 1) + struct.pack("<I", 3) + b"a\xffb" + struct.pack("<QQ", 8, 0)
    rec = struct.pack("<IQI", sch.id, 5, len(payload)) + payload
    data = stream_bytes([rec])
    raw = RawStream("h", 1, 1, "stream_1_1.bin", data)
    exc = make_exception(_err(HG_ERR_UTF8, 0, 0, off=16, aux=12), raw, flat)
    assert isinstance(exc, errors.CorruptRecordError) and exc.offset == 16
    assert str(exc).startswith("'utf-8' codec can't decode byte 0xff in position 1")
    exc = make_exception(_err(HG_ERR_UNKNOWN_SCHEMA, 0, 0, off=16, aux=777), raw, flat)
    assert str(exc) == "unknown schema id 777 (stream stream_1_1.bin, byte offset 16)"
    exc = make_exception(_err(HG_ERR_ORDER, 0, 9), raw, flat)
    assert isinstance(exc, errors.MuxOrderingError) and exc.index == 9


def test_tally_render_golden_and_wire_form():
    """The reference's own tally golden (tests/golden/tally_fixture.txt, sinks.py render)."""
    exp = json.loads((GOLDEN / "expected" / "tally_fixture.json").read_text())
    rep = TallyReport(fingerprint=None, backends=("BACKEND_HIP", "BACKEND_ZE"),
                      hostnames=frozenset({"aurora-node"}), processes=frozenset({("aurora-node", 1)}),
                      threads=frozenset({("aurora-node", 1, 1)}))
    for name, total, calls in exp["rows"]:
        rep.rows[("host", name)] = TallyRow(name, "host", total, calls, total // calls, total // calls)
    assert render_tally(rep) == exp["render"]
    assert TallyReport.from_json(rep.to_json()) == rep


def test_fmt_duration_vectors():
    # sinks.py fmt_duration vectors (test_sinks.py:222-228)
    assert [fmt_duration(x) for x in (4_730_000_000, 500_910_000, 394_500_000, 1, 0, 1_500)] == [
        "4.73s", "500.91ms", "394.50ms", "1.00ns", "0.00ns", "1.50us"]


def _rand_report(rng, rank):
    rep = TallyReport(fingerprint="f" * 16, backends=("BACKEND_ZE",), hostnames=frozenset({f"n{rank % 2}"}),
                      processes=frozenset({(f"n{rank % 2}", rank)}),
                      threads=frozenset({(f"n{rank % 2}", rank, rank)}))
    for name in rng.sample("abcdef", rng.randint(1, 6)):
        times = [rng.randint(1, 10**6) for _ in range(rng.randint(1, 8))]
        rep.rows[("host", name)] = TallyRow(name, "host", sum(times), len(times), min(times), max(times),
                                            rng.randint(0, len(times)))
    if rng.random() < 0.4:
        rep.dropped[(f"n{rank % 2}", rank, rank)] = rng.randint(1, 9)
    return rep


def test_merge_is_a_commutative_monoid():
    rng = random.Random(7)
    for i in range(200):
        a, b, c = (_rand_report(rng, 3 * i + k) for k in range(3))
        assert merge_tallies([a, empty_report()]) == a
        assert merge_tallies([a, b]) == merge_tallies([b, a])
        assert merge_tallies([merge_tallies([a, b]), c]) == merge_tallies([a, merge_tallies([b, c])])
    with pytest.raises(errors.FingerprintMismatchError):
        merge_tallies([TallyReport(fingerprint="a" * 16), TallyReport(fingerprint="b" * 16)])


def test_synth_streams_are_well_formed():
    wl = config("c2", 0.0002)
    raws = generate(wl)
    assert len(raws) == 256
    for r in raws[:8]:
        assert r.data[:4] == struct.pack("<I", 0x54485049)
        assert count_records(r.data) == r.info.event_count
        # record chain ends exactly at the end of the file
        off = 16
        while off < len(r.data):
            off += 16 + struct.unpack_from("<I", r.data, off + 12)[0]
        assert off == len(r.data)
    # deterministic
    again = generate(config("c2", 0.0002))
    assert [r.data for r in raws[:4]] == [r.data for r in again[:4]]


def test_synth_reproduces_committed_goldens():
    """The C generator still writes the committed syn_c1 / syn_c2 fixture bytes (make_golden.py)."""
    from golden_util import trace_dir
    from paper_2504_03683_b200.tracefile import open_trace_reader

    for name, cfg, scale in (("syn_c1", "c1", 0.008), ("syn_c2", "c2", 0.0003)):
        ours = {(r.hostname, r.pid, r.tid): r.data for r in generate(config(cfg, scale))}
        committed = {(r.hostname, r.pid, r.tid): r.data for r in open_trace_reader(trace_dir(name)).raw_streams()}
        assert ours == committed, name


def test_merge_same_identity_matches_identity_keyed_oracle():
    """Splitting streams into same-identity halves and merging them back (pipeline.merge_same_identity)
    gives what the oracle -- which keys its stacks by identity like pipeline.py:156-161 -- computes
    on the split streams; the dup_identity golden pins that oracle to the reference."""
    from oracle import oracle
    from paper_2504_03683_b200.pipeline import merge_same_identity

    wl = config("c2", 0.0005)
    raws = generate(wl)[:8]
    rng = random.Random(5)
    split = []
    for r in raws:
        parts, off = ([], []), 16
        while off < len(r.data):
            plen = struct.unpack_from("<I", r.data, off + 12)[0]
            parts[rng.random() < 0.5].append(r.data[off: off + 16 + plen])
            off += 16 + plen
        for i, p in enumerate(parts):
            split.append(RawStream(r.hostname, r.pid, r.tid, f"{r.name}.{i}", stream_bytes(p)))
    merged = merge_same_identity(split)
    assert len(merged) == len(raws)
    a = oracle.run(split, wl.registry, want_timeline=True)
    b = oracle.run(merged, wl.registry, want_timeline=True)
    assert a.report == b.report and a.stats == b.stats and a.orphans == b.orphans and a.timeline == b.timeline
    assert oracle.run(raws, wl.registry).report == b.report  # the split lost nothing


def test_passive_sink_detection():
    from paper_2504_03683_b200.pipeline import Sink, _is_passive

    class Diag(Sink):
        def on_diagnostics(self, orphans):
            pass

    class Ref:  # a sink deriving from a foreign base class named Sink with a no-op on_message
        pass

    RefSink = type("Sink", (), {"on_message": lambda self, msg: None, "name": "s"})
    RefDiag = type("RefDiag", (RefSink,), {"on_diagnostics": lambda self, o: None})

    class Busy(Sink):
        def on_message(self, msg):
            print(msg)

    assert _is_passive(Diag()) and _is_passive(RefDiag()) and not _is_passive(Busy())
    assert _is_passive(Ref())
