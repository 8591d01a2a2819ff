"""Numeric and size edges through the GPU engine, against the CPU oracle (bit-exact).

* C1 at its stated size (1M events, one stream) on the single pass and on the exact path;
* wide values: host durations of 2^32..2^33 ns (the 128-bit global fold), timestamps from
  about 2^60 (CPython float repr beyond 2^53 in the timeline), device spans of +-2^40 ns
  (negative when end < start: the signed 128-bit device fold);
* more than 16,384 distinct device names (the name dictionary grows and the run repeats);
* the timeline of a device-heavy trace of about 2M events;
* streams that share one (hostname, pid, tid) identity (one LIFO stack, pipeline.py:156-161).
"""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


def _check(engine, raws, wl, path=0, timeline=False, want=None):
    from oracle import oracle
    from paper_2504_03683_b200.engine import OPT_PATH

    infos = [r.info for r in raws]
    engine.set_option(OPT_PATH, path)
    try:
        got = engine.run(raws, wl.registry, infos, want_timeline=timeline)
    finally:
        engine.set_option(OPT_PATH, 0)
    if want is None:
        want = oracle.run(raws, wl.registry, infos, want_timeline=timeline)
    assert got.error is None and want.error is None, (got.error, want.error)
    assert got.stats == want.stats
    assert got.report == want.report
    assert got.orphans == want.orphans
    if timeline:
        assert got.timeline == want.timeline.encode()
    return got, want


@pytest.fixture(scope="module")
def c1_full():
    from paper_2504_03683_b200 import synth

    wl = synth.config("c1", 1.0)
    return wl, synth.generate(wl)


@pytest.mark.parametrize("path,expect", [(0, 1), (1, 0)])
def test_c1_full_size(engine, c1_full, path, expect):
    """BASELINE config 1 (1M events, one stream) bit-exact on both phase-1 paths."""
    wl, raws = c1_full
    assert sum(r.info.event_count for r in raws) == 1_000_000
    _check(engine, raws, wl, path=path)
    assert engine.last_path()[0] == expect


def _wide(n_streams=12, per=40_000, seed=0):
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec("wide", P + 100 * (i % 3), P + 100 * (i % 3) + i, per + 101 * i, 31_000 + 17 * seed + i)
               for i in range(n_streams)]
    params = dict(gap_lo=1 << 32, gap_hi=1 << 33, ts0_hi=1 << 60, prof_p=0.4, close_at_end=0, max_depth=6,
                  dev_off_hi=1 << 41, dev_lo=-(1 << 40), dev_hi=1 << 40)
    return synth.Workload("wide", synth.ze_registry(), streams, params, kernel_names=synth.kernel_pool(64))


@pytest.mark.parametrize("path", [0, 1])
def test_wide_durations_and_timestamps(engine, path):
    from paper_2504_03683_b200 import synth

    wl = _wide()
    raws = synth.generate(wl)
    got, want = _check(engine, raws, wl, path=path)
    rows = want.report.rows
    assert any(r.max_ns >= 1 << 32 for (sec, _), r in rows.items() if sec == "host")
    assert any(r.min_ns < 0 for (sec, _), r in rows.items() if sec == "device")
    assert want.last_ts >= 1 << 53


def test_wide_values_timeline(engine):
    from paper_2504_03683_b200 import synth

    wl = _wide(n_streams=4, per=6000, seed=1)
    _check(engine, synth.generate(wl), wl, timeline=True)


def test_more_than_16k_device_names(engine):
    """20,000 kernel names over 16 streams: past the 16,384-row dictionary, which grows and reruns."""
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    streams = [synth.StreamSpec("names", P, P + i, 60_000, 41_000 + i) for i in range(16)]
    wl = synth.Workload("names", synth.ze_registry(), streams, dict(prof_p=1.0),
                        kernel_names=synth.kernel_pool(20_000, ascii_only=True))
    raws = synth.generate(wl)
    got, want = _check(engine, raws, wl)
    n_dev = sum(1 for (sec, _) in want.report.rows if sec == "device")
    assert n_dev > 16_384
    got2, _ = _check(engine, raws, wl, want=want)  # a second run on the grown dictionary


def test_timeline_device_heavy_2m_events(engine):
    from paper_2504_03683_b200 import synth

    wl = synth.config("c5", 0.02)
    raws = synth.generate(wl)
    assert sum(r.info.event_count for r in raws) >= 2_000_000
    _check(engine, raws, wl, timeline=True)


@pytest.mark.parametrize("name_len", [300, 4000])
def test_timeline_long_names(engine, name_len):
    """Kernel names of hundreds to thousands of bytes (escapes and non-ASCII among them): formatting
    tiles larger than the shared staging buffer are written straight to the output."""
    from paper_2504_03683_b200 import synth

    P = synth.PID_BASE
    names = [("k%d_" % i) + ("x\u00e9\"" if i % 3 == 0 else "y") * (name_len // 4) for i in range(24)]
    names = [n.encode().decode("unicode_escape") for n in names]
    streams = [synth.StreamSpec("long", P, P + i, 4_000, 77_000 + i) for i in range(6)]
    wl = synth.Workload("long", synth.ze_registry(), streams, dict(prof_p=0.8), kernel_names=names)
    _check(engine, synth.generate(wl), wl, timeline=True)


def test_shared_identity_streams_merge(engine):
    """Two cursors per identity with interleaved calls (entries in one, exits in the other)
    through run_pipeline: one merged stream per identity, equal to the oracle that keys
    stacks by identity the way the reference does."""
    import struct

    from oracle import oracle
    from paper_2504_03683_b200 import run_pipeline, synth
    from paper_2504_03683_b200.pipeline import TallySink, TimelineSink
    from paper_2504_03683_b200.tracefile import RawStream, stream_bytes

    wl = synth.config("c2", 0.001)
    raws = synth.generate(wl)[:6]
    # split every stream's records alternately into two files with the same identity
    split = []
    for r in raws:
        recs, off = [], 16
        while off < len(r.data):
            plen = struct.unpack_from("<I", r.data, off + 12)[0]
            recs.append(r.data[off: off + 16 + plen])
            off += 16 + plen
        for part in (recs[0::2], recs[1::2]):
            split.append(RawStream(r.hostname, r.pid, r.tid, f"{r.name}.{len(split)}", stream_bytes(part)))

    class Src:
        registry = wl.registry

        def raw_streams(self):
            return list(split)

    want = oracle.run(split, wl.registry, None, want_timeline=True)
    res = run_pipeline(Src(), [TallySink(), TimelineSink()])
    assert res["tally"] == want.report
    assert vars(res.stats) == want.stats
    assert res.orphans == want.orphans
    assert res["timeline"] == __import__("json").loads(want.timeline)


def test_truncation_flush_order_with_none_hostnames(engine):
    """Record-list sources with hostname None: the muxer orders streams by (hostname or "", ...) but
    the reference flushes open calls by (str(hostname), pid, tid) (pipeline.py:230), so the
    truncated spans of the None stream come between "A..." and "Zed" in the timeline."""
    import json

    from oracle import oracle
    from paper_2504_03683_b200 import run_pipeline, synth
    from paper_2504_03683_b200.pipeline import TallySink, TimelineSink, _raw_from_records
    from paper_2504_03683_b200.tracefile import EventRecord

    ze = synth.ze_registry()
    sid = {s.name: s.id for s in ze.schemas}

    def rec(name, ts, host, pid, tid):
        sc = ze.by_id[sid[f"ze:{name}"]]
        payload = {f.name: ("" if f.kind == "string" else b"" if f.kind == "blob" else 0) for f in sc.fields}
        return EventRecord(sc.id, ts, payload, host, pid, tid)

    cursors = []
    for k, (host, pid) in enumerate([(None, 5), ("Alpha", 1), ("Zed", 2), (None, 3), ("Beta", 9)]):
        cursors.append([rec("zeMockInit_entry", 10 + k, host, pid, pid), rec("zeMockMemAlloc_entry", 20 + k, host, pid, pid),
                        rec("zeMockMemAlloc_exit", 30 + k, host, pid, pid), rec("zeMockMemFree_entry", 40 + k, host, pid, pid)])
    raws = _raw_from_records(cursors, ze)
    want = oracle.run(raws, ze, None, want_timeline=True)
    res = run_pipeline(cursors, [TallySink(), TimelineSink()], registry=ze)
    assert res["tally"] == want.report and vars(res.stats) == want.stats
    assert res["timeline"] == json.loads(want.timeline)
    names = [o.get("pid") for o in json.loads(want.timeline) if o.get("args", {}).get("truncated")]
    assert names[:2] == [1, 1] and names[-2:] == [2, 2]  # Alpha first, Zed last
