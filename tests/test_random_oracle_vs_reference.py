"""The oracle against the reference itself on seeded random traces (tests/random_traces.py): tally
JSON, IntervalStats, orphans, timeline bytes, pretty-print text and validation findings -- or the
same exception -- for every seed.  Needs /root/reference (the build container); skipped elsewhere."""

import json
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="the reference is importable only in the build container")

SEEDS = list(range(200))


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import hapitrace.harness as harness
    import hapitrace.pipeline as pipeline
    import hapitrace.sinks as sinks
    import hapitrace.tracefile as tracefile

    return harness, pipeline, sinks, tracefile


@pytest.mark.parametrize("seed", SEEDS)
def test_oracle_equals_reference(ref, seed, tmp_path):
    from random_traces import random_trace

    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.pipeline import merge_same_identity
    from paper_2504_03683_b200.tracefile import open_trace_reader
    from paper_2504_03683_b200.validation import ValidationRules

    harness, pipeline, sinks, tracefile = ref
    ze, raws = random_trace(seed)
    d = tmp_path / "t"
    synth.write(synth.Workload("r", ze, []), raws, d)

    class Diag(pipeline.Sink):
        name = "diag"

        def on_diagnostics(self, orphans):
            self.orphans = [list(o) for o in orphans]

    diag = Diag()
    tl_path = tmp_path / "tl.json"
    want_exc = None
    try:
        res = pipeline.run_pipeline(tracefile.open_trace_reader(d),
                                    [sinks.TallySink(), sinks.TimelineSink(out_path=tl_path), sinks.PrettyPrintSink(),
                                     sinks.ValidationSink(harness.bundled_model()), diag])
    except Exception as e:  # noqa: BLE001
        want_exc = e
    reader = open_trace_reader(d)
    mine = merge_same_identity(reader.raw_streams())
    got = oracle.run(mine, reader.registry, reader.stream_infos(), want_timeline=True)
    if want_exc is not None:
        assert got.error is not None, f"reference raised {want_exc!r}, oracle did not"
        assert type(got.error).__name__ == type(want_exc).__name__ and str(got.error) == str(want_exc)
        assert [list(o) for o in got.orphans] == diag.orphans
        return
    assert got.error is None, got.error
    assert json.loads(got.report.to_json()) == json.loads(res["tally"].to_json())
    assert got.stats == {k: getattr(res.stats, k) for k in got.stats}
    assert [list(o) for o in got.orphans] == diag.orphans
    assert got.timeline.encode() == tl_path.read_bytes()
    assert oracle.pretty(mine, reader.registry) == res["pretty"]
    rules = ValidationRules.from_model(harness.bundled_model(), reader.registry)
    findings = oracle.validate(mine, reader.registry, rules, got.orphans)
    assert [list(f) for f in findings] == [[f.rule, f.subject, f.stream, f.timestamp_ns, f.message]
                                          for f in res["validate"]]
