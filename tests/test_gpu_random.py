"""The GPU engine against the oracle on seeded random traces (tests/random_traces.py) through
run_pipeline with every sink the engine serves: tally, timeline, pretty-print and validation -- or the
same exception and the orphans delivered before it -- on the default path, and the tally alone on
the exact path (the single pass falls back there for corrupt seeds)."""

import json

import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

RULES = json.loads((GOLDEN / "expected" / "validation_rules.json").read_text())


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


@pytest.mark.parametrize("seed", list(range(150)))
def test_engine_equals_oracle_on_random_traces(engine, seed):
    from random_traces import random_trace

    from oracle import oracle
    from paper_2504_03683_b200 import (PrettyPrintSink, TallySink, TimelineSink, ValidationRules, ValidationSink,
                                       run_pipeline)
    from paper_2504_03683_b200.pipeline import Sink, merge_same_identity

    ze, raws = random_trace(seed)

    class Src:
        registry = ze

        def raw_streams(self):
            return raws

        def stream_infos(self):
            return [r.info for r in raws]

    class Diag(Sink):
        name = "diag"

        def on_diagnostics(self, orphans):
            self.orphans = orphans

    rules = ValidationRules.from_dict(RULES)
    mine = merge_same_identity(raws)
    want = oracle.run(mine, ze, [r.info for r in raws], want_timeline=True)
    diag = Diag()
    sinks = [TallySink(), TimelineSink(), PrettyPrintSink(), ValidationSink(rules=rules), diag]
    if want.error is not None:
        with pytest.raises(Exception) as ei:
            run_pipeline(Src(), sinks, engine=engine)
        assert type(ei.value).__name__ == type(want.error).__name__ and str(ei.value) == str(want.error)
        assert diag.orphans == want.orphans
        return
    res = run_pipeline(Src(), sinks, engine=engine)
    assert res["tally"] == want.report and vars(res.stats) == want.stats and res.orphans == want.orphans
    assert res["timeline"] == json.loads(want.timeline)
    assert res["pretty"] == oracle.pretty(mine, ze)
    findings = oracle.validate(mine, ze, rules, want.orphans)
    assert [tuple(vars(f).values()) for f in res["validate"]] == [tuple(f) for f in findings]


@pytest.mark.parametrize("seed", list(range(0, 150, 3)))
@pytest.mark.parametrize("path", [0, 1])
def test_tally_paths_on_random_traces(engine, seed, path):
    from random_traces import random_trace

    from oracle import oracle
    from paper_2504_03683_b200.engine import OPT_PATH
    from paper_2504_03683_b200.pipeline import merge_same_identity

    ze, raws = random_trace(seed)
    mine = merge_same_identity(raws)
    want = oracle.run(mine, ze, [r.info for r in raws])
    engine.set_option(OPT_PATH, path)
    try:
        got = engine.run(mine, ze, [r.info for r in raws])
    finally:
        engine.set_option(OPT_PATH, 0)
    if want.error is not None:
        assert got.error is not None and type(got.error) is type(want.error) and str(got.error) == str(want.error)
        assert got.orphans == want.orphans
        return
    assert got.error is None and got.report == want.report and got.stats == want.stats and got.orphans == want.orphans


@pytest.mark.parametrize("seed", list(range(1, 150, 5)))
@pytest.mark.parametrize("range_bytes", [32, 112, 600])
def test_single_pass_small_ranges_on_random_traces(engine, seed, range_bytes):
    """Many speculative ranges per stream (escaped names, wide values, orphans, mismatches, unclosed calls
    crossing range cuts): the single pass either vouches for the exact result or falls back."""
    from random_traces import random_trace

    from oracle import oracle
    from paper_2504_03683_b200.engine import OPT_RANGE_BYTES
    from paper_2504_03683_b200.pipeline import merge_same_identity

    ze, raws = random_trace(seed, corrupt=False)
    mine = merge_same_identity(raws)
    want = oracle.run(mine, ze, [r.info for r in raws])
    engine.set_option(OPT_RANGE_BYTES, range_bytes)
    try:
        got = engine.run(mine, ze, [r.info for r in raws])
    finally:
        engine.set_option(OPT_RANGE_BYTES, 0)
    if want.error is not None:
        assert got.error is not None and str(got.error) == str(want.error)
        return
    assert got.error is None and got.report == want.report and got.stats == want.stats and got.orphans == want.orphans


@pytest.mark.parametrize("range_bytes", [0, 112])
@pytest.mark.parametrize("seed", list(range(120)))
def test_single_pass_timeline_on_random_traces(engine, seed, range_bytes):
    """Tally + timeline runs take the single pass (per-range messages, compose's cross-range spans
    with the result bits of pending exits); 112-byte ranges split the streams into many ranges."""
    from random_traces import random_trace

    from oracle import oracle
    from paper_2504_03683_b200.engine import OPT_RANGE_BYTES
    from paper_2504_03683_b200.pipeline import merge_same_identity

    ze, raws = random_trace(seed)
    mine = merge_same_identity(raws)
    infos = [r.info for r in mine]
    want = oracle.run(mine, ze, infos, want_timeline=True)
    engine.set_option(OPT_RANGE_BYTES, range_bytes)
    try:
        got = engine.run(mine, ze, infos, want_timeline=True)
    finally:
        engine.set_option(OPT_RANGE_BYTES, 0)
    assert (got.error is None) == (want.error is None), (got.error, want.error)
    if want.error is not None:
        assert type(got.error) is type(want.error) and str(got.error) == str(want.error)
        return
    assert got.report == want.report and got.stats == want.stats and got.orphans == want.orphans
    assert got.timeline == want.timeline.encode()
    if range_bytes == 0:
        assert engine.last_path()[0] == 1


@pytest.mark.parametrize("range_bytes", [0, 112])
@pytest.mark.parametrize("seed", list(range(100)))
def test_single_pass_events_on_random_traces(engine, seed, range_bytes):
    """PrettyPrintSink + ValidationSink runs (no timeline) take the single pass: every record in its
    range's list, then the muxer's order by the merge passes."""
    from random_traces import random_trace

    from oracle import oracle
    from paper_2504_03683_b200 import PrettyPrintSink, TallySink, ValidationRules, ValidationSink, run_pipeline
    from paper_2504_03683_b200.engine import OPT_RANGE_BYTES
    from paper_2504_03683_b200.pipeline import Sink, merge_same_identity

    ze, raws = random_trace(seed)

    class Src:
        registry = ze

        def raw_streams(self):
            return raws

        def stream_infos(self):
            return [r.info for r in raws]

    class Diag(Sink):
        name = "diag"

        def on_diagnostics(self, orphans):
            self.orphans = orphans

    rules = ValidationRules.from_dict(RULES)
    mine = merge_same_identity(raws)
    want = oracle.run(mine, ze, [r.info for r in raws])
    diag = Diag()
    sinks = [TallySink(), PrettyPrintSink(), ValidationSink(rules=rules), diag]
    engine.set_option(OPT_RANGE_BYTES, range_bytes)
    try:
        if want.error is not None:
            with pytest.raises(Exception) as ei:
                run_pipeline(Src(), sinks, engine=engine)
            assert type(ei.value).__name__ == type(want.error).__name__ and str(ei.value) == str(want.error)
            assert diag.orphans == want.orphans
            return
        res = run_pipeline(Src(), sinks, engine=engine)
    finally:
        engine.set_option(OPT_RANGE_BYTES, 0)
    assert res["tally"] == want.report and vars(res.stats) == want.stats and res.orphans == want.orphans
    assert res["pretty"] == oracle.pretty(mine, ze)
    findings = oracle.validate(mine, ze, rules, want.orphans)
    assert [tuple(vars(f).values()) for f in res["validate"]] == [tuple(f) for f in findings]
    if range_bytes == 0:
        assert engine.last_path()[0] == 1
