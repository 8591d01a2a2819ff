"""ValidationSink on the GPU (csrc/validate.cu): the reference's findings on
every golden trace of the bundled registry (incl. the three w1 defect injections of
test_acceptance.py:214-231), and the oracle restatement's on synthetic traces with many handles."""

import json

import pytest

from golden_util import GOLDEN

pytestmark = pytest.mark.gpu

INDEX = json.loads((GOLDEN / "expected" / "validation_index.json").read_text())
RULES = json.loads((GOLDEN / "expected" / "validation_rules.json").read_text())


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


def _sink():
    from paper_2504_03683_b200 import ValidationRules, ValidationSink

    return ValidationSink(rules=ValidationRules.from_dict(RULES))


@pytest.mark.parametrize("name", sorted(INDEX))
def test_validation_matches_reference_golden(engine, name):
    from paper_2504_03683_b200 import open_trace_reader, run_pipeline

    want = INDEX[name]
    reader = open_trace_reader(GOLDEN / "traces" / name)
    if "raises" in want:
        with pytest.raises(Exception) as ei:
            run_pipeline(reader, [_sink()], engine=engine)
        assert type(ei.value).__name__ == want["raises"] and str(ei.value) == want["str"]
        return
    got = run_pipeline(reader, [_sink()], engine=engine)["validate"]
    assert [[f.rule, f.subject, f.stream, f.timestamp_ns, f.message] for f in got] == want["findings"]


@pytest.mark.parametrize("name,scale", [("c2", 0.0005), ("c5", 0.0005), ("c1", 0.02)])
def test_validation_synthetic_with_pretty_and_tally(engine, name, scale):
    from oracle import oracle
    from paper_2504_03683_b200 import PrettyPrintSink, TallySink, ValidationRules, run_pipeline, synth

    wl = synth.config(name, scale)
    raws = synth.generate(wl)

    class Src:
        registry = wl.registry

        def raw_streams(self):
            return raws

        def stream_infos(self):
            return [r.info for r in raws]

    res = run_pipeline(Src(), [TallySink(), _sink(), PrettyPrintSink()], engine=engine)
    want = oracle.run(raws, wl.registry, [r.info for r in raws])
    findings = oracle.validate(raws, wl.registry, ValidationRules.from_dict(RULES), want.orphans)
    got = [tuple([f.rule, f.subject, f.stream, f.timestamp_ns, f.message]) for f in res["validate"]]
    assert got == [tuple(f) for f in findings] and len(got) > 10
    assert res["tally"] == want.report and res["pretty"] == oracle.pretty(raws, wl.registry)
