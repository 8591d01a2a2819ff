"""The ValidationSink restatement in oracle/oracle.py, and ValidationRules, against the reference's
own findings on every golden trace of the bundled registry (make_validation_golden.py)."""

import json

import pytest

from golden_util import GOLDEN

INDEX = json.loads((GOLDEN / "expected" / "validation_index.json").read_text())
RULES = json.loads((GOLDEN / "expected" / "validation_rules.json").read_text())
CLEAN = sorted(k for k, v in INDEX.items() if "findings" in v)


@pytest.mark.parametrize("name", CLEAN)
def test_oracle_validation_matches_reference(name):
    from oracle import oracle
    from paper_2504_03683_b200.pipeline import merge_same_identity
    from paper_2504_03683_b200.tracefile import open_trace_reader
    from paper_2504_03683_b200.validation import ValidationRules

    reader = open_trace_reader(GOLDEN / "traces" / name)
    raws = merge_same_identity(reader.raw_streams())
    orphans = oracle.run(raws, reader.registry, reader.stream_infos()).orphans
    got = oracle.validate(raws, reader.registry, ValidationRules.from_dict(RULES), orphans)
    assert [list(f) for f in got] == INDEX[name]["findings"]


def test_rules_round_trip():
    from paper_2504_03683_b200.validation import ValidationRules

    r = ValidationRules.from_dict(RULES)
    assert r.to_dict() == RULES and r.pnext and r.creators and r.releasers and r.execute and r.resets


def test_injected_defects_each_found_once():
    """test_acceptance.py:214-231: one injected defect, exactly that rule."""
    for tag, rule in (("uninit_pnext", "uninit_pnext"), ("leak_event", "leaked_event"),
                      ("no_reset_cmdlist", "cmdlist_not_reset")):
        assert [f[0] for f in INDEX[f"val_w1_{tag}"]["findings"]] == [rule]
    assert INDEX["w1_default"]["findings"] == []
