"""The CPU oracle reproduces the reference's outputs on every golden fixture.

This pins the oracle before it is trusted as the checker for the GPU path
(fixtures and expected outputs come from the reference itself, see
tests/golden/make_golden.py)."""

import pytest

from golden_util import check, expected, names, trace_dir
from oracle import oracle
from paper_2504_03683_b200.tally import render_tally
from paper_2504_03683_b200.tracefile import open_trace_reader


def _oracle(name, timeline):
    try:
        reader = open_trace_reader(trace_dir(name))
        raws = reader.raw_streams()
    except Exception as e:  # header-level errors surface while opening cursors
        return None, e
    r = oracle.run(raws, reader.registry, reader.stream_infos(), want_timeline=timeline,
                   labels=[f"{s.hostname}/{s.pid}/{s.tid}" for s in raws])
    return r, r.error


@pytest.mark.parametrize("name", names())
@pytest.mark.parametrize("mode", ["tally", "tally+timeline"])
def test_oracle_matches_reference(name, mode):
    exp = expected(name)[mode]
    r, err = _oracle(name, mode == "tally+timeline")
    if r is None:
        check(exp, error=err)
        return
    check(exp, error=err, report=r.report, render=render_tally(r.report), stats=r.stats,
          orphans=r.orphans, timeline=r.timeline if mode == "tally+timeline" else None)
