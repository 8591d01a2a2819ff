"""GPU parity: run_pipeline on libhapigpu reproduces the reference on every golden fixture."""

import pytest

from golden_util import Diag_factory, check, expected, names, trace_dir

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2504_03683_b200.engine import Engine

    eng = Engine(device=0)
    yield eng
    eng.close()


@pytest.mark.parametrize("name", names())
def test_tally_matches_reference(engine, name):
    from paper_2504_03683_b200 import TallySink, open_trace_reader, render_tally, run_pipeline

    exp = expected(name)["tally"]
    diag = Diag_factory()
    try:
        res = run_pipeline(open_trace_reader(trace_dir(name)), [TallySink(), diag], engine=engine)
    except Exception as e:  # noqa: BLE001
        check(exp, error=e, orphans=diag.orphans)
        return
    rep = res["tally"]
    stats = {k: getattr(res.stats, k) for k in exp["stats"]} if "stats" in exp else None
    check(exp, error=None, report=rep, render=render_tally(rep), stats=stats, orphans=res.orphans)
    assert diag.orphans == res.orphans


@pytest.mark.parametrize("name", names())
def test_timeline_matches_reference(engine, name):
    """tally + timeline sinks: the GPU's JSON bytes equal json.dump of the reference's objects."""
    from paper_2504_03683_b200 import TallySink, TimelineSink, open_trace_reader, render_tally, run_pipeline

    exp = expected(name)["tally+timeline"]
    diag = Diag_factory()
    tl = TimelineSink()
    try:
        res = run_pipeline(open_trace_reader(trace_dir(name)), [TallySink(), tl, diag], engine=engine)
    except Exception as e:  # noqa: BLE001
        check(exp, error=e, orphans=diag.orphans)
        return
    rep = res["tally"]
    stats = {k: getattr(res.stats, k) for k in exp["stats"]} if "stats" in exp else None
    check(exp, error=None, report=rep, render=render_tally(rep), stats=stats, orphans=res.orphans,
          timeline=tl.json_bytes)
    assert "timeline_sha256" in exp
