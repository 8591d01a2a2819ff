"""Shared helpers: load a golden fixture's expected outputs and compare a result to them."""

import hashlib
import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def names():
    return json.loads((GOLDEN / "expected" / "index.json").read_text())


def expected(name):
    return json.loads((GOLDEN / "expected" / f"{name}.json").read_text())


def trace_dir(name):
    return GOLDEN / "traces" / name


def describe_exc(e):
    attrs = {k: getattr(e, k) for k in ("stream", "offset", "index") if hasattr(e, k)}
    return {"type": type(e).__name__, "str": str(e), "attrs": attrs}


def check(exp, *, error, report=None, render=None, stats=None, orphans=None, timeline=None):
    """Compare one pipeline mode's outcome with the golden record ``exp``."""
    if "error" in exp:
        assert error is not None, f"expected {exp['error']['type']}: {exp['error']['str']}"
        got = describe_exc(error)
        want = {k: exp["error"][k] for k in ("type", "str", "attrs")}
        assert got == want
        if orphans is not None:
            assert [list(o) for o in orphans] == exp["orphans"]
        return
    assert error is None, f"unexpected {type(error).__name__}: {error}"
    assert report.to_json() == exp["tally_json"]
    if render is not None:
        assert render == exp["render"]
    if stats is not None:
        assert stats == exp["stats"]
    if orphans is not None:
        assert [list(o) for o in orphans] == exp["orphans"]
    if timeline is not None and "timeline_sha256" in exp:
        blob = timeline if isinstance(timeline, bytes) else timeline.encode()
        assert len(blob) == exp["timeline_len"]
        assert hashlib.sha256(blob).hexdigest() == exp["timeline_sha256"]


def Diag_factory():
    """A diagnostics-only sink (no on_message override): collects on_diagnostics orphans."""
    from paper_2504_03683_b200.pipeline import Sink

    class Diag(Sink):
        name = "diag"
        consumes = "intervals"

        def __init__(self):
            self.orphans = None

        def on_diagnostics(self, orphans):
            self.orphans = list(orphans)

        def on_finish(self):
            return self.orphans

    return Diag()
