"""The PrettyPrintSink restatement in oracle/oracle.py against the reference's own output on every
clean golden trace (tests/golden/expected/pretty_index.json, made by make_pretty_golden.py)."""

import hashlib
import json

import pytest

from golden_util import GOLDEN

INDEX = json.loads((GOLDEN / "expected" / "pretty_index.json").read_text())
CLEAN = sorted(k for k, v in INDEX.items() if "sha256" in v)


@pytest.mark.parametrize("name", CLEAN)
def test_oracle_pretty_matches_reference(name):
    from oracle import oracle
    from paper_2504_03683_b200.pipeline import merge_same_identity
    from paper_2504_03683_b200.tracefile import open_trace_reader

    reader = open_trace_reader(GOLDEN / "traces" / name)
    text = oracle.pretty(merge_same_identity(reader.raw_streams()), reader.registry).encode("utf-8")
    want = INDEX[name]
    assert len(text) == want["bytes"] and hashlib.sha256(text).hexdigest() == want["sha256"]


def test_pretty_memcpy_fixture_line():
    """tests/golden/pretty_memcpy.txt of the reference (test_acceptance.py:311-336) through the oracle."""
    from oracle import oracle
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.pipeline import _raw_from_records
    from paper_2504_03683_b200.tracefile import EventRecord

    ze = synth.ze_registry()
    sc = ze.schema("ze:zeMockCommandListAppendMemoryCopy_entry")
    ts = (21 * 3600 + 41 * 60 + 26) * 10**9 + 240059291
    rec = EventRecord(sc.id, ts, {"hCommandList": 0x0508AEA8, "dstptr": 0xFF007FFFFFF90000,
                                  "srcptr": 0x00007FFFEDCEAB98, "size": 472, "hSignalEvent": 0x05165898,
                                  "numWaitEvents": 0, "phWaitEvents": 0, "phWaitEvents_vals": b""},
                      hostname="x4204c0s1b0n0", pid=124765, tid=124765)
    raws = _raw_from_records([[rec]], ze)
    assert oracle.pretty(raws, ze) == (GOLDEN / "pretty_memcpy.txt").read_text()
