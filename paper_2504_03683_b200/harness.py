"""Convenience entry points mirroring `/root/reference/pkg/src/hapitrace/harness.py:117-129`."""

from __future__ import annotations

from pathlib import Path

from .pipeline import TallySink, run_pipeline
from .tally import TallyReport
from .tracefile import open_trace_reader


def tally_trace(trace_dir, engine=None, distributed=False) -> TallyReport:
    """One GPU pipeline pass producing the tally report for a finalized trace (harness.py:117-121).
    ``distributed``: shard the streams over the ranks of a torch.distributed group (run_pipeline)."""
    reader = open_trace_reader(trace_dir)
    return run_pipeline(reader, sinks=[TallySink()], engine=engine, distributed=distributed)["tally"]


def write_tally_json(report: TallyReport, path):
    Path(path).write_text(report.to_json())


def read_tally_json(path) -> TallyReport:
    return TallyReport.from_json(Path(path).read_text())
