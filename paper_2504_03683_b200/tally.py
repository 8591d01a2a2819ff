"""Tally report: the reduced output of the hot path, its wire form and text form.

Value semantics follow `/root/reference/pkg/src/hapitrace/sinks.py:113-303`
(row fold, JSON wire form, fixed-width rendering with truncated percentages)
and `aggregator.py:30-76` (commutative-monoid merge).  The numbers inside a
report are produced on the GPU (`engine.py`); this module only holds them and
renders them, so text output is byte-identical to the reference for equal
reports.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

from .errors import FingerprintMismatchError

_UNITS = ((1_000_000_000, "s"), (1_000_000, "ms"), (1_000, "us"), (1, "ns"))


def fmt_duration(ns: int) -> str:
    """Largest unit with magnitude >= 1, two decimals (sinks.py:36-41)."""
    for div, unit in _UNITS:
        if ns >= div:
            return f"{ns / div:.2f}{unit}"
    return "0.00ns"


@dataclass
class TallyRow:
    name: str
    section: str  # "host" | "device"
    time_ns: int = 0
    count: int = 0
    min_ns: int = 0
    max_ns: int = 0
    error_count: int = 0

    def fold(self, duration_ns: int, error: bool):
        if self.count:
            self.min_ns = min(self.min_ns, duration_ns)
            self.max_ns = max(self.max_ns, duration_ns)
        else:
            self.min_ns = self.max_ns = duration_ns
        self.count += 1
        self.time_ns += duration_ns
        self.error_count += 1 if error else 0

    @property
    def average_ns(self) -> float:
        return self.time_ns / self.count if self.count else 0.0


@dataclass
class TallyReport:
    fingerprint: str | None = None
    backends: tuple = ()
    hostnames: frozenset = frozenset()
    processes: frozenset = frozenset()
    threads: frozenset = frozenset()
    rows: dict = field(default_factory=dict)  # (section, name) -> TallyRow
    dropped: dict = field(default_factory=dict)  # (hostname, pid, tid) -> count

    def section_rows(self, section: str) -> list:
        picked = [r for r in self.rows.values() if r.section == section]
        picked.sort(key=lambda r: (-r.time_ns, r.name))
        return picked

    def total_dropped(self) -> int:
        return sum(self.dropped.values())

    def to_json(self) -> str:
        rows = []
        for _key, r in sorted(self.rows.items()):
            rows.append(
                {
                    "section": r.section,
                    "name": r.name,
                    "time_ns": r.time_ns,
                    "count": r.count,
                    "min_ns": r.min_ns,
                    "max_ns": r.max_ns,
                    "error_count": r.error_count,
                }
            )
        doc = {
            "format_version": 1,
            "fingerprint": self.fingerprint,
            "backends": sorted(self.backends),
            "hostnames": sorted(self.hostnames),
            "processes": sorted(list(p) for p in self.processes),
            "threads": sorted(list(t) for t in self.threads),
            "rows": rows,
            "dropped": [
                {"hostname": h, "pid": p, "tid": t, "count": c}
                for (h, p, t), c in sorted(self.dropped.items())
            ],
        }
        return json.dumps(doc, indent=1)

    @classmethod
    def from_json(cls, text: str) -> "TallyReport":
        doc = json.loads(text)
        rows = {}
        for r in doc["rows"]:
            rows[(r["section"], r["name"])] = TallyRow(
                r["name"], r["section"], r["time_ns"], r["count"], r["min_ns"], r["max_ns"],
                r["error_count"],
            )
        return cls(
            fingerprint=doc["fingerprint"],
            backends=tuple(doc["backends"]),
            hostnames=frozenset(doc["hostnames"]),
            processes=frozenset(tuple(p) for p in doc["processes"]),
            threads=frozenset(tuple(t) for t in doc["threads"]),
            rows=rows,
            dropped={(d["hostname"], d["pid"], d["tid"]): d["count"] for d in doc["dropped"]},
        )


def _pct(part: int, total: int) -> str:
    # truncation, never rounding (sinks.py:251-254)
    basis = int(part * 10000 // total) if total else 0
    return f"{basis // 100}.{basis % 100:02d}"


def _table(rows: list) -> list:
    total = sum(r.time_ns for r in rows)
    head = ("Name", "Time", "Time(%)", "Calls", "Average", "Min", "Max")
    body = [
        (
            r.name,
            fmt_duration(r.time_ns),
            _pct(r.time_ns, total),
            str(r.count),
            fmt_duration(int(r.average_ns)),
            fmt_duration(r.min_ns),
            fmt_duration(r.max_ns),
        )
        for r in rows
    ]
    width = [max([len(head[c])] + [len(b[c]) for b in body]) for c in range(len(head))]
    out = [" | ".join(h.rjust(width[c]) for c, h in enumerate(head))]
    out.extend(" | ".join(v.rjust(width[c]) for c, v in enumerate(b)) for b in body)
    return out


def render_tally(report: TallyReport) -> str:
    """Fixed-width text: banner, host table, device table, drops (sinks.py:281-303)."""
    lines = [
        ",".join(sorted(report.backends))
        + f" | {len(report.hostnames)} Hostnames"
        + f" | {len(report.processes)} Processes"
        + f" | {len(report.threads)} Threads | ",
        "",
    ]
    host = report.section_rows("host")
    if host:
        lines += _table(host)
    device = report.section_rows("device")
    if device:
        lines += ["", "Device commands:", ""] + _table(device)
    n_dropped = report.total_dropped()
    if n_dropped:
        detail = ", ".join(f"{h}/{p}/{t}: {c}" for (h, p, t), c in sorted(report.dropped.items()))
        lines += ["", f"Dropped events: {n_dropped} ({detail})"]
    return "\n".join(lines) + "\n"


def empty_report() -> TallyReport:
    """Merge identity (aggregator.py:30-32)."""
    return TallyReport()


def merge_tallies(reports) -> TallyReport:
    """Commutative-monoid merge by (section, name) (aggregator.py:35-76)."""
    reports = list(reports)
    fps = {r.fingerprint for r in reports if r.fingerprint is not None}
    if len(fps) > 1:
        raise FingerprintMismatchError(f"cannot merge reports from different models: {sorted(fps)}")
    out = TallyReport(fingerprint=next(iter(fps)) if fps else None)
    backends, hosts, procs, threads = set(), set(), set(), set()
    for r in reports:
        backends |= set(r.backends)
        hosts |= r.hostnames
        procs |= r.processes
        threads |= r.threads
        for key, row in r.rows.items():
            acc = out.rows.get(key)
            if acc is None:
                out.rows[key] = TallyRow(row.name, row.section, row.time_ns, row.count,
                                         row.min_ns, row.max_ns, row.error_count)
                continue
            acc.time_ns += row.time_ns
            acc.count += row.count
            acc.min_ns = min(acc.min_ns, row.min_ns)
            acc.max_ns = max(acc.max_ns, row.max_ns)
            acc.error_count += row.error_count
        for key, n in r.dropped.items():
            out.dropped[key] = out.dropped.get(key, 0) + n
    out.backends = tuple(sorted(backends))
    out.hostnames = frozenset(hosts)
    out.processes = frozenset(procs)
    out.threads = frozenset(threads)
    return out
