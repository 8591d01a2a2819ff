"""Turn engine outputs (dense rows, error candidates, orphans) into reference objects.

Everything here is O(rows + streams + candidates): assembling the
`TallyReport` dataclass (sinks.py:139-248 semantics), choosing which trace
error the reference's single-threaded muxer would have hit first, and
formatting that exception exactly as the reference does.
"""

from __future__ import annotations

import struct

from .abi import (
    HG_ERR_FEED, HG_ERR_LEN_MISMATCH, HG_ERR_ORDER, HG_ERR_RESULT, HG_ERR_STRUCT, HG_ERR_TELEMETRY,
    HG_ERR_TRAILING, HG_ERR_TRUNC_HEADER, HG_ERR_TRUNC_PAYLOAD, HG_ERR_TRUNC_VAR, HG_ERR_UNKNOWN_SCHEMA,
    HG_ERR_UTF8, i128,
)
from .errors import CorruptRecordError, HapitraceError, MuxOrderingError, UnknownSchemaError
from .tally import TallyReport, TallyRow

_DECODE_CODES = {
    HG_ERR_TRUNC_HEADER, HG_ERR_TRUNC_PAYLOAD, HG_ERR_UNKNOWN_SCHEMA, HG_ERR_LEN_MISMATCH,
    HG_ERR_TRUNC_VAR, HG_ERR_TRAILING, HG_ERR_UTF8, HG_ERR_STRUCT, HG_ERR_ORDER,
}
_CORRUPT_TEXT = {
    HG_ERR_TRUNC_HEADER: "truncated record header",
    HG_ERR_TRUNC_PAYLOAD: "truncated record payload",
    HG_ERR_LEN_MISMATCH: "payload length mismatch",
    HG_ERR_TRUNC_VAR: "truncated variable field",
    HG_ERR_TRAILING: "trailing payload bytes",
}


def build_report(flat, rows, device_names, stream_infos, stream_idents, stream_spans) -> TallyReport:
    """TallySink.on_finish equivalent from native rows.

    rows: iterable of (section, name_id, count, errors, sum, min, max) ints.
    stream_infos: StreamInfo list when the source had an index (on_streams), else None.
    stream_idents / stream_spans: (hostname, pid, tid) and span count per stream.
    """
    reg = flat.registry
    report = TallyReport(fingerprint=reg.fingerprint, backends=(f"BACKEND_{reg.api_name.upper()}",))
    for section, name_id, count, errs, total, mn, mx in rows:
        if section == 0:
            name, sec = flat.function_names[name_id], "host"
        else:
            name, sec = device_names[name_id], "device"
        report.rows[(sec, name)] = TallyRow(name, sec, total, count, mn, mx, errs)
    hosts, procs, threads = set(), set(), set()
    if stream_infos is not None:
        for i in stream_infos:
            hosts.add(i.hostname)
            procs.add((i.hostname, i.pid))
            threads.add((i.hostname, i.pid, i.tid))
            if i.dropped_count:
                report.dropped[(i.hostname, i.pid, i.tid)] = i.dropped_count
    for (h, p, t), n in zip(stream_idents, stream_spans):
        if n:
            hosts.add(h)
            procs.add((h, p))
            threads.add((h, p, t))
    report.hostnames = frozenset(hosts)
    report.processes = frozenset(procs)
    report.threads = frozenset(threads)
    return report


def rows_from_native(native_rows) -> list:
    return [
        (r.section, r.name_id, r.count, r.error_count, i128(r.time_lo, r.time_hi),
         i128(r.min_lo, r.min_hi), i128(r.max_lo, r.max_hi))
        for r in native_rows
    ]


def error_key(e):
    """Position at which the reference's pull-based muxer raises this error.

    Priming reads (record 0 of each stream, pipeline.py:80-91) come first in
    stream order; a later decode/ordering failure at record k surfaces right
    after record k-1 of that stream was delivered (pipeline.py:93-99); an
    interval-stage failure surfaces while its own record is delivered.
    """
    if e.code in _DECODE_CODES:
        if e.seq == 0:
            return (0, 0, e.stream, 0, 0)
        return (1, e.prev_ts, e.stream, e.seq - 1, 1)
    return (1, e.ts, e.stream, e.seq, 0)


def first_error(candidates):
    """Per stream keep the decode/order failure with the lowest record index and
    drop interval-stage candidates at or beyond it, then take the earliest."""
    cut = {}
    for e in candidates:
        if e.code in _DECODE_CODES:
            if e.stream not in cut or e.seq < cut[e.stream].seq:
                cut[e.stream] = e
    live = list(cut.values())
    for e in candidates:
        if e.code not in _DECODE_CODES:
            c = cut.get(e.stream)
            if c is None or e.seq < c.seq:
                live.append(e)
    return min(live, key=error_key) if live else None


def make_exception(e, stream, flat):
    """Build the exact exception object the reference raises for candidate ``e``.

    ``stream``: RawStream (label + bytes).  Message texts that come from the
    Python runtime itself (UnicodeDecodeError, struct.error, int(nan)) are
    reproduced by re-running that one operation on the failing record's bytes.
    """
    name = stream.name
    code = e.code
    if code in _CORRUPT_TEXT:
        return CorruptRecordError(_CORRUPT_TEXT[code], name, e.offset)
    if code == HG_ERR_UNKNOWN_SCHEMA:
        return UnknownSchemaError(f"unknown schema id {e.aux} (stream {name}, byte offset {e.offset})")
    data = stream.data
    if code in (HG_ERR_UTF8, HG_ERR_STRUCT):
        (plen,) = struct.unpack_from("<I", data, e.offset + 12)
        payload = data[e.offset + 16: e.offset + 16 + plen]
        if code == HG_ERR_UTF8:
            (ln,) = struct.unpack_from("<I", payload, e.aux - 4)
            try:
                payload[e.aux: e.aux + ln].decode("utf-8")
            except UnicodeDecodeError as u:
                return CorruptRecordError(str(u), name, e.offset)
            raise AssertionError("engine flagged valid UTF-8")
        pos, size = e.aux >> 8, e.aux & 0xFF
        try:
            struct.unpack_from("<Q" if size == 8 else "<I", payload, pos)
        except struct.error as s:
            return s
        raise AssertionError("engine flagged a readable field")
    if code == HG_ERR_ORDER:
        return MuxOrderingError(name, e.seq)
    if code == HG_ERR_FEED:
        return flat.feed_errors[e.aux]()
    sid = struct.unpack_from("<I", data, e.offset)[0]
    schema = flat.registry.by_id[sid]
    if code == HG_ERR_TELEMETRY:
        counter, _ = flat.telemetry[sid]
        field = next(f for f in reversed(schema.fields) if f.name == "value")
        value = _field_value(field.kind, e.aux)
        if counter in ("compute_engine", "copy_engine"):
            return HapitraceError(f"utilization out of range: {value}")
        return HapitraceError(f"{counter} must be non-negative: {value}")
    if code == HG_ERR_RESULT:
        try:
            int(struct.unpack("<d", struct.pack("<Q", e.aux))[0])
        except (ValueError, OverflowError) as x:
            return x
        raise AssertionError("engine flagged a convertible result")
    return HapitraceError(f"engine error code {code}")


def _field_value(kind, bits):
    if kind == "f64":
        return struct.unpack("<d", struct.pack("<Q", bits))[0]
    if kind == "i64":
        return struct.unpack("<q", struct.pack("<Q", bits))[0]
    return bits


def orphan_list(orphans, labels, flat, cutoff=None, cut_streams=None):
    """IntervalBuilder.orphans in mux order: (f"{host}/{pid}/{tid}", ts, fn)."""
    keyed = []
    for o in orphans:
        if cut_streams is not None and o.stream in cut_streams and o.seq >= cut_streams[o.stream]:
            continue
        k = (1, o.ts, o.stream, o.seq, 0)
        if cutoff is not None and not k < cutoff:
            continue
        keyed.append((k, o))
    keyed.sort(key=lambda x: x[0])
    return [(labels[o.stream], o.ts, flat.function_names[o.function]) for _, o in keyed]
