"""TEST INFRASTRUCTURE ONLY -- ctypes front of the CPU oracle (hapi_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) import this module.  It runs the literal CPU restatement of
the reference path and returns results in the same shapes the GPU engine's
Python front returns, so tests compare like with like:

    OracleResult.report      TallyReport        (sinks.py:139-248)
    OracleResult.stats       IntervalStats dict (pipeline.py:117-129)
    OracleResult.orphans     [(label, ts, fn)]  (pipeline.py:138, 163-168)
    OracleResult.error       the exception the reference raises, or None
    OracleResult.timeline    json.dump(objs, indent=1) text (sinks.py:414-418)
"""

from __future__ import annotations

import ctypes as C
import os
import struct
import subprocess
from dataclasses import dataclass
from pathlib import Path

from paper_2504_03683_b200.abi import (
    HgOrphan, HgStats, HgTallyRow, HgTraceError, flatten_registry, i128,
)
from paper_2504_03683_b200.results import build_report, make_exception, orphan_list, rows_from_native
from paper_2504_03683_b200.timeline import TimelineBuilder
from paper_2504_03683_b200.registry import COUNTER_KINDS

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
SRC = HERE / "hapi_oracle.c"


class TlItem(C.Structure):
    _fields_ = [
        ("kind", C.c_uint8), ("truncated", C.c_uint8), ("value_kind", C.c_uint8), ("pad", C.c_uint8),
        ("stream", C.c_uint32), ("name", C.c_int32), ("cmdkind", C.c_int32),
        ("start", C.c_uint64), ("end", C.c_uint64), ("result", C.c_uint64),
        ("tile", C.c_uint64), ("engine", C.c_uint64),
        ("counter_kind", C.c_int64), ("counter_domain", C.c_int64),
    ]


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", str(LIB), str(SRC), "-lpthread"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.oracle_run.restype = vp
        L.oracle_run.argtypes = [vp, u32, C.c_char_p, u32, u32, vp, vp, u32, vp, vp]
        L.oracle_tally_threads.restype = vp
        L.oracle_tally_threads.argtypes = [vp, u32, C.c_char_p, u32, u32, vp, vp, u32, vp]
        L.oracle_tally_threads_at.restype = vp
        L.oracle_tally_threads_at.argtypes = [vp, u32, C.c_char_p, u32, u32, vp, vp, u32, vp, u64]
        L.oracle_free.argtypes = [vp]
        L.oracle_has_error.argtypes = [vp, vp]
        L.oracle_has_error.restype = C.c_int
        L.oracle_stats.argtypes = [vp, vp]
        L.oracle_rows.argtypes = [vp, vp, u64]
        L.oracle_rows.restype = u64
        L.oracle_names.argtypes = [vp, C.c_int, vp, u64, vp, u64]
        L.oracle_names.restype = u64
        L.oracle_name_bytes.argtypes = [vp, C.c_int]
        L.oracle_name_bytes.restype = u64
        L.oracle_orphans.argtypes = [vp, vp, u64]
        L.oracle_orphans.restype = u64
        L.oracle_stream_spans.argtypes = [vp, vp, u64]
        L.oracle_stream_spans.restype = u64
        L.oracle_timeline.argtypes = [vp, vp, u64]
        L.oracle_timeline.restype = u64
        L.oracle_tl_item_size.restype = u64
        L.oracle_last_ts.argtypes = [vp]
        L.oracle_last_ts.restype = u64
        assert L.oracle_tl_item_size() == C.sizeof(TlItem)
        _lib = L
    return _lib


@dataclass
class OracleResult:
    report: object
    stats: dict
    orphans: list
    error: BaseException | None
    timeline: str | None
    last_ts: int


def _names(L, h, which):
    nb = L.oracle_name_bytes(h, which)
    n = L.oracle_names(h, which, None, 0, None, 0)
    buf = (C.c_uint8 * max(nb, 1))()
    offs = (C.c_uint64 * (n + 1))()
    L.oracle_names(h, which, buf, nb, offs, n + 1)
    raw = bytes(buf)[:nb]
    return [raw[offs[i]:offs[i + 1]].decode("utf-8") for i in range(n)]


def _py_value(kind, bits):
    if kind == 2:  # f64
        return struct.unpack("<d", struct.pack("<Q", bits))[0]
    if kind == 1:  # i64
        return struct.unpack("<q", struct.pack("<Q", bits))[0]
    return bits


def run(raw_streams, registry, stream_infos=None, want_timeline=False, threads=0, device_index=0,
        labels=None, floor_last_ts=0) -> OracleResult:
    """Run the oracle over RawStream objects in (hostname, pid, tid) order.

    threads > 0: the sharded tally (no timeline, no orphan list); floor_last_ts then lower-bounds the
    truncation end -- the global last timestamp when the streams are one rank's shard."""
    L = lib()
    flat = flatten_registry(registry)
    n = len(raw_streams)
    bufs = [C.create_string_buffer(s.data, len(s.data)) if s.data else None for s in raw_streams]
    ptrs = (C.c_void_p * max(n, 1))(*[C.cast(b, C.c_void_p) if b is not None else None for b in bufs])
    sizes = (C.c_uint64 * max(n, 1))(*[len(s.data) for s in raw_streams])
    # streams sharing one (hostname, pid, tid) share a stack (pipeline.py:156-161)
    first, grp = {}, []
    for i, s in enumerate(raw_streams):
        grp.append(first.setdefault((s.hostname, s.pid, s.tid), i))
    group = (C.c_uint32 * max(n, 1))(*grp) if len(first) < n else None
    # the reference flushes open calls per stack sorted by (str(hostname), pid, tid) (pipeline.py:230)
    fo = sorted(range(n), key=lambda i: (str(raw_streams[i].hostname), raw_streams[i].pid or 0,
                                         raw_streams[i].tid or 0, i))
    flush = (C.c_uint32 * max(n, 1))(*fo) if fo != list(range(n)) else None
    if threads:
        h = L.oracle_tally_threads_at(flat.schemas, flat.n_schemas, flat.kinds, len(flat.function_names), n,
                                      ptrs, sizes, threads, group, int(floor_last_ts))
    else:
        h = L.oracle_run(flat.schemas, flat.n_schemas, flat.kinds, len(flat.function_names), n, ptrs, sizes,
                         1 if want_timeline else 0, group, flush)
    if not h:
        raise RuntimeError("oracle: registry ids too large")
    try:
        return _collect(L, h, flat, raw_streams, stream_infos, want_timeline, device_index, labels)
    finally:
        L.oracle_free(h)


def _collect(L, h, flat, raw_streams, stream_infos, want_timeline, device_index, labels):
    n = len(raw_streams)
    idents = [(s.hostname, s.pid, s.tid) for s in raw_streams]
    if labels is None:
        labels = [f"{s.hostname}/{s.pid}/{s.tid}" for s in raw_streams]
    st = HgStats()
    L.oracle_stats(h, C.byref(st))
    stats = {k: getattr(st, k) for k, _ in HgStats._fields_}
    n_orph = L.oracle_orphans(h, None, 0)
    orph = (HgOrphan * max(n_orph, 1))()
    L.oracle_orphans(h, orph, n_orph)
    orphans_raw = list(orph)[:n_orph]
    err = HgTraceError()
    error = None
    if L.oracle_has_error(h, C.byref(err)):
        error = make_exception(err, raw_streams[err.stream], flat)
    # the oracle stops at the first error, so every collected orphan precedes it
    orphans = orphan_list(orphans_raw, labels, flat)
    n_rows = L.oracle_rows(h, None, 0)
    rows = (HgTallyRow * max(n_rows, 1))()
    L.oracle_rows(h, rows, n_rows)
    names = _names(L, h, 0)
    spans = (C.c_uint64 * max(n, 1))()
    L.oracle_stream_spans(h, spans, n)
    report = build_report(flat, rows_from_native(list(rows)[:n_rows]), names, stream_infos, idents, list(spans)[:n])
    timeline = None
    if want_timeline and error is None:
        cmdkinds = _names(L, h, 1)
        n_items = L.oracle_timeline(h, None, 0)
        items = (TlItem * max(n_items, 1))()
        L.oracle_timeline(h, items, n_items)
        tb = TimelineBuilder(device_index)
        for it in list(items)[:n_items]:
            s = raw_streams[it.stream]
            if it.kind == 0:
                tb.host_span(flat.function_names[it.name], s.hostname, s.pid, s.tid, it.start, it.end,
                             _py_value(it.value_kind, it.result) if it.value_kind != 2 else
                             int(_py_value(2, it.result)), bool(it.truncated))
            elif it.kind == 1:
                start = struct.unpack("<q", struct.pack("<Q", it.start))[0] if it.value_kind & 1 else it.start
                end = struct.unpack("<q", struct.pack("<Q", it.end))[0] if it.value_kind & 2 else it.end
                tb.device_span(names[it.name], start, end, it.tile, it.engine,
                               cmdkinds[it.cmdkind] if it.cmdkind >= 0 else "")
            else:
                tb.sample(COUNTER_KINDS[it.counter_kind], it.counter_domain, it.start,
                          _py_value(it.value_kind, it.result), it.tile)
        timeline = tb.dumps()
    return OracleResult(report, stats, orphans, error, timeline, L.oracle_last_ts(h))


def run_dir(directory, want_timeline=False, threads=0, device_index=0) -> OracleResult:
    from paper_2504_03683_b200.tracefile import open_trace_reader

    reader = open_trace_reader(directory)
    return run(reader.raw_streams(), reader.registry, reader.stream_infos(), want_timeline, threads,
               device_index)


# ---------------------------------------------------------------------------
# PrettyPrintSink (event sink) restatement -- TEST INFRASTRUCTURE, pinned by
# tests/golden/expected/pretty_index.json (the reference's own output on every golden trace)

def _fmt_timestamp(ns: int) -> str:  # sinks.py:43-46
    s, frac = divmod(ns, 1_000_000_000)
    s %= 86400
    return f"{s // 3600:02d}:{s % 3600 // 60:02d}:{s % 60:02d}.{frac:09d}"


def _fmt_value(kind: str, value) -> str:  # sinks.py:49-59
    import json

    if kind == "address":
        return f"0x{value:016x}"
    if kind == "string":
        return json.dumps(value)
    if kind == "blob":
        return "[ " + ", ".join(str(b) for b in value) + " ]"
    if kind == "f64":
        return repr(float(value))
    return str(value)


def _decode_stream(data: bytes, registry):
    """(ts, schema, payload dict) of every record (tracefile.py:147-215 on a clean stream)."""
    out = []
    off = 16
    while off + 16 <= len(data):
        sid, ts, plen = struct.unpack_from("<IQI", data, off)
        schema = registry.by_id[sid]
        p = off + 16
        payload = {}
        for f in schema.fields:
            if f.kind in ("string", "blob"):
                (n,) = struct.unpack_from("<I", data, p)
                raw = data[p + 4: p + 4 + n]
                payload[f.name] = raw.decode("utf-8") if f.kind == "string" else raw
                p += 4 + n
            else:
                fmt = {"u64": "<Q", "i64": "<q", "f64": "<d", "address": "<Q"}[f.kind]
                (payload[f.name],) = struct.unpack_from(fmt, data, p)
                p += 8
        out.append((ts, schema, payload))
        off += 16 + plen
    return out


def pretty(raw_streams, registry) -> str:
    """PrettyPrintSink.on_finish text over mux_streams order (pipeline.py:68-114, sinks.py:66-106)."""
    import heapq

    heap = []
    decoded = [_decode_stream(r.data, registry) if r.data else [] for r in raw_streams]
    for idx, (r, recs) in enumerate(zip(raw_streams, decoded)):
        if recs:
            heap.append((recs[0][0], r.hostname or "", r.pid or 0, r.tid or 0, 0, idx))
    heapq.heapify(heap)
    lines = []
    while heap:
        ts, _h, _p, _t, seq, idx = heapq.heappop(heap)
        r = raw_streams[idx]
        _, schema, payload = decoded[idx][seq]
        fields = ", ".join(f"{f.name}: {_fmt_value(f.kind, payload[f.name])}" for f in schema.fields)
        lines.append(f"{_fmt_timestamp(ts)} - {r.hostname} - vpid: {r.pid}, vtid: {r.tid} - {schema.name}: "
                     + ("{ " + fields + " }" if fields else "{ }"))
        if seq + 1 < len(decoded[idx]):
            heapq.heappush(heap, (decoded[idx][seq + 1][0], _h, _p, _t, seq + 1, idx))
    return "\n".join(lines) + ("\n" if lines else "")


# ---------------------------------------------------------------------------
# ValidationSink restatement -- TEST INFRASTRUCTURE, pinned by
# tests/golden/expected/validation_index.json (the reference's own findings)

def validate(raw_streams, registry, rules, orphans):
    """ValidationSink.on_message over mux_streams order, then on_finish (sinks.py:518-594);
    ``rules``: paper_2504_03683_b200.validation.ValidationRules; ``orphans``: the interval stage's."""
    import heapq

    findings, live, executed, pending = [], {}, {}, {}
    decoded = [_decode_stream(r.data, registry) if r.data else [] for r in raw_streams]
    heap = [(recs[0][0], r.hostname or "", r.pid or 0, r.tid or 0, 0, idx)
            for idx, (r, recs) in enumerate(zip(raw_streams, decoded)) if recs]
    heapq.heapify(heap)
    while heap:
        ts, _h, _p, _t, seq, idx = heapq.heappop(heap)
        r = raw_streams[idx]
        _, schema, payload = decoded[idx][seq]
        if seq + 1 < len(decoded[idx]):
            heapq.heappush(heap, (decoded[idx][seq + 1][0], _h, _p, _t, seq + 1, idx))
        label = f"{r.hostname}/{r.pid}/{r.tid}"
        sid = schema.id
        if sid in rules.pnext:
            fn_name, blob_field = rules.pnext[sid]
            blob = payload.get(blob_field, b"")
            if len(blob) >= 8:
                pnext = int.from_bytes(blob[:8], "little")
                if pnext != 0:
                    findings.append(("uninit_pnext", pnext, label, ts,
                                     f"{fn_name}: extension slot pNext is 0x{pnext:x}, must be NULL"))
        key = (r.hostname, r.pid, r.tid)
        if schema.event_class == "host_entry":
            pending[(key, schema.function)] = payload
            if sid in rules.execute:
                h = int(payload[rules.execute[sid]])
                if executed.get(h):
                    findings.append(("cmdlist_not_reset", h, label, ts,
                                     f"command list 0x{h:x} executed again without a reset"))
                executed[h] = True
            continue
        if schema.event_class != "host_exit":
            continue
        result = int(payload.get("result", 0))
        if sid in rules.creators and result == 0:
            fn_name, out_field = rules.creators[sid]
            h = int(payload[out_field])
            live[h] = ("leaked_event", h, label, ts, f"handle 0x{h:x} from {fn_name} never released")
        elif sid in rules.releasers and result == 0:
            fn_name, _entry_id, handle_param = rules.releasers[sid]
            entry = pending.get((key, fn_name))
            if entry is not None:
                live.pop(int(entry[handle_param]), None)
        elif sid in rules.resets and result == 0:
            _entry_id, handle_param = rules.resets[sid]
            entry = pending.get((key, schema.function))
            if entry is not None:
                executed[int(entry[handle_param])] = False
    leaks = sorted(live.values(), key=lambda f: f[1])
    orph = [("orphan_exit", 0, stream, ts, f"exit of {fn} without matching entry") for stream, ts, fn in orphans]
    return findings + leaks + orph
