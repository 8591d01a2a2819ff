"""`run_pipeline` and the sink plugin API, served by the GPU engine.

Mirrors `/root/reference/pkg/src/hapitrace/pipeline.py:250-314` and the tally
and timeline sinks of `sinks.py:209-248, 341-418`: same sink contract
(`name`, `consumes`, `on_start`, `on_streams`, `on_diagnostics`, `on_finish`),
same duplicate-name and missing-registry errors, same `PipelineResult` /
`IntervalStats` shapes.  The difference is where the work happens: the
decode -> mux -> pair -> tally/timeline loop runs as CUDA kernels
(csrc/engine.cu) instead of a per-event Python loop.

Supported sinks: TallySink and TimelineSink from this package, plus any sink
that does not override `on_message` (diagnostics-only sinks).  Sinks that
need per-message callbacks are rejected with UnsupportedTraceError -- there
is no CPU fallback path.
"""

from __future__ import annotations

import json
import os
import threading
from dataclasses import dataclass, field

from .errors import HapitraceError, PipelineError, UnsupportedTraceError
from .registry import SchemaRegistry
from .tally import TallyReport
from .tracefile import RECORD_HEADER, RawStream, encode_record, stream_bytes

END_OF_STREAM = "end_of_stream"


@dataclass(frozen=True)
class Message:
    kind: str
    event: object = None
    span: object = None
    sample: object = None


@dataclass(frozen=True)
class Span:
    name: str
    kind: str
    hostname: str
    pid: int
    tid: int
    start_ns: int
    end_ns: int
    entry_payload: dict = field(default_factory=dict)
    exit_payload: dict = field(default_factory=dict)
    result: int = 0
    truncated: bool = False

    @property
    def duration_ns(self) -> int:
        return self.end_ns - self.start_ns


@dataclass
class IntervalStats:
    events_in: int = 0
    passed: int = 0
    host_spans: int = 0
    truncated_spans: int = 0
    device_spans: int = 0
    samples: int = 0
    orphan_exits: int = 0

    def converted_events(self) -> int:
        return 2 * self.host_spans + self.truncated_spans + self.device_spans + self.samples


class Sink:
    """Base class for analysis sinks (pipeline.py:250-263)."""

    name = "sink"
    consumes = "intervals"

    def on_start(self, registry):
        pass

    def on_message(self, msg):
        pass

    def on_finish(self):
        return None


@dataclass
class PipelineResult:
    sink_results: dict
    stats: IntervalStats
    orphans: list = field(default_factory=list)
    timing: dict = field(default_factory=dict)

    def __getitem__(self, sink_name):
        return self.sink_results[sink_name]


class TallySink(Sink):
    """Tally sink whose fold runs on the GPU (sinks.py:209-248 semantics)."""

    name = "tally"
    consumes = "intervals"

    def on_start(self, registry):
        self.report = TallyReport(fingerprint=registry.fingerprint,
                                  backends=(f"BACKEND_{registry.api_name.upper()}",))

    def on_message(self, msg):
        raise UnsupportedTraceError("hapigpu's TallySink is fed by the GPU engine through run_pipeline")

    def _gpu_result(self, report: TallyReport):
        self.report = report

    def on_finish(self) -> TallyReport:
        return self.report


class TimelineSink(Sink):
    """Chrome-trace timeline whose JSON bytes are produced on the GPU (sinks.py:341-418)."""

    name = "timeline"
    consumes = "intervals"

    def __init__(self, out_path=None, device_index: int = 0, objects: bool = True):
        """objects=False: on_finish returns the JSON bytes instead of the parsed object list (the
        reference returns the list, sinks.py:414-418; parsing GBs of JSON on the host is optional)."""
        self.out_path = out_path
        self.device_index = device_index
        self.objects = objects
        self._bytes = b"[]"

    def on_message(self, msg):
        raise UnsupportedTraceError("hapigpu's TimelineSink is fed by the GPU engine through run_pipeline")

    def _gpu_result(self, blob: bytes):
        self._bytes = blob

    @property
    def json_bytes(self) -> bytes:
        return self._bytes

    def on_finish(self):
        if self.out_path is not None:
            with open(self.out_path, "wb") as fh:
                fh.write(self._bytes)
        return json.loads(self._bytes) if self.objects else self._bytes


class PrettyPrintSink(Sink):
    """One text line per event in mux order, rendered on the GPU (sinks.py:66-106 semantics):
    ``HH:MM:SS.nnnnnnnnn - <hostname> - vpid: P, vtid: T - <schema>: { f: v, ... }``."""

    name = "pretty"
    consumes = "events"

    def __init__(self, write=None):
        self._write = write
        self._lines: list = []

    def on_start(self, registry):
        self._registry = registry

    def on_message(self, msg):
        raise UnsupportedTraceError("hapigpu's PrettyPrintSink is fed by the GPU engine through run_pipeline")

    def on_finish(self) -> str:
        return "\n".join(self._lines) + ("\n" if self._lines else "")


def _is_pretty(sink) -> bool:
    """This package's PrettyPrintSink, or the reference's (same name and state: _write, _lines)."""
    return isinstance(sink, PrettyPrintSink) or (
        type(sink).__name__ == "PrettyPrintSink" and hasattr(sink, "_lines") and hasattr(sink, "_write"))


def _feed_pretty(sink, text: bytes):
    lines = text.decode("utf-8").split("\n")[:-1] if text else []
    if sink._write is not None:
        for line in lines:
            sink._write(line)
    else:
        sink._lines = lines


def _is_passive(sink) -> bool:
    """A sink that never looks at messages: no on_message, or one inherited unchanged from a base
    class named ``Sink`` (this package's or the reference's, pipeline.py:250-263)."""
    if not hasattr(sink, "on_message"):
        return True
    for klass in type(sink).__mro__:
        if "on_message" in klass.__dict__:
            return klass is Sink or (klass.__name__ == "Sink" and _is_noop(klass.__dict__["on_message"]))
    return True


def _is_noop(fn) -> bool:
    code = getattr(fn, "__code__", None)
    if code is None:
        return False
    # a body that is just `pass` (or a docstring) compiles to RETURN_CONST None
    import dis

    ops = [i.opname for i in dis.get_instructions(code) if i.opname not in ("RESUME", "NOP")]
    return ops in (["RETURN_CONST"], ["LOAD_CONST", "RETURN_VALUE"])


# ---------------------------------------------------------------------------
# sources


def _stream_label(cur, idx):
    name = getattr(cur, "name", None)
    if name:
        return name
    host = getattr(cur, "hostname", None)
    if host is not None:
        return f"{host}/{getattr(cur, 'pid', '?')}/{getattr(cur, 'tid', '?')}"
    return f"input[{idx}]"


def _raw_from_records(cursors, registry):
    """Encode in-memory record iterables (pipeline.py:286 list sources) to stream bytes."""
    raws, labels = [], []
    for idx, cur in enumerate(cursors):
        recs = list(cur)
        label = _stream_label(cur, idx)
        idents = {(r.hostname, r.pid, r.tid) for r in recs}
        if len(idents) > 1:
            raise UnsupportedTraceError(f"stream {label} mixes record identities {sorted(map(str, idents))}")
        host, pid, tid = idents.pop() if idents else (None, None, None)
        body = []
        for r in recs:
            if r.timestamp_ns is None:
                raise UnsupportedTraceError("records without timestamps")
            schema = registry.by_id.get(r.schema_id)
            if schema is None:
                raise UnsupportedTraceError(f"record with unknown schema id {r.schema_id}")
            try:
                body.append(encode_record(schema, r.timestamp_ns, r.payload))
            except Exception as e:  # noqa: BLE001
                raise UnsupportedTraceError(f"payload does not match its schema: {e}") from None
        raws.append(RawStream(host, pid, tid, label, stream_bytes(body) if recs else b""))
        labels.append(label)
    # mux order: (hostname or "", pid or 0, tid or 0, input index)  (pipeline.py:88-91)
    order = sorted(range(len(raws)), key=lambda i: (raws[i].hostname or "", raws[i].pid or 0, raws[i].tid or 0, i))
    return merge_same_identity([raws[i] for i in order])


def _walk(raw):
    """(offsets, timestamps) of every record of a stream; None if a header or payload is cut."""
    data, off, offs, tss = raw.data, 16, [], []
    n = len(data)
    while off < n:
        if off + 16 > n:
            return None
        _, ts, plen = RECORD_HEADER.unpack_from(data, off)
        if off + 16 + plen > n:
            return None
        offs.append(off)
        tss.append(ts)
        off += 16 + plen
    return offs, tss


def merge_same_identity(raws):
    """Streams that share one (hostname, pid, tid) identity share one LIFO stack in the reference
    (pipeline.py:156-161) and meet in the muxer by (ts, seq, input index) (pipeline.py:88-91).  The
    engine pairs per stream, so such streams are merged here into one stream in exactly that order.
    ``raws`` is in mux order (identity, then input index); a group whose records cannot be walked
    or are not timestamp-monotone (the reference would raise mid-run) is refused."""
    out, i = [], 0
    while i < len(raws):
        j = i + 1
        key = (raws[i].hostname, raws[i].pid, raws[i].tid)
        while j < len(raws) and (raws[j].hostname, raws[j].pid, raws[j].tid) == key:
            j += 1
        if j - i == 1:
            out.append(raws[i])
            i = j
            continue
        group = [r for r in raws[i:j] if r.data]
        if len(group) <= 1:
            out.append(group[0] if group else raws[i])
            i = j
            continue
        walks = []
        for r in group:
            w = _walk(r)
            if w is None or any(b < a for a, b in zip(w[1], w[1][1:])):
                raise UnsupportedTraceError(
                    f"streams sharing identity {key} need a clean, timestamp-ordered record walk to be merged")
            walks.append(w)
        import heapq

        heap = [(w[1][0], 0, g) for g, w in enumerate(walks) if w[0]]
        heapq.heapify(heap)
        parts = [group[0].data[:16]]
        while heap:
            ts, seq, g = heapq.heappop(heap)
            offs, tss = walks[g]
            a = offs[seq]
            b = offs[seq + 1] if seq + 1 < len(offs) else len(group[g].data)
            parts.append(group[g].data[a:b])
            if seq + 1 < len(offs):
                heapq.heappush(heap, (tss[seq + 1], seq + 1, g))
        out.append(RawStream(key[0], key[1], key[2], group[0].name, b"".join(parts), group[0].info))
        i = j
    return out


def _resolve_source(source, registry):
    if hasattr(source, "dir") and (hasattr(source, "metadata") or hasattr(source, "file_streams")):
        # a trace directory (ours or the reference's TraceReader): the engine reads the files itself
        from .tracefile import open_trace_reader

        ours = source if hasattr(source, "file_streams") else open_trace_reader(source.dir)
        return merge_same_identity(ours.file_streams()), ours.stream_infos()
    if hasattr(source, "raw_streams"):
        return (merge_same_identity(source.raw_streams()),
                source.stream_infos() if hasattr(source, "stream_infos") else None)
    cursors = source.streams() if hasattr(source, "streams") else list(source)
    infos = source.stream_infos() if hasattr(source, "stream_infos") else None
    return _raw_from_records(cursors, registry), infos


# ---------------------------------------------------------------------------

_engines = threading.local()


def default_engine():
    eng = getattr(_engines, "engine", None)
    if eng is None:
        from .engine import Engine

        eng = Engine()
        _engines.engine = eng
    return eng


def run_pipeline(source, sinks=(), registry=None, engine=None, distributed=False) -> PipelineResult:
    """One GPU pass: decode, mux-order semantics, interval pairing, sinks' results.

    ``distributed``: False (this process's GPU does the whole trace), True (the default
    torch.distributed group) or a ProcessGroup: every rank calls run_pipeline on the same source,
    owns the streams `distributed.partition_streams` gives it, and every rank returns the result of
    the whole trace (streams per rank, last-ts and tally merges as collectives)."""
    if registry is None:
        registry = getattr(source, "registry", None)
        if registry is None:
            raise PipelineError("a registry is required when source is not a TraceReader")
    if not isinstance(registry, SchemaRegistry):  # e.g. a reference registry object
        registry = SchemaRegistry.from_dict(registry.to_dict())
    comm = None
    if distributed is not False:
        from .distributed import Comm

        comm = Comm(None if distributed is True else distributed)
        if comm.world == 1 and os.environ.get("HAPIGPU_COLLECTIVES") != "1":
            comm = None
    if comm is None:
        raws, infos = _resolve_source(source, registry)
    else:
        shard = _resolve_sharded(source, registry, comm)
        infos = shard.infos
    names = [s.name for s in sinks]
    if len(set(names)) != len(names):
        raise PipelineError(f"duplicate sink names: {names}")
    tally = [s for s in sinks if isinstance(s, TallySink)]
    timeline = [s for s in sinks if isinstance(s, TimelineSink)]
    pretty = [s for s in sinks if _is_pretty(s)]
    from .validation import ValidationSink

    validate = [s for s in sinks if isinstance(s, ValidationSink)]
    if len(validate) > 1:
        raise UnsupportedTraceError("several ValidationSinks in one run")
    for s in sinks:
        if not isinstance(s, (TallySink, TimelineSink, ValidationSink)) and not _is_pretty(s) and not _is_passive(s):
            raise UnsupportedTraceError(
                f"sink {s.name!r} needs per-message callbacks; hapigpu serves TallySink/TimelineSink/PrettyPrintSink")
    # in a multi-rank run the timeline is merged across ranks (rank 0 formats it, ShardedRun.timeline);
    # the event sinks (every record in global mux order) are served by rank 0 from the whole trace;
    # the other ranks return None for these sinks
    ordered = timeline + pretty + validate
    device_index = {s.device_index for s in timeline}
    if len(device_index) > 1:
        raise UnsupportedTraceError("several TimelineSinks with different device_index")
    for s in sinks:
        s.on_start(registry)
        if infos is not None and hasattr(s, "on_streams"):
            s.on_streams(infos)
    eng = engine or default_engine()
    res = None
    try:
        if comm is None:
            labels = [r.name for r in raws]
            olabels = [f"{r.hostname}/{r.pid}/{r.tid}" for r in raws]
            res = eng.run(raws, registry, infos, want_timeline=bool(timeline), labels=labels,
                          orphan_labels=olabels, timeline_device_index=next(iter(device_index), 0),
                          want_events=bool(pretty), validation=validate[0].rules if validate else None)
        else:
            res = _run_sharded(eng, registry, shard, comm, timeline_device=next(iter(device_index), 0)
                               if timeline else None)
            if (pretty or validate) and res.error is None and comm.rank == 0:
                full, _ = _resolve_source(source, registry)
                r0 = eng.run(full, registry, infos, labels=[r.name for r in full],
                             orphan_labels=[f"{r.hostname}/{r.pid}/{r.tid}" for r in full], want_events=bool(pretty),
                             validation=validate[0].rules if validate else None)
                res.events, res.findings = r0.events, r0.findings
    finally:  # diagnostics reach interested sinks even when the run fails (pipeline.py:307-312)
        for s in sinks:
            hook = getattr(s, "on_diagnostics", None)
            if hook is not None:
                hook(list(res.orphans) if res is not None else [])
    if res.error is not None:
        raise res.error
    for s in tally:
        s._gpu_result(res.report)
    root = comm is None or comm.rank == 0
    if root:
        for s in timeline:
            s._gpu_result(res.timeline)
        for s in pretty:
            _feed_pretty(s, res.events)
        for s in validate:
            s._gpu_result(res.findings)
    results = {s.name: (s.on_finish() if root or not any(s is o for o in ordered) else None) for s in sinks}
    stats = IntervalStats(**res.stats)
    timing = {"kernel_ms": res.kernel_ms, "total_ms": res.total_ms, "h2d_bytes": res.h2d_bytes,
              "d2h_bytes": res.d2h_bytes, "launches": res.launches}
    return PipelineResult(results, stats, res.orphans, timing)


# ---------------------------------------------------------------------------
# multi-rank runs


@dataclass
class _Shard:
    raws: list            # this rank's streams (identity-merged), in mux order
    stream_global: list   # their global indices
    global_streams: list  # identities + labels of the whole trace, in mux order
    infos: list | None
    input_error: tuple | None  # (global index, exception) met while reading this rank's files


def _resolve_sharded(source, registry, comm) -> _Shard:
    """This rank's part of the source.  Trace directories: sizes from the file system, each rank reads
    only its own files (grouped by identity, pipeline.py:156-161).  In-memory sources: every rank holds
    the whole trace already and keeps its part."""
    from .distributed import partition_streams
    from .tracefile import open_trace_reader

    reader = None
    if hasattr(source, "dir") and (hasattr(source, "metadata") or hasattr(source, "stream_sizes")):
        reader = open_trace_reader(source.dir) if not hasattr(source, "stream_sizes") else source
    if reader is None:
        raws, infos = _resolve_source(source, registry)
        parts = partition_streams([len(r.data) for r in raws], comm.world)
        mine = parts[comm.rank]
        ids = [RawStream(r.hostname, r.pid, r.tid, r.name, b"") for r in raws]
        return _Shard([raws[i] for i in mine], mine, ids, infos, None)
    infos = reader.stream_infos()
    entries = reader._entries
    keys = [(e["hostname"], e["pid"], e["tid"]) for e in entries]
    parts = partition_streams(reader.stream_sizes(), comm.world, keys)
    mine = parts[comm.rank]
    ids = [RawStream(e["hostname"], e["pid"], e["tid"], e["file"], b"") for e in entries]
    raws, err = [], None
    for i in mine:
        try:
            raws.extend(reader.file_streams(select=[i]))
        except HapitraceError as e:
            err = (i, e)
            break
    if err is not None:
        return _Shard([], [], ids, infos, err)
    merged = merge_same_identity(raws)
    # a merged identity keeps the global index of its first file
    first = {}
    for i in mine:
        first.setdefault(keys[i], i)
    return _Shard(merged, [first[(r.hostname, r.pid, r.tid)] for r in merged], ids, infos, None)


def _run_sharded(eng, registry, shard, comm, timeline_device=None):
    """timeline_device: the TimelineSink's device_index when the run also builds the timeline (every
    rank's messages merged by rank 0, ShardedRun.timeline)."""
    from .abi import HG_WANT_TALLY, HG_WANT_TL_ITEMS
    from .distributed import ShardedRun
    from .engine import RunResult

    eng.set_registry(registry)
    eng.set_streams(shard.raws)
    run = ShardedRun(eng, registry, comm, shard.stream_global, shard.global_streams)
    want = HG_WANT_TALLY | (HG_WANT_TL_ITEMS if timeline_device is not None else 0)
    info = run.step(want=want, input_error=shard.input_error)
    labels = [s.name for s in shard.global_streams]
    olabels = [f"{s.hostname}/{s.pid}/{s.tid}" for s in shard.global_streams]
    report, stats, orphans, error = run.result(shard.infos, labels, olabels)
    timeline = None
    if timeline_device is not None and error is None:
        timeline = run.timeline(timeline_device)
    return RunResult(report, stats, orphans, error, timeline, info["phase1_ms"], info["device_ms"], info["h2d_bytes"],
                     info["d2h_bytes"], info["launches"])
