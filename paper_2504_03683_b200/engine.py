"""Engine: one GPU pipeline context (hg_ctx) behind a small Python class.

`Engine.run(raw_streams, registry, ...)` replaces the body of the reference's
`run_pipeline` for tally/timeline sinks (pipeline.py:275-314): it hands the
undecoded stream bytes to libhapigpu, which decodes, pairs and reduces them
on the GPU, and returns the reference objects (TallyReport, IntervalStats
values, orphan list) or the exception the reference would raise.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import native
from .abi import (
    HG_OK, HG_TRACE_ERROR, HG_WANT_EVENTS, HG_WANT_TALLY, HG_WANT_TIMELINE, HG_WANT_VALIDATE, HgConfig, HgFinding,
    HgValidationRule, HgOrphan, HgStats, HgTallyRow,
    HgTraceError, flatten_registry,
)
from .errors import EngineError, UnsupportedTraceError
from .tracefile import FileStream
from .results import build_report, error_key, first_error, make_exception, orphan_list, rows_from_native

HG_EUNSUPPORTED = -5
MERGE_STATS = 8  # IntervalStats counters + trace-error ranks at the head of the merge buffer (csrc/merge.cu)
OPT_PATH = 1
OPT_RANGE_BYTES = 2
PATH_AUTO, PATH_EXACT, PATH_FAST = 0, 1, 2


def _ident(v):
    """pid / tid for hg_add_stream: None travels as INT64_MIN (printed "None" by event sinks)."""
    return -(1 << 63) if v is None else int(v)


@dataclass
class RunResult:
    report: object | None
    stats: dict
    orphans: list
    error: BaseException | None
    timeline: bytes | None
    kernel_ms: float
    total_ms: float
    h2d_bytes: int
    d2h_bytes: int
    launches: int
    events: bytes | None = None
    findings: list | None = None


class Engine:
    """A GPU pipeline context bound to one CUDA device."""

    def __init__(self, device: int = 0, timeline_device_index: int = 0, seg_bytes: int = 0):
        self._L = native.lib()
        self._ctx = C.c_void_p()
        cfg = HgConfig(device=device, tile_bytes=seg_bytes, flags=0, timeline_device_index=timeline_device_index)
        rc = self._L.hg_create(C.byref(cfg), C.byref(self._ctx))
        if rc != HG_OK:
            msg = self._L.hg_last_error(self._ctx).decode() if self._ctx else "hg_create failed"
            self.close()
            raise EngineError(msg)
        self.device = device
        self._flat = None
        self._registry_key = None
        self._keep = []
        self._streams = []

    # -- lifecycle
    def close(self):
        if getattr(self, "_ctx", None):
            self._L.hg_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def _check(self, rc, what):
        if rc == HG_OK:
            return
        msg = self._L.hg_last_error(self._ctx).decode(errors="replace")
        if rc == HG_EUNSUPPORTED:
            raise UnsupportedTraceError(f"{what}: {msg}")
        raise EngineError(f"{what} failed ({rc}): {msg}")

    # -- inputs
    def set_registry(self, registry):
        if self._registry_key is registry:
            return self._flat
        flat = flatten_registry(registry)
        self._check(self._L.hg_set_registry(self._ctx, flat.schemas, flat.n_schemas, flat.kinds, len(flat.kinds),
                                            len(flat.function_names)), "hg_set_registry")
        names = [("" if n is None else str(n)).encode("utf-8") for n in flat.function_names]
        offs = [0]
        for b in names:
            offs.append(offs[-1] + len(b))
        blob = b"".join(names)
        null = bytes(1 if n is None else 0 for n in flat.function_names)
        n = len(names)
        self._check(self._L.hg_set_function_names(
            self._ctx, C.c_char_p(blob) if blob else None, (C.c_uint64 * (n + 1))(*offs),
            C.c_char_p(null) if null else None, n), "hg_set_function_names")
        self._set_schema_names(flat)
        self._flat = flat
        self._registry_key = registry
        return flat

    def _set_schema_names(self, flat):
        """EventSchema / FieldSpec names for event sinks (hg_set_schema_names), in flat order."""
        by_id = flat.registry.by_id
        schemas = [by_id[h.id] for h in flat.schemas]
        names = [s.name.encode("utf-8") for s in schemas]
        fields = [f.name.encode("utf-8") for s in schemas for f in s.fields]

        def blob(parts):
            offs = [0]
            for b in parts:
                offs.append(offs[-1] + len(b))
            return b"".join(parts), (C.c_uint64 * len(offs))(*offs)

        nb, no = blob(names)
        fb, fo = blob(fields)
        self._check(self._L.hg_set_schema_names(self._ctx, nb, no, len(names), fb, fo, len(fields)),
                    "hg_set_schema_names")
        self._event_ok = all(len({f.name for f in s.fields}) == len(s.fields) and
                             all(f.kind in ("u64", "i64", "f64", "address", "string", "blob") for f in s.fields)
                             for s in schemas)

    def set_streams(self, raw_streams):
        """raw_streams: RawStream list in mux order (hostname, pid, tid)."""
        self._check(self._L.hg_clear_streams(self._ctx), "hg_clear_streams")
        self._keep = []
        self._streams = list(raw_streams)
        for s in self._streams:
            if isinstance(s, FileStream):
                self.add_stream_file(s.hostname, s.pid, s.tid, s.path, 0, s.size)
            else:
                self.add_stream_ptr(s.hostname, s.pid, s.tid, s.data)
        self._set_flush_order()

    def _set_flush_order(self):
        """Truncated spans flush per stack in (str(hostname), pid, tid) order (pipeline.py:230); the
        streams are in (hostname or "", pid or 0, tid or 0) order -- they differ only around None."""
        idents = [(s.hostname, s.pid, s.tid) for s in self._streams]
        if not any(h is None for h, _, _ in idents):
            return
        order = sorted(range(len(idents)), key=lambda i: (str(idents[i][0]), idents[i][1] or 0, idents[i][2] or 0, i))
        if order == list(range(len(idents))):
            return
        rank = [0] * len(order)
        for r, i in enumerate(order):
            rank[i] = r
        self._check(self._L.hg_set_flush_order(self._ctx, (C.c_uint32 * len(rank))(*rank), len(rank)),
                    "hg_set_flush_order")

    def set_streams_pinned(self, idents, tensors):
        """Streams from pinned host tensors (torch.uint8); the next run copies them H2D."""
        from .tracefile import RawStream

        self._check(self._L.hg_clear_streams(self._ctx), "hg_clear_streams")
        self._keep = list(tensors)
        self._streams = [RawStream(h, p, t, "", b"") for h, p, t in idents]
        for (h, p, t), ten in zip(idents, tensors):
            self.add_stream_ptr(h, p, t, ten.data_ptr() if ten.numel() else 0, ten.numel())

    def add_stream_file(self, hostname, pid, tid, path, offset, size):
        """hg_add_stream_file: the engine reads the stream file itself (csrc/ingest.cu)."""
        h = hostname.encode() if hostname is not None else None
        self._check(self._L.hg_add_stream_file(self._ctx, h, _ident(pid), _ident(tid), str(path).encode(),
                                               offset, size), "hg_add_stream_file")

    def add_stream_device(self, hostname, pid, tid, tensor):
        """hg_add_stream_device: stream bytes already in this GPU's memory (a CUDA uint8 tensor)."""
        h = hostname.encode() if hostname is not None else None
        n = tensor.numel() * tensor.element_size()
        self._keep.append(tensor)
        self._check(self._L.hg_add_stream_device(self._ctx, h, _ident(pid), _ident(tid),
                                                 C.c_void_p(tensor.data_ptr() if n else 0), n),
                    "hg_add_stream_device")

    def set_streams_device(self, idents, tensors):
        """Streams whose bytes are CUDA tensors on this engine's GPU (GDS, another kernel, a peer copy)."""
        from .tracefile import RawStream

        self._check(self._L.hg_clear_streams(self._ctx), "hg_clear_streams")
        self._keep = []
        self._streams = [RawStream(h, p, t, "", b"") for h, p, t in idents]
        for (h, p, t), ten in zip(idents, tensors):
            self.add_stream_device(h, p, t, ten)

    def ingest_stats(self) -> dict:
        """hg_ingest_stats of the last staging: bytes per source kind, host ms, threads."""
        a, b, c, d = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        ms, th = C.c_float(), C.c_uint32()
        self._check(self._L.hg_ingest_stats(self._ctx, C.byref(a), C.byref(b), C.byref(c), C.byref(d), C.byref(ms),
                                            C.byref(th)), "hg_ingest_stats")
        return {"pinned_bytes": a.value, "pageable_bytes": b.value, "file_bytes": c.value, "device_bytes": d.value,
                "ms": ms.value, "threads": th.value}

    def events_text(self) -> bytes:
        """PrettyPrintSink's text of the last HG_WANT_EVENTS run (every record in mux order)."""
        n = C.c_uint64()
        self._check(self._L.hg_events_size(self._ctx, C.byref(n)), "hg_events_size")
        buf = (C.c_char * max(n.value, 1))()
        self._check(self._L.hg_get_events(self._ctx, buf, n.value), "hg_get_events")
        return bytes(buf)[: n.value]

    def event_order(self):
        """The mux order of the last HG_WANT_EVENTS run: (stream index, record index) per event."""
        n = C.c_uint64()
        self._check(self._L.hg_get_event_order(self._ctx, None, None, 0, C.byref(n)), "hg_get_event_order")
        st = (C.c_uint32 * max(n.value, 1))()
        sq = (C.c_uint64 * max(n.value, 1))()
        self._check(self._L.hg_get_event_order(self._ctx, st, sq, n.value, C.byref(n)), "hg_get_event_order")
        return list(zip(list(st)[: n.value], list(sq)[: n.value]))

    def set_validation_rules(self, rows):
        arr = (HgValidationRule * max(len(rows), 1))(*rows)
        self._check(self._L.hg_set_validation_rules(self._ctx, arr, len(rows)), "hg_set_validation_rules")

    def findings_raw(self):
        n = C.c_uint64()
        self._check(self._L.hg_get_findings(self._ctx, None, 0, C.byref(n)), "hg_get_findings")
        arr = (HgFinding * max(n.value, 1))()
        self._check(self._L.hg_get_findings(self._ctx, arr, n.value, C.byref(n)), "hg_get_findings")
        return list(arr)[: n.value]

    def events_ms(self) -> float:
        ms = C.c_float()
        self._check(self._L.hg_events_ms(self._ctx, C.byref(ms)), "hg_events_ms")
        return ms.value

    def add_stream_ptr(self, hostname, pid, tid, data, size=None):
        """data: bytes (kept alive here) or an integer host address (+ size)."""
        if isinstance(data, int):
            ptr, n = (data or None), size
        else:
            buf = C.c_char_p(data) if data else None
            self._keep.append(data)
            ptr, n = (C.cast(buf, C.c_void_p).value if buf else None), len(data)
        h = hostname.encode() if hostname is not None else None  # NULL: hostname None
        self._check(self._L.hg_add_stream(self._ctx, h, _ident(pid), _ident(tid), ptr, n), "hg_add_stream")

    def stage(self):
        self._check(self._L.hg_stage(self._ctx), "hg_stage")

    def set_option(self, key: int, value: int):
        """hg_set_option: OPT_PATH (0 auto, 1 exact, 2 single pass only), OPT_RANGE_BYTES."""
        self._check(self._L.hg_set_option(self._ctx, key, value), "hg_set_option")

    def last_path(self):
        """(path of the last phase 1: 1 single pass / 0 exact, discarded single passes so far, range bytes)"""
        p, f, r = C.c_uint32(), C.c_uint64(), C.c_uint32()
        self._check(self._L.hg_last_path(self._ctx, C.byref(p), C.byref(f), C.byref(r)), "hg_last_path")
        return p.value, f.value, r.value

    # -- execution
    def run_raw(self, want=HG_WANT_TALLY):
        rc = self._L.hg_run(self._ctx, want)
        if rc not in (HG_OK, HG_TRACE_ERROR):
            self._check(rc, "hg_run")
        return rc

    def set_timeline_device(self, index: int):
        self._check(self._L.hg_set_timeline_device(self._ctx, int(index)), "hg_set_timeline_device")

    def tensor_device(self):
        import torch

        return torch.device("cuda", self.device)

    # -- split run for sharded (multi-GPU) use: distributed.ShardedRun
    def run_local(self, want=HG_WANT_TALLY):
        """hg_run_local: phase 1 over this context's streams; raises on an engine failure."""
        self._check(self._L.hg_run_local(self._ctx, want), "hg_run_local")

    def local_flags(self) -> int:
        """hg_local_flags after run_local: 1 = a device span beyond +-2^63 ns."""
        f = C.c_uint32()
        self._check(self._L.hg_local_flags(self._ctx, C.byref(f)), "hg_local_flags")
        return f.value

    def local_last_ts(self) -> int:
        last = C.c_uint64()
        self._check(self._L.hg_local_last_ts(self._ctx, C.byref(last), None), "hg_local_last_ts")
        return last.value

    def finish(self, global_last_ts: int) -> int:
        """hg_finish: composition and truncation at the global last timestamp; HG_OK or HG_TRACE_ERROR."""
        rc = self._L.hg_finish(self._ctx, global_last_ts)
        if rc not in (HG_OK, HG_TRACE_ERROR):
            self._check(rc, "hg_finish")
        return rc

    def merge_size(self, n_dev_global: int, n_streams_global: int):
        """(total int64 elements, elements of the SUM region) of the merge buffer (csrc/merge.cu)."""
        sum_n = C.c_uint64()
        total = self._L.hg_merge_size(len(self._flat.function_names), n_dev_global, n_streams_global,
                                      C.byref(sum_n))
        return total, sum_n.value

    def merge_export(self, dst_ptr: int, dev_map, n_dev_global: int, stream_global, n_streams_global: int):
        """hg_merge_export into device memory at dst_ptr (a torch tensor on this engine's GPU)."""
        dm = (C.c_uint32 * max(len(dev_map), 1))(*dev_map)
        sg = (C.c_uint32 * max(len(stream_global), 1))(*stream_global)
        self._check(self._L.hg_merge_export(self._ctx, C.c_void_p(dst_ptr), dm, len(dev_map), n_dev_global, sg,
                                            n_streams_global), "hg_merge_export")

    def merge_import(self, host_ptr: int, names, n_streams_global: int):
        """hg_merge_import from host memory: the reduced buffer plus the global device-name list."""
        enc = [n.encode("utf-8") for n in names]
        offs = [0]
        for b in enc:
            offs.append(offs[-1] + len(b))
        self._check(self._L.hg_merge_import(self._ctx, C.c_void_p(host_ptr), len(names), n_streams_global,
                                            b"".join(enc), (C.c_uint64 * len(offs))(*offs)), "hg_merge_import")

    def timing(self):
        k, t = C.c_float(), C.c_float()
        h2d, d2h, nl = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._L.hg_last_timing(self._ctx, C.byref(k), C.byref(t), C.byref(h2d), C.byref(d2h), C.byref(nl))
        return k.value, t.value, h2d.value, d2h.value, nl.value

    def stats(self) -> dict:
        st = HgStats()
        self._check(self._L.hg_get_stats(self._ctx, C.byref(st)), "hg_get_stats")
        return {k: getattr(st, k) for k, _ in HgStats._fields_}

    def tally_rows(self):
        n = C.c_uint64()
        self._check(self._L.hg_get_tally(self._ctx, None, 0, C.byref(n)), "hg_get_tally")
        rows = (HgTallyRow * max(n.value, 1))()
        self._check(self._L.hg_get_tally(self._ctx, rows, n.value, C.byref(n)), "hg_get_tally")
        return rows_from_native(list(rows)[: n.value])

    def device_names(self):
        nn, nb = C.c_uint64(), C.c_uint64()
        self._check(self._L.hg_get_device_names(self._ctx, None, 0, None, 0, C.byref(nn), C.byref(nb)), "names")
        buf = (C.c_char * max(nb.value, 1))()
        offs = (C.c_uint64 * (nn.value + 1))()
        self._check(self._L.hg_get_device_names(self._ctx, buf, nb.value, offs, nn.value + 1, C.byref(nn),
                                                C.byref(nb)), "names")
        raw = bytes(buf)[: nb.value]
        return [raw[offs[i]: offs[i + 1]].decode("utf-8") for i in range(nn.value)]

    def stream_spans(self):
        n = len(self._streams)
        arr = (C.c_uint64 * max(n, 1))()
        self._check(self._L.hg_get_stream_spans(self._ctx, arr, n), "hg_get_stream_spans")
        return list(arr)[:n]

    def orphans_raw(self):
        n = C.c_uint64()
        self._check(self._L.hg_get_orphans(self._ctx, None, 0, C.byref(n)), "hg_get_orphans")
        arr = (HgOrphan * max(n.value, 1))()
        self._check(self._L.hg_get_orphans(self._ctx, arr, n.value, C.byref(n)), "hg_get_orphans")
        return list(arr)[: n.value]

    def errors_raw(self):
        n = C.c_uint64()
        self._check(self._L.hg_get_trace_errors(self._ctx, None, 0, C.byref(n)), "hg_get_trace_errors")
        arr = (HgTraceError * max(n.value, 1))()
        self._check(self._L.hg_get_trace_errors(self._ctx, arr, n.value, C.byref(n)), "hg_get_trace_errors")
        return list(arr)[: n.value]

    def phase_timing(self):
        """(walk, chain, decode) device ms of the last run's phase 1."""
        a, b, c = C.c_float(), C.c_float(), C.c_float()
        self._check(self._L.hg_phase_timing(self._ctx, C.byref(a), C.byref(b), C.byref(c)), "hg_phase_timing")
        return a.value, b.value, c.value

    def timeline_ms(self) -> float:
        ms = C.c_float()
        self._check(self._L.hg_timeline_ms(self._ctx, C.byref(ms)), "hg_timeline_ms")
        return ms.value

    def timeline_bytes(self) -> bytes:
        n = C.c_uint64()
        self._check(self._L.hg_timeline_size(self._ctx, C.byref(n)), "hg_timeline_size")
        buf = (C.c_char * max(n.value, 1))()
        self._check(self._L.hg_get_timeline(self._ctx, buf, n.value), "hg_get_timeline")
        return bytes(buf)[: n.value]

    # -- the drop-in
    def run(self, raw_streams, registry, stream_infos=None, want_timeline=False, labels=None,
            orphan_labels=None, timeline_device_index=0, reuse_streams=False, want_events=False,
            validation=None) -> RunResult:
        """validation: ValidationRules of a ValidationSink (its findings land in RunResult.findings)."""
        """reuse_streams: run again over the streams of the previous call (still resident in HBM)."""
        flat = self.set_registry(registry)
        self._check(self._L.hg_set_timeline_device(self._ctx, int(timeline_device_index)), "hg_set_timeline_device")
        if not reuse_streams:
            self.set_streams(raw_streams)
        if want_events and not self._event_ok:
            raise UnsupportedTraceError("event sinks: a schema with duplicate field names or an unknown field kind")
        want = HG_WANT_TALLY | (HG_WANT_TIMELINE if want_timeline else 0) | (HG_WANT_EVENTS if want_events else 0)
        if validation is not None:
            from .validation import rule_rows

            self.set_validation_rules(rule_rows(validation, flat))
            want |= HG_WANT_VALIDATE
        rc = self.run_raw(want)
        k, t, h2d, d2h, nl = self.timing()
        stats = self.stats()
        if orphan_labels is None:
            orphan_labels = [f"{s.hostname}/{s.pid}/{s.tid}" for s in raw_streams]
        orphans = self.orphans_raw()
        error = None
        if rc == HG_TRACE_ERROR:
            cands = self.errors_raw()
            e = first_error(cands)
            cut = {}
            for c in cands:
                if c.code in (1, 2, 3, 4, 5, 6, 7, 8, 9) and (c.stream not in cut or c.seq < cut[c.stream]):
                    cut[c.stream] = c.seq
            named = raw_streams[e.stream]
            if labels is not None:
                from .tracefile import RawStream

                named = RawStream(named.hostname, named.pid, named.tid, labels[e.stream], named.data, named.info)
            error = make_exception(e, named, flat)
            olist = orphan_list(orphans, orphan_labels, flat, cutoff=error_key(e), cut_streams=cut)
            return RunResult(None, stats, olist, error, None, k, t, h2d, d2h, nl)
        olist = orphan_list(orphans, orphan_labels, flat)
        idents = [(s.hostname, s.pid, s.tid) for s in raw_streams]
        report = build_report(flat, self.tally_rows(), self.device_names(), stream_infos, idents, self.stream_spans())
        timeline = self.timeline_bytes() if want_timeline else None
        r = RunResult(report, stats, olist, None, timeline, k, t, h2d, d2h, nl)
        if want_events:
            r.events = self.events_text()
        if validation is not None:
            from .validation import findings_from_native

            r.findings = findings_from_native(self.findings_raw(), validation, raw_streams)
        return r
