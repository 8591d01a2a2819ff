"""ctypes mirror of include/hapigpu.h and the registry flattening it consumes.

`flatten_registry` resolves, once per trace, everything the reference looks
up by name per event (pipeline.py:153-215, sinks.py:381-402): the event
class, the pairing key (function name -> dense id), the `result` field of
exits, the profiling fields of device records, the telemetry counter key.
Registry shapes the GPU decoder does not implement raise
UnsupportedTraceError here, before any work starts.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from .errors import HapitraceError, UnsupportedTraceError
from .registry import CLASS_CODE, COUNTER_KINDS, KIND_CODE, SchemaRegistry, parse_counter_key

HG_NUM_ROLES = 10
ROLE = {
    "result": 0, "device_start_ns": 1, "device_end_ns": 2, "name": 3, "tile": 4,
    "engine": 5, "command_kind": 6, "value": 7, "device": 8,
}
ROLE_RESULT, ROLE_START, ROLE_END, ROLE_NAME, ROLE_TILE, ROLE_ENGINE, ROLE_CMDKIND, ROLE_VALUE, ROLE_DEVICE = range(9)

FEED_NONE, FEED_ALWAYS, FEED_TIMELINE = 0, 1, 2

HG_OK, HG_TRACE_ERROR = 0, 1
HG_WANT_TALLY, HG_WANT_TIMELINE, HG_WANT_EVENTS, HG_WANT_VALIDATE, HG_WANT_TL_ITEMS = 1, 2, 4, 8, 16

(HG_ERR_TRUNC_HEADER, HG_ERR_TRUNC_PAYLOAD, HG_ERR_UNKNOWN_SCHEMA, HG_ERR_LEN_MISMATCH,
 HG_ERR_TRUNC_VAR, HG_ERR_TRAILING, HG_ERR_UTF8, HG_ERR_STRUCT, HG_ERR_ORDER, HG_ERR_FEED,
 HG_ERR_TELEMETRY, HG_ERR_RESULT) = range(1, 13)

_INT_KINDS = ("u64", "i64", "address")


class HgSchema(C.Structure):
    _fields_ = [
        ("id", C.c_uint32),
        ("event_class", C.c_uint8),
        ("n_fields", C.c_uint8),
        ("counter_kind", C.c_uint8),
        ("feed_error", C.c_uint8),
        ("function", C.c_int32),
        ("counter_domain", C.c_int32),
        ("kinds_offset", C.c_uint32),
        ("role", C.c_int16 * HG_NUM_ROLES),
    ]


class HgConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("tile_bytes", C.c_uint32), ("flags", C.c_uint32),
                ("timeline_device_index", C.c_int32)]


class HgStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "events_in", "passed", "host_spans", "truncated_spans", "device_spans", "samples", "orphan_exits")]


class HgTallyRow(C.Structure):
    _fields_ = [
        ("section", C.c_uint32), ("name_id", C.c_uint32),
        ("count", C.c_uint64), ("error_count", C.c_uint64),
        ("time_lo", C.c_uint64), ("time_hi", C.c_int64),
        ("min_lo", C.c_uint64), ("min_hi", C.c_int64),
        ("max_lo", C.c_uint64), ("max_hi", C.c_int64),
    ]


class HgOrphan(C.Structure):
    _fields_ = [("stream", C.c_uint32), ("function", C.c_int32), ("ts", C.c_uint64), ("seq", C.c_uint64)]


class HgValidationRule(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("pnext", C.c_int16), ("exec", C.c_int16), ("create", C.c_int16),
                ("rel", C.c_int16), ("rst", C.c_int16), ("result", C.c_int16)]


class HgFinding(C.Structure):
    _fields_ = [("rule", C.c_uint32), ("sid", C.c_uint32), ("stream", C.c_uint32), ("pad", C.c_uint32),
                ("pos", C.c_uint64), ("ts", C.c_uint64), ("subject_lo", C.c_uint64), ("subject_hi", C.c_int64)]


class HgTraceError(C.Structure):
    _fields_ = [("code", C.c_uint32), ("stream", C.c_uint32), ("seq", C.c_uint64), ("offset", C.c_uint64),
                ("ts", C.c_uint64), ("prev_ts", C.c_uint64), ("aux", C.c_uint64)]


def i128(lo: int, hi: int) -> int:
    return (hi << 64) | lo


@dataclass
class FlatRegistry:
    registry: SchemaRegistry
    schemas: C.Array            # HgSchema[n]
    kinds: bytes
    function_names: list        # id -> name (str or None)
    feed_errors: dict           # schema id -> zero-arg callable building the exception
    telemetry: dict             # schema id -> (counter kind str, domain)

    @property
    def n_schemas(self) -> int:
        return len(self.schemas)


def _feed_key_error(key):
    return lambda: KeyError(key)


def flatten_registry(registry: SchemaRegistry) -> FlatRegistry:
    by_id = registry.by_id  # later duplicates win (dict semantics)
    fn_ids: dict = {}
    fn_names: list = []
    kinds = bytearray()
    rows = []
    feed_errors = {}
    telemetry = {}

    def fn_id(name):
        if name not in fn_ids:
            fn_ids[name] = len(fn_names)
            fn_names.append(name)
        return fn_ids[name]

    for sid in sorted(by_id):
        s = by_id[sid]
        if sid < 0 or sid >= 1 << 32:
            continue  # cannot appear in a u32 record header
        if len(s.fields) > 255:
            raise UnsupportedTraceError(f"schema {s.name}: more than 255 fields")
        h = HgSchema()
        h.id = sid
        cls = CLASS_CODE.get(s.event_class, CLASS_CODE["meta"])  # unknown classes pass through
        h.event_class = cls
        h.n_fields = len(s.fields)
        h.kinds_offset = len(kinds)
        for f in s.fields:
            kinds.append(KIND_CODE.get(f.kind, KIND_CODE["blob"]))  # _SchemaCodec treats others as blob
        for r in range(HG_NUM_ROLES):
            h.role[r] = -1
        names = {}
        for i, f in enumerate(s.fields):
            names.setdefault(f.name, i)  # payload dict keeps the LAST duplicate; see below
        for i, f in enumerate(s.fields):
            names[f.name] = i
        kind_of = {f.name: f.kind for f in s.fields}
        h.function = -1
        if cls in (CLASS_CODE["host_entry"], CLASS_CODE["host_exit"]):
            h.function = fn_id(s.function)
        if cls == CLASS_CODE["host_exit"] and "result" in names:
            k = kind_of["result"]
            if k not in _INT_KINDS and k != "f64":
                raise UnsupportedTraceError(f"schema {s.name}: result field of kind {k}")
            h.role[ROLE_RESULT] = names["result"]
        if cls == CLASS_CODE["device_profiling"]:
            for key in ("name", "device_start_ns", "device_end_ns"):
                if key not in names:
                    feed_errors[sid] = _feed_key_error(key)
                    h.feed_error = FEED_ALWAYS
                    break
            if not h.feed_error:
                if kind_of["name"] != "string":
                    raise UnsupportedTraceError(f"schema {s.name}: device name of kind {kind_of['name']}")
                for key in ("device_start_ns", "device_end_ns"):
                    if kind_of[key] not in _INT_KINDS:
                        raise UnsupportedTraceError(f"schema {s.name}: {key} of kind {kind_of[key]}")
            for key in ("tile", "engine"):
                if key in names and kind_of[key] not in _INT_KINDS:
                    raise UnsupportedTraceError(f"schema {s.name}: {key} of kind {kind_of[key]}")
            if "command_kind" in names and kind_of["command_kind"] != "string":
                raise UnsupportedTraceError(f"schema {s.name}: command_kind of kind {kind_of['command_kind']}")
            for key in ("device_start_ns", "device_end_ns", "name", "tile", "engine", "command_kind"):
                if key in names:
                    h.role[ROLE[key]] = names[key]
        if cls == CLASS_CODE["telemetry_sample"]:
            try:
                counter, domain = parse_counter_key(s.name)
            except (HapitraceError, ValueError) as e:
                err = e
                feed_errors[sid] = lambda err=err: type(err)(*err.args)
                h.feed_error = FEED_ALWAYS
            else:
                h.counter_kind = COUNTER_KINDS.index(counter)
                h.counter_domain = domain if -(1 << 31) <= domain < (1 << 31) else -1
                telemetry[sid] = (counter, domain)
                for key in ("value", "device"):
                    if key not in names:
                        feed_errors[sid] = _feed_key_error(key)
                        h.feed_error = FEED_ALWAYS
                        break
                if not h.feed_error:
                    if kind_of["value"] not in _INT_KINDS and kind_of["value"] != "f64":
                        raise UnsupportedTraceError(f"schema {s.name}: telemetry value of kind {kind_of['value']}")
                    if kind_of["device"] not in _INT_KINDS:
                        raise UnsupportedTraceError(f"schema {s.name}: telemetry device of kind {kind_of['device']}")
                    h.role[ROLE_VALUE] = names["value"]
                    h.role[ROLE_DEVICE] = names["device"]
                    # no timeline track for this (counter, domain): only a timeline sink raises
                    from .timeline import COUNTER_TRACKS

                    if (counter, domain) not in COUNTER_TRACKS:
                        h.feed_error = FEED_TIMELINE
                        feed_errors[sid] = (
                            lambda c=counter, d=domain: HapitraceError(f"no timeline track for counter {c}|{d}")
                        )
        rows.append(h)
    arr = (HgSchema * len(rows))(*rows)
    return FlatRegistry(registry, arr, bytes(kinds), fn_names, feed_errors, telemetry)
