"""Trace directories: index/metadata loading, raw stream bytes, record encoding.

The reader side follows `/root/reference/pkg/src/hapitrace/tracefile.py:477-553`
for everything that happens *before* record decoding (metadata.json
completeness check, registry rebuild, `(hostname, pid, tid)` sort of the
streams.json index, 16-byte file-header check with identical error text).
Record decoding itself is NOT done here: the raw bytes of every stream are
handed to the native engine, which decodes them on the GPU.

The encoder (`encode_record`) produces the record byte layout of
`tracefile.py:106-145` / docs/trace-format.md; it is used to build synthetic
traces and to feed in-memory record sources to the engine.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from pathlib import Path

from .errors import CorruptRecordError, HapitraceError, TraceDirectoryError
from .registry import SchemaRegistry

MAGIC = 0x54485049
FORMAT_VERSION = 1
FILE_HEADER = struct.Struct("<IIQ")
RECORD_HEADER = struct.Struct("<IQI")
_FIXED = {"u64": "<Q", "i64": "<q", "f64": "<d", "address": "<Q"}


@dataclass
class EventRecord:
    schema_id: int
    timestamp_ns: int | None
    payload: dict
    hostname: str | None = field(default=None, compare=False)
    pid: int | None = field(default=None, compare=False)
    tid: int | None = field(default=None, compare=False)


@dataclass(frozen=True)
class StreamInfo:
    hostname: str
    pid: int
    tid: int
    event_count: int
    dropped_count: int


@dataclass
class RawStream:
    """One stream file's identity plus its undecoded bytes (header included)."""

    hostname: str | None
    pid: int | None
    tid: int | None
    name: str  # label used in CorruptRecordError / MuxOrderingError
    data: bytes
    info: StreamInfo | None = None


class FileStream:
    """A stream file the engine stages itself (hg_add_stream_file: pinned double-buffered reads
    overlapped with the PCIe copies, csrc/ingest.cu); its 16-byte header is already checked.  The
    bytes are read on the host only if host-side code asks for ``data`` (error formatting)."""

    def __init__(self, hostname, pid, tid, name, path, size, info=None):
        self.hostname, self.pid, self.tid, self.name = hostname, pid, tid, name
        self.path, self.size, self.info = str(path), size, info
        self._data = None

    @property
    def data(self) -> bytes:
        if self._data is None:
            self._data = Path(self.path).read_bytes()
        return self._data


class TraceReader:
    """Finalized trace directory (tracefile.py:518-549 semantics up to decode)."""

    def __init__(self, directory):
        self.dir = Path(directory)
        meta_path = self.dir / "metadata.json"
        if not meta_path.exists():
            raise TraceDirectoryError(f"{self.dir} is not a trace directory (no metadata.json)")
        meta = json.loads(meta_path.read_text())
        if not meta.get("complete", False):
            raise TraceDirectoryError(f"{self.dir} holds an unfinalized or incomplete trace")
        self.metadata = meta
        self.mode = meta["mode"]
        self.clock_kind = meta["clock"]
        self.registry = SchemaRegistry.from_dict(meta["registry"])
        index = json.loads((self.dir / "streams.json").read_text())
        self._entries = sorted(index["streams"], key=lambda e: (e["hostname"], e["pid"], e["tid"]))

    def stream_infos(self) -> list:
        return [
            StreamInfo(e["hostname"], e["pid"], e["tid"], e["event_count"], e["dropped_count"])
            for e in self._entries
        ]

    def stream_sizes(self) -> list:
        """Byte size of every stream file in index order, without reading it (0 for unread files);
        the multi-GPU partitioner balances ranks by these."""
        return [(self.dir / e["file"]).stat().st_size if e["event_count"] else 0 for e in self._entries]

    def file_streams(self, select=None) -> list:
        """Like raw_streams, but the files are left for the engine to read (FileStream); only the
        16-byte headers are read here, in index order, for the reference's errors."""
        out = []
        select = None if select is None else set(select)
        for i, e in enumerate(self._entries):
            if select is not None and i not in select:
                continue
            name = e["file"]
            info = StreamInfo(e["hostname"], e["pid"], e["tid"], e["event_count"], e["dropped_count"])
            if not e["event_count"]:
                out.append(RawStream(e["hostname"], e["pid"], e["tid"], name, b"", info))
                continue
            path = self.dir / name
            with open(path, "rb") as fh:
                head = fh.read(FILE_HEADER.size)
            if not head:  # an empty file yields no records and is not checked (tracefile.py:489-490)
                out.append(RawStream(e["hostname"], e["pid"], e["tid"], name, b"", info))
                continue
            check_file_header(head, name)
            out.append(FileStream(e["hostname"], e["pid"], e["tid"], name, path, path.stat().st_size, info))
        return out

    def raw_streams(self, select=None) -> list:
        """Read every stream file (or the index positions in ``select``) in index order, validating
        its 16-byte header."""
        out = []
        select = None if select is None else set(select)
        for i, e in enumerate(self._entries):
            if select is not None and i not in select:
                continue
            name = e["file"]
            data = (self.dir / name).read_bytes() if e["event_count"] else b""
            check_file_header(data, name)
            info = StreamInfo(e["hostname"], e["pid"], e["tid"], e["event_count"], e["dropped_count"])
            out.append(RawStream(e["hostname"], e["pid"], e["tid"], name, data, info))
        return out

    # the reference API name; our "cursors" are raw byte streams
    streams = raw_streams


def open_trace_reader(directory) -> TraceReader:
    return TraceReader(directory)


def check_file_header(data: bytes, name: str):
    """File-header validation with the reference's messages (tracefile.py:491-499)."""
    if not data:
        return
    if len(data) < FILE_HEADER.size:
        raise CorruptRecordError("truncated file header", name, 0)
    magic, version, _ = FILE_HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise CorruptRecordError(f"bad magic 0x{magic:08x}", name, 0)
    if version != FORMAT_VERSION:
        raise CorruptRecordError(f"unsupported format version {version}", name, 4)


# ---------------------------------------------------------------------------
# encoding (trace production helpers; not on the analysis hot path)


def encode_payload(schema, payload: dict) -> bytes:
    parts = []
    if len(payload) != len(schema.fields):
        raise HapitraceError(
            f"schema {schema.name}: expected {len(schema.fields)} fields, got {len(payload)}"
        )
    for f in schema.fields:
        v = payload[f.name]
        code = _FIXED.get(f.kind)
        if code is not None:
            parts.append(struct.pack(code, v))
        else:
            b = v.encode("utf-8") if f.kind == "string" else bytes(v)
            parts.append(struct.pack("<I", len(b)))
            parts.append(b)
    return b"".join(parts)


def encode_record(schema, timestamp_ns: int, payload: dict) -> bytes:
    body = encode_payload(schema, payload)
    return RECORD_HEADER.pack(schema.id, timestamp_ns, len(body)) + body


def stream_bytes(records: bytes | list) -> bytes:
    """File header + concatenated records."""
    if isinstance(records, list):
        records = b"".join(records)
    return FILE_HEADER.pack(MAGIC, FORMAT_VERSION, 0) + records


def write_trace(directory, registry: SchemaRegistry, streams, mode="default", clock="virtual",
                buffer_capacity=65536):
    """Write a finalized trace directory in the reference layout (trace-format.md).

    ``streams``: iterable of dicts with hostname, pid, tid, data (full file bytes
    incl. header, or b""), event_count, dropped_count and optional file name.
    """
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    index = []
    for s in streams:
        fname = s.get("file") or f"stream_{s['pid']}_{s['tid']}.bin"
        if s["data"]:
            (d / fname).write_bytes(s["data"])
        index.append(
            {
                "hostname": s["hostname"],
                "pid": s["pid"],
                "tid": s["tid"],
                "event_count": s["event_count"],
                "dropped_count": s.get("dropped_count", 0),
                "file": fname,
            }
        )
    (d / "streams.json").write_text(json.dumps({"streams": index}, indent=1))
    meta = {
        "format_version": FORMAT_VERSION,
        "api_name": registry.api_name,
        "mode": mode,
        "clock": clock,
        "buffer_capacity": buffer_capacity,
        "complete": True,
        "registry": registry.to_dict(),
    }
    (d / "metadata.json").write_text(json.dumps(meta, indent=1))
    return d
