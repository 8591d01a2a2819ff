"""ctypes front of libztrc.so: the reference's five-function C writer binding, implemented natively
(include/ztrc_writer.h, csrc/ztrc_writer.c; reference: pkg/cinterpose/src/writer_binding.h:14-19,
pkg/docs/writer-binding.md).  Producer side of the traces the GPU engine analyses.

    export_metadata(registry, path)         # harness.py:132-143: the pregenerated metadata.json
    w = CWriter(); w.open(dir, path, cap)   # ztrc_open
    s = w.acquire()                         # ztrc_stream_acquire (per calling thread)
    w.emit(s, schema, ts, payload_dict)     # encode (tracefile.encode_payload) + ztrc_emit
    w.close()                               # ztrc_close: streams.json, complete: true
"""

from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

from .tracefile import encode_payload

HERE = Path(__file__).resolve().parent
LIB = HERE / "libztrc.so"
SRC = HERE / "csrc" / "ztrc_writer.c"
DEFAULT_BUFFER_CAPACITY = 1 << 16  # tracefile.py:43


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", str(LIB), str(SRC), "-lpthread"])
    return LIB


def export_metadata(registry, path, mode: str = "full", clock_kind: str = "monotonic-wall"):
    """Standalone metadata.json for out-of-process writers (harness.py:132-143)."""
    meta = {"format_version": 1, "api_name": registry.api_name, "mode": mode, "clock": clock_kind,
            "buffer_capacity": DEFAULT_BUFFER_CAPACITY, "complete": False, "registry": registry.to_dict()}
    Path(path).write_text(json.dumps(meta, indent=1))


class CWriter:
    def __init__(self):
        build()
        L = C.CDLL(str(LIB))
        L.ztrc_open.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64]
        L.ztrc_open.restype = C.c_int
        L.ztrc_stream_acquire.argtypes = []
        L.ztrc_stream_acquire.restype = C.c_void_p
        L.ztrc_emit.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_char_p, C.c_uint32]
        L.ztrc_emit.restype = C.c_int
        L.ztrc_clock_ns.restype = C.c_uint64
        L.ztrc_close.restype = C.c_int
        L.ztrc_debug_pause_drainer.argtypes = [C.c_int]
        self.L = L

    def open(self, directory, metadata_path, buffer_capacity=DEFAULT_BUFFER_CAPACITY) -> int:
        return self.L.ztrc_open(str(directory).encode(), str(metadata_path).encode(), buffer_capacity)

    def acquire(self):
        return self.L.ztrc_stream_acquire()

    def emit_raw(self, stream, schema_id: int, ts: int, payload: bytes) -> int:
        return self.L.ztrc_emit(stream, schema_id, ts, payload, len(payload))

    def emit(self, stream, schema, ts: int, payload: dict) -> int:
        return self.emit_raw(stream, schema.id, ts, encode_payload(schema, payload))

    def clock_ns(self) -> int:
        return self.L.ztrc_clock_ns()

    def close(self) -> int:
        return self.L.ztrc_close()

    def pause_drainer(self, paused: bool):
        self.L.ztrc_debug_pause_drainer(1 if paused else 0)
