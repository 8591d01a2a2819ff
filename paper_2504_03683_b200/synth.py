"""Synthetic trace workloads, generated natively.

Bench and test input only: the C generator (csrc/synth.c) writes stream files
in the reference byte format; tests/golden/make_golden.py decodes C-generated
fixtures with the reference reader to pin the encoding.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path

from .abi import ROLE_CMDKIND, ROLE_NAME, flatten_registry
from .registry import SchemaRegistry, TELEMETRY_COUNTERS
from .tracefile import RawStream, StreamInfo, write_trace

HERE = Path(__file__).resolve().parent
SRC = HERE / "csrc" / "synth.c"
LIB = HERE / "libhapisynth.so"

PID_BASE = 4202000  # harness.py:27-28
PID_STRIDE = 100
SAMPLER_TID_OFFSET = 99  # sampler.py:31

# test pool: includes non-ASCII names to exercise UTF-8 validation and JSON escaping
KERNEL_POOL_SMALL = ["lrn_conv1d", "gemm_f32", "reduce_sum", "softmax", "ядро_σ", "カーネル", "axpy", "stencil7"]
# benchmark pool: kernel names are C/C++ symbols in real traces (ASCII)
KERNEL_POOL_ASCII = ["lrn_conv1d", "gemm_f32", "reduce_sum", "softmax", "layernorm_bwd", "attention_fwd", "axpy",
                     "stencil7"]


def kernel_pool(n: int, ascii_only: bool = False) -> list:
    base = list(KERNEL_POOL_ASCII if ascii_only else KERNEL_POOL_SMALL)
    i = 0
    while len(base) < n:
        base.append(f"kernel_{i:04d}_{'abcdefgh'[i % 8] * (1 + i % 5)}")
        i += 1
    return base[:n]


class SynthParams(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("n_events", C.c_uint64), ("max_depth", C.c_uint32), ("pad0", C.c_uint32),
        ("gap_lo", C.c_uint64), ("gap_hi", C.c_uint64), ("ts0_hi", C.c_uint64),
        ("push_p", C.c_double), ("err_p", C.c_double), ("prof_p", C.c_double), ("meta_p", C.c_double),
        ("orphan_p", C.c_double), ("mismatch_p", C.c_double), ("zipf_s", C.c_double),
        ("n_layers", C.c_uint32), ("close_at_end", C.c_int32), ("meta_sid", C.c_int32),
        ("dev_off_hi", C.c_uint64), ("dev_lo", C.c_int64), ("dev_hi", C.c_int64),
    ]


class SynthFn(C.Structure):
    _fields_ = [("entry_sid", C.c_uint32), ("exit_sid", C.c_uint32), ("prof_sid", C.c_int32),
                ("layer", C.c_uint32), ("memcpy", C.c_int32)]


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", str(LIB), str(SRC), "-lm"])
    return LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.synth_stream.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_char_p, C.c_void_p, C.c_uint32,
                                   C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.synth_stream.restype = C.c_int
        L.synth_sampler.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.synth_sampler.restype = C.c_int
        L.synth_last_ts.argtypes = [C.c_char_p, C.c_uint64]
        L.synth_last_ts.restype = C.c_uint64
        _lib = L
    return _lib


def ze_registry() -> SchemaRegistry:
    """The bundled mock Level-Zero registry (38 schemas, fingerprint f2471ee59addbe96)."""
    return SchemaRegistry.from_dict(json.loads((HERE / "data" / "ze_registry.json").read_text()))


def layered_registry(n_top: int = 1000, n_low: int = 1000, top="sycl", low="ze", api="sycl_ze") -> SchemaRegistry:
    """Two-layer API model registry (config C4): top-layer functions wrap lower-layer ones."""
    schemas = []

    def add(name, cls, fields, fn=None):
        schemas.append({"id": len(schemas), "name": f"{api}:{name}", "class": cls, "function": fn,
                        "mode_mask": ["default", "full", "minimal"],
                        "fields": [{"name": n, "kind": k, "origin": o} for n, k, o in fields]})

    fns = [f"{top}Api{i:04d}" for i in range(n_top)] + [f"{low}Api{i:04d}" for i in range(n_low)]
    for i, fn in enumerate(fns):
        entry = [("handle", "address", "stack_arg"), ("size", "u64", "stack_arg")]
        if i % 7 == 0:
            entry.append(("flags", "i64", "stack_arg"))
        add(f"{fn}_entry", "host_entry", entry, fn)
        add(f"{fn}_exit", "host_exit", [("result", "i64", "result")], fn)
    add("annotation", "meta", [("label", "string", "stack_arg")])
    for key, _ in TELEMETRY_COUNTERS:
        add(f"telemetry_{key}", "telemetry_sample", [("device", "u64", "telemetry"), ("value", "f64", "telemetry")])
    return SchemaRegistry.from_dict({"api_name": api, "fingerprint": "c4c4c4c4c4c4c4c4", "schemas": schemas})


def functions_of(registry: SchemaRegistry, layers: dict | None = None) -> list:
    """Entry/exit/profiling schema ids per function, in registry order."""
    entry, exit_, prof, order = {}, {}, {}, []
    for s in registry.schemas:
        if s.event_class == "host_entry":
            entry[s.function] = s.id
            order.append(s.function)
        elif s.event_class == "host_exit":
            exit_[s.function] = s.id
        elif s.event_class == "device_profiling":
            prof[s.function] = s.id
    out = []
    for fn in order:
        if fn in exit_:
            out.append((fn, entry[fn], exit_[fn], prof.get(fn, -1), (layers or {}).get(fn, 0),
                        1 if "MemoryCopy" in (fn or "") else 0))
    return out


@dataclass
class StreamSpec:
    hostname: str
    pid: int
    tid: int
    n_events: int
    seed: int
    kind: str = "calls"  # or "sampler"
    file: str | None = None


@dataclass
class Workload:
    name: str
    registry: SchemaRegistry
    streams: list
    params: dict = field(default_factory=dict)
    layers: dict | None = None
    kernel_names: list = field(default_factory=lambda: list(KERNEL_POOL_SMALL))
    sampler_period_ns: int = 50_000


DEFAULTS = dict(max_depth=4, gap_lo=1, gap_hi=600, ts0_hi=1000, push_p=0.5, err_p=0.02, prof_p=0.25,
                meta_p=0.0, orphan_p=0.0, mismatch_p=0.0, zipf_s=0.0, n_layers=1, close_at_end=1,
                dev_off_hi=10_000, dev_lo=1_000, dev_hi=100_000)


def _buffer(cap: int):
    """An uninitialised byte buffer for the C generator (zero-filling GBs of ctypes arrays cost more than
    generating the records) and its address."""
    import numpy as np

    a = np.empty(cap, dtype=np.uint8)
    return a, a.ctypes.data


def generate_stream(wl: Workload, spec: StreamSpec, flat=None, until_ns=None, counts=None) -> bytes:
    """One stream's file bytes; ``counts`` (a list) receives its record count."""
    L = _L()
    flat = flat or flatten_registry(wl.registry)
    max_id = max(s.id for s in flat.schemas)
    by_id = (type(flat.schemas[0]) * (max_id + 1))()
    for s in flat.schemas:
        by_id[s.id] = s
    if spec.kind == "sampler":
        sids = (C.c_uint32 * 9)(*[wl.registry.schema(f"{wl.registry.api_name}:telemetry_{k}").id
                                 for k, _ in TELEMETRY_COUNTERS])
        n_inst = (until_ns or 0) // wl.sampler_period_ns + 1
        cap = 16 + n_inst * 9 * 32
        arr, buf = _buffer(cap)
        ln, ev = C.c_uint64(), C.c_uint64()
        rc = L.synth_sampler(sids, 0, 0, wl.sampler_period_ns, until_ns or 0, spec.seed, buf, cap,
                             C.byref(ln), C.byref(ev))
        assert rc == 0
        if counts is not None:
            counts.append(ev.value)
        return arr[: ln.value].tobytes()
    p = dict(DEFAULTS)
    p.update(wl.params)
    fns = functions_of(wl.registry, wl.layers)
    farr = (SynthFn * len(fns))(*[SynthFn(e, x, pr, lay, mc) for _, e, x, pr, lay, mc in fns])
    names = [n.encode() for n in wl.kernel_names]
    name_arr = (C.c_char_p * max(len(names), 1))(*names)
    meta = [s.id for s in wl.registry.schemas if s.event_class == "meta"]
    P = SynthParams(seed=spec.seed, n_events=spec.n_events, meta_sid=meta[0] if meta else -1,
                    **{k: v for k, v in p.items()})
    cap = 16 + spec.n_events * (96 + max((len(n) for n in names), default=0)) + 4096
    arr, buf = _buffer(cap)
    ln, ev = C.c_uint64(), C.c_uint64()
    rc = L.synth_stream(C.byref(P), by_id, max_id + 1, flat.kinds, farr, len(fns), name_arr, len(names),
                        buf, cap, C.byref(ln), C.byref(ev))
    if rc != 0:
        raise RuntimeError(f"synth_stream failed ({rc})")
    if counts is not None:
        counts.append(ev.value)
    return arr[: ln.value].tobytes()


def last_timestamp(data: bytes) -> int:
    """ts of the final record (streams are ts-monotone), by a header walk in C."""
    return _L().synth_last_ts(data, len(data))


def generate(wl: Workload, threads: int | None = None) -> list:
    """All streams of a workload as RawStream objects in (hostname, pid, tid) order."""
    flat = flatten_registry(wl.registry)
    calls = [s for s in wl.streams if s.kind == "calls"]
    def one(s, until=None):
        c = []
        d = generate_stream(wl, s, flat, until_ns=until, counts=c)
        return d, c[0]

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 4) as ex:
        datas = list(ex.map(one, calls))
    out = {}
    for s, dn in zip(calls, datas):
        out[(s.hostname, s.pid, s.tid)] = (s, dn)
    samplers = [s for s in wl.streams if s.kind == "sampler"]
    if samplers:
        until = max(last_timestamp(d) for d, _ in datas) if datas else 0
        for s in samplers:
            out[(s.hostname, s.pid, s.tid)] = (s, one(s, until))
    raws = []
    for key in sorted(out):
        s, (d, n) = out[key]
        name = s.file or f"stream_{s.pid}_{s.tid}.bin"
        raws.append(RawStream(s.hostname, s.pid, s.tid, name, d, StreamInfo(s.hostname, s.pid, s.tid, n, 0)))
    return raws


def count_records(data: bytes) -> int:
    import struct

    off, n = 16, 0
    while off + 16 <= len(data):
        plen = struct.unpack_from("<I", data, off + 12)[0]
        off += 16 + plen
        n += 1
    return n


def write(wl: Workload, raws: list, directory) -> Path:
    return write_trace(
        directory, wl.registry,
        [{"hostname": r.hostname, "pid": r.pid, "tid": r.tid, "data": r.data, "event_count": r.info.event_count,
          "dropped_count": r.info.dropped_count, "file": r.name} for r in raws],
    )


# ---------------------------------------------------------------------------
# SURVEY.md §8(d) configurations (scale= shrinks event counts for tests)


def config(name: str, scale: float = 1.0) -> Workload:
    ze = ze_registry()
    if name == "c1":
        n = max(1, int(1_000_000 * scale))
        return Workload("c1", ze, [StreamSpec("synth0", PID_BASE, PID_BASE, n, 42)], {"prof_p": 0.12},
                        kernel_names=list(KERNEL_POOL_ASCII))
    if name == "c2":
        per = max(1, int(390_625 * scale))
        streams = []
        for p in range(4):
            pid = PID_BASE + PID_STRIDE * p
            for t in range(64):
                streams.append(StreamSpec("synth0", pid, pid + t, per, 43_000 + p * 64 + t))
        return Workload("c2", ze, streams, {"prof_p": 0.12}, kernel_names=list(KERNEL_POOL_ASCII))
    if name == "c3":
        per = max(1, int(976_562 * scale))
        streams = []
        for h in range(8):
            for p in range(4):
                pid = PID_BASE + PID_STRIDE * p
                for t in range(32):
                    streams.append(StreamSpec(f"node{h:02d}", pid, pid + t, per, 44_000 + (h * 4 + p) * 32 + t,
                                              file=f"stream_node{h:02d}_{pid}_{pid + t}.bin"))
        return Workload("c3", ze, streams, {"prof_p": 0.12}, kernel_names=list(KERNEL_POOL_ASCII))
    if name == "c4":
        reg = layered_registry()
        layers = {s.function: (0 if s.function.startswith("sycl") else 1)
                  for s in reg.schemas if s.event_class == "host_entry"}
        per = max(1, int(390_625 * scale))
        streams = []
        for p in range(4):
            pid = PID_BASE + PID_STRIDE * p
            for t in range(64):
                streams.append(StreamSpec("synth0", pid, pid + t, per, 45_000 + p * 64 + t))
        return Workload("c4", reg, streams, {"max_depth": 64, "push_p": 0.55, "zipf_s": 1.1, "n_layers": 2},
                        layers=layers)
    if name == "c5":
        per = max(1, int(390_625 * scale))
        streams = []
        for p in range(4):
            pid = PID_BASE + PID_STRIDE * p
            for t in range(64):
                streams.append(StreamSpec("synth0", pid, pid + t, per, 46_000 + p * 64 + t))
        streams.append(StreamSpec("synth0", PID_BASE, PID_BASE + SAMPLER_TID_OFFSET, 0, 46_999, kind="sampler"))
        return Workload("c5", ze, streams, {"prof_p": 0.9}, kernel_names=kernel_pool(500))
    raise KeyError(name)
