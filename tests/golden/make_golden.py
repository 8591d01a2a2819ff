"""Generate the golden fixtures that pin the oracle and the GPU engine to the reference.

Run in the build container (the reference is importable there, not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For every fixture it writes a trace directory under tests/golden/traces/<name>/
and the reference's own outputs under tests/golden/expected/:
  <name>.json           tally JSON + rendered text + IntervalStats + orphans, or
                        the raised exception (type, str, attributes) and the
                        orphans delivered to on_diagnostics before it; for a
                        tally-only pipeline and for tally+timeline
  <name>.timeline.json  the TimelineSink file bytes (when the run succeeds)
Traces come from the reference's own writer/workloads (w1-w3), from this
repo's C generator (decoded by the reference reader here, which pins the
generator's encoding), and from hand-built byte mutations for every error
path of the decoder and muxer.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import random
import shutil
import struct
import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

from hapitrace import harness as ref_harness  # noqa: E402
from hapitrace.pipeline import Sink, run_pipeline  # noqa: E402
from hapitrace.sinks import TallySink, TimelineSink, render_tally  # noqa: E402
from hapitrace.tracefile import open_trace_reader  # noqa: E402

from paper_2504_03683_b200 import synth  # noqa: E402
from paper_2504_03683_b200.registry import SchemaRegistry  # noqa: E402
from paper_2504_03683_b200.tracefile import encode_record, stream_bytes, write_trace  # noqa: E402

TRACES = HERE / "traces"
EXPECTED = HERE / "expected"


class Diag(Sink):
    name = "diag"
    consumes = "intervals"

    def __init__(self):
        self.orphans = None

    def on_diagnostics(self, orphans):
        self.orphans = [list(o) for o in orphans]

    def on_finish(self):
        return self.orphans


def _exc(e):
    attrs = {k: getattr(e, k) for k in ("stream", "offset", "index") if hasattr(e, k)}
    return {"type": type(e).__name__, "str": str(e), "args": [repr(a) for a in e.args], "attrs": attrs}


def run_reference(d: Path, name: str):
    out = {"name": name}
    for mode in ("tally", "tally+timeline"):
        diag = Diag()
        sinks = [TallySink()]
        tl = EXPECTED / f"{name}.timeline.json"
        if mode == "tally+timeline":
            sinks.append(TimelineSink(out_path=tl))
        sinks.append(diag)
        res = {}
        try:
            r = run_pipeline(open_trace_reader(d), sinks)
        except Exception as e:  # noqa: BLE001 -- recording the reference's behaviour
            res["error"] = _exc(e)
            res["orphans"] = diag.orphans
            if tl.exists() and mode == "tally+timeline":
                tl.unlink()
        else:
            if mode == "tally+timeline":
                blob = tl.read_bytes()
                res["timeline_sha256"] = hashlib.sha256(blob).hexdigest()
                res["timeline_len"] = len(blob)
                if len(blob) > 64_000:
                    tl.unlink()
            res["tally_json"] = r["tally"].to_json()
            res["render"] = render_tally(r["tally"])
            res["stats"] = dataclasses.asdict(r.stats)
            res["orphans"] = r["diag"]
        out[mode] = res
    (EXPECTED / f"{name}.json").write_text(json.dumps(out, indent=1))
    return out


# ---------------------------------------------------------------------------
# fixture builders


def fx_workloads():
    ze = ref_harness.bundled_workload
    yield "w1_default", lambda d: ref_harness.trace_workload(ze("w1"), d, hostname="goldenhost")
    yield "w1_full_sampled", lambda d: ref_harness.trace_workload(
        ze("w1"), d, mode="full", sample=True, sample_period_ns=50_000, hostname="goldenhost")
    yield "w1_injected", lambda d: ref_harness.trace_workload(
        ze("w1"), d, mode="full", inject=("leak_event", "no_reset_cmdlist", "uninit_pnext"), hostname="goldenhost")
    yield "w2_full_sampled", lambda d: ref_harness.trace_workload(
        ze("w2"), d, mode="full", sample=True, sample_period_ns=20_000, hostname="goldenhost")
    yield "w3_minimal", lambda d: ref_harness.trace_workload(ze("w3"), d, mode="minimal", hostname="goldenhost")
    yield "w3_full_drops", lambda d: ref_harness.trace_workload(
        ze("w3"), d, mode="full", buffer_capacity=512, hostname="goldenhost")


def _wl(name, reg, streams, **params):
    return synth.Workload(name, reg, streams, params)


def fx_synthetic():
    ze = synth.ze_registry()
    P = synth.PID_BASE

    def gen(wl, kernel_names=None):
        if kernel_names:
            wl.kernel_names = kernel_names

        def make(d):
            synth.write(wl, synth.generate(wl), d)
        return make

    yield "syn_c1", gen(synth.config("c1", 0.008))
    yield "syn_c2", gen(synth.config("c2", 0.0003))
    yield "syn_c4", gen(_wl("c4s", synth.layered_registry(150, 150),
                            [synth.StreamSpec("synth0", P, P + t, 2500, 450 + t) for t in range(6)],
                            max_depth=64, push_p=0.6, zipf_s=1.1, n_layers=2), None)
    c4 = synth.config("c4", 0.0)
    yield "syn_c4_layers", gen(synth.Workload(
        "c4l", c4.registry, [synth.StreamSpec("synth0", P, P + t, 3000, 451 + t) for t in range(4)],
        {"max_depth": 64, "push_p": 0.55, "zipf_s": 1.1, "n_layers": 2}, layers=c4.layers))
    c5 = synth.Workload("c5s", ze, [synth.StreamSpec("synth0", P + 100 * p, P + 100 * p + t, 1500, 460 + 8 * p + t)
                                    for p in range(2) for t in range(4)]
                        + [synth.StreamSpec("synth0", P, P + 99, 0, 469, kind="sampler")],
                        {"prof_p": 0.9}, kernel_names=synth.kernel_pool(40))
    c5.sampler_period_ns = 20_000
    yield "syn_c5", gen(c5)
    yield "syn_multihost", gen(_wl("mh", ze, [
        synth.StreamSpec(h, P + 100 * p, P + 100 * p + t, 700, 500 + 20 * i + 4 * p + t,
                         file=f"stream_{h}_{P + 100 * p}_{P + 100 * p + t}.bin")
        for i, h in enumerate(("node02", "node00", "node01")) for p in range(2) for t in range(3)], prof_p=0.3))
    yield "syn_orphans", gen(_wl("orph", ze, [synth.StreamSpec("synth0", P, P + t, 2000, 600 + t) for t in range(5)],
                                 orphan_p=0.02, mismatch_p=0.05, meta_p=0.05, close_at_end=0, max_depth=6))
    yield "syn_ties", gen(_wl("ties", ze, [synth.StreamSpec("synth0", P + 100 * (t % 2), P + t, 1500, 700 + t)
                                           for t in range(6)], gap_lo=0, gap_hi=2, close_at_end=0))
    yield "syn_deep", gen(_wl("deep", ze, [synth.StreamSpec("synth0", P, P, 6000, 800)],
                              max_depth=300, push_p=0.8, close_at_end=0, mismatch_p=0.01))
    # wide values: host gaps in [2^32, 2^33] ns, timestamps from ~2^60 (CPython float repr
    # beyond 2^53), device spans of +-2^40 ns (negative: end < start)
    yield "syn_wide", gen(_wl("wide", ze, [synth.StreamSpec("synth0", P, P + t, 1200, 900 + t) for t in range(4)],
                              gap_lo=1 << 32, gap_hi=1 << 33, ts0_hi=1 << 60, prof_p=0.5, close_at_end=0,
                              dev_off_hi=1 << 41, dev_lo=-(1 << 40), dev_hi=1 << 40))


def fx_dup_identity():
    """Two stream files with one (hostname, pid, tid): they share a LIFO stack
    (pipeline.py:156-161) and tie-break by seq then input index (pipeline.py:88-91)."""
    ze = synth.ze_registry()
    by = {s.name: s.id for s in ze.schemas}

    def rec(name, ts, **payload):
        sc = ze.by_id[by[f"ze:{name}"]]
        full = {}
        for f in sc.fields:
            full[f.name] = payload.get(f.name, "" if f.kind == "string" else b"" if f.kind == "blob" else 0)
        return encode_record(sc, ts, full)

    def make(d):
        a = [rec("zeMockInit_entry", 10), rec("zeMockMemAlloc_entry", 30), rec("zeMockMemAlloc_exit", 40),
             rec("zeMockMemFree_entry", 50), rec("zeMockInit_exit", 70, result=3), rec("zeMockMemFree_entry", 90)]
        b = [rec("zeMockMemFree_exit", 50), rec("zeMockMemFree_exit", 60), rec("zeMockEventCreate_entry", 70),
             rec("zeMockEventCreate_exit", 75), rec("zeMockInit_entry", 95)]
        c = [rec("zeMockInit_entry", 5), rec("zeMockInit_exit", 50)]
        entries = [{"hostname": "dup", "pid": 7, "tid": 7, "data": stream_bytes(a), "event_count": len(a),
                    "dropped_count": 0, "file": "stream_7_7_a.bin"},
                   {"hostname": "dup", "pid": 7, "tid": 7, "data": stream_bytes(b), "event_count": len(b),
                    "dropped_count": 0, "file": "stream_7_7_b.bin"},
                   {"hostname": "dup", "pid": 7, "tid": 8, "data": stream_bytes(c), "event_count": len(c),
                    "dropped_count": 0, "file": "stream_7_8.bin"}]
        write_trace(d, ze, entries)
    yield "dup_identity", make


# --- hand-built registries and byte-level fixtures --------------------------


def custom_registry():
    """Sparse ids, f64 results, duplicate function names, i64 device
    timestamps, a device schema with no tile/engine/command_kind, meta class."""
    S = []

    def add(sid, name, cls, fields, fn=None):
        S.append({"id": sid, "name": name, "class": cls, "function": fn, "mode_mask": ["default", "full"],
                  "fields": [{"name": n, "kind": k, "origin": "stack_arg"} for n, k in fields]})

    add(7, "cx:alpha_entry", "host_entry", [("x", "u64")], "alpha")
    add(3000, "cx:alpha_exit", "host_exit", [("result", "f64")], "alpha")
    add(100, "cx:beta_entry", "host_entry", [("s", "string"), ("b", "blob")], "beta")
    add(101, "cx:beta_exit", "host_exit", [("result", "u64"), ("tag", "string")], "beta")
    add(102, "cx:beta2_entry", "host_entry", [], "beta")  # same function name, different schema
    add(103, "cx:beta2_exit", "host_exit", [], "beta")    # no result field -> result 0
    add(5, "cx:gamma_entry", "host_entry", [], "gamma")
    add(6, "cx:gamma_exit", "host_exit", [("result", "i64")], "gamma")
    add(50, "cx:dev_profiling", "device_profiling",
        [("device_start_ns", "i64"), ("device_end_ns", "i64"), ("name", "string")], "beta")
    add(51, "cx:dev2_profiling", "device_profiling",
        [("device_start_ns", "u64"), ("device_end_ns", "u64"), ("command_kind", "string"), ("name", "string"),
         ("tile", "u64"), ("engine", "u64")], "alpha")
    add(60, "cx:note", "meta", [("label", "string")])
    add(61, "cx:weird", "not_a_class", [("v", "u64")])
    add(70, "cx:telemetry_power_domain_1", "telemetry_sample", [("device", "u64"), ("value", "f64")])
    add(71, "cx:telemetry_copy_tile_0", "telemetry_sample", [("device", "u64"), ("value", "i64")])
    return SchemaRegistry.from_dict({"api_name": "cx", "fingerprint": "0123456789abcdef", "schemas": S})


def _enc(reg, sid, ts, payload):
    return encode_record(reg.by_id[sid], ts, payload)


def fx_custom():
    reg = custom_registry()
    rng = random.Random(2026)

    def stream(seed, n_ops, with_dev=True):
        rng = random.Random(seed)
        recs, stack, ts = [], [], rng.randint(0, 50)
        pairs = [(7, 3000), (100, 101), (102, 103), (5, 6)]
        for _ in range(n_ops):
            ts += rng.randint(0, 40)
            u = rng.random()
            if u < 0.05:
                recs.append(_enc(reg, 60, ts, {"label": rng.choice(["phase", "ω-step", ""])}))
            elif u < 0.08:
                recs.append(_enc(reg, 61, ts, {"v": 5}))
            elif u < 0.14 and with_dev:
                a = rng.randint(0, 10**6)
                b = a + rng.randint(-5000, 5000)  # negative device durations are legal
                recs.append(_enc(reg, 50, ts, {"device_start_ns": a, "device_end_ns": b,
                                               "name": rng.choice(["kérnel", "k2", "\U0001f680go"])}))
            elif u < 0.18 and with_dev:
                a = rng.randint(0, 10**9)
                recs.append(_enc(reg, 51, ts, {"device_start_ns": a, "device_end_ns": a + rng.randint(0, 10**6),
                                               "command_kind": "kernel", "name": "k2", "tile": rng.randint(0, 2),
                                               "engine": rng.randint(0, 1)}))
            elif u < 0.22:
                recs.append(_enc(reg, 70, ts, {"device": rng.randint(0, 2), "value": rng.uniform(0, 300)}))
            elif u < 0.25:
                recs.append(_enc(reg, 71, ts, {"device": 0, "value": rng.randint(0, 1)}))
            elif stack and (rng.random() < 0.5 or len(stack) > 5):
                en, ex = stack.pop()
                if rng.random() < 0.06:  # wrong exit: typed mismatch
                    ex = rng.choice(pairs)[1]
                    stack.append((en, None))
                payload = {}
                for f in reg.by_id[ex].fields:
                    payload[f.name] = {"f64": rng.choice([0.0, 0.5, -0.99, 2.5, -3.7, 1e18]), "u64": rng.choice([0, 0, 7]),
                                       "i64": rng.choice([0, -2]), "string": "t"}[f.kind]
                recs.append(_enc(reg, ex, ts, payload))
                if stack and stack[-1][1] is None:
                    stack.pop()
            else:
                en, ex = rng.choice(pairs)
                stack.append((en, ex))
                payload = {f.name: {"u64": 1, "string": "sü", "blob": b"\x00\x01"}[f.kind]
                           for f in reg.by_id[en].fields}
                recs.append(_enc(reg, en, ts, payload))
        return stream_bytes(recs)

    def make(d):
        streams = []
        for i, (h, p, t) in enumerate([("hA", 10, 11), ("hA", 10, 12), ("hB", 3, 3), ("hA", 2, 99)]):
            data = stream(100 + i, 900)
            streams.append({"hostname": h, "pid": p, "tid": t, "data": data,
                            "event_count": synth.count_records(data), "dropped_count": i % 2 * 3,
                            "file": f"s_{h}_{p}_{t}.bin"})
        streams.append({"hostname": "hC", "pid": 5, "tid": 5, "data": b"", "event_count": 0, "dropped_count": 17})
        write_trace(d, reg, streams)

    yield "custom_registry", make

    def empty(d):
        write_trace(d, reg, [])

    yield "empty_trace", empty


def _base_streams(n=3, per=400, seed=900, **kw):
    ze = synth.ze_registry()
    P = synth.PID_BASE
    wl = _wl("base", ze, [synth.StreamSpec("synth0", P, P + t, per, seed + t) for t in range(n)], **kw)
    return ze, synth.generate(wl)


def _offsets(data):
    offs, off = [], 16
    while off + 16 <= len(data):
        offs.append(off)
        off += 16 + struct.unpack_from("<I", data, off + 12)[0]
    return offs


def _write_raws(d, reg, raws, mutate):
    streams = []
    for i, r in enumerate(raws):
        data = mutate(i, bytearray(r.data)) if mutate else bytes(r.data)
        streams.append({"hostname": r.hostname, "pid": r.pid, "tid": r.tid, "data": bytes(data),
                        "event_count": r.info.event_count, "dropped_count": 0, "file": r.name})
    write_trace(d, reg, streams)


def fx_errors():
    ze, raws = _base_streams()

    def mut(which, fn):
        def make(d):
            _write_raws(d, ze, raws, lambda i, b: fn(b) if i == which else b)
        return make

    def cut_tail(b):
        return b[:-5]

    def unknown_sid(b):
        o = _offsets(b)[150]
        struct.pack_into("<I", b, o, 777)
        return b

    def bad_magic(b):
        b[0] ^= 0xFF
        return b

    def bad_version(b):
        struct.pack_into("<I", b, 4, 2)
        return b

    def short_header(b):
        return b[:10]

    def first_fixed(b, start=0):
        for o in _offsets(b)[start:]:
            sid = struct.unpack_from("<I", b, o)[0]
            if all(f.kind not in ("string", "blob") for f in ze.by_id[sid].fields):
                return o
        raise AssertionError

    def len_mismatch(b):
        o = first_fixed(b, 200)
        plen = struct.unpack_from("<I", b, o + 12)[0]
        struct.pack_into("<I", b, o + 12, plen + 8)
        return b[:o + 16 + plen] + b"\x00" * 8 + b[o + 16 + plen:]

    def var_record(b, start, sid_filter=None):
        for o in _offsets(b)[start:]:
            sid = struct.unpack_from("<I", b, o)[0]
            if any(f.kind in ("string", "blob") for f in ze.by_id[sid].fields):
                if sid_filter is None or sid in sid_filter:
                    return o, sid
        raise AssertionError

    def trailing(b):
        o, _ = var_record(b, 120)
        plen = struct.unpack_from("<I", b, o + 12)[0]
        struct.pack_into("<I", b, o + 12, plen + 4)
        return b[:o + 16 + plen] + b"\xab\xcd\xef\x01" + b[o + 16 + plen:]

    def trunc_var(b):
        o, sid = var_record(b, 90)
        # first var field's length prefix -> too long for the payload
        p = 0
        for f in ze.by_id[sid].fields:
            if f.kind in ("string", "blob"):
                break
            p += 8
        struct.pack_into("<I", b, o + 16 + p, 10_000)
        return b

    launch = ze.schema("ze:zeMockCommandListAppendLaunchKernel_entry").id

    def struct_err(b):
        o = _offsets(b)[60]
        # replace record 60 with a launch-kernel entry whose payload stops inside the u64 groupCount
        body = struct.pack("<Q", 0x1234) + struct.pack("<I", 3) + b"abc" + b"\x01\x02\x03\x04"
        ts = struct.unpack_from("<Q", b, o + 4)[0]
        nxt = o + 16 + struct.unpack_from("<I", b, o + 12)[0]
        return b[:o] + struct.pack("<IQI", launch, ts, len(body)) + body + b[nxt:]

    def utf8_err(bad):
        def f(b):
            o = _offsets(b)[75]
            ts = struct.unpack_from("<Q", b, o + 4)[0]
            nxt = o + 16 + struct.unpack_from("<I", b, o + 12)[0]
            body = struct.pack("<Q", 1) + struct.pack("<I", len(bad)) + bad + struct.pack("<QQ", 8, 0)
            return b[:o] + struct.pack("<IQI", launch, ts, len(body)) + body + b[nxt:]
        return f

    def order_err(b, at=50):
        o = _offsets(b)[at]
        prev = _offsets(b)[at - 1]
        pts = struct.unpack_from("<Q", b, prev + 4)[0]
        struct.pack_into("<Q", b, o + 4, max(pts - 1, 0) if pts else 0)
        if pts == 0:
            struct.pack_into("<Q", b, prev + 4, 5)
        return b

    yield "err_trunc_tail", mut(1, cut_tail)
    yield "err_unknown_schema", mut(2, unknown_sid)
    yield "err_bad_magic", mut(1, bad_magic)
    yield "err_bad_version", mut(0, bad_version)
    yield "err_short_header", mut(2, short_header)
    yield "err_len_mismatch", mut(0, len_mismatch)
    yield "err_trailing", mut(2, trailing)
    yield "err_trunc_var", mut(1, trunc_var)
    yield "err_struct", mut(0, struct_err)
    yield "err_utf8_start", mut(1, utf8_err(b"ab\xffcd"))
    yield "err_utf8_cont", mut(1, utf8_err(b"x\xe2\x82"))
    yield "err_utf8_surrogate", mut(2, utf8_err(b"\xed\xa0\x80z"))
    yield "err_order", mut(1, order_err)
    yield "err_order_first", mut(2, lambda b: order_err(b, 1))

    def two_errors(d):
        def m(i, b):
            if i == 0:
                return order_err(b, 300)
            if i == 2:
                return unknown_sid(b)
            return b
        _write_raws(d, ze, raws, m)

    yield "err_two_streams", two_errors

    # telemetry value out of range, on a sampler stream next to call streams
    def telemetry_err(d):
        c5 = synth.Workload("t", ze, [synth.StreamSpec("synth0", synth.PID_BASE, synth.PID_BASE, 500, 31),
                                      synth.StreamSpec("synth0", synth.PID_BASE, synth.PID_BASE + 99, 0, 32,
                                                       kind="sampler")], {"prof_p": 0.5})
        c5.sampler_period_ns = 5_000
        rs = synth.generate(c5)

        def m(i, b):
            if i != 1:
                return b
            o = _offsets(b)[9 * 7 + 5]  # compute_tile_0 sample of the 8th instant
            struct.pack_into("<d", b, o + 16 + 8, 1.5)
            return b
        _write_raws(d, ze, rs, m)

    yield "err_telemetry", telemetry_err

    # custom-registry error paths
    def custom_err(kind):
        def make(d):
            S = [
                {"id": 0, "name": "e:f_entry", "class": "host_entry", "function": "f", "mode_mask": ["full"],
                 "fields": []},
                {"id": 1, "name": "e:f_exit", "class": "host_exit", "function": "f", "mode_mask": ["full"],
                 "fields": [{"name": "result", "kind": "f64", "origin": "result"}]},
                {"id": 2, "name": "e:telemetry_bogus_1", "class": "telemetry_sample", "function": None,
                 "mode_mask": ["full"], "fields": [{"name": "device", "kind": "u64", "origin": "t"},
                                                   {"name": "value", "kind": "f64", "origin": "t"}]},
                {"id": 3, "name": "e:telemetry_compute_tile_3", "class": "telemetry_sample", "function": None,
                 "mode_mask": ["full"], "fields": [{"name": "device", "kind": "u64", "origin": "t"},
                                                   {"name": "value", "kind": "f64", "origin": "t"}]},
                {"id": 4, "name": "e:k_profiling", "class": "device_profiling", "function": "f",
                 "mode_mask": ["full"], "fields": [{"name": "device_start_ns", "kind": "u64", "origin": "p"},
                                                   {"name": "device_end_ns", "kind": "u64", "origin": "p"}]},
            ]
            reg = SchemaRegistry.from_dict({"api_name": "e", "fingerprint": "eeeeeeeeeeeeeeee", "schemas": S})
            recs = []
            ts = 0
            for i in range(40):
                ts += 10
                recs.append(_enc(reg, 0, ts, {}))
                ts += 10
                val = 0.5
                if kind == "nan" and i == 25:
                    val = float("nan")
                if kind == "inf" and i == 25:
                    val = float("-inf")
                recs.append(_enc(reg, 1, ts, {"result": val}))
                if i == 30:
                    if kind == "bogus":
                        recs.append(_enc(reg, 2, ts + 1, {"device": 0, "value": 1.0}))
                    if kind == "track":
                        recs.append(_enc(reg, 3, ts + 1, {"device": 0, "value": 0.25}))
                    if kind == "keyerr":
                        recs.append(_enc(reg, 4, ts + 1, {"device_start_ns": 1, "device_end_ns": 2}))
            data = stream_bytes(recs)
            write_trace(d, reg, [{"hostname": "h", "pid": 1, "tid": 1, "data": data,
                                  "event_count": len(recs), "dropped_count": 0}])
        return make

    for k in ("nan", "inf", "bogus", "track", "keyerr"):
        yield f"err_custom_{k}", custom_err(k)


def tally_fixture():
    """The reference's paper-style tally render (its test_sinks.py:382-408 fixture)."""
    from hapitrace.sinks import TallyReport, TallyRow

    rows = [("hipDeviceSynchronize", 4_730_000_000, 1), ("zeEventHostSynchronize", 4_680_000_000, 9),
            ("hipMemcpy", 1_770_000_000, 3), ("__hipUnregisterFatBinary", 500_910_000, 1),
            ("zeCommandListAppendMemoryCopy", 394_500_000, 5), ("hipLaunchKernel", 262_700_000, 2),
            ("zeModuleCreate", 256_090_000, 1), ("other", 55_800_000, 4)]
    rep = TallyReport(fingerprint=None, backends=("BACKEND_HIP", "BACKEND_ZE"),
                      hostnames=frozenset({"aurora-node"}), processes=frozenset({("aurora-node", 1)}),
                      threads=frozenset({("aurora-node", 1, 1)}))
    for n, t, c in rows:
        rep.rows[("host", n)] = TallyRow(n, "host", time_ns=t, count=c, min_ns=t // c, max_ns=t // c)
    (EXPECTED / "tally_fixture.json").write_text(json.dumps(
        {"rows": rows, "render": render_tally(rep),
         "source": "reference sinks.render_tally on test_sinks.py:382-408 fixture"}, indent=1))


def main(only=None):
    EXPECTED.mkdir(parents=True, exist_ok=True)
    TRACES.mkdir(parents=True, exist_ok=True)
    index = []
    for group in (fx_workloads, fx_synthetic, fx_dup_identity, fx_custom, fx_errors):
        for name, make in group():
            if only and name not in only:
                continue
            d = TRACES / name
            if d.exists():
                shutil.rmtree(d)
            make(d)
            res = run_reference(d, name)
            index.append(name)
            status = res["tally"].get("error", {}).get("type", "ok")
            print(f"{name:24s} {status}")
    if not only:
        (EXPECTED / "index.json").write_text(json.dumps(sorted(index), indent=1))
        tally_fixture()


if __name__ == "__main__":
    main(sys.argv[1:] or None)
