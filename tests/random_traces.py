"""TEST INFRASTRUCTURE: seeded random traces of the bundled ze registry, in the reference format.

Each seed gives a few streams (identities that collide across hosts, duplicate pids), with nested
calls, orphan and typed-mismatch exits, unclosed calls, device-profiling records (kernel names with
escapes and non-ASCII UTF-8, negative spans), telemetry samples (valid values, occasionally an
out-of-range one), annotations, equal timestamps, timestamps near 2^60, blobs, and -- for a share of
the seeds -- one corruption (unknown schema id, truncated record, bad UTF-8, a timestamp going
backwards, trailing bytes).  Used to compare the engine with the oracle and the oracle with the
reference beyond the fixed fixtures."""

from __future__ import annotations

import random
import struct

from paper_2504_03683_b200 import synth
from paper_2504_03683_b200.tracefile import RawStream, StreamInfo, encode_record, stream_bytes

NAMES = ["k_gemm", "kélté", "k\"quote\"", "k\\slash", "k\ttab", "memcpy(H2D)", "漢字", "k" * 40,
         "a", "k\U0001f600", "kernel_" + "x" * 17]


def _payload(schema, rnd, big):
    out = {}
    for f in schema.fields:
        if f.kind == "string":
            out[f.name] = rnd.choice(NAMES) if f.name in ("name", "label") else rnd.choice(["kernel", "memcpy", ""])
        elif f.kind == "blob":
            out[f.name] = bytes(rnd.getrandbits(8) for _ in range(rnd.choice([0, 0, 8, 16, 3])))
        elif f.kind == "f64":  # telemetry values: utilisation counters must stay in [0, 1] (sampler.py:44-48)
            out[f.name] = rnd.choice([0.0, 0.5, 1.0, 0.25, 1e-9, 0.1 + 0.2])
        elif f.kind == "i64":
            out[f.name] = rnd.choice([0, 0, 0, 3, -7, (1 << 62), -(1 << 63)])
        else:
            out[f.name] = rnd.getrandbits(64 if big else 40)
    return out


def random_trace(seed: int, corrupt: bool | None = None):
    """(registry, [RawStream]) in (hostname, pid, tid) order."""
    rnd = random.Random(seed)
    ze = synth.ze_registry()
    by_cls = {}
    for s in ze.schemas:
        by_cls.setdefault(s.event_class, []).append(s)
    entries = {s.function: s for s in by_cls["host_entry"]}
    exits = {s.function: s for s in by_cls["host_exit"]}
    fns = sorted(entries)
    big = rnd.random() < 0.3
    n_streams = rnd.randint(1, 6)
    idents = set()
    while len(idents) < n_streams:
        idents.add((rnd.choice(["h0", "h1", "né", "zz"]), rnd.choice([1, 2, 4202000]), rnd.randint(1, 6)))
    raws = []
    for host, pid, tid in sorted(idents):
        ts = rnd.choice([0, 1000, (1 << 60) - 5000]) if big else rnd.randint(0, 1000)
        stack, recs = [], []
        for _ in range(rnd.randint(0, 120)):
            ts += rnd.choice([0, 0, 1, 7, 500]) if not big else rnd.choice([0, 1 << 33, 12345])
            u = rnd.random()
            if u < 0.35 and len(stack) < 12:
                f = rnd.choice(fns)
                stack.append(f)
                sc = entries[f]
            elif u < 0.7 and stack:
                f = stack.pop() if rnd.random() < 0.9 else rnd.choice(fns)  # occasional typed mismatch
                sc = exits[f]
            elif u < 0.75:
                sc = exits[rnd.choice(fns)]  # orphan exit
            elif u < 0.87:
                sc = rnd.choice(by_cls["device_profiling"])
            elif u < 0.95:
                sc = rnd.choice(by_cls["telemetry_sample"])
            else:
                sc = by_cls["meta"][0]
            p = _payload(sc, rnd, big)
            if sc.event_class == "device_profiling" and rnd.random() < 0.2:
                p["device_end_ns"], p["device_start_ns"] = p["device_start_ns"], p["device_end_ns"]  # negative span
            if sc.event_class == "telemetry_sample" and rnd.random() < 0.004:
                p["value"] = rnd.choice([-1.0, 1.5])  # a range check error (sampler.py:44-48)
            recs.append(encode_record(sc, ts, p))
        data = stream_bytes(recs) if recs else b""
        raws.append(RawStream(host, pid, tid, f"stream_{host}_{pid}_{tid}.bin", data,
                              StreamInfo(host, pid, tid, len(recs), rnd.choice([0, 0, 0, 5]))))
    if corrupt is None:
        corrupt = rnd.random() < 0.3
    if corrupt:
        cands = [i for i, r in enumerate(raws) if len(r.data) > 40]
        if cands:
            i = rnd.choice(cands)
            r = raws[i]
            d = bytearray(r.data)
            offs, off = [], 16
            while off + 16 <= len(d):
                offs.append(off)
                off += 16 + struct.unpack_from("<I", d, off + 12)[0]
            at = rnd.choice(offs)
            kind = rnd.randrange(6)
            if kind == 5:  # bad UTF-8 in a device record's command_kind string, else fall back to an unknown id
                devs = [o for o in offs if struct.unpack_from("<I", d, o)[0] in (26, 27) and
                        struct.unpack_from("<I", d, o + 32)[0] > 0]
                if devs:
                    d[rnd.choice(devs) + 36] = 0xFF
                else:
                    kind = 0
            if kind == 0:
                d[at:at + 4] = struct.pack("<I", 999)  # unknown schema id
            elif kind == 1:
                d = d[: at + rnd.randint(1, 20)]  # truncated header / payload
            elif kind == 2:
                ts = struct.unpack_from("<Q", d, at + 4)[0]
                d[at + 4:at + 12] = struct.pack("<Q", max(ts, 1) - 1 if at > 16 else ts)  # may go backwards
                if at > 16:
                    d[at + 4:at + 12] = struct.pack("<Q", 0)
            elif kind == 3:
                d[at + 12:at + 16] = struct.pack("<I", struct.unpack_from("<I", d, at + 12)[0] + 1)  # length off
            else:
                d += b"\xff\xfe"  # trailing garbage after the last record
            raws[i] = RawStream(r.hostname, r.pid, r.tid, r.name, bytes(d), r.info)
    return ze, raws
