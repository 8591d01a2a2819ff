"""Multi-GPU runs: one process per GPU, streams sharded per rank, collectives for the real exchanges.

The interval state is per (hostname, pid, tid) stream (pipeline.py:158-161) and
the tally is a commutative monoid (aggregator.py:1-9), so ranks own disjoint
stream sets (`partition_streams`: LPT by bytes) and exchange:

  1. MAX of [local last timestamp, failure status] -- truncated spans end at the
     GLOBAL last ts (pipeline.py:152, :235), and a rank whose engine failed
     stops every rank instead of leaving them in the next collective;
  2. the device-name lists (all-gather of bytes) -> one global name order;
  3. the tally merge (aggregator.py:35-76): every rank's engine writes its
     device-resident rows, IntervalStats and span counts into one int64 buffer
     in a rank-independent layout (hg_merge_export, csrc/merge.cu); a SUM and a
     MAX all-reduce over that buffer ARE merge_tallies; hg_merge_import installs
     the result.  No row crosses Python on the way;
  4. only when some rank hit one: the trace errors (the first in the
     reference's pull order wins, results.error_key over GLOBAL stream
     indices) and the orphan exits (gathered, then put in mux order).

`Comm` wraps torch.distributed: tensors live on the GPU for NCCL and on the
CPU for gloo, so the same code runs in the world-size-2 CPU tests.
"""

from __future__ import annotations

import os
from types import SimpleNamespace

from .abi import HG_TRACE_ERROR, HG_WANT_TALLY
from .errors import EngineError
from .results import build_report, error_key, first_error, make_exception, orphan_list

STATUS_OK, STATUS_TRACE, STATUS_ENGINE, STATUS_INPUT = 0, 1, 2, 3
_BIAS = 1 << 63


def partition_streams(sizes, world_size: int, keys=None) -> list:
    """Assign whole streams to ranks by LPT on byte size: largest first onto the
    least-loaded rank (ties: lower rank).  Streams with equal ``keys`` entries (one (hostname, pid,
    tid) identity, which shares one LIFO stack, pipeline.py:156-161) go to one rank together.
    Returns, per rank, its global stream indices in ascending (= mux) order."""
    n = len(sizes)
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    groups = {}
    for i in range(n):
        groups.setdefault(keys[i] if keys is not None else i, []).append(i)
    units = sorted(groups.values(), key=lambda g: (-sum(sizes[i] for i in g), g[0]))
    load = [0] * world_size
    out = [[] for _ in range(world_size)]
    for g in units:
        r = min(range(world_size), key=lambda k: (load[k], k))
        out[r].extend(g)
        load[r] += sum(sizes[i] for i in g)
    return [sorted(x) for x in out]


def pack_exception(e: BaseException):
    """(class, str, attributes): exceptions whose __init__ formats its arguments do not unpickle."""
    return (type(e), str(e), dict(getattr(e, "__dict__", {})))


def unpack_exception(packed) -> BaseException:
    cls, text, attrs = packed
    e = cls.__new__(cls)
    BaseException.__init__(e, text)
    e.__dict__.update(attrs)
    return e


class Comm:
    """torch.distributed collectives on int64 / uint8 tensors (GPU for NCCL, CPU for gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        nccl = dist.get_backend(group) == "nccl"
        self.device = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")

    def max_i64(self, values):
        t = self.torch.tensor(values, dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t.tolist()

    def all_reduce_(self, t, op: str):
        ops = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX, "min": self.dist.ReduceOp.MIN}
        self.dist.all_reduce(t, op=ops[op], group=self.group)

    def all_gather_bytes(self, blob: bytes) -> list:
        torch = self.torch
        n = torch.tensor([len(blob)], dtype=torch.int64, device=self.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        cap = max(max(sizes), 1)
        mine = torch.zeros(cap, dtype=torch.uint8)
        if blob:
            mine[: len(blob)] = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
        mine = mine.to(self.device)
        bufs = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(bufs, mine, group=self.group)
        return [bytes(b[:k].cpu().numpy().tobytes()) for b, k in zip(bufs, sizes)]

    def all_gather_object(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def gather_to0(self, t, sizes):
        """Rank 0 receives every rank's 1-D uint8 tensor (sizes[r] bytes each; point-to-point sends)."""
        torch = self.torch
        on_dev = self.device.type == "cuda"
        if self.rank != 0:
            if sizes[self.rank]:
                self.dist.send(t if on_dev else t.cpu(), dst=0, group=self.group)
            return None
        out = [t]
        for r in range(1, self.world):
            buf = torch.empty(sizes[r], dtype=torch.uint8, device=self.device)
            if sizes[r]:
                self.dist.recv(buf, src=r, group=self.group)
            out.append(buf)
        return out


def _all_gather_i64(comm, values):
    """Every rank's small int list, concatenated in rank order."""
    torch = comm.torch
    t = torch.tensor(values, dtype=torch.int64, device=comm.device)
    out = [torch.zeros_like(t) for _ in range(comm.world)]
    comm.dist.all_gather(out, t, group=comm.group)
    return [int(x) for o in out for x in o.tolist()]


def _names_blob(names):
    enc = [n.encode("utf-8") for n in names]
    offs = [0]
    for b in enc:
        offs.append(offs[-1] + len(b))
    return b"".join(enc), offs


def _split_names(blob: bytes) -> list:
    """Inverse of the per-rank blob: u32 count, u32 lengths, then the bytes."""
    import struct

    if not blob:
        return []
    (n,) = struct.unpack_from("<I", blob, 0)
    lens = struct.unpack_from(f"<{n}I", blob, 4)
    out, at = [], 4 + 4 * n
    for k in lens:
        out.append(blob[at: at + k].decode("utf-8"))
        at += k
    return out


def _join_names(names) -> bytes:
    import struct

    enc = [n.encode("utf-8") for n in names]
    return struct.pack(f"<I{len(enc)}I", len(enc), *map(len, enc)) + b"".join(enc)


class ShardedRun:
    """Drive one engine over this rank's streams and merge across ranks.

    ``stream_global[i]``: global index of local stream i in the whole trace's (hostname, pid, tid)
    order; ``global_streams``: the whole trace's RawStream-like objects (hostname, pid, tid, name)
    in that order (labels, identities); ``comm``: a Comm, or None for one rank."""

    def __init__(self, engine, registry, comm=None, stream_global=None, global_streams=None):
        self.engine = engine
        self.registry = registry
        self.comm = comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        # the multi-rank protocol (split run, collectives, merge); HAPIGPU_COLLECTIVES=1 keeps it at
        # world size 1 (tests of the NCCL flavour on one GPU)
        self.multi = comm is not None and (self.world > 1 or os.environ.get("HAPIGPU_COLLECTIVES") == "1")
        self.stream_global = stream_global
        self.global_streams = global_streams
        self.global_last_ts = None
        self.rc = 0
        self._merged = None
        self._names = None

    # ------------------------------------------------------------------ step
    def step(self, want=HG_WANT_TALLY, input_error=None) -> dict:
        """Phase 1, the last-ts exchange, composition and the tally merge.  ``input_error``: an exception
        this rank met before the engine (e.g. a stream file header, tracefile.py:491-499), keyed by the
        global index of the stream it belongs to; every rank raises the first such error."""
        eng = self.engine
        sg = self.stream_global if self.stream_global is not None else list(range(len(eng._streams)))
        status, failure, last = STATUS_OK, None, 0
        if not self.multi and input_error is None:  # one rank: hg_run (the fused single-rank path)
            self.rc = eng.run_raw(want)
            self.global_last_ts = eng.local_last_ts()
            k, tot, h2d, d2h, nl = eng.timing()
            walk, chain, decode = eng.phase_timing()
            return {"device_ms": tot, "phase1_ms": k, "walk_ms": walk, "chain_ms": chain, "decode_ms": decode,
                    "h2d_bytes": h2d, "d2h_bytes": d2h, "launches": nl, "rc": self.rc}
        if input_error is not None:
            status, failure = STATUS_INPUT, ((0, input_error[0]), pack_exception(input_error[1]))
        else:
            try:
                eng.run_local(want)
                last = eng.local_last_ts()
                if eng.local_flags() & 1:
                    from .errors import UnsupportedTraceError

                    raise UnsupportedTraceError("multi-rank merge of device spans beyond the signed 64-bit range")
            except Exception as e:  # noqa: BLE001  (an engine failure: reported to every rank)
                status, failure = STATUS_ENGINE, ((2, self.rank), pack_exception(e))
        g, gstatus = last, status
        if self.multi:
            g, gstatus = self.comm.max_i64([last - _BIAS, status])
            g += _BIAS
        if gstatus:
            self._raise_first(failure)
        self.global_last_ts = g
        self.rc = eng.finish(g)
        if self.multi:
            self._merge(sg)
        k, tot, h2d, d2h, nl = eng.timing()
        walk, chain, decode = eng.phase_timing()
        return {"device_ms": tot, "phase1_ms": k, "walk_ms": walk, "chain_ms": chain, "decode_ms": decode,
                "h2d_bytes": h2d, "d2h_bytes": d2h, "launches": nl, "rc": self.rc}

    def _raise_first(self, failure):
        packed = [failure] if not self.multi else self.comm.all_gather_object(failure)
        key, exc = min((f for f in packed if f is not None), key=lambda f: f[0])
        if key[0] == 2 and failure is None:
            raise EngineError(f"rank {key[1]} failed: {unpack_exception(exc)}")
        raise unpack_exception(exc)

    def _merge(self, sg):
        """Names agreement, then the device-resident tally merge (two all-reduces, csrc/merge.cu)."""
        import numpy as np
        import torch

        eng, comm = self.engine, self.comm
        names = eng.device_names()
        gathered = [_split_names(b) for b in comm.all_gather_bytes(_join_names(names))]
        gnames = sorted({n for g in gathered for n in g})
        pos = {n: i for i, n in enumerate(gnames)}
        n_gs = len(self.global_streams) if self.global_streams is not None else max(sg, default=-1) + 1
        total, sum_n = eng.merge_size(len(gnames), n_gs)
        buf = torch.empty(total, dtype=torch.int64, device=eng.tensor_device())
        eng.merge_export(buf.data_ptr(), [pos[n] for n in names], len(gnames), sg, n_gs)
        coll = buf if buf.device == comm.device else buf.to(comm.device)
        comm.all_reduce_(coll[:sum_n], "sum")
        comm.all_reduce_(coll[sum_n:], "max")
        host = np.ascontiguousarray(coll.cpu().numpy())
        eng.merge_import(host.ctypes.data, gnames, n_gs)
        self._names = gnames
        self._merged = host
        self._n_gs = n_gs

    # ------------------------------------------------------------------ results
    def stats(self) -> dict:
        return self.engine.stats()

    def _global_spans(self):
        from .engine import MERGE_STATS

        return [int(x) for x in self._merged[MERGE_STATS: MERGE_STATS + self._n_gs]]

    def result(self, stream_infos=None, labels=None, orphan_labels=None):
        """(report, stats, orphans) of the whole trace, or raise the trace error the reference's single
        pipeline would raise (the same one on every rank)."""
        from .engine import MERGE_STATS

        eng = self.engine
        flat = eng._flat
        stats = self.stats()
        if not self.multi:
            gs = eng._streams
            idents = [(s.hostname, s.pid, s.tid) for s in gs]
            spans = eng.stream_spans()
            sg = list(range(len(gs)))
            any_error = self.rc == HG_TRACE_ERROR
        else:
            gs = self.global_streams
            idents = [(s.hostname, s.pid, s.tid) for s in gs]
            spans = self._global_spans()
            sg = self.stream_global
            any_error = int(self._merged[MERGE_STATS - 1]) > 0
        if orphan_labels is None:
            orphan_labels = [f"{s.hostname}/{s.pid}/{s.tid}" for s in gs]
        if labels is None:
            labels = [getattr(s, "name", "") for s in gs]
        orph_local = [SimpleNamespace(stream=sg[o.stream], function=o.function, ts=o.ts, seq=o.seq)
                      for o in eng.orphans_raw()]
        if any_error:
            err = self._first_error(sg, labels)
            orphans = orph_local if not self.multi else [o for g in self.comm.all_gather_object(orph_local) for o in g]
            key, exc, cut = err
            olist = orphan_list(orphans, orphan_labels, flat, cutoff=key, cut_streams=cut)
            return None, stats, olist, unpack_exception(exc)
        if self.multi and stats["orphan_exits"]:
            orphans = [o for g in self.comm.all_gather_object(orph_local) for o in g]
        else:
            orphans = orph_local
        olist = orphan_list(orphans, orphan_labels, flat)
        report = build_report(flat, eng.tally_rows(), eng.device_names(), stream_infos, idents, spans)
        return report, stats, olist, None

    def _first_error(self, sg, labels):
        """The error the reference's muxer raises first: per rank the local first candidate (global
        stream indices), then the minimum of error_key over all ranks."""
        from .tracefile import RawStream

        eng = self.engine
        cands = [SimpleNamespace(code=c.code, stream=sg[c.stream], seq=c.seq, offset=c.offset, ts=c.ts,
                                 prev_ts=c.prev_ts, aux=c.aux, local=c.stream) for c in eng.errors_raw()]
        cut = {}
        for c in cands:
            if c.code in (1, 2, 3, 4, 5, 6, 7, 8, 9) and (c.stream not in cut or c.seq < cut[c.stream]):
                cut[c.stream] = c.seq
        mine = None
        e = first_error(cands)
        if e is not None:
            s = eng._streams[e.local]
            named = RawStream(s.hostname, s.pid, s.tid, labels[e.stream], s.data, getattr(s, "info", None))
            mine = (error_key(e), pack_exception(make_exception(e, named, eng._flat)), cut)
        allc = [mine] if not self.multi else self.comm.all_gather_object(mine)
        key, exc, _ = min((c for c in allc if c is not None), key=lambda c: c[0])
        cuts = {}
        for c in allc:
            if c is not None:
                cuts.update(c[2])
        return key, exc, cuts

    def timeline(self, device_index=0):
        """The whole trace's TimelineSink JSON after a step with HG_WANT_TL_ITEMS (collective (6) of
        SURVEY.md §8e): every rank exports its sorted messages with global stream keys
        (hg_tl_export), rank 0 receives them and merges + formats them (hg_tl_import).  Returns the
        bytes on rank 0, None on the other ranks."""
        import ctypes as C

        import torch

        eng, comm = self.engine, self.comm
        L, ctx = eng._L, eng._ctx
        gs = self.global_streams
        n_gs = len(gs)
        order = sorted(range(n_gs), key=lambda i: (str(gs[i].hostname), gs[i].pid or 0, gs[i].tid or 0, i))
        flush_rank = [0] * n_gs
        for k, i in enumerate(order):
            flush_rank[i] = k
        sg = self.stream_global
        ns = len(sg)
        n, pb, ndev = C.c_uint64(), C.c_uint64(), C.c_uint64()
        eng._check(L.hg_tl_export(ctx, None, None, None, None, C.byref(n), C.byref(pb), C.byref(ndev)), "hg_tl_export")
        dev = eng.tensor_device()
        items = torch.empty(max(40 * n.value, 1), dtype=torch.uint8, device=dev)
        pay = torch.empty(max(pb.value, 1), dtype=torch.uint8, device=dev)
        smap = (C.c_uint32 * max(ns, 1))(*sg)
        fmap = (C.c_uint32 * max(ns, 1))(*[flush_rank[g] for g in sg])
        eng._check(L.hg_tl_export(ctx, smap, fmap, C.c_void_p(items.data_ptr()), C.c_void_p(pay.data_ptr()),
                                  C.byref(n), C.byref(pb), C.byref(ndev)), "hg_tl_export")
        meta = [int(x) for x in _all_gather_i64(comm, [n.value, pb.value, ndev.value])]
        counts, pays, devs = meta[0::3], meta[1::3], meta[2::3]
        got_items = comm.gather_to0(items[: 40 * n.value], [40 * c for c in counts])
        got_pay = comm.gather_to0(pay[: pb.value], pays)
        if comm.rank != 0:
            return None
        run0, pay0, a, b = [], [], 0, 0
        for c, p_ in zip(counts, pays):
            run0.append(a)
            pay0.append(b)
            a += c
            b += p_
        all_items = torch.cat([t.to(dev) for t in got_items] + [items[:40]])  # + padding: never empty
        all_pay = torch.cat([t.to(dev) for t in got_pay] + [pay[:1]])
        hosts = (C.c_char_p * max(n_gs, 1))(*[None if x.hostname is None else str(x.hostname).encode() for x in gs])
        pids = (C.c_int64 * max(n_gs, 1))(*[-(1 << 63) if x.pid is None else int(x.pid) for x in gs])
        tids = (C.c_int64 * max(n_gs, 1))(*[-(1 << 63) if x.tid is None else int(x.tid) for x in gs])
        eng._check(L.hg_set_timeline_device(ctx, int(device_index)), "hg_set_timeline_device")
        eng._check(L.hg_tl_import(ctx, C.c_void_p(all_items.data_ptr()), a, (C.c_uint64 * len(run0))(*run0),
                                  (C.c_uint64 * len(pay0))(*pay0), len(run0), C.c_void_p(all_pay.data_ptr()), hosts,
                                  pids, tids, n_gs, (C.c_uint32 * max(n_gs, 1))(*order), sum(devs),
                                  self.global_last_ts), "hg_tl_import")
        return eng.timeline_bytes()

    # the round-1 name, kept for callers that only want the tally
    def report(self, stream_infos=None):
        rep, _, _, err = self.result(stream_infos)
        if err is not None:
            raise err
        return rep
