"""TEST INFRASTRUCTURE: a CPU stand-in for engine.Engine in the multi-rank host-logic tests.

It implements the Engine surface that distributed.ShardedRun and pipeline.run_pipeline(distributed=...)
drive (set_registry / set_streams / run_local / local_last_ts / finish / merge_* / result getters) with
the CPU oracle doing the per-rank work, and restates csrc/merge.cu's buffer layout in numpy, so the
collectives, the name agreement, the error / orphan reconciliation and the partitioner run for real
over gloo on CPU.  The GPU version of the same flow is tests/test_gpu_distributed.py.
"""

from __future__ import annotations

import ctypes as C
from types import SimpleNamespace

import numpy as np

MERGE_STATS = 8
BIAS = 1 << 63
M64 = (1 << 64) - 1


def _key(u):  # (int64)(u ^ 2^63)
    v = (u ^ BIAS) & M64
    return v - (1 << 64) if v >> 63 else v


class FakeEngine:
    def __init__(self, fail_run=False):
        self.device = -1
        self._flat = None
        self._streams = []
        self.fail_run = fail_run

    # inputs
    def set_registry(self, registry):
        from paper_2504_03683_b200.abi import flatten_registry

        self.registry = registry
        self._flat = flatten_registry(registry)
        return self._flat

    def set_streams(self, raws):
        self._streams = list(raws)

    def tensor_device(self):
        import torch

        return torch.device("cpu")

    # run
    def run_local(self, want=1):
        """The sequential oracle over this rank's streams: last ts, raw orphans, the raw first error."""
        from oracle import oracle
        from paper_2504_03683_b200.abi import HgOrphan, HgStats, HgTraceError
        from paper_2504_03683_b200.errors import EngineError

        if self.fail_run:
            raise EngineError("injected engine failure")
        L = oracle.lib()
        flat = self._flat
        n = len(self._streams)
        bufs = [C.create_string_buffer(s.data, len(s.data)) if s.data else None for s in self._streams]
        ptrs = (C.c_void_p * max(n, 1))(*[C.cast(b, C.c_void_p) if b is not None else None for b in bufs])
        sizes = (C.c_uint64 * max(n, 1))(*[len(s.data) for s in self._streams])
        h = L.oracle_run(flat.schemas, flat.n_schemas, flat.kinds, len(flat.function_names), n, ptrs, sizes, 0,
                         None, None)
        try:
            self._last = L.oracle_last_ts(h)
            st = HgStats()
            L.oracle_stats(h, C.byref(st))
            self._orphan_total = st.orphan_exits
            k = L.oracle_orphans(h, None, 0)
            arr = (HgOrphan * max(k, 1))()
            L.oracle_orphans(h, arr, k)
            self._orph = [SimpleNamespace(stream=o.stream, function=o.function, ts=o.ts, seq=o.seq)
                          for o in list(arr)[:k]]
            e = HgTraceError()
            self._errors = []
            if L.oracle_has_error(h, C.byref(e)):
                self._errors = [SimpleNamespace(code=e.code, stream=e.stream, seq=e.seq, offset=e.offset, ts=e.ts,
                                                prev_ts=e.prev_ts, aux=e.aux)]
        finally:
            L.oracle_free(h)

    def local_last_ts(self):
        return self._last

    def local_flags(self):
        return 0

    def finish(self, g):
        """Rows, names, stats and span identities with truncation at the global last ts g."""
        from oracle import oracle

        r = oracle.run(self._streams, self.registry, None, threads=1, floor_last_ts=g)
        fnid = {n: i for i, n in enumerate(self._flat.function_names)}
        self._names = sorted(k[1] for k in r.report.rows if k[0] == "device")
        did = {n: i for i, n in enumerate(self._names)}
        self._rows = []
        for (sec, name), row in r.report.rows.items():
            nid = fnid[name] if sec == "host" else did[name]
            self._rows.append((0 if sec == "host" else 1, nid, row.count, row.error_count, row.time_ns, row.min_ns,
                               row.max_ns))
        self._stats = dict(r.stats)
        self._stats["orphan_exits"] = self._orphan_total
        idents = {(s.hostname, s.pid, s.tid): i for i, s in enumerate(self._streams)}
        self._spans = [0] * len(self._streams)
        for ident in r.report.threads:
            if ident in idents:
                self._spans[idents[ident]] = 1
        return 1 if self._errors else 0

    # merge (numpy restatement of csrc/merge.cu)
    def merge_size(self, n_dev_global, n_gs):
        R = len(self._flat.function_names) + n_dev_global
        return MERGE_STATS + n_gs + 7 * R, MERGE_STATS + n_gs + 5 * R

    def merge_export(self, ptr, dev_map, n_dev_global, stream_global, n_gs):
        n_fn = len(self._flat.function_names)
        R = n_fn + n_dev_global
        total = MERGE_STATS + n_gs + 7 * R
        b = np.ctypeslib.as_array((C.c_int64 * total).from_address(ptr))
        keys = ("events_in", "passed", "host_spans", "truncated_spans", "device_spans", "samples", "orphan_exits")
        b[:] = 0
        for i, k in enumerate(keys):
            b[i] = self._stats[k]
        b[7] = 1 if self._errors else 0
        for i, g in enumerate(stream_global):
            b[MERGE_STATS + g] = self._spans[i]
        rows = MERGE_STATS + n_gs
        mn, mx = rows + 5 * R, rows + 6 * R
        b[mn: mn + R] = ~0x7FFFFFFFFFFFFFFF
        b[mx: mx + R] = -(1 << 63)
        for sec, nid, count, errs, total_ns, lo, hi in self._rows:
            g = nid if sec == 0 else n_fn + dev_map[nid]
            t = total_ns & ((1 << 128) - 1)
            lo64, hi64 = t & M64, t >> 64
            b[rows + 5 * g: rows + 5 * g + 5] = [count, errs, lo64 & 0xFFFFFFFF, lo64 >> 32,
                                                hi64 - (1 << 64) if hi64 >> 63 else hi64]
            u_lo = lo & M64 if sec == 0 else (lo + BIAS) & M64
            u_hi = hi & M64 if sec == 0 else (hi + BIAS) & M64
            b[mn + g] = ~_key(u_lo)
            b[mx + g] = _key(u_hi)

    def merge_import(self, ptr, names, n_gs):
        n_fn = len(self._flat.function_names)
        R = n_fn + len(names)
        total = MERGE_STATS + n_gs + 7 * R
        b = [int(x) for x in np.ctypeslib.as_array((C.c_int64 * total).from_address(ptr))]
        keys = ("events_in", "passed", "host_spans", "truncated_spans", "device_spans", "samples", "orphan_exits")
        self._stats = {k: b[i] for i, k in enumerate(keys)}
        rows = MERGE_STATS + n_gs
        mn, mx = rows + 5 * R, rows + 6 * R
        self._rows, self._names = [], list(names)
        for g in range(R):
            count, errs, l0, l1, h = b[rows + 5 * g: rows + 5 * g + 5]
            if not count:
                continue
            total_ns = l0 + (l1 << 32) + (h << 64)
            u_lo = ((~b[mn + g]) & M64) ^ BIAS
            u_hi = (b[mx + g] & M64) ^ BIAS
            if g < n_fn:
                self._rows.append((0, g, count, errs, total_ns, u_lo, u_hi))
            else:
                s = lambda u: u - (1 << 64) if u >> 63 else u  # noqa: E731
                self._rows.append((1, g - n_fn, count, errs, total_ns, s((u_lo - BIAS) & M64), s((u_hi - BIAS) & M64)))

    # getters
    def timing(self):
        return 0.0, 0.0, 0, 0, 0

    def phase_timing(self):
        return 0.0, 0.0, 0.0

    def stats(self):
        return dict(self._stats)

    def tally_rows(self):
        return list(self._rows)

    def device_names(self):
        return list(self._names)

    def stream_spans(self):
        return list(self._spans)

    def orphans_raw(self):
        return list(self._orph)

    def errors_raw(self):
        return list(self._errors)
