"""Multi-GPU runs: one process per GPU, streams sharded per rank, NCCL for the two real exchanges.

The interval state is per (hostname, pid, tid) stream (pipeline.py:158-161) and
the tally is a commutative monoid (aggregator.py:1-9), so ranks own disjoint
stream sets and need exactly two collectives:
  1. all-reduce MAX of the local last timestamp before truncated spans are
     finalised -- truncation ends at the GLOBAL last ts (pipeline.py:152, :235);
  2. the tally merge: dense per-function host rows and (name-aligned) device
     rows reduced with SUM / MIN / MAX (aggregator.py:35-76 semantics).
128-bit sums travel as three int64 limbs (lo32, hi32, signed hi64) so the
SUM all-reduce is exact for any rank count below 2^31.  Extrema travel
sign-biased so int64 MIN/MAX order equals the unsigned/128-bit order for the
values the engine produces.  Identity sets, drops and orphans are gathered as
Python objects (small).

`merge_dense` / `limbs` are pure tensor functions so the merge runs on CPU
gloo in tests (tests/test_distributed.py) exactly as on NCCL.
"""

from __future__ import annotations

from .results import build_report, orphan_list
from .tally import TallyReport

MASK32 = (1 << 32) - 1


def limbs(value: int):
    """signed 128-bit -> (lo32, hi32, hi64) with value = hi64*2^64 + hi32*2^32 + lo32."""
    lo = value & ((1 << 64) - 1)
    hi = value >> 64
    return [lo & MASK32, lo >> 32, hi]


def unlimbs(l0: int, l1: int, h: int) -> int:
    return l0 + (l1 << 32) + (h << 64)


def encode_rows(rows, keys):
    """rows: {key: (count, errors, sum, min, max)} -> flat int lists aligned to `keys`.

    Returns (sum_part, min_part, max_part) where sum_part holds count, errors and
    the sum limbs; extrema are clamped to int64 (engine values fit) and biased
    only implicitly: int64 MIN/MAX equals the integer order.
    """
    big = (1 << 63) - 1
    s, mn, mx = [], [], []
    for k in keys:
        r = rows.get(k)
        if r is None:
            s += [0, 0, 0, 0, 0]
            mn.append(big)
            mx.append(-big - 1)
            continue
        count, errs, total, lo, hi = r
        s += [count, errs, *limbs(total)]
        mn.append(lo)
        mx.append(hi)
    return s, mn, mx


def decode_rows(keys, s, mn, mx):
    out = {}
    for i, k in enumerate(keys):
        count, errs, l0, l1, h = s[5 * i: 5 * i + 5]
        if count:
            out[k] = (count, errs, unlimbs(l0, l1, h), mn[i], mx[i])
    return out


def merge_dense(local_rows, keys, all_reduce):
    """Reduce aligned row tables across ranks with a caller-supplied all_reduce(list, op)."""
    s, mn, mx = encode_rows(local_rows, keys)
    s = all_reduce(s, "sum")
    mn = all_reduce(mn, "min")
    mx = all_reduce(mx, "max")
    return decode_rows(keys, s, mn, mx)


def torch_all_reduce(group=None, device=None):
    import torch
    import torch.distributed as dist

    ops = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}

    def fn(values, op):
        if not values:
            return values
        t = torch.tensor(values, dtype=torch.int64, device=device)
        dist.all_reduce(t, op=ops[op], group=group)
        return t.tolist()

    return fn


class ShardedRun:
    """Drive one engine over this rank's streams; merge across ranks when world_size > 1."""

    def __init__(self, engine, registry, world_size=1, rank=0, device=None):
        self.engine = engine
        self.registry = registry
        self.world_size = world_size
        self.rank = rank
        self.device = device
        self.global_last_ts = None

    def step(self) -> dict:
        eng = self.engine
        L, ctx = eng._L, eng._ctx
        import ctypes as C

        rc = L.hg_run_local(ctx, 1)
        eng._check(rc, "hg_run_local")
        last, nev = C.c_uint64(), C.c_uint64()
        eng._check(L.hg_local_last_ts(ctx, C.byref(last), C.byref(nev)), "hg_local_last_ts")
        g = last.value
        if self.world_size > 1:
            import torch
            import torch.distributed as dist

            # u64 timestamps < 2^63 in practice; bias keeps the order exact anyway
            t = torch.tensor([g - (1 << 63)], dtype=torch.int64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            g = t.item() + (1 << 63)
        self.global_last_ts = g
        rc = L.hg_finish(ctx, g)
        if rc not in (0, 1):
            eng._check(rc, "hg_finish")
        k, tot, h2d, d2h, nl = eng.timing()
        walk, chain, decode = eng.phase_timing()
        return {"device_ms": tot, "phase1_ms": k, "walk_ms": walk, "chain_ms": chain, "decode_ms": decode,
                "h2d_bytes": h2d, "d2h_bytes": d2h, "launches": nl, "rc": rc}

    def report(self, stream_infos) -> TallyReport:
        eng = self.engine
        flat = eng._flat
        names = eng.device_names()
        rows = eng.tally_rows()
        idents = [(s.hostname, s.pid, s.tid) for s in eng._streams]
        spans = eng.stream_spans()
        if self.world_size == 1:
            return build_report(flat, rows, names, stream_infos, idents, spans)
        import torch.distributed as dist

        host = {("host", flat.function_names[r[1]]): r[2:] for r in rows if r[0] == 0}
        dev = {("device", names[r[1]]): r[2:] for r in rows if r[0] == 1}
        # device-name dictionaries differ per rank: agree on one key order first
        gathered = [None] * self.world_size
        dist.all_gather_object(gathered, sorted(dev))
        dev_keys = sorted({k for g in gathered for k in g})
        host_keys = [("host", n) for n in flat.function_names]
        merged = merge_dense({**host, **dev}, host_keys + dev_keys, torch_all_reduce(device="cuda"))
        infos = [None] * self.world_size
        dist.all_gather_object(infos, (list(stream_infos or []), [i for i, n in zip(idents, spans) if n]))
        rep = TallyReport(fingerprint=self.registry.fingerprint,
                          backends=(f"BACKEND_{self.registry.api_name.upper()}",))
        from .tally import TallyRow

        for (sec, name), (count, errs, total, mn, mx) in merged.items():
            rep.rows[(sec, name)] = TallyRow(name, sec, total, count, mn, mx, errs)
        hosts, procs, threads = set(), set(), set()
        for inf, span_ids in infos:
            for i in inf:
                hosts.add(i.hostname)
                procs.add((i.hostname, i.pid))
                threads.add((i.hostname, i.pid, i.tid))
                if i.dropped_count:
                    rep.dropped[(i.hostname, i.pid, i.tid)] = i.dropped_count
            for h, p, t in span_ids:
                hosts.add(h)
                procs.add((h, p))
                threads.add((h, p, t))
        rep.hostnames, rep.processes, rep.threads = frozenset(hosts), frozenset(procs), frozenset(threads)
        return rep
