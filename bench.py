"""Benchmark: events/s for decode+pair+tally on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2] [--scale 1.0]

A "step" is one pass of the hot path (decode -> pair -> tally, SURVEY.md §8a
rows a2-a5) over one synthetic trace of the named configuration.  N=1: config
C2 (100M events, 4 procs x 64 threads = 256 streams, bundled ze registry).
N>1 (one process per GPU; `--gpus N` relaunches itself under torchrun): config
C3 (1B events, 1,024 streams) sharded over the ranks by the product's LPT
partitioner -- each rank generates only its streams -- with the last-ts
exchange and the device-resident tally merge (NCCL) inside every timed step
(strong scaling).

Rank 0 prints ONE JSON line.  `value` = whole-job events / max-over-ranks
device time per step with the trace resident in HBM; `e2e` = the same metric
through the public API with the trace in pinned host memory, H2D and result
D2H inside the timed region; `parity` = the timed run's TallyReport and
IntervalStats against the CPU oracle over the same streams at full size (the
run exits non-zero on a mismatch).  `--impl reference` times the CPU oracle (C
restatement of the reference path, oracle/hapi_oracle.c) with all host cores
on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "events/sec decode+pair+tally at 1/2/4/8 B200; % of HBM roofline"


def _peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def loop():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(0.1)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_name(args, ws):
    """C2 (100M events, one B200) at N=1; C3 (1B events, 8 hosts x 4 procs x 32 threads) sharded over
    the ranks at N>1 -- BASELINE.json configs[1] and configs[2]."""
    if args.config:
        return args.config
    return "c2" if ws == 1 else "c3"


DESCR = {
    "c2": "SURVEY.md §8(d) C2: 100M-event synthetic L0-style trace, 4 procs x 64 threads (256 streams), bundled ze "
          "registry, one B200",
    "c3": "SURVEY.md §8(d) C3: 1B-event multi-host trace, 8 hosts x 4 procs x 32 threads (1,024 streams), streams "
          "sharded over the ranks by LPT on bytes, NCCL merge",
}


def shared_config(name, scale, ws):
    """The `config` both arms print (same dict -> the driver sees the same workload)."""
    from paper_2504_03683_b200 import synth

    wl = synth.config(name, scale)
    events = sum(s.n_events for s in wl.streams if s.kind == "calls")
    return {"workload": f"{name} x{scale}: {DESCR.get(name, name)}", "events": events,
            "streams": len(wl.streams), "n_gpus": ws}


def my_streams(name, scale, ws, rank):
    """This rank's part of the workload: the product's partitioner over the streams' expected sizes
    (event counts); only those streams are generated.  Returns (workload, global index list)."""
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.distributed import partition_streams

    wl = synth.config(name, scale)
    order = sorted(range(len(wl.streams)), key=lambda i: (wl.streams[i].hostname, wl.streams[i].pid,
                                                          wl.streams[i].tid))
    specs = [wl.streams[i] for i in order]
    mine = partition_streams([s.n_events for s in specs], ws)[rank] if ws > 1 else list(range(len(specs)))
    sub = synth.Workload(wl.name, wl.registry, [specs[i] for i in mine], wl.params, wl.layers, wl.kernel_names,
                         wl.sampler_period_ns)
    return sub, mine, specs


def oracle_check(raws, registry, threads, floor_last_ts=0, with_infos=True):
    """The CPU oracle (C restatement of the reference path, test infrastructure) over these streams,
    sharded over host threads: the parity reference for the timed run."""
    from oracle import oracle

    t = time.perf_counter()
    r = oracle.run(raws, registry, [x.info for x in raws] if with_infos else None, threads=threads,
                   floor_last_ts=floor_last_ts)
    return r, time.perf_counter() - t


def cpu_baseline(raws, registry, target_s=10.0, max_events=None):
    """Oracle (C restatement) tally with all host threads on a bounded sample of the workload."""
    from oracle import oracle

    cores = os.cpu_count() or 1
    total = sum(r.info.event_count for r in raws)
    # probe on a small slice to size the sample for ~target_s seconds
    k = max(1, min(len(raws), cores))
    probe = raws[:k]
    t = time.perf_counter()
    oracle.run(probe, registry, [r.info for r in probe], threads=cores)
    dt = time.perf_counter() - t
    rate = sum(r.info.event_count for r in probe) / max(dt, 1e-9)
    want_events = min(total, int(rate * target_s), max_events or total)
    n = k
    acc = sum(r.info.event_count for r in raws[:n])
    while n < len(raws) and acc < want_events:
        acc += raws[n].info.event_count
        n += 1
    sample = raws[:n]
    ev = sum(r.info.event_count for r in sample)
    t = time.perf_counter()
    oracle.run(sample, registry, [r.info for r in sample], threads=cores)
    dt = time.perf_counter() - t
    return {"value": ev / dt, "unit": "events/s", "cores": cores, "kind": "port",
            "sample": f"{n} of {len(raws)} streams ({ev} events) of the same workload, oracle/hapi_oracle.c "
                      f"sharded over {cores} threads, {dt:.2f} s"}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from paper_2504_03683_b200 import synth

    name = workload_name(args, ws)
    cfg = shared_config(name, args.scale, ws)
    wl = synth.config(name, args.scale)
    # a bounded sample of the workload: the first streams in mux order, about 100M events at most
    specs = sorted([s for s in wl.streams if s.kind == "calls"], key=lambda s: (s.hostname, s.pid, s.tid))
    keep, acc = [], 0
    for s in specs:
        if acc >= 100_000_000:
            break
        keep.append(s)
        acc += s.n_events
    if len(keep) < len(specs):
        wl = synth.Workload(wl.name, wl.registry, keep, wl.params, wl.layers, wl.kernel_names, wl.sampler_period_ns)
    raws = synth.generate(wl)
    times = []
    base = None
    for i in range(args.warmup + args.steps):
        b = cpu_baseline(raws, wl.registry, target_s=args.ref_seconds)
        if i >= args.warmup:
            times.append(b["value"])
            base = b
    value = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {**base, "value": value},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _parity_line(got_rep, got_stats, want_rep, want_stats):
    if got_rep == want_rep and got_stats == want_stats:
        return "exact"
    diff = [k for k in set(got_rep.rows) | set(want_rep.rows) if got_rep.rows.get(k) != want_rep.rows.get(k)]
    return f"MISMATCH: stats {got_stats != want_stats}, rows {sorted(diff)[:5]}"


def run_ours(args):
    import torch

    ws, rank, local = _dist()
    comm = None
    dev = local % max(torch.cuda.device_count(), 1)  # == local on a real node; >1 rank per GPU only with gloo
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(dev)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:  # gloo: the N>1 code path on one GPU (tests), collectives through host memory
            dist.init_process_group("gloo")
        from paper_2504_03683_b200.distributed import Comm

        comm = Comm()
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.distributed import ShardedRun
    from paper_2504_03683_b200.engine import Engine
    from paper_2504_03683_b200.tally import merge_tallies
    from paper_2504_03683_b200.tracefile import RawStream

    name = workload_name(args, ws)
    cfg = shared_config(name, args.scale, ws)
    t0 = time.perf_counter()
    sub, mine, specs = my_streams(name, args.scale, ws, rank)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    threads = max(1, (os.cpu_count() or 1) // local_world)
    raws = synth.generate(sub, threads=threads)
    gen_s = time.perf_counter() - t0
    n_events = sum(r.info.event_count for r in raws)
    n_bytes = sum(len(r.data) for r in raws)
    infos = [r.info for r in raws]
    gstreams = [RawStream(s.hostname, s.pid, s.tid, s.file or f"stream_{s.pid}_{s.tid}.bin", b"") for s in specs]

    eng = Engine(device=dev)
    runner = ShardedRun(eng, sub.registry, comm, stream_global=mine, global_streams=gstreams)

    # ---- device-resident timing (value): the trace is in HBM before the timed region
    eng.set_registry(sub.registry)
    eng.set_streams(raws)
    eng.stage()
    for _ in range(args.warmup):
        runner.step()
    step_ms, dec_ms, ph1_ms, launches = [], [], [], 0
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clk = Clocks(dev)
    with clk:
        for i in range(args.steps):
            ev0[i].record()
            info = runner.step()
            ev1[i].record()
            dec_ms.append(info["decode_ms"])
            ph1_ms.append(info["phase1_ms"])
            step_ms.append(info["device_ms"])
            launches += info["launches"]
    torch.cuda.synchronize()
    if ws > 1:  # the whole step incl. the merge collectives, on the device clock of the current stream
        step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    ms = statistics.mean(step_ms)
    tms = statistics.mean(dec_ms)
    p1 = statistics.mean(ph1_ms)
    tot_events, tot_bytes = n_events, n_bytes
    if ws > 1:
        t = torch.tensor([ms, tms, p1], dtype=torch.float64, device=comm.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, tms_max, p1 = t.tolist()
        e = torch.tensor([n_events, n_bytes], dtype=torch.int64, device=comm.device)
        torch.distributed.all_reduce(e)
        tot_events, tot_bytes = e.tolist()
    value = tot_events / (ms / 1e3)
    rep, stats, _, err = runner.result(infos if ws == 1 else None)
    if err is not None:
        raise err

    # ---- parity of the timed run against the CPU oracle, at full size
    t_or = time.perf_counter()
    want, or_s = oracle_check(raws, sub.registry, threads, floor_last_ts=runner.global_last_ts,
                              with_infos=ws == 1)
    if ws > 1:  # per-shard oracle reports merged the reference's way (aggregator.py:35-76)
        reps = comm.all_gather_object((want.report, want.stats))
        want_rep = merge_tallies([r for r, _ in reps])
        want_stats = {k: sum(s[k] for _, s in reps) for k in want.stats}
    else:
        want_rep, want_stats = want.report, want.stats
    parity = _parity_line(rep, stats, want_rep, want_stats)
    parity_s = time.perf_counter() - t_or

    # ---- end to end through the public API from pinned host memory (e2e)
    pinned = []
    for r in raws:
        t = torch.empty(len(r.data), dtype=torch.uint8, pin_memory=True)
        if len(r.data):
            t.copy_(torch.frombuffer(bytearray(r.data), dtype=torch.uint8))
        pinned.append(t)
    e2e_s = []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        eng.set_streams_pinned([(r.hostname, r.pid, r.tid) for r in raws], pinned)
        info = runner.step()
        rep2, _, _, _ = runner.result(infos if ws == 1 else None)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            e2e_s.append(dt)
            h2d, d2h = info["h2d_bytes"], info["d2h_bytes"]
    e2e = statistics.mean(e2e_s)
    if ws > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device=comm.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = t.item()
    if rep2 != rep:
        parity = "MISMATCH: e2e run differs from the resident run"

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        if parity != "exact":
            sys.exit(1)
        return
    peak, peak_src = _peaks()
    path, fallbacks, range_bytes = eng.last_path()
    single = path == 1
    achieved = (n_bytes / (tms / 1e3)) / 1e9  # rank 0: its trace bytes over its decode kernel time
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "events/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic",
        "config": cfg,
        "parity": parity,
        "workload_detail": {
            "events_per_gpu_rank0": n_events,
            "bytes_per_gpu_rank0": n_bytes,
            "bytes_per_event": n_bytes / max(n_events, 1),
            "total_events": tot_events,
            "total_bytes": tot_bytes,
            "parallelism": (f"{ws} ranks, streams by LPT on bytes (distributed.partition_streams); per step: "
                            "MAX all-reduce of [last ts, status], device-name all-gather, SUM + MAX all-reduce of "
                            "the device-resident tally buffer (csrc/merge.cu), all inside the timed step")
            if ws > 1 else "1 GPU",
            "timing": "engine CUDA events (staging -> results on host)" if ws == 1 else
                      "CUDA events on the current stream around the whole step incl. merge, max over ranks",
            "l2": "input (GBs) >> 126 MB L2: no flush needed between steps",
            "generation_s": round(gen_s, 2),
            "parity_check": f"timed run's TallyReport + IntervalStats vs oracle/hapi_oracle.c over the same "
                            f"{'streams' if ws == 1 else 'shards (merged with merge_tallies)'} at full size, "
                            f"{threads} host threads, {or_s:.2f} s",
        },
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": None,
            "kernel": "fast_scan_kernel + fast_kernel" if single else "seg_decode_kernel",
            "kernel_ms": tms,
            "algorithmic_bytes_per_launch": n_bytes,
            "peak_source": peak_src,
            "phase1": {"kernels": ("fast_scan_kernel + fast_kernel + fast_verify_kernel + fast_orphan_fix_kernel" if single
                                   else "seg_walk_kernel + seg_chain_kernel + seg_decode_kernel"),
                       "path": "single pass over HBM (csrc/fast.cuh)" if single else "exact three-kernel path",
                       "range_bytes": range_bytes, "fallbacks": fallbacks, "ms": p1,
                       "achieved": (n_bytes / (p1 / 1e3)) / 1e9,
                       "frac": (n_bytes / (p1 / 1e3)) / 1e9 / peak},
        },
        "cpu_baseline": cpu_baseline(raws, sub.registry, target_s=args.ref_seconds, max_events=100_000_000),
        "e2e": {"value": tot_events / e2e, "unit": "events/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "Engine.set_streams_pinned + ShardedRun.step + ShardedRun.result (hg_add_stream host "
                        "pointers into pinned memory; hg_run at N=1, hg_run_local/hg_finish + merge at N>1), wall "
                        "clock per step, max over ranks"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if ws == 1 and not args.no_dropin:
        line["e2e_dropin"] = dropin_side(eng, sub, raws, rep, stats, args)
        if line["e2e_dropin"].get("parity", "exact") != "exact":
            parity = line["parity"] = "MISMATCH in e2e_dropin"
    if ws == 1 and not args.no_timeline:
        line["timeline"] = timeline_side(eng, threads)
        if line["timeline"]["parity"] != "exact" and parity == "exact":
            parity = line["parity"] = "MISMATCH in timeline"
    if ws == 1 and not args.no_configs:
        line["other_configs"] = configs_side(eng, threads)
    traffic = REPO / "profiles" / ("fast_kernel_traffic.json" if single else "seg_decode_traffic.json")
    if traffic.exists():
        tr = json.loads(traffic.read_text())
        line["roofline"]["traffic"] = tr.get("dram_bytes_per_launch")
        line["roofline"]["traffic_source"] = tr.get("source")
    bad = [c for c in line.get("other_configs", []) if c.get("parity") != "exact"]
    if bad and parity == "exact":
        parity = "MISMATCH in other_configs: " + ", ".join(c["config"] for c in bad)
        line["parity"] = parity
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    if parity != "exact":
        sys.exit(1)


def dropin_side(eng, wl, raws, rep, stats, args):
    """The reference's own call on files (harness.py:117-121 / pipeline.py:275-314):
    run_pipeline(open_trace_reader(dir), [TallySink()]) over the workload written to disk, the engine
    reading the stream files itself (csrc/ingest.cu: pinned double-buffered chunks, reads overlapped
    with the PCIe copies).  Page cache warm (the files were just written)."""
    import shutil
    import tempfile

    from paper_2504_03683_b200 import TallySink, open_trace_reader, run_pipeline, synth

    total = sum(len(r.data) for r in raws)
    tmp = Path(os.environ.get("HAPIGPU_BENCH_TMP", tempfile.gettempdir()))
    if shutil.disk_usage(tmp).free < 2 * total + (1 << 30):
        return {"skipped": f"not enough space in {tmp} for {total} bytes"}
    d = Path(tempfile.mkdtemp(prefix="hapigpu_dropin_", dir=tmp))
    try:
        t = time.perf_counter()
        synth.write(wl, raws, d / "trace")
        write_s = time.perf_counter() - t
        walls, ing = [], None
        res = None
        for i in range(args.warmup + max(3, args.steps // 4)):
            t = time.perf_counter()
            res = run_pipeline(open_trace_reader(d / "trace"), [TallySink()], engine=eng)
            dt = time.perf_counter() - t
            if i >= args.warmup:
                walls.append(dt)
                ing = eng.ingest_stats()
        ev = stats["events_in"]
        ok = res["tally"] == rep and vars(res.stats) == stats
        return {"value": ev / statistics.mean(walls), "unit": "events/s", "wall_ms": 1e3 * statistics.mean(walls),
                "ingest": ing, "ingest_gb_per_s": ing["file_bytes"] / ing["ms"] / 1e6 if ing["ms"] else None,
                "trace_write_s": round(write_s, 2), "parity": "exact" if ok else "MISMATCH",
                "path": "run_pipeline(open_trace_reader(dir), [TallySink()]) from stream files, page cache warm; "
                        "wall clock per call incl. index/header reads, file -> pinned -> HBM, kernels, report"}
    finally:
        shutil.rmtree(d, ignore_errors=True)


def timeline_side(eng, threads, config="c5", scale=1.0):
    """Row a8 (TimelineSink) on the device-heavy config at full size: tally + Chrome-trace JSON of
    SURVEY.md §8(d) C5 (100M events, 30%+ device-profiling records).  Device time of phase 1 and of the
    ordering + JSON formatting; roofline bytes = the trace read once + the JSON written once.  Checks
    (size-independent): object count = interval messages + metadata objects, json.dump framing, the
    tally of the timeline run equal to the CPU oracle's."""
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.abi import HG_WANT_TALLY, HG_WANT_TIMELINE
    from paper_2504_03683_b200.results import build_report

    wl = synth.config(config, scale)
    raws = synth.generate(wl, threads=threads)
    infos = [r.info for r in raws]
    in_bytes = sum(len(r.data) for r in raws)
    eng.set_registry(wl.registry)
    eng.set_streams(raws)
    eng.stage()
    p1, tlm = [], []
    for i in range(3):
        eng.run_raw(HG_WANT_TALLY | HG_WANT_TIMELINE)
        k, t, *_ = eng.timing()
        if i:
            p1.append(k)
            tlm.append(eng.timeline_ms())
    st = eng.stats()
    rep = build_report(eng._flat, eng.tally_rows(), eng.device_names(), infos,
                       [(r.hostname, r.pid, r.tid) for r in raws], eng.stream_spans())
    tl = eng.timeline_bytes()
    msgs = st["host_spans"] + st["truncated_spans"] + st["device_spans"] + st["samples"]
    n_obj = tl.count(b"\n {\n  \"name\": ")
    n_meta = tl.count(b"\"ph\": \"M\"")
    want, _ = oracle_check(raws, wl.registry, threads)
    ok = tl[:3] == b"[\n " and tl[-2:] == b"\n]" and n_obj - n_meta == msgs and rep == want.report and \
        st == want.stats
    ph1, ms = statistics.mean(p1), statistics.mean(tlm)
    peak, _ = _peaks()
    gbs = (in_bytes + len(tl)) / ((ph1 + ms) / 1e3) / 1e9
    return {"workload": f"{config} x{scale}: SURVEY.md §8(d) C5 (device-profiling heavy) + full timeline export",
            "events": st["events_in"], "messages": msgs, "trace_bytes": in_bytes, "json_bytes": len(tl),
            "phase1_ms": ph1, "timeline_ms": ms, "json_gb_per_s": len(tl) / ms / 1e6,
            "events_per_s": st["events_in"] / ((ph1 + ms) / 1e3),
            "roofline": {"bytes": in_bytes + len(tl), "achieved_gb_per_s": gbs, "frac": gbs / peak},
            "parity": "exact" if ok else "MISMATCH",
            "path": ("single pass (fast_kernel<kTL>: per-range message lists)" if eng.last_path()[0] == 1 else
                     "exact three-kernel phase 1 (record-indexed messages)") +
                    " + k-way merge of the per-stream runs by mux key + JSON formatting",
            "checks": "object count = messages + metadata, json.dump framing, tally + IntervalStats == CPU oracle"}


def configs_side(eng, threads, plan=(("c1", 1.0), ("c3", 0.1), ("c4", 1.0), ("c5", 1.0))):
    """The other SURVEY.md §8(d) shapes (tally, device-resident, single pass unless it falls back):
    phase-1 device time and events/s at a bounded scale each, and the tally + IntervalStats of the
    last run against the CPU oracle over the same streams."""
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.abi import HG_WANT_TALLY
    from paper_2504_03683_b200.results import build_report

    out = []
    for name, scale in plan:
        wl = synth.config(name, scale)
        raws = synth.generate(wl)
        eng.set_registry(wl.registry)
        eng.set_streams(raws)
        eng.stage()
        ms = []
        for i in range(4):
            eng.run_raw(HG_WANT_TALLY)
            k, t, *_ = eng.timing()
            if i:
                ms.append(t)
        st = eng.stats()
        path, fallbacks, rb = eng.last_path()
        rep = build_report(eng._flat, eng.tally_rows(), eng.device_names(), [r.info for r in raws],
                           [(r.hostname, r.pid, r.tid) for r in raws], eng.stream_spans())
        want, _ = oracle_check(raws, wl.registry, threads)
        d = statistics.mean(ms)
        nb = sum(len(r.data) for r in raws)
        out.append({"config": name, "scale": scale, "events": st["events_in"], "streams": len(raws),
                    "bytes": nb, "device_ms": d, "events_per_s": st["events_in"] / (d / 1e3),
                    "roofline_frac": nb / (d / 1e3) / 1e9 / _peaks()[0],
                    "path": "single pass" if path == 1 else "exact", "range_bytes": rb,
                    "parity": _parity_line(rep, st, want.report, want.stats)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="workload (default: c2 at N=1, c3 sharded at N>1)")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 collectives (gloo: several ranks on one GPU, for tests)")
    ap.add_argument("--no-timeline", action="store_true", help="skip the row-a8 timeline side measurement")
    ap.add_argument("--no-dropin", action="store_true", help="skip the run_pipeline-from-files measurement")
    ap.add_argument("--no-configs", action="store_true", help="skip the other-configuration side measurements")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torchrun (the driver does the same)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), *sys.argv]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
