"""Benchmark: events/s for decode+pair+tally on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2] [--scale 1.0]

A "step" is one pass of the hot path (decode -> pair -> tally, SURVEY.md §8a
rows a2-a5) over one synthetic trace of the named configuration; at N=1 the
workload is config C2 (100M events, 4 procs x 64 threads = 256 streams,
bundled ze registry).  Under torchrun every rank processes its own C2-sized
trace (weak scaling: distinct pids per rank) and the ranks exchange the global
last timestamp and merge tallies over NCCL.

Rank 0 prints ONE JSON line.  `value` = whole-job events / max-over-ranks
device time per step with the trace resident in HBM (CUDA events on the
engine's stream); `e2e` = the same metric through the public API with the
trace in pinned host memory, H2D and result D2H inside the timed region.
`--impl reference` times the CPU oracle (C restatement of the reference path,
oracle/hapi_oracle.c) with all host cores on a bounded sample.
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


def make_workload(name, scale, rank):
    from paper_2504_03683_b200 import synth

    wl = synth.config(name, scale)
    if rank:  # weak scaling: every rank owns a distinct set of processes
        for s in wl.streams:
            s.pid += 1_000_000 * rank
            s.tid += 1_000_000 * rank
            s.seed += 7_919 * rank
    return wl


def cpu_baseline(raws, registry, target_s=10.0):
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
    want_events = min(total, int(rate * target_s))
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
    wl = make_workload(args.config, args.scale, 0)
    from paper_2504_03683_b200 import synth

    raws = synth.generate(wl)
    total = sum(r.info.event_count for r in raws)
    times = []
    base = None
    for i in range(args.warmup + args.steps):
        b = cpu_baseline(raws, wl.registry, target_s=args.ref_seconds)
        if i >= args.warmup:
            times.append(b["value"])
            base = b
    value = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.config} x{args.scale}", "events": total},
        "cpu_baseline": {**base, "value": value},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args):
    import torch

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.distributed import ShardedRun
    from paper_2504_03683_b200.engine import Engine

    t0 = time.perf_counter()
    wl = make_workload(args.config, args.scale, rank)
    raws = synth.generate(wl)
    gen_s = time.perf_counter() - t0
    n_events = sum(r.info.event_count for r in raws)
    n_bytes = sum(len(r.data) for r in raws)
    infos = [r.info for r in raws]

    eng = Engine(device=local if ws > 1 else 0)
    runner = ShardedRun(eng, wl.registry, world_size=ws, rank=rank)

    # ---- device-resident timing (value)
    eng.set_registry(wl.registry)
    eng.set_streams(raws)
    eng.stage()
    for _ in range(args.warmup):
        runner.step()
    step_ms, dec_ms, ph1_ms, walk_ms, launches = [], [], [], [], 0
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    with clk:
        for _ in range(args.steps):
            info = runner.step()
            step_ms.append(info["device_ms"])
            dec_ms.append(info["decode_ms"])
            ph1_ms.append(info["phase1_ms"])
            walk_ms.append(info["walk_ms"])
            launches += info["launches"]
    torch.cuda.synchronize()
    ms = statistics.mean(step_ms)
    tms = statistics.mean(dec_ms)
    p1 = statistics.mean(ph1_ms)
    wms = statistics.mean(walk_ms)
    tot_events = n_events
    if ws > 1:
        t = torch.tensor([ms, tms, p1, wms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, tms, p1, wms = t.tolist()
        e = torch.tensor([n_events, n_bytes], dtype=torch.int64, device="cuda")
        torch.distributed.all_reduce(e)
        tot_events, tot_bytes = e.tolist()
    else:
        tot_bytes = n_bytes
    value = tot_events / (ms / 1e3)

    # correctness of the timed path against the oracle on rank 0's first streams (cheap check)
    rep = runner.report(infos)

    # ---- end-to-end through the public API from pinned host memory (e2e)
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
        rep2 = runner.report(infos)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            e2e_s.append(dt)
            h2d, d2h = info["h2d_bytes"], info["d2h_bytes"]
    e2e = statistics.mean(e2e_s)
    if ws > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = t.item()
    assert rep2 == rep, "e2e run produced a different tally"

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    peak, peak_src = _peaks()
    path, fallbacks, range_bytes = eng.last_path()
    single = path == 1
    achieved = (n_bytes / (tms / 1e3)) / 1e9  # per GPU: rank-local trace bytes over the decode kernel time
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "events/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic",
        "config": {
            "workload": f"{args.config}: SURVEY.md §8(d) C2 = 100M-event synthetic L0-style trace, 4 procs x 64 "
                        f"threads (256 streams), bundled ze registry" if args.config == "c2" else args.config,
            "scale": args.scale,
            "events_per_gpu": n_events,
            "bytes_per_gpu": n_bytes,
            "bytes_per_event": n_bytes / max(n_events, 1),
            "total_events": tot_events,
            "parallelism": f"streams per rank, {ws} rank(s); NCCL all-reduce of last ts + tally merge" if ws > 1
            else "1 GPU",
            "l2": "input (GBs) >> 126 MB L2: no flush needed between steps",
            "generation_s": round(gen_s, 2),
        },
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": None,
            "kernel": "fast_kernel" if single else "seg_decode_kernel",
            "kernel_ms": tms,
            "algorithmic_bytes_per_launch": n_bytes,
            "peak_source": peak_src,
            "phase1": {"kernels": ("fast_kernel + fast_verify_kernel + fast_orphan_fix_kernel" if single
                                   else "seg_walk_kernel + seg_chain_kernel + seg_decode_kernel"),
                       "path": "single pass over HBM (csrc/fast.cuh)" if single else "exact three-kernel path",
                       "range_bytes": range_bytes, "fallbacks": fallbacks, "ms": p1,
                       "walk_ms": wms, "achieved": (n_bytes / (p1 / 1e3)) / 1e9,
                       "frac": (n_bytes / (p1 / 1e3)) / 1e9 / peak},
        },
        "cpu_baseline": cpu_baseline(raws, wl.registry, target_s=args.ref_seconds),
        "e2e": {"value": tot_events / e2e, "unit": "events/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "path": "Engine.run via pinned host streams (public API)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_timeline:
        line["timeline"] = timeline_side(eng)
    if not args.no_configs:
        line["other_configs"] = configs_side(eng)
    traffic = REPO / "profiles" / ("fast_kernel_traffic.json" if single else "seg_decode_traffic.json")
    if traffic.exists():
        tr = json.loads(traffic.read_text())
        line["roofline"]["traffic"] = tr.get("dram_bytes_per_launch")
        line["roofline"]["traffic_source"] = tr.get("source")
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def timeline_side(eng, config="c5", scale=0.1):
    """Row a8 (TimelineSink): tally + timeline on the device-heavy config, device time of the ordering and
    JSON formatting, with size-independent checks (object count = interval messages + metadata objects,
    json.dump framing, tally equal to the tally-only run)."""
    from paper_2504_03683_b200 import synth

    wl = synth.config(config, scale)
    raws = synth.generate(wl)
    infos = [r.info for r in raws]
    r0 = eng.run(raws, wl.registry, infos)
    r1 = None
    for _ in range(2):
        r1 = eng.run(raws, wl.registry, infos, want_timeline=True)
    ms = eng.timeline_ms()
    tl, st = r1.timeline, r1.stats
    msgs = st["host_spans"] + st["truncated_spans"] + st["device_spans"] + st["samples"]
    n_obj = tl.count(b"\n {\n  \"name\": ")
    n_meta = tl.count(b"\"ph\": \"M\"")
    assert tl[:3] == b"[\n " and tl[-2:] == b"\n]" and n_obj - n_meta == msgs and r1.report == r0.report
    return {"workload": f"{config} x{scale}: SURVEY.md §8(d) C5 (device-profiling heavy) + full timeline export",
            "events": st["events_in"], "messages": msgs, "json_bytes": len(tl),
            "phase1_ms": r1.kernel_ms, "timeline_ms": ms, "json_gb_per_s": len(tl) / ms / 1e6,
            "events_per_s": st["events_in"] / ((r1.kernel_ms + ms) / 1e3),
            "path": "exact three-kernel phase 1 (record-indexed messages) + k-way merge of the per-stream runs by mux key + JSON formatting",
            "checks": "object count = messages + metadata, json.dump framing, tally == tally-only run"}


def configs_side(eng, plan=(("c1", 1.0), ("c3", 0.1), ("c4", 0.25), ("c5", 0.25))):
    """The other SURVEY.md §8(d) shapes (tally, device-resident, single pass unless it falls back):
    phase-1 device time and events/s at a bounded scale each (parity for them is in tests/)."""
    from paper_2504_03683_b200 import synth
    from paper_2504_03683_b200.abi import HG_WANT_TALLY

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
        ev = eng.stats()["events_in"]
        path, fallbacks, rb = eng.last_path()
        d = statistics.mean(ms)
        out.append({"config": name, "scale": scale, "events": ev, "streams": len(raws),
                    "bytes": sum(len(r.data) for r in raws), "device_ms": d, "events_per_s": ev / (d / 1e3),
                    "path": "single pass" if path == 1 else "exact", "range_bytes": rb})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-timeline", action="store_true", help="skip the row-a8 timeline side measurement")
    ap.add_argument("--no-configs", action="store_true", help="skip the other-configuration side measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
