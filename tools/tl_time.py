"""Time the GPU timeline (ordering + JSON formatting) on a synthetic workload.

    python tools/tl_time.py [config] [scale]

Prints tally-only and tally+timeline device times, the timeline's own device
time and size, plus size-independent checks of the JSON (element count equals
the interval-stage messages + metadata objects; bracket framing)."""

import sys
import time

sys.path.insert(0, ".")

from paper_2504_03683_b200 import synth  # noqa: E402
from paper_2504_03683_b200.engine import Engine  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    wl = synth.config(name, scale)
    t = time.time()
    raws = synth.generate(wl)
    print(f"generated {name} x{scale}: {sum(len(r.data) for r in raws) / 1e9:.2f} GB in {time.time() - t:.1f}s")
    eng = Engine(0)
    infos = [r.info for r in raws]
    for _ in range(2):
        r0 = eng.run(raws, wl.registry, infos)
    print(f"tally only: tile kernel {r0.kernel_ms:.2f} ms, run {r0.total_ms:.2f} ms")
    for _ in range(2):
        t = time.time()
        r1 = eng.run(raws, wl.registry, infos, want_timeline=True)
        wall = time.time() - t
    ms = eng.timeline_ms()
    tl = r1.timeline
    st = r1.stats
    msgs = st["host_spans"] + st["truncated_spans"] + st["device_spans"] + st["samples"]
    n_obj = tl.count(b"\n {\n  \"name\": ")
    n_meta = tl.count(b"\"ph\": \"M\"")
    print(f"tally+timeline: tile kernel {r1.kernel_ms:.2f} ms, run {r1.total_ms:.2f} ms, timeline {ms:.2f} ms "
          f"(device), {len(tl) / 1e9:.3f} GB -> {len(tl) / ms / 1e6:.1f} GB/s of JSON, {msgs / ms / 1e6:.1f} M msgs/ms... "
          f"wall {wall:.1f}s")
    assert tl[:3] == b"[\n " and tl[-2:] == b"\n]", (tl[:10], tl[-10:])
    assert n_obj - n_meta == msgs, (n_obj, n_meta, msgs)
    assert r1.report == r0.report
    print(f"checks ok: {n_obj} objects = {msgs} messages + {n_meta} metadata")


if __name__ == "__main__":
    main()
