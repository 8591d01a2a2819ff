"""Time the GPU event path (mux order of every record + PrettyPrintSink lines) on a synthetic workload.

    python tools/ev_time.py [config] [scale]"""

import sys

sys.path.insert(0, ".")

from paper_2504_03683_b200 import synth  # noqa: E402
from paper_2504_03683_b200.abi import HG_WANT_EVENTS, HG_WANT_TALLY  # noqa: E402
from paper_2504_03683_b200.engine import Engine  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
    wl = synth.config(name, scale)
    raws = synth.generate(wl)
    eng = Engine(0)
    eng.set_registry(wl.registry)  # (schema names for the event lines too)
    eng.set_streams(raws)
    eng.stage()
    for _ in range(3):
        eng.run_raw(HG_WANT_TALLY | HG_WANT_EVENTS)
        k, t, *_ = eng.timing()
        print(f"{name} x{scale}: phase1 {k:.2f} ms, run {t:.2f} ms, events {eng.events_ms():.2f} ms, "
              f"path {eng.last_path()[0]}")


if __name__ == "__main__":
    main()
