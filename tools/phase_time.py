"""Phase-1 kernel times (segment walk / chain / decode) on a synthetic workload.

    python tools/phase_time.py [config] [scale] [seg_bytes]"""

import sys

sys.path.insert(0, ".")

from paper_2504_03683_b200 import synth  # noqa: E402
from paper_2504_03683_b200.abi import HG_WANT_TALLY  # noqa: E402
from paper_2504_03683_b200.engine import Engine  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    seg = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    wl = synth.config(name, scale)
    raws = synth.generate(wl)
    nbytes = sum(len(r.data) for r in raws)
    eng = Engine(0, seg_bytes=seg) if seg else Engine(0)
    eng.set_registry(wl.registry)
    eng.set_streams(raws)
    eng.stage()
    for i in range(4):
        eng.run_raw(HG_WANT_TALLY)
        k, t, *_ = eng.timing()
        w, c, d = eng.phase_timing()
        ev = eng.stats()["events_in"]
        print(f"{name} x{scale} seg={seg or 'default'}: phase1 {k:.3f} ms (walk {w:.3f}, chain {c:.3f}, decode {d:.3f}) "
              f"{ev / k / 1e6:.0f} M ev/s, {nbytes / k / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
