"""fast_kernel time vs single-pass range size (hg_set_option HG_OPT_RANGE_BYTES) on one workload.

    python tools/range_sweep.py [config] [scale] [range bytes ...]"""

import sys

sys.path.insert(0, ".")

from paper_2504_03683_b200 import synth  # noqa: E402
from paper_2504_03683_b200.abi import HG_WANT_TALLY  # noqa: E402
from paper_2504_03683_b200.engine import OPT_RANGE_BYTES, Engine  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    sizes = [int(x) for x in sys.argv[3:]] or [0]
    wl = synth.config(name, scale)
    raws = synth.generate(wl)
    eng = Engine(0)
    eng.set_registry(wl.registry)
    eng.set_streams(raws)
    for rb in sizes:
        eng.set_option(OPT_RANGE_BYTES, rb)
        eng.stage()
        ts = []
        for i in range(5):
            eng.run_raw(HG_WANT_TALLY)
            k, t, *_ = eng.timing()
            if i:
                ts.append((k, t))
        path, fb, used = eng.last_path()
        print(f"{name} x{scale} range {used} B (asked {rb}): fast {min(k for k, _ in ts):.3f} ms, "
              f"run {min(t for _, t in ts):.3f} ms, path {path}")


if __name__ == "__main__":
    main()
