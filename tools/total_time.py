"""Whole-run device time (phase 1 + compose + result copies) of tally runs: python tools/total_time.py config scale"""
import sys

sys.path.insert(0, ".")
from paper_2504_03683_b200 import synth  # noqa: E402
from paper_2504_03683_b200.abi import HG_WANT_TALLY  # noqa: E402
from paper_2504_03683_b200.engine import Engine  # noqa: E402

name, scale = sys.argv[1], float(sys.argv[2])
wl = synth.config(name, scale)
raws = synth.generate(wl)
eng = Engine(0)
eng.set_registry(wl.registry)
eng.set_streams(raws)
eng.stage()
for i in range(4):
    eng.run_raw(HG_WANT_TALLY)
k, t, *_ = eng.timing()
print(f"{name} x{scale}: phase1 {k:.3f} ms, whole run {t:.3f} ms, path {eng.last_path()}")
