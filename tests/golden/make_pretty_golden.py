"""Pin PrettyPrintSink to the reference: for every golden trace directory,
run the reference's own run_pipeline(open_trace_reader(d), [PrettyPrintSink()]) and record the
text's length and sha256 (or the exception it raises) in tests/golden/expected/pretty_index.json.

Run in the build container (the reference is importable there, not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pretty_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from hapitrace.pipeline import run_pipeline  # noqa: E402
from hapitrace.sinks import PrettyPrintSink  # noqa: E402
from hapitrace.tracefile import open_trace_reader  # noqa: E402


def main():
    out = {}
    for d in sorted((HERE / "traces").iterdir()):
        if not (d / "metadata.json").exists():
            continue
        try:
            text = run_pipeline(open_trace_reader(d), [PrettyPrintSink()])["pretty"]
        except Exception as e:  # noqa: BLE001
            out[d.name] = {"raises": type(e).__name__, "str": str(e)}
            continue
        b = text.encode("utf-8")
        out[d.name] = {"bytes": len(b), "lines": text.count("\n"), "sha256": hashlib.sha256(b).hexdigest(),
                       "head": text[:2000]}
    (HERE / "expected" / "pretty_index.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"{len(out)} traces")


if __name__ == "__main__":
    main()
