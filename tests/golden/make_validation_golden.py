"""Pin ValidationSink to the reference.

Writes, from the reference itself (importable in the build container only):
  traces/val_w1_<tag>/            w1 traced with one defect injected (test_acceptance.py:214-231)
  expected/validation_rules.json  ValidationRules.from_model(bundled_model(), bundled_registry())
  expected/validation_index.json  per golden trace of the bundled registry: the reference's
                                  ValidationSink(bundled_model()) findings, or the exception

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_validation_golden.py
"""

from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

from hapitrace import harness as ref_harness  # noqa: E402
from hapitrace.pipeline import run_pipeline  # noqa: E402
from hapitrace.sinks import ValidationSink  # noqa: E402
from hapitrace.tracefile import open_trace_reader  # noqa: E402

from paper_2504_03683_b200.registry import SchemaRegistry  # noqa: E402
from paper_2504_03683_b200.validation import ValidationRules  # noqa: E402


def main():
    model = ref_harness.bundled_model()
    reg = ref_harness.bundled_registry()
    for tag in ("uninit_pnext", "leak_event", "no_reset_cmdlist"):
        d = HERE / "traces" / f"val_w1_{tag}"
        shutil.rmtree(d, ignore_errors=True)
        ref_harness.trace_workload(ref_harness.bundled_workload("w1"), d, mode="full", inject=(tag,),
                                   hostname="goldenhost")
    ours = SchemaRegistry.from_dict(reg.to_dict())
    rules = ValidationRules.from_model(model, ours)
    (HERE / "expected" / "validation_rules.json").write_text(json.dumps(rules.to_dict(), indent=1) + "\n")
    out = {}
    for d in sorted((HERE / "traces").iterdir()):
        if not (d / "metadata.json").exists():
            continue
        meta = json.loads((d / "metadata.json").read_text())
        if meta.get("registry", {}).get("fingerprint") != reg.fingerprint:
            continue
        try:
            found = run_pipeline(open_trace_reader(d), [ValidationSink(model)])["validate"]
        except Exception as e:  # noqa: BLE001
            out[d.name] = {"raises": type(e).__name__, "str": str(e)}
            continue
        out[d.name] = {"findings": [[f.rule, f.subject, f.stream, f.timestamp_ns, f.message] for f in found]}
    (HERE / "expected" / "validation_index.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print({k: (len(v["findings"]) if "findings" in v else v["raises"]) for k, v in out.items()})


if __name__ == "__main__":
    main()
