"""ValidationSink served by the GPU engine (reference sinks.py:435-605).

The reference checks four post-mortem rules over the raw events in mux order:
  uninit_pnext       a property-query entry whose struct blob leads with a non-NULL pNext
  cmdlist_not_reset  a command list executed again without a reset in between
  leaked_event       a handle created (result 0) and never released
  orphan_exit        forwarded from the interval stage (on_diagnostics)
Its rule tables come from the API model (ValidationSink.on_start, sinks.py:461-516).  Here they are
`ValidationRules` -- built from the reference's model object (duck-typed, a literal restatement of
on_start) or loaded from their JSON form -- and the per-event work runs on the GPU (csrc/validate.cu):
per record classification in mux order, the "last entry of this function on this stream" lookups
(pending_entries, sinks.py:526-527) as a sort + segmented max-scan, and the per-handle state machines
(live handles, executed command lists) as sorts by (handle, mux position) with neighbour tests.
The host only formats the few findings.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass, field

from .errors import FingerprintMismatchError, UnsupportedTraceError


@dataclass(frozen=True)
class ValidationFinding:
    rule: str  # uninit_pnext | leaked_event | cmdlist_not_reset | orphan_exit
    subject: int  # offending handle or address value
    stream: str
    timestamp_ns: int
    message: str


@dataclass
class ValidationRules:
    """The rule tables of ValidationSink.on_start (sinks.py:461-516), keyed by schema id."""

    fingerprint: str
    pnext: dict = field(default_factory=dict)      # entry sid -> (function name, blob field name)
    creators: dict = field(default_factory=dict)   # exit sid -> (function name, out field name)
    releasers: dict = field(default_factory=dict)  # exit sid -> (function name, entry sid, handle param)
    execute: dict = field(default_factory=dict)    # entry sid -> handle param
    resets: dict = field(default_factory=dict)     # exit sid -> (entry sid, handle param)

    @classmethod
    def from_model(cls, model, registry) -> "ValidationRules":
        """Literal restatement of ValidationSink.on_start over the reference's ApiModel object."""
        mod = sys.modules.get(type(model).__module__)
        fp_fn = getattr(mod, "model_fingerprint", None)
        fp = fp_fn(model) if fp_fn is not None else getattr(model, "fingerprint", None)
        if registry.fingerprint != fp:
            raise FingerprintMismatchError("validator model does not match the trace registry")
        r = cls(fingerprint=fp)
        api = model.api_name
        for fn in model.functions:
            for p in fn.params:
                if p.deref is None or p.deref.kind != "blob":
                    continue
                base, _ = model.base_type(p.c_type)
                sd = model.struct_defs.get(base)
                if sd and sd.fields and sd.fields[0].name == "pNext":
                    entry = registry.schema(f"{api}:{fn.name}_entry")
                    r.pnext[entry.id] = (fn.name, f"{p.name}_vals")
        for fn in model.functions:
            if "creates_handle" in fn.attrs:
                ex = registry.schema(f"{api}:{fn.name}_exit")
                out_field = next((f.name for f in ex.fields if f.origin == "deref_out" and f.kind == "address"), None)
                if out_field:
                    r.creators[ex.id] = (fn.name, out_field)
            if "releases_handle" in fn.attrs:
                ex = registry.schema(f"{api}:{fn.name}_exit")
                handle_param = next((p.name for p in fn.params if p.is_handle), None)
                if handle_param:
                    en = registry.schema(f"{api}:{fn.name}_entry")
                    r.releasers[ex.id] = (fn.name, en.id, handle_param)
        for fn in model.functions:
            if "CommandList" not in fn.name:
                continue
            handle_param = next((p.name for p in fn.params if p.is_handle), None)
            if handle_param is None:
                continue
            ex = registry.schema(f"{api}:{fn.name}_exit")
            en = registry.schema(f"{api}:{fn.name}_entry")
            if fn.name.endswith("Execute"):
                r.execute[en.id] = handle_param
            elif fn.name.endswith("Reset"):
                r.resets[ex.id] = (en.id, handle_param)
        return r

    def to_dict(self) -> dict:
        return {"fingerprint": self.fingerprint,
                "pnext": {str(k): list(v) for k, v in self.pnext.items()},
                "creators": {str(k): list(v) for k, v in self.creators.items()},
                "releasers": {str(k): list(v) for k, v in self.releasers.items()},
                "execute": {str(k): v for k, v in self.execute.items()},
                "resets": {str(k): list(v) for k, v in self.resets.items()}}

    @classmethod
    def from_dict(cls, d) -> "ValidationRules":
        return cls(d["fingerprint"], {int(k): tuple(v) for k, v in d["pnext"].items()},
                   {int(k): tuple(v) for k, v in d["creators"].items()},
                   {int(k): tuple(v) for k, v in d["releasers"].items()},
                   {int(k): v for k, v in d["execute"].items()},
                   {int(k): tuple(v) for k, v in d["resets"].items()})


VK_PNEXT, VK_EXEC, VK_CREATE, VK_RELEASE, VK_RESET, VK_TRACK = 1, 2, 4, 8, 16, 32
_INT_KINDS = ("u64", "i64", "address")


def rule_rows(rules: ValidationRules, flat):
    """hg_validation_rule rows in the registry's flat order (csrc/validate.cu); refuses layouts whose
    reference behaviour the rows cannot express (UnsupportedTraceError, never a silent difference)."""
    from .abi import HgValidationRule

    by_id = flat.registry.by_id
    rel_fn = {fn: param for fn, _en, param in rules.releasers.values()}
    rst_fn = {}
    for ex_id, (_en, param) in rules.resets.items():
        rst_fn[by_id[ex_id].function] = param
    rows = []
    for h in flat.schemas:
        sc = by_id[h.id]
        idx = {}
        for i, f in enumerate(sc.fields):
            idx[f.name] = i  # payload dicts keep the last duplicate
        kinds = {f.name: f.kind for f in sc.fields}

        def fld(name, allowed):
            if name not in idx:
                return -1
            if kinds[name] not in allowed:
                raise UnsupportedTraceError(f"validation: field {sc.name}.{name} of kind {kinds[name]}")
            return idx[name]

        r = HgValidationRule(0, -1, -1, -1, -1, -1, -1)
        if sc.id in rules.pnext:
            r.pnext = fld(rules.pnext[sc.id][1], ("blob",))
            if r.pnext >= 0:
                r.kind |= VK_PNEXT
        if sc.event_class == "host_entry":
            if sc.id in rules.execute:
                r.exec = fld(rules.execute[sc.id], _INT_KINDS)
                if r.exec < 0:
                    raise UnsupportedTraceError(f"validation: {sc.name} lacks {rules.execute[sc.id]}")
                r.kind |= VK_EXEC
            for fnmap, attr in ((rel_fn, "rel"), (rst_fn, "rst")):
                if sc.function in fnmap:
                    i = fld(fnmap[sc.function], _INT_KINDS)
                    if i < 0:
                        raise UnsupportedTraceError(f"validation: {sc.name} lacks {fnmap[sc.function]}")
                    setattr(r, attr, i)
                    r.kind |= VK_TRACK
        elif sc.event_class == "host_exit":
            if "result" in idx:
                r.result = fld("result", ("u64", "i64"))
            if sc.id in rules.creators:
                r.create = fld(rules.creators[sc.id][1], _INT_KINDS)
                if r.create < 0:
                    raise UnsupportedTraceError(f"validation: {sc.name} lacks {rules.creators[sc.id][1]}")
                r.kind |= VK_CREATE
            elif sc.id in rules.releasers:
                if rules.releasers[sc.id][0] != sc.function:
                    raise UnsupportedTraceError(f"validation: releaser {sc.name} of another function")
                r.kind |= VK_RELEASE
            elif sc.id in rules.resets:
                r.kind |= VK_RESET
        rows.append(r)
    return rows


def findings_from_native(native, rules: ValidationRules, streams) -> list:
    """ValidationFinding objects in the reference's order: in-order findings (mux position), then the
    leaked handles sorted by subject (sinks.py:592-594)."""
    in_order, leaks = [], []
    for f in native:
        s = streams[f.stream]
        label = f"{s.hostname}/{s.pid}/{s.tid}"
        if f.rule == 1:
            pn = f.subject_lo
            in_order.append((f.pos, ValidationFinding("uninit_pnext", pn, label, f.ts,
                                                      f"{rules.pnext[f.sid][0]}: extension slot pNext is 0x{pn:x}, "
                                                      "must be NULL")))
            continue
        h = (f.subject_hi << 64) + f.subject_lo - (1 << 63)
        if f.rule == 2:
            in_order.append((f.pos, ValidationFinding("cmdlist_not_reset", h, label, f.ts,
                                                      f"command list 0x{h:x} executed again without a reset")))
        else:
            leaks.append(ValidationFinding("leaked_event", h, label, f.ts,
                                           f"handle 0x{h:x} from {rules.creators[f.sid][0]} never released"))
    in_order.sort(key=lambda x: x[0])
    return [x[1] for x in in_order] + sorted(leaks, key=lambda f: f.subject)


class ValidationSink:
    """Post-mortem rule checks (sinks.py:448-594); the events are examined by the GPU engine."""

    name = "validate"
    consumes = "events"

    def __init__(self, model=None, rules: ValidationRules | None = None):
        if model is None and rules is None:
            raise TypeError("ValidationSink needs the API model (or its ValidationRules)")
        self.model = model
        self.rules = rules
        self._findings: list = []
        self._orphans: list = []

    def on_start(self, registry):
        if self.rules is None:
            self.rules = ValidationRules.from_model(self.model, registry)
        elif registry.fingerprint != self.rules.fingerprint:
            raise FingerprintMismatchError("validator model does not match the trace registry")
        self.registry = registry

    def on_message(self, msg):
        raise UnsupportedTraceError("hapigpu's ValidationSink is fed by the GPU engine through run_pipeline")

    def _gpu_result(self, findings):
        self._findings = findings

    def on_diagnostics(self, orphans):
        self._orphans = [ValidationFinding("orphan_exit", 0, stream, ts, f"exit of {fn} without matching entry")
                         for stream, ts, fn in orphans]

    def on_finish(self) -> list:
        return self._findings + self._orphans


def render_findings(findings: list) -> str:
    """sinks.py:597-605."""
    if not findings:
        return "validation: clean, 0 findings\n"
    lines = [f"validation: {len(findings)} finding(s)"]
    for f in findings:
        lines.append(f"  [{f.rule}] {f.message} (stream {f.stream}, t={f.timestamp_ns})")
    return "\n".join(lines) + "\n"
