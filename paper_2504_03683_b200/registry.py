"""Schema registry: the decode contract embedded in every trace's metadata.json.

Mirrors the read side of the reference registry
(`/root/reference/pkg/src/hapitrace/registry.py:23-129`): field kinds, event
classes, the dict wire form and the telemetry counter naming.  Registry
*generation* from API models is out of scope; traces carry
their registry, and `from_dict` rebuilds it.

`flatten()` turns a registry into the fixed-width tables the native engine
consumes (`include/hapigpu.h`, `hg_schema`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import HapitraceError, RegistryError

FIELD_KINDS = ("u64", "i64", "f64", "address", "string", "blob")
EVENT_CLASSES = ("host_entry", "host_exit", "device_profiling", "telemetry_sample", "meta")

# registry.py:30-40 -- (counter key, timeline track)
TELEMETRY_COUNTERS = (
    ("power_domain_0", "Power|Domain 0"),
    ("power_domain_1", "Power|Domain 1"),
    ("power_domain_2", "Power|Domain 2"),
    ("frequency_domain_0", "GPU Frequency|Domain 0"),
    ("frequency_domain_1", "GPU Frequency|Domain 1"),
    ("compute_tile_0", "Compute Engine|Tile 0"),
    ("compute_tile_1", "Compute Engine|Tile 1"),
    ("copy_tile_0", "Copy Engine|Tile 0"),
    ("copy_tile_1", "Copy Engine|Tile 1"),
)

# native codes (include/hapigpu.h)
KIND_CODE = {"u64": 0, "i64": 1, "f64": 2, "address": 3, "string": 4, "blob": 5}
CLASS_CODE = {"host_entry": 0, "host_exit": 1, "device_profiling": 2, "telemetry_sample": 3, "meta": 4}
COUNTER_KINDS = ("power", "frequency", "compute_engine", "copy_engine")


@dataclass(frozen=True)
class FieldSpec:
    name: str
    kind: str
    origin: str


@dataclass(frozen=True)
class EventSchema:
    id: int
    name: str
    event_class: str
    fields: tuple
    mode_mask: frozenset
    function: str | None = None

    def field_names(self) -> tuple:
        return tuple(f.name for f in self.fields)


@dataclass(frozen=True)
class SchemaRegistry:
    api_name: str
    fingerprint: str
    schemas: tuple
    by_id: dict = field(default_factory=dict, compare=False, repr=False)
    by_name: dict = field(default_factory=dict, compare=False, repr=False)

    def __post_init__(self):
        for s in self.schemas:  # later duplicates win, as dict(...) does in the reference
            self.by_id[s.id] = s
            self.by_name[s.name] = s

    def schema(self, name: str) -> EventSchema:
        try:
            return self.by_name[name]
        except KeyError:
            raise RegistryError(f"no schema named {name!r}") from None

    def to_dict(self) -> dict:
        return {
            "api_name": self.api_name,
            "fingerprint": self.fingerprint,
            "schemas": [
                {
                    "id": s.id,
                    "name": s.name,
                    "class": s.event_class,
                    "function": s.function,
                    "mode_mask": sorted(s.mode_mask),
                    "fields": [{"name": f.name, "kind": f.kind, "origin": f.origin} for f in s.fields],
                }
                for s in self.schemas
            ],
        }

    @classmethod
    def from_dict(cls, doc: dict) -> "SchemaRegistry":
        schemas = []
        for s in doc["schemas"]:
            fields = tuple(FieldSpec(f["name"], f["kind"], f["origin"]) for f in s["fields"])
            schemas.append(
                EventSchema(
                    id=int(s["id"]),
                    name=s["name"],
                    event_class=s["class"],
                    fields=fields,
                    mode_mask=frozenset(s["mode_mask"]),
                    function=s.get("function"),
                )
            )
        return cls(api_name=doc["api_name"], fingerprint=doc["fingerprint"], schemas=tuple(schemas))


def parse_counter_key(schema_name: str):
    """Telemetry schema name -> (counter kind, domain); sampler.py:51-64 semantics.

    Raises ValueError (non-integer suffix) or HapitraceError (unknown prefix)
    exactly where the reference does.
    """
    tail = schema_name.rsplit("telemetry_", 1)[-1]
    prefix, _, idx = tail.rpartition("_")
    domain = int(idx)
    kind = {
        "power_domain": "power",
        "frequency_domain": "frequency",
        "compute_tile": "compute_engine",
        "copy_tile": "copy_engine",
    }.get(prefix)
    if kind is None:
        raise HapitraceError(f"not a telemetry schema: {schema_name!r}")
    return kind, domain
