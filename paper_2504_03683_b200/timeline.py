"""Timeline (Chrome trace event JSON) constants and the reference object model.

The GPU engine formats the JSON bytes itself (csrc/timeline.cu); this module
holds the track tables (sinks.py:309-328) and `TimelineBuilder`, a restatement
of TimelineSink's per-span object construction (sinks.py:341-418) that the
test oracle uses to produce reference-identical bytes via json.dump.
"""

from __future__ import annotations

import json

from .errors import HapitraceError

DEVICE_TRACK_PID_BASE = 9_000_000

COUNTER_TRACKS = {
    ("power", 0): "Power|Domain 0",
    ("power", 1): "Power|Domain 1",
    ("power", 2): "Power|Domain 2",
    ("frequency", 0): "GPU Frequency|Domain 0",
    ("frequency", 1): "GPU Frequency|Domain 1",
    ("compute_engine", 0): "Compute Engine|Tile 0",
    ("compute_engine", 1): "Compute Engine|Tile 1",
    ("copy_engine", 0): "Copy Engine|Tile 0",
    ("copy_engine", 1): "Copy Engine|Tile 1",
}

DEVICE_TRACK_NAMES = {
    (0, 0): "Tile 0 Compute",
    (0, 1): "Tile 0 Copy",
    (1, 0): "Tile 1 Compute",
    (1, 1): "Tile 1 Copy",
}

TIMELINE_REQUIRED_KEYS = ("name", "ph", "ts", "pid", "tid")


def check_timeline_object(obj: dict) -> bool:
    if any(k not in obj for k in TIMELINE_REQUIRED_KEYS):
        return False
    if obj["ph"] == "C" and "args" not in obj:
        return False
    if obj["ph"] == "X" and "dur" not in obj:
        return False
    return True


class TimelineBuilder:
    """Object list in emission order, as TimelineSink.on_message builds it."""

    def __init__(self, device_index: int = 0):
        self.device_pid = DEVICE_TRACK_PID_BASE + device_index
        self.objects = []
        self._seen = set()

    def _meta(self, pid, tid, name, kind):
        key = (pid, tid, kind)
        if key in self._seen:
            return
        self._seen.add(key)
        self.objects.append({"name": kind, "ph": "M", "ts": 0, "pid": pid, "tid": tid, "args": {"name": name}})

    def host_span(self, name, hostname, pid, tid, start, end, result, truncated):
        self._meta(pid, 0, f"Host {hostname} pid {pid}", "process_name")
        args = {"result": result}
        if truncated:
            args["truncated"] = True
        self.objects.append({"name": name, "ph": "X", "ts": start / 1000.0, "dur": (end - start) / 1000.0,
                             "pid": pid, "tid": tid, "args": args})

    def device_span(self, name, start, end, tile, engine, command_kind):
        tid = tile * 2 + engine
        self._meta(self.device_pid, 0, "Device 0", "process_name")
        self._meta(self.device_pid, tid, DEVICE_TRACK_NAMES.get((tile, engine), "Device"), "thread_name")
        self.objects.append({"name": name, "ph": "X", "ts": start / 1000.0, "dur": (end - start) / 1000.0,
                             "pid": self.device_pid, "tid": tid, "args": {"kind": command_kind}})

    def sample(self, counter, domain, ts, value, device):
        track = COUNTER_TRACKS.get((counter, domain))
        if track is None:
            raise HapitraceError(f"no timeline track for counter {counter}|{domain}")
        self.objects.append({"name": track, "ph": "C", "ts": ts / 1000.0, "pid": DEVICE_TRACK_PID_BASE + device,
                             "tid": 0, "args": {"value": value}})

    def dumps(self) -> str:
        return json.dumps(self.objects, indent=1)
