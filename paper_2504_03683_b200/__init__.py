"""hapigpu -- B200-native trace post-processing (decode -> pair -> tally/timeline).

Drop-in for the analysis path of the reference `hapitrace` package (THAPI
re-created, /root/reference/pkg): same `run_pipeline` / `TallySink` /
`TimelineSink` / `tally_trace` / `merge_tallies` API, with the per-event work
done by hand-written sm_100a CUDA kernels in libhapigpu.so (csrc/engine.cu).
"""

from .errors import (  # noqa: F401
    CorruptRecordError, EngineError, FingerprintMismatchError, HapitraceError, MuxOrderingError, PipelineError,
    TraceDirectoryError, TraceError, UnknownSchemaError, UnsupportedTraceError,
)
from .pipeline import (  # noqa: F401
    END_OF_STREAM, IntervalStats, Message, PipelineResult, PrettyPrintSink, Sink, Span, TallySink, TimelineSink,
    run_pipeline,
)
from .registry import EventSchema, FieldSpec, SchemaRegistry  # noqa: F401
from .tally import TallyReport, TallyRow, empty_report, fmt_duration, merge_tallies, render_tally  # noqa: F401
from .timeline import check_timeline_object  # noqa: F401
from .tracefile import EventRecord, StreamInfo, TraceReader, open_trace_reader  # noqa: F401
from .harness import read_tally_json, tally_trace, write_tally_json  # noqa: F401
from .validation import ValidationFinding, ValidationRules, ValidationSink, render_findings  # noqa: F401

__version__ = "0.1.0"
