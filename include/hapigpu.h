/*
 * hapigpu.h -- C ABI of the B200 trace post-processing engine (libhapigpu.so).
 *
 * The reference (THAPI re-created as the Python package `hapitrace`) has no
 * FFI on this path: its boundary is the Python plugin API
 *   run_pipeline(source, sinks, registry)      pipeline.py:275-314
 *   TallySink / TallyReport                     sinks.py:113-248
 *   TimelineSink                                sinks.py:341-418
 *   merge_tallies                               aggregator.py:35-76
 * Each entry point below names the reference interface it replaces.  The
 * Python package `paper_2504_03683_b200` binds this header with ctypes and
 * re-exposes the reference API on top of it.
 *
 * Conventions: plain C types only; return 0 (HG_OK) on success, a negative
 * HG_E* code on an engine failure (text via hg_last_error), or HG_TRACE_ERROR
 * (> 0) when the trace itself is malformed -- the caller then reads the
 * per-stream error candidates (hg_get_trace_errors) and raises the same
 * exception the reference would (CorruptRecordError, UnknownSchemaError,
 * MuxOrderingError, HapitraceError ...).  One context per pipeline; a context
 * is not reentrant, distinct contexts may run concurrently.  The library owns
 * all device memory; output arrays are caller-allocated.
 */
#ifndef HAPIGPU_H
#define HAPIGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_ABI_VERSION 1

/* return codes */
#define HG_OK 0
#define HG_TRACE_ERROR 1
#define HG_EARG (-1)
#define HG_ESTATE (-2)
#define HG_ECUDA (-3)
#define HG_ENOMEM (-4)
#define HG_EUNSUPPORTED (-5)

/* field kinds (registry.py:23 FIELD_KINDS order) */
enum { HG_KIND_U64 = 0, HG_KIND_I64 = 1, HG_KIND_F64 = 2, HG_KIND_ADDRESS = 3, HG_KIND_STRING = 4, HG_KIND_BLOB = 5 };
/* event classes (registry.py:24 EVENT_CLASSES order) */
enum { HG_CLASS_ENTRY = 0, HG_CLASS_EXIT = 1, HG_CLASS_DEVICE = 2, HG_CLASS_TELEMETRY = 3, HG_CLASS_META = 4 };
/* field roles resolved by name on the host (pipeline.py:183, 192-214; sinks.py:381-395) */
enum {
  HG_ROLE_RESULT = 0,   /* host_exit "result"                  */
  HG_ROLE_START = 1,    /* device "device_start_ns"            */
  HG_ROLE_END = 2,      /* device "device_end_ns"              */
  HG_ROLE_NAME = 3,     /* device "name"                       */
  HG_ROLE_TILE = 4,     /* device "tile"                       */
  HG_ROLE_ENGINE = 5,   /* device "engine"                     */
  HG_ROLE_CMDKIND = 6,  /* device "command_kind"               */
  HG_ROLE_VALUE = 7,    /* telemetry "value"                   */
  HG_ROLE_DEVICE = 8,   /* telemetry "device"                  */
  HG_NUM_ROLES = 10
};
/* telemetry counter kinds (sampler.py:51-64) */
enum { HG_COUNTER_POWER = 0, HG_COUNTER_FREQUENCY = 1, HG_COUNTER_COMPUTE = 2, HG_COUNTER_COPY = 3 };

/* One schema of the registry, flattened (registry.py:61-71 EventSchema).
 * feed_error != 0: every event of this schema raises when it reaches the
 * interval stage (e.g. a telemetry schema whose name parse_counter_key
 * rejects); the host keeps the exception text, the engine reports where. */
typedef struct hg_schema {
  uint32_t id;             /* schema id as stored in records                 */
  uint8_t event_class;     /* HG_CLASS_*                                     */
  uint8_t n_fields;
  uint8_t counter_kind;    /* HG_COUNTER_* (telemetry only)                  */
  uint8_t feed_error;      /* 0 = none                                       */
  int32_t function;        /* function-name id (pairing/tally key), -1: None */
  int32_t counter_domain;  /* telemetry domain index                         */
  uint32_t kinds_offset;   /* first field kind in the kinds[] array          */
  int16_t role[HG_NUM_ROLES]; /* field index per HG_ROLE_*, -1 if absent     */
} hg_schema;

typedef struct hg_config {
  int32_t device;          /* CUDA device ordinal                            */
  uint32_t tile_bytes;     /* exact-path segment bytes (0 = sized to the trace) */
  uint32_t flags;          /* reserved                                       */
  int32_t timeline_device_index; /* TimelineSink(device_index=) (sinks.py:347-349) */
} hg_config;

typedef struct hg_stats {  /* IntervalStats (pipeline.py:117-129) */
  uint64_t events_in, passed, host_spans, truncated_spans, device_spans, samples, orphan_exits;
} hg_stats;

/* one tally row (TallyRow, sinks.py:113-136).  Sums and extrema are exact
 * signed 128-bit integers split into (lo, hi) words. */
typedef struct hg_tally_row {
  uint32_t section;        /* 0 host, 1 device                               */
  uint32_t name_id;        /* host: function id; device: device-name id      */
  uint64_t count, error_count;
  uint64_t time_lo; int64_t time_hi;
  uint64_t min_lo;  int64_t min_hi;
  uint64_t max_lo;  int64_t max_hi;
} hg_tally_row;

/* orphan exit diagnostic (pipeline.py:163-168), unordered; the host sorts
 * by (ts, stream, seq) = mux order. */
typedef struct hg_orphan {
  uint32_t stream;         /* stream index as added                          */
  int32_t function;
  uint64_t ts;
  uint64_t seq;            /* record index within the stream                 */
} hg_orphan;

/* trace error candidates: the first failing record of each stream
 * (pipeline.py:92-100, tracefile.py:198-215) and value-dependent
 * interval-stage errors (sampler.py:44-48).  The host picks the one the
 * reference's muxer would hit first and formats the exception. */
enum {
  HG_ERR_TRUNC_HEADER = 1,   /* CorruptRecordError "truncated record header"  */
  HG_ERR_TRUNC_PAYLOAD = 2,  /* CorruptRecordError "truncated record payload" */
  HG_ERR_UNKNOWN_SCHEMA = 3, /* UnknownSchemaError                            */
  HG_ERR_LEN_MISMATCH = 4,   /* CorruptRecordError "payload length mismatch"  */
  HG_ERR_TRUNC_VAR = 5,      /* CorruptRecordError "truncated variable field" */
  HG_ERR_TRAILING = 6,       /* CorruptRecordError "trailing payload bytes"   */
  HG_ERR_UTF8 = 7,           /* CorruptRecordError from UnicodeDecodeError    */
  HG_ERR_STRUCT = 8,         /* struct.error escaping _decode_one             */
  HG_ERR_ORDER = 9,          /* MuxOrderingError                              */
  HG_ERR_FEED = 10,          /* schema feed_error at this event               */
  HG_ERR_TELEMETRY = 11,     /* TelemetrySample range check                   */
  HG_ERR_RESULT = 12         /* int(result) of a NaN/inf f64 result           */
};
typedef struct hg_trace_error {
  uint32_t code;           /* HG_ERR_*                                       */
  uint32_t stream;
  uint64_t seq;            /* index of the failing record                    */
  uint64_t offset;         /* its byte offset in the stream file             */
  uint64_t ts;             /* its timestamp (if decodable)                   */
  uint64_t prev_ts;        /* timestamp of record seq-1 (pull position)      */
  uint64_t aux;            /* code-specific: schema id, utf-8 position ...   */
} hg_trace_error;

typedef struct hg_ctx hg_ctx;

/* create/destroy a pipeline context bound to one GPU
 * replaces: run_pipeline's per-call IntervalBuilder/sink set-up (pipeline.py:282-299) */
int hg_create(const hg_config* cfg, hg_ctx** out);
void hg_destroy(hg_ctx* ctx);
const char* hg_last_error(hg_ctx* ctx);
int hg_abi_version(void);

/* install the decode contract: TraceReader registry + _CodecTable
 * (tracefile.py:172-180, 530-531; registry.py:116-129) */
int hg_set_registry(hg_ctx* ctx, const hg_schema* schemas, uint32_t n_schemas,
                    const uint8_t* kinds, uint32_t n_kinds, uint32_t n_functions);

/* add one stream file (bytes incl. the 16-byte header, already validated by
 * the host) in (hostname, pid, tid) order; replaces StreamCursor
 * (tracefile.py:477-508).  `data` is a host pointer that must stay valid
 * until hg_run returns.  hostname NULL stands for None (record-list sources):
 * it orders as "" and prints as "None" in timeline metadata (sinks.py:367);
 * pid / tid INT64_MIN stand for None in pretty-printed lines. */
int hg_add_stream(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid,
                  const void* data, uint64_t size);
int hg_clear_streams(hg_ctx* ctx);

/* the same stream, its bytes already in DEVICE memory of this context's GPU (a torch
 * tensor's data_ptr, a GPUDirect-Storage buffer): staged with one HBM->HBM copy, no
 * PCIe.  Caller-owned until hg_run returns. */
int hg_add_stream_device(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid,
                         const void* device_ptr, uint64_t size);
/* the same stream, read by the engine from a FILE (bytes [offset, offset+size)); the
 * 16-byte file header must already be validated (tracefile.py:491-499 messages).
 * Replaces StreamCursor's whole-file read (tracefile.py:489): staging reads files and
 * pageable host buffers through per-thread double-buffered pinned chunks, so file
 * reads and PCIe transfers overlap; pinned host buffers go straight to DMA. */
int hg_add_stream_file(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid,
                       const char* path, uint64_t offset, uint64_t size);
/* how the last staging moved the bytes: per source kind, host wall ms of the whole
 * staging (file reads + copies), host threads used */
int hg_ingest_stats(hg_ctx* ctx, uint64_t* pinned_bytes, uint64_t* pageable_bytes, uint64_t* file_bytes,
                    uint64_t* device_bytes, float* ms, uint32_t* threads);

/* copy all added streams to HBM now; later runs reuse the resident copy
 * (used to time the device-resident path separately from ingest). */
int hg_stage(hg_ctx* ctx);

/* run decode -> pair -> tally (+ timeline) over all streams:
 * replaces run_pipeline(reader, [TallySink(), TimelineSink()]) (pipeline.py:275-314) */
#define HG_WANT_TALLY 1u
#define HG_WANT_TIMELINE 2u
#define HG_WANT_EVENTS 4u   /* every record in mux order + PrettyPrintSink's text (events.cu) */
#define HG_WANT_VALIDATE 8u /* ValidationSink's rules over the mux order (validate.cu) */
#define HG_WANT_TL_ITEMS 16u /* this rank's timeline messages, sorted, for hg_tl_export (tldist.cu) */
int hg_run(hg_ctx* ctx, uint32_t want);

/* split form for sharded (multi-GPU) runs: phase 1 over the local streams,
 * then the caller all-reduces the max timestamp (pipeline.py:152, :235) and
 * finishes with the global value. */
int hg_run_local(hg_ctx* ctx, uint32_t want);
int hg_local_last_ts(hg_ctx* ctx, uint64_t* last_ts, uint64_t* n_events);
int hg_finish(hg_ctx* ctx, uint64_t global_last_ts);
/* after hg_run_local: HG_FLAG_WIDE_DEVICE = some device span is beyond +-2^63 ns (its tally row keeps
 * 128-bit extrema; the multi-rank merge carries 64-bit extrema and refuses such runs) */
#define HG_FLAG_WIDE_DEVICE 1u
int hg_local_flags(hg_ctx* ctx, uint32_t* flags);

/* results */
int hg_get_stats(hg_ctx* ctx, hg_stats* out);                       /* IntervalStats */
int hg_get_tally(hg_ctx* ctx, hg_tally_row* rows, uint64_t cap, uint64_t* n_rows); /* TallySink.on_finish */
int hg_get_device_names(hg_ctx* ctx, char* bytes, uint64_t cap, uint64_t* offsets,
                        uint64_t n_offsets, uint64_t* n_names, uint64_t* n_bytes);
int hg_get_stream_spans(hg_ctx* ctx, uint64_t* per_stream, uint64_t n); /* span identities (sinks.py:240-242) */
int hg_get_orphans(hg_ctx* ctx, hg_orphan* out, uint64_t cap, uint64_t* n); /* IntervalBuilder.orphans */
int hg_get_trace_errors(hg_ctx* ctx, hg_trace_error* out, uint64_t cap, uint64_t* n);

/* function names (UTF-8, id = index, offsets[n] = end; is_null[i] != 0 for a
 * None name, may be NULL): the "name" of host-span timeline objects
 * (sinks.py:369, registry.py:61-71 EventSchema.function).  Required before a
 * run with HG_WANT_TIMELINE. */
int hg_set_function_names(hg_ctx* ctx, const char* bytes, const uint64_t* offsets, const uint8_t* is_null,
                          uint32_t n);

/* timeline: Chrome-trace JSON bytes exactly as json.dump(objs, fh, indent=1)
 * writes them (TimelineSink, sinks.py:341-418), built on the GPU by the run
 * that had HG_WANT_TIMELINE (and no trace error). */
int hg_timeline_size(hg_ctx* ctx, uint64_t* n_bytes);
int hg_get_timeline(hg_ctx* ctx, char* out, uint64_t cap);
int hg_timeline_ms(hg_ctx* ctx, float* ms);  /* device time of the ordering + formatting */
/* phase-1 kernel times of the last run (segment walk, chain, decode), CUDA events */
int hg_phase_timing(hg_ctx* ctx, float* walk_ms, float* chain_ms, float* decode_ms);
/* order in which open calls are flushed as truncated spans at the end of the run:
 * the reference sorts its stacks by (str(hostname), pid, tid) (pipeline.py:230), which
 * differs from the (hostname or "", pid or 0, tid or 0) stream order when hostnames are
 * None.  rank[s] = position of stream s in the flush order (a permutation of the added
 * streams); NULL restores stream order.  Reset by hg_clear_streams. */
int hg_set_flush_order(hg_ctx* ctx, const uint32_t* rank, uint32_t n);
/* event sinks (`consumes = "events"`, pipeline.py:250-263): a run with HG_WANT_EVENTS orders
 * every record as mux_streams does (pipeline.py:68-114) and renders PrettyPrintSink's lines
 * (sinks.py:66-106; "\n"-terminated, UTF-8).  Schema and field names (EventSchema.name,
 * FieldSpec.name; fields in kinds[] order) are required first.  hg_get_event_order returns the
 * mux order itself: (stream index, record index within the stream) per event. */
int hg_set_schema_names(hg_ctx* ctx, const char* names, const uint64_t* offsets, uint32_t n_schemas,
                        const char* field_names, const uint64_t* field_offsets, uint32_t n_fields);
int hg_events_size(hg_ctx* ctx, uint64_t* n_bytes);
int hg_get_events(hg_ctx* ctx, char* out, uint64_t cap);
int hg_get_event_order(hg_ctx* ctx, uint32_t* stream, uint64_t* seq, uint64_t cap, uint64_t* n);
int hg_events_ms(hg_ctx* ctx, float* ms);  /* device time of ordering + rendering */
/* ValidationSink (sinks.py:448-594).  One rule row per schema (hg_set_registry order): kind bits
 * 1 uninit-pNext check (field `pnext`: the struct blob), 2 command-list execution (`exec`: the
 * handle), 4 creates a handle (`create`: the deref-out address; exits), 8 releases / 16 resets a
 * handle (exits: the handle comes from the latest entry of the same function on the same stream,
 * sinks.py:526-527, whose rule row has kind bit 32 and `rel` / `rst` = that parameter), `result`:
 * the exit's result field (-1: none, treated as 0).  A run with HG_WANT_VALIDATE returns the
 * findings: uninit_pnext / cmdlist_not_reset at their mux position, leaked handles (the host
 * sorts them by subject); orphan_exit findings come from the orphan list. */
enum { HG_FIND_PNEXT = 1, HG_FIND_CMDLIST = 2, HG_FIND_LEAK = 3 };
typedef struct hg_validation_rule {
  uint32_t kind;
  int16_t pnext, exec, create, rel, rst, result;
} hg_validation_rule;
typedef struct hg_finding {
  uint32_t rule;           /* HG_FIND_*                                       */
  uint32_t sid;            /* schema id of the record that raised it           */
  uint32_t stream;         /* its stream                                       */
  uint32_t pad;
  uint64_t pos;            /* its position in the mux order                    */
  uint64_t ts;             /* its timestamp                                    */
  uint64_t subject_lo;     /* subject = subject_hi * 2^64 + subject_lo - 2^63 for handles (65-bit key), */
  int64_t subject_hi;      /* the pNext value itself (hi 0) for uninit_pnext   */
} hg_finding;
int hg_set_validation_rules(hg_ctx* ctx, const hg_validation_rule* rules, uint32_t n_schemas);
int hg_get_findings(hg_ctx* ctx, hg_finding* out, uint64_t cap, uint64_t* n);
/* multi-rank timeline (collective (6) of SURVEY.md §8e): every rank runs with HG_WANT_TL_ITEMS
 * (phase 1 + its timeline messages in mux order), then hg_tl_export writes them into device memory
 * (`items`: 40-byte records, `payload`: the bytes of the device / telemetry records they print) with
 * stream keys made global (stream_global[s], flush_global[s]: the stream's index in the whole trace's
 * (hostname, pid, tid) order and in its (str(hostname), pid, tid) flush order).  Call once with NULL
 * destinations for the sizes.  Rank 0 concatenates the ranks' exports (NCCL) and hg_tl_import merges
 * the runs by mux key and formats the JSON exactly as a single run over the whole trace would
 * (hg_get_timeline).  hosts / pids / tids: the whole trace's identities (NULL host = None, INT64_MIN
 * pid / tid = None); flush_stream[k] = global stream of flush rank k. */
int hg_tl_export(hg_ctx* ctx, const uint32_t* stream_global, const uint32_t* flush_global, void* items, void* payload,
                 uint64_t* n_items, uint64_t* payload_bytes, uint64_t* n_device_spans);
int hg_tl_import(hg_ctx* ctx, void* items, uint64_t n_items, const uint64_t* run_start, const uint64_t* payload_start,
                 uint32_t n_runs, const void* payload, const char* const* hosts, const int64_t* pids, const int64_t* tids,
                 uint32_t n_streams, const uint32_t* flush_stream, uint64_t n_device_spans, uint64_t global_last_ts);
/* TimelineSink(device_index=) (sinks.py:347-349): device pid 9000000 + index */
int hg_set_timeline_device(hg_ctx* ctx, int32_t device_index);

/* device-resident dense tally: host rows are function-indexed, 6 x u64 each (count,
 * errors, sum lo, sum hi, min, max).  Returns a device pointer owned by the context. */
int hg_device_tally(hg_ctx* ctx, void** host_rows, uint64_t* n_host_rows);

/* multi-GPU merge (aggregator.py:35-76 merge_tallies as two collectives).  After
 * hg_finish, hg_merge_export writes this rank's tally, IntervalStats and per-stream
 * span counts into `dst` (DEVICE memory on this context's GPU, hg_merge_size int64
 * elements) in a rank-independent layout: rows of the n_fn functions, then the
 * n_dev_global device names of the global name order (dev_map[d] = global row of
 * local device row d, host array), span counts at stream_global[s] (host array, one
 * entry per local stream).  The caller all-reduces elements [0, sum_elems) with SUM
 * and the rest with MAX (NCCL), copies the buffer to host memory and hands it to
 * hg_merge_import together with the global device-name list (UTF-8, offsets[n] =
 * end); hg_get_tally / hg_get_device_names / hg_get_stats then return the merged
 * results.  Layout: see merge.cu. */
uint64_t hg_merge_size(uint32_t n_fn, uint32_t n_dev_global, uint32_t n_streams_global, uint64_t* sum_elems);
int hg_merge_export(hg_ctx* ctx, void* dst, const uint32_t* dev_map, uint32_t n_dev_local, uint32_t n_dev_global,
                    const uint32_t* stream_global, uint32_t n_streams_global);
int hg_merge_import(hg_ctx* ctx, const void* src, uint32_t n_dev_global, uint32_t n_streams_global,
                    const char* names, const uint64_t* name_offsets);

/* timing of the last run, CUDA events on the engine's stream: kernel_ms = the
 * dominant kernel (fast_scan_kernel + fast_kernel on the single pass, the decode kernel on the exact path), total_ms = whole run from staging to results
 * on the host; bytes moved host<->device and kernel launches of that run */
int hg_last_timing(hg_ctx* ctx, float* kernel_ms, float* total_ms, uint64_t* h2d_bytes, uint64_t* d2h_bytes,
                   uint64_t* kernel_launches);

/* engine options.  HG_OPT_PATH: 0 = single pass over HBM (fast.cuh) with the
 * exact three-kernel path as fallback whenever the single pass cannot vouch for
 * its result (any trace error, a wrong range speculation), 1 = exact path only,
 * 2 = single pass only (a trace it rejects fails with HG_ESTATE; tests).
 * HG_OPT_RANGE_BYTES: bytes per single-pass range (0 = sized so that one range
 * runs per resident lane).  The environment variable HAPIGPU_PATH sets the
 * default path at hg_create. */
#define HG_OPT_PATH 1u
#define HG_OPT_RANGE_BYTES 2u
int hg_set_option(hg_ctx* ctx, uint32_t key, uint64_t value);
/* which phase-1 path produced the last result (1 single pass, 0 exact), how many
 * single-pass results were discarded so far, and the range size used */
int hg_last_path(hg_ctx* ctx, uint32_t* path, uint64_t* fallbacks, uint32_t* range_bytes);

#ifdef __cplusplus
}
#endif
#endif /* HAPIGPU_H */
