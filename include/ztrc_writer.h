/*
 * ztrc_writer.h -- the five-function trace writer of the reference's C interposer layer,
 * implemented natively (libztrc.so, paper_2504_03683_b200/csrc/ztrc_writer.c).
 *
 * Replaces: the declarations of pkg/cinterpose/src/writer_binding.h:14-19 (which ship without an
 * implementation; contract in pkg/docs/writer-binding.md:10-45) and mirrors the Python
 * TraceWriter it stands for (tracefile.py:222-441): per-thread stream files
 * stream_<pid>_<tid>.bin with the 16-byte header, records [u32 schema_id][u64 ts][u32 len]
 * [payload] (trace-format.md), a single-producer ring per stream with drop-newest overflow
 * accounting counted in records, one drainer thread, and at close a streams.json index
 * (json.dumps(indent=1) layout, sorted by (hostname, pid, tid), silent streams omitted) and the
 * metadata flipped to "complete": true.  The trace it writes is read by open_trace_reader and
 * analysed by run_pipeline like any other.
 *
 * Identity: hostname = gethostname(), pid = getpid(), tid = gettid() of the emitting thread.
 */
#ifndef ZTRC_WRITER_H
#define ZTRC_WRITER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ztrc_stream ztrc_stream_t;

/* Create the trace directory (absent or empty), copy the pregenerated metadata.json from
 * metadata_path (it must carry "complete": false), start the drainer.  buffer_capacity: ring
 * slots (records) per stream, >= 1.  Returns 0 on success, -1 on failure. */
int ztrc_open(const char* dir, const char* metadata_path, uint64_t buffer_capacity);

/* The calling thread's stream, created on first use.  NULL only when the trace is not open. */
ztrc_stream_t* ztrc_stream_acquire(void);

/* Non-blocking enqueue of one encoded payload: 0 written, 1 dropped (ring full), -1 not open. */
int ztrc_emit(ztrc_stream_t* s, uint32_t schema_id, uint64_t timestamp_ns, const uint8_t* payload,
              uint32_t payload_len);

/* CLOCK_MONOTONIC in nanoseconds. */
uint64_t ztrc_clock_ns(void);

/* Quiesce (no emits may be in flight), flush every ring, write streams.json, flip the metadata
 * complete flag.  Returns 0 on success, -1 on failure (the trace stays marked incomplete). */
int ztrc_close(void);

/* test hooks: stop the drainer so rings fill deterministically (1) or restart it (0); drain now */
void ztrc_debug_pause_drainer(int paused);
void ztrc_debug_drain(void);

#ifdef __cplusplus
}
#endif
#endif /* ZTRC_WRITER_H */
