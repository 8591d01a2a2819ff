// ctx.h -- the engine context (hg_ctx) shared by the host translation units of libhapigpu.so:
// engine.cu (C ABI, staging, composition), fast.cu (single pass), seg.cu (exact path),
// timeline.cu (timeline ordering and formatting).  Kernel definitions stay in the one TU that
// launches them (HG_*_KERNELS guards in the .cuh files), so the TUs compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "timeline.cuh"
#include "seg.cuh"
#include "fast.cuh"

using namespace hg;

// ===========================================================================
// host side: the C ABI (include/hapigpu.h)

template <class T>
struct DBuf {
  T* ptr = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t want) {
    if (want <= n) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr; n = 0;
    cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(want, 1) * sizeof(T));
    if (e == cudaSuccess) n = want;
    return e;
  }
  void release() { if (ptr) cudaFree(ptr); ptr = nullptr; n = 0; }
};

enum StreamSource { SRC_HOST = 0, SRC_DEVICE = 1, SRC_FILE = 2 };

struct HostStream {
  std::string host;
  int64_t pid, tid;
  const uint8_t* data;  // host (SRC_HOST) or device (SRC_DEVICE) bytes; null for files
  uint64_t size;
  bool host_none;  // hostname None (record sources): "Host None pid .." in the timeline (sinks.py:367)
  bool pid_none = false, tid_none = false;  // pid / tid None (record sources): printed "None"
  int src = SRC_HOST;
  std::string path;       // SRC_FILE
  uint64_t file_off = 0;  // SRC_FILE: offset of the stream's first byte in the file
};

struct IngestStats {
  uint64_t pinned_bytes = 0, pageable_bytes = 0, file_bytes = 0, device_bytes = 0;
  float ms = 0;
  int threads = 0;
};
struct IngestPool;  // ingest.cu

// timeline sources (timeline.cu): a context's own messages, or the merged runs of several ranks
struct TlStreamName {
  std::string host;
  bool host_none;
  int64_t pid;
  bool pid_none;
  int64_t tid;
  bool tid_none;
};
struct TlSource {
  const TlItem* items = nullptr;
  uint32_t nrec_slots = 0, N = 0, ncomp = 0, n = 0;  // record region, all slots, compose's messages, messages
  const unsigned long long* rec_off = nullptr;        // first slot of every record-region run (device)
  uint32_t n_runs = 0;
  std::vector<TlStreamName> streams;                  // identities the stream field of the keys indexes
  const uint32_t* flush_stream = nullptr;             // device: flush rank -> stream (truncated spans)
  uint64_t n_dev = 0;                                 // device spans (thread-name table bound)
  // messages of the single pass (tl_ranges): range r's at items[r * rcap ...], rn[r] of them
  bool ranges = false;
  uint32_t n_ranges = 0, rcap = 0;
  const uint32_t* rn = nullptr;
  const uint32_t* range_stream = nullptr;
  const unsigned long long* range_base = nullptr;
  const uint32_t* stream_range0 = nullptr;
};

struct hg_ctx {
  hg_config cfg{};
  std::string err;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};  // 0 run start, 1 after staging, 2 after compose, 3 results on host, 4/5 phase 1, 6 after walk, 7 after chain
  int sm_count = 0;
  // registry
  std::vector<DSchema> schemas;
  std::vector<int32_t> sid_map;
  std::vector<uint2> desc;
  DBuf<uint2> d_desc;
  std::vector<uint8_t> kinds, field_role;
  uint32_t n_fn = 0, max_sid = 0;
  DBuf<DSchema> d_schemas;
  DBuf<int32_t> d_sid_map;
  DBuf<uint8_t> d_kinds, d_field_role;
  // streams
  std::vector<HostStream> streams;
  bool staged = false;
  std::vector<uint64_t> base, sizes;
  uint64_t total_bytes = 0;
  DBuf<uint8_t> d_data;
  DBuf<uint64_t> d_base, d_size;
  std::vector<uint32_t> tile_stream, stream_tile0;  // segment -> stream, stream -> first segment
  DBuf<uint32_t> d_tile_stream, d_stream_tile0;
  // scratch
  DBuf<SegState> d_state;
  uint32_t epoch = 0;
  DBuf<SumEntry> d_pool, d_stack;
  uint64_t pool_cap = 0, stack_cap = 0;
  DBuf<unsigned long long> d_host_acc, d_dev_acc, d_dev_wide;
  DBuf<unsigned long long> d_counters;  // misc counters, see below
  DBuf<hg_orphan> d_orphans;
  uint64_t orphan_cap = 0;
  DBuf<hg_trace_error> d_errors;
  uint32_t error_cap = 0;
  DBuf<unsigned long long> d_stream_spans;
  // name dict
  DBuf<unsigned long long> d_keys;
  DBuf<uint32_t> d_vals, d_name_len, d_small;
  DBuf<uint64_t> d_name_off;
  DBuf<uint8_t> d_arena;
  uint64_t dict_mask = 0, arena_cap = 0;
  uint32_t row_cap = 0;
  // results (host copies)
  bool have_results = false;
  uint32_t want = 0;
  std::vector<unsigned long long> counters;
  std::vector<unsigned long long> host_acc, dev_acc, dev_wide;
  std::vector<uint8_t> arena;
  std::vector<uint64_t> name_off;
  std::vector<uint32_t> name_len;
  uint32_t n_dev_rows = 0;
  std::vector<hg_orphan> orphans;
  std::vector<hg_trace_error> errors;
  std::vector<unsigned long long> stream_spans;
  uint64_t local_last_ts = 0, local_events = 0;
  bool phase1_done = false;
  float kernel_ms = 0, total_ms = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0, launches = 0;
  // timeline
  std::vector<std::string> fn_names;
  std::vector<uint8_t> fn_null;
  bool have_fn_names = false;
  DBuf<TlItem> d_tl_items;
  uint64_t tl_cap = 0;
  // timeline messages from the single pass: per range, in record order (Params::tl_ritems)
  bool tl_ranges = false;          // the last timeline run's messages are per range
  uint32_t tl_rcap = 0;            // message slots per range
  DBuf<uint32_t> d_tl_rn;          // messages per range
  DBuf<unsigned long long> d_tl_pres;  // result bits of the first pending exits per range
  DBuf<uint32_t> d_tl_rpre;        // exclusive scan of d_tl_rn
  bool ev_ranges = false;          // the last event run's records are per range (d_ev_items, d_ev_rn)
  DBuf<uint32_t> d_ev_rn;
  DBuf<unsigned long long> d_ev_seq;  // hg_get_event_order scratch
  DBuf<ulonglong2> d_tl_keys[2];
  DBuf<uint32_t> d_tl_idx[2];
  DBuf<uint32_t> d_tl_ro[2], d_tl_tcnt, d_tl_tile0, d_tl_split;  // sort: run offsets, tile counts, merge splits
  DBuf<uint32_t> d_tl_lens, d_tl_stream_proc;
  DBuf<uint64_t> d_tl_offs, d_tl_bsum, d_tl_fnq_off, d_tl_sstr_off;
  DBuf<char> d_tl_fnq, d_tl_sstr, d_tl_out, d_tl_devpid;
  DBuf<unsigned int> d_tl_proc_first, d_tl_th_state, d_tl_th_first;
  DBuf<unsigned long long> d_tl_th_hi, d_tl_th_lo;
  uint64_t tl_size = 0;
  bool tl_ready = false;
  const uint32_t* tl_order = nullptr;  // HG_WANT_TL_ITEMS: the messages' mux order (run_timeline_order)
  uint32_t tl_n = 0;
  DBuf<uint32_t> d_tlx_len, d_tlx_map;       // multi-rank export: payload lengths, stream maps
  DBuf<uint64_t> d_tlx_off;
  DBuf<unsigned long long> d_tlx_runs;       // multi-rank import: run starts
  DBuf<uint32_t> d_tlx_flush;
  float tl_ms = 0;
  uint64_t tl_comp_base = 0;
  float walk_ms = 0, chain_ms = 0, decode_ms = 0;
  // segments
  uint32_t seg_bytes = 8192;
  DBuf<SegW> d_segw;
  DBuf<SegInfo> d_seginfo;
  DBuf<unsigned long long> d_stream_nrec, d_tl_rec_off;
  DBuf<SumEntry> d_deep;
  uint64_t deep_cap = 0;
  DBuf<Params> d_params;
  // single-pass range path (fast.cuh)
  int path_opt = 0;                 // 0 auto (fast, exact on anomaly), 1 exact only, 2 fast only
  uint32_t range_opt = 0;           // forced range bytes (0 = sized to the resident lanes)
  uint32_t range_bytes = 0, n_ranges = 0, fast_warps = 0;
  std::vector<uint32_t> range_stream, stream_range0;
  DBuf<uint32_t> d_range_stream, d_stream_range0;
  DBuf<RangeState> d_rstate;
  DBuf<SegState> d_rseg;
  DBuf<unsigned long long> d_range_base;
  std::vector<uint32_t> vplan;
  DBuf<uint32_t> d_vplan;
  std::vector<uint4> fdesc, dplan;
  bool has_dev = true;
  int desc_mode = 0;                // fast_kernel descriptors: 0 global (L1), 1 shared uint4, 2 shared compact              // some schema is device-profiling (the range kernel's name cache)
  DBuf<uint4> d_fdesc, d_dplan;
  int last_path = 0;                // 1 = the last run's phase 1 was the single pass
  uint64_t fallbacks = 0;
  uint32_t last_anom = 0;
  uint32_t range_shift = 0;  // extra bytes per range (retry after a failed speculation)
  uint64_t retries = 0;
  uint32_t max_rps = 0;      // most ranges in one stream (fast_verify_kernel's width)
  bool deep_inline = false;  // fast_kernel<_, true>: overflow chunks handled inline
  int smem_optin = 0;
  // compose blocks (single pass)
  uint32_t n_blk = 0;
  std::vector<uint32_t> blk_stream, blk_u0, stream_blk0;
  DBuf<uint32_t> d_blk_stream, d_blk_u0, d_stream_blk0;
  DBuf<SegState> d_blk_state;
  // truncation flush order (hg_set_flush_order)
  bool flush_order = false;
  DBuf<uint32_t> d_flush_rank, d_flush_stream;
  // event sinks (events.cu): schema / field names, the mux-ordered records and their text
  bool have_schema_names = false;
  std::vector<std::string> schema_names, field_names;
  DBuf<TlItem> d_ev_items;
  DBuf<char> d_ev_spre, d_ev_sname, d_ev_fname, d_ev_out;
  DBuf<uint64_t> d_ev_spre_off, d_ev_sname_off, d_ev_fname_off, d_ev_offs;
  DBuf<uint32_t> d_ev_lens;
  const uint32_t* ev_order = nullptr;
  uint64_t ev_size = 0;
  bool ev_ready = false;
  float ev_ms = 0;
  // validation (validate.cu)
  std::vector<hg_validation_rule> val_rules;
  DBuf<hg_validation_rule> d_val_rules;
  DBuf<unsigned int> d_val_cnt;
  DBuf<uint32_t> d_val_order;
  DBuf<TlItem> d_val_eq, d_val_xr, d_val_cr;
  DBuf<hg_finding> d_val_fnd;
  std::vector<hg_finding> val_findings;
  bool val_ready = false;
  size_t compose_smem = 0;  // compose_kernel's dynamic shared memory attribute as last set
  // pinned host staging of small results (counters, tally rows, names, orphans, errors): one sync
  uint8_t* pin = nullptr;
  size_t pin_cap = 0;
  // ingest (ingest.cu): pinned staging pool and the last staging's numbers
  IngestPool* ingest = nullptr;
  IngestStats ingest_stats;
  // multi-GPU merge (merge.cu): results replaced by the all-reduced ones
  bool merged = false;
  DBuf<uint32_t> d_merge_map;
};

// counter slots in d_counters
enum {
  C_STATS = 0,            // 7 slots
  C_LAST_TS = 8,
  C_POOL_USED = 9,
  C_STACK_USED = 10,
  C_N_ORPHANS = 11,
  C_N_ERRORS = 12,        // unsigned int in a u64 slot
  C_WORK = 13,            // unsigned int
  C_ARENA_USED = 14,
  C_N_ROWS = 15,          // unsigned int
  C_OVERFLOW = 16,        // unsigned int
  C_WIDE = 17,            // unsigned int
  C_WATCHDOG = 18,        // unsigned int
  C_TL_N = 19,            // timeline messages appended
  C_TL_TOTAL = 20,        // timeline body bytes (scan total)
  C_TL_TH_OVF = 21,       // unsigned int: thread-name table overflow
  C_DEEP_USED = 22,       // deep lane-stack chunks handed out
  C_TL_N2 = 23,           // timeline messages appended by compose
  C_REC_TOTAL = 24,       // records of all streams (timeline slots)
  C_ANOM = 25,            // unsigned int: single-pass result void (fast.cuh)
  C_NUM = 26
};

static inline int fail(hg_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail(ctx, HG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// json.dumps(str) with ensure_ascii (json/encoder.py) of a valid UTF-8 string
static inline std::string json_quote(const std::string& s) {
  static const char* hx = "0123456789abcdef";
  std::string o = "\"";
  auto u4 = [&](uint32_t v) {
    o += "\\u";
    o += hx[(v >> 12) & 15]; o += hx[(v >> 8) & 15]; o += hx[(v >> 4) & 15]; o += hx[v & 15];
  };
  for (size_t i = 0; i < s.size();) {
    uint32_t c = (uint8_t)s[i], cp;
    auto b = [&](size_t k) { return (uint32_t)(k < s.size() ? (uint8_t)s[k] : 0x80) & 0x3F; };
    if (c < 0x80) { cp = c; i += 1; }
    else if (c < 0xE0) { cp = ((c & 0x1F) << 6) | b(i + 1); i += 2; }
    else if (c < 0xF0) { cp = ((c & 0x0F) << 12) | (b(i + 1) << 6) | b(i + 2); i += 3; }
    else { cp = ((c & 0x07) << 18) | (b(i + 1) << 12) | (b(i + 2) << 6) | b(i + 3); i += 4; }
    if (cp == '"') o += "\\\"";
    else if (cp == '\\') o += "\\\\";
    else if (cp >= 0x20 && cp < 0x7F) o += (char)cp;
    else if (cp == '\n') o += "\\n";
    else if (cp == '\r') o += "\\r";
    else if (cp == '\t') o += "\\t";
    else if (cp == '\b') o += "\\b";
    else if (cp == '\f') o += "\\f";
    else if (cp < 0x10000) u4(cp);
    else { uint32_t v = cp - 0x10000; u4(0xD800 | (v >> 10)); u4(0xDC00 | (v & 0x3FF)); }
  }
  o += "\"";
  return o;
}

template <class T>
static cudaError_t upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
  cudaError_t e = d.ensure(std::max<size_t>(h.size(), 1));
  if (e != cudaSuccess || h.empty()) return e;
  return cudaMemcpyAsync(d.ptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st);
}


// shared between the host translation units (C linkage: engine.cu defines them inside its extern "C" block)
extern "C" {
Params make_params(hg_ctx* ctx);
int init_run(hg_ctx* ctx);
int launch_fast(hg_ctx* ctx);      // fast.cu
int launch_phase1(hg_ctx* ctx);    // seg.cu
int run_timeline(hg_ctx* ctx, uint64_t global_last_ts);  // timeline.cu
int ingest_streams(hg_ctx* ctx);   // ingest.cu
int run_events(hg_ctx* ctx);       // events.cu
int run_validation(hg_ctx* ctx);   // validate.cu
int tl_sort(hg_ctx* ctx, const TlItem* items, uint32_t nrec_slots, uint32_t N, uint32_t ncomp, uint32_t n,
            const uint32_t** order);                                                   // timeline.cu
int tl_sort_runs(hg_ctx* ctx, const TlItem* items, uint32_t nrec_slots, uint32_t N, uint32_t ncomp, uint32_t n,
                 const unsigned long long* rec_off, uint32_t n_runs, const uint32_t** order);  // timeline.cu
int run_timeline_order(hg_ctx* ctx);                                                   // timeline.cu
int tl_merge_passes(hg_ctx* ctx, uint32_t R, uint32_t n, const uint32_t** order);          // timeline.cu
int tl_sort_ranges(hg_ctx* ctx, const TlSource& S, uint32_t* n_out, const uint32_t** order);  // timeline.cu
int timeline_from(hg_ctx* ctx, const TlSource& S, uint64_t global_last_ts);            // timeline.cu
int tl_scan(hg_ctx* ctx, const uint32_t* lens, uint32_t n, uint64_t* offs, uint64_t* total);  // timeline.cu
void ingest_free(hg_ctx* ctx);     // ingest.cu
}
