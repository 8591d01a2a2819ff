// engine.cu -- hapigpu: B200 (sm_100a) trace post-processing engine.
//
// Hot path: decode the per-thread stream files,
// pair host entry/exit records per stream into spans, fold spans into the
// tally.  Reference semantics:
//   record format / decode errors     tracefile.py:147-215, docs/trace-format.md
//   per-stream monotonicity           pipeline.py:95-100
//   LIFO pairing, typed mismatch      pipeline.py:156-185
//   device spans, telemetry samples   pipeline.py:186-215, sampler.py:36-48
//   truncation at the global last ts  pipeline.py:152, 220-240
//   tally fold                        sinks.py:123-132, 230-242
//
// Kernel structure (one pass over the trace bytes):
//   tile_kernel     persistent; one warp per 4 KiB stream tile.  The warp stages
//                   the tile (+overhang) in shared memory, finds record
//                   boundaries speculatively per lane, verifies them against the
//                   preceding tile through a decoupled look-back on a tile-state
//                   array, then decodes 32 records per round and runs the stack
//                   automaton with ballot/shuffle elimination.  Completed spans
//                   fold into a CTA-shared tally table; unresolved exits (empty
//                   stack) and residual entries go to a small per-tile summary.
//   compose_kernel  per stream, composes the tile summaries in order (the same
//                   automaton over a tiny sequence), emits cross-tile spans,
//                   orphans and the truncated spans at the global last ts.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hg_device.cuh"

using namespace hg;

namespace {

constexpr int kTile = 4096;                    // stream bytes per warp tile
constexpr int kLaneBytes = kTile / kWarp;      // 128
constexpr int kMaxRecLane = kLaneBytes / 16;   // 8
constexpr int kMaxRecTile = kTile / 16;        // 256
constexpr int kOverhang = 1024;
constexpr int kWinBytes = kTile + kOverhang;   // staged window
constexpr int kWarpsPerCta = 8;
constexpr int kCtaThreads = kWarpsPerCta * kWarp;
constexpr uint32_t kSmemFnMax = 2048;          // host rows tallied in shared memory up to this many functions

struct Elem {        // pending exit (bottom of the array) or stack frame (above)
  uint64_t ts;
  uint64_t result;
  int32_t fn;
  uint16_t seq;      // record index within the tile
  uint16_t flags;    // bit0 exit, bit1 error, bit2 bad f64 result
};

struct WarpSmem {
  uint32_t win[kWinBytes / 4 + 4];
  uint16_t roff[kMaxRecTile];
  Elem elems[kMaxRecTile];
};

struct SmemRow {     // per-CTA host row accumulator
  uint32_t count, err;
  uint32_t s0, s1, s2, pad;   // 96-bit sum
  unsigned long long mn, mx;
};

enum Stat { ST_EVENTS = 0, ST_PASSED, ST_HOST, ST_TRUNC, ST_DEVICE, ST_SAMPLES, ST_ORPHANS, ST_N };

struct Params {
  const uint8_t* data;
  const uint64_t* stream_base;
  const uint64_t* stream_size;
  const uint32_t* tile_stream;    // stream-major tile id -> stream
  const uint32_t* stream_tile0;   // stream -> first stream-major tile id
  const uint32_t* order;          // processing order -> stream-major tile id
  uint32_t n_tiles, n_streams;
  const DSchema* schemas;
  const int32_t* sid_map;
  uint32_t max_sid;
  const uint8_t* kinds;
  const uint8_t* field_role;
  uint32_t n_fn;
  TileState* state;
  uint32_t epoch;
  SumEntry* pool;
  unsigned long long* pool_used;
  uint64_t pool_cap;
  unsigned long long* host_acc;   // n_fn x 6: count, err, sum_lo, sum_hi, min, max
  unsigned long long* dev_acc;    // row_cap x 6: count, err, sum_lo, sum_hi, min_b, max_b
  uint32_t* wide_flag;
  NameDict names;
  hg_orphan* orphans;
  unsigned long long* n_orphans;
  uint64_t orphan_cap;
  hg_trace_error* errors;
  unsigned int* n_errors;
  uint32_t error_cap;
  unsigned long long* stats;
  unsigned long long* last_ts;
  unsigned long long* stream_spans;
  unsigned int* work_counter;
  uint32_t* watchdog;
  uint32_t want;
  // compose
  SumEntry* stack_scratch;
  unsigned long long* stack_used;
  uint64_t stack_cap;
  uint64_t global_last_ts;
};

// ---------------------------------------------------------------------------
// small device helpers

__device__ __forceinline__ const DSchema* schema_of(const Params& p, uint32_t sid) {
  if (sid > p.max_sid) return nullptr;
  int32_t si = __ldg(&p.sid_map[sid]);
  return si < 0 ? nullptr : &p.schemas[si];
}

// header-level validity used to walk a chain (tracefile.py:199-210 order)
__device__ __forceinline__ bool header_walkable(const Params& p, const Window& w, uint64_t off, uint64_t& next) {
  if (off + 16 > w.size) return false;
  uint32_t sid = rd32(w, off);
  uint32_t plen = rd32(w, off + 12);
  if (off + 16 + plen > w.size) return false;
  if (!schema_of(p, sid)) return false;
  next = off + 16 + plen;
  return true;
}

// stricter plausibility used to pick speculative sync points
__device__ __forceinline__ bool header_plausible(const Params& p, const Window& w, uint64_t off, uint64_t& next, uint64_t& ts) {
  if (off + 16 > w.size) return false;
  uint32_t sid = rd32(w, off);
  const DSchema* s = schema_of(p, sid);
  if (!s) return false;
  uint32_t plen = rd32(w, off + 12);
  if (off + 16 + plen > w.size) return false;
  if (s->flags & SF_VAR) { if (plen < s->fixed_len) return false; }
  else if (plen != s->fixed_len) return false;
  next = off + 16 + plen;
  ts = rd64(w, off + 4);
  return true;
}

__device__ __forceinline__ bool sync_ok(const Params& p, const Window& w, uint64_t off) {
  uint64_t next, ts, n2, ts2;
  if (!header_plausible(p, w, off, next, ts)) return false;
  if (next == w.size) return true;
  if (!header_plausible(p, w, next, n2, ts2)) return false;
  return ts2 >= ts;
}

// walk records from `entry` while they start before `sub1`; offsets go to roff
__device__ __forceinline__ void lane_walk(const Params& p, const Window& w, uint64_t t0, uint64_t entry, uint64_t sub1,
                                          uint16_t* roff_lane, uint32_t& cnt, uint64_t& exit, bool& fail,
                                          uint64_t& fail_off) {
  uint64_t off = entry;
  cnt = 0;
  fail = false;
  while (off < sub1) {
    uint64_t next;
    if (!header_walkable(p, w, off, next)) { fail = true; fail_off = off; exit = kNone; return; }
    roff_lane[cnt++] = (uint16_t)(off - t0);
    off = next;
  }
  exit = off;
}

// intra-warp consistency of lane walks given the tile entry e0 (kNone = dead)
__device__ void warp_verify(const Params& p, const Window& w, uint64_t t0, uint64_t sub1, uint16_t* roff_lane,
                            uint64_t e0, uint64_t& hyp, uint32_t& cnt, uint64_t& exit, bool& fail, uint64_t& fail_off) {
  const uint32_t lane = lane_id();
  for (int it = 0; it < 2 * kWarp + 2; it++) {
    uint64_t up = __shfl_up_sync(0xffffffffu, exit, 1);
    uint64_t e_in = lane == 0 ? e0 : up;
    bool good;
    if (e_in == kNone) good = true;  // behind a failed lane: dead
    else if (e_in >= sub1) good = (cnt == 0 && !fail && exit == e_in);
    else good = (hyp == e_in);
    if (__all_sync(0xffffffffu, good)) return;
    if (!good) {
      if (e_in >= sub1) { cnt = 0; fail = false; exit = e_in; hyp = e_in; }
      else { hyp = e_in; lane_walk(p, w, t0, e_in, sub1, roff_lane, cnt, exit, fail, fail_off); }
    }
  }
}

// ---------------------------------------------------------------------------
// tile-state publication (decoupled look-back)

__device__ __forceinline__ uint32_t st_status(const TileState* s) { return *(volatile const uint32_t*)&s->status; }
__device__ __forceinline__ uint64_t vld(const uint64_t* a) { return *(volatile const uint64_t*)a; }
__device__ __forceinline__ uint32_t vld32(const uint32_t* a) { return *(volatile const uint32_t*)a; }

// state fields: spec_* and done_* never alias (see TileState in hg_device.cuh)
struct Look {
  uint64_t entry;  // true entry offset of this tile (kNone: predecessor chain failed)
  uint64_t base;   // records of the stream before this tile
  uint64_t prev_ts;
  bool has_prev;
};

__device__ __forceinline__ uint32_t wait_status(const Params& p, const TileState* s, bool need_final) {
  long long t_start = clock64();
  for (uint32_t spins = 0;; spins++) {
    uint32_t st = st_status(s);
    if ((st >> 2) == p.epoch) {
      uint32_t c = st & 3u;
      if (c == TS_DONE || c == TS_ERROR || (!need_final && c == TS_SPEC)) { __threadfence(); return c; }
    }
    __nanosleep(64);
    // watchdog: a predecessor that never publishes is an engine bug; fail loudly instead of hanging
    if ((spins & 1023u) == 1023u && clock64() - t_start > (long long)8e9) {
      atomicExch(p.watchdog, 1u);
      return TS_ERROR;
    }
  }
}

// layout of the two publications inside TileState
//   SPEC : spec_entry, exit (=spec exit), n_local (spec count), last_ts (spec last ts)
//   DONE : pool_* unused here; done values in `incl`, `has_last`, and exit/last in
//          the second half (we reuse pad fields through a side array, see below)
struct DoneState { uint64_t exit, incl, last_ts; uint32_t has_last, pad; };

__device__ Look lookback(const Params& p, const DoneState* done, uint32_t g0, uint32_t g, uint64_t size) {
  Look L;
  uint32_t k = g - 1;
  for (;;) {  // walk back to the nearest final tile
    uint32_t c = wait_status(p, &p.state[k], false);
    if (c != TS_SPEC) break;
    k--;  // the stream's first tile never publishes SPEC
  }
  for (;;) {
    uint32_t c = wait_status(p, &p.state[k], true);
    if (c == TS_ERROR) { L.entry = kNone; L.base = 0; L.prev_ts = 0; L.has_prev = false; return L; }
    uint64_t e = vld(&done[k].exit);
    uint64_t base = vld(&done[k].incl);
    uint64_t last = vld(&done[k].last_ts);
    bool has = vld32(&done[k].has_last) != 0;
    bool broken = false;
    uint32_t i = k + 1;
    for (; i < g; i++) {
      uint32_t ci = wait_status(p, &p.state[i], false);
      if (ci == TS_ERROR) { L.entry = kNone; L.base = 0; L.prev_ts = 0; L.has_prev = false; return L; }
      if (ci == TS_DONE) {
        e = vld(&done[i].exit); base = vld(&done[i].incl); last = vld(&done[i].last_ts); has = vld32(&done[i].has_last) != 0;
        continue;
      }
      const TileState* s = &p.state[i];
      uint64_t se = vld(&s->spec_entry), sx = vld(&s->exit);
      uint32_t sn = vld32(&s->n_local);
      uint64_t t1 = min(16 + (uint64_t)(i - g0 + 1) * kTile, size);  // tile end (stream offset)
      bool ok;
      if (se == kNone) ok = (e >= t1);          // pass-through tile
      else ok = (e == se) && sx != kNone;
      if (!ok) { broken = true; break; }
      if (se != kNone) {
        e = sx;
        base += sn;
        if (sn) { last = vld(&s->last_ts); has = true; }
      }
    }
    if (!broken) { L.entry = e; L.base = base; L.prev_ts = last; L.has_prev = has; return L; }
    wait_status(p, &p.state[i], true);  // tile i repairs itself; continue from it
    k = i;
  }
}

__device__ __forceinline__ void publish(TileState* s, uint32_t epoch, uint32_t code) {
  __threadfence();
  *(volatile uint32_t*)&s->status = (epoch << 2) | code;
}

// ---------------------------------------------------------------------------
// host-row folding (CTA shared table or global)

__device__ __forceinline__ void smem_min_u64(unsigned long long* a, unsigned long long v) {
  if (v < *(volatile unsigned long long*)a) atomicMin(a, v);
}
__device__ __forceinline__ void smem_max_u64(unsigned long long* a, unsigned long long v) {
  if (v > *(volatile unsigned long long*)a) atomicMax(a, v);
}

__device__ void fold_host_lane(const Params& p, SmemRow* tab, int32_t fn, uint64_t dur, bool err) {
  if (tab) {
    SmemRow* r = &tab[fn];
    atomicAdd(&r->count, 1u);
    if (err) atomicAdd(&r->err, 1u);
    uint32_t lo = (uint32_t)dur, hi = (uint32_t)(dur >> 32);
    uint32_t o0 = atomicAdd(&r->s0, lo);
    uint32_t c0 = (o0 + lo) < o0;
    uint32_t add1 = hi + c0;
    uint32_t c1 = (add1 < hi);  // hi + c0 overflowed
    uint32_t o1 = atomicAdd(&r->s1, add1);
    c1 += (o1 + add1) < o1;
    if (c1) atomicAdd(&r->s2, c1);
    smem_min_u64(&r->mn, dur);
    smem_max_u64(&r->mx, dur);
  } else {
    unsigned long long* a = p.host_acc + 6ull * fn;
    atomicAdd(&a[0], 1ull);
    if (err) atomicAdd(&a[1], 1ull);
    add_i128(&a[2], &a[3], dur, 0);
    atomicMin(&a[4], dur);
    atomicMax(&a[5], dur);
  }
}

// fold this round's completed host spans, aggregating lanes with the same function
__device__ void fold_host_round(const Params& p, SmemRow* tab, bool paired, int32_t fn, uint64_t dur, bool err) {
  uint32_t todo = __ballot_sync(0xffffffffu, paired);
  bool wide = __any_sync(0xffffffffu, paired && dur >= (1ull << 32));
  if (wide || !tab) {
    if (paired) fold_host_lane(p, tab, fn, dur, err);
    return;
  }
  const uint32_t lane = lane_id();
  while (todo) {
    int leader = __ffs(todo) - 1;
    int32_t f = __shfl_sync(0xffffffffu, fn, leader);
    bool in = paired && fn == f;
    uint32_t grp = __ballot_sync(0xffffffffu, in);
    uint32_t errs = __ballot_sync(0xffffffffu, in && err);
    if (in) {
      uint32_t d = (uint32_t)dur;
      uint32_t lo = __reduce_add_sync(grp, d & 0xffffu);
      uint32_t hi = __reduce_add_sync(grp, d >> 16);
      uint32_t mn = __reduce_min_sync(grp, d);
      uint32_t mx = __reduce_max_sync(grp, d);
      if ((int)lane == leader) {
        SmemRow* r = &tab[f];
        atomicAdd(&r->count, (uint32_t)__popc(grp));
        if (errs) atomicAdd(&r->err, (uint32_t)__popc(errs));
        uint64_t sum = (uint64_t)lo + ((uint64_t)hi << 16);  // < 2^37
        uint32_t slo = (uint32_t)sum, shi = (uint32_t)(sum >> 32);
        uint32_t o0 = atomicAdd(&r->s0, slo);
        uint32_t add1 = shi + ((o0 + slo) < o0 ? 1u : 0u);
        if (add1) {
          uint32_t o1 = atomicAdd(&r->s1, add1);
          if ((o1 + add1) < o1) atomicAdd(&r->s2, 1u);
        }
        smem_min_u64(&r->mn, mn);
        smem_max_u64(&r->mx, mx);
      }
    }
    todo &= ~grp;
  }
}

__device__ __forceinline__ void fold_device(const Params& p, uint32_t row, uint64_t d_lo, int64_t d_hi) {
  unsigned long long* a = p.dev_acc + 6ull * row;
  atomicAdd(&a[0], 1ull);
  add_i128(&a[2], &a[3], d_lo, d_hi);
  // i128 (d_hi:d_lo) fits in i64 iff d_hi is the sign extension of d_lo
  if (d_hi == ((int64_t)d_lo >> 63)) {
    atomicMin(&a[4], bias64((int64_t)d_lo));
    atomicMax(&a[5], bias64((int64_t)d_lo));
  } else {
    atomicExch(p.wide_flag, 1u);
  }
}

__device__ void push_error(const Params& p, uint32_t code, uint32_t stream, uint64_t seq, uint64_t off, uint64_t ts,
                           uint64_t prev_ts, uint64_t aux) {
  unsigned int i = atomicAdd(p.n_errors, 1u);
  if (i < p.error_cap) {
    hg_trace_error e;
    e.code = code; e.stream = stream; e.seq = seq; e.offset = off; e.ts = ts; e.prev_ts = prev_ts; e.aux = aux;
    p.errors[i] = e;
  }
}

__device__ void push_orphans(const Params& p, bool is_orphan, uint32_t stream, int32_t fn, uint64_t ts, uint64_t seq) {
  uint32_t m = __ballot_sync(0xffffffffu, is_orphan);
  if (!m) return;
  unsigned long long base = 0;
  if (lane_id() == 0) base = atomicAdd(p.n_orphans, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (is_orphan) {
    uint64_t i = base + __popc(m & lanemask_lt());
    if (i < p.orphan_cap) { hg_orphan o; o.stream = stream; o.function = fn; o.ts = ts; o.seq = seq; p.orphans[i] = o; }
  }
}

// ---------------------------------------------------------------------------
// per-record decode (tracefile.py:147-169 + pipeline.py:150-218 classification)

enum RecKind : uint32_t { RK_NONE = 0, RK_ENTRY = 1, RK_EXIT = 2 };

struct RecOut {
  uint32_t kind;     // RK_*
  int32_t fn;
  uint64_t ts;
  uint64_t result;
  uint32_t flags;    // bit1 error, bit2 bad f64 result
  uint32_t dec_err;  // HG_ERR_* decode-level (pull) error
  uint64_t dec_aux;
  uint32_t feed_err; // HG_ERR_FEED / HG_ERR_TELEMETRY at this record
  uint64_t feed_aux;
};

__device__ void decode_record(const Params& p, const Window& w, uint64_t off, uint32_t stream, RecOut& o,
                              uint32_t& dev_spans, uint32_t& samples, uint32_t& passed) {
  o.kind = RK_NONE; o.flags = 0; o.dec_err = 0; o.feed_err = 0; o.result = 0; o.fn = -1;
  uint32_t sid = rd32(w, off);
  o.ts = rd64(w, off + 4);
  uint32_t plen = rd32(w, off + 12);
  const uint64_t body = off + 16;
  const DSchema* s = schema_of(p, sid);  // non-null: checked by the walk
  uint64_t role_off[HG_NUM_ROLES];
  #pragma unroll
  for (int r = 0; r < HG_NUM_ROLES; r++) role_off[r] = 0;
  uint32_t name_len = 0;
  if (!(s->flags & SF_VAR)) {
    if (plen != s->fixed_len) { o.dec_err = HG_ERR_LEN_MISMATCH; return; }
    #pragma unroll
    for (int r = 0; r < HG_NUM_ROLES; r++) if (s->role[r] >= 0) role_off[r] = body + 8u * (uint32_t)s->role[r];
  } else {
    uint64_t q = 0;
    const uint8_t* kd = p.kinds + s->kinds_off;
    const uint8_t* fr = p.field_role + s->kinds_off;
    for (uint32_t i = 0; i < s->nfields; i++) {
      uint8_t k = __ldg(&kd[i]);
      uint8_t role = __ldg(&fr[i]);
      if (k < HG_KIND_STRING) {
        if (q + 8 > plen) { o.dec_err = HG_ERR_STRUCT; o.dec_aux = (q << 8) | 8; return; }
        if (role != 0xff) role_off[role] = body + q;
        q += 8;
      } else {
        if (q + 4 > plen) { o.dec_err = HG_ERR_STRUCT; o.dec_aux = (q << 8) | 4; return; }
        uint32_t ln = rd32(w, body + q);
        q += 4;
        if (q + ln > plen) { o.dec_err = HG_ERR_TRUNC_VAR; return; }
        if (k == HG_KIND_STRING && !utf8_valid(w, body + q, ln)) { o.dec_err = HG_ERR_UTF8; o.dec_aux = q; return; }
        if (role != 0xff) {
          role_off[role] = body + q;
          if (role == HG_ROLE_NAME) name_len = ln;
        }
        q += ln;
      }
    }
    if (q != plen) { o.dec_err = HG_ERR_TRAILING; return; }
  }
  switch (s->cls) {
    case HG_CLASS_ENTRY:
      o.kind = RK_ENTRY; o.fn = s->fn;
      return;
    case HG_CLASS_EXIT: {
      o.kind = RK_EXIT; o.fn = s->fn;
      if (s->flags & SF_RESULT) {
        uint64_t bits = rd64(w, role_off[HG_ROLE_RESULT]);
        o.result = bits;
        if (s->flags & SF_RESULT_F64) {
          double x = __longlong_as_double((long long)bits);
          if (isnan(x) || isinf(x)) o.flags |= 4;
          else if (x >= 1.0 || x <= -1.0) o.flags |= 2;
        } else if (bits != 0) {
          o.flags |= 2;
        }
      }
      return;
    }
    case HG_CLASS_DEVICE: {
      if (s->flags & SF_FEED_ALWAYS) { o.feed_err = HG_ERR_FEED; o.feed_aux = sid; return; }
      uint64_t a = rd64(w, role_off[HG_ROLE_START]);
      uint64_t b = rd64(w, role_off[HG_ROLE_END]);
      int64_t ah = (s->role_kind[HG_ROLE_START] == HG_KIND_I64 && (int64_t)a < 0) ? -1 : 0;
      int64_t bh = (s->role_kind[HG_ROLE_END] == HG_KIND_I64 && (int64_t)b < 0) ? -1 : 0;
      uint64_t d_lo = b - a;
      int64_t d_hi = bh - ah - (b < a ? 1 : 0);
      uint32_t row = name_lookup(p.names, w, role_off[HG_ROLE_NAME], name_len);
      if (row != 0xffffffffu) fold_device(p, row, d_lo, d_hi);
      dev_spans++;
      return;
    }
    case HG_CLASS_TELEMETRY: {
      if (s->flags & SF_FEED_ALWAYS) { o.feed_err = HG_ERR_FEED; o.feed_aux = sid; return; }
      uint64_t bits = rd64(w, role_off[HG_ROLE_VALUE]);
      uint8_t vk = s->role_kind[HG_ROLE_VALUE];
      bool util = s->counter_kind >= HG_COUNTER_COMPUTE;
      bool bad;
      if (vk == HG_KIND_F64) {
        double v = __longlong_as_double((long long)bits);
        bad = util ? !(v >= 0.0 && v <= 1.0) : (v < 0.0);
      } else if (vk == HG_KIND_I64) {
        int64_t v = (int64_t)bits;
        bad = util ? !(v >= 0 && v <= 1) : (v < 0);
      } else {
        bad = util ? (bits > 1) : false;
      }
      if (bad) { o.feed_err = HG_ERR_TELEMETRY; o.feed_aux = bits; return; }
      samples++;
      if ((s->flags & SF_FEED_TIMELINE) && (p.want & HG_WANT_TIMELINE)) { o.feed_err = HG_ERR_FEED; o.feed_aux = sid; }
      return;
    }
    default:
      passed++;
      return;
  }
}

// ---------------------------------------------------------------------------
// the tile kernel

__global__ void __launch_bounds__(kCtaThreads) tile_kernel(Params p, DoneState* done) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SmemRow* tab = nullptr;
  size_t tab_bytes = 0;
  if (p.n_fn <= kSmemFnMax) {
    tab = reinterpret_cast<SmemRow*>(smem_raw);
    tab_bytes = ((sizeof(SmemRow) * p.n_fn + 127) / 128) * 128;
    for (uint32_t i = threadIdx.x; i < p.n_fn; i += blockDim.x) {
      SmemRow z; z.count = z.err = z.s0 = z.s1 = z.s2 = z.pad = 0; z.mn = ~0ull; z.mx = 0;
      tab[i] = z;
    }
  }
  WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem_raw + tab_bytes) + (threadIdx.x >> 5);
  __syncthreads();

  const uint32_t lane = lane_id();
  uint32_t st_events = 0, st_passed = 0, st_host = 0, st_dev = 0, st_samples = 0, st_orph = 0;
  uint64_t my_last_ts = 0;

  for (;;) {
    uint32_t work = 0;
    if (lane == 0) work = atomicAdd(p.work_counter, 1u);
    work = __shfl_sync(0xffffffffu, work, 0);
    if (work >= p.n_tiles) break;
    const uint32_t g = p.order[work];
    const uint32_t s = p.tile_stream[g];
    const uint32_t g0 = p.stream_tile0[s];
    const uint32_t j = g - g0;
    const uint64_t size = p.stream_size[s];
    const uint8_t* gbase = p.data + p.stream_base[s];
    const uint64_t t0 = 16 + (uint64_t)j * kTile;
    const uint64_t t1 = min(t0 + kTile, size);

    // ---- stage [t0, t0 + kWinBytes) (clipped to the padded stream end) in shared memory
    Window w;
    w.s = ws->win;
    w.win_start = t0;
    w.g = gbase;
    w.size = size;
    {
      uint64_t want_end = min(t0 + (uint64_t)kWinBytes, (uint64_t)((size + 15) & ~(uint64_t)15));
      uint32_t nvec = (uint32_t)((want_end - t0 + 15) / 16);
      const uint4* src = reinterpret_cast<const uint4*>(gbase + t0);
      uint4* dst = reinterpret_cast<uint4*>(ws->win);
      for (uint32_t v = lane; v < nvec; v += kWarp) dst[v] = __ldg(&src[v]);
      // staged bytes usable by rd32/rd64 (they read up to 8 bytes past off)
      w.win_end = t0 + (uint64_t)nvec * 16;
      if (lane < 4) ws->win[nvec * 4 + lane] = 0;
    }
    __syncwarp();

    // ---- pass A: speculative boundaries per lane
    const uint64_t sub0 = min(t0 + (uint64_t)lane * kLaneBytes, t1);
    const uint64_t sub1 = min(sub0 + kLaneBytes, t1);
    uint16_t* roff_lane = ws->roff + lane * kMaxRecLane;
    uint64_t hyp = kNone, exit = kNone, fail_off = 0;
    uint32_t cnt = 0;
    bool fail = false;
    for (uint64_t o = sub0; o < sub1; o++) {
      if (sync_ok(p, w, o)) { hyp = o; break; }
    }
    if (hyp != kNone) lane_walk(p, w, t0, hyp, sub1, roff_lane, cnt, exit, fail, fail_off);
    // tile hypothesis: first lane's sync point
    uint32_t hmask = __ballot_sync(0xffffffffu, hyp != kNone);
    uint64_t S = hmask ? __shfl_sync(0xffffffffu, hyp, __ffs(hmask) - 1) : kNone;
    if (S != kNone) warp_verify(p, w, t0, sub1, roff_lane, S, hyp, cnt, exit, fail, fail_off);

    // ---- look-back: true entry, record base, previous ts
    Look L;
    if (j == 0) {
      L.entry = 16; L.base = 0; L.prev_ts = 0; L.has_prev = false;
    } else {
      // publish the speculation
      uint32_t n_spec = __reduce_add_sync(0xffffffffu, cnt);
      uint64_t x31 = __shfl_sync(0xffffffffu, exit, 31);
      // last record under the speculation
      uint32_t lastmask = __ballot_sync(0xffffffffu, cnt > 0);
      uint64_t spec_last = 0;
      if (lastmask) {
        int ll = 31 - __clz(lastmask);
        uint64_t lo = 0;
        if ((int)lane == ll) lo = rd64(w, t0 + roff_lane[cnt - 1] + 4);
        spec_last = __shfl_sync(0xffffffffu, lo, ll);
      }
      bool spec_failed = __any_sync(0xffffffffu, fail && exit == kNone && hyp != kNone);
      if (lane == 0) {
        TileState* st = &p.state[g];
        st->spec_entry = S;
        st->exit = (S == kNone) ? kNone : (spec_failed ? kNone : x31);
        st->n_local = S == kNone ? 0 : n_spec;
        st->last_ts = spec_last;
        publish(st, p.epoch, TS_SPEC);
        L = lookback(p, done, g0, g, size);
      }
      L.entry = __shfl_sync(0xffffffffu, L.entry, 0);
      L.base = __shfl_sync(0xffffffffu, L.base, 0);
      L.prev_ts = __shfl_sync(0xffffffffu, L.prev_ts, 0);
      L.has_prev = __shfl_sync(0xffffffffu, L.has_prev, 0);
      if (L.entry == kNone) {  // the stream died in an earlier tile
        if (lane == 0) publish(&p.state[g], p.epoch, TS_ERROR);
        if (lane == 0) { p.state[g].pool_n_pending = 0; p.state[g].pool_n_resid = 0; }
        continue;
      }
      bool consistent = (S == kNone) ? (L.entry >= t1) : (L.entry == S);
      if (!consistent) {
        if (S == kNone) { hyp = kNone; cnt = 0; exit = kNone; fail = false; }
        warp_verify(p, w, t0, sub1, roff_lane, L.entry, hyp, cnt, exit, fail, fail_off);
      }
    }
    if (j == 0) {
      if (S != 16) warp_verify(p, w, t0, sub1, roff_lane, 16, hyp, cnt, exit, fail, fail_off);
    }
    // pass-through tile (entry beyond it) cannot fail and owns nothing
    if (L.entry >= t1) { cnt = 0; fail = false; exit = L.entry; }

    // ---- header-level failure: first failing lane whose walk started at its true entry
    uint64_t e_up = __shfl_up_sync(0xffffffffu, exit, 1);
    uint64_t e_in = lane == 0 ? L.entry : e_up;
    bool real_fail = fail && e_in != kNone && hyp == e_in;
    uint32_t fmask = __ballot_sync(0xffffffffu, real_fail);
    int fl = fmask ? __ffs(fmask) - 1 : 32;
    if ((int)lane > fl) cnt = 0;
    // inclusive count before each lane
    uint32_t incl = cnt;
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) { uint32_t v = __shfl_up_sync(0xffffffffu, incl, d); if ((int)lane >= d) incl += v; }
    const uint32_t n_rec = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t lane_base = incl - cnt;
    // compact record offsets into tile order
    uint16_t tmp[kMaxRecLane];
    #pragma unroll
    for (int k = 0; k < kMaxRecLane; k++) tmp[k] = (k < (int)cnt) ? roff_lane[k] : 0;
    __syncwarp();
    #pragma unroll
    for (int k = 0; k < kMaxRecLane; k++) if (k < (int)cnt) ws->roff[lane_base + k] = tmp[k];
    __syncwarp();
    uint64_t tile_last_ts = 0;
    if (n_rec) {
      uint64_t v = 0;
      if (lane == 0) v = rd64(w, t0 + ws->roff[n_rec - 1] + 4);
      tile_last_ts = __shfl_sync(0xffffffffu, v, 0);
    }
    uint64_t true_exit = __shfl_sync(0xffffffffu, exit, 31);
    if (lane == 0) {
      DoneState* d = &done[g];
      d->exit = true_exit;
      d->incl = L.base + n_rec;
      d->last_ts = n_rec ? tile_last_ts : L.prev_ts;
      d->has_last = (n_rec || L.has_prev) ? 1u : 0u;
    }
    uint64_t ffo = __shfl_sync(0xffffffffu, fail_off, fl < 32 ? fl : 0);
    if (lane == 0) {
      if (fmask) {
        uint32_t code;
        uint64_t aux = 0;
        uint64_t ts_f = 0;
        if (ffo + 16 > size) code = HG_ERR_TRUNC_HEADER;
        else {
          uint32_t sid = rd32(w, ffo);
          uint32_t plen = rd32(w, ffo + 12);
          ts_f = rd64(w, ffo + 4);
          if (ffo + 16 + plen > size) code = HG_ERR_TRUNC_PAYLOAD;
          else { code = HG_ERR_UNKNOWN_SCHEMA; aux = sid; }
        }
        uint64_t prev = n_rec ? tile_last_ts : L.prev_ts;
        push_error(p, code, s, L.base + n_rec, ffo, ts_f, prev, aux);
        publish(&p.state[g], p.epoch, TS_ERROR);
      } else {
        publish(&p.state[g], p.epoch, TS_DONE);
      }
    }

    // ---- passes B + C: decode 32 records per round, run the stack automaton
    uint32_t n_pend = 0, top = 0;   // elems[0, n_pend) pending exits, [n_pend, top) stack
    uint64_t prev_round_ts = L.prev_ts;
    bool have_prev = L.has_prev;
    bool cut = false;
    uint32_t feed_done = 0, dec_done = 0;
    uint32_t tile_spans = 0;
    for (uint32_t rb = 0; rb < n_rec && !cut; rb += kWarp) {
      const uint32_t r = rb + lane;
      const bool act = r < n_rec;
      RecOut ro;
      ro.kind = RK_NONE; ro.dec_err = 0; ro.feed_err = 0; ro.flags = 0; ro.ts = 0; ro.fn = -1; ro.result = 0;
      uint64_t off = 0;
      uint32_t dsp = 0;
      if (act) {
        off = t0 + ws->roff[r];
        decode_record(p, w, off, s, ro, dsp, st_samples, st_passed);
      }
      // monotonicity (pipeline.py:98-99): against the previous record of the stream
      uint64_t up_ts = __shfl_up_sync(0xffffffffu, ro.ts, 1);
      bool has_p = lane == 0 ? have_prev : true;
      uint64_t pts = lane == 0 ? prev_round_ts : up_ts;
      if (act && ro.dec_err == 0 && has_p && ro.ts < pts) ro.dec_err = HG_ERR_ORDER;
      // first decode-level error in the round cuts the stream
      uint32_t dm = __ballot_sync(0xffffffffu, act && ro.dec_err != 0);
      int dl = dm ? __ffs(dm) - 1 : 32;
      if (dm) {
        cut = true;
        if ((int)lane == dl && !dec_done) {
          push_error(p, ro.dec_err, s, L.base + r, off, ro.ts, has_p ? pts : 0, ro.dec_aux);
        }
        dec_done = 1;
      }
      bool live = act && (int)lane < dl;
      if (live) {
        st_events++;
        st_dev += dsp;
        if (ro.ts > my_last_ts) my_last_ts = ro.ts;
      }
      tile_spans += __reduce_add_sync(0xffffffffu, live ? dsp : 0u);
      prev_round_ts = __shfl_sync(0xffffffffu, ro.ts, 31);
      if (n_rec - rb < 32) prev_round_ts = __shfl_sync(0xffffffffu, ro.ts, (n_rec - rb - 1) & 31);
      have_prev = true;

      // ---- stack automaton over this round (pipeline.py:156-185)
      const bool isE = live && ro.kind == RK_ENTRY;
      const bool isX = live && ro.kind == RK_EXIT;
      uint32_t unres = __ballot_sync(0xffffffffu, isE || isX);
      const uint32_t Emask = __ballot_sync(0xffffffffu, isE);
      bool paired = false, orphan = false, me_unres = isE || isX;
      uint64_t entry_ts = 0;
      for (int it = 0; it < kWarp; it++) {
        uint32_t pm = unres & lanemask_lt();
        int pred = pm ? 31 - __clz(pm) : 0;
        int32_t pfn = __shfl_sync(0xffffffffu, ro.fn, pred);
        uint64_t pts2 = __shfl_sync(0xffffffffu, ro.ts, pred);
        bool act2 = isX && me_unres && pm && ((Emask >> pred) & 1u);
        bool m = act2 && pfn == ro.fn;
        bool o = act2 && pfn != ro.fn;
        uint32_t Mx = __ballot_sync(0xffffffffu, m);
        uint32_t Ox = __ballot_sync(0xffffffffu, o);
        if (!(Mx | Ox)) break;
        // entries claimed by a matching exit: the next unresolved element after them
        uint32_t nm = unres & lanemask_gt();
        int succ = nm ? __ffs(nm) - 1 : 0;
        bool claimed = isE && me_unres && nm && ((Mx >> succ) & 1u);
        uint32_t Ce = __ballot_sync(0xffffffffu, claimed);
        if (m) { paired = true; entry_ts = pts2; me_unres = false; }
        if (o) { orphan = true; me_unres = false; }
        if (claimed) me_unres = false;
        unres &= ~(Mx | Ox | Ce);
      }
      // remaining: X* E*.  Resolve the leading exits against the tile stack.
      uint32_t Xs = __ballot_sync(0xffffffffu, isX && me_unres);
      while (Xs) {
        int jx = __ffs(Xs) - 1;
        int32_t fj = __shfl_sync(0xffffffffu, ro.fn, jx);
        if (top > n_pend) {
          Elem tp = ws->elems[top - 1];
          if (tp.fn == fj) {
            if ((int)lane == jx) { paired = true; entry_ts = tp.ts; }
            top--;
          } else if ((int)lane == jx) {
            orphan = true;
          }
        } else {
          // empty tile stack: pending until composed with the preceding tiles
          if ((int)lane == jx) {
            Elem e; e.ts = ro.ts; e.result = ro.result; e.fn = ro.fn; e.seq = (uint16_t)r;
            e.flags = (uint16_t)(1u | (ro.flags & 6u));
            ws->elems[n_pend] = e;
          }
          n_pend++; top++;
        }
        __syncwarp();
        Xs &= Xs - 1;
      }
      // push the round's unresolved entries
      uint32_t Es = __ballot_sync(0xffffffffu, isE && me_unres);
      if (isE && me_unres) {
        Elem e; e.ts = ro.ts; e.result = 0; e.fn = ro.fn; e.seq = (uint16_t)r; e.flags = 0;
        ws->elems[top + __popc(Es & lanemask_lt())] = e;
      }
      top += __popc(Es);
      __syncwarp();
      // interval-stage errors (first per tile): device/telemetry feed errors, and
      // NaN/inf f64 results, which only raise when the exit pairs (pipeline.py:169-183)
      bool bad_res = paired && (ro.flags & 4u);
      uint32_t fm = __ballot_sync(0xffffffffu, (live && ro.feed_err != 0) || bad_res);
      if (fm && !feed_done) {
        if ((int)lane == __ffs(fm) - 1) {
          if (bad_res) push_error(p, HG_ERR_RESULT, s, L.base + r, off, ro.ts, 0, ro.result);
          else push_error(p, ro.feed_err, s, L.base + r, off, ro.ts, 0, ro.feed_aux);
        }
        feed_done = 1;
      }
      fold_host_round(p, tab, paired, ro.fn, ro.ts - entry_ts, (ro.flags & 2u) != 0);
      if (paired) st_host++;
      tile_spans += __popc(__ballot_sync(0xffffffffu, paired));
      push_orphans(p, orphan, s, ro.fn, ro.ts, L.base + r);
      if (orphan) st_orph++;
    }

    // ---- tile summary for the composition pass
    if (lane == 0) {
      unsigned long long off = top ? atomicAdd(p.pool_used, (unsigned long long)top) : 0ull;
      p.state[g].pool_off = off;
      p.state[g].pool_n_pending = n_pend;
      p.state[g].pool_n_resid = top - n_pend;
      if (tile_spans) atomicAdd(&p.stream_spans[s], (unsigned long long)tile_spans);
    }
    unsigned long long poff = 0;
    if (lane == 0) poff = p.state[g].pool_off;
    poff = __shfl_sync(0xffffffffu, poff, 0);
    __syncwarp();
    for (uint32_t i = lane; i < top; i += kWarp) {
      if (poff + i < p.pool_cap) {
        Elem e = ws->elems[i];
        SumEntry o;
        o.ts = e.ts; o.seq = L.base + e.seq; o.fn = e.fn; o.flags = e.flags; o.result = e.result;
        p.pool[poff + i] = o;
      }
    }
    __syncwarp();
  }

  // ---- flush per-lane statistics
  auto wsum = [](uint32_t v) { return __reduce_add_sync(0xffffffffu, v); };
  uint32_t a0 = wsum(st_events), a1 = wsum(st_passed), a2 = wsum(st_host), a3 = wsum(st_dev), a4 = wsum(st_samples),
           a5 = wsum(st_orph);
  uint64_t mts = my_last_ts;
  #pragma unroll
  for (int d = 16; d; d >>= 1) { uint64_t v = __shfl_xor_sync(0xffffffffu, mts, d); mts = v > mts ? v : mts; }
  if (lane == 0) {
    if (a0) atomicAdd(&p.stats[ST_EVENTS], (unsigned long long)a0);
    if (a1) atomicAdd(&p.stats[ST_PASSED], (unsigned long long)a1);
    if (a2) atomicAdd(&p.stats[ST_HOST], (unsigned long long)a2);
    if (a3) atomicAdd(&p.stats[ST_DEVICE], (unsigned long long)a3);
    if (a4) atomicAdd(&p.stats[ST_SAMPLES], (unsigned long long)a4);
    if (a5) atomicAdd(&p.stats[ST_ORPHANS], (unsigned long long)a5);
    atomicMax(p.last_ts, (unsigned long long)mts);
  }
  // ---- flush the CTA host table
  __syncthreads();
  if (tab) {
    for (uint32_t f = threadIdx.x; f < p.n_fn; f += blockDim.x) {
      SmemRow r = tab[f];
      if (!r.count) continue;
      unsigned long long* a = p.host_acc + 6ull * f;
      atomicAdd(&a[0], (unsigned long long)r.count);
      if (r.err) atomicAdd(&a[1], (unsigned long long)r.err);
      uint64_t lo = (uint64_t)r.s0 | ((uint64_t)r.s1 << 32);
      add_i128(&a[2], &a[3], lo, (int64_t)r.s2);
      atomicMin(&a[4], r.mn);
      atomicMax(&a[5], r.mx);
    }
  }
}

// ---------------------------------------------------------------------------
// composition of tile summaries per stream (exact automaton from an empty stack)

__global__ void compose_kernel(Params p) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p.n_streams) return;
  const uint32_t g0 = p.stream_tile0[s];
  const uint32_t g1 = (s + 1 < p.n_streams) ? p.stream_tile0[s + 1] : p.n_tiles;
  uint64_t need = 0;
  uint32_t gend = g1;
  for (uint32_t g = g0; g < g1; g++) {
    need += p.state[g].pool_n_resid;
    if ((p.state[g].status & 3u) == TS_ERROR) { gend = g + 1; break; }
  }
  unsigned long long sbase = need ? atomicAdd(p.stack_used, (unsigned long long)need) : 0ull;
  if (sbase + need > p.stack_cap) return;  // host detects via stack_used
  SumEntry* st = p.stack_scratch + sbase;
  uint64_t top = 0;
  uint32_t host = 0, orph = 0, trunc = 0, spans = 0;
  for (uint32_t g = g0; g < gend; g++) {
    const TileState& ts = p.state[g];
    const SumEntry* e = p.pool + ts.pool_off;
    uint32_t np = ts.pool_n_pending, nr = ts.pool_n_resid;
    if (ts.pool_off + np + nr > p.pool_cap) return;
    for (uint32_t i = 0; i < np; i++) {
      SumEntry x = e[i];
      if (top && st[top - 1].fn == x.fn) {
        SumEntry en = st[--top];
        if (x.flags & 4u) push_error(p, HG_ERR_RESULT, s, x.seq, 0, x.ts, 0, x.result);
        uint64_t dur = x.ts - en.ts;
        unsigned long long* a = p.host_acc + 6ull * x.fn;
        atomicAdd(&a[0], 1ull);
        if (x.flags & 2u) atomicAdd(&a[1], 1ull);
        add_i128(&a[2], &a[3], dur, 0);
        atomicMin(&a[4], dur);
        atomicMax(&a[5], dur);
        host++; spans++;
      } else {
        unsigned long long k = atomicAdd(p.n_orphans, 1ull);
        if (k < p.orphan_cap) { hg_orphan o; o.stream = s; o.function = x.fn; o.ts = x.ts; o.seq = x.seq; p.orphans[k] = o; }
        orph++;
      }
    }
    for (uint32_t i = 0; i < nr; i++) st[top++] = e[np + i];
  }
  // truncated spans at the global last timestamp, innermost first (pipeline.py:220-240)
  while (top) {
    SumEntry en = st[--top];
    uint64_t dur = p.global_last_ts - en.ts;
    unsigned long long* a = p.host_acc + 6ull * en.fn;
    atomicAdd(&a[0], 1ull);
    add_i128(&a[2], &a[3], dur, 0);
    atomicMin(&a[4], dur);
    atomicMax(&a[5], dur);
    trunc++; spans++;
  }
  if (host) atomicAdd(&p.stats[ST_HOST], (unsigned long long)host);
  if (orph) atomicAdd(&p.stats[ST_ORPHANS], (unsigned long long)orph);
  if (trunc) atomicAdd(&p.stats[ST_TRUNC], (unsigned long long)trunc);
  if (spans) atomicAdd(&p.stream_spans[s], (unsigned long long)spans);
}

__global__ void init_acc_kernel(unsigned long long* host_acc, uint32_t n_fn, unsigned long long* dev_acc, uint32_t n_dev) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_fn) {
    unsigned long long* a = host_acc + 6ull * i;
    a[0] = a[1] = a[2] = a[3] = 0; a[4] = ~0ull; a[5] = 0;
  }
  if (i < n_dev) {
    unsigned long long* a = dev_acc + 6ull * i;
    a[0] = a[1] = a[2] = a[3] = 0; a[4] = ~0ull; a[5] = 0;
  }
}

}  // namespace

// ===========================================================================
// host side: the C ABI (include/hapigpu.h)

namespace {

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

struct HostStream {
  std::string host;
  int64_t pid, tid;
  const uint8_t* data;
  uint64_t size;
};

}  // namespace

struct hg_ctx {
  hg_config cfg{};
  std::string err;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};
  int sm_count = 0;
  // registry
  std::vector<DSchema> schemas;
  std::vector<int32_t> sid_map;
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
  std::vector<uint32_t> tile_stream, stream_tile0, order;
  DBuf<uint32_t> d_tile_stream, d_stream_tile0, d_order;
  // scratch
  DBuf<TileState> d_state;
  DBuf<DoneState> d_done;
  uint32_t epoch = 0;
  DBuf<SumEntry> d_pool, d_stack;
  uint64_t pool_cap = 0, stack_cap = 0;
  DBuf<unsigned long long> d_host_acc, d_dev_acc;
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
  std::vector<unsigned long long> host_acc, dev_acc;
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
  C_NUM = 19
};

static int fail(hg_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail(ctx, HG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

extern "C" {

int hg_abi_version(void) { return HG_ABI_VERSION; }

const char* hg_last_error(hg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int hg_create(const hg_config* cfg, hg_ctx** out) {
  if (!out) return HG_EARG;
  hg_ctx* ctx = new hg_ctx();
  if (cfg) ctx->cfg = *cfg;
  *out = ctx;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(ctx, HG_ECUDA, "no CUDA device available");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  for (auto& ev : ctx->ev) CK(cudaEventCreate(&ev));
  CK(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
  return HG_OK;
}

void hg_destroy(hg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->d_schemas.release(); ctx->d_sid_map.release(); ctx->d_kinds.release(); ctx->d_field_role.release();
  ctx->d_data.release(); ctx->d_base.release(); ctx->d_size.release();
  ctx->d_tile_stream.release(); ctx->d_stream_tile0.release(); ctx->d_order.release();
  ctx->d_state.release(); ctx->d_done.release(); ctx->d_pool.release(); ctx->d_stack.release();
  ctx->d_host_acc.release(); ctx->d_dev_acc.release(); ctx->d_counters.release();
  ctx->d_orphans.release(); ctx->d_errors.release(); ctx->d_stream_spans.release();
  ctx->d_keys.release(); ctx->d_vals.release(); ctx->d_name_len.release(); ctx->d_small.release();
  ctx->d_name_off.release(); ctx->d_arena.release();
  for (auto& ev : ctx->ev) if (ev) cudaEventDestroy(ev);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int hg_set_registry(hg_ctx* ctx, const hg_schema* schemas, uint32_t n_schemas, const uint8_t* kinds, uint32_t n_kinds,
                    uint32_t n_functions) {
  if (!ctx || (n_schemas && !schemas)) return HG_EARG;
  uint32_t max_sid = 0;
  for (uint32_t i = 0; i < n_schemas; i++) max_sid = std::max(max_sid, schemas[i].id);
  if (n_schemas && max_sid > (1u << 24)) return fail(ctx, HG_EUNSUPPORTED, "schema ids above 2^24 are not supported");
  ctx->schemas.clear();
  ctx->sid_map.assign(n_schemas ? max_sid + 1 : 1, -1);
  ctx->kinds.assign(kinds, kinds + n_kinds);
  ctx->field_role.assign(n_kinds, 0xff);
  for (uint32_t i = 0; i < n_schemas; i++) {
    const hg_schema& h = schemas[i];
    DSchema d{};
    d.kinds_off = h.kinds_offset;
    d.fn = h.function;
    d.cls = h.event_class;
    d.nfields = h.n_fields;
    d.counter_kind = h.counter_kind;
    uint32_t fixed = 0, minlen = 0;
    bool var = false;
    for (uint32_t f = 0; f < h.n_fields; f++) {
      uint8_t k = kinds[h.kinds_offset + f];
      if (k >= HG_KIND_STRING) { var = true; minlen += 4; } else { fixed += 8; minlen += 8; }
    }
    if ((var ? minlen : fixed) > 0xffff) return fail(ctx, HG_EUNSUPPORTED, "schema payload too large");
    d.fixed_len = (uint16_t)(var ? minlen : fixed);
    d.flags = var ? SF_VAR : 0;
    for (int r = 0; r < HG_NUM_ROLES; r++) {
      d.role[r] = (int8_t)(h.role[r] > 127 ? -1 : h.role[r]);
      d.role_kind[r] = h.role[r] >= 0 ? kinds[h.kinds_offset + h.role[r]] : 0xff;
      if (h.role[r] >= 0) ctx->field_role[h.kinds_offset + h.role[r]] = (uint8_t)r;
    }
    if (h.event_class == HG_CLASS_EXIT && h.role[HG_ROLE_RESULT] >= 0) {
      d.flags |= SF_RESULT;
      if (d.role_kind[HG_ROLE_RESULT] == HG_KIND_F64) d.flags |= SF_RESULT_F64;
    }
    if (h.feed_error == 1) d.flags |= SF_FEED_ALWAYS;
    if (h.feed_error == 2) d.flags |= SF_FEED_TIMELINE;
    ctx->sid_map[h.id] = (int32_t)ctx->schemas.size();
    ctx->schemas.push_back(d);
  }
  ctx->n_fn = n_functions;
  ctx->max_sid = n_schemas ? max_sid : 0;
  cudaSetDevice(ctx->cfg.device);
  CK(ctx->d_schemas.ensure(std::max<size_t>(ctx->schemas.size(), 1)));
  CK(ctx->d_sid_map.ensure(ctx->sid_map.size()));
  CK(ctx->d_kinds.ensure(std::max<size_t>(n_kinds, 1)));
  CK(ctx->d_field_role.ensure(std::max<size_t>(n_kinds, 1)));
  if (!ctx->schemas.empty())
    CK(cudaMemcpy(ctx->d_schemas.ptr, ctx->schemas.data(), ctx->schemas.size() * sizeof(DSchema), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_sid_map.ptr, ctx->sid_map.data(), ctx->sid_map.size() * 4, cudaMemcpyHostToDevice));
  if (n_kinds) {
    CK(cudaMemcpy(ctx->d_kinds.ptr, kinds, n_kinds, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_field_role.ptr, ctx->field_role.data(), n_kinds, cudaMemcpyHostToDevice));
  }
  ctx->have_results = false;
  return HG_OK;
}

int hg_add_stream(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid, const void* data, uint64_t size) {
  if (!ctx || (size && !data)) return HG_EARG;
  ctx->streams.push_back(HostStream{hostname ? hostname : "", pid, tid, (const uint8_t*)data, size});
  ctx->staged = false;
  ctx->have_results = false;
  return HG_OK;
}

int hg_clear_streams(hg_ctx* ctx) {
  if (!ctx) return HG_EARG;
  ctx->streams.clear();
  ctx->staged = false;
  ctx->have_results = false;
  return HG_OK;
}

static int build_layout(hg_ctx* ctx) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  ctx->base.resize(ns);
  ctx->sizes.resize(ns);
  uint64_t off = 0;
  for (uint32_t s = 0; s < ns; s++) {
    ctx->base[s] = off;
    ctx->sizes[s] = ctx->streams[s].size;
    off += (ctx->streams[s].size + 255) & ~255ull;
  }
  ctx->total_bytes = off;
  // tiles
  ctx->tile_stream.clear();
  ctx->stream_tile0.assign(ns, 0);
  std::vector<uint32_t> ntiles(ns, 0);
  uint32_t maxt = 0;
  for (uint32_t s = 0; s < ns; s++) {
    ctx->stream_tile0[s] = (uint32_t)ctx->tile_stream.size();
    uint64_t sz = ctx->sizes[s];
    uint32_t nt = sz > 16 ? (uint32_t)((sz - 16 + kTile - 1) / kTile) : 0;
    ntiles[s] = nt;
    maxt = std::max(maxt, nt);
    for (uint32_t t = 0; t < nt; t++) ctx->tile_stream.push_back(s);
  }
  // processing order: tile index major, streams interleaved (predecessors finish early)
  ctx->order.clear();
  ctx->order.reserve(ctx->tile_stream.size());
  for (uint32_t t = 0; t < maxt; t++)
    for (uint32_t s = 0; s < ns; s++)
      if (t < ntiles[s]) ctx->order.push_back(ctx->stream_tile0[s] + t);
  return HG_OK;
}

static int stage(hg_ctx* ctx) {
  cudaSetDevice(ctx->cfg.device);
  build_layout(ctx);
  const uint32_t ns = (uint32_t)ctx->streams.size();
  const size_t pad = kWinBytes + 4096;
  CK(ctx->d_data.ensure(ctx->total_bytes + pad));
  CK(cudaMemsetAsync(ctx->d_data.ptr + ctx->total_bytes, 0, pad, ctx->stream));
  ctx->h2d_bytes = 0;
  for (uint32_t s = 0; s < ns; s++) {
    if (!ctx->streams[s].size) continue;
    CK(cudaMemcpyAsync(ctx->d_data.ptr + ctx->base[s], ctx->streams[s].data, ctx->streams[s].size, cudaMemcpyHostToDevice,
                       ctx->stream));
    ctx->h2d_bytes += ctx->streams[s].size;
  }
  CK(ctx->d_base.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_size.ensure(std::max<uint32_t>(ns, 1)));
  if (ns) {
    CK(cudaMemcpyAsync(ctx->d_base.ptr, ctx->base.data(), ns * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_size.ptr, ctx->sizes.data(), ns * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  size_t nt = ctx->tile_stream.size();
  CK(ctx->d_tile_stream.ensure(std::max<size_t>(nt, 1)));
  CK(ctx->d_order.ensure(std::max<size_t>(nt, 1)));
  CK(ctx->d_stream_tile0.ensure(std::max<uint32_t>(ns, 1)));
  if (nt) {
    CK(cudaMemcpyAsync(ctx->d_tile_stream.ptr, ctx->tile_stream.data(), nt * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_order.ptr, ctx->order.data(), nt * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ns) CK(cudaMemcpyAsync(ctx->d_stream_tile0.ptr, ctx->stream_tile0.data(), ns * 4, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->d_state.n < nt) {
    CK(ctx->d_state.ensure(nt));
    CK(cudaMemsetAsync(ctx->d_state.ptr, 0, nt * sizeof(TileState), ctx->stream));
    ctx->epoch = 0;
  }
  CK(ctx->d_done.ensure(std::max<size_t>(nt, 1)));
  ctx->staged = true;
  return HG_OK;
}

int hg_stage(hg_ctx* ctx) {
  if (!ctx) return HG_EARG;
  int rc = stage(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return HG_OK;
}

static size_t tile_smem_bytes(uint32_t n_fn) {
  size_t tab = n_fn <= kSmemFnMax ? ((sizeof(SmemRow) * n_fn + 127) / 128) * 128 : 0;
  return tab + sizeof(WarpSmem) * kWarpsPerCta;
}

static int ensure_scratch(hg_ctx* ctx, uint64_t n_records_bound) {
  const size_t nt = ctx->tile_stream.size();
  const uint32_t ns = (uint32_t)ctx->streams.size();
  if (ctx->pool_cap == 0) ctx->pool_cap = std::max<uint64_t>(1 << 20, nt * 16);
  if (ctx->stack_cap == 0) ctx->stack_cap = ctx->pool_cap;
  if (ctx->orphan_cap == 0) ctx->orphan_cap = 1 << 16;
  if (ctx->error_cap == 0) ctx->error_cap = (uint32_t)std::max<size_t>(4096, 2 * nt + 16);
  if (ctx->row_cap == 0) {
    ctx->row_cap = 1 << 14;
    ctx->dict_mask = (1 << 16) - 1;
    ctx->arena_cap = 1 << 22;
  }
  (void)n_records_bound;
  CK(ctx->d_pool.ensure(ctx->pool_cap));
  CK(ctx->d_stack.ensure(ctx->stack_cap));
  CK(ctx->d_orphans.ensure(ctx->orphan_cap));
  CK(ctx->d_errors.ensure(ctx->error_cap));
  CK(ctx->d_host_acc.ensure(6ull * std::max<uint32_t>(ctx->n_fn, 1)));
  CK(ctx->d_dev_acc.ensure(6ull * ctx->row_cap));
  CK(ctx->d_counters.ensure(C_NUM));
  CK(ctx->d_stream_spans.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_keys.ensure(ctx->dict_mask + 1));
  CK(ctx->d_vals.ensure(ctx->dict_mask + 1));
  CK(ctx->d_name_len.ensure(ctx->row_cap));
  CK(ctx->d_name_off.ensure(ctx->row_cap));
  CK(ctx->d_arena.ensure(ctx->arena_cap));
  return HG_OK;
}

static Params make_params(hg_ctx* ctx) {
  Params p{};
  p.data = ctx->d_data.ptr;
  p.stream_base = ctx->d_base.ptr;
  p.stream_size = ctx->d_size.ptr;
  p.tile_stream = ctx->d_tile_stream.ptr;
  p.stream_tile0 = ctx->d_stream_tile0.ptr;
  p.order = ctx->d_order.ptr;
  p.n_tiles = (uint32_t)ctx->tile_stream.size();
  p.n_streams = (uint32_t)ctx->streams.size();
  p.schemas = ctx->d_schemas.ptr;
  p.sid_map = ctx->d_sid_map.ptr;
  p.max_sid = ctx->max_sid;
  p.kinds = ctx->d_kinds.ptr;
  p.field_role = ctx->d_field_role.ptr;
  p.n_fn = ctx->n_fn;
  p.state = ctx->d_state.ptr;
  p.epoch = ctx->epoch;
  p.pool = ctx->d_pool.ptr;
  unsigned long long* C = ctx->d_counters.ptr;
  p.pool_used = C + C_POOL_USED;
  p.pool_cap = ctx->pool_cap;
  p.host_acc = ctx->d_host_acc.ptr;
  p.dev_acc = ctx->d_dev_acc.ptr;
  p.wide_flag = reinterpret_cast<uint32_t*>(C + C_WIDE);
  p.names.keys = ctx->d_keys.ptr;
  p.names.vals = ctx->d_vals.ptr;
  p.names.mask = ctx->dict_mask;
  p.names.arena = ctx->d_arena.ptr;
  p.names.arena_used = C + C_ARENA_USED;
  p.names.arena_cap = ctx->arena_cap;
  p.names.name_off = ctx->d_name_off.ptr;
  p.names.name_len = ctx->d_name_len.ptr;
  p.names.n_rows = reinterpret_cast<uint32_t*>(C + C_N_ROWS);
  p.names.row_cap = ctx->row_cap;
  p.names.overflow = reinterpret_cast<uint32_t*>(C + C_OVERFLOW);
  p.orphans = ctx->d_orphans.ptr;
  p.n_orphans = C + C_N_ORPHANS;
  p.orphan_cap = ctx->orphan_cap;
  p.errors = ctx->d_errors.ptr;
  p.n_errors = reinterpret_cast<unsigned int*>(C + C_N_ERRORS);
  p.error_cap = ctx->error_cap;
  p.stats = C + C_STATS;
  p.last_ts = C + C_LAST_TS;
  p.stream_spans = ctx->d_stream_spans.ptr;
  p.work_counter = reinterpret_cast<unsigned int*>(C + C_WORK);
  p.watchdog = reinterpret_cast<uint32_t*>(C + C_WATCHDOG);
  p.want = ctx->want;
  p.stack_scratch = ctx->d_stack.ptr;
  p.stack_used = C + C_STACK_USED;
  p.stack_cap = ctx->stack_cap;
  return p;
}

static int launch_phase1(hg_ctx* ctx) {
  const uint32_t nt = (uint32_t)ctx->tile_stream.size();
  const uint32_t ns = (uint32_t)ctx->streams.size();
  ctx->epoch++;
  if (ctx->epoch >= (1u << 29)) {
    CK(cudaMemsetAsync(ctx->d_state.ptr, 0, ctx->d_state.n * sizeof(TileState), ctx->stream));
    ctx->epoch = 1;
  }
  CK(cudaMemsetAsync(ctx->d_counters.ptr, 0, C_NUM * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_stream_spans.ptr, 0, std::max<uint32_t>(ns, 1) * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_keys.ptr, 0, (ctx->dict_mask + 1) * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_vals.ptr, 0, (ctx->dict_mask + 1) * 4, ctx->stream));
  uint32_t nmax = std::max(ctx->n_fn, ctx->row_cap);
  init_acc_kernel<<<(nmax + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_host_acc.ptr, ctx->n_fn, ctx->d_dev_acc.ptr,
                                                                ctx->row_cap);
  ctx->launches = 1;
  if (nt) {
    Params p = make_params(ctx);
    size_t smem = tile_smem_bytes(ctx->n_fn);
    CK(cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_kernel, kCtaThreads, smem));
    if (per_sm < 1) return fail(ctx, HG_ECUDA, "tile kernel does not fit on an SM");
    uint32_t grid = std::min<uint32_t>((uint32_t)(per_sm * ctx->sm_count), (nt + kWarpsPerCta - 1) / kWarpsPerCta);
    grid = std::max<uint32_t>(grid, 1);
    tile_kernel<<<grid, kCtaThreads, smem, ctx->stream>>>(p, ctx->d_done.ptr);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  return HG_OK;
}

static int read_counters(hg_ctx* ctx) {
  ctx->counters.resize(C_NUM);
  CK(cudaMemcpyAsync(ctx->counters.data(), ctx->d_counters.ptr, C_NUM * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return HG_OK;
}

int hg_run_local(hg_ctx* ctx, uint32_t want) {
  if (!ctx) return HG_EARG;
  cudaSetDevice(ctx->cfg.device);
  ctx->want = want;
  ctx->have_results = false;
  ctx->phase1_done = false;
  for (int attempt = 0; attempt < 6; attempt++) {
    CK(cudaEventRecord(ctx->ev[0], ctx->stream));
    uint64_t h2d = 0;
    if (!ctx->staged) {
      int rc = stage(ctx);
      if (rc) return rc;
      h2d = ctx->h2d_bytes;
    }
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    int rc = ensure_scratch(ctx, 0);
    if (rc) return rc;
    rc = launch_phase1(ctx);
    if (rc) return rc;
    rc = read_counters(ctx);
    if (rc) return rc;
    ctx->h2d_bytes = h2d;
    bool grow = false;
    unsigned long long* C = ctx->counters.data();
    if (C[C_POOL_USED] > ctx->pool_cap) { ctx->pool_cap = C[C_POOL_USED] + (C[C_POOL_USED] >> 2); ctx->stack_cap = ctx->pool_cap; grow = true; }
    if (C[C_N_ORPHANS] > ctx->orphan_cap) { ctx->orphan_cap = C[C_N_ORPHANS] * 2; grow = true; }
    if ((uint32_t)C[C_N_ERRORS] > ctx->error_cap) { ctx->error_cap = (uint32_t)C[C_N_ERRORS] * 2; grow = true; }
    if ((uint32_t)C[C_OVERFLOW]) {
      ctx->row_cap *= 4; ctx->dict_mask = ctx->dict_mask * 4 + 3; ctx->arena_cap = std::max<uint64_t>(ctx->arena_cap * 4, C[C_ARENA_USED] * 2);
      grow = true;
    }
    if (!grow) break;
    if (attempt == 5) return fail(ctx, HG_ENOMEM, "scratch buffers kept overflowing");
  }
  if ((uint32_t)ctx->counters[C_WATCHDOG])
    return fail(ctx, HG_ECUDA, "tile look-back watchdog fired (engine bug)");
  if ((uint32_t)ctx->counters[C_WIDE])
    return fail(ctx, HG_EUNSUPPORTED, "device span durations beyond the signed 64-bit range");
  ctx->local_last_ts = ctx->counters[C_LAST_TS];
  ctx->local_events = ctx->counters[C_STATS + ST_EVENTS];
  ctx->phase1_done = true;
  return HG_OK;
}

int hg_local_last_ts(hg_ctx* ctx, uint64_t* last_ts, uint64_t* n_events) {
  if (!ctx || !ctx->phase1_done) return HG_ESTATE;
  if (last_ts) *last_ts = ctx->local_last_ts;
  if (n_events) *n_events = ctx->local_events;
  return HG_OK;
}

int hg_finish(hg_ctx* ctx, uint64_t global_last_ts) {
  if (!ctx || !ctx->phase1_done) return HG_ESTATE;
  cudaSetDevice(ctx->cfg.device);
  const uint32_t ns = (uint32_t)ctx->streams.size();
  for (int attempt = 0; attempt < 3; attempt++) {
    if (ns) {
      Params p = make_params(ctx);
      p.global_last_ts = global_last_ts;
      unsigned long long zero = 0;
      CK(cudaMemcpyAsync(p.stack_used, &zero, 8, cudaMemcpyHostToDevice, ctx->stream));
      // the tally accumulators already hold phase-1 spans; compose adds the rest
      compose_kernel<<<(ns + 127) / 128, 128, 0, ctx->stream>>>(p);
      CK(cudaGetLastError());
      ctx->launches++;
    }
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    int rc = read_counters(ctx);
    if (rc) return rc;
    if (ctx->counters[C_STACK_USED] <= ctx->stack_cap && ctx->counters[C_N_ORPHANS] <= ctx->orphan_cap) break;
    return fail(ctx, HG_ENOMEM, "composition scratch overflow");  // TODO: rerun the whole pipeline with larger buffers
  }
  // results to the host
  unsigned long long* C = ctx->counters.data();
  ctx->n_dev_rows = (uint32_t)std::min<unsigned long long>(C[C_N_ROWS], ctx->row_cap);
  ctx->host_acc.resize(6ull * ctx->n_fn);
  ctx->dev_acc.resize(6ull * ctx->n_dev_rows);
  ctx->d2h_bytes = C_NUM * 8;
  if (ctx->n_fn) CK(cudaMemcpyAsync(ctx->host_acc.data(), ctx->d_host_acc.ptr, ctx->host_acc.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->n_dev_rows) CK(cudaMemcpyAsync(ctx->dev_acc.data(), ctx->d_dev_acc.ptr, ctx->dev_acc.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->name_off.resize(ctx->n_dev_rows);
  ctx->name_len.resize(ctx->n_dev_rows);
  uint64_t arena_used = std::min<uint64_t>(C[C_ARENA_USED], ctx->arena_cap);
  ctx->arena.resize(arena_used);
  if (ctx->n_dev_rows) {
    CK(cudaMemcpyAsync(ctx->name_off.data(), ctx->d_name_off.ptr, ctx->n_dev_rows * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->name_len.data(), ctx->d_name_len.ptr, ctx->n_dev_rows * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (arena_used) CK(cudaMemcpyAsync(ctx->arena.data(), ctx->d_arena.ptr, arena_used, cudaMemcpyDeviceToHost, ctx->stream));
  uint64_t n_orph = std::min<uint64_t>(C[C_N_ORPHANS], ctx->orphan_cap);
  ctx->orphans.resize(n_orph);
  if (n_orph) CK(cudaMemcpyAsync(ctx->orphans.data(), ctx->d_orphans.ptr, n_orph * sizeof(hg_orphan), cudaMemcpyDeviceToHost, ctx->stream));
  uint32_t n_err = (uint32_t)std::min<unsigned long long>((uint32_t)C[C_N_ERRORS], ctx->error_cap);
  ctx->errors.resize(n_err);
  if (n_err) CK(cudaMemcpyAsync(ctx->errors.data(), ctx->d_errors.ptr, n_err * sizeof(hg_trace_error), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->stream_spans.resize(ns);
  if (ns) CK(cudaMemcpyAsync(ctx->stream_spans.data(), ctx->d_stream_spans.ptr, ns * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->ev[3], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->d2h_bytes += ctx->host_acc.size() * 8 + ctx->dev_acc.size() * 8 + arena_used + n_orph * sizeof(hg_orphan) +
                    n_err * sizeof(hg_trace_error) + ns * 8 + ctx->n_dev_rows * 12;
  float k_ms = 0, t_ms = 0;
  cudaEventElapsedTime(&k_ms, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&t_ms, ctx->ev[0], ctx->ev[3]);
  ctx->kernel_ms = k_ms;
  ctx->total_ms = t_ms;
  ctx->have_results = true;
  return ctx->errors.empty() ? HG_OK : HG_TRACE_ERROR;
}

int hg_run(hg_ctx* ctx, uint32_t want) {
  int rc = hg_run_local(ctx, want);
  if (rc) return rc;
  return hg_finish(ctx, ctx->local_last_ts);
}

int hg_get_stats(hg_ctx* ctx, hg_stats* out) {
  if (!ctx || !out) return HG_EARG;
  if (!ctx->have_results) return HG_ESTATE;
  const unsigned long long* C = ctx->counters.data() + C_STATS;
  out->events_in = C[ST_EVENTS];
  out->passed = C[ST_PASSED];
  out->host_spans = C[ST_HOST];
  out->truncated_spans = C[ST_TRUNC];
  out->device_spans = C[ST_DEVICE];
  out->samples = C[ST_SAMPLES];
  out->orphan_exits = C[ST_ORPHANS];
  return HG_OK;
}

int hg_get_tally(hg_ctx* ctx, hg_tally_row* rows, uint64_t cap, uint64_t* n_rows) {
  if (!ctx || !n_rows) return HG_EARG;
  if (!ctx->have_results) return HG_ESTATE;
  uint64_t n = 0;
  for (uint32_t f = 0; f < ctx->n_fn; f++) {
    const unsigned long long* a = &ctx->host_acc[6ull * f];
    if (!a[0]) continue;
    if (rows && n < cap) {
      hg_tally_row& r = rows[n];
      r.section = 0; r.name_id = f; r.count = a[0]; r.error_count = a[1];
      r.time_lo = a[2]; r.time_hi = (int64_t)a[3];
      r.min_lo = a[4]; r.min_hi = 0; r.max_lo = a[5]; r.max_hi = 0;
    }
    n++;
  }
  for (uint32_t d = 0; d < ctx->n_dev_rows; d++) {
    const unsigned long long* a = &ctx->dev_acc[6ull * d];
    if (!a[0]) continue;
    if (rows && n < cap) {
      hg_tally_row& r = rows[n];
      r.section = 1; r.name_id = d; r.count = a[0]; r.error_count = a[1];
      r.time_lo = a[2]; r.time_hi = (int64_t)a[3];
      int64_t mn = (int64_t)(a[4] ^ 0x8000000000000000ull), mx = (int64_t)(a[5] ^ 0x8000000000000000ull);
      r.min_lo = (uint64_t)mn; r.min_hi = mn < 0 ? -1 : 0;
      r.max_lo = (uint64_t)mx; r.max_hi = mx < 0 ? -1 : 0;
    }
    n++;
  }
  *n_rows = n;
  return HG_OK;
}

int hg_get_device_names(hg_ctx* ctx, char* bytes, uint64_t cap, uint64_t* offsets, uint64_t n_offsets,
                        uint64_t* n_names, uint64_t* n_bytes) {
  if (!ctx) return HG_EARG;
  if (!ctx->have_results) return HG_ESTATE;
  uint64_t total = 0;
  for (uint32_t d = 0; d < ctx->n_dev_rows; d++) total += ctx->name_len[d];
  if (n_names) *n_names = ctx->n_dev_rows;
  if (n_bytes) *n_bytes = total;
  if (!bytes) return HG_OK;
  uint64_t o = 0;
  for (uint32_t d = 0; d < ctx->n_dev_rows; d++) {
    if (offsets && d < n_offsets) offsets[d] = o;
    uint32_t l = ctx->name_len[d];
    if (o + l <= cap) memcpy(bytes + o, ctx->arena.data() + ctx->name_off[d], l);
    o += l;
  }
  if (offsets && ctx->n_dev_rows < n_offsets) offsets[ctx->n_dev_rows] = o;
  return HG_OK;
}

int hg_get_stream_spans(hg_ctx* ctx, uint64_t* per_stream, uint64_t n) {
  if (!ctx || !per_stream) return HG_EARG;
  if (!ctx->have_results) return HG_ESTATE;
  for (uint64_t i = 0; i < n && i < ctx->stream_spans.size(); i++) per_stream[i] = ctx->stream_spans[i];
  return HG_OK;
}

int hg_get_orphans(hg_ctx* ctx, hg_orphan* out, uint64_t cap, uint64_t* n) {
  if (!ctx || !n) return HG_EARG;
  if (!ctx->have_results) return HG_ESTATE;
  *n = ctx->orphans.size();
  if (out) memcpy(out, ctx->orphans.data(), sizeof(hg_orphan) * std::min<uint64_t>(cap, ctx->orphans.size()));
  return HG_OK;
}

int hg_get_trace_errors(hg_ctx* ctx, hg_trace_error* out, uint64_t cap, uint64_t* n) {
  if (!ctx || !n) return HG_EARG;
  if (!ctx->have_results) return HG_ESTATE;
  *n = ctx->errors.size();
  if (out) memcpy(out, ctx->errors.data(), sizeof(hg_trace_error) * std::min<uint64_t>(cap, ctx->errors.size()));
  return HG_OK;
}

int hg_timeline_size(hg_ctx* ctx, uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return HG_EARG;
  return fail(ctx, HG_EUNSUPPORTED, "timeline export not built yet");
}

int hg_get_timeline(hg_ctx* ctx, char* out, uint64_t cap) {
  (void)out; (void)cap;
  return fail(ctx, HG_EUNSUPPORTED, "timeline export not built yet");
}

int hg_device_tally(hg_ctx* ctx, void** host_rows, uint64_t* n_host_rows) {
  if (!ctx) return HG_EARG;
  if (host_rows) *host_rows = ctx->d_host_acc.ptr;
  if (n_host_rows) *n_host_rows = ctx->n_fn;
  return HG_OK;
}

int hg_last_timing(hg_ctx* ctx, float* kernel_ms, float* total_ms, uint64_t* h2d_bytes, uint64_t* d2h_bytes,
                   uint64_t* kernel_launches) {
  if (!ctx) return HG_EARG;
  if (kernel_ms) *kernel_ms = ctx->kernel_ms;
  if (total_ms) *total_ms = ctx->total_ms;
  if (h2d_bytes) *h2d_bytes = ctx->h2d_bytes;
  if (d2h_bytes) *d2h_bytes = ctx->d2h_bytes;
  if (kernel_launches) *kernel_launches = ctx->launches;
  return HG_OK;
}

}  // extern "C"
