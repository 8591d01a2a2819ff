// kernels.cuh -- shared device building blocks of the hapigpu kernels (sm_100a).
//
// Launch parameters, the compact schema descriptors (screened from shared
// memory), error/orphan sinks, tally folding (per-lane columns, CTA tables,
// exact 128-bit global rows, CTA device-row cache), the exact LIFO automaton
// round used by compose_kernel (pipeline.py:156-168) and the generic payload
// field walk (tracefile.py:152-169).  Phase 1 lives in seg.cuh.
#pragma once
#include "hg_device.cuh"

namespace hg {

// dynamic shared memory of the tile kernel; every shared pointer is derived from this
// symbol in the function that uses it so accesses compile to LDS/STS
extern __shared__ __align__(128) uint8_t g_smem[];

constexpr uint32_t kSmallF = 16;               // per-lane tally columns up to this many functions
constexpr uint32_t kSmemFnMax = 2048;          // CTA-shared tally table up to this many functions
#ifndef HG_DEV_SLOTS
#define HG_DEV_SLOTS 64
#endif
constexpr int kDevSlots = HG_DEV_SLOTS;        // CTA cache of device rows
constexpr int kSdescMax = 512;                 // schema ids screened from shared memory

// function id field of packed stack metadata: fn (19 bits), M_FN = none
constexpr uint32_t M_FN = 0x7FFFFu;
__device__ __forceinline__ int32_t m_fn(uint32_t m) { return (m & M_FN) == M_FN ? -1 : (int32_t)(m & M_FN); }

struct SmemRow {   // CTA-shared host row (larger function sets); durations >= 2^32 go to global
  uint32_t count, err;
  uint32_t s0, s1;             // 64-bit sum
  uint32_t mn, mx;
};

struct DevRow {    // CTA-shared device row cache entry
  uint32_t tag;    // row + 1, 0 = free
  uint32_t count;
  uint32_t s0, s1, s2;          // 96-bit two's complement sum
  uint32_t mn, mx;              // biased signed 32-bit extrema (wider values go to global)
  uint32_t pad;
};

struct NameSlot {
  unsigned long long hash;
  uint32_t row;
  uint32_t pad;
};

enum Stat { ST_EVENTS = 0, ST_PASSED, ST_HOST, ST_TRUNC, ST_DEVICE, ST_SAMPLES, ST_ORPHANS, ST_N };

struct Params {
  const uint8_t* data;
  const uint64_t* stream_base;
  const uint64_t* stream_size;
  const uint32_t* tile_stream;    // stream-major tile id -> stream
  const uint32_t* stream_tile0;   // stream -> first stream-major tile id
  uint32_t n_tiles, n_streams;
  const DSchema* schemas;
  const int32_t* sid_map;
  const uint2* desc;              // compact per-sid descriptor (see make_desc)
  uint32_t max_sid;
  const uint8_t* kinds;
  const uint8_t* field_role;
  uint32_t n_fn;
  SegState* state;
  uint32_t epoch;
  SumEntry* pool;
  unsigned long long* pool_used;
  uint64_t pool_cap;
  unsigned long long* host_acc;   // n_fn x 6: count, err, sum_lo, sum_hi, min, max
  unsigned long long* dev_acc;    // row_cap x 6: count, err, sum_lo, sum_hi, min_b, max_b
  unsigned long long* dev_wide;   // row_cap x 6: lock, count, min lo/hi, max lo/hi of spans beyond +-2^63 ns
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
  uint32_t last_ts_dev;            // compose: the global last ts is *last_ts (one-rank fused run)
  // timeline messages (nullptr unless HG_WANT_TIMELINE): slots [0, tl_comp_base) are
  // indexed by global record number (segment decode), compose appends after them
  TlItem* tl_items;
  unsigned long long* tl_n;        // messages written by the segment decode
  unsigned long long* tl_n2;       // messages appended by compose
  uint64_t tl_comp_base;
  uint64_t tl_cap;
  const unsigned long long* tl_rec_off;  // per stream: global record number of its first record
  // timeline messages of the single pass (nullptr unless a timeline run takes it): range r's
  // messages in record order at tl_ritems[r * tl_rcap ...], their number in tl_rn[r], klo = the
  // record's index within the range (tl_range_compact makes it the mux key); tl_pres: result bits
  // of each range's first kRLP pending exits (compose's cross-range spans)
  TlItem* tl_ritems;
  uint32_t tl_rcap;
  uint32_t* tl_rn;
  unsigned long long* tl_pres;
  // every record of the single pass for event sinks (nullptr unless an event run takes it): range
  // r's records at ev_ritems[r * tl_rcap + k] (k: index in the range), ev_rn[r] of them
  TlItem* ev_ritems;
  uint32_t* ev_rn;
  // segments
  uint32_t seg_bytes;
  SumEntry* deep;                  // per-lane automaton chunks of deep segments
  unsigned long long* deep_used;
  uint64_t deep_cap;
  // single-pass range path (fast.cuh)
  const uint32_t* range_stream;    // range -> stream
  const uint32_t* stream_range0;   // stream -> first range
  uint32_t n_ranges;
  uint32_t range_bytes;
  struct RangeState* rstate;
  unsigned long long* range_base;  // record index of each range's first record (verify kernel)
  uint32_t* anom;                  // nonzero: the single-pass result is void, run the exact path
  const uint32_t* vplan;           // per schema id: single-var-field payload plan (fast.cuh)
  const uint4* fdesc;              // per schema id (+ one sentinel): inline-record descriptor (fast.cuh)
  const uint4* dplan;              // per schema id: device-record layout for the drain (fast.cuh)
  const uint32_t* flush_rank;      // stream -> rank in the truncation flush order (nullptr: stream order)
  uint32_t has_dev;                // the registry has device-profiling schemas (fast.cuh: CTA name cache)
  uint32_t prescan;                // range starts found by fast_scan_kernel (rstate[r].entry), not by each lane
};

// compact descriptor: x = fn(20) | cls(3)<<20 | flags(8)<<23 ; y = fixed_len(16) | result field index(8)<<16 | counter(8)<<24
__device__ __forceinline__ uint32_t d_fn(uint2 d) { return d.x & 0xFFFFFu; }
__device__ __forceinline__ uint32_t d_cls(uint2 d) { return (d.x >> 20) & 7u; }
__device__ __forceinline__ uint32_t d_flags(uint2 d) { return d.x >> 23; }
__device__ __forceinline__ uint32_t d_fixed(uint2 d) { return d.y & 0xFFFFu; }
__device__ __forceinline__ uint32_t d_resfield(uint2 d) { return (d.y >> 16) & 0xFFu; }
constexpr uint32_t D_PRESENT = 0x80000000u;  // stored in flags' top bit position of x

// compact descriptors live at the start of the tile kernel's shared memory when the
// registry's ids fit (kSdescMax); otherwise they are read through L1
__device__ __forceinline__ uint2 desc_of(const Params& p, uint32_t sid) {
  if (sid > p.max_sid) return make_uint2(0, 0);
  if (p.max_sid < (uint32_t)kSdescMax) return reinterpret_cast<const uint2*>(g_smem)[sid];
  return __ldg(&p.desc[sid]);
}
__device__ __forceinline__ bool d_present(uint2 d) { return (d.x & D_PRESENT) != 0; }

__device__ __forceinline__ const DSchema* schema_of(const Params& p, uint32_t sid) {
  if (sid > p.max_sid) return nullptr;
  int32_t si = __ldg(&p.sid_map[sid]);
  return si < 0 ? nullptr : &p.schemas[si];
}

// ---------------------------------------------------------------------------
// error / orphan sinks

static __device__ __noinline__ void push_error(const Params& p, uint32_t code, uint32_t stream, uint64_t seq, uint64_t off, uint64_t ts,
                           uint64_t prev_ts, uint64_t aux) {
  unsigned int i = atomicAdd(p.n_errors, 1u);
  if (i < p.error_cap) {
    hg_trace_error e;
    e.code = code; e.stream = stream; e.seq = seq; e.offset = off; e.ts = ts; e.prev_ts = prev_ts; e.aux = aux;
    p.errors[i] = e;
  }
}

static __device__ __noinline__ void push_orphan(const Params& p, uint32_t stream, int32_t fn, uint64_t ts, uint64_t seq) {
  unsigned long long i = atomicAdd(p.n_orphans, 1ull);
  if (i < p.orphan_cap) { hg_orphan o; o.stream = stream; o.function = fn; o.ts = ts; o.seq = seq; p.orphans[i] = o; }
}

// ---------------------------------------------------------------------------
// tally folding

// per-lane host columns for small function sets: [fn][lane] count and 64-bit sum
// (no atomics), per-warp error count and extrema (shared atomics, mostly skipped
// by a plain pre-check)
struct LaneTab {
  uint32_t* cnt; uint32_t* slo; uint32_t* shi;   // [fn * 32 + lane]
  uint32_t* err; uint32_t* mn; uint32_t* mx;     // [fn]
};

static __device__ __noinline__ void fold_host_global(const Params& p, int32_t fn, uint64_t dur, bool err) {
  unsigned long long* a = p.host_acc + 6ull * fn;
  atomicAdd(&a[0], 1ull);
  if (err) atomicAdd(&a[1], 1ull);
  add_i128(&a[2], &a[3], dur, 0);
  atomicMin(&a[4], dur);
  atomicMax(&a[5], dur);
}

__device__ __forceinline__ void smem_min_u64(unsigned long long* a, unsigned long long v) {
  if (v < *(volatile unsigned long long*)a) atomicMin(a, v);
}
__device__ __forceinline__ void smem_max_u64(unsigned long long* a, unsigned long long v) {
  if (v > *(volatile unsigned long long*)a) atomicMax(a, v);
}

struct HostFold {
  LaneTab lt;      // valid when small
  SmemRow* tab;    // CTA table when medium
  bool small;

  __device__ __forceinline__ void fold(const Params& p, int32_t fn, uint64_t dur, bool err) const {
    if (small && (dur >> 32) == 0) {
      uint32_t i = (uint32_t)fn * kWarp + lane_id();
      uint32_t d = (uint32_t)dur;
      lt.cnt[i] += 1;
      uint32_t lo = lt.slo[i] + d;
      lt.shi[i] += lo < d ? 1u : 0u;
      lt.slo[i] = lo;
      if (err) atomicAdd(&lt.err[fn], 1u);
      if (d < *(volatile uint32_t*)&lt.mn[fn]) atomicMin(&lt.mn[fn], d);
      if (d > *(volatile uint32_t*)&lt.mx[fn]) atomicMax(&lt.mx[fn], d);
    } else if (tab && (dur >> 32) == 0) {
      SmemRow* r = &tab[fn];
      uint32_t d = (uint32_t)dur;
      atomicAdd(&r->count, 1u);
      if (err) atomicAdd(&r->err, 1u);
      uint32_t o0 = atomicAdd(&r->s0, d);
      if (o0 + d < o0) atomicAdd(&r->s1, 1u);
      if (d < *(volatile uint32_t*)&r->mn) atomicMin(&r->mn, d);
      if (d > *(volatile uint32_t*)&r->mx) atomicMax(&r->mx, d);
    } else {
      fold_host_global(p, fn, dur, err);
    }
  }
};

// device rows: CTA cache keyed by the global row id, global atomics on a miss
// signed 128-bit a < b
__device__ __forceinline__ bool lt128(int64_t ahi, uint64_t alo, int64_t bhi, uint64_t blo) {
  return ahi < bhi || (ahi == bhi && alo < blo);
}

// a device span beyond +-2^63 ns (Python ints have no width, sinks.py:123-132): 128-bit extrema of
// the row under a per-row lock (rare: negative or huge device_end - device_start)
static __device__ __noinline__ void fold_device_wide(const Params& p, uint32_t row, uint64_t d_lo, int64_t d_hi) {
  unsigned long long* w = p.dev_wide + 6ull * row;
  while (atomicCAS(&w[0], 0ull, 1ull) != 0ull) {
  }
  __threadfence();
  volatile unsigned long long* v = w;
  v[1] = v[1] + 1;
  if (lt128(d_hi, d_lo, (int64_t)v[3], v[2])) { v[2] = d_lo; v[3] = (uint64_t)d_hi; }
  if (lt128((int64_t)v[5], v[4], d_hi, d_lo)) { v[4] = d_lo; v[5] = (uint64_t)d_hi; }
  __threadfence();
  atomicExch(&w[0], 0ull);
  atomicExch(p.wide_flag, 1u);  // the multi-rank merge carries 64-bit extrema only
}

static __device__ __noinline__ void fold_device_global(const Params& p, uint32_t row, uint64_t d_lo, int64_t d_hi) {
  unsigned long long* a = p.dev_acc + 6ull * row;
  atomicAdd(&a[0], 1ull);
  add_i128(&a[2], &a[3], d_lo, d_hi);
  if (d_hi == ((int64_t)d_lo >> 63)) {
    atomicMin(&a[4], bias64((int64_t)d_lo));
    atomicMax(&a[5], bias64((int64_t)d_lo));
  } else {
    fold_device_wide(p, row, d_lo, d_hi);
  }
}

__device__ __forceinline__ void fold_device(const Params& p, DevRow* cache, uint32_t row, uint64_t d_lo, int64_t d_hi) {
  DevRow* r = &cache[row % kDevSlots];
  uint32_t tag = *(volatile uint32_t*)&r->tag;
  if (tag == 0) { tag = atomicCAS(&r->tag, 0u, row + 1); if (tag == 0) tag = row + 1; }
  const bool fits32 = d_hi == ((int64_t)d_lo >> 63) && (int64_t)d_lo >= INT32_MIN && (int64_t)d_lo <= INT32_MAX;
  if (tag != row + 1 || !fits32) { fold_device_global(p, row, d_lo, d_hi); return; }
  atomicAdd(&r->count, 1u);
  // 96-bit two's complement accumulation of a sign-extended 32-bit value
  const uint32_t lo = (uint32_t)d_lo;
  const uint32_t ext = (int32_t)lo < 0 ? 0xFFFFFFFFu : 0u;
  const uint32_t o0 = atomicAdd(&r->s0, lo);
  const uint32_t c0 = (o0 + lo) < o0 ? 1u : 0u;
  const uint32_t add1 = ext + c0;  // 0, 1, 0xFFFFFFFF or 0 (wrapped)
  if (add1) {
    const uint32_t o1 = atomicAdd(&r->s1, add1);
    const uint32_t c1 = (o1 + add1) < o1 ? 1u : 0u;
    const uint32_t add2 = ext + c1;
    if (add2) atomicAdd(&r->s2, add2);
  }
  const uint32_t b = lo ^ 0x80000000u;
  if (b < *(volatile uint32_t*)&r->mn) atomicMin(&r->mn, b);
  if (b > *(volatile uint32_t*)&r->mx) atomicMax(&r->mx, b);
}

// ---------------------------------------------------------------------------
// one round of the LIFO automaton over 32 consecutive elements (lane order =
// sequence order), against a stack kept in global memory (warp-uniform view).
// Exact semantics of pipeline.py:156-168: an exit pops only a same-function
// top; otherwise it is an orphan and does not pop.  With allow_pending, exits
// that meet an empty stack are kept (at the stack bottom) for a later
// composition instead of being orphans.

struct GStack {
  SumEntry* base;      // positions >= n_fast (global scratch)
  SumEntry* fast;      // positions < n_fast (the warp's shared-memory slice; nullptr: none)
  uint32_t n_fast;
  uint32_t n_pend;
  uint32_t top;
  __device__ __forceinline__ SumEntry& at(uint32_t i) const { return i < n_fast ? fast[i] : base[i]; }
};

struct RoundOut {
  uint64_t ets;      // entry timestamp of a matched pair
  uint32_t flags;    // bit0 paired, bit1 orphan
  uint32_t n_pend;   // updated stack (warp-uniform)
  uint32_t top;
};

static __device__ __noinline__ RoundOut round_resolve(GStack st, bool allow_pending, bool isE, bool isX, int32_t fn,
                                               uint64_t ts, SumEntry mine) {
  const uint32_t lane = lane_id();
  bool paired = false, orphan = false;
  uint64_t entry_ts = 0;
  uint32_t unres = __ballot_sync(0xffffffffu, isE || isX);
  const uint32_t Emask = __ballot_sync(0xffffffffu, isE);
  bool me_unres = isE || isX;
  for (int it = 0; it < kWarp; it++) {
    uint32_t pm = unres & lanemask_lt();
    int pred = pm ? 31 - __clz(pm) : 0;
    int32_t pfn = __shfl_sync(0xffffffffu, fn, pred);
    uint64_t pts = __shfl_sync(0xffffffffu, ts, pred);
    bool act = isX && me_unres && pm && ((Emask >> pred) & 1u);
    bool m = act && pfn == fn;
    bool o = act && pfn != fn;
    uint32_t Mx = __ballot_sync(0xffffffffu, m);
    uint32_t Ox = __ballot_sync(0xffffffffu, o);
    if (!(Mx | Ox)) break;
    uint32_t nm = unres & lanemask_gt();
    int succ = nm ? __ffs(nm) - 1 : 0;
    bool claimed = isE && me_unres && nm && ((Mx >> succ) & 1u);
    uint32_t Ce = __ballot_sync(0xffffffffu, claimed);
    if (m) { paired = true; entry_ts = pts; me_unres = false; }
    if (o) { orphan = true; me_unres = false; }
    if (claimed) me_unres = false;
    unres &= ~(Mx | Ox | Ce);
  }
  // leading exits against the stack, in order
  uint32_t Xs = __ballot_sync(0xffffffffu, isX && me_unres);
  while (Xs) {
    int jx = __ffs(Xs) - 1;
    int32_t fj = __shfl_sync(0xffffffffu, fn, jx);
    if (st.top > st.n_pend) {
      SumEntry tp = st.at(st.top - 1);
      if (tp.fn == fj) {
        if ((int)lane == jx) { paired = true; entry_ts = tp.ts; }
        st.top--;
      } else if ((int)lane == jx) {
        orphan = true;
      }
    } else if (allow_pending) {
      if ((int)lane == jx) st.at(st.n_pend) = mine;
      st.n_pend++;
      st.top++;
    } else if ((int)lane == jx) {
      orphan = true;
    }
    __syncwarp();
    Xs &= Xs - 1;
  }
  uint32_t Es = __ballot_sync(0xffffffffu, isE && me_unres);
  if (isE && me_unres) st.at(st.top + __popc(Es & lanemask_lt())) = mine;
  st.top += __popc(Es);
  __syncwarp();
  RoundOut out;
  out.ets = entry_ts;
  out.flags = (paired ? 1u : 0u) | (orphan ? 2u : 0u);
  out.n_pend = st.n_pend;
  out.top = st.top;
  return out;
}

// append one timeline message per lane with `on` (warp-aggregated slot claim);
// called by all 32 lanes
static __device__ __noinline__ void tl_emit(const Params& p, bool on, uint64_t khi, uint64_t klo, uint64_t a, uint64_t b,
                                     uint32_t kind, uint32_t x) {
  const uint32_t m = __ballot_sync(0xffffffffu, on);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if ((int)lane_id() == leader) base = atomicAdd(p.tl_n2, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (on) {
    const unsigned long long i = p.tl_comp_base + base + __popc(m & lanemask_lt());
    if (i < p.tl_cap) {
      TlItem it;
      it.khi = khi; it.klo = klo; it.a = a; it.b = b; it.kind = kind; it.x = x;
      p.tl_items[i] = it;
    }
  }
}

// variable-payload field walk (tracefile.py:152-169); returns 0 or an HG_ERR_* code.
// role_off receives stream offsets of role fields, name_len the name string length.
template <class RD32>
static __device__ __noinline__ uint32_t walk_fields(const Params& p, uint2 d, uint32_t sid, uint64_t body, uint32_t plen,
                                                RD32 rd, const Window& w, uint64_t* role_off, uint32_t& name_len,
                                                uint64_t& aux) {
  const DSchema* s = schema_of(p, sid);
  const uint8_t* kd = p.kinds + s->kinds_off;
  const uint8_t* fr = p.field_role + s->kinds_off;
  uint32_t q = 0;
  for (uint32_t i = 0; i < s->nfields; i++) {
    uint8_t k = __ldg(&kd[i]);
    uint8_t role = __ldg(&fr[i]);
    if (k < HG_KIND_STRING) {
      if (q + 8 > plen) { aux = ((uint64_t)q << 8) | 8; return HG_ERR_STRUCT; }
      if (role != 0xff) role_off[role] = body + q;
      q += 8;
    } else {
      if (q + 4 > plen) { aux = ((uint64_t)q << 8) | 4; return HG_ERR_STRUCT; }
      uint32_t ln = rd(body + q);
      q += 4;
      if ((uint64_t)q + ln > plen) return HG_ERR_TRUNC_VAR;
      if (k == HG_KIND_STRING && !utf8_valid(w, body + q, ln)) { aux = q; return HG_ERR_UTF8; }
      if (role != 0xff) {
        role_off[role] = body + q;
        if (role == HG_ROLE_NAME) name_len = ln;
      }
      q += ln;
    }
  }
  (void)d;
  if (q != plen) return HG_ERR_TRAILING;
  return 0;
}


// segment start selector for a schema's variable-payload plan
__device__ __forceinline__ uint32_t seg_sel(const uint32_t seg[5], uint32_t k) {
  uint32_t v = seg[0];
  v = k == 1 ? seg[1] : v;
  v = k == 2 ? seg[2] : v;
  v = k == 3 ? seg[3] : v;
  v = k == 4 ? seg[4] : v;
  return v;
}

}  // namespace hg
