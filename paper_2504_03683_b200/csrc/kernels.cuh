// kernels.cuh -- the decode -> pair -> tally kernels of hapigpu (sm_100a).
//
// tile_kernel (persistent, one warp per 8 KiB tile of one stream file)
//   stage    TMA bulk copy (cp.async.bulk + mbarrier) of tile+overhang into the
//            warp's shared window; the next tile is prefetched into L2
//            (cp.async.bulk.prefetch.L2) while this one is processed.
//   pass A   each lane owns 256 bytes: speculative sync to a plausible record
//            header and a header walk (tracefile.py:198-210 checks); an
//            intra-warp consistency loop and a decoupled look-back over the
//            previous tiles of the stream fix the true record boundaries.
//   rounds   32 records per round in lockstep, one per lane: decode + payload
//            validation (tracefile.py:147-169), monotonicity (pipeline.py:98),
//            then the LIFO pairing (pipeline.py:156-185) as a depth computation
//            (ballot prefix counts, clamped at zero for exits that meet an
//            empty stack) and level matching with match.any; the typed check
//            entry.fn == exit.fn guards the fast path, and the first round that
//            fails it (or overflows the shared level table) switches the rest of
//            the tile to an exact ballot/shuffle elimination (round_resolve).
//            Matched pairs fold into per-lane tally columns (no atomics).
//   summary  pending exits + open entries go to a small per-tile summary.
// compose_kernel (one warp per stream) runs round_resolve over the tile
//   summaries in tile order from an empty stack, then closes the stream's open
//   calls as truncated spans at the global last timestamp (pipeline.py:220-240).
#pragma once
#include "hg_device.cuh"

namespace hg {

// dynamic shared memory of the tile kernel; every shared pointer is derived from this
// symbol in the function that uses it so accesses compile to LDS/STS
extern __shared__ __align__(128) uint8_t g_smem[];

constexpr int kLaneBytes = 256;                // stream bytes per lane in pass A
constexpr int kTile = kWarp * kLaneBytes;      // 8 KiB per warp tile
constexpr int kMaxRecLane = kLaneBytes / 16;   // records per lane (16-byte minimum)
constexpr int kMaxRecTile = kTile / 16;
constexpr int kOverhang = 512;
constexpr int kWinBytes = kTile + kOverhang;
constexpr int kWinWords = kWinBytes / 4 + 4;
constexpr int kWarpsPerCta = 12;
constexpr int kCtaThreads = kWarpsPerCta * kWarp;
constexpr uint32_t kSmallF = 16;               // per-lane tally columns up to this many functions
constexpr uint32_t kSmemFnMax = 2048;          // CTA-shared tally table up to this many functions
constexpr int kDevSlots = 64;                  // CTA cache of device rows
constexpr int kNameSlots = 64;                 // CTA cache of device-name hashes
constexpr int kLevels = 64;                    // depth levels tracked in shared memory (fast path)
constexpr int kPendCap = 64;                   // pending exits kept in shared memory (fast path)
constexpr int kQCap = 64;                      // deferred-record queue per warp
constexpr int kSyncSpan = 48;                  // bytes a lane scans for a speculative record start
constexpr int kSdescMax = 512;                 // schema ids screened from shared memory

// packed record meta used in residues and level slots
//   fn (19 bits) | exit (bit 19) | error (bit 20) | bad f64 result (bit 21) | NaN (bit 22) | tile record index (bits 23..31)
constexpr uint32_t M_FN = 0x7FFFFu;
constexpr uint32_t M_EXIT = 1u << 19, M_ERR = 1u << 20, M_BAD = 1u << 21, M_NAN = 1u << 22;
__device__ __forceinline__ int32_t m_fn(uint32_t m) { return (m & M_FN) == M_FN ? -1 : (int32_t)(m & M_FN); }
__device__ __forceinline__ uint32_t m_rec(uint32_t m) { return m >> 23; }

struct alignas(16) WarpSmem {
  uint32_t win[kWinWords];
  unsigned long long mbar;
  uint32_t pad0;
  uint16_t roff[kMaxRecLane][kWarp];     // pass A: record offsets (window-relative), [k][lane]
  uint16_t rlist[kMaxRecTile];           // record offsets in tile order
  uint32_t q[kQCap];                     // deferred records: window offset | tile record index << 16
  uint64_t lvl_ts[kLevels];              // open entry per depth level (fast path)
  uint32_t lvl_meta[kLevels];
  uint64_t pend_ts[kPendCap];            // pending exits (fast path)
  uint64_t pend_res[kPendCap];
  uint32_t pend_meta[kPendCap];
};

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
  const uint32_t* order;          // processing order -> stream-major tile id
  uint32_t n_tiles, n_streams;
  const DSchema* schemas;
  const int32_t* sid_map;
  const uint2* desc;              // compact per-sid descriptor (see make_desc)
  uint32_t max_sid;
  const uint8_t* kinds;
  const uint8_t* field_role;
  uint32_t n_fn;
  TileState* state;
  uint32_t epoch;
  SumEntry* pool;
  unsigned long long* pool_used;
  uint64_t pool_cap;
  SumEntry* warp_scratch;         // per resident warp: kMaxRecTile entries (pass C tile stack)
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
  // timeline messages (nullptr unless HG_WANT_TIMELINE): slots [0, tl_comp_base) are
  // indexed by global record number (segment decode), compose appends after them
  TlItem* tl_items;
  unsigned long long* tl_n;        // messages written by the segment decode
  unsigned long long* tl_n2;       // messages appended by compose
  uint64_t tl_comp_base;
  uint64_t tl_cap;
  const unsigned long long* tl_rec_off;  // per stream: global record number of its first record
  // segments
  uint32_t seg_bytes;
  SumEntry* deep;                  // per-lane automaton chunks of deep segments
  unsigned long long* deep_used;
  uint64_t deep_cap;
};

// compact descriptor: x = fn(20) | cls(3)<<20 | flags(8)<<23 ; y = fixed_len(16) | result field index(8)<<16 | counter(8)<<24
__device__ __forceinline__ uint32_t d_fn(uint2 d) { return d.x & 0xFFFFFu; }
__device__ __forceinline__ uint32_t d_cls(uint2 d) { return (d.x >> 20) & 7u; }
__device__ __forceinline__ uint32_t d_flags(uint2 d) { return d.x >> 23; }
__device__ __forceinline__ uint32_t d_fixed(uint2 d) { return d.y & 0xFFFFu; }
__device__ __forceinline__ uint32_t d_resfield(uint2 d) { return (d.y >> 16) & 0xFFu; }
constexpr uint32_t D_PRESENT = 0x80000000u;  // stored in flags' top bit position of x

// ---------------------------------------------------------------------------
// fast shared-memory reads (record fully inside the staged window)

__device__ __forceinline__ uint32_t s32(const uint32_t* w, uint32_t o) {
  return __funnelshift_r(w[o >> 2], w[(o >> 2) + 1], (o & 3) * 8);
}
__device__ __forceinline__ uint64_t s64(const uint32_t* w, uint32_t o) {
  uint32_t i = o >> 2, sh = (o & 3) * 8;
  uint32_t a = w[i], b = w[i + 1], c = w[i + 2];
  return ((uint64_t)__funnelshift_r(b, c, sh) << 32) | __funnelshift_r(a, b, sh);
}

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
// pass A: record boundaries

// header checks needed to walk a chain (tracefile.py:199-210); window-relative offsets
__device__ __forceinline__ bool walkable(const Params& p, const uint32_t* win, uint64_t t0, uint64_t size, uint32_t o,
                                         uint32_t& next) {
  uint64_t a = t0 + o;
  if (a + 16 > size) return false;
  uint32_t sid = s32(win, o);
  uint32_t plen = s32(win, o + 12);
  if (a + 16 + plen > size) return false;
  if (!d_present(desc_of(p, sid))) return false;
  next = o + 16 + plen;
  return true;
}

// stricter plausibility for speculative sync points (two consistent headers)
__device__ __forceinline__ bool plausible(const Params& p, const uint32_t* win, uint64_t t0, uint64_t size,
                                          uint32_t win_len, uint32_t o, uint32_t& next, uint64_t& ts) {
  if (o + 16 > win_len) return false;
  uint32_t sid = s32(win, o);
  if (sid > p.max_sid) return false;
  uint2 d = desc_of(p, sid);
  if (!d_present(d)) return false;
  uint32_t plen = s32(win, o + 12);
  if (t0 + o + 16 + plen > size) return false;
  if (d_flags(d) & SF_VAR) { if (plen < d_fixed(d)) return false; }
  else if (plen != d_fixed(d)) return false;
  next = o + 16 + plen;
  ts = s64(win, o + 4);
  return true;
}

__device__ __forceinline__ bool sync_ok(const Params& p, const uint32_t* win, uint64_t t0, uint64_t size,
                                        uint32_t win_len, uint32_t o) {
  uint32_t next, n2;
  uint64_t ts, ts2;
  if (!plausible(p, win, t0, size, win_len, o, next, ts)) return false;
  if (t0 + next == size) return true;
  if (!plausible(p, win, t0, size, win_len, next, n2, ts2)) return false;
  return ts2 >= ts;
}

// walk from `entry` while records start before sub1 (window-relative); kNone32 = failure
constexpr uint32_t kNone32 = 0xFFFFFFFFu;

__device__ __forceinline__ void lane_walk(const Params& p, WarpSmem* ws, const uint32_t* win, uint64_t t0,
                                          uint64_t size, uint32_t entry, uint32_t sub1, uint32_t& cnt,
                                          uint32_t& exit, bool& fail, uint32_t& fail_off) {
  const uint32_t lane = lane_id();
  uint32_t o = entry;
  cnt = 0;
  fail = false;
  while (o < sub1) {
    uint32_t next;
    if (!walkable(p, win, t0, size, o, next)) { fail = true; fail_off = o; exit = kNone32; return; }
    ws->roff[cnt][lane] = (uint16_t)o;
    cnt++;
    o = next;
  }
  exit = o;
}

// offsets are window-relative u32; kNone32 marks "dead/unknown"
__device__ __noinline__ void warp_verify(const Params& p, uint32_t ws_off, uint64_t t0, uint64_t size,
                                         uint32_t sub1, uint32_t e0, uint32_t& hyp, uint32_t& cnt, uint32_t& exit,
                                         bool& fail, uint32_t& fail_off) {
  WarpSmem* ws = reinterpret_cast<WarpSmem*>(g_smem + ws_off);
  const uint32_t* win = ws->win;
  const uint32_t lane = lane_id();
  for (int it = 0; it < 2 * kWarp + 2; it++) {
    uint32_t up = __shfl_up_sync(0xffffffffu, exit, 1);
    uint32_t e_in = lane == 0 ? e0 : up;
    bool good;
    if (e_in == kNone32) good = true;
    else if (e_in >= sub1) good = (cnt == 0 && !fail && exit == e_in);
    else good = (hyp == e_in);
    if (__all_sync(0xffffffffu, good)) return;
    if (!good) {
      if (e_in >= sub1) { cnt = 0; fail = false; exit = e_in; hyp = e_in; }
      else { hyp = e_in; lane_walk(p, ws, win, t0, size, e_in, sub1, cnt, exit, fail, fail_off); }
    }
  }
}

// ---------------------------------------------------------------------------
// decoupled look-back over the stream's previous tiles

struct DoneState { uint64_t exit, incl, last_ts; uint32_t has_last, pad; };

struct Look {
  uint64_t entry;   // true entry offset (stream offset); kNone: the stream failed earlier
  uint64_t base;    // records of the stream before this tile
  uint64_t prev_ts;
  bool has_prev;
};

__device__ __forceinline__ uint32_t st_status(const TileState* s) { return *(volatile const uint32_t*)&s->status; }
__device__ __forceinline__ uint64_t vld(const uint64_t* a) { return *(volatile const uint64_t*)a; }
__device__ __forceinline__ uint32_t vld32(const uint32_t* a) { return *(volatile const uint32_t*)a; }

__device__ __forceinline__ uint32_t wait_status(const Params& p, const TileState* s, bool need_final) {
  long long t_start = clock64();
  for (uint32_t spins = 0;; spins++) {
    uint32_t st = st_status(s);
    if ((st >> 2) == p.epoch) {
      uint32_t c = st & 3u;
      if (c == TS_DONE || c == TS_ERROR || (!need_final && c == TS_SPEC)) { __threadfence(); return c; }
    }
    __nanosleep(32);
    // watchdog: a predecessor that never publishes is an engine bug; fail loudly instead of hanging
    if ((spins & 1023u) == 1023u && clock64() - t_start > (long long)8e9) {
      atomicExch(p.watchdog, 1u);
      return TS_ERROR;
    }
  }
}

__device__ __noinline__ Look lookback(const Params& p, const DoneState* done, uint32_t g0, uint32_t g, uint64_t size) {
  Look L;
  uint32_t k = g - 1;
  for (;;) {  // nearest tile with a final state (the stream's first tile never publishes SPEC)
    uint32_t c = wait_status(p, &p.state[k], false);
    if (c != TS_SPEC) break;
    k--;
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
      uint64_t t1 = min(16 + (uint64_t)(i - g0 + 1) * kTile, size);
      bool ok = (se == kNone) ? (e >= t1) : (e == se && sx != kNone);
      if (!ok) { broken = true; break; }
      if (se != kNone) {
        e = sx;
        base += sn;
        if (sn) { last = vld(&s->last_ts); has = true; }
      }
    }
    if (!broken) { L.entry = e; L.base = base; L.prev_ts = last; L.has_prev = has; return L; }
    wait_status(p, &p.state[i], true);  // tile i repairs its speculation; resume from it
    k = i;
  }
}

__device__ __forceinline__ void publish(TileState* s, uint32_t epoch, uint32_t code) {
  __threadfence();
  *(volatile uint32_t*)&s->status = (epoch << 2) | code;
}

// ---------------------------------------------------------------------------
// error / orphan sinks

__device__ __noinline__ void push_error(const Params& p, uint32_t code, uint32_t stream, uint64_t seq, uint64_t off, uint64_t ts,
                           uint64_t prev_ts, uint64_t aux) {
  unsigned int i = atomicAdd(p.n_errors, 1u);
  if (i < p.error_cap) {
    hg_trace_error e;
    e.code = code; e.stream = stream; e.seq = seq; e.offset = off; e.ts = ts; e.prev_ts = prev_ts; e.aux = aux;
    p.errors[i] = e;
  }
}

__device__ __noinline__ void push_orphan(const Params& p, uint32_t stream, int32_t fn, uint64_t ts, uint64_t seq) {
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

__device__ __noinline__ void fold_host_global(const Params& p, int32_t fn, uint64_t dur, bool err) {
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
__device__ __noinline__ void fold_device_global(const Params& p, uint32_t row, uint64_t d_lo, int64_t d_hi) {
  unsigned long long* a = p.dev_acc + 6ull * row;
  atomicAdd(&a[0], 1ull);
  add_i128(&a[2], &a[3], d_lo, d_hi);
  if (d_hi == ((int64_t)d_lo >> 63)) {
    atomicMin(&a[4], bias64((int64_t)d_lo));
    atomicMax(&a[5], bias64((int64_t)d_lo));
  } else {
    atomicExch(p.wide_flag, 1u);
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

// device-name row: CTA hash cache verified by full comparison with the row's stored bytes
__device__ __forceinline__ bool arena_equal(const NameDict& d, uint32_t row, const uint32_t* win, uint32_t o, uint32_t n) {
  if (d.name_len[row] != n) return false;
  const uint8_t* a = d.arena + d.name_off[row];
  for (uint32_t i = 0; i < n; i++)
    if (a[i] != (uint8_t)(s32(win, o + i) & 0xff)) return false;
  return true;
}

__device__ uint64_t hash_smem(const uint32_t* win, uint32_t o, uint32_t n) {
  uint64_t h = 0x9E3779B97F4A7C15ull ^ ((uint64_t)n * 0xff51afd7ed558ccdull);
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4) {
    h ^= s32(win, o + i);
    h *= 0x100000001b3ull;
    h ^= h >> 29;
  }
  if (i < n) {
    uint32_t x = s32(win, o + i) & (0xffffffffu >> (8 * (4 - (n - i))));
    h ^= x;
    h *= 0x100000001b3ull;
  }
  h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return h | 1ull;
}

// ---------------------------------------------------------------------------
// one round of the LIFO automaton over 32 consecutive elements (lane order =
// sequence order), against a stack kept in global memory (warp-uniform view).
// Exact semantics of pipeline.py:156-168: an exit pops only a same-function
// top; otherwise it is an orphan and does not pop.  With allow_pending, exits
// that meet an empty stack are kept (at the stack bottom) for a later
// composition instead of being orphans.

struct GStack {
  SumEntry* base;
  uint32_t n_pend;
  uint32_t top;
};

struct RoundOut {
  uint64_t ets;      // entry timestamp of a matched pair
  uint32_t flags;    // bit0 paired, bit1 orphan
  uint32_t n_pend;   // updated stack (warp-uniform)
  uint32_t top;
};

__device__ __noinline__ RoundOut round_resolve(GStack st, bool allow_pending, bool isE, bool isX, int32_t fn,
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
      SumEntry tp = st.base[st.top - 1];
      if (tp.fn == fj) {
        if ((int)lane == jx) { paired = true; entry_ts = tp.ts; }
        st.top--;
      } else if ((int)lane == jx) {
        orphan = true;
      }
    } else if (allow_pending) {
      if ((int)lane == jx) st.base[st.n_pend] = mine;
      st.n_pend++;
      st.top++;
    } else if ((int)lane == jx) {
      orphan = true;
    }
    __syncwarp();
    Xs &= Xs - 1;
  }
  uint32_t Es = __ballot_sync(0xffffffffu, isE && me_unres);
  if (isE && me_unres) st.base[st.top + __popc(Es & lanemask_lt())] = mine;
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
__device__ __noinline__ void tl_emit(const Params& p, bool on, uint64_t khi, uint64_t klo, uint64_t a, uint64_t b,
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

// ---------------------------------------------------------------------------
// pass B: one lane decodes its records and runs the automaton locally

struct LaneOut {
  uint32_t np, sp;          // residue: [0,np) pending exits, [np,sp) open entries
  uint32_t dec_err;         // first decode-level error (cuts the stream)
  uint32_t dec_k;           // its lane-local record index
  uint64_t dec_aux, dec_ts, dec_prev;
  uint32_t feed_err;        // first interval-stage error
  uint32_t feed_k;
  uint64_t feed_aux, feed_ts;
  uint32_t spans;           // host pairs + device spans (identity bookkeeping)
};

// generic (bounds-checked) field reads for records that leave the staged window
struct GAcc {
  Window w;
  __device__ __forceinline__ uint32_t r32(uint64_t a) const { return rd32(w, a); }
  __device__ __forceinline__ uint64_t r64(uint64_t a) const { return rd64(w, a); }
};

// variable-payload field walk (tracefile.py:152-169); returns 0 or an HG_ERR_* code.
// role_off receives stream offsets of role fields, name_len the name string length.
template <class RD32>
__device__ __noinline__ uint32_t walk_fields(const Params& p, uint2 d, uint32_t sid, uint64_t body, uint32_t plen,
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


// ---------------------------------------------------------------------------
// fast paths for records entirely inside the staged window

// strict UTF-8 (tracefile.py:165 semantics) over window bytes: multi-byte sequences
__device__ __noinline__ bool utf8_window_slow(const uint32_t* win, uint32_t o, uint32_t n) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(win);
  uint32_t i = 0;
  while (i < n) {
    uint32_t c = b[o + i];
    if (c < 0x80) { i++; continue; }
    uint32_t need, lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) need = 1;
    else if (c >= 0xE0 && c <= 0xEF) { need = 2; lo = c == 0xE0 ? 0xA0 : 0x80; hi = c == 0xED ? 0x9F : 0xBF; }
    else if (c >= 0xF0 && c <= 0xF4) { need = 3; lo = c == 0xF0 ? 0x90 : 0x80; hi = c == 0xF4 ? 0x8F : 0xBF; }
    else return false;
    if (i + need >= n) return false;
    uint32_t d1 = b[o + i + 1];
    if (d1 < lo || d1 > hi) return false;
    for (uint32_t k = 2; k <= need; k++) {
      uint32_t dk = b[o + i + k];
      if (dk < 0x80 || dk > 0xBF) return false;
    }
    i += need + 1;
  }
  return true;
}

// ASCII 4 bytes at a time; anything else through the strict validator
__device__ __forceinline__ bool utf8_window(const uint32_t* win, const Window& w, uint32_t o, uint32_t n) {
  (void)w;
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4)
    if (s32(win, o + i) & 0x80808080u) return utf8_window_slow(win, o, n);
  if (i < n && (s32(win, o + i) & (0xffffffffu >> (8 * (4 - (n - i))))) & 0x80808080u)
    return utf8_window_slow(win, o, n);
  return true;
}

// variable payload through the schema's plan; false -> take the generic walk
// (which also produces the exact error for malformed records)
__device__ __forceinline__ bool var_plan(const DSchema* sc, const uint32_t* win, const Window& w, uint32_t body,
                                         uint32_t plen, uint32_t seg[5]) {
  const uint32_t nv = sc->nvar;
  if (nv == kNoPlan) return false;
  uint32_t q = 0;
  seg[0] = 0;
  #pragma unroll
  for (uint32_t i = 0; i < 4; i++) {
    if (i < nv) {
      q += sc->lead[i];
      if (q + 4 > plen) return false;
      uint32_t ln = s32(win, body + q);
      q += 4;
      if ((uint64_t)q + ln > plen) return false;
      if (sc->vkind[i] && !utf8_window(win, w, body + q, ln)) return false;
      q += ln;
      seg[i + 1] = q;
    }
  }
  q += sc->lead[nv];
  return q == plen;
}

__device__ __forceinline__ uint32_t seg_sel(const uint32_t seg[5], uint32_t k) {
  uint32_t v = seg[0];
  v = k == 1 ? seg[1] : v;
  v = k == 2 ? seg[2] : v;
  v = k == 3 ? seg[3] : v;
  v = k == 4 ? seg[4] : v;
  return v;
}

__device__ __forceinline__ uint64_t hash_window(const uint32_t* win, uint32_t o, uint32_t n) {
  uint64_t h = 0x9E3779B97F4A7C15ull ^ ((uint64_t)n * 0xff51afd7ed558ccdull);
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4) {
    h ^= s32(win, o + i);
    h *= 0x100000001b3ull;
    h ^= h >> 29;
  }
  if (i < n) {
    uint32_t x = s32(win, o + i) & (0xffffffffu >> (8 * (4 - (n - i))));
    h ^= x;
    h *= 0x100000001b3ull;
  }
  h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return h | 1ull;
}

// word-wise comparison of a window string with a dictionary row (arena rows are 4-aligned)
__device__ __forceinline__ bool name_equal_window(const NameDict& d, uint32_t row, const uint32_t* win, uint32_t o,
                                                  uint32_t n) {
  if (__ldg(&d.name_len[row]) != n) return false;
  const uint32_t* a = reinterpret_cast<const uint32_t*>(d.arena + d.name_off[row]);
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4)
    if (a[i >> 2] != s32(win, o + i)) return false;
  if (i < n) {
    uint32_t m = 0xffffffffu >> (8 * (4 - (n - i)));
    if ((a[i >> 2] & m) != (s32(win, o + i) & m)) return false;
  }
  return true;
}

}  // namespace hg
