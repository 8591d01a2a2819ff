// hg_device.cuh -- device-side building blocks of the hapigpu engine (sm_100a).
//
// Byte access into stream bytes in HBM, strict UTF-8 validation with CPython's
// acceptance rules (tracefile.py:165 `raw.decode("utf-8")`), the device-name
// dictionary layout, exact 128-bit tally accumulators, the per-segment state and
// the timeline message record.  Included by engine.cu only.
#pragma once
#include <cstdint>

#include "../../include/hapigpu.h"

namespace hg {

constexpr int kWarp = 32;
constexpr uint64_t kNone = ~0ull;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__device__ __forceinline__ uint32_t lanemask_gt() { uint32_t m; asm("mov.u32 %0, %%lanemask_gt;" : "=r"(m)); return m; }

// ---------------------------------------------------------------------------
// schema table (flattened registry, see include/hapigpu.h hg_schema)

enum : uint8_t {
  SF_VAR = 1,          // has string/blob fields (variable payload)
  SF_RESULT = 2,       // exit with a "result" field
  SF_RESULT_F64 = 4,   // ... of kind f64
  SF_FEED_ALWAYS = 8,  // raises when fed (host holds the exception)
  SF_FEED_TIMELINE = 16,
  SF_RESULT_I64 = 32,  // ... of kind i64 (else u64/address)
  SF_NOINLINE = 64,    // range kernel: never decoded inline (f64 result, feed error, payload plan needs HBM)
};

// result kind of an exit schema for the timeline's int(result) (pipeline.py:183):
// 0 unsigned, 1 signed (absent result -> 0), 2 f64
__host__ __device__ inline uint32_t result_kind(uint32_t fl) {
  if (!(fl & SF_RESULT)) return 1;
  if (fl & SF_RESULT_F64) return 2;
  return (fl & SF_RESULT_I64) ? 1u : 0u;
}

struct DSchema {
  uint32_t kinds_off;
  int32_t fn;
  uint16_t fixed_len;   // exact payload length (fixed-only) or minimum (var)
  uint8_t cls;
  uint8_t flags;
  uint8_t nfields;
  uint8_t counter_kind;
  int8_t role[HG_NUM_ROLES];
  uint8_t role_kind[HG_NUM_ROLES];
  // fast plan for variable payloads: var items and the fixed bytes around them
  uint8_t nvar;                       // number of string/blob fields; kNoPlan: use the generic walk
  uint8_t vkind[4];                   // 1 string (UTF-8 checked), 0 blob
  uint16_t lead[5];                   // fixed bytes before var item i; lead[nvar] = trailing fixed bytes
  uint8_t role_seg[HG_NUM_ROLES];     // segment (0..nvar) holding the role field
  uint16_t role_delta[HG_NUM_ROLES];  // bytes from the segment start to the field (var field: its u32 length)
  uint8_t track;                      // telemetry: timeline counter track (0..8), 0xFF none
};
constexpr uint8_t kNoPlan = 0xFF;

// ---------------------------------------------------------------------------
// stream window: a warp-staged copy of [win_start, win_end) of one stream in
// shared memory, with a global-memory fallback outside it.

struct Window {
  const uint32_t* s;     // shared words; s[0] holds stream byte win_start (4-aligned)
  uint64_t win_start;    // stream offset of s[0]
  uint64_t win_end;      // staged bytes end (stream offset)
  const uint8_t* g;      // stream base in global memory (256-aligned)
  uint64_t size;         // stream file size
};

__device__ __forceinline__ uint32_t g_word(const uint8_t* g, uint64_t widx) {
  return __ldg(reinterpret_cast<const uint32_t*>(g) + widx);
}

// little-endian u32 at any byte offset (caller guarantees off+4 <= size + padding)
__device__ __forceinline__ uint32_t rd32(const Window& w, uint64_t off) {
  uint32_t sh = (uint32_t)(off & 3) * 8;
  if (off + 8 <= w.win_end) {
    uint64_t wi = (off - w.win_start) >> 2;
    return __funnelshift_r(w.s[wi], w.s[wi + 1], sh);
  }
  uint64_t wi = off >> 2;
  return __funnelshift_r(g_word(w.g, wi), g_word(w.g, wi + 1), sh);
}

__device__ __forceinline__ uint64_t rd64(const Window& w, uint64_t off) {
  uint32_t sh = (uint32_t)(off & 3) * 8;
  uint32_t a, b, c;
  if (off + 12 <= w.win_end) {
    uint64_t wi = (off - w.win_start) >> 2;
    a = w.s[wi]; b = w.s[wi + 1]; c = w.s[wi + 2];
  } else {
    uint64_t wi = off >> 2;
    a = g_word(w.g, wi); b = g_word(w.g, wi + 1); c = g_word(w.g, wi + 2);
  }
  uint32_t lo = __funnelshift_r(a, b, sh), hi = __funnelshift_r(b, c, sh);
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint8_t rd8(const Window& w, uint64_t off) {
  return (uint8_t)(rd32(w, off) & 0xff);
}

// Strict UTF-8 (no overlongs, no surrogates, <= U+10FFFF).  Returns true if valid.
static __device__ __noinline__ bool utf8_valid(const Window& w, uint64_t p, uint32_t n) {
  uint32_t i = 0;
  // ASCII fast path, 4 bytes at a time
  while (i + 4 <= n) {
    uint32_t x = rd32(w, p + i);
    if (x & 0x80808080u) break;
    i += 4;
  }
  while (i < n) {
    uint32_t c = rd8(w, p + i);
    if (c < 0x80) { i++; continue; }
    uint32_t need;
    uint32_t lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) need = 1;
    else if (c >= 0xE0 && c <= 0xEF) { need = 2; if (c == 0xE0) lo = 0xA0; if (c == 0xED) hi = 0x9F; }
    else if (c >= 0xF0 && c <= 0xF4) { need = 3; if (c == 0xF0) lo = 0x90; if (c == 0xF4) hi = 0x8F; }
    else return false;
    if (i + need >= n) return false;  // "unexpected end of data"
    for (uint32_t k = 1; k <= need; k++) {
      uint32_t d = rd8(w, p + i + k);
      if (k == 1 ? (d < lo || d > hi) : (d < 0x80 || d > 0xBF)) return false;
    }
    i += need + 1;
  }
  return true;
}

// ---------------------------------------------------------------------------
// device-name dictionary (device rows are keyed by the profiling payload's
// "name" string, pipeline.py:192; first-seen order assigns row ids)

struct NameDict {
  unsigned long long* keys;   // hash or 0
  uint32_t* vals;             // row + 1, 0 while being published
  uint64_t mask;
  uint8_t* arena;             // name bytes
  unsigned long long* arena_used;
  uint64_t arena_cap;
  uint64_t* name_off;         // per row
  uint32_t* name_len;
  uint32_t* n_rows;
  uint32_t row_cap;
  uint32_t* overflow;
};

// ---------------------------------------------------------------------------
// exact accumulators

// 128-bit signed sum in two u64 words, updated with global atomics
__device__ __forceinline__ void add_i128(unsigned long long* lo, unsigned long long* hi, uint64_t v_lo, int64_t v_hi) {
  unsigned long long old = atomicAdd(lo, (unsigned long long)v_lo);
  unsigned long long carry = (old + v_lo) < old ? 1ull : 0ull;
  unsigned long long h = (unsigned long long)v_hi + carry;
  if (h) atomicAdd(hi, h);
}

// order-preserving map of a signed 64-bit value onto u64
__device__ __forceinline__ uint64_t bias64(int64_t x) { return (uint64_t)x ^ 0x8000000000000000ull; }

// ---------------------------------------------------------------------------
// per-segment state read by compose_kernel

enum : uint32_t { TS_INVALID = 0, TS_DONE = 2, TS_ERROR = 3 };

struct SegState {
  uint32_t status;     // (epoch << 2) | TS_*, raised with atomicMax (a deferred error wins)
  uint32_t pool_n_pending;
  uint64_t pool_off;   // summary entries in the pool
  uint32_t pool_n_resid;
  uint32_t pad;
};

struct SumEntry {      // segment summary: pending exit or residual entry
  uint64_t ts;
  uint64_t seq;
  int32_t fn;
  uint32_t flags;      // bit0 exit, bit1 error, bit2 bad (NaN/inf) f64 result, bit3 NaN, bits4-5 result kind
  uint64_t result;     // exit result bits (timeline)
};

// ---------------------------------------------------------------------------
// timeline item: one message of the interval stage that TimelineSink turns into
// a JSON object (sinks.py:363-410).  Sorted by (khi, klo) = mux order of the
// triggering record (pipeline.py:68-114): ts, stream rank, record index; the
// truncated spans of finish() (pipeline.py:220-240) carry klo bit 63 and sort
// after everything, stream by stream, innermost first.
enum : uint32_t { TL_HOST = 0, TL_DEVICE = 1, TL_SAMPLE = 2, TL_TRUNC = 1u << 8 };
struct TlItem {
  uint64_t khi;        // ts of the triggering record (~0 for truncated spans)
  uint64_t klo;        // trunc << 63 | stream << 40 | record index (truncated: pop order)
  uint64_t a;          // host: entry ts; device/sample: payload address in HBM
  uint64_t b;          // host: result bits
  uint32_t kind;       // TL_* | result kind << 4 (host)
  uint32_t x;          // host: function id; device/sample: schema id
};
__host__ __device__ inline uint64_t tl_klo(uint32_t s, uint64_t seq) { return ((uint64_t)s << 40) | seq; }

}  // namespace hg
