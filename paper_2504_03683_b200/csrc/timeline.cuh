// timeline.cuh -- the Chrome-trace JSON of TimelineSink, produced on the GPU.
//
// Phase 1 / compose append one TlItem per interval-stage message that the
// reference's TimelineSink turns into an object (sinks.py:363-410): host spans
// at their exit record, device spans and telemetry samples at their record,
// truncated spans at finish().  This file orders and prints them:
//
//   tl_count / tl_compact / tl_tilesort / tl_pairs / tl_split / tl_merge
//        order by (khi, klo) = mux order (pipeline.py:68-114): the streams are
//        sorted runs already; empty slots dropped, runs merged pairwise with
//        merge-path partitioned passes (keys are unique)
//   tl_len_kernel     exact byte length of every item's JSON text, and the first
//        sorted position of every metadata key (pid, tid, kind) -- TimelineSink._meta
//        emits at first sight (sinks.py:351-359)
//   tl_meta_len_kernel   the lengths of the items that carry metadata objects
//   tl_scan*          exclusive scan -> byte offsets
//   tl_write_kernel   formats each CTA's kTlTile consecutive items (grouped by kind)
//        into a shared staging buffer, then stores it with aligned 16-byte writes
//
// The bytes equal json.dump(objects, fh, indent=1) (sinks.py:414-418): floats
// via numfmt.cuh (CPython repr), strings JSON-escaped with ensure_ascii.
#pragma once
#include "kernels.cuh"
#include "numfmt.cuh"

namespace hg {

struct TlTables {
  const TlItem* items;
  uint32_t n;
  const uint32_t* order;          // sorted position -> item index
  const char* fnq;                // JSON-quoted function names
  const uint64_t* fnq_off;        // n_fn + 1
  const char* sstr;               // per stream: pid, tid, quoted "Host {h} pid {pid}"
  const uint64_t* sstr_off;       // 3 * n_streams + 1
  const uint32_t* stream_proc;    // process_name meta id per stream
  uint32_t dev_proc;              // meta id of (device_pid, 0, process_name)
  const char* dev_pid;            // decimal device pid (9000000 + device_index)
  uint32_t dev_pid_len;
  unsigned int* proc_first;       // first sorted position per process meta id
  unsigned int* th_state;         // device thread_name metas: table keyed by tid
  unsigned long long* th_hi;
  unsigned long long* th_lo;
  unsigned int* th_first;
  uint32_t th_mask;
  unsigned int* th_overflow;
  const DSchema* schemas;
  const int32_t* sid_map;
  const uint8_t* kinds;
  uint32_t max_sid;
  uint64_t last_ts;               // global last timestamp: end of truncated spans
  const uint32_t* flush_stream;   // truncated items carry their flush rank: rank -> stream (nullptr: identity)
  uint32_t* lens;
  uint64_t* offs;
  char* out;                      // output buffer; item text starts at 1 + offs[i]
  uint32_t stage_cap;             // tl_write_kernel: staging bytes per tile
};

// ---------------------------------------------------------------------------
// byte writer (p == nullptr: count only)

struct TW {        // writes the bytes
  static constexpr bool kWrite = true;
  char* p;
  uint64_t n;
  __device__ __forceinline__ void c(char ch) { p[n++] = ch; }
  // the destination's head bytes, then 4-byte stores of funnel-shifted source words, then the
  // tail; every source word read holds a byte of the string (no read past its last word)
  __device__ __forceinline__ void s(const char* q, uint32_t l) {
    char* d = p + n;
    n += l;
    uint32_t i = 0;
    while (i < l && (reinterpret_cast<uintptr_t>(d + i) & 3)) { d[i] = q[i]; i++; }
    if (i + 4 <= l) {
      const char* qs = q + i;
      const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(qs) & ~(uintptr_t)3);
      const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(qs) & 3) * 8;
      uint32_t* dw = reinterpret_cast<uint32_t*>(d + i);
      uint32_t a = w[0];
      for (uint32_t k = 1; i + 4 <= l; i += 4, k++) {
        const uint32_t b = (sh || i + 8 <= l) ? w[k] : 0u;
        *dw++ = __funnelshift_r(a, b, sh);
        a = b;
      }
    }
    for (; i < l; i++) d[i] = q[i];
  }
  template <int N>
  __device__ __forceinline__ void lit(const char (&q)[N]) {
    #pragma unroll
    for (int i = 0; i < N - 1; i++) p[n + i] = q[i];
    n += N - 1;
  }
  __device__ __forceinline__ char* at() { return p + n; }
};
struct TC {        // counts them (tl_len_kernel)
  static constexpr bool kWrite = false;
  uint64_t n;
  __device__ __forceinline__ void c(char) { n++; }
  __device__ __forceinline__ void s(const char*, uint32_t l) { n += l; }
  template <int N>
  __device__ __forceinline__ void lit(const char (&)[N]) { n += N - 1; }
};

// unaligned little-endian loads from the stream bytes in HBM (aligned words + funnel shifts;
// the data array is zero-padded, so the word after the last byte is readable)
__device__ __forceinline__ uint32_t ldu32(const uint8_t* q) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(q) & ~(uintptr_t)3);
  return __funnelshift_r(w[0], w[1], (uint32_t)(reinterpret_cast<uintptr_t>(q) & 3) * 8);
}
__device__ __forceinline__ uint64_t ldu64(const uint8_t* q) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(q) & ~(uintptr_t)3);
  const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(q) & 3) * 8;
  const uint32_t a = w[0], b = w[1], c = w[2];
  return ((uint64_t)__funnelshift_r(b, c, sh) << 32) | __funnelshift_r(a, b, sh);
}

template <class W>
__device__ __forceinline__ void hex4(W& w, uint32_t v) {
  const char* hx = "0123456789abcdef";
  w.c('\\'); w.c('u');
  w.c(hx[(v >> 12) & 15]); w.c(hx[(v >> 8) & 15]); w.c(hx[(v >> 4) & 15]); w.c(hx[v & 15]);
}

// json.dumps(str) with ensure_ascii of validated UTF-8 bytes (json/encoder.py ESCAPE_ASCII)
template <class W>
__device__ __forceinline__ void json_str(W& w, const uint8_t* s, uint32_t len) {
  {  // plain printable ASCII without quote or backslash (kernel names): the bytes themselves.
     // Four bytes per step (exact SWAR byte tests: < 0x20, >= 0x7F, == '"', == '\\')
    uint32_t bad = 0;
    for (uint32_t i = 0; i < len; i += 4) {
      uint32_t x = ldu32(s + i);
      if (len - i < 4) {
        const uint32_t m = 0xffffffffu >> (8u * (4u - (len - i)));
        x = (x & m) | (0x61616161u & ~m);  // past the end: 'a'
      }
      const uint32_t y = x ^ 0x22222222u, z = x ^ 0x5C5C5C5Cu;
      bad |= ((x - 0x20202020u) & ~x) | (x + 0x01010101u) | x | ((y - 0x01010101u) & ~y) | ((z - 0x01010101u) & ~z);
    }
    if (!(bad & 0x80808080u)) {
      w.c('"');
      if (W::kWrite) w.s(reinterpret_cast<const char*>(s), len);
      else w.s(nullptr, len);
      w.c('"');
      return;
    }
  }
  w.c('"');
  for (uint32_t i = 0; i < len;) {
    uint32_t c = s[i], cp;
    if (c < 0x80) { cp = c; i += 1; }
    else if (c < 0xE0) { cp = ((c & 0x1F) << 6) | (s[i + 1] & 0x3F); i += 2; }
    else if (c < 0xF0) { cp = ((c & 0x0F) << 12) | ((s[i + 1] & 0x3F) << 6) | (s[i + 2] & 0x3F); i += 3; }
    else { cp = ((c & 0x07) << 18) | ((s[i + 1] & 0x3F) << 12) | ((s[i + 2] & 0x3F) << 6) | (s[i + 3] & 0x3F); i += 4; }
    if (cp == '"') { w.c('\\'); w.c('"'); }
    else if (cp == '\\') { w.c('\\'); w.c('\\'); }
    else if (cp >= 0x20 && cp < 0x7F) w.c((char)cp);
    else if (cp == '\n') { w.c('\\'); w.c('n'); }
    else if (cp == '\r') { w.c('\\'); w.c('r'); }
    else if (cp == '\t') { w.c('\\'); w.c('t'); }
    else if (cp == '\b') { w.c('\\'); w.c('b'); }
    else if (cp == '\f') { w.c('\\'); w.c('f'); }
    else if (cp < 0x10000) hex4(w, cp);
    else { const uint32_t v = cp - 0x10000; hex4(w, 0xD800 | (v >> 10)); hex4(w, 0xDC00 | (v & 0x3FF)); }
  }
  w.c('"');
}

// ---------------------------------------------------------------------------
// payload fields of a device/telemetry record (already validated by phase 1)

struct TlFields {
  const uint8_t* at[HG_NUM_ROLES];
  uint32_t len[HG_NUM_ROLES];
};

static __device__ __noinline__ void tl_locate(const TlTables& T, const DSchema* sc, const uint8_t* pay, TlFields& F) {
  for (int r = 0; r < HG_NUM_ROLES; r++) { F.at[r] = nullptr; F.len[r] = 0; }
  if (sc->nvar != kNoPlan) {  // payload plan: variable-field starts, then every role at its segment + delta
    uint32_t seg[5];
    uint32_t q = 0;
    seg[0] = 0;
    for (uint32_t i = 0; i < sc->nvar; i++) {
      q += sc->lead[i];
      q += 4 + ldu32(pay + q);
      seg[i + 1] = q;
    }
    for (int r = 0; r < HG_NUM_ROLES; r++) {
      if (sc->role[r] < 0) continue;
      const uint32_t at = seg_sel(seg, sc->role_seg[r]) + sc->role_delta[r];
      if (sc->role_kind[r] >= HG_KIND_STRING) { F.len[r] = ldu32(pay + at); F.at[r] = pay + at + 4; }
      else F.at[r] = pay + at;
    }
    return;
  }
  uint32_t off = 0;
  for (uint32_t f = 0; f < sc->nfields; f++) {
    const uint8_t k = T.kinds[sc->kinds_off + f];
    int role = -1;
    for (int r = 0; r < HG_NUM_ROLES; r++)
      if (sc->role[r] == (int)f) role = r;
    if (k >= HG_KIND_STRING) {
      const uint32_t l = ldu32(pay + off);
      if (role >= 0) { F.at[role] = pay + off + 4; F.len[role] = l; }
      off += 4 + l;
    } else {
      if (role >= 0) F.at[role] = pay + off;
      off += 8;
    }
  }
}

struct I128 { int64_t hi; uint64_t lo; };

// Python int of an integer field (absent -> 0, payload.get(key, 0))
__device__ __forceinline__ I128 int_field(const TlFields& F, const DSchema* sc, int role) {
  I128 r{0, 0};
  if (!F.at[role]) return r;
  r.lo = ldu64(F.at[role]);
  r.hi = (sc->role_kind[role] == HG_KIND_I64 && (int64_t)r.lo < 0) ? -1 : 0;
  return r;
}
__device__ __forceinline__ I128 add128(I128 a, I128 b) {
  I128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}
__device__ __forceinline__ I128 sub128(I128 a, I128 b) {
  I128 r;
  r.lo = a.lo - b.lo;
  r.hi = a.hi - b.hi - (a.lo < b.lo ? 1 : 0);
  return r;
}
__device__ __forceinline__ bool eq128(I128 a, I128 b) { return a.hi == b.hi && a.lo == b.lo; }

// decimal digit count of v by comparisons only (the counting writer's fast path)
__device__ __forceinline__ uint32_t ndig(uint64_t v) {
  if (v < 10000000000ull) {
    if (v < 100000ull) return v < 100ull ? (v < 10ull ? 1 : 2) : (v < 1000ull ? 3 : (v < 10000ull ? 4 : 5));
    return v < 10000000ull ? (v < 1000000ull ? 6 : 7) : (v < 100000000ull ? 8 : (v < 1000000000ull ? 9 : 10));
  }
  if (v < 1000000000000000ull)
    return v < 1000000000000ull ? (v < 100000000000ull ? 11 : 12) : (v < 10000000000000ull ? 13 : (v < 100000000000000ull ? 14 : 15));
  return v < 100000000000000000ull ? (v < 10000000000000000ull ? 16 : 17) : (v < 1000000000000000000ull ? 18 : (v < 10000000000000000000ull ? 19 : 20));
}

template <class W>
__device__ __forceinline__ void w_i128(W& w, I128 v) {
  if (!W::kWrite && (v.hi == 0 || (v.hi == -1 && (int64_t)v.lo < 0))) {  // fits in 64 bits: count
    w.s(nullptr, v.hi == 0 ? ndig(v.lo) : 1u + ndig(0 - v.lo));
    return;
  }
  if constexpr (W::kWrite) {
    w.n += nf::fmt_i128(v.hi, v.lo, w.at());
  } else {
    char b[48];
    w.s(b, (uint32_t)nf::fmt_i128(v.hi, v.lo, b));
  }
}
template <class W>
__device__ __forceinline__ void w_us(W& w, I128 ns) {  // ns / 1000.0
  if (!W::kWrite && ns.hi == 0 && ns.lo < 8796093022208000ull) {  // fmt_ns_div1000's exact-decimal case
    const uint64_t ip = ns.lo / 1000;
    const uint32_t fp = (uint32_t)(ns.lo - ip * 1000);
    w.s(nullptr, ndig(ip) + 1u + (fp == 0 ? 1u : (fp % 10u ? 3u : (fp % 100u ? 2u : 1u))));
    return;
  }
  if constexpr (W::kWrite) {
    w.n += nf::fmt_ns_div1000(ns.hi, ns.lo, w.at());
  } else {
    char b[40];
    w.s(b, (uint32_t)nf::fmt_ns_div1000(ns.hi, ns.lo, b));
  }
}

// device track id tile * 2 + engine (sinks.py:379-381)
__device__ __forceinline__ I128 dev_tid(I128 tile, I128 engine) {
  I128 t2;
  t2.lo = tile.lo << 1;
  t2.hi = (int64_t)(((uint64_t)tile.hi << 1) | (tile.lo >> 63));
  return add128(t2, engine);
}

// thread_name meta table (keyed by tid): th_first[tid] for tid < kThDirect, else th_first[kThDirect +
// slot of an open-addressing table]
constexpr uint32_t kThDirect = 1024;

static __device__ __noinline__ int th_slot_hash(const TlTables& T, I128 tid, bool insert);

__device__ __forceinline__ int th_slot(const TlTables& T, I128 tid, bool insert) {
  if (tid.hi == 0 && tid.lo < kThDirect) return (int)tid.lo;
  const int h = th_slot_hash(T, tid, insert);
  return h < 0 ? h : (int)kThDirect + h;
}

static __device__ __noinline__ int th_slot_hash(const TlTables& T, I128 tid, bool insert) {
  uint64_t h = (tid.lo * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)tid.hi * 0xC2B2AE3D27D4EB4Full);
  h ^= h >> 29;
  for (uint32_t probe = 0, slot = (uint32_t)h & T.th_mask; probe <= T.th_mask; probe++, slot = (slot + 1) & T.th_mask) {
    uint32_t st = *(volatile unsigned int*)&T.th_state[slot];
    if (st == 0) {
      if (!insert) return -1;
      st = atomicCAS(&T.th_state[slot], 0u, 1u);
      if (st == 0) {
        T.th_hi[slot] = (unsigned long long)tid.hi;
        T.th_lo[slot] = tid.lo;
        __threadfence();
        atomicExch(&T.th_state[slot], 2u);
        return (int)slot;
      }
    }
    while ((st = *(volatile unsigned int*)&T.th_state[slot]) == 1u) __nanosleep(20);
    __threadfence();
    if (*(volatile unsigned long long*)&T.th_hi[slot] == (unsigned long long)tid.hi &&
        *(volatile unsigned long long*)&T.th_lo[slot] == tid.lo)
      return (int)slot;
  }
  if (insert) atomicExch(T.th_overflow, 1u);
  return -1;
}

__device__ __forceinline__ uint32_t tl_stream(uint64_t klo) { return (uint32_t)((klo >> 40) & 0x7FFFFFu); }

__device__ __forceinline__ const DSchema* tl_schema(const TlTables& T, uint32_t sid) {
  if (sid > T.max_sid) return nullptr;
  const int32_t si = T.sid_map[sid];
  return si < 0 ? nullptr : &T.schemas[si];
}

__device__ __forceinline__ void first_min(unsigned int* a, uint32_t i) {
  if (*(volatile unsigned int*)a > i) atomicMin(a, i);
}

// ---------------------------------------------------------------------------
// sort

constexpr int kSortTile = 2048;
constexpr int kSortThreads = 256;

__device__ __forceinline__ bool key_lt(ulonglong2 a, ulonglong2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

// The slots of the record region hold each stream's messages at their record index, so every
// stream is already a sorted run (per-stream timestamps never decrease, the record index breaks
// ties); the empty slots (records that emit nothing) are dropped first.  Compose's messages (in
// claim order) are sorted per tile.  The runs are then merged pairwise -- the k-way merge of the
// reference's muxer (heapq.merge over the streams) as log2(streams) merge-path passes.

// messages per tile of the record region (empty slots: key ~0)
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kSortThreads) tl_count_kernel(const TlItem* items, uint32_t nrec, uint32_t* tcnt) {
  __shared__ uint32_t wsum[kSortThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
  uint32_t c = 0;
  for (uint32_t t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    const uint64_t g = base + t;
    if (g < nrec) c += (items[g].khi != ~0ull || items[g].klo != ~0ull) ? 1u : 0u;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kSortThreads / 32; w++) s += wsum[w];
    tcnt[blockIdx.x] = s;
  }
}
#endif  // HG_TL_KERNELS

// exclusive scan of n counts in place by one 1024-thread CTA (all threads call it); a[n] = total
__device__ __forceinline__ void cta_excl_scan(uint32_t* a, uint32_t n) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < n; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < n ? a[i] : 0u;
    uint32_t x = v;
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if ((threadIdx.x & 31) >= (uint32_t)d) x += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t w = ws[threadIdx.x];
      #pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (threadIdx.x >= (uint32_t)d) w += y;
      }
      ws[threadIdx.x] = w;
    }
    __syncthreads();
    const uint32_t incl = carry + x + ((threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0u);
    if (i < n) a[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) a[n] = carry;
}

#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(1024) tl_small_scan_kernel(uint32_t* a, uint32_t n) { cta_excl_scan(a, n); }
#endif  // HG_TL_KERNELS

// drop the empty slots: keys + item index of every message, record region then compose's
// messages; run_off[s] = first message of stream s, then one run per compose tile, run_off[R] = n
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kSortThreads) tl_compact_kernel(const TlItem* items, uint32_t nrec_slots, uint32_t n_slots,
                                                                  const uint32_t* tpre, uint32_t n_rtiles,
                                                                  const unsigned long long* rec_off, uint32_t ns,
                                                                  uint32_t nrec, uint32_t n, ulonglong2* keys,
                                                                  uint32_t* idx, uint32_t* run_off) {
  constexpr uint32_t kPer = kSortTile / kSortThreads;
  __shared__ uint32_t wsum[kSortThreads / 32];
  __shared__ uint32_t s_pre[kSortThreads];
  if (blockIdx.x >= n_rtiles) {  // compose's messages: no empty slots
    const uint64_t c0 = (uint64_t)(blockIdx.x - n_rtiles) * kSortTile;
    for (uint32_t t = threadIdx.x; t < kSortTile; t += blockDim.x) {
      const uint64_t g = nrec_slots + c0 + t;
      if (g < n_slots) {
        keys[nrec + c0 + t] = make_ulonglong2(items[g].khi, items[g].klo);
        idx[nrec + c0 + t] = (uint32_t)g;
      }
    }
    if (blockIdx.x == n_rtiles) {
      const uint32_t R0 = ns;
      for (uint32_t c = threadIdx.x; nrec + (uint64_t)c * kSortTile < n; c += blockDim.x) run_off[R0 + c] = nrec + c * kSortTile;
      const uint32_t ntc = (n - nrec + kSortTile - 1) / kSortTile;
      if (threadIdx.x == 0) run_off[R0 + ntc] = n;
      for (uint32_t s = threadIdx.x; s < ns; s += blockDim.x)  // streams whose records start at the end
        if (rec_off[s] >= nrec_slots) run_off[s] = nrec;
    }
    return;
  }
  const uint64_t base = (uint64_t)blockIdx.x * kSortTile + (uint64_t)threadIdx.x * kPer;  // kPer slots per thread
  ulonglong2 k[kPer];
  uint32_t m = 0;
  #pragma unroll
  for (uint32_t j = 0; j < kPer; j++) {
    const uint64_t g = base + j;
    k[j] = g < nrec_slots ? make_ulonglong2(items[g].khi, items[g].klo) : make_ulonglong2(~0ull, ~0ull);
    m |= (k[j].x != ~0ull || k[j].y != ~0ull) ? 1u << j : 0u;
  }
  const uint32_t c = __popc(m);
  uint32_t x = c;  // inclusive warp scan, then across warps
  #pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if ((threadIdx.x & 31) >= (uint32_t)d) x += y;
  }
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  uint32_t wo = 0;
  for (uint32_t w = 0; w < (threadIdx.x >> 5); w++) wo += wsum[w];
  const uint32_t ex = tpre[blockIdx.x] + wo + x - c;  // first output of this thread
  s_pre[threadIdx.x] = ex;
  uint32_t o = ex;
  #pragma unroll
  for (uint32_t j = 0; j < kPer; j++) {
    if (m >> j & 1u) {
      keys[o] = k[j];
      idx[o] = (uint32_t)(base + j);
      o++;
    }
  }
  __syncthreads();
  // streams starting in this tile: their first message is the first at or after the start slot
  if (threadIdx.x < 32) {
    const uint64_t t0 = (uint64_t)blockIdx.x * kSortTile, t1 = t0 + kSortTile;
    uint32_t lo = 0, hi = ns;  // first stream with rec_off >= t0
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (rec_off[mid] < t0) lo = mid + 1;
      else hi = mid;
    }
    for (uint32_t s = lo + threadIdx.x; s < ns; s += 32) {
      const uint64_t r = rec_off[s];
      if (r >= t1 || r >= nrec_slots) break;
      const uint32_t th = (uint32_t)(r - t0) / kPer, j = (uint32_t)(r - t0) % kPer;
      uint32_t before = s_pre[th];
      for (uint32_t q = 0; q < j; q++) {
        const uint64_t g = t0 + (uint64_t)th * kPer + q;
        before += (items[g].khi != ~0ull || items[g].klo != ~0ull) ? 1u : 0u;
      }
      run_off[s] = before;
    }
  }
}
#endif  // HG_TL_KERNELS

// the single pass's messages (per range, in record order, klo = index in the range): one warp per
// range writes the mux keys (stream << 40 | range_base + index: the record's index in its stream)
// back into the items and appends keys + item indices at the range's offset rpre[r], so every
// stream's ranges form one sorted run; blocks past the ranges copy compose's messages like
// tl_compact_kernel and write the run offsets
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kSortThreads) tl_range_compact_kernel(
    TlItem* items, uint32_t n_ranges, uint32_t rcap, const uint32_t* rn, const uint32_t* rpre,
    const uint32_t* range_stream, const unsigned long long* range_base, const uint32_t* stream_range0, uint32_t ns,
    uint64_t comp_base, uint32_t ncomp, uint32_t nrec, ulonglong2* keys, uint32_t* idx, uint32_t* run_off) {
  constexpr uint32_t kWarpsPerBlock = kSortThreads / 32;
  const uint32_t nrb = (n_ranges + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const uint32_t lane = threadIdx.x & 31;
  if (blockIdx.x < nrb) {
    const uint32_t r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (r >= n_ranges) return;
    const uint32_t cnt = rn[r], base = rpre[r];
    const uint64_t hi = (uint64_t)range_stream[r] << 40, rb = range_base[r];
    for (uint32_t j = lane; j < cnt; j += 32) {
      const uint64_t g = (uint64_t)r * rcap + j;
      const uint64_t khi = items[g].khi, klo = hi | (rb + items[g].klo);
      items[g].klo = klo;
      keys[base + j] = make_ulonglong2(khi, klo);
      idx[base + j] = (uint32_t)g;
    }
    return;
  }
  const uint64_t c0 = (uint64_t)(blockIdx.x - nrb) * kSortTile;
  for (uint32_t t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    const uint64_t c = c0 + t;
    if (c < ncomp) {
      const uint64_t g = comp_base + c;
      keys[nrec + c] = make_ulonglong2(items[g].khi, items[g].klo);
      idx[nrec + c] = (uint32_t)g;
    }
  }
  if (blockIdx.x == nrb) {
    for (uint32_t s = threadIdx.x; s < ns; s += blockDim.x) run_off[s] = rpre[stream_range0[s]];
    const uint32_t ntc = (ncomp + kSortTile - 1) / kSortTile;
    for (uint32_t c = threadIdx.x; c < ntc; c += blockDim.x) run_off[ns + c] = nrec + c * kSortTile;
    if (threadIdx.x == 0) run_off[ns + ntc] = nrec + ncomp;
  }
}
#endif  // HG_TL_KERNELS

// one compose tile sorted in place (bitonic, 2048 keys); the last tile is padded with ~0 keys
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kSortThreads) tl_tilesort_kernel(ulonglong2* keys, uint32_t* idx, uint32_t base,
                                                                   uint32_t count) {
  __shared__ ulonglong2 sk[kSortTile];
  __shared__ uint32_t si[kSortTile];
  const uint64_t b0 = base + (uint64_t)blockIdx.x * kSortTile;
  const uint64_t end = (uint64_t)base + count;
  for (uint32_t t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    const uint64_t g = b0 + t;
    if (g < end) { sk[t] = keys[g]; si[t] = idx[g]; }
    else { sk[t] = make_ulonglong2(~0ull, ~0ull); si[t] = 0xFFFFFFFFu; }
  }
  __syncthreads();
  for (uint32_t k = 2; k <= (uint32_t)kSortTile; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < kSortTile; t += blockDim.x) {
        const uint32_t u = t ^ j;
        if (u > t) {
          const bool up = (t & k) == 0;
          const ulonglong2 a = sk[t], b = sk[u];
          if (key_lt(b, a) == up) {
            sk[t] = b; sk[u] = a;
            const uint32_t x = si[t]; si[t] = si[u]; si[u] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    const uint64_t g = b0 + t;
    if (g < end) { keys[g] = sk[t]; idx[g] = si[t]; }
  }
}
#endif  // HG_TL_KERNELS

// merge-path co-rank: how many of the first k merged elements come from A
template <class F, class G>
__device__ __forceinline__ uint64_t corank(uint64_t k, uint64_t na, uint64_t nb, F A, G B) {
  uint64_t lo = k > nb ? k - nb : 0, hi = k < na ? k : na;
  while (lo < hi) {
    const uint64_t i = (lo + hi) >> 1;
    if (key_lt(A(i), B(k - i - 1))) lo = i + 1;
    else hi = i;
  }
  return lo;
}

// one merge pass over R runs: pair p = runs 2p, 2p+1 (the last may be alone); output tiles of
// kSortTile per pair, tile0[p] = first tile of pair p (exclusive scan), nro = the merged runs
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(1024) tl_pairs_kernel(const uint32_t* ro, uint32_t R, uint32_t* tile0, uint32_t* nro) {
  const uint32_t P = (R + 1) / 2;
  for (uint32_t p = threadIdx.x; p < P; p += blockDim.x) {
    const uint32_t len = ro[min(2 * p + 2, R)] - ro[2 * p];
    tile0[p] = (len + kSortTile - 1) / kSortTile;
    nro[p] = ro[2 * p];
  }
  if (threadIdx.x == 0) nro[P] = ro[R];
  __syncthreads();
  cta_excl_scan(tile0, P);
}
#endif  // HG_TL_KERNELS

// co-rank of every output tile's first element within its pair
#ifdef HG_TL_KERNELS
__global__ void tl_split_kernel(const ulonglong2* ki, const uint32_t* ro, uint32_t R, const uint32_t* tile0,
                                uint32_t* split) {
  const uint32_t P = (R + 1) / 2;
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= tile0[P]) return;
  uint32_t lo = 0, hi = P;  // last pair with tile0 <= b
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (tile0[mid] <= b) lo = mid;
    else hi = mid;
  }
  const uint32_t p = lo;
  const uint32_t a0 = ro[2 * p], a1 = ro[min(2 * p + 1, R)], b1 = ro[min(2 * p + 2, R)];
  const uint32_t na = a1 - a0, nb = b1 - a1;
  const uint64_t k = (uint64_t)(b - tile0[p]) * kSortTile;
  split[b] = (uint32_t)corank(k, na, nb, [&](uint64_t x) { return ki[a0 + x]; }, [&](uint64_t x) { return ki[a1 + x]; });
}
#endif  // HG_TL_KERNELS

#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kSortThreads) tl_merge_kernel(const ulonglong2* ki, const uint32_t* ii, ulonglong2* ko,
                                                                uint32_t* io, const uint32_t* ro, uint32_t R,
                                                                const uint32_t* tile0, const uint32_t* split) {
  // keys as two 8-byte arrays (the merge compares the high words first: half the shared-memory
  // wavefronts of 16-byte keys)
  __shared__ unsigned long long kx[kSortTile], ky[kSortTile];
  __shared__ uint32_t si[kSortTile];
  __shared__ uint16_t src[kSortTile];
  const uint32_t P = (R + 1) / 2;
  const uint32_t b = blockIdx.x;
  if (b >= tile0[P]) return;
  uint32_t lo = 0, hi = P;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (tile0[mid] <= b) lo = mid;
    else hi = mid;
  }
  const uint32_t p = lo;
  const uint32_t a0 = ro[2 * p], a1 = ro[min(2 * p + 1, R)], b1 = ro[min(2 * p + 2, R)];
  const uint32_t na = a1 - a0, nb = b1 - a1;
  const uint32_t k0 = (b - tile0[p]) * kSortTile, k1 = min(k0 + (uint32_t)kSortTile, na + nb);
  const uint32_t i0 = split[b], i1 = b + 1 < tile0[p + 1] ? split[b + 1] : na;
  const uint32_t j0 = k0 - i0, j1 = k1 - i1;
  const uint32_t la = i1 - i0, lb = j1 - j0;
  for (uint32_t t = threadIdx.x; t < la + lb; t += blockDim.x) {
    const uint32_t g = t < la ? a0 + i0 + t : a1 + j0 + (t - la);
    const ulonglong2 k = ki[g];
    kx[t] = k.x;
    ky[t] = k.y;
    si[t] = ii[g];
  }
  __syncthreads();
  auto lt = [&](uint32_t x, uint32_t y) { return kx[x] < kx[y] || (kx[x] == kx[y] && ky[x] < ky[y]); };
  constexpr uint32_t per = kSortTile / kSortThreads;
  const uint32_t kk = threadIdx.x * per;
  if (kk < la + lb) {
    uint32_t i, j;
    {  // co-rank of kk
      uint32_t l = kk > lb ? kk - lb : 0, h = kk < la ? kk : la;
      while (l < h) {
        const uint32_t m = (l + h) >> 1;
        if (lt(m, la + kk - m - 1)) l = m + 1;
        else h = m;
      }
      i = l;
      j = kk - l;
    }
    const uint32_t end = min(kk + per, la + lb);
    for (uint32_t k = kk; k < end; k++) {
      const bool takeA = j >= lb || (i < la && lt(i, la + j));
      src[k] = (uint16_t)(takeA ? i++ : la + j++);
    }
  }
  __syncthreads();
  const uint32_t out0 = a0 + k0;  // the merged run starts where run 2p did
  for (uint32_t t = threadIdx.x; t < la + lb; t += blockDim.x) {
    const uint32_t q = src[t];
    ko[out0 + t] = make_ulonglong2(kx[q], ky[q]);
    io[out0 + t] = si[q];
  }
}
#endif  // HG_TL_KERNELS

// ---------------------------------------------------------------------------
// metadata first occurrences

// ---------------------------------------------------------------------------
// one item's JSON text: [metas] + object, each element prefixed by ",\n " ("\n " first)

template <class W>
__device__ __forceinline__ void elem_open(W& w, bool first) {
  if (!first) w.c(',');
  w.lit("\n {\n  \"name\": ");
}

template <class W>
__device__ __forceinline__ void meta_obj(W& w, bool first, bool thread, const char* pid, uint32_t pid_len, I128 tid,
                                      const char* nameq, uint32_t name_len, const uint8_t* raw_name, uint32_t raw_len) {
  elem_open(w, first);
  if (thread) w.lit("\"thread_name\""); else w.lit("\"process_name\"");
  w.lit(",\n  \"ph\": \"M\",\n  \"ts\": 0,\n  \"pid\": ");
  w.s(pid, pid_len);
  w.lit(",\n  \"tid\": ");
  w_i128(w, tid);
  w.lit(",\n  \"args\": {\n   \"name\": ");
  if (raw_name) json_str(w, raw_name, raw_len);
  else w.s(nameq, name_len);
  w.lit("\n  }\n }");
}

// kLen: the length pass -- the item's own text only, while recording the first occurrences of
// its metadata keys (TimelineSink._meta, sinks.py:351-359); tl_meta_len_kernel then measures
// the items that carry metadata again, with it
// meta: the item opens a metadata key (flagged by tl_meta_len_kernel; the write pass looks the
// keys up only then)
template <class W, bool kLen = false>
__device__ __forceinline__ void tl_format(const TlTables& T, uint32_t i, const TlItem& it, W& w, bool meta = true) {
  const uint32_t kind = it.kind & 3u;
  bool first = i == 0;
  if (kind == TL_HOST) {
    const uint32_t s = ((it.kind & TL_TRUNC) && T.flush_stream) ? T.flush_stream[tl_stream(it.klo)] : tl_stream(it.klo);
    const uint64_t* so = T.sstr_off + 3ull * s;
    if (kLen) {
      first_min(&T.proc_first[T.stream_proc[s]], i);
    } else if (meta && T.proc_first[T.stream_proc[s]] == i) {
      meta_obj(w, first, false, T.sstr + so[0], (uint32_t)(so[1] - so[0]), I128{0, 0}, T.sstr + so[2],
               (uint32_t)(so[3] - so[2]), nullptr, 0);
      first = false;
    }
    const bool trunc = (it.kind & TL_TRUNC) != 0;
    const uint64_t end = trunc ? T.last_ts : it.khi;
    elem_open(w, first);
    w.s(T.fnq + T.fnq_off[it.x], (uint32_t)(T.fnq_off[it.x + 1] - T.fnq_off[it.x]));
    w.lit(",\n  \"ph\": \"X\",\n  \"ts\": ");
    w_us(w, I128{0, it.a});
    w.lit(",\n  \"dur\": ");
    w_us(w, I128{0, end - it.a});
    w.lit(",\n  \"pid\": ");
    w.s(T.sstr + so[0], (uint32_t)(so[1] - so[0]));
    w.lit(",\n  \"tid\": ");
    w.s(T.sstr + so[1], (uint32_t)(so[2] - so[1]));
    w.lit(",\n  \"args\": {\n   \"result\": ");
    {
      const uint32_t rk = (it.kind >> 4) & 3u;
      if (!W::kWrite && rk != 2) {  // integer result: count its digits
        const bool neg = rk == 1 && (int64_t)it.b < 0;
        w.s(nullptr, neg ? 1u + ndig(0 - it.b) : ndig(it.b));
      } else if (rk != 2 && W::kWrite) {
        if constexpr (W::kWrite) w.n += rk == 1 ? nf::fmt_i64((int64_t)it.b, w.at()) : nf::fmt_u64(it.b, w.at());
      } else {
        char b[400];
        const int l = nf::fmt_int_of_double(__longlong_as_double((long long)it.b), b);
        w.s(b, (uint32_t)l);
      }
    }
    if (trunc) w.lit(",\n   \"truncated\": true");
    w.lit("\n  }\n }");
    return;
  }
  const DSchema* sc = tl_schema(T, it.x);
  TlFields F;
  tl_locate(T, sc, reinterpret_cast<const uint8_t*>(it.a), F);
  if (kind == TL_DEVICE) {
    const I128 tile = int_field(F, sc, HG_ROLE_TILE), engine = int_field(F, sc, HG_ROLE_ENGINE);
    const I128 tid = dev_tid(tile, engine);
    if (kLen) {
      first_min(&T.proc_first[T.dev_proc], i);
      const int slot = th_slot(T, tid, true);
      if (slot >= 0) first_min(&T.th_first[slot], i);
    } else if (meta && T.proc_first[T.dev_proc] == i) {
      meta_obj(w, first, false, T.dev_pid, T.dev_pid_len, I128{0, 0}, "\"Device 0\"", 10, nullptr, 0);
      first = false;
    }
    const int slot = (kLen || !meta) ? -1 : th_slot(T, tid, false);
    if (slot >= 0 && T.th_first[slot] == i) {
      // _DEVICE_TRACK_NAMES (sinks.py:323-328)
      const bool known = tile.hi == 0 && engine.hi == 0 && tile.lo <= 1 && engine.lo <= 1;
      char nm[20];
      uint32_t nl = 0;
      if (known) {
        const char* base = engine.lo ? "\"Tile 0 Copy\"" : "\"Tile 0 Compute\"";
        for (; base[nl]; nl++) nm[nl] = base[nl];
        nm[6] = (char)('0' + tile.lo);
      } else {
        const char* base = "\"Device\"";
        for (; base[nl]; nl++) nm[nl] = base[nl];
      }
      meta_obj(w, first, true, T.dev_pid, T.dev_pid_len, tid, nm, nl, nullptr, 0);
      first = false;
    }
    const I128 st = int_field(F, sc, HG_ROLE_START), en = int_field(F, sc, HG_ROLE_END);
    elem_open(w, first);
    json_str(w, F.at[HG_ROLE_NAME], F.len[HG_ROLE_NAME]);
    w.lit(",\n  \"ph\": \"X\",\n  \"ts\": ");
    w_us(w, st);
    w.lit(",\n  \"dur\": ");
    w_us(w, sub128(en, st));
    w.lit(",\n  \"pid\": ");
    w.s(T.dev_pid, T.dev_pid_len);
    w.lit(",\n  \"tid\": ");
    w_i128(w, tid);
    w.lit(",\n  \"args\": {\n   \"kind\": ");
    if (F.at[HG_ROLE_CMDKIND]) json_str(w, F.at[HG_ROLE_CMDKIND], F.len[HG_ROLE_CMDKIND]);
    else w.lit("\"\"");
    w.lit("\n  }\n }");
    return;
  }
  // telemetry sample (sinks.py:397-410)
  elem_open(w, first);
  {
    const uint32_t t = sc->track;
    if (t < 3) w.lit("\"Power|Domain ");
    else if (t < 5) w.lit("\"GPU Frequency|Domain ");
    else if (t < 7) w.lit("\"Compute Engine|Tile ");
    else w.lit("\"Copy Engine|Tile ");
    w.c((char)('0' + (t < 3 ? t : (t - 3) & 1)));
    w.c('"');
  }
  w.lit(",\n  \"ph\": \"C\",\n  \"ts\": ");
  w_us(w, I128{0, it.khi});
  w.lit(",\n  \"pid\": ");
  w_i128(w, add128(I128{0, 9000000ull}, int_field(F, sc, HG_ROLE_DEVICE)));
  w.lit(",\n  \"tid\": 0,\n  \"args\": {\n   \"value\": ");
  {
    char b[40];
    const uint64_t bits = ldu64(F.at[HG_ROLE_VALUE]);
    const uint8_t vk = sc->role_kind[HG_ROLE_VALUE];
    int l;
    if (vk == HG_KIND_F64) l = nf::fmt_double(__longlong_as_double((long long)bits), b);
    else if (vk == HG_KIND_I64) l = nf::fmt_i64((int64_t)bits, b);
    else l = nf::fmt_u64(bits, b);
    w.s(b, (uint32_t)l);
  }
  w.lit("\n  }\n }");
}

// Items are formatted in CTA tiles of kTlTile consecutive sorted positions, gathered once into
// shared memory and handed to the threads grouped by kind (host spans, device spans, samples), so
// that a warp runs one kind's formatting code instead of all three.  With kTlRounds > 1 every
// thread formats kTlRounds items of the kind-sorted list, kTlThreads apart: a warp's rounds mix
// cheap and costly kinds, which evens out the warps' times before the tile's barrier.
#ifndef HG_TL_TILE
#define HG_TL_TILE 128  // small tiles: the CTA barrier waits for its slowest item, more CTAs per SM hide that
#endif
#ifndef HG_TL_ROUNDS
#define HG_TL_ROUNDS 1
#endif
constexpr int kTlTile = HG_TL_TILE;
constexpr int kTlRounds = HG_TL_ROUNDS;
constexpr int kTlThreads = kTlTile / kTlRounds;
constexpr uint32_t kTlMeta = 1u << 31;  // lens[i] flag: the item carries metadata objects

struct TlTileSmem {
  TlItem it[kTlTile];
  uint16_t list[kTlTile];   // tile positions grouped by kind
  uint32_t cur[4];
};

// gathers the tile's items and groups them by kind; returns the number of items in the tile
__device__ __forceinline__ uint32_t tl_tile_group(const TlTables& T, uint64_t i0, TlTileSmem& S) {
  const uint32_t t = threadIdx.x, lane = t & 31;
  uint32_t kind[kTlRounds];
  #pragma unroll
  for (int r = 0; r < kTlRounds; r++) {
    const uint32_t q = t + r * kTlThreads;
    kind[r] = 3;
    if (i0 + q < T.n) {
      const TlItem it = T.items[T.order[i0 + q]];
      S.it[q] = it;
      kind[r] = it.kind & 3u;
    }
  }
  if (t < 4) S.cur[t] = 0;
  __syncthreads();
  uint32_t pos[kTlRounds];
  #pragma unroll
  for (int r = 0; r < kTlRounds; r++) {
    pos[r] = 0;
    #pragma unroll
    for (uint32_t k = 0; k < 3; k++) {
      const uint32_t m = __ballot_sync(0xffffffffu, kind[r] == k);
      if (m) {
        const uint32_t leader = __ffs(m) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&S.cur[k], (uint32_t)__popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (kind[r] == k) pos[r] = base + __popc(m & ((1u << lane) - 1u));
      }
    }
  }
  __syncthreads();
  const uint32_t n0 = S.cur[0], n1 = S.cur[1];
  #pragma unroll
  for (int r = 0; r < kTlRounds; r++)
    if (kind[r] < 3) S.list[kind[r] == 0 ? pos[r] : kind[r] == 1 ? n0 + pos[r] : n0 + n1 + pos[r]] =
        (uint16_t)(t + r * kTlThreads);
  const uint32_t cnt = n0 + n1 + S.cur[2];
  __syncthreads();
  return cnt;
}

#ifndef HG_TL_LEN_MINB
#define HG_TL_LEN_MINB (1280 / kTlThreads)  // 48 registers: 1.26 -> 1.05 ms at C5 x0.25 (vs 80)
#endif
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kTlThreads, HG_TL_LEN_MINB) tl_len_kernel(TlTables T) {
  __shared__ TlTileSmem S;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kTlTile; i0 < T.n; i0 += (uint64_t)gridDim.x * kTlTile) {
    const uint32_t cnt = tl_tile_group(T, i0, S);
    #pragma unroll
    for (int r = 0; r < kTlRounds; r++) {
      const uint32_t q = threadIdx.x + r * kTlThreads;
      if (q < cnt) {
        const uint32_t j = S.list[q];
        TC w{0};
        tl_format<TC, true>(T, (uint32_t)(i0 + j), S.it[j], w);
        T.lens[i0 + j] = (uint32_t)w.n;
      }
    }
    __syncthreads();
  }
}
#endif  // HG_TL_KERNELS

// the items that open a metadata key: their length with the metadata objects, flagged for the
// write pass (two keys may share an item: both threads store the same value)
#ifdef HG_TL_KERNELS
__global__ void tl_meta_len_kernel(TlTables T, uint32_t n_proc, uint32_t th_size) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (uint64_t)n_proc + th_size;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = e < n_proc ? T.proc_first[e] : T.th_first[e - n_proc];
    if (f >= T.n) continue;
    TC w{0};
    tl_format<TC, false>(T, f, T.items[T.order[f]], w);
    T.lens[f] = (uint32_t)w.n | kTlMeta;
  }
}
#endif  // HG_TL_KERNELS

// ---------------------------------------------------------------------------
// exclusive scan of lens -> offs (three kernels, 1024 per block)

constexpr int kScanBlock = 1024;

__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* total) {
  __shared__ uint64_t wsum[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, x, d);
    if ((int)lane >= d) x += t;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t y = lane < (blockDim.x >> 5) ? wsum[lane] : 0;
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, y, d);
      if ((int)lane >= d) y += t;
    }
    wsum[lane] = y;
  }
  __syncthreads();
  const uint64_t before = (warp ? wsum[warp - 1] : 0) + x - v;
  if (total) *total = wsum[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kScanBlock) tl_scan1_kernel(const uint32_t* lens, uint32_t n, uint64_t* bsum) {
  const uint64_t i = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  uint64_t tot;
  block_excl_scan(i < n ? lens[i] & ~kTlMeta : 0, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
#endif  // HG_TL_KERNELS

#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kScanBlock) tl_scan2_kernel(uint64_t* bsum, uint32_t nb, uint64_t* grand) {
  uint64_t carry = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += kScanBlock) {
    const uint32_t b = b0 + threadIdx.x;
    const uint64_t v = b < nb ? bsum[b] : 0;
    uint64_t tot;
    const uint64_t ex = block_excl_scan(v, &tot);
    if (b < nb) bsum[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *grand = carry;
}
#endif  // HG_TL_KERNELS

#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kScanBlock) tl_scan3_kernel(const uint32_t* lens, uint32_t n, const uint64_t* bsum,
                                                              uint64_t* offs) {
  const uint64_t i = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const uint64_t ex = block_excl_scan(i < n ? lens[i] & ~kTlMeta : 0, nullptr);
  if (i < n) offs[i] = bsum[blockIdx.x] + ex;
}
#endif  // HG_TL_KERNELS

// ---------------------------------------------------------------------------
// writer: a CTA formats a tile of items (grouped by kind) into a shared staging buffer at their
// offsets, then stores the tile's contiguous byte range with aligned 16-byte writes

// The staging buffer is sized at launch from this timeline's average object length (TlTables::
// stage_cap, 1/16 above kTlTile x the average: a tile rarely exceeds it, and one that does is
// written straight to HBM) -- as small as the objects allow, for 8 CTAs per SM.

struct TlWriteSmem {
  TlTileSmem g;
  uint32_t rel[kTlTile];    // offset of the item's text in the staging buffer
  uint64_t o0, oend;
  __align__(16) char stage[16];  // stage_cap + 16 bytes (dynamic shared memory)
};

inline size_t tl_write_smem(uint32_t stage_cap) { return sizeof(TlWriteSmem) + stage_cap; }

#ifndef HG_TL_WRITE_MINB
#define HG_TL_WRITE_MINB (1024 / kTlThreads)  // 64 registers: 8 CTAs per SM (3.25 -> 2.81 ms at C5 x0.25 vs 6)
#endif
#ifdef HG_TL_KERNELS
__global__ void __launch_bounds__(kTlThreads, HG_TL_WRITE_MINB) tl_write_kernel(TlTables T) {
  extern __shared__ __align__(16) char tl_smem[];
  TlWriteSmem& S = *reinterpret_cast<TlWriteSmem*>(tl_smem);
  const uint32_t t = threadIdx.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kTlTile; i0 < T.n; i0 += (uint64_t)gridDim.x * kTlTile) {
    const uint64_t last = min((uint64_t)T.n, i0 + kTlTile) - 1;
    uint64_t off[kTlRounds];
    uint32_t len[kTlRounds];
    #pragma unroll
    for (int r = 0; r < kTlRounds; r++) {
      const uint64_t i = i0 + t + r * kTlThreads;
      off[r] = 0;
      len[r] = 0;
      if (i <= last) {
        off[r] = 1 + T.offs[i];
        len[r] = T.lens[i];
        if (i == i0) S.o0 = off[r];
        if (i == last) S.oend = off[r] + (len[r] & ~kTlMeta);
      }
    }
    const uint32_t cnt = tl_tile_group(T, i0, S.g);  // (its barriers publish o0 / oend)
    const uint64_t al = S.o0 & ~15ull, total = S.oend - al;
    const bool staged = total <= (uint64_t)T.stage_cap;
    #pragma unroll
    for (int r = 0; r < kTlRounds; r++)
      if (i0 + t + r * kTlThreads <= last) S.rel[t + r * kTlThreads] = (uint32_t)(off[r] - al) | (len[r] & kTlMeta);
    __syncthreads();
    #pragma unroll
    for (int r = 0; r < kTlRounds; r++) {
      const uint32_t q = t + r * kTlThreads;
      if (q < cnt) {
        const uint32_t j = S.g.list[q];
        const uint32_t rl = S.rel[j];
        const uint64_t gi = i0 + j;
        if (staged) {
          TW w{S.stage + (rl & ~kTlMeta), 0};
          tl_format(T, (uint32_t)gi, S.g.it[j], w, (rl & kTlMeta) != 0);
        } else {
          TW w{T.out + al + (rl & ~kTlMeta), 0};
          tl_format(T, (uint32_t)gi, S.g.it[j], w, (rl & kTlMeta) != 0);
        }
      }
    }
    __syncthreads();
    if (staged) {  // bytes [head, end) of the 16-byte aligned window at al
      char* gout = T.out + al;
      const uint32_t head = (uint32_t)(S.o0 - al), end = (uint32_t)total;
      const uint32_t full_end = end & ~15u;
      for (uint32_t b0 = 16u * t + (head ? 16u : 0u); b0 < full_end; b0 += 16u * kTlThreads)
        *reinterpret_cast<uint4*>(gout + b0) = *reinterpret_cast<const uint4*>(S.stage + b0);
      if (t < 16) {  // the partial first and last chunks, a byte per thread
        if (head && head + t < 16u && head + t < end) gout[head + t] = S.stage[head + t];
        const uint32_t b = full_end + t;
        if (b < end && (b >= 16u || !head)) gout[b] = S.stage[b];
      }
      __syncthreads();
    }
  }
}
#endif  // HG_TL_KERNELS

}  // namespace hg
