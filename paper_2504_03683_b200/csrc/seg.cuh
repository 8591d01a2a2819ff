// seg.cuh -- phase 1 of hapigpu as three segment kernels (sm_100a).
//
// Every stream file is cut into fixed-size byte segments (8 KiB by default);
// a record belongs to the segment its header starts in.  One THREAD owns one
// segment and runs the reference's sequential algorithm over it, so the only
// parallelisation cost is one speculative synchronisation per segment:
//
//   seg_walk_kernel    thread per segment: find the first record header at or
//                      after the segment start (three consistent headers,
//                      tracefile.py:198-210 checks), walk the record chain to the
//                      segment end: record count, exit offset, last timestamp.
//   seg_chain_kernel   warp per stream: the true entry of segment k is the exit
//                      of segment k-1; mis-speculated segments are re-walked;
//                      header-level errors (truncated header/payload, unknown
//                      schema) cut the stream; record bases and the timestamp
//                      before each segment (monotonicity, pipeline.py:98).
//   seg_decode_kernel  thread per segment from its verified entry: full decode
//                      with every payload check (tracefile.py:147-215), the
//                      mux ordering check, the IntervalBuilder automaton
//                      (pipeline.py:142-218) on a per-lane stack in shared
//                      memory (global chunk when deep), device spans and
//                      telemetry samples, tally folds into per-lane columns,
//                      timeline messages.  Exits that meet an empty local stack
//                      and open entries at the end form the segment summary that
//                      compose_kernel resolves across segments.
#pragma once
#include "kernels.cuh"

namespace hg {

constexpr int kSegWarps = 4;
constexpr size_t kDataPad = 8192;  // zero bytes after the last stream (look-ahead reads and prefetches)
constexpr int kSegThreads = kSegWarps * kWarp;
constexpr int kLS = 8;   // open entries per lane in shared memory
constexpr int kLP = 4;   // pending exits per lane in shared memory

struct SegW {            // speculative walk of one segment
  uint64_t spec_entry;   // kNone: no synchronisation point found
  uint64_t exit;         // offset after the last walked record (kNone: walk failed)
  uint64_t last_ts;
  uint64_t fail_off;     // first non-walkable header (fail != 0)
  uint32_t n;
  uint32_t fail;
};

enum : uint32_t { SI_HAS_PREV = 1, SI_DEAD = 2, SI_HDR_FAIL = 4 };

struct SegInfo {         // verified segment
  uint64_t entry;
  uint64_t base;         // records of the stream before this segment
  uint64_t prev_ts;
  uint32_t n;            // records to decode
  uint32_t flags;        // SI_*
};

struct SegGeom {
  uint32_t g, s, j;
  uint64_t size, t0, t1;
  const uint8_t* gbase;
};

__device__ __forceinline__ SegGeom seg_geom(const Params& p, uint32_t g) {
  SegGeom G;
  G.g = g;
  G.s = p.tile_stream[g];
  G.j = g - p.stream_tile0[G.s];
  G.size = p.stream_size[G.s];
  G.gbase = p.data + p.stream_base[G.s];
  G.t0 = 16 + (uint64_t)G.j * p.seg_bytes;
  G.t1 = min(G.t0 + (uint64_t)p.seg_bytes, G.size);
  return G;
}

// unaligned little-endian reads from a 256-aligned, zero-padded stream in HBM
__device__ __forceinline__ uint32_t g32(const uint8_t* g, uint64_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(g) + (off >> 2);
  return __funnelshift_r(__ldg(w), __ldg(w + 1), (uint32_t)(off & 3) * 8);
}
__device__ __forceinline__ uint64_t g64(const uint8_t* g, uint64_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(g) + (off >> 2);
  const uint32_t sh = (uint32_t)(off & 3) * 8;
  const uint32_t a = __ldg(w), b = __ldg(w + 1), c = __ldg(w + 2);
  return ((uint64_t)__funnelshift_r(b, c, sh) << 32) | __funnelshift_r(a, b, sh);
}

// record header (sid, ts, plen) from the five words covering [off, off + 16)
struct Hdr { uint32_t sid, plen; uint64_t ts; };
__device__ __forceinline__ Hdr g_hdr(const uint8_t* g, uint64_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(g) + (off >> 2);
  const uint32_t sh = (uint32_t)(off & 3) * 8;
  const uint32_t a = __ldg(w), b = __ldg(w + 1), c = __ldg(w + 2), d = __ldg(w + 3), e = __ldg(w + 4);
  Hdr h;
  h.sid = __funnelshift_r(a, b, sh);
  h.ts = ((uint64_t)__funnelshift_r(c, d, sh) << 32) | __funnelshift_r(b, c, sh);
  h.plen = __funnelshift_r(d, e, sh);
  return h;
}

__device__ __forceinline__ Window g_window(const SegGeom& G) {
  Window w;
  w.s = nullptr; w.win_start = 0; w.win_end = 0; w.g = G.gbase; w.size = G.size;
  return w;
}

// plausible record header at `o` (known schema, payload length consistent with it)
__device__ __forceinline__ bool seg_plausible(const Params& p, const uint8_t* g, uint64_t size, uint64_t o,
                                              uint64_t& next, uint64_t& ts) {
  if (o + 16 > size) return false;
  const Hdr h = g_hdr(g, o);
  if (h.sid > p.max_sid) return false;
  const uint2 d = desc_of(p, h.sid);
  if (!d_present(d)) return false;
  if (o + 16 + h.plen > size) return false;
  if (d_flags(d) & SF_VAR) { if (h.plen < d_fixed(d)) return false; }
  else if (h.plen != d_fixed(d)) return false;
  next = o + 16 + h.plen;
  ts = h.ts;
  return true;
}

// walk the chain from `entry` while records start before t1 (tracefile.py:198-210 header checks)
static __device__ __noinline__ SegW seg_walk_from(const Params& p, const uint8_t* g, uint64_t size, uint64_t entry, uint64_t t1) {
  SegW W;
  W.spec_entry = entry;
  W.n = 0;
  W.fail = 0;
  W.fail_off = 0;
  uint64_t o = entry, last = kNone;
  while (o < t1) {
    if (o + 16 > size) { W.fail = 1; break; }
    const uint32_t sid = g32(g, o), plen = g32(g, o + 12);
    if (o + 16 + plen > size || !d_present(desc_of(p, sid))) { W.fail = 1; break; }
    last = o;
    W.n++;
    o += 16 + plen;
  }
  W.fail_off = o;
  W.exit = W.fail ? kNone : o;
  W.last_ts = last != kNone ? g64(g, last + 4) : 0;
  return W;
}

__device__ __forceinline__ void seg_load_desc(const Params& p) {
  if (p.max_sid < (uint32_t)kSdescMax) {
    uint2* t = reinterpret_cast<uint2*>(g_smem);
    for (uint32_t i = threadIdx.x; i <= p.max_sid; i += blockDim.x) t[i] = __ldg(&p.desc[i]);
  }
  __syncthreads();
}

#ifdef HG_SEG_KERNELS
__global__ void __launch_bounds__(256) seg_walk_kernel(Params p, SegW* segw) {
  seg_load_desc(p);
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < p.n_tiles; g += gridDim.x * blockDim.x) {
    const SegGeom G = seg_geom(p, g);
    uint64_t entry = kNone;
    if (G.j == 0) {
      entry = 16;
    } else {
      // first offset with three consistent headers (or a chain that ends the file)
      for (uint64_t o = G.t0; o < G.t1; o++) {
        uint64_t n1, n2, n3, ts0, ts1, ts2;
        if (!seg_plausible(p, G.gbase, G.size, o, n1, ts0)) continue;
        if (n1 != G.size) {
          if (!seg_plausible(p, G.gbase, G.size, n1, n2, ts1) || ts1 < ts0) continue;
          if (n2 != G.size && (!seg_plausible(p, G.gbase, G.size, n2, n3, ts2) || ts2 < ts1)) continue;
        }
        entry = o;
        break;
      }
    }
    SegW W;
    if (entry == kNone) {
      W.spec_entry = kNone; W.exit = kNone; W.last_ts = 0; W.fail_off = 0; W.n = 0; W.fail = 0;
    } else {
      W = seg_walk_from(p, G.gbase, G.size, entry, G.t1);
    }
    segw[g] = W;
  }
}
#endif  // HG_SEG_KERNELS

// ---------------------------------------------------------------------------
// chain: warp per stream

#ifdef HG_SEG_KERNELS
__global__ void __launch_bounds__(128) seg_chain_kernel(Params p, SegW* segw, SegInfo* info, unsigned long long* stream_nrec) {
  seg_load_desc(p);
  const uint32_t lane = lane_id();
  const uint32_t s = blockIdx.x * (blockDim.x / kWarp) + (threadIdx.x >> 5);
  if (s >= p.n_streams) return;
  const uint32_t g0 = p.stream_tile0[s];
  const uint32_t g1 = (s + 1 < p.n_streams) ? p.stream_tile0[s + 1] : p.n_tiles;
  const uint64_t size = p.stream_size[s];
  const uint8_t* gbase = p.data + p.stream_base[s];
  uint64_t c_exit = 16, c_base = 0, c_last = 0;
  bool c_has = false, c_dead = false;
  for (uint32_t gb = g0; gb < g1; gb += kWarp) {
    const uint32_t g = gb + lane;
    const bool valid = g < g1;
    const uint64_t t1 = valid ? min(16 + (uint64_t)(g - g0 + 1) * p.seg_bytes, size) : 0;
    SegW W;
    if (valid) W = segw[g];
    else { W.spec_entry = kNone; W.exit = kNone; W.last_ts = 0; W.fail_off = 0; W.n = 0; W.fail = 0; }
    // resolve the chain: lane k's entry is lane k-1's exit (lane 0: the carry)
    uint32_t fixed = 0;
    for (;;) {
      uint64_t pe = __shfl_up_sync(0xffffffffu, W.exit, 1);
      const uint32_t pf = __shfl_up_sync(0xffffffffu, W.fail, 1);
      if (lane == 0) pe = c_exit;
      const bool pfail = lane == 0 ? false : pf != 0;
      bool ok = true;
      if (valid && !pfail && !c_dead) {
        if (pe >= t1) ok = (W.n == 0 && W.exit == pe && !W.fail);   // a record spans the whole segment
        else ok = W.spec_entry == pe;
      }
      const uint32_t bad = __ballot_sync(0xffffffffu, !ok) & ~fixed;
      if (!bad) break;
      const int j = __ffs(bad) - 1;
      if ((int)lane == j) {
        if (pe >= t1) { W.spec_entry = pe; W.exit = pe; W.n = 0; W.fail = 0; W.last_ts = 0; W.fail_off = 0; }
        else W = seg_walk_from(p, gbase, size, pe, t1);
      }
      fixed |= 1u << j;
    }
    // header-level failure cuts the stream: the first failing lane (from its true entry)
    const uint32_t fm = __ballot_sync(0xffffffffu, valid && W.fail);
    const int fl = (c_dead) ? -1 : (fm ? __ffs(fm) - 1 : 32);
    const bool dead = c_dead || (int)lane > fl;
    // record bases and the timestamp before each segment
    uint64_t n = (valid && !dead) ? W.n : 0;
    uint64_t incl = n;
    for (int d = 1; d < 32; d <<= 1) { const uint64_t v = __shfl_up_sync(0xffffffffu, incl, d); if ((int)lane >= d) incl += v; }
    const uint64_t base = c_base + incl - n;
    // last ts of the nearest preceding segment with records
    int src = n ? (int)lane : -1;
    int pre = __shfl_up_sync(0xffffffffu, src, 1);
    if (lane == 0) pre = -1;
    for (int d = 1; d < 32; d <<= 1) { const int v = __shfl_up_sync(0xffffffffu, pre, d); if ((int)lane >= d) pre = max(pre, v); }
    const uint64_t pl = __shfl_sync(0xffffffffu, W.last_ts, pre < 0 ? 0 : pre);
    const uint64_t prev_ts = pre >= 0 ? pl : c_last;
    const bool has_prev = pre >= 0 || c_has;
    if (valid) {
      SegInfo I;
      I.entry = W.spec_entry;
      I.base = base;
      I.prev_ts = prev_ts;
      I.n = (uint32_t)n;
      I.flags = (has_prev ? SI_HAS_PREV : 0u) | (dead ? SI_DEAD : 0u) | ((int)lane == fl ? SI_HDR_FAIL : 0u);
      info[g] = I;
      if ((int)lane == fl) {  // the failing header: the error the muxer would hit on that stream
        const uint64_t a = W.fail_off;
        uint32_t code;
        uint64_t aux = 0, ts_f = 0;
        if (a + 16 > size) code = HG_ERR_TRUNC_HEADER;
        else {
          const uint32_t sid = g32(gbase, a), plen = g32(gbase, a + 12);
          ts_f = g64(gbase, a + 4);
          if (a + 16 + plen > size) code = HG_ERR_TRUNC_PAYLOAD;
          else { code = HG_ERR_UNKNOWN_SCHEMA; aux = sid; }
        }
        const uint64_t plast = n ? W.last_ts : prev_ts;
        push_error(p, code, s, base + n, a, ts_f, (n || has_prev) ? plast : 0, aux);
      }
    }
    // carry to the next 32 segments
    const uint64_t tot = __shfl_sync(0xffffffffu, incl, 31);
    c_base += tot;
    int lastw = -1;
    {
      const uint32_t m = __ballot_sync(0xffffffffu, n != 0);
      lastw = m ? 31 - __clz(m) : -1;
    }
    if (lastw >= 0) { c_last = __shfl_sync(0xffffffffu, W.last_ts, lastw); c_has = true; }
    c_exit = __shfl_sync(0xffffffffu, W.exit, 31);
    if (fl < 32) c_dead = true;
  }
  if (lane == 0) {
    stream_nrec[s] = c_base;
    // IntervalStats.events_in and the global last timestamp (pipeline.py:152): every
    // record of an error-free run is decoded, and timestamps rise along each stream
    if (c_base) atomicAdd(&p.stats[ST_EVENTS], (unsigned long long)c_base);
    if (c_has) atomicMax(p.last_ts, (unsigned long long)c_last);
  }
}
#endif  // HG_SEG_KERNELS

// ---------------------------------------------------------------------------
// decode + pair + tally: thread per segment, warp-convergent loop
//
// Each iteration of the warp loop every lane either decodes one record of its
// current segment or closes it and opens its next one.  Host entry/exit records
// (the bulk) are handled inline; work whose cost varies per record -- payload
// validation of variable records (strings: strict UTF-8), device-profiling and
// telemetry records -- is queued per warp and drained 32 at a time with every
// lane active, so one lane's long record does not stall the other 31.

constexpr int kSQ = 64;            // deferred payload validations per warp (drained at 32)
constexpr int kSQD = 40;           // deferred device/telemetry records per warp (drained at 8)
constexpr int kSegNameSlots = 128; // CTA cache of device-name hashes

struct SegSmem {
  uint32_t tab, lanetab, lanetab_warp, dcache, ncache, warps, warp_bytes, total;
};

__host__ __device__ inline SegSmem seg_smem_layout(uint32_t n_fn) {
  SegSmem L;
  uint32_t off = (uint32_t)(((sizeof(uint2) * kSdescMax) + 127) & ~(size_t)127);
  const bool small = n_fn <= kSmallF;
  L.tab = off;
  if (!small && n_fn <= kSmemFnMax) off += (uint32_t)((sizeof(SmemRow) * n_fn + 127) & ~(size_t)127);
  L.lanetab = off;
  L.lanetab_warp = small ? (uint32_t)((((size_t)3 * n_fn * kWarp + 3 * n_fn) * 4 + 127) & ~(size_t)127) : 0u;
  off += L.lanetab_warp * kSegWarps;
  L.dcache = off;
  off += (uint32_t)((sizeof(DevRow) * kDevSlots + 127) & ~(size_t)127);
  L.ncache = off;
  off += (uint32_t)((sizeof(NameSlot) * kSegNameSlots + 127) & ~(size_t)127);
  L.warps = off;
  // per warp: open-entry stack [kLS][32] (ts 8, meta 4, seq 4), pending exits [kLP][32]
  // (ts 8, result 8, meta 4, seq 4), two deferred queues (off 8, seq 8, prev 8, s 4, g 4, sid 4, plen 4)
  L.warp_bytes = (uint32_t)(kLS * kWarp * 16 + kLP * kWarp * 24 + (kSQ + kSQD) * 40);
  off += L.warp_bytes * kSegWarps;
  L.total = off;
  return L;
}

struct LaneStack {
  uint64_t* e_ts;    // [kLS][32] (pointers pre-offset by lane)
  uint32_t* e_meta;
  uint32_t* e_seq;
  uint64_t* p_ts;    // [kLP][32]
  uint64_t* p_res;
  uint32_t* p_meta;  // fn | SumEntry flags << 19
  uint32_t* p_seq;
  SumEntry* deep;    // global chunk [pending..., entries...] once the shared slots overflow
  uint32_t np, ne;
};

struct SegQ {        // per-warp deferred queue (shared, SoA)
  uint64_t* off;
  uint64_t* seq;
  uint64_t* prev;
  uint32_t* s;
  uint32_t* g;       // segment | order-violation flag << 31
  uint32_t* sid;
  uint32_t* plen;
};

__device__ __forceinline__ uint8_t* seg_warp_base(const SegSmem& L) {
  return g_smem + L.warps + (threadIdx.x >> 5) * L.warp_bytes;
}

__device__ __forceinline__ LaneStack lane_stack(const SegSmem& L) {
  const uint32_t lane = lane_id();
  uint8_t* b = seg_warp_base(L);
  LaneStack S;
  S.e_ts = reinterpret_cast<uint64_t*>(b) + lane;
  S.e_meta = reinterpret_cast<uint32_t*>(b + kLS * kWarp * 8) + lane;
  S.e_seq = reinterpret_cast<uint32_t*>(b + kLS * kWarp * 12) + lane;
  uint8_t* q = b + kLS * kWarp * 16;
  S.p_ts = reinterpret_cast<uint64_t*>(q) + lane;
  S.p_res = reinterpret_cast<uint64_t*>(q + kLP * kWarp * 8) + lane;
  S.p_meta = reinterpret_cast<uint32_t*>(q + kLP * kWarp * 16) + lane;
  S.p_seq = reinterpret_cast<uint32_t*>(q + kLP * kWarp * 20) + lane;
  S.deep = nullptr;
  S.np = S.ne = 0;
  return S;
}

// queue 0: payload validations (kSQ entries); queue 1: device/telemetry work (kSQD)
__device__ __forceinline__ SegQ seg_queue(const SegSmem& L, int which) {
  const uint32_t cap = which ? kSQD : kSQ;
  uint8_t* b = seg_warp_base(L) + kLS * kWarp * 16 + kLP * kWarp * 24 + (which ? kSQ * 40 : 0);
  SegQ Q;
  Q.off = reinterpret_cast<uint64_t*>(b);
  Q.seq = reinterpret_cast<uint64_t*>(b + cap * 8);
  Q.prev = reinterpret_cast<uint64_t*>(b + cap * 16);
  Q.s = reinterpret_cast<uint32_t*>(b + cap * 24);
  Q.g = reinterpret_cast<uint32_t*>(b + cap * 28);
  Q.sid = reinterpret_cast<uint32_t*>(b + cap * 32);
  Q.plen = reinterpret_cast<uint32_t*>(b + cap * 36);
  return Q;
}

__device__ __forceinline__ uint32_t* seg_lanetab(const SegSmem& L) {
  return reinterpret_cast<uint32_t*>(g_smem + L.lanetab + (threadIdx.x >> 5) * L.lanetab_warp);
}

// move the lane's automaton state to a global chunk (capacity: the segment's record count)
__device__ __forceinline__ bool go_deep(const Params& p, LaneStack& S, uint64_t base, uint32_t cap) {
  const unsigned long long off = atomicAdd(p.deep_used, (unsigned long long)cap);
  if (off + cap > p.deep_cap) return false;  // the host grows the pool and reruns
  SumEntry* d = p.deep + off;
  for (uint32_t i = 0; i < S.np; i++) {
    SumEntry e;
    e.ts = S.p_ts[i * kWarp]; e.result = S.p_res[i * kWarp];
    const uint32_t m = S.p_meta[i * kWarp];
    e.fn = (m & M_FN) == M_FN ? -1 : (int32_t)(m & M_FN);
    e.flags = m >> 19;
    e.seq = base + S.p_seq[i * kWarp];
    d[i] = e;
  }
  for (uint32_t i = 0; i < S.ne; i++) {
    SumEntry e;
    e.ts = S.e_ts[i * kWarp]; e.result = 0;
    const uint32_t m = S.e_meta[i * kWarp];
    e.fn = m == M_FN ? -1 : (int32_t)m;
    e.flags = 0;
    e.seq = base + S.e_seq[i * kWarp];
    d[S.np + i] = e;
  }
  S.deep = d;
  return true;
}

struct SegCounters {
  uint32_t passed, host, dev, samples, orph, items;
};

// the lane's current segment
struct LaneSeg {
  const uint8_t* gbase;
  uint64_t o;          // next record offset
  uint64_t base;       // stream record index of the segment's first record
  uint64_t prev_ts;
  uint64_t slot0;      // timeline slot of the segment's first record
  Hdr nh;              // header of record k, loaded one record ahead
  uint32_t g, s, n, k;
  uint32_t spans;
  bool have_prev, failed, res_done, hdr_fail;
};

// ---- strict UTF-8 / hashing / comparison on HBM bytes

static __device__ __noinline__ bool g_utf8_slow(const uint8_t* g, uint64_t o, uint32_t n) {
  uint32_t i = 0;
  while (i < n) {
    const uint32_t c = g32(g, o + i) & 0xffu;
    if (c < 0x80) { i++; continue; }
    uint32_t need, lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) need = 1;
    else if (c >= 0xE0 && c <= 0xEF) { need = 2; lo = c == 0xE0 ? 0xA0 : 0x80; hi = c == 0xED ? 0x9F : 0xBF; }
    else if (c >= 0xF0 && c <= 0xF4) { need = 3; lo = c == 0xF0 ? 0x90 : 0x80; hi = c == 0xF4 ? 0x8F : 0xBF; }
    else return false;
    if (i + need >= n) return false;
    const uint32_t d1 = g32(g, o + i + 1) & 0xffu;
    if (d1 < lo || d1 > hi) return false;
    for (uint32_t k = 2; k <= need; k++) {
      const uint32_t dk = g32(g, o + i + k) & 0xffu;
      if (dk < 0x80 || dk > 0xBF) return false;
    }
    i += need + 1;
  }
  return true;
}

__device__ __forceinline__ bool g_utf8(const uint8_t* g, uint64_t o, uint32_t n) {
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4)
    if (g32(g, o + i) & 0x80808080u) return g_utf8_slow(g, o, n);
  if (i < n && (g32(g, o + i) & (0xffffffffu >> (8 * (4 - (n - i))))) & 0x80808080u) return g_utf8_slow(g, o, n);
  return true;
}

__device__ __forceinline__ uint64_t g_hash(const uint8_t* g, uint64_t o, uint32_t n) {
  uint64_t h = 0x9E3779B97F4A7C15ull ^ ((uint64_t)n * 0xff51afd7ed558ccdull);
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4) {
    h ^= g32(g, o + i);
    h *= 0x100000001b3ull;
    h ^= h >> 29;
  }
  if (i < n) {
    h ^= g32(g, o + i) & (0xffffffffu >> (8 * (4 - (n - i))));
    h *= 0x100000001b3ull;
  }
  h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return h | 1ull;
}

// the row's length, offset and bytes were written by another SM during this kernel (published by
// its fence + vals store).  A read through L1 / the read-only cache can only be stale the other way
// (a sector cached before the row was written): equal bytes there mean equal names (a stale match
// would need a 64-bit hash collision), a mismatch is confirmed at L2 (ld.global.cg) before the
// lookup believes it -- else a stale line could make a second row for one name
template <bool kL2>
__device__ __forceinline__ bool g_name_equal_at(const NameDict& d, uint32_t row, const uint8_t* g, uint64_t o, uint32_t n) {
  const uint32_t len = kL2 ? __ldcg(&d.name_len[row]) : d.name_len[row];
  if (len != n) return false;
  const uint64_t off = kL2 ? (uint64_t)__ldcg(reinterpret_cast<const unsigned long long*>(d.name_off) + row) : d.name_off[row];
  const uint32_t* a = reinterpret_cast<const uint32_t*>(d.arena + off);
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4)
    if ((kL2 ? __ldcg(a + (i >> 2)) : a[i >> 2]) != g32(g, o + i)) return false;
  if (i < n) {
    const uint32_t m = 0xffffffffu >> (8 * (4 - (n - i)));
    if (((kL2 ? __ldcg(a + (i >> 2)) : a[i >> 2]) & m) != (g32(g, o + i) & m)) return false;
  }
  return true;
}

__device__ __forceinline__ bool g_name_equal(const NameDict& d, uint32_t row, const uint8_t* g, uint64_t o, uint32_t n) {
  return g_name_equal_at<false>(d, row, g, o, n) || g_name_equal_at<true>(d, row, g, o, n);
}

// device-name dictionary lookup/insert (same layout, hash and probing as name_lookup)
static __device__ __noinline__ uint32_t g_name_lookup(const NameDict& d, const uint8_t* g, uint64_t o, uint32_t n, uint64_t h) {
  for (uint64_t slot = h & d.mask, probes = 0; probes <= d.mask; slot = (slot + 1) & d.mask, probes++) {
    // a plain read first: names already in the dictionary cost no atomic (hot names are shared by
    // every SM, so an atomicCAS per lookup would serialise on a few L2 lines)
    unsigned long long k = *(volatile unsigned long long*)&d.keys[slot];
    if (k == 0ull) k = atomicCAS(&d.keys[slot], 0ull, (unsigned long long)h);
    if (k == 0ull) {
      const uint32_t row = atomicAdd(d.n_rows, 1u);
      const unsigned long long off = atomicAdd(d.arena_used, (unsigned long long)((n + 3u) & ~3u));
      if (row >= d.row_cap || off + n > d.arena_cap) {
        atomicExch(d.overflow, 1u);
        atomicExch(&d.vals[slot], 0xffffffffu);
        return 0xffffffffu;
      }
      uint32_t* dst = reinterpret_cast<uint32_t*>(d.arena + off);
      for (uint32_t i = 0; i < n; i += 4) {
        uint32_t wv = g32(g, o + i);
        if (n - i < 4) wv &= 0xffffffffu >> (8 * (4 - (n - i)));
        dst[i >> 2] = wv;
      }
      d.name_off[row] = off;
      d.name_len[row] = n;
      __threadfence();
      atomicExch(&d.vals[slot], row + 1);
      return row;
    }
    if (k == h) {
      uint32_t v;
      while ((v = *(volatile uint32_t*)&d.vals[slot]) == 0) __nanosleep(32);
      if (v == 0xffffffffu) return 0xffffffffu;
      __threadfence();
      if (g_name_equal(d, v - 1, g, o, n)) return v - 1;
    }
  }
  atomicExch(d.overflow, 1u);
  return 0xffffffffu;
}

// variable payload through the schema's plan, reading HBM (tracefile.py:152-169);
// false -> the generic walk decides (and names the exact error)
__device__ __forceinline__ bool g_var_plan(const DSchema* sc, const uint8_t* g, uint64_t body, uint32_t plen,
                                           uint32_t seg[5]) {
  const uint32_t nv = sc->nvar;
  if (nv == kNoPlan) return false;
  uint32_t q = 0;
  seg[0] = 0;
  #pragma unroll
  for (uint32_t i = 0; i < 4; i++) {
    if (i < nv) {
      q += sc->lead[i];
      if (q + 4 > plen) return false;
      const uint32_t ln = g32(g, body + q);
      q += 4;
      if ((uint64_t)q + ln > plen) return false;
      if (sc->vkind[i] && !g_utf8(g, body + q, ln)) return false;
      q += ln;
      seg[i + 1] = q;
    }
  }
  q += sc->lead[nv];
  return q == plen;
}

// payload validation + role field locations of one record (var records: plan or
// generic walk).  role_ptr: field data (var fields: first byte after the length);
// role_len: var field lengths.
static __device__ __noinline__ uint32_t seg_fields(const Params& p, const uint8_t* g, uint64_t size, uint64_t a, uint32_t sid,
                                           uint32_t plen, uint64_t* role_ptr, uint32_t* role_len, uint64_t& aux,
                                           uint32_t roles) {
  // roles: bit mask of the HG_ROLE_* fields wanted (their schemas have them)
  const uint2 d = desc_of(p, sid);
  const DSchema* sc = schema_of(p, sid);
  const uint64_t body = a + 16;
  if (!(d_flags(d) & SF_VAR)) {
    for (uint32_t m = roles; m; m &= m - 1) {
      const int r = __ffs(m) - 1;
      role_ptr[r] = body + 8u * (uint32_t)sc->role[r];
    }
    return 0;
  }
  uint32_t seg[5];
  if (g_var_plan(sc, g, body, plen, seg)) {
    for (uint32_t m = roles; m; m &= m - 1) {
      const int r = __ffs(m) - 1;
      const uint64_t at = body + seg_sel(seg, sc->role_seg[r]) + sc->role_delta[r];
      if (sc->role_kind[r] >= HG_KIND_STRING) { role_len[r] = g32(g, at); role_ptr[r] = at + 4; }
      else role_ptr[r] = at;
    }
    return 0;
  }
  for (int r = 0; r < HG_NUM_ROLES; r++) { role_ptr[r] = 0; role_len[r] = 0; }
  Window w;
  w.s = nullptr; w.win_start = 0; w.win_end = 0; w.g = g; w.size = size;
  uint32_t name_len = 0;
  const uint32_t e = walk_fields(p, d, sid, body, plen, [&](uint64_t x) { return g32(g, x); }, w, role_ptr, name_len, aux);
  if (e) return e;
  for (int r = 0; r < HG_NUM_ROLES; r++)
    if (sc->role[r] >= 0 && sc->role_kind[r] >= HG_KIND_STRING) role_len[r] = g32(g, role_ptr[r] - 4);
  return 0;
}

// device-profiling record (pipeline.py:186-202): duration into its name's row
static __device__ __noinline__ uint32_t seg_device(const Params& p, const SegSmem L, const uint8_t* g, uint64_t size,
                                           uint32_t sid, const uint64_t* rp, const uint32_t* rl, uint64_t& aux) {
  const uint2 d = desc_of(p, sid);
  if (d_flags(d) & SF_FEED_ALWAYS) { aux = sid; return HG_ERR_FEED; }
  const DSchema* sc = schema_of(p, sid);
  const uint64_t ua = g64(g, rp[HG_ROLE_START]), ub = g64(g, rp[HG_ROLE_END]);
  const int64_t ah = (sc->role_kind[HG_ROLE_START] == HG_KIND_I64 && (int64_t)ua < 0) ? -1 : 0;
  const int64_t bh = (sc->role_kind[HG_ROLE_END] == HG_KIND_I64 && (int64_t)ub < 0) ? -1 : 0;
  const uint64_t d_lo = ub - ua;
  const int64_t d_hi = bh - ah - (ub < ua ? 1 : 0);
  const uint64_t no = rp[HG_ROLE_NAME];
  const uint32_t nl = rl[HG_ROLE_NAME];
  DevRow* dcache = reinterpret_cast<DevRow*>(g_smem + L.dcache);
  NameSlot* ncache = reinterpret_cast<NameSlot*>(g_smem + L.ncache);
  const uint64_t h = g_hash(g, no, nl);
  NameSlot* slot = &ncache[h % kSegNameSlots];
  const unsigned long long ch = *(volatile unsigned long long*)&slot->hash;
  const uint32_t cr = *(volatile uint32_t*)&slot->row;
  uint32_t row = 0xffffffffu;
  if (ch == h && cr < *(volatile uint32_t*)p.names.n_rows && g_name_equal(p.names, cr, g, no, nl)) row = cr;
  if (row == 0xffffffffu) {
    (void)size;
    row = g_name_lookup(p.names, g, no, nl, h);
    if (row != 0xffffffffu) { slot->row = row; __threadfence_block(); slot->hash = h; }
  }
  if (row != 0xffffffffu) fold_device(p, dcache, row, d_lo, d_hi);
  return 0;
}

// telemetry sample checks (pipeline.py:203-215; sampler.py:44-48)
static __device__ __noinline__ uint32_t seg_telemetry(const Params& p, const uint8_t* g, uint32_t sid, const uint64_t* rp,
                                              uint64_t& aux) {
  const uint2 d = desc_of(p, sid);
  const uint32_t fl = d_flags(d);
  if (fl & SF_FEED_ALWAYS) { aux = sid; return HG_ERR_FEED; }
  const DSchema* sc = schema_of(p, sid);
  const uint64_t bits = g64(g, rp[HG_ROLE_VALUE]);
  const uint8_t vk = sc->role_kind[HG_ROLE_VALUE];
  const bool util = sc->counter_kind >= HG_COUNTER_COMPUTE;
  bool bad;
  if (vk == HG_KIND_F64) {
    const double v = __longlong_as_double((long long)bits);
    bad = util ? !(v >= 0.0 && v <= 1.0) : (v < 0.0);
  } else if (vk == HG_KIND_I64) {
    const int64_t v = (int64_t)bits;
    bad = util ? !(v >= 0 && v <= 1) : (v < 0);
  } else {
    bad = util ? (bits > 1) : false;
  }
  if (bad) { aux = bits; return HG_ERR_TELEMETRY; }
  if ((fl & SF_FEED_TIMELINE) && (p.want & (HG_WANT_TIMELINE | HG_WANT_TL_ITEMS))) { aux = sid; return HG_ERR_FEED; }
  return 0;
}

__device__ __forceinline__ void seg_item(const Params& p, uint64_t slot, uint64_t khi, uint64_t klo, uint64_t a,
                                         uint64_t b, uint32_t kind, uint32_t x) {
  TlItem it;
  it.khi = khi; it.klo = klo; it.a = a; it.b = b; it.kind = kind; it.x = x;
  p.tl_items[slot] = it;
}

__device__ __forceinline__ void seg_hole(const Params& p, uint64_t slot) {
  p.tl_items[slot].khi = ~0ull;
  p.tl_items[slot].klo = ~0ull;
}

// a segment's final state; deferred errors may raise it to TS_ERROR later (max)
__device__ __forceinline__ void seg_status(const Params& p, uint32_t g, uint32_t code) {
  __threadfence();
  atomicMax(&p.state[g].status, (p.epoch << 2) | code);
}

// drain n deferred records, one per lane
// payload validation of variable records (tracefile.py:152-169); the exact error
// (and the ordering error it takes precedence over) comes from the full walk
static __device__ __noinline__ void seg_drain_v(const Params& p, const SegSmem L, uint32_t n) {
  const SegQ Q = seg_queue(L, 0);
  const uint32_t lane = lane_id();
  if (lane < n) {
    const uint64_t a = Q.off[lane];
    const uint32_t s = Q.s[lane], sid = Q.sid[lane], plen = Q.plen[lane];
    const uint8_t* gb = p.data + p.stream_base[s];
    uint32_t segs[5];
    if (!g_var_plan(schema_of(p, sid), gb, a + 16, plen, segs)) {
      uint64_t rp[HG_NUM_ROLES];
      uint32_t rl[HG_NUM_ROLES];
      uint64_t aux = 0;
      const uint32_t err = seg_fields(p, gb, p.stream_size[s], a, sid, plen, rp, rl, aux, 0u);
      if (err) {
        push_error(p, err, s, Q.seq[lane], a, g64(gb, a + 4), Q.prev[lane], aux);
        seg_status(p, Q.g[lane] & 0x7FFFFFFFu, TS_ERROR);
      }
    }
  }
  __syncwarp();
}

// device-profiling / telemetry records and ordering-failed variable records
static __device__ __noinline__ uint4 seg_drain(const Params& p, const SegSmem L, uint32_t n) {
  uint4 K = make_uint4(0, 0, 0, 0);  // device spans, samples, timeline messages
  const SegQ Q = seg_queue(L, 1);
  const uint32_t lane = lane_id();
  if (lane < n) {
    const uint64_t a = Q.off[lane], seq = Q.seq[lane], prev = Q.prev[lane];
    const uint32_t s = Q.s[lane], gq = Q.g[lane];
    const uint32_t g = gq & 0x7FFFFFFFu;
    const bool order_bad = (gq >> 31) != 0;
    const uint8_t* gb = p.data + p.stream_base[s];
    const uint64_t size = p.stream_size[s];
    const Hdr h = g_hdr(gb, a);
    const uint2 d = desc_of(p, h.sid);
    const uint32_t cls = d_cls(d);
    uint64_t rp[HG_NUM_ROLES];
    uint32_t rl[HG_NUM_ROLES];
    uint64_t aux = 0;
    uint32_t err = 0;
    const uint32_t roles = cls == HG_CLASS_DEVICE ? ((1u << HG_ROLE_START) | (1u << HG_ROLE_END) | (1u << HG_ROLE_NAME))
                           : cls == HG_CLASS_TELEMETRY ? (1u << HG_ROLE_VALUE) : 0u;
    const bool feed_always = (d_flags(d) & SF_FEED_ALWAYS) != 0;  // role fields may be missing
    uint32_t segs[5];
    if (roles || !g_var_plan(schema_of(p, h.sid), gb, a + 16, h.plen, segs))  // validation only: the plan suffices
      err = seg_fields(p, gb, size, a, h.sid, h.plen, rp, rl, aux, feed_always ? 0u : roles);
    bool feed = false;
    if (!err && order_bad) err = HG_ERR_ORDER;
    if (!err && !order_bad) {
      if (cls == HG_CLASS_DEVICE) err = seg_device(p, L, gb, size, h.sid, rp, rl, aux);
      else if (cls == HG_CLASS_TELEMETRY) err = seg_telemetry(p, gb, h.sid, rp, aux);
      feed = err != 0;
    }
    if (err) {
      push_error(p, err, s, seq, a, h.ts, feed ? 0 : prev, aux);
      seg_status(p, g, TS_ERROR);
    } else if (cls == HG_CLASS_DEVICE || cls == HG_CLASS_TELEMETRY) {
      const bool dev = cls == HG_CLASS_DEVICE;
      if (dev) { K.x++; atomicAdd(&p.stream_spans[s], 1ull); }
      else K.y++;
      if (p.tl_items) {
        seg_item(p, p.tl_rec_off[s] + seq, h.ts, tl_klo(s, seq), (uint64_t)(gb + a + 16), 0, dev ? TL_DEVICE : TL_SAMPLE,
                 h.sid);
        K.z++;
      }
    }
  }
  __syncwarp();
  return K;
}

// open the lane's next live segment at or after g (dead ones are closed on the way)
__device__ __forceinline__ bool seg_begin(const Params& p, const SegInfo* info, uint32_t g, LaneSeg& C) {
  for (; g < p.n_tiles; g += gridDim.x * blockDim.x) {
    const SegInfo I = info[g];
    if (I.flags & SI_DEAD) {
      SegState* st = &p.state[g];
      st->pool_n_pending = 0; st->pool_n_resid = 0; st->pool_off = 0;
      seg_status(p, g, TS_ERROR);
      continue;
    }
    const uint32_t s = p.tile_stream[g];
    C.g = g; C.s = s;
    C.gbase = p.data + p.stream_base[s];
    C.o = I.entry; C.base = I.base; C.prev_ts = I.prev_ts; C.n = I.n; C.k = 0;
    if (I.n) C.nh = g_hdr(C.gbase, I.entry);
    C.have_prev = (I.flags & SI_HAS_PREV) != 0;
    C.hdr_fail = (I.flags & SI_HDR_FAIL) != 0;
    C.failed = false; C.res_done = false; C.spans = 0;
    C.slot0 = p.tl_items ? p.tl_rec_off[s] + I.base : 0;
    return true;
  }
  C.g = p.n_tiles;
  return false;
}

// segment summary for compose_kernel: pending exits, then open entries bottom..top
__device__ __forceinline__ void seg_end(const Params& p, LaneSeg& C, LaneStack& S) {
  const uint32_t sum_n = S.np + S.ne;
  const unsigned long long poff = sum_n ? atomicAdd(p.pool_used, (unsigned long long)sum_n) : 0ull;
  SegState* st = &p.state[C.g];
  st->pool_off = poff;
  st->pool_n_pending = S.np;
  st->pool_n_resid = S.ne;
  if (C.spans) atomicAdd(&p.stream_spans[C.s], (unsigned long long)C.spans);
  if (poff + sum_n <= p.pool_cap) {
    for (uint32_t i = 0; i < sum_n; i++) {
      SumEntry e;
      if (S.deep) {
        e = S.deep[i];
      } else if (i < S.np) {
        e.ts = S.p_ts[i * kWarp]; e.result = S.p_res[i * kWarp];
        const uint32_t m = S.p_meta[i * kWarp];
        e.fn = (m & M_FN) == M_FN ? -1 : (int32_t)(m & M_FN);
        e.flags = m >> 19;
        e.seq = C.base + S.p_seq[i * kWarp];
      } else {
        const uint32_t j = i - S.np;
        e.ts = S.e_ts[j * kWarp]; e.result = 0;
        const uint32_t m = S.e_meta[j * kWarp];
        e.fn = m == M_FN ? -1 : (int32_t)m;
        e.flags = 0;
        e.seq = C.base + S.e_seq[j * kWarp];
      }
      p.pool[poff + i] = e;
    }
  }
  seg_status(p, C.g, (C.failed || C.hdr_fail) ? TS_ERROR : TS_DONE);
  S.deep = nullptr;
  S.np = S.ne = 0;
}

// result offset of a variable-payload exit whose result follows a string/blob (rare)
static __device__ __noinline__ uint64_t var_result_off(const Params& p, const uint8_t* g, uint64_t size, uint64_t a, uint32_t sid,
                                               uint32_t plen) {
  uint64_t rp[HG_NUM_ROLES];
  uint32_t rl[HG_NUM_ROLES];
  uint64_t aux = 0;
  if (seg_fields(p, g, size, a, sid, plen, rp, rl, aux, 1u << HG_ROLE_RESULT)) return kNone;  // invalid payload: the drain reports it
  return rp[HG_ROLE_RESULT];
}

static __device__ __noinline__ void seg_prologue(const Params& p, const SegSmem L) {
  const uint32_t lane = lane_id();
  if (p.max_sid < (uint32_t)kSdescMax) {
    uint2* t = reinterpret_cast<uint2*>(g_smem);
    for (uint32_t i = threadIdx.x; i <= p.max_sid; i += blockDim.x) t[i] = __ldg(&p.desc[i]);
  }
  if (p.n_fn <= kSmallF) {
    uint32_t* b = seg_lanetab(L);
    const uint32_t n = p.n_fn * kWarp;
    for (uint32_t i = lane; i < 3 * n; i += kWarp) b[i] = 0;
    for (uint32_t i = lane; i < p.n_fn; i += kWarp) { b[3 * n + i] = 0; b[3 * n + p.n_fn + i] = 0xFFFFFFFFu; b[3 * n + 2 * p.n_fn + i] = 0; }
  } else if (p.n_fn <= kSmemFnMax) {
    SmemRow* tab = reinterpret_cast<SmemRow*>(g_smem + L.tab);
    for (uint32_t i = threadIdx.x; i < p.n_fn; i += blockDim.x) {
      SmemRow z; z.count = z.err = z.s0 = z.s1 = 0; z.mn = 0xFFFFFFFFu; z.mx = 0;
      tab[i] = z;
    }
  }
  DevRow* dcache = reinterpret_cast<DevRow*>(g_smem + L.dcache);
  for (uint32_t i = threadIdx.x; i < kDevSlots; i += blockDim.x) {
    DevRow z; z.tag = 0; z.count = 0; z.s0 = z.s1 = z.s2 = z.pad = 0; z.mn = 0xFFFFFFFFu; z.mx = 0;
    dcache[i] = z;
  }
  NameSlot* ncache = reinterpret_cast<NameSlot*>(g_smem + L.ncache);
  for (uint32_t i = threadIdx.x; i < kSegNameSlots; i += blockDim.x) { ncache[i].hash = 0; ncache[i].row = 0; }
  __syncthreads();
}

static __device__ __noinline__ void seg_epilogue(const Params& p, const SegSmem L, const SegCounters K) {
  const uint32_t lane = lane_id();
  auto wsum = [](uint32_t v) { return __reduce_add_sync(0xffffffffu, v); };
  // events and the last timestamp come from the chain (every record of an error-free run is decoded)
  const uint32_t a1 = wsum(K.passed), a2 = wsum(K.host), a3 = wsum(K.dev), a4 = wsum(K.samples),
                 a5 = wsum(K.orph), a6 = wsum(K.items);
  if (lane == 0) {
    if (a1) atomicAdd(&p.stats[ST_PASSED], (unsigned long long)a1);
    if (a2) atomicAdd(&p.stats[ST_HOST], (unsigned long long)a2);
    if (a3) atomicAdd(&p.stats[ST_DEVICE], (unsigned long long)a3);
    if (a4) atomicAdd(&p.stats[ST_SAMPLES], (unsigned long long)a4);
    if (a5) atomicAdd(&p.stats[ST_ORPHANS], (unsigned long long)a5);
    if (a6) atomicAdd(p.tl_n, (unsigned long long)a6);  // record-indexed timeline messages
  }
  __syncthreads();
  const uint32_t nn = p.n_fn * kWarp;
  if (p.n_fn <= kSmallF) {
    const uint32_t* lt = seg_lanetab(L);
    for (uint32_t f = 0; f < p.n_fn; f++) {
      const uint32_t i = f * kWarp + lane;
      uint64_t cc = lt[i], sum = ((uint64_t)lt[2 * nn + i] << 32) | lt[nn + i];
      if (!__any_sync(0xffffffffu, cc != 0)) continue;
      for (int d = 16; d; d >>= 1) {
        cc += __shfl_xor_sync(0xffffffffu, cc, d);
        sum += __shfl_xor_sync(0xffffffffu, sum, d);
      }
      if (lane == 0 && cc) {
        unsigned long long* a = p.host_acc + 6ull * f;
        atomicAdd(&a[0], (unsigned long long)cc);
        if (lt[3 * nn + f]) atomicAdd(&a[1], (unsigned long long)lt[3 * nn + f]);
        add_i128(&a[2], &a[3], sum, 0);
        atomicMin(&a[4], (unsigned long long)lt[3 * nn + p.n_fn + f]);
        atomicMax(&a[5], (unsigned long long)lt[3 * nn + 2 * p.n_fn + f]);
      }
    }
  } else if (p.n_fn <= kSmemFnMax) {
    const SmemRow* tab = reinterpret_cast<const SmemRow*>(g_smem + L.tab);
    for (uint32_t f = threadIdx.x; f < p.n_fn; f += blockDim.x) {
      const SmemRow r = tab[f];
      if (!r.count) continue;
      unsigned long long* a = p.host_acc + 6ull * f;
      atomicAdd(&a[0], (unsigned long long)r.count);
      if (r.err) atomicAdd(&a[1], (unsigned long long)r.err);
      add_i128(&a[2], &a[3], (uint64_t)r.s0 | ((uint64_t)r.s1 << 32), 0);
      atomicMin(&a[4], (unsigned long long)r.mn);
      atomicMax(&a[5], (unsigned long long)r.mx);
    }
  }
  const DevRow* dcache = reinterpret_cast<const DevRow*>(g_smem + L.dcache);
  for (uint32_t i = threadIdx.x; i < kDevSlots; i += blockDim.x) {
    const DevRow r = dcache[i];
    if (!r.tag || !r.count) continue;
    unsigned long long* a = p.dev_acc + 6ull * (r.tag - 1);
    atomicAdd(&a[0], (unsigned long long)r.count);
    add_i128(&a[2], &a[3], (uint64_t)r.s0 | ((uint64_t)r.s1 << 32), (int64_t)(int32_t)r.s2);
    atomicMin(&a[4], bias64((int64_t)(int32_t)(r.mn ^ 0x80000000u)));
    atomicMax(&a[5], bias64((int64_t)(int32_t)(r.mx ^ 0x80000000u)));
  }
}

// one record with every check and rare case (errors, variable payloads, pending or
// orphan exits, deep stacks, f64 results); returns true when the record is deferred
// returns 0 (nothing deferred), 1 (payload validation queue) or 2 (device/telemetry queue)
__device__ __forceinline__ uint32_t seg_record_full(const Params& p, LaneSeg& C, LaneStack& S, SegCounters& K,
                                                    HostFold& hf, bool tl, uint64_t& q_off, uint64_t& q_prev,
                                                    bool& order_bad, uint32_t& q_sid, uint32_t& q_plen) {
  uint32_t defer = 0;
  const uint32_t k = C.k++;
  const uint64_t a = C.o;
  const Hdr h = C.nh;
  C.o = a + 16 + h.plen;
  C.nh = g_hdr(C.gbase, C.o);
  const uint2 d = desc_of(p, h.sid);
  const uint32_t cls = d_cls(d), fl = d_flags(d);
  const bool var = (fl & SF_VAR) != 0;
  const bool ob = C.have_prev && h.ts < C.prev_ts;   // pipeline.py:98
  if (!var && h.plen != d_fixed(d)) {                 // tracefile.py:210
    push_error(p, HG_ERR_LEN_MISMATCH, C.s, C.base + k, a, h.ts, C.have_prev ? C.prev_ts : 0, 0);
    C.failed = true;
  } else if (ob && !var) {
    push_error(p, HG_ERR_ORDER, C.s, C.base + k, a, h.ts, C.prev_ts, 0);
    C.failed = true;
  } else {
    // payload checks of variable records, device and telemetry work: deferred
    const bool dt = cls == HG_CLASS_DEVICE || cls == HG_CLASS_TELEMETRY;
    defer = (dt || ob) ? 2u : (var ? 1u : 0u);
    q_off = a;
    q_prev = C.have_prev ? C.prev_ts : 0;
    q_sid = h.sid;
    q_plen = h.plen;
    order_bad = ob;
    if (ob) C.failed = true;  // var record: the drain names payload error or ordering
  }
  if (C.failed) return defer;
  C.prev_ts = h.ts;
  C.have_prev = true;
  bool item = cls == HG_CLASS_DEVICE || cls == HG_CLASS_TELEMETRY;  // written by the drain
  if (cls == HG_CLASS_ENTRY) {
    const uint32_t m = d.x & M_FN;
    if (!S.deep && S.ne < (uint32_t)kLS) {
      S.e_ts[S.ne * kWarp] = h.ts; S.e_meta[S.ne * kWarp] = m; S.e_seq[S.ne * kWarp] = k;
    } else {
      if (!S.deep && !go_deep(p, S, C.base, C.n)) C.failed = true;
      if (S.deep) {
        SumEntry e;
        e.ts = h.ts; e.seq = C.base + k; e.fn = (m == M_FN) ? -1 : (int32_t)m; e.flags = 0; e.result = 0;
        S.deep[S.np + S.ne] = e;
      }
    }
    S.ne++;
  } else if (cls == HG_CLASS_EXIT) {
    const int32_t fn = (d.x & M_FN) == M_FN ? -1 : (int32_t)(d.x & M_FN);
    uint64_t res = 0;
    uint32_t xf = 1u | (result_kind(fl) << 4);  // SumEntry flags: exit | err | bad | nan | kind << 4
    if (fl & SF_RESULT) {
      uint64_t ro = a + 16 + 8u * d_resfield(d);
      if (var) {
        const DSchema* sc = schema_of(p, h.sid);
        ro = (sc->role_seg[HG_ROLE_RESULT] == 0 && sc->nvar != kNoPlan && sc->role_delta[HG_ROLE_RESULT] + 8u <= h.plen)
                 ? a + 16 + sc->role_delta[HG_ROLE_RESULT]
                 : var_result_off(p, C.gbase, p.stream_size[C.s], a, h.sid, h.plen);
      }
      res = ro == kNone ? 0 : g64(C.gbase, ro);
      if (fl & SF_RESULT_F64) {
        const double xv = __longlong_as_double((long long)res);
        if (isnan(xv)) xf |= 4u | 8u;
        else if (isinf(xv)) xf |= 4u;
        else if (xv >= 1.0 || xv <= -1.0) xf |= 2u;
      } else if (res) {
        xf |= 2u;
      }
    }
    if (S.ne) {  // pipeline.py:156-168: pops a same-function top, else an orphan that does not pop
      uint64_t ets;
      int32_t tfn;
      if (!S.deep) {
        ets = S.e_ts[(S.ne - 1) * kWarp];
        const uint32_t m = S.e_meta[(S.ne - 1) * kWarp];
        tfn = m == M_FN ? -1 : (int32_t)m;
      } else {
        const SumEntry e = S.deep[S.np + S.ne - 1];
        ets = e.ts; tfn = e.fn;
      }
      if (tfn == fn) {
        S.ne--;
        hf.fold(p, fn, h.ts - ets, (xf & 2u) != 0);
        K.host++;
        C.spans++;
        if ((xf & 4u) && !C.res_done) {  // int(NaN/inf) raises only when the exit pairs
          push_error(p, HG_ERR_RESULT, C.s, C.base + k, a, h.ts, 0, res);
          C.res_done = true;
        }
        if (tl) {
          seg_item(p, C.slot0 + k, h.ts, tl_klo(C.s, C.base + k), ets, res, TL_HOST | (((xf >> 4) & 3u) << 4),
                   (uint32_t)fn);
          K.items++;
          item = true;
        }
      } else {
        push_orphan(p, C.s, fn, h.ts, C.base + k);
        K.orph++;
      }
    } else {  // no local entry: the summary decides (compose_kernel)
      if (!S.deep && S.np < (uint32_t)kLP) {
        S.p_ts[S.np * kWarp] = h.ts; S.p_res[S.np * kWarp] = res;
        S.p_meta[S.np * kWarp] = (fn < 0 ? M_FN : (uint32_t)fn) | (xf << 19);
        S.p_seq[S.np * kWarp] = k;
      } else {
        if (!S.deep && !go_deep(p, S, C.base, C.n)) C.failed = true;
        if (S.deep) {
          SumEntry e;
          e.ts = h.ts; e.seq = C.base + k; e.fn = fn; e.flags = xf; e.result = res;
          S.deep[S.np] = e;
        }
      }
      S.np++;
    }
  } else if (cls != HG_CLASS_DEVICE && cls != HG_CLASS_TELEMETRY) {
    K.passed++;
  }
  if (tl && !item) seg_hole(p, C.slot0 + k);
  return defer;
}

#ifdef HG_SEG_KERNELS
__global__ void __launch_bounds__(kSegThreads, 3) seg_decode_kernel(Params p, const SegInfo* info, const Params* gp) {
  // noinline helpers read the parameters from a global copy: taking the address of the
  // kernel parameter block would move every hot-loop parameter read to local memory
  const Params& gpr = *gp;
  const SegSmem L = seg_smem_layout(p.n_fn);
  seg_prologue(gpr, L);
  const uint32_t lane = lane_id();
  SegCounters K;
  K.passed = K.host = K.dev = K.samples = K.orph = K.items = 0;
  HostFold hf;
  hf.small = p.n_fn <= kSmallF;
  hf.tab = (!hf.small && p.n_fn <= kSmemFnMax) ? reinterpret_cast<SmemRow*>(g_smem + L.tab) : nullptr;
  if (hf.small) {
    uint32_t* b = seg_lanetab(L);
    const uint32_t nn = p.n_fn * kWarp;
    hf.lt.cnt = b; hf.lt.slo = b + nn; hf.lt.shi = b + 2 * nn;
    hf.lt.err = b + 3 * nn; hf.lt.mn = b + 3 * nn + p.n_fn; hf.lt.mx = b + 3 * nn + 2 * p.n_fn;
  }
  LaneStack S = lane_stack(L);
  const SegQ QV = seg_queue(L, 0), QD = seg_queue(L, 1);
  const bool tl = p.tl_items != nullptr;
  const bool small = hf.small;
  const uint32_t nn = p.n_fn * kWarp;
  const uint32_t stride = gridDim.x * blockDim.x;
  LaneSeg C;
  bool have = seg_begin(p, info, blockIdx.x * blockDim.x + threadIdx.x, C);
  uint32_t qn = 0, qd = 0;
  while (__any_sync(0xffffffffu, have)) {
    const bool act = have && C.k < C.n && !C.failed;
    // ---- fast path: entry push, matching exit pop, device/telemetry/meta pass-through
    // (in order, shallow stack, integer result; payload checks of variable records
    // other than exits are deferred).  Straight-line code.
    const Hdr h = C.nh;
    const uint64_t a = C.o;
    const uint2 d = act ? desc_of(p, h.sid) : make_uint2(0, 0);
    const uint32_t cls = d_cls(d), fl = d_flags(d);
    const uint32_t fnm = d.x & M_FN;
    const bool isE = cls == HG_CLASS_ENTRY, isX = cls == HG_CLASS_EXIT;
    const bool var = (fl & SF_VAR) != 0;
    // variable exits qualify when their result precedes every string/blob (resfield set)
    const bool ok = act && !(fl & SF_RESULT_F64) &&
                    (var ? (h.plen >= d_fixed(d) && (!isX || !(fl & SF_RESULT) || d_resfield(d) != 0xFFu))
                         : h.plen == d_fixed(d)) &&
                    !(C.have_prev && h.ts < C.prev_ts) && !S.deep;
    const uint32_t top = (S.ne && S.ne <= (uint32_t)kLS ? S.ne - 1 : 0) * kWarp;
    const uint64_t ets = S.e_ts[top];
    const uint32_t tm = S.e_meta[top];
    const bool f_entry = ok && isE && S.ne < (uint32_t)kLS;
    const bool f_exit = ok && isX && S.ne != 0 && tm == fnm;
    const bool f_other = ok && !isE && !isX;
    const bool fast = f_entry || f_exit || f_other;
    uint32_t defer = 0;  // 1: validation queue, 2: device/telemetry queue
    bool order_bad = false;
    uint64_t q_off = a, q_prev = C.prev_ts;
    uint32_t q_sid = h.sid, q_plen = h.plen;
    if (fast) {
      const uint32_t k = C.k++;
      C.o = a + 16 + h.plen;
      C.nh = g_hdr(C.gbase, C.o);  // next header in flight while this record is handled
      if (((C.o + 256) ^ (a + 256)) >> 7)  // entering a new 128-byte line: pull the one two lines ahead into L1
        asm volatile("prefetch.global.L1 [%0];" ::"l"(C.gbase + C.o + 256));

      C.prev_ts = h.ts;
      C.have_prev = true;
      if (f_entry) {
        const uint32_t at = S.ne * kWarp;
        S.e_ts[at] = h.ts; S.e_meta[at] = fnm; S.e_seq[at] = k;
        S.ne++;
      }
      const bool dev_or_tel = cls == HG_CLASS_DEVICE || cls == HG_CLASS_TELEMETRY;
      defer = dev_or_tel ? 2u : (var ? 1u : 0u);
      if (f_other && !dev_or_tel) K.passed++;
      uint64_t res = 0;
      if (f_exit) {
        S.ne--;
        if (fl & SF_RESULT) res = g64(C.gbase, a + 16 + 8u * d_resfield(d));
        const uint64_t dur = h.ts - ets;
        const bool err = res != 0;
        if (small && (dur >> 32) == 0) {
          const uint32_t i = fnm * kWarp + lane, du = (uint32_t)dur;
          hf.lt.cnt[i] += 1;
          const uint32_t lo = hf.lt.slo[i] + du;
          hf.lt.shi[i] += lo < du ? 1u : 0u;
          hf.lt.slo[i] = lo;
          if (err) atomicAdd(&hf.lt.err[fnm], 1u);
          if (du < *(volatile uint32_t*)&hf.lt.mn[fnm]) atomicMin(&hf.lt.mn[fnm], du);
          if (du > *(volatile uint32_t*)&hf.lt.mx[fnm]) atomicMax(&hf.lt.mx[fnm], du);
        } else {
          hf.fold(gpr, (int32_t)fnm, dur, err);
        }
        K.host++;
        C.spans++;
      }
      if (tl) {
        if (f_exit) {
          seg_item(p, C.slot0 + k, h.ts, tl_klo(C.s, C.base + k), ets, res,
                   TL_HOST | (result_kind(fl) << 4), fnm);
          K.items++;
        } else if (!dev_or_tel) {
          seg_hole(p, C.slot0 + k);
        }
      }
    }
    const bool slow = act && !fast;
    if (__any_sync(0xffffffffu, slow)) {
      if (slow) defer = seg_record_full(gpr, C, S, K, hf, tl, q_off, q_prev, order_bad, q_sid, q_plen);
    }
    const bool ending = have && !act;
    if (__any_sync(0xffffffffu, ending)) {
      if (ending) {
        seg_end(p, C, S);
        have = seg_begin(p, info, C.g + stride, C);
      }
    }
    const uint32_t qm = __ballot_sync(0xffffffffu, defer == 1u);
    if (qm) {
      if (defer == 1u) {
        const uint32_t i = qn + __popc(qm & lanemask_lt());
        QV.off[i] = q_off; QV.seq[i] = C.base + C.k - 1; QV.prev[i] = q_prev; QV.s[i] = C.s; QV.g[i] = C.g;
        QV.sid[i] = q_sid; QV.plen[i] = q_plen;
      }
      qn += __popc(qm);
      __syncwarp();
      if (qn >= (uint32_t)kWarp) {
        seg_drain_v(gpr, L, kWarp);
        qn -= kWarp;
        if (lane < qn) {
          QV.off[lane] = QV.off[kWarp + lane]; QV.seq[lane] = QV.seq[kWarp + lane]; QV.prev[lane] = QV.prev[kWarp + lane];
          QV.s[lane] = QV.s[kWarp + lane]; QV.g[lane] = QV.g[kWarp + lane];
          QV.sid[lane] = QV.sid[kWarp + lane]; QV.plen[lane] = QV.plen[kWarp + lane];
        }
        __syncwarp();
      }
    }
    const uint32_t dm = __ballot_sync(0xffffffffu, defer == 2u);
    if (dm) {
      if (defer == 2u) {
        const uint32_t i = qd + __popc(dm & lanemask_lt());
        QD.off[i] = q_off; QD.seq[i] = C.base + C.k - 1; QD.prev[i] = q_prev; QD.s[i] = C.s;
        QD.g[i] = C.g | (order_bad ? 0x80000000u : 0u);
        QD.sid[i] = q_sid; QD.plen[i] = q_plen;
      }
      qd += __popc(dm);
      __syncwarp();
      if (qd >= 8u) {  // device work is rarer: drain smaller batches to keep the queue short
        const uint32_t nd = qd < (uint32_t)kWarp ? qd : (uint32_t)kWarp;
        const uint4 dk = seg_drain(gpr, L, nd);
        K.dev += dk.x; K.samples += dk.y; K.items += dk.z;
        qd -= nd;
        if (lane < qd) {
          QD.off[lane] = QD.off[nd + lane]; QD.seq[lane] = QD.seq[nd + lane]; QD.prev[lane] = QD.prev[nd + lane];
          QD.s[lane] = QD.s[nd + lane]; QD.g[lane] = QD.g[nd + lane];
          QD.sid[lane] = QD.sid[nd + lane]; QD.plen[lane] = QD.plen[nd + lane];
        }
        __syncwarp();
      }
    }
  }
  (void)nn;
  if (qn) seg_drain_v(gpr, L, qn);
  if (qd) {
    const uint4 dk = seg_drain(gpr, L, qd);
    K.dev += dk.x; K.samples += dk.y; K.items += dk.z;
  }
  seg_epilogue(gpr, L, K);
}
#endif  // HG_SEG_KERNELS

// exclusive scan of per-stream record totals -> timeline slot offset of each stream
#ifdef HG_SEG_KERNELS
__global__ void __launch_bounds__(1024) seg_rec_off_kernel(const unsigned long long* stream_nrec, uint32_t n,
                                                           unsigned long long* off, unsigned long long* total) {
  unsigned long long carry = 0;
  for (uint32_t b0 = 0; b0 < n; b0 += 1024) {
    const uint32_t i = b0 + threadIdx.x;
    const uint64_t v = i < n ? stream_nrec[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_excl_scan(v, &tot);
    if (i < n) off[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}
#endif  // HG_SEG_KERNELS

}  // namespace hg
