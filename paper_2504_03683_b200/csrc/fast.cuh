// fast.cuh -- phase 1 in ONE pass over HBM: the range kernel (sm_100a).
//
// Every stream is cut into contiguous byte ranges, one range per resident lane
// (total_bytes / resident lanes each, so the grid is a single wave).  A lane
// runs the reference's sequential algorithm over its range:
//   decode every record (tracefile.py:147-215), the per-stream ordering check
//   (pipeline.py:98), the IntervalBuilder LIFO automaton (pipeline.py:156-185)
//   and the tally fold (sinks.py:123-132, 230-242),
// reading the bytes from a private 256-byte ring in shared memory (8 slots of
// 32 B, read with wrapped word indices).  Every iteration a lane whose oldest slot
// is consumed copies its next 32 bytes itself with two 16-byte cp.async.cg
// (LDGSTS: L2 -> shared, bypassing L1); one commit group per iteration and
// `cp.async.wait_group kRLag` prove every fill older than kRLag iterations
// complete, so readiness is a popcount of the lane's request shift register.  HBM
// is read once; every record access on the inline path is an LDS.
//
// Range starts are speculative (first offset with eight consistent record
// headers).  fast_verify_kernel then checks, per stream, that every range
// starts where the previous one ended and that timestamps keep rising across
// ranges; it turns the range summaries into compose_kernel's input (pending
// exits, open entries) and the record bases.  Anything the single pass does
// not reproduce exactly -- any decode / ordering / telemetry error, a wrong
// speculation, a NaN/inf f64 result -- sets `anom`, and the host discards the
// pass and runs the exact three-kernel path (seg.cuh), which reports errors
// with the reference's precedence.  A clean trace therefore costs one read.
#pragma once
#include "seg.cuh"

namespace hg {

constexpr uint32_t kRChunk = 32;                    // bytes per ring slot (one sector)
#ifndef HG_RING_SLOTS
#define HG_RING_SLOTS 8
#endif
#ifndef HG_RINLINE
#define HG_RINLINE 128
#endif
#ifndef HG_FAST_WARPS
#define HG_FAST_WARPS 12
#endif
constexpr uint32_t kRSlots = HG_RING_SLOTS;         // slots per lane
constexpr uint32_t kRRing = kRChunk * kRSlots;      // 256-byte ring
constexpr uint32_t kRWordMask = kRRing / 4 - 1;
constexpr uint32_t kRMirror = 0;                    // (no mirror: header words are read with wrapped indices)
constexpr uint32_t kRStride = kRRing + kRMirror;    // ring bytes per lane: header + first field need no wrap
constexpr uint32_t kRInline = HG_RINLINE;           // records up to this long are decoded from the ring
#ifndef HG_RLAG
#define HG_RLAG 2  // C2 x1.0 phase 1: lag 1 1.888 ms, 2 1.875, 3 1.880
#endif
constexpr int kRLag = HG_RLAG;                            // iterations before a fill group is waited for
constexpr int kRLS = 4;                             // open entries per lane in shared memory: the stack's top
                                                    // window (depth d in slot d % kRLS), older ones spilled
constexpr int kRLP = 4;                             // pending exits per lane in shared memory
constexpr int kRQ = 64;                             // deferred-record queues per warp (drained at 32)
constexpr uint32_t kRDeepHalf = 64;                 // per-lane overflow chunk (SumEntry): pending exits beyond
constexpr uint32_t kRDepthMax = 72;                 // kRLP at [0, 64), open entries of depth d at 64 + d
constexpr uint32_t kRDeep = kRDeepHalf + kRDepthMax;
#ifndef HG_RNAMES
#define HG_RNAMES 512  // 64 -> 256 slots of 64 B: C2 phase 1 1.99 -> 1.90 ms, C5 x0.25 1.96 -> 1.91 ms; 512 of 32 B, 2-way
#endif
constexpr uint32_t kRNames = HG_RNAMES;    // CTA name cache: 2-way sets of 32-byte slots (seq, row | len << 24,
constexpr uint32_t kRNameMax = 40;         // hash bits 32-63, name); register strings up to kRNameMax bytes
constexpr uint32_t kRNameCache = 20;       // names up to this long are cached
#ifndef HG_RWAYS
#define HG_RWAYS 1  // C5 x1.0 phase 1: 1 way 6.71 ms, 2 ways 6.94, 4 ways 7.21 (probes cost more than misses)
#endif
constexpr uint32_t kRWays = HG_RWAYS;      // ways per set

struct RangeState {
  uint64_t entry;      // speculative first record (kNone: no plausible header in the range)
  uint64_t exit;       // offset after the last record
  uint64_t first_ts, last_ts;
  uint64_t pool_off;   // summary: np pending exits, then ne open entries (bottom..top)
  uint32_t n, np, ne, pad;
};

// single-field variable payload plan per schema id (vplan): valid << 31 | string << 30 |
// trailing fixed bytes << 14 | leading fixed bytes
constexpr uint32_t VP_VALID = 1u << 31, VP_STR = 1u << 30;

struct RSmem {
  uint32_t tab, lanetab, lanetab_warp, dcache, ncache, fdesc, warps, warp_bytes, total;
  uint32_t ring, st_ts, st_fn, pd_ts, pd_meta, pd_k, q_off, q_s, qs_off, qs_s, ftab, ferr;  // within a warp block
};

__host__ __device__ inline uint32_t r_align(uint32_t x) { return (x + 127u) & ~127u; }

// n_fd: inline-record descriptors staged in shared memory as uint4 (0: read through L1); n_cd: the
// same as 4-byte compact descriptors (large registries: max_sid >= kSdescMax, desc_of reads HBM, so
// they take its place); dev: the registry has device schemas (else no CTA name cache)
__host__ __device__ inline RSmem fast_smem_layout(uint32_t n_fn, uint32_t nw, uint32_t n_fd, uint32_t n_cd = 0,
                                                  bool dev = true) {
  RSmem L;
  // desc_of's table (kernels.cuh; max_sid + 1 entries when max_sid < kSdescMax, else it reads HBM) or cdesc
  uint32_t off = n_cd ? r_align(4u * n_cd) : n_fd ? r_align(8u * n_fd) : 0u;
  const bool small = n_fn <= kSmallF;
  L.tab = off;
  if (!small && n_fn <= kSmemFnMax) off += r_align((uint32_t)sizeof(SmemRow) * n_fn);
  L.lanetab = off;  // unused (the per-lane fold table lives in the warp block)
  L.lanetab_warp = 0;
  L.dcache = off;
  off += r_align((uint32_t)sizeof(DevRow) * kDevSlots);
  L.ncache = off;  // kRNames x 64 B seqlocked name cache (fast.cuh), not seg.cuh's NameSlot table
  off += dev ? 32u * kRNames : 0u;
  L.fdesc = off;
  off += r_align(16u * n_fd);
  L.warps = off;
  uint32_t w = 0;
  L.ring = w;    w += kRStride * kWarp;
  L.ftab = w;    w += small ? 8u * n_fn * kWarp : 0u;   // [fn][lane] count << 44 | sum
  L.ferr = w;    w += small ? 12u * n_fn : 0u;          // [fn] error count, min, max
  w = (w + 15u) & ~15u;
  L.st_ts = w;   w += 8u * kRLS * kWarp;
  L.st_fn = w;   w += 4u * kRLS * kWarp;
  L.pd_ts = w;   w += 8u * kRLP * kWarp;
  L.pd_meta = w; w += 4u * kRLP * kWarp;
  L.pd_k = w;    w += 4u * kRLP * kWarp;
  L.q_off = w;   w += 8u * kRQ;   // device / telemetry records
  L.qs_off = w;  w += 8u * kRQ;   // string payloads to validate
  L.q_s = w;     w += 4u * kRQ;
  L.qs_s = w;    w += 4u * kRQ;
  L.warp_bytes = r_align(w);
  off += L.warp_bytes * nw;
  L.total = off;
  return L;
}

// SegSmem view of the shared tables, for the helpers shared with seg.cuh
__device__ __forceinline__ SegSmem r_segsmem(const RSmem& R) {
  SegSmem L;
  L.tab = R.tab; L.lanetab = R.lanetab; L.lanetab_warp = R.lanetab_warp; L.dcache = R.dcache; L.ncache = R.ncache;
  L.warps = R.warps; L.warp_bytes = R.warp_bytes; L.total = R.total;
  return L;
}

__device__ __forceinline__ uint32_t s_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- ring reads (the ring word index wraps)

__device__ __forceinline__ uint32_t r_u32(const uint32_t* ring, uint32_t bp) {
  const uint32_t wi = bp >> 2;
  return __funnelshift_r(ring[wi & kRWordMask], ring[(wi + 1) & kRWordMask], (bp & 3u) << 3);
}
__device__ __forceinline__ uint64_t r_u64(const uint32_t* ring, uint32_t bp) {
  const uint32_t wi = bp >> 2, sh = (bp & 3u) << 3;
  const uint32_t a = ring[wi & kRWordMask], b = ring[(wi + 1) & kRWordMask], c = ring[(wi + 2) & kRWordMask];
  return ((uint64_t)__funnelshift_r(b, c, sh) << 32) | __funnelshift_r(a, b, sh);
}

// ---- the lane's range (offsets relative to C0, the 128-aligned start of ring chunk 0)

struct RLane {
  const uint8_t* g;     // stream bytes from C0
  uint64_t C0;          // stream offset of chunk 0
  uint64_t size;        // stream size - C0
  uint32_t size32;      // min(size, 2^32 - 1)
  uint64_t prev_ts, first_ts;
  SumEntry* deep;       // overflow chunk (nullptr until needed)
  uint32_t o, t1, entry;
  uint32_t r, s, n, spans;
  uint32_t ci, clast;   // chunks requested, last chunk this range reads
  uint32_t recent;      // bit i: a chunk was requested i iterations ago (its fill group may be pending)
  uint32_t np, ne;
  uint32_t nw;          // open entries in the shared top window (depths ne - nw .. ne - 1); kept once `deep`
                        // exists (before, nothing was spilled: the window holds all ne)
  uint32_t ti;          // timeline messages of this range so far (timeline runs)
  bool bad;
  bool fresh;           // no requests until every pending fill of this lane completed (slot reuse)
};

// one record of the lane's range for the event sinks: slot k of the range (its index in the range);
// a = the record's offset in the data array (ev_line)
__device__ __forceinline__ void r_event(const Params& p, const RLane& R, uint32_t k, uint64_t ts, uint64_t o,
                                        uint32_t sid) {
  TlItem it;
  it.khi = ts; it.klo = k; it.a = (uint64_t)(R.g - p.data) + o; it.b = 0; it.kind = 0; it.x = sid;
  p.ev_ritems[(uint64_t)R.r * p.tl_rcap + k] = it;
}

// one timeline message of the lane's range, in record order (k: the record's index in the range)
__device__ __forceinline__ void r_item(const Params& p, RLane& R, uint64_t khi, uint64_t k, uint64_t a, uint64_t b,
                                       uint32_t kind, uint32_t x) {
  TlItem it;
  it.khi = khi; it.klo = k; it.a = a; it.b = b; it.kind = kind; it.x = x;
  p.tl_ritems[(uint64_t)R.r * p.tl_rcap + R.ti++] = it;
}

// first offset in [t0, t1) that starts a chain of kScanDepth plausible headers with
// non-decreasing timestamps (or a shorter one that ends exactly at the stream end).
// A wrong guess is caught by fast_verify_kernel and costs a whole exact pass, so the
// single pass demands a longer chain than the segment walk (seg_walk_kernel: three).
#ifndef HG_SCAN_DEPTH
#define HG_SCAN_DEPTH 8
#endif
constexpr int kScanDepth = HG_SCAN_DEPTH;

__device__ __forceinline__ bool r_scan_at(const Params& p, const uint8_t* g, uint64_t size, uint64_t o) {
  uint64_t cur = o, nxt, ts, prev = 0;
  int k = 0;
  for (; k < kScanDepth; k++) {
    if (!seg_plausible(p, g, size, cur, nxt, ts) || (k && ts < prev)) break;
    prev = ts;
    cur = nxt;
    if (cur == size) { k = kScanDepth; break; }
  }
  return k == kScanDepth;
}

static __device__ __noinline__ uint64_t r_scan(const Params& p, const uint8_t* g, uint64_t size, uint64_t t0, uint64_t t1) {
  for (uint64_t o = t0; o < t1; o++)
    if (r_scan_at(p, g, size, o)) return o;
  return kNone;
}

// every range's speculative start before the range kernel, one warp per range testing 32
// consecutive offsets at once (the same first offset as r_scan: the lowest lane that passes).
// A lane of the range kernel scanning alone paid one dependent L2/HBM round trip per offset
// at kernel start (4% of C2's stall samples, profiles/r21_*).
#ifdef HG_FAST_KERNELS
__global__ void __launch_bounds__(256) fast_scan_kernel(Params p) {
  if (p.max_sid < (uint32_t)kSdescMax) {  // desc_of reads shared memory for such registries
    uint2* t = reinterpret_cast<uint2*>(g_smem);
    for (uint32_t i = threadIdx.x; i <= p.max_sid; i += blockDim.x) t[i] = __ldg(&p.desc[i]);
    __syncthreads();
  }
  const uint32_t lane = lane_id();
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < p.n_ranges; r += nwarps) {
    const uint32_t s = p.range_stream[r];
    const uint32_t j = r - p.stream_range0[s];
    uint64_t found = j == 0 ? 16ull : kNone;
    if (j) {
      const uint64_t size = p.stream_size[s];
      const uint8_t* g = p.data + p.stream_base[s];
      const uint64_t t0 = 16 + (uint64_t)j * p.range_bytes;
      const uint64_t t1 = min(t0 + (uint64_t)p.range_bytes, size);
      for (uint64_t base = t0; base < t1; base += kWarp) {
        const uint64_t o = base + lane;
        const uint32_t m = __ballot_sync(0xffffffffu, o < t1 && r_scan_at(p, g, size, o));
        if (m) { found = base + (uint32_t)(__ffs(m) - 1); break; }
      }
    }
    if (lane == 0) p.rstate[r].entry = found;
  }
}
#endif

// open the lane's next range (ranges without a plausible header are recorded and skipped)
__device__ __forceinline__ bool r_begin(const Params& p, RLane& R, uint32_t r, uint32_t stride) {
  for (; r < p.n_ranges; r += stride) {
    const uint32_t s = p.range_stream[r];
    const uint32_t j = r - p.stream_range0[s];
    const uint64_t size = p.stream_size[s];
    const uint8_t* g = p.data + p.stream_base[s];
    const uint64_t t0 = 16 + (uint64_t)j * p.range_bytes;
    const uint64_t t1 = min(t0 + (uint64_t)p.range_bytes, size);
    const uint64_t entry = j == 0 ? 16ull : p.prescan ? p.rstate[r].entry : r_scan(p, g, size, t0, t1);
    if (entry == kNone) {
      RangeState st;
      st.entry = kNone; st.exit = kNone; st.first_ts = 0; st.last_ts = 0; st.pool_off = 0;
      st.n = 0; st.np = 0; st.ne = 0; st.pad = 0;
      p.rstate[r] = st;
      if (p.tl_rn) p.tl_rn[r] = 0;
      if (p.ev_rn) p.ev_rn[r] = 0;
      continue;
    }
    R.C0 = entry & ~(uint64_t)(kRChunk - 1);
    R.g = g + R.C0;
    R.size = size - R.C0;
    R.size32 = R.size < 0xFFFFFFFFull ? (uint32_t)R.size : 0xFFFFFFFFu;
    R.o = (uint32_t)(entry - R.C0);
    R.entry = R.o;
    R.t1 = (uint32_t)(t1 - R.C0);
    // chunks this range can read from the ring: records that start before t1 and fit kRInline
    R.clast = (uint32_t)min((size - 1 - R.C0) / kRChunk, (uint64_t)(R.t1 + kRInline - 1) / kRChunk);
    R.ci = 0; R.fresh = true;
    R.prev_ts = 0; R.first_ts = 0;
    R.deep = nullptr;
    R.r = r; R.s = s; R.n = 0; R.spans = 0; R.np = 0; R.ne = 0; R.nw = 0; R.ti = 0; R.bad = false;
    return true;
  }
  R.r = p.n_ranges;
  R.o = R.t1 = R.entry = 0; R.C0 = 0; R.size = 0; R.size32 = 0; R.g = p.data;
  R.n = R.np = R.ne = R.nw = R.ci = R.clast = R.ti = 0;
  R.bad = false; R.fresh = true;
  return false;
}

struct RTabs {           // the lane's views of its warp block
  uint64_t* st_ts; uint32_t* st_fn;                     // [kRLS][32], pre-offset by lane
  uint64_t* pd_ts; uint32_t* pd_meta; uint32_t* pd_k;   // [kRLP][32]
};

__device__ __forceinline__ RTabs r_tabs(const RSmem& L) {
  const uint32_t lane = lane_id();
  uint8_t* b = g_smem + L.warps + (threadIdx.x >> 5) * L.warp_bytes;
  RTabs T;
  T.st_ts = reinterpret_cast<uint64_t*>(b + L.st_ts) + lane;
  T.st_fn = reinterpret_cast<uint32_t*>(b + L.st_fn) + lane;
  T.pd_ts = reinterpret_cast<uint64_t*>(b + L.pd_ts) + lane;
  T.pd_meta = reinterpret_cast<uint32_t*>(b + L.pd_meta) + lane;
  T.pd_k = reinterpret_cast<uint32_t*>(b + L.pd_k) + lane;
  return T;
}

// summary + range state.  Fills still in flight for this lane's slots are harmless:
// the next range requests its chunks in later groups and reads them only once those
// groups are proven complete (groups complete in order).
__device__ __forceinline__ void r_end(const Params& p, RLane& R, const RTabs& T) {
  const uint32_t sum_n = R.np + R.ne;
  const unsigned long long poff = sum_n ? atomicAdd(p.pool_used, (unsigned long long)sum_n) : 0ull;
  if (poff + sum_n <= p.pool_cap) {
    for (uint32_t i = 0; i < R.np; i++) {
      SumEntry e;
      if (i < (uint32_t)kRLP) {
        e.ts = T.pd_ts[i * kWarp];
        e.result = p.tl_pres ? p.tl_pres[(uint64_t)R.r * kRLP + i] : 0ull;  // result bits: the timeline only
        const uint32_t m = T.pd_meta[i * kWarp];
        e.fn = m_fn(m); e.flags = m >> 19; e.seq = T.pd_k[i * kWarp];
      } else {
        e = R.deep[i - kRLP];
      }
      p.pool[poff + i] = e;
    }
    for (uint32_t i = 0; i < R.ne; i++) {
      SumEntry e;
      if (!R.deep || i + R.nw >= R.ne) {  // in the top window
        const uint32_t j = (i & (kRLS - 1)) * kWarp;
        e.ts = T.st_ts[j];
        e.fn = m_fn(T.st_fn[j]);
      } else {                 // spilled (ts and fn only)
        const SumEntry* d = R.deep + kRDeepHalf + i;
        e.ts = d->ts;
        e.fn = d->fn;
      }
      e.seq = 0; e.flags = 0; e.result = 0;
      p.pool[poff + R.np + i] = e;
    }
  }
  RangeState st;
  st.entry = R.C0 + R.entry; st.exit = R.C0 + R.o; st.first_ts = R.first_ts; st.last_ts = R.prev_ts;
  st.pool_off = poff;
  st.n = R.n; st.np = R.np; st.ne = R.ne; st.pad = 0;
  p.rstate[R.r] = st;
  if (p.tl_rn) p.tl_rn[R.r] = R.ti;
  if (p.ev_rn) p.ev_rn[R.r] = R.n;
  if (R.spans) atomicAdd(&p.stream_spans[R.s], (unsigned long long)R.spans);
  if (R.bad) atomicOr(p.anom, 1u);   // anomaly reasons (bits): 1 record, 2 drain, 4 string, 8 chain, 16 order
}

// close the lane's range and open its next one, out of line (rare; the lane state travels by value
// so the hot loop keeps it in registers)
static __device__ __noinline__ RLane r_switch(const Params& p, RLane R, const RTabs T, uint32_t stride) {
  r_end(p, R, T);
  r_begin(p, R, R.r + stride, stride);
  return R;
}

// a per-lane overflow chunk for deep stacks / many pending exits
__device__ __forceinline__ bool r_deep(const Params& p, RLane& R) {
  if (R.deep) return true;
  const unsigned long long off = atomicAdd(p.deep_used, (unsigned long long)kRDeep);
  if (off + kRDeep > p.deep_cap) return false;  // the host grows the pool and reruns
  R.deep = p.deep + off;
  R.nw = R.ne;  // nothing spilled yet
  return true;
}

// the top window is full and depth i is pushed: its slot holds depth i - kRLS, which moves to the chunk
__device__ __forceinline__ void r_spill(RLane& R, const RTabs& T, uint32_t i) {
  const uint32_t j = (i & (kRLS - 1)) * kWarp;
  SumEntry* d = R.deep + kRDeepHalf + (i - kRLS);
  d->ts = T.st_ts[j];
  d->fn = m_fn(T.st_fn[j]);
}

// every record the inline path does not take, decoded from HBM: long records,
// payload plans other than one variable field, deep stacks, orphans, f64 results.
// Returns true when the record goes to the deferred queue.
__device__ __forceinline__ bool r_record_slow(const Params& p, RLane& R, const RTabs& T, SegCounters& K,
                                              const HostFold& hf) {
  const uint64_t a = R.o;  // relative to C0
  if (a + 16 > R.size) { R.bad = true; return false; }           // truncated header
  const Hdr h = g_hdr(R.g, a);
  const uint2 d = desc_of(p, h.sid);
  if (!d_present(d)) { R.bad = true; return false; }             // unknown schema
  const uint64_t L = 16ull + h.plen;
  if (a + L > R.size) { R.bad = true; return false; }            // truncated payload
  const uint32_t cls = d_cls(d), fl = d_flags(d);
  const bool var = (fl & SF_VAR) != 0;
  if (var ? h.plen < d_fixed(d) : h.plen != d_fixed(d)) { R.bad = true; return false; }
  if (R.n && h.ts < R.prev_ts) { R.bad = true; return false; }  // MuxOrderingError
  if (fl & SF_FEED_ALWAYS) { R.bad = true; return false; }
  const bool dt = cls == HG_CLASS_DEVICE || cls == HG_CLASS_TELEMETRY;
  uint64_t rp[HG_NUM_ROLES];
  uint32_t rl[HG_NUM_ROLES];
  uint64_t aux = 0;
  const bool want_res = cls == HG_CLASS_EXIT && (fl & SF_RESULT);
  if (var && !dt) {  // stream offsets for seg_fields: C0 is 128-aligned, so alignment is unchanged
    if (seg_fields(p, R.g, R.size, a, h.sid, h.plen, rp, rl, aux, want_res ? (1u << HG_ROLE_RESULT) : 0u)) {
      R.bad = true;
      return false;
    }
  }
  const uint32_t k = R.n++;
  if (!k) R.first_ts = h.ts;
  R.prev_ts = h.ts;
  R.o = (uint32_t)(a + L);
  if (p.ev_ritems) r_event(p, R, k, h.ts, a, h.sid);
  if (dt) {
    if (cls == HG_CLASS_DEVICE) R.spans++;  // a device span's identity (sinks.py:240-242)
    if (p.tl_ritems) r_item(p, R, h.ts, k, reinterpret_cast<uint64_t>(R.g + a + 16), 0,
                            cls == HG_CLASS_DEVICE ? TL_DEVICE : TL_SAMPLE, h.sid);
    return true;
  }
  const uint32_t fnm = d.x & M_FN;
  if (cls == HG_CLASS_ENTRY) {
    const uint32_t i = R.ne;
    if (i >= kRDepthMax) { R.bad = true; return false; }
    if (R.deep || i >= (uint32_t)kRLS) {
      if (!r_deep(p, R)) { R.bad = true; return false; }
      if (R.nw == (uint32_t)kRLS) r_spill(R, T, i);  // the window is full: its oldest entry (depth i - kRLS, same slot) moves
      else R.nw++;
    }
    T.st_ts[(i & (kRLS - 1)) * kWarp] = h.ts; T.st_fn[(i & (kRLS - 1)) * kWarp] = fnm;
    R.ne = i + 1;
  } else if (cls == HG_CLASS_EXIT) {
    uint64_t res = 0;
    uint32_t xf = 1u | (result_kind(fl) << 4);
    if (want_res) {
      const uint64_t ro = var ? rp[HG_ROLE_RESULT] : a + 16 + 8u * (uint32_t)schema_of(p, h.sid)->role[HG_ROLE_RESULT];
      res = g64(R.g, ro);
      if (fl & SF_RESULT_F64) {
        const double xv = __longlong_as_double((long long)res);
        if (isnan(xv) || isinf(xv)) { R.bad = true; return false; }  // int() raises if it pairs: exact path
        if (xv >= 1.0 || xv <= -1.0) xf |= 2u;
      } else if (res) {
        xf |= 2u;
      }
    }
    const uint32_t ne = R.ne;
    if (ne) {  // pipeline.py:156-168
      uint64_t ets;
      uint32_t tfn;
      if (!R.deep || R.nw) {
        ets = T.st_ts[((ne - 1) & (kRLS - 1)) * kWarp]; tfn = T.st_fn[((ne - 1) & (kRLS - 1)) * kWarp];
      } else {
        const SumEntry* e = R.deep + kRDeepHalf + ne - 1;
        ets = e->ts; tfn = e->fn < 0 ? M_FN : (uint32_t)e->fn;
      }
      if (tfn == fnm) {
        R.ne = ne - 1;
        R.nw -= R.nw ? 1u : 0u;
        hf.fold(p, (int32_t)fnm, h.ts - ets, (xf & 2u) != 0);
        K.host++;
        R.spans++;
        if (p.tl_ritems) r_item(p, R, h.ts, k, ets, res, TL_HOST | (result_kind(fl) << 4), fnm);
      } else {
        push_orphan(p, R.s, m_fn(fnm), h.ts, (1ull << 63) | ((uint64_t)R.r << 24) | k);
        K.orph++;
      }
    } else {  // no local entry: compose decides
      const uint32_t i = R.np;
      if (i < (uint32_t)kRLP) {
        T.pd_ts[i * kWarp] = h.ts; T.pd_meta[i * kWarp] = fnm | (xf << 19);
        T.pd_k[i * kWarp] = k;
        if (p.tl_pres) p.tl_pres[(uint64_t)R.r * kRLP + i] = res;
      } else {
        if (i >= (uint32_t)kRLP + kRDeepHalf || !r_deep(p, R)) { R.bad = true; return false; }
        SumEntry e;
        e.ts = h.ts; e.seq = k; e.fn = m_fn(fnm); e.flags = xf; e.result = res;
        R.deep[i - kRLP] = e;
      }
      R.np = i + 1;
    }
  } else {
    K.passed++;
  }
  return false;
}

// ---- device-name cache: (hash, row, name bytes) slots under a sequence lock in shared memory,
// filled by the drain after a global dictionary lookup; a hit avoids the dictionary's atomics

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// ---- strings of up to kRNameMax bytes in registers: the words are loaded in one round trip
// (aligned loads, funnel-shifted with a static index), then checked, hashed and compared there
constexpr uint32_t kDW = kRNameMax / 4;

// the kRNameMax bytes at o as words (the stream is 256-aligned and the data buffer zero-padded by
// kDataPad, so reading past a short string is safe); every load is issued before any is used
__device__ __forceinline__ void r_words(const uint8_t* g, uint64_t o, uint32_t (&w)[kDW]) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(g) + (o >> 2);
  const uint32_t sh = (uint32_t)(o & 3) * 8;
  uint32_t r[kDW + 1];
  #pragma unroll
  for (uint32_t j = 0; j <= kDW; j++) r[j] = __ldg(p + j);
  #pragma unroll
  for (uint32_t j = 0; j < kDW; j++) w[j] = __funnelshift_r(r[j], r[j + 1], sh);
}

// zero every byte from n on (n <= kRNameMax)
__device__ __forceinline__ void r_words_mask(uint32_t (&w)[kDW], uint32_t n) {
  #pragma unroll
  for (uint32_t j = 0; j < kDW; j++)
    w[j] = 4 * j >= n ? 0u : 4 * j + 4 <= n ? w[j] : w[j] & (0xffffffffu >> (8 * (4 - (n - 4 * j))));
}

__device__ __forceinline__ bool r_words_ascii(const uint32_t (&w)[kDW]) {
  uint32_t acc = 0;
  #pragma unroll
  for (uint32_t j = 0; j < kDW; j++) acc |= w[j];
  return (acc & 0x80808080u) == 0;
}

// strict UTF-8 (tracefile.py:165) of n bytes at o: all-ASCII checked kRNameMax bytes per round trip
// (g_utf8's word loop waits for every load before the next), anything else by the byte automaton
__device__ __forceinline__ bool r_utf8(const uint8_t* g, uint64_t o, uint32_t n) {
  for (uint32_t i = 0; i < n; i += kRNameMax) {
    uint32_t w[kDW];
    r_words(g, o + i, w);
    r_words_mask(w, min(n - i, kRNameMax));
    if (!r_words_ascii(w)) return g_utf8_slow(g, o, n);
  }
  return true;
}

// g_hash (seg.cuh) over register words
__device__ __forceinline__ uint64_t r_words_hash(const uint32_t (&w)[kDW], uint32_t n) {
  uint64_t h = 0x9E3779B97F4A7C15ull ^ ((uint64_t)n * 0xff51afd7ed558ccdull);
  #pragma unroll
  for (uint32_t j = 0; j < kDW; j++) {
    if (4 * j + 4 <= n) {
      h ^= w[j];
      h *= 0x100000001b3ull;
      h ^= h >> 29;
    } else if (4 * j < n) {
      h ^= w[j];
      h *= 0x100000001b3ull;
    }
  }
  h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return h | 1ull;
}

// CTA name cache (device rows by kernel name): set h % (kRNames / kRWays), kRWays 32-byte ways (one: direct mapped) under a
// sequence lock each; a hit needs the length, hash bits 32-63 and every name byte to match, so the
// cache never changes which row a name gets (the global dictionary decides, seg.cuh g_name_lookup)
__device__ __forceinline__ uint32_t r_name_probe_w(uint32_t nc_s, uint64_t h, const uint32_t (&w)[kDW], uint32_t nl) {
  if (nl > kRNameCache) return 0xffffffffu;
  const uint32_t set = nc_s + (uint32_t)(h & (kRNames / kRWays - 1)) * 32u * kRWays;
  #pragma unroll
  for (uint32_t way = 0; way < kRWays; way++) {
    const uint32_t slot = set + 32u * way;
    uint32_t s1;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(s1) : "r"(slot) : "memory");
    if (!s1 || (s1 & 1u)) continue;
    const uint32_t rl = lds32(slot + 4), hh = lds32(slot + 8);
    if ((rl >> 24) != nl || hh != (uint32_t)(h >> 32)) continue;
    uint32_t diff = 0;
    #pragma unroll
    for (uint32_t j = 0; j < kRNameCache / 4; j++)
      if (4 * j < nl) diff |= lds32(slot + 12 + 4 * j) ^ w[j];  // both zero beyond nl
    if (diff) continue;
    uint32_t s2;
    asm volatile("membar.cta; ld.volatile.shared.u32 %0, [%1];" : "=r"(s2) : "r"(slot) : "memory");
    if (s2 == s1) return rl & 0xFFFFFFu;
  }
  return 0xffffffffu;
}

// fill a way of the name's set (an empty one, else the way picked by hash bits 40-)
__device__ __forceinline__ void r_name_fill_w(uint32_t nc_s, uint64_t h, uint32_t row, const uint32_t (&w)[kDW],
                                              uint32_t nl) {
  if (nl > kRNameCache || row > 0xFFFFFFu) return;
  const uint32_t set = nc_s + (uint32_t)(h & (kRNames / kRWays - 1)) * 32u * kRWays;
  uint32_t way = (uint32_t)(h >> 40) & (kRWays - 1), s = 0;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(s) : "r"(set + 32u * way) : "memory");
  #pragma unroll
  for (uint32_t k = 0; k < kRWays; k++) {
    uint32_t sk;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(sk) : "r"(set + 32u * k) : "memory");
    if (!sk && s) { way = k; s = 0; }
  }
  const uint32_t slot = set + 32u * way;
  if (s & 1u) return;
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(slot), "r"(s), "r"(s + 1u) : "memory");
  if (old != s) return;
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(slot + 4), "r"(row | (nl << 24)) : "memory");
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(slot + 8), "r"((uint32_t)(h >> 32)) : "memory");
  #pragma unroll
  for (uint32_t j = 0; j < kRNameCache / 4; j++)
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(slot + 12 + 4 * j), "r"(w[j]) : "memory");
  asm volatile("membar.cta; st.volatile.shared.u32 [%0], %1;" ::"r"(slot), "r"(s + 2u) : "memory");
}

// deferred records, one per lane, read from HBM (L2): device-profiling and telemetry
// records (fold / range checks) and string payloads of inline records (UTF-8)
static __device__ __noinline__ uint2 r_drain(const Params& p, const SegSmem L, const uint64_t* q_off, const uint32_t* q_s,
                                      uint32_t n, uint32_t nc_s) {
  uint2 K = make_uint2(0, 0);
  const uint32_t lane = lane_id();
  if (lane < n) {
    const uint64_t a = q_off[lane];
    const uint32_t s = q_s[lane];
    const uint8_t* gb = p.data + p.stream_base[s];
    const uint64_t size = p.stream_size[s];
    const Hdr h = g_hdr(gb, a);
    const uint2 d = desc_of(p, h.sid);
    const uint32_t cls = d_cls(d);
    const uint32_t roles = cls == HG_CLASS_DEVICE ? ((1u << HG_ROLE_START) | (1u << HG_ROLE_END) | (1u << HG_ROLE_NAME))
                           : cls == HG_CLASS_TELEMETRY ? (1u << HG_ROLE_VALUE) : 0u;
    uint64_t rp[HG_NUM_ROLES];
    uint32_t rl[HG_NUM_ROLES];
    uint64_t aux = 0;
    uint32_t err = 0;
    const uint4 dp = cls == HG_CLASS_DEVICE ? __ldg(&p.dplan[h.sid]) : make_uint4(0, 0, 0, 0);
    uint32_t nw_[kDW];     // the name in registers (nreg) when it is at most kRNameMax bytes
    bool nreg = false;
    uint64_t ua_ = 0, ub_ = 0;
    if (dp.y >> 31) {  // usual device layout (dplan): start / end and the first length in one round trip,
                       // the second length and both strings' words in the next
      const uint32_t lead0 = dp.x & 0xFFFFu, lead1 = dp.x >> 16, lead2 = dp.y & 0xFFFFu;
      const uint64_t body = a + 16;
      const uint32_t l0 = g32(gb, body + lead0);
      rp[HG_ROLE_START] = body + (dp.z & 0xFFFFu);
      rp[HG_ROLE_END] = body + (dp.z >> 16);
      ua_ = g64(gb, rp[HG_ROLE_START]);
      ub_ = g64(gb, rp[HG_ROLE_END]);
      if ((uint64_t)lead0 + 4u + l0 + lead1 + 4u > h.plen) {
        err = HG_ERR_TRUNC_VAR;
      } else {
        const uint64_t b1 = body + lead0 + 4u + l0 + lead1;
        const bool second = (dp.y >> 16) & 1u;
        const uint64_t s0 = body + lead0 + 4u, s1 = b1 + 4u;
        const uint32_t l1 = g32(gb, b1);
        uint32_t ow[kDW];  // the other string, when short
        r_words(gb, second ? s0 : s1, ow);
        r_words(gb, second ? s1 : s0, nw_);
        const uint32_t nl = second ? l1 : l0, ol = second ? l0 : l1;
        if ((uint64_t)lead0 + 4u + l0 + lead1 + 4u + l1 + lead2 != h.plen) {
          err = HG_ERR_TRAILING;
        } else {
          const bool nstr = ((dp.y >> (second ? 18 : 17)) & 1u) != 0, ostr = ((dp.y >> (second ? 17 : 18)) & 1u) != 0;
          nreg = nl <= kRNameMax;
          if (nreg) r_words_mask(nw_, nl);
          if (ostr) {
            bool ok;
            if (ol <= kRNameMax) { r_words_mask(ow, ol); ok = r_words_ascii(ow) || g_utf8_slow(gb, second ? s0 : s1, ol); }
            else ok = r_utf8(gb, second ? s0 : s1, ol);
            if (!ok) err = HG_ERR_UTF8;
          }
          if (nstr && !err && !(nreg ? r_words_ascii(nw_) || g_utf8_slow(gb, second ? s1 : s0, nl) : r_utf8(gb, second ? s1 : s0, nl)))
            err = HG_ERR_UTF8;
        }
        rp[HG_ROLE_NAME] = second ? s1 : s0;
        rl[HG_ROLE_NAME] = nl;
      }
    } else if (roles) {
      err = seg_fields(p, gb, size, a, h.sid, h.plen, rp, rl, aux, roles);
    } else {  // the inline record's one string field (length already checked): strict UTF-8
      const uint32_t vp = __ldg(&p.vplan[h.sid]);
      const uint64_t at = a + 16 + (vp & 0x3FFFu);
      if (!r_utf8(gb, at + 4, g32(gb, at))) err = HG_ERR_UTF8;
    }
    if (!err && cls == HG_CLASS_DEVICE) {  // seg_device with the global dictionary, then fill the CTA cache
      if (d_flags(d) & SF_FEED_ALWAYS) {
        err = HG_ERR_FEED;
      } else {
        const DSchema* sc = schema_of(p, h.sid);
        const uint64_t ua = (dp.y >> 31) ? ua_ : g64(gb, rp[HG_ROLE_START]);
        const uint64_t ub = (dp.y >> 31) ? ub_ : g64(gb, rp[HG_ROLE_END]);
        const bool si = (dp.y >> 31) ? ((dp.y >> 19) & 1u) != 0 : sc->role_kind[HG_ROLE_START] == HG_KIND_I64;
        const bool ei = (dp.y >> 31) ? ((dp.y >> 20) & 1u) != 0 : sc->role_kind[HG_ROLE_END] == HG_KIND_I64;
        const int64_t ah = (si && (int64_t)ua < 0) ? -1 : 0;
        const int64_t bh = (ei && (int64_t)ub < 0) ? -1 : 0;
        const uint64_t no = rp[HG_ROLE_NAME];
        const uint32_t nl = rl[HG_ROLE_NAME];
        const uint64_t hh = nreg ? r_words_hash(nw_, nl) : g_hash(gb, no, nl);
        // CTA cache: no global atomics on a hit
        uint32_t row = nreg ? r_name_probe_w(nc_s, hh, nw_, nl) : 0xffffffffu;
        if (row == 0xffffffffu) {
          row = g_name_lookup(p.names, gb, no, nl, hh);
          if (row != 0xffffffffu && nreg) r_name_fill_w(nc_s, hh, row, nw_, nl);
        }
        if (row != 0xffffffffu) {
          fold_device(p, reinterpret_cast<DevRow*>(g_smem + L.dcache), row, ub - ua, bh - ah - (ub < ua ? 1 : 0));
        }
      }
    } else if (!err && cls == HG_CLASS_TELEMETRY) {
      err = seg_telemetry(p, gb, h.sid, rp, aux);
    }
    if (err) {
      atomicOr(p.anom, 2u);
    } else if (cls == HG_CLASS_DEVICE) {
      K.x++;  // its span identity was counted by the record's lane (RLane::spans)
    } else if (cls == HG_CLASS_TELEMETRY) {
      K.y++;
    }
  }
  __syncwarp();
  return K;
}

constexpr int kRMaxThreads = HG_FAST_WARPS * kWarp;

// strict UTF-8 of the one string field of inline records (tracefile.py:165), one per lane, from HBM
static __device__ __noinline__ void r_drain_str(const Params& p, const uint64_t* q_off, const uint32_t* q_s, uint32_t n) {
  const uint32_t lane = lane_id();
  if (lane < n) {
    const uint64_t a = q_off[lane];
    const uint8_t* gb = p.data + p.stream_base[q_s[lane]];
    const uint32_t vp = __ldg(&p.vplan[g32(gb, a)]);
    const uint64_t at = a + 16 + (vp & 0x3FFFu);
    if (!r_utf8(gb, at + 4, g32(gb, at))) atomicOr(p.anom, 4u);
  }
  __syncwarp();
}

// inline-record descriptor (fdesc, one uint4 per schema id, built by hg_set_registry):
// x = function (19 bits) | kind << 20 | flags; y = min payload | max inline payload << 16;
// z = fixed bytes before | after the one variable field (blob / string)
enum : uint32_t { FK_ENTRY = 0, FK_EXIT = 1, FK_PASS = 2, FK_DEFER = 3, FK_NEVER = 7 };
constexpr uint32_t FD_STR = 1u << 23, FD_VAR = 1u << 24, FD_RES = 1u << 25;  // result kind at bits 26-27
constexpr uint32_t FD_ISDEV = 1u << 28;  // device-profiling class

__device__ __forceinline__ void r_cp16p(uint32_t dst, const void* src, uint32_t pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p cp.async.cg.shared.global [%0], [%1], 16; }"
               ::"r"(dst), "l"(src), "r"(pred) : "memory");
}

__device__ __forceinline__ void r_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// per-lane fold table entry: count << 44 | sum (u64), min, max; flushed to the global
// row before the sum can reach 2^44 or the count 2^20 (sinks.py:123-132 TallyRow.fold)
constexpr uint64_t kFCount = 1ull << 44;
constexpr uint64_t kFLimit = (1ull << 43) | (1ull << 63);

static __device__ __noinline__ void r_fold_flush(const Params& p, uint32_t fn, uint64_t cs) {
  unsigned long long* a = p.host_acc + 6ull * fn;
  atomicAdd(&a[0], (unsigned long long)(cs >> 44));
  add_i128(&a[2], &a[3], cs & (kFCount - 1), 0);
}

// 4-byte inline descriptor (large registries): valid << 31 | fdesc.x bits 20-28 (kind, flags) |
// fixed payload length << 12 | function (0xFFF: M_FN); records with a variable field, a function
// id >= 0xFFF or a payload range keep the uint4 (valid = 0: read through L1)
__host__ __device__ inline uint32_t r_compact(uint4 D) {
  const uint32_t fn = D.x & M_FN, lo = D.y & 0xFFFFu, hi = D.y >> 16;
  const uint32_t kind = (D.x >> 20) & 7u;
  if (kind == FK_NEVER) return 0x80000FFFu | (FK_NEVER << 20);
  if ((D.x & FD_VAR) || lo != hi || lo > 0xFFu || (fn >= 0xFFFu && fn != M_FN)) return 0u;
  return 0x80000000u | (D.x & 0x1FF00000u) | (lo << 12) | (fn == M_FN ? 0xFFFu : fn);
}

__device__ __forceinline__ uint4 r_expand(uint32_t c) {
  const uint32_t fn = c & 0xFFFu, len = (c >> 12) & 0xFFu;
  return make_uint4((fn == 0xFFFu ? M_FN : fn) | (c & 0x1FF00000u), len | (len << 16), 0u, 0u);
}

// descriptor mode of the range kernel: 1 uint4 table in shared memory (small registries), 2 compact
// table (fits next to 12 warps), 0 through L1
inline int fast_desc_mode(uint32_t max_sid, uint32_t n_fn, bool dev, uint32_t optin, uint32_t& n_fd, uint32_t& n_cd) {
  n_fd = n_cd = 0;
  if (max_sid < (uint32_t)kSdescMax) { n_fd = max_sid + 2; return 1; }
  if (fast_smem_layout(n_fn, HG_FAST_WARPS, 0, max_sid + 2, dev).total <= optin) { n_cd = max_sid + 2; return 2; }
  return 0;
}

__device__ __forceinline__ void r_prologue(const Params& p, const RSmem& RL, uint32_t nw, uint32_t n_fd, uint32_t n_cd) {
  uint4* fd = reinterpret_cast<uint4*>(g_smem + RL.fdesc);
  for (uint32_t i = threadIdx.x; i < n_fd; i += blockDim.x) fd[i] = __ldg(&p.fdesc[i]);
  if (p.max_sid < (uint32_t)kSdescMax) {
    uint2* t = reinterpret_cast<uint2*>(g_smem);
    for (uint32_t i = threadIdx.x; i <= p.max_sid; i += blockDim.x) t[i] = __ldg(&p.desc[i]);
  }
  if (p.n_fn > kSmallF && p.n_fn <= kSmemFnMax) {
    SmemRow* tab = reinterpret_cast<SmemRow*>(g_smem + RL.tab);
    for (uint32_t i = threadIdx.x; i < p.n_fn; i += blockDim.x) {
      SmemRow z; z.count = z.err = z.s0 = z.s1 = 0; z.mn = 0xFFFFFFFFu; z.mx = 0;
      tab[i] = z;
    }
  }
  if (p.n_fn <= kSmallF) {
    uint8_t* wb = g_smem + RL.warps + (threadIdx.x >> 5) * RL.warp_bytes;
    uint64_t* ft = reinterpret_cast<uint64_t*>(wb + RL.ftab);
    for (uint32_t i = lane_id(); i < p.n_fn * kWarp; i += kWarp) ft[i] = 0;
    uint32_t* fe = reinterpret_cast<uint32_t*>(wb + RL.ferr);
    for (uint32_t i = lane_id(); i < p.n_fn; i += kWarp) { fe[i] = 0; fe[p.n_fn + i] = 0xFFFFFFFFu; fe[2 * p.n_fn + i] = 0; }
  }
  DevRow* dcache = reinterpret_cast<DevRow*>(g_smem + RL.dcache);
  for (uint32_t i = threadIdx.x; i < kDevSlots; i += blockDim.x) {
    DevRow z; z.tag = 0; z.count = 0; z.s0 = z.s1 = z.s2 = z.pad = 0; z.mn = 0xFFFFFFFFu; z.mx = 0;
    dcache[i] = z;
  }
  uint32_t* ncache = reinterpret_cast<uint32_t*>(g_smem + RL.ncache);
  if (p.has_dev)
    for (uint32_t i = threadIdx.x; i < kRNames; i += blockDim.x) ncache[8 * i] = 0;  // seq 0: empty
  uint32_t* cd = reinterpret_cast<uint32_t*>(g_smem);
  for (uint32_t i = threadIdx.x; i < n_cd; i += blockDim.x) cd[i] = r_compact(__ldg(&p.fdesc[i]));
  (void)nw;
  __syncthreads();
}

static __device__ __noinline__ void r_epilogue(const Params& p, const RSmem RL, const SegCounters K) {
  const uint32_t lane = lane_id();
  const uint32_t a1 = __reduce_add_sync(0xffffffffu, K.passed), a2 = __reduce_add_sync(0xffffffffu, K.host),
                 a3 = __reduce_add_sync(0xffffffffu, K.dev), a4 = __reduce_add_sync(0xffffffffu, K.samples),
                 a5 = __reduce_add_sync(0xffffffffu, K.orph);
  if (lane == 0) {
    if (a1) atomicAdd(&p.stats[ST_PASSED], (unsigned long long)a1);
    if (a2) atomicAdd(&p.stats[ST_HOST], (unsigned long long)a2);
    if (a3) atomicAdd(&p.stats[ST_DEVICE], (unsigned long long)a3);
    if (a4) atomicAdd(&p.stats[ST_SAMPLES], (unsigned long long)a4);
    if (a5) atomicAdd(&p.stats[ST_ORPHANS], (unsigned long long)a5);
  }
  if (p.n_fn <= kSmallF) {  // per-lane table of this warp
    const uint8_t* wb = g_smem + RL.warps + (threadIdx.x >> 5) * RL.warp_bytes;
    const uint64_t* ft = reinterpret_cast<const uint64_t*>(wb + RL.ftab);
    const uint32_t* fe = reinterpret_cast<const uint32_t*>(wb + RL.ferr);
    for (uint32_t f = 0; f < p.n_fn; f++) {
      const uint64_t cs = ft[f * kWarp + lane];
      uint64_t cnt = cs >> 44, sum = cs & (kFCount - 1);
      const bool seen = fe[2 * p.n_fn + f] != 0 || fe[p.n_fn + f] != 0xFFFFFFFFu;  // flushed spans count too
      if (!__any_sync(0xffffffffu, cnt != 0) && !seen) continue;
      for (int dd = 16; dd; dd >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, dd);
        sum += __shfl_xor_sync(0xffffffffu, sum, dd);
      }
      if (lane == 0) {
        unsigned long long* a = p.host_acc + 6ull * f;
        if (cnt) atomicAdd(&a[0], (unsigned long long)cnt);
        if (fe[f]) atomicAdd(&a[1], (unsigned long long)fe[f]);
        if (sum) add_i128(&a[2], &a[3], sum, 0);
        atomicMin(&a[4], (unsigned long long)fe[p.n_fn + f]);
        atomicMax(&a[5], (unsigned long long)fe[2 * p.n_fn + f]);
      }
    }
  }
  __syncthreads();
  if (p.n_fn > kSmallF && p.n_fn <= kSmemFnMax) {
    const SmemRow* tab = reinterpret_cast<const SmemRow*>(g_smem + RL.tab);
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
  const DevRow* dcache = reinterpret_cast<const DevRow*>(g_smem + RL.dcache);
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

// kSD: descriptor mode (fast_desc_mode): 1 the registry's inline descriptors in shared memory (max_sid <
// kSdescMax), 2 compact descriptors in shared memory, 0 through L1;
// kDeep: stacks deeper than kRLS stay on the inline path (overflow chunk) -- chosen by the host
// once a run of the trace needed overflow chunks; kMode bits: 1 a timeline run (every host span,
// device span and sample also leaves a message in its range's list, r_item), 2 an event run
// (every record, r_event)
template <int kSD, bool kDeep, int kMode>
__global__ void __launch_bounds__(kRMaxThreads, 1) fast_kernel(Params p, const Params* gp) {
  const Params& gpr = *gp;
  const uint32_t nw = blockDim.x >> 5;
  const uint32_t n_fd = kSD == 1 ? p.max_sid + 2 : 0u, n_cd = kSD == 2 ? p.max_sid + 2 : 0u;
  const RSmem RL = fast_smem_layout(p.n_fn, nw, n_fd, n_cd, p.has_dev != 0);
  const uint32_t* cdesc_s = reinterpret_cast<const uint32_t*>(g_smem);
  const uint4* fdesc_s = reinterpret_cast<const uint4*>(g_smem + RL.fdesc);
  const SegSmem L = r_segsmem(RL);
  const uint32_t lane = lane_id();
  uint8_t* wb = g_smem + RL.warps + (threadIdx.x >> 5) * RL.warp_bytes;
  const uint32_t* ring = reinterpret_cast<const uint32_t*>(wb + RL.ring + lane * kRStride);
  const uint32_t ring_s = s_addr(ring);
  const uint32_t nc_s = s_addr(g_smem + RL.ncache);
  r_prologue(p, RL, nw, n_fd, n_cd);
  SegCounters K;
  K.passed = K.host = K.dev = K.samples = K.orph = K.items = 0;
  HostFold hf;  // the slow path's fold: CTA table (medium function sets) or global rows
  hf.small = false;
  hf.tab = (p.n_fn > kSmallF && p.n_fn <= kSmemFnMax) ? reinterpret_cast<SmemRow*>(g_smem + RL.tab) : nullptr;
  const bool small = p.n_fn <= kSmallF;
  uint64_t* ftab = reinterpret_cast<uint64_t*>(wb + RL.ftab) + lane;
  uint32_t* ferr = reinterpret_cast<uint32_t*>(wb + RL.ferr);
  const RTabs T = r_tabs(RL);
  uint64_t* q_off = reinterpret_cast<uint64_t*>(wb + RL.q_off);
  uint32_t* q_s = reinterpret_cast<uint32_t*>(wb + RL.q_s);
  uint64_t* qs_off = reinterpret_cast<uint64_t*>(wb + RL.qs_off);
  uint32_t* qs_s = reinterpret_cast<uint32_t*>(wb + RL.qs_s);
  uint32_t qsn = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  constexpr uint32_t kPend = (1u << kRLag) - 1u;
  RLane R;
  R.recent = 0;
  bool live = r_begin(gpr, R, blockIdx.x * blockDim.x + threadIdx.x, stride);
  uint32_t qd = 0;
  const uint32_t sid_cap = p.max_sid + 1;  // fdesc[max_sid + 1]: never inline (unknown ids, slow path names them)
  while (__any_sync(0xffffffffu, live)) {
    const bool ending = live && (R.o >= R.t1 || R.bad);
    if (__any_sync(0xffffffffu, ending)) {
      if (ending) {
        R = r_switch(gpr, R, T, stride);
        live = R.r < p.n_ranges;
      }
    }
    const bool act = live && R.o < R.t1 && !R.bad;
    const uint32_t o_start = R.o;
    // ---- ring refill: the lane copies its next line itself (8 x 16 B cp.async, + the mirror for slot 0)
    const uint32_t cons = R.o / kRChunk;
    if (act && cons > R.ci) { R.ci = cons; R.fresh = true; }  // a long record jumped over chunks
    if (!(R.recent & kPend)) R.fresh = false;
    const bool want = act && !R.fresh && R.ci <= R.clast && R.ci < cons + kRSlots;
    {
      const uint32_t q = R.ci & (kRSlots - 1);
      const uint8_t* src = R.g + (uint64_t)R.ci * kRChunk;
      const uint32_t dst = ring_s + q * kRChunk;
      const uint32_t pw = want ? 1u : 0u, pm = (want && q == 0) ? 1u : 0u;
      #pragma unroll
      for (uint32_t k = 0; k < kRChunk; k += 16) r_cp16p(dst + k, src + k, pw);
      (void)pm;
    }
    R.ci += want ? 1u : 0u;
    R.recent = (R.recent << 1) | (want ? 1u : 0u);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kRLag) : "memory");
    __syncwarp();
    // ---- every chunk requested before the last kRLag iterations is in the ring; first the header
    // (right after a range switch ci restarts at 0 while the old range's last fills may still be
    // pending: nothing of the new range is in the ring yet -- no wrap-around to "all ready")
    const uint32_t pend = __popc(R.recent & kPend);
    const uint32_t cr = R.ci > pend ? R.ci - pend : 0u;
    const bool ready = act && min((R.o + 15u) / kRChunk, R.clast) < cr;
    const uint32_t pos = R.o & (kRRing - 1);
    const uint32_t wb0 = pos >> 2;
    const uint32_t sh = (pos & 3u) << 3;
    const uint32_t w0 = ring[wb0], w1 = ring[(wb0 + 1) & kRWordMask], w2 = ring[(wb0 + 2) & kRWordMask],
                   w3 = ring[(wb0 + 3) & kRWordMask], w4 = ring[(wb0 + 4) & kRWordMask],
                   w5 = ring[(wb0 + 5) & kRWordMask], w6 = ring[(wb0 + 6) & kRWordMask];
    const uint32_t sid = __funnelshift_r(w0, w1, sh);
    const uint64_t ts = ((uint64_t)__funnelshift_r(w2, w3, sh) << 32) | __funnelshift_r(w1, w2, sh);
    const uint32_t plen = __funnelshift_r(w3, w4, sh);
    uint4 D;
    if (kSD == 1) {
      D = fdesc_s[min(sid, sid_cap)];
    } else if (kSD == 2) {
      const uint32_t c = cdesc_s[min(sid, sid_cap)];
      D = (c >> 31) ? r_expand(c) : __ldg(&p.fdesc[min(sid, sid_cap)]);
    } else {
      D = __ldg(&p.fdesc[min(sid, sid_cap)]);
    }
    const uint32_t fnm = D.x & M_FN;
    const uint32_t kind = (D.x >> 20) & 7u;
    const uint32_t ne = R.ne, np = R.np;
    const uint32_t topi = ((ne - 1u) & (uint32_t)(kRLS - 1)) * kWarp;
    uint64_t ets = T.st_ts[topi];
    uint32_t tfn = T.st_fn[topi];
    // the window is empty: the top was spilled to the lane's overflow chunk (HBM, L1); only an exit
    // needs it (every iteration of a lane in that state waited for the load, 22% of C4's stall samples)
    if (kDeep && ne && R.deep && !R.nw && kind == FK_EXIT) {
      const SumEntry* de = R.deep + kRDeepHalf + (ne - 1u);
      ets = de->ts;
      tfn = de->fn < 0 ? M_FN : (uint32_t)de->fn;
    }
    // inline: the whole record in the ring, in order, with a length its schema allows (lo <= plen <= hi <= 112)
    const uint32_t lo = D.y & 0xFFFFu, hi = D.y >> 16;
    const bool good = ready && plen - lo <= hi - lo && (R.o + 15u + plen) / kRChunk < cr &&
                      R.o + 16u + plen <= R.size32 && (R.n == 0 || ts >= R.prev_ts);
    const bool stall = ready && !good && plen <= kRInline - 16u && (R.o + 15u + plen) / kRChunk >= cr &&
                       (uint64_t)R.o + 16u + plen <= R.size;
    // a push spills when the window is full, a pop reads the chunk when it is empty (kDeep, chunk allocated)
    // (without kDeep a lane whose range allocated a chunk leaves every push / pop to the slow path)
    const bool fE = good && kind == FK_ENTRY && (kDeep ? ne < kRDepthMax && (R.deep || ne < (uint32_t)kRLS)
                                                       : ne < (uint32_t)kRLS && !R.deep);
    const bool fXp = good && kind == FK_EXIT && ne && (kDeep || !R.deep) && tfn == fnm;  // pops a same-function top
    // pending (compose decides); with kDeep beyond kRLP into the lane's chunk (a range that starts deep
    // in a call stack meets tens of exits before its first entry: they took the slow path, C4)
    const bool fXq = good && kind == FK_EXIT && ne == 0 &&
                     (np < (uint32_t)kRLP || (kDeep && R.deep && np < (uint32_t)kRLP + kRDeepHalf));
    const bool fO = good && (kind == FK_PASS || kind == FK_DEFER);
    // one variable field (blob / string): exact length here, UTF-8 of strings in the drain
    const uint32_t lead0 = D.z & 0xFFFFu, lead1 = D.z >> 16;
    const bool chk = (D.x & FD_VAR) != 0;
    const uint32_t ln = r_u32(ring, pos + 16u + lead0);
    const bool lenbad = (fE || fXp || fXq || fO) && chk && lead0 + 4u + (uint64_t)ln + lead1 != plen;
    if (lenbad) R.bad = true;  // CorruptRecordError: the exact path names it
    const bool fast = (fE || fXp || fXq || fO) && !lenbad;
    bool qflag = fast && kind == FK_DEFER;
    R.spans += (qflag && (D.x & FD_ISDEV)) ? 1u : 0u;  // a device span's identity (sinks.py:240-242)
    bool sflag = fast && (D.x & FD_STR) && ln;
    if (sflag && ln <= 16u) {  // short strings (kernel names): all-ASCII from the ring, else the drain decides
      const uint32_t sp = pos + 20u + lead0, sw = sp >> 2, s0 = (sp & 3u) << 3;
      const uint32_t e = sp + ln, ew = (e - 1u) >> 2;  // last word holding a string byte
      uint32_t acc = 0;
      #pragma unroll
      for (uint32_t k = 0; k < 5; k++) {
        const uint32_t wk = sw + k;
        uint32_t x = ring[wk & kRWordMask];
        if (k == 0) x &= 0xffffffffu << s0;
        if (wk == ew) x &= 0xffffffffu >> (8u * ((4u - (e & 3u)) & 3u));
        acc |= wk <= ew ? x : 0u;
      }
      sflag = (acc & 0x80808080u) != 0;
    }
    const uint64_t res = (D.x & FD_RES) ? ((uint64_t)__funnelshift_r(w5, w6, sh) << 32) | __funnelshift_r(w4, w5, sh) : 0ull;
    const bool err = res != 0;
    if (fast) {
      if (kMode & 2) r_event(p, R, R.n, ts, o_start, sid);
      R.first_ts = R.n ? R.first_ts : ts;
      R.n++;
      R.prev_ts = ts;
      R.o += 16u + plen;
    }
    if (fE) {
      if (kDeep && R.deep && R.nw == (uint32_t)kRLS) r_spill(R, T, ne);
      T.st_ts[(ne & (kRLS - 1)) * kWarp] = ts;
      T.st_fn[(ne & (kRLS - 1)) * kWarp] = fnm;
    }
    if (kDeep) R.nw = R.nw + ((fE && R.nw < (uint32_t)kRLS) ? 1u : 0u) - ((fXp && R.nw) ? 1u : 0u);
    if (fXq) {
      const uint32_t xf = 1u | (err ? 2u : 0u) | (((D.x >> 26) & 3u) << 4);
      if (kDeep && np >= (uint32_t)kRLP) {  // as r_record_slow stores it
        SumEntry e;
        e.ts = ts; e.seq = R.n - 1; e.fn = m_fn(fnm); e.flags = xf; e.result = res;
        R.deep[np - kRLP] = e;
      } else {
        const uint32_t i = np * kWarp;
        T.pd_ts[i] = ts;
        T.pd_meta[i] = fnm | (xf << 19);
        T.pd_k[i] = R.n - 1;
        if (kMode & 1) p.tl_pres[(uint64_t)R.r * kRLP + np] = res;
      }
    }
    if (kMode & 1) {
      if (fXp) r_item(p, R, ts, R.n - 1, ets, res, TL_HOST | (((D.x >> 26) & 3u) << 4), fnm);
      if (qflag) r_item(p, R, ts, R.n - 1, reinterpret_cast<uint64_t>(R.g + o_start + 16u), 0,
                        (D.x & FD_ISDEV) ? TL_DEVICE : TL_SAMPLE, sid);
    }
    R.ne = ne + (fE ? 1u : 0u) - (fXp ? 1u : 0u);
    R.np = np + (fXq ? 1u : 0u);
    if (fXp) {
      const uint64_t dur = ts - ets;
      if (small && (dur >> 32) == 0) {
        const uint32_t du = (uint32_t)dur;
        uint64_t cs = ftab[fnm * kWarp] + kFCount + du;
        if (cs & kFLimit) {  // flush before the packed count or sum can overflow
          r_fold_flush(gpr, fnm, cs);
          cs = 0;
        }
        ftab[fnm * kWarp] = cs;
        if (err) atomicAdd(&ferr[fnm], 1u);
        atomicMin(&ferr[p.n_fn + fnm], du);
        atomicMax(&ferr[2 * p.n_fn + fnm], du);
      } else {
        hf.fold(gpr, (int32_t)fnm, dur, err);
      }
      K.host++;
      R.spans++;
    }
    K.passed += (fO && kind == FK_PASS) ? 1u : 0u;
    // everything else from HBM (the ring is only a cache of the stream)
    const bool slow = ready && !fast && !R.bad && !stall;  // unknown ids, long records, deep stacks, orphans ...
    if (__any_sync(0xffffffffu, slow)) {
      if (slow) qflag = r_record_slow(gpr, R, T, K, hf);
    }
    // deferred records (already consumed): string UTF-8 checks, device folds and telemetry checks
    const uint32_t sm = __ballot_sync(0xffffffffu, sflag);
    if (sm) {
      if (sflag) {
        const uint32_t i = qsn + __popc(sm & lanemask_lt());
        qs_off[i] = R.C0 + o_start;
        qs_s[i] = R.s;
      }
      qsn += __popc(sm);
      __syncwarp();
      if (qsn >= (uint32_t)kWarp) {
        r_drain_str(gpr, qs_off, qs_s, kWarp);
        qsn -= kWarp;
        if (lane < qsn) { qs_off[lane] = qs_off[kWarp + lane]; qs_s[lane] = qs_s[kWarp + lane]; }
        __syncwarp();
      }
    }
    const uint32_t dm = __ballot_sync(0xffffffffu, qflag);
    if (dm) {
      if (qflag) {
        const uint32_t i = qd + __popc(dm & lanemask_lt());
        q_off[i] = R.C0 + o_start;
        q_s[i] = R.s;
      }
      qd += __popc(dm);
      __syncwarp();
      if (qd >= (uint32_t)kWarp) {
        const uint2 dk = r_drain(gpr, L, q_off, q_s, kWarp, nc_s);
        K.dev += dk.x; K.samples += dk.y;
        qd -= kWarp;
        if (lane < qd) { q_off[lane] = q_off[kWarp + lane]; q_s[lane] = q_s[kWarp + lane]; }
        __syncwarp();
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (qsn) r_drain_str(gpr, qs_off, qs_s, qsn);
  if (qd) {
    const uint2 dk = r_drain(gpr, L, q_off, q_s, qd, nc_s);
    K.dev += dk.x; K.samples += dk.y;
  }
  __syncwarp();
  r_epilogue(gpr, RL, K);
}

// per stream (one CTA): verify the range chain, record bases, compose_kernel's per-range state.
// Thread t owns a contiguous block of the stream's ranges: a local pass composes the block
// (exit carry, last timestamp, record count and what the block needs from its predecessor), a
// CTA scan hands every block its incoming carry, a second pass writes the per-range outputs.
// kVThreads: 128 threads per stream; 512 when a stream has many ranges (one huge stream: the
// two sequential passes shrink 4x, the carry scan over the blocks grows)
template <int kVThreads>
__global__ void __launch_bounds__(kVThreads) fast_verify_kernel(Params p, unsigned long long* stream_nrec) {
  __shared__ unsigned long long sx[kVThreads], st_[kVThreads], sb[kVThreads];
  __shared__ uint32_t sflags[kVThreads];
  const uint32_t s = blockIdx.x, t = threadIdx.x;
  const uint32_t r0 = p.stream_range0[s];
  const uint32_t r1 = (s + 1 < p.n_streams) ? p.stream_range0[s + 1] : p.n_ranges;
  const uint64_t size = p.stream_size[s];
  const uint32_t nr = r1 - r0, per = (nr + kVThreads - 1) / kVThreads;
  const uint32_t a = min(r0 + t * per, r1), b = min(a + per, r1);
  bool chain_ok = true, order_ok = true;
  bool hx = false, ht = false, need_e = false, need_t = false;
  uint64_t lx = 0, lt = 0, sum = 0, first_e = 0, first_t = 0, lead_t1 = 0;
  for (uint32_t r = a; r < b; r++) {
    const RangeState st = p.rstate[r];
    const uint64_t t1 = min(16 + (uint64_t)(r - r0 + 1) * p.range_bytes, size);
    if (st.entry != kNone) {  // starts where the previous range ended
      if (!hx) { need_e = true; first_e = st.entry; }
      else if (st.entry != lx) chain_ok = false;
      hx = true;
      lx = st.exit;
    } else {                  // no plausible header: a record of an earlier range spans it
      if (!hx) lead_t1 = max(lead_t1, t1);
      else if (lx < t1) chain_ok = false;
    }
    if (st.n) {               // timestamps keep rising across ranges (pipeline.py:98)
      if (!ht) { need_t = true; first_t = st.first_ts; }
      else if (st.first_ts < lt) order_ok = false;
      ht = true;
      lt = st.last_ts;
    }
    sum += st.n;
  }
  sx[t] = lx; st_[t] = lt; sb[t] = sum;
  sflags[t] = (hx ? 1u : 0u) | (ht ? 2u : 0u);
  __syncthreads();
  if (t == 0) {  // exclusive scan of the block carries (the exit before range 0 is the header end, 16)
    unsigned long long cx = 16, ct = 0, cb = 0;
    bool cht = false;
    for (uint32_t i = 0; i < kVThreads; i++) {
      const unsigned long long x = sx[i], ts = st_[i], n = sb[i];
      const uint32_t f = sflags[i];
      sx[i] = cx; st_[i] = ct; sb[i] = cb;
      sflags[i] = (f & 3u) | (cht ? 4u : 0u);
      if (f & 1u) cx = x;
      if (f & 2u) { ct = ts; cht = true; }
      cb += n;
    }
    stream_nrec[s] = cb;
    if (cb) atomicAdd(&p.stats[ST_EVENTS], cb);
    if (cht) atomicMax(p.last_ts, ct);  // IntervalStats.events_in, the global last ts (pipeline.py:152)
  }
  __syncthreads();
  const uint64_t in_x = sx[t], in_t = st_[t];
  const bool in_ht = (sflags[t] & 4u) != 0;
  if (need_e && first_e != in_x) chain_ok = false;
  if (lead_t1 > in_x) chain_ok = false;
  if (need_t && in_ht && first_t < in_t) order_ok = false;
  if (!chain_ok) atomicOr(p.anom, 8u);
  if (!order_ok) atomicOr(p.anom, 16u);
  uint64_t base = sb[t];
  for (uint32_t r = a; r < b; r++) {
    const RangeState st = p.rstate[r];
    p.range_base[r] = base;
    SegState ss;
    ss.status = (p.epoch << 2) | TS_DONE;
    ss.pool_n_pending = st.np;
    ss.pool_off = st.pool_off;
    ss.pool_n_resid = st.ne;
    ss.pad = 0;
    p.state[r] = ss;
    if (st.pool_off + st.np + st.ne <= p.pool_cap)
      for (uint32_t i = 0; i < st.np; i++) p.pool[st.pool_off + i].seq += base;
    base += st.n;
  }
}

// orphans found inside a range carry (range, index in range); make them stream indices
#ifdef HG_FAST_KERNELS
__global__ void fast_orphan_fix_kernel(Params p) {
  const unsigned long long n = min(*(volatile unsigned long long*)p.n_orphans, (unsigned long long)p.orphan_cap);
  for (unsigned long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t q = p.orphans[i].seq;
    if (q >> 63) p.orphans[i].seq = p.range_base[(q >> 24) & ((1ull << 39) - 1)] + (q & 0xFFFFFFull);
  }
}
#endif  // HG_FAST_KERNELS

}  // namespace hg
