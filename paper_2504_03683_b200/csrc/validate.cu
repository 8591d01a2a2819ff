// validate.cu -- ValidationSink's rules on the GPU (sinks.py:435-594).
//
// The reference walks the events in mux order with three dictionaries: pending_entries (last entry
// payload per (stream, function)), live_created (handle -> finding) and executed (command-list
// handle -> bool).  Each dictionary's history is a per-key sequence in mux order, so the walk
// becomes sorts + neighbour tests (after run_events has the mux order of every record):
//   val_classify_kernel<count / emit>  per mux position: uninit_pnext findings; E items (entries of
//        the functions releases / resets look up: their handle parameter), X items (command-list
//        executions), C items (creates with result 0), Q items (releases / resets with result 0)
//   tl_sort (E+Q by stream, function, type, record index) + val_resolve_kernel (one CTA, max-scan
//        of the latest E): each Q gets pending_entries[(stream, function)][param] -> R items
//   tl_sort (C + released handles by handle, position) + val_leak_kernel: a handle is leaked iff its
//        last event is a create (live_created.pop / re-insert, sinks.py:574-586)
//   tl_sort (X + reset handles by handle, position) + val_cmdlist_kernel: an execution whose
//        previous event of the same handle is an execution (sinks.py:540-551)
// Findings carry their mux position (in-order findings) or handle (leaks, sorted by subject); the
// host formats the messages.
#define HG_VAL_KERNELS
#include "ctx.h"

namespace {

enum : uint32_t { VK_PNEXT = 1, VK_EXEC = 2, VK_CREATE = 4, VK_RELEASE = 8, VK_RESET = 16, VK_TRACK = 32 };
enum : uint32_t { IT_E = 0, IT_Q = 1, IT_X = 2, IT_C = 3, IT_R = 4 };

using VRule = hg_validation_rule;  // per schema index: kind VK_*, field indices (-1: absent)

struct VTables {
  const TlItem* ev;       // records in slot order (run_events)
  const uint32_t* order;  // mux order
  uint32_t n;
  const uint8_t* data;
  const int32_t* sid_map;
  const DSchema* schemas;
  const uint8_t* kinds;
  const VRule* rules;
  TlItem* eq; TlItem* xr; TlItem* cr;   // E+Q, X+reset, C+release
  unsigned int* cnt;                    // [0] eq, [1] xr, [2] cr, [3] findings
  hg_finding* fnd;
  uint32_t cap_eq, cap_xr, cap_cr, cap_f;
};

// payload address of field f (fields before it walked: 8 bytes, or u32 length + bytes)
__device__ __forceinline__ const uint8_t* field_at(const VTables& T, const DSchema& sc, const uint8_t* q, int f) {
  for (int k = 0; k < f; k++) {
    const uint8_t kind = T.kinds[sc.kinds_off + k];
    q += (kind == HG_KIND_STRING || kind == HG_KIND_BLOB) ? 4u + ldu32(q) : 8u;
  }
  return q;
}

// Python int value of an integer field as a 65-bit key: v + 2^63 (u64 / address and i64 share one order)
__device__ __forceinline__ void hkey(const VTables& T, const DSchema& sc, const uint8_t* q, int f, uint64_t& hi,
                                     uint64_t& lo) {
  const uint64_t v = ldu64(field_at(T, sc, q, f));
  const bool sgn = T.kinds[sc.kinds_off + f] == HG_KIND_I64;
  // v' = v + 2^63 (signed) or v + 2^63 (unsigned, may carry into bit 64)
  lo = v + 0x8000000000000000ull;
  hi = sgn ? 0ull : (v >= 0x8000000000000000ull ? 1ull : 0ull);
}

__device__ __forceinline__ void put(TlItem* a, unsigned int* c, uint32_t cap, uint64_t khi, uint64_t klo, uint64_t av,
                                    uint64_t bv, uint32_t kind, uint32_t x) {
  const unsigned int i = atomicAdd(c, 1u);
  if (i < cap) {
    TlItem it;
    it.khi = khi; it.klo = klo; it.a = av; it.b = bv; it.kind = kind; it.x = x;
    a[i] = it;
  }
}

// sort key of a handle-keyed item: (v' >> 1, (v' & 1) << 63 | position)
__device__ __forceinline__ void hsort(uint64_t hi, uint64_t lo, uint32_t pos, uint64_t& khi, uint64_t& klo) {
  khi = (hi << 63) | (lo >> 1);
  klo = ((lo & 1ull) << 63) | pos;
}

__device__ __forceinline__ void add_finding(const VTables& T, uint32_t rule, uint32_t sid, uint32_t s, uint64_t pos,
                                            uint64_t ts, uint64_t hi, uint64_t lo) {
  const unsigned int i = atomicAdd(&T.cnt[3], 1u);
  if (i < T.cap_f) {
    hg_finding f;
    f.rule = rule; f.sid = sid; f.stream = s; f.pad = 0; f.pos = pos; f.ts = ts; f.subject_lo = lo;
    f.subject_hi = (int64_t)hi;
    T.fnd[i] = f;
  }
}

__global__ void __launch_bounds__(256) val_classify_kernel(VTables T) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < T.n; i += gridDim.x * blockDim.x) {
    const TlItem it = T.ev[T.order[i]];
    const int32_t si = T.sid_map[it.x];
    const VRule r = T.rules[si];
    if (!r.kind) continue;
    const DSchema& sc = T.schemas[si];
    const uint8_t* q = T.data + it.a + 16;
    const uint32_t s = (uint32_t)(it.klo >> 40);
    const uint64_t seq = it.klo & ((1ull << 40) - 1);
    if (r.kind & VK_PNEXT) {  // sinks.py:523-537
      const uint8_t* b = field_at(T, sc, q, r.pnext);
      if (ldu32(b) >= 8) {
        const uint64_t pn = ldu64(b + 4);
        if (pn) add_finding(T, HG_FIND_PNEXT, it.x, s, i, it.khi, 0, pn);
      }
    }
    const uint64_t grp = ((uint64_t)s << 21) | ((uint64_t)(uint32_t)sc.fn << 1);
    if (sc.cls == HG_CLASS_ENTRY) {
      uint64_t hi, lo;
      if (r.kind & VK_TRACK) {  // pending_entries[(stream, function)] = payload (sinks.py:540)
        if (r.rel >= 0) { hkey(T, sc, q, r.rel, hi, lo); put(T.eq, &T.cnt[0], T.cap_eq, grp, seq << 1, lo, hi, IT_E, it.x); }
        if (r.rst >= 0) { hkey(T, sc, q, r.rst, hi, lo); put(T.eq, &T.cnt[0], T.cap_eq, grp | 1u, seq << 1, lo, hi, IT_E, it.x); }
      }
      if (r.kind & VK_EXEC) {
        uint64_t kh, kl;
        hkey(T, sc, q, r.exec, hi, lo);
        hsort(hi, lo, i, kh, kl);
        put(T.xr, &T.cnt[1], T.cap_xr, kh, kl, lo, hi, IT_X, it.x);
      }
      continue;
    }
    if (sc.cls != HG_CLASS_EXIT) continue;
    if (r.result >= 0 && ldu64(field_at(T, sc, q, r.result)) != 0) continue;  // int(result) != 0
    if (r.kind & VK_CREATE) {
      uint64_t hi, lo, kh, kl;
      hkey(T, sc, q, r.create, hi, lo);
      hsort(hi, lo, i, kh, kl);
      put(T.cr, &T.cnt[2], T.cap_cr, kh, kl, lo, hi, IT_C, it.x);
    } else if (r.kind & (VK_RELEASE | VK_RESET)) {
      put(T.eq, &T.cnt[0], T.cap_eq, grp | ((r.kind & VK_RESET) ? 1u : 0u), (seq << 1) | 1u, i, 0, IT_Q, it.x);
    }
  }
}

// E+Q sorted by (group, record index): every Q takes the handle of the latest E of its group --
// one CTA, a running max-scan of "index of the latest E" carried across 1024-item chunks
__global__ void __launch_bounds__(1024) val_resolve_kernel(const TlItem* eq, const uint32_t* order, uint32_t n,
                                                           TlItem* xr, TlItem* cr, unsigned int* cnt, uint32_t cap_xr,
                                                           uint32_t cap_cr) {
  __shared__ int s_w[32];
  __shared__ int s_carry;
  if (threadIdx.x == 0) s_carry = -1;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < n; b0 += 1024) {
    const uint32_t j = b0 + threadIdx.x;
    TlItem it;
    int v = -1;
    if (j < n) {
      it = eq[order[j]];
      if (it.kind == IT_E) v = (int)j;
    }
    int x = v;  // inclusive max-scan
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if ((threadIdx.x & 31) >= (uint32_t)d) x = max(x, y);
    }
    if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
    __syncthreads();
    int pre = s_carry;
    for (uint32_t w = 0; w < (threadIdx.x >> 5); w++) pre = max(pre, s_w[w]);
    const int last = max(pre, x);
    if (j < n && it.kind == IT_Q && last >= 0) {
      const TlItem e = eq[order[last]];
      if (e.khi == it.khi) {  // same stream, function and rule type
        uint64_t kh, kl;
        hsort(e.b, e.a, (uint32_t)it.a, kh, kl);
        if (it.khi & 1u) put(xr, &cnt[1], cap_xr, kh, kl, e.a, e.b, IT_R, it.x);  // reset
        else put(cr, &cnt[2], cap_cr, kh, kl, e.a, e.b, IT_R, it.x);               // release
      }
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = last;
    __syncthreads();
  }
}

__device__ __forceinline__ bool same_handle(const TlItem& a, const TlItem& b) { return a.a == b.a && a.b == b.b; }

// C + releases by (handle, position): a handle whose last event is a create is leaked
__global__ void __launch_bounds__(256) val_leak_kernel(VTables T, const TlItem* cr, const uint32_t* order, uint32_t n) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const TlItem it = cr[order[j]];
    if (it.kind != IT_C) continue;
    if (j + 1 < n && same_handle(cr[order[j + 1]], it)) continue;
    const uint32_t pos = (uint32_t)(it.klo & 0xFFFFFFFFull);
    const TlItem ev = T.ev[T.order[pos]];
    add_finding(T, HG_FIND_LEAK, it.x, (uint32_t)(ev.klo >> 40), pos, ev.khi, it.b, it.a);
  }
}

// X + resets by (handle, position): an execution right after an execution of the same handle
__global__ void __launch_bounds__(256) val_cmdlist_kernel(VTables T, const TlItem* xr, const uint32_t* order, uint32_t n) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const TlItem it = xr[order[j]];
    if (it.kind != IT_X || j == 0) continue;
    const TlItem pv = xr[order[j - 1]];
    if (pv.kind != IT_X || !same_handle(pv, it)) continue;
    const uint32_t pos = (uint32_t)(it.klo & 0xFFFFFFFFull);
    const TlItem ev = T.ev[T.order[pos]];
    add_finding(T, HG_FIND_CMDLIST, it.x, (uint32_t)(ev.klo >> 40), pos, ev.khi, it.b, it.a);
  }
}

}  // namespace

// after run_events: the four rules over the mux-ordered records
int run_validation(hg_ctx* ctx) {
  ctx->val_ready = false;
  if (!ctx->ev_ready) return fail(ctx, HG_ESTATE, "validation needs the event order (HG_WANT_EVENTS)");
  if (ctx->val_rules.size() != ctx->schemas.size() || ctx->val_rules.empty())
    return fail(ctx, HG_ESTATE, "hg_set_validation_rules first");
  cudaStream_t st = ctx->stream;
  const uint32_t n = (uint32_t)ctx->counters[C_STATS + ST_EVENTS];
  CK(upload(ctx->d_val_rules, ctx->val_rules, st));
  CK(ctx->d_val_cnt.ensure(4));
  // the events' order: a private copy (the sorts below reuse the timeline sort's buffers)
  CK(ctx->d_val_order.ensure(std::max<uint32_t>(n, 1)));
  if (n) CK(cudaMemcpyAsync(ctx->d_val_order.ptr, ctx->ev_order, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  VTables T{};
  T.ev = ctx->d_ev_items.ptr;
  T.order = ctx->d_val_order.ptr;
  T.n = n;
  T.data = ctx->d_data.ptr;
  T.sid_map = ctx->d_sid_map.ptr;
  T.schemas = ctx->d_schemas.ptr;
  T.kinds = ctx->d_kinds.ptr;
  T.rules = ctx->d_val_rules.ptr;
  T.cnt = ctx->d_val_cnt.ptr;
  const uint32_t g = std::max<uint32_t>(1, std::min<uint32_t>((n + 255) / 256, (uint32_t)ctx->sm_count * 16));
  unsigned int c[4] = {0, 0, 0, 0};
  for (int pass = 0; pass < 2; pass++) {  // count, then emit into exact-size buffers
    CK(cudaMemsetAsync(T.cnt, 0, 16, st));
    T.eq = ctx->d_val_eq.ptr; T.xr = ctx->d_val_xr.ptr; T.cr = ctx->d_val_cr.ptr; T.fnd = ctx->d_val_fnd.ptr;
    T.cap_eq = pass ? c[0] : 0; T.cap_xr = pass ? c[1] + c[0] : 0; T.cap_cr = pass ? c[2] + c[0] : 0;
    T.cap_f = pass ? c[3] + c[1] + c[2] + 16 : 0;
    if (n) val_classify_kernel<<<g, 256, 0, st>>>(T);
    CK(cudaGetLastError());
    ctx->launches++;
    if (!pass) {
      CK(cudaMemcpyAsync(c, T.cnt, 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(ctx->d_val_eq.ensure(std::max(c[0], 1u)));
      CK(ctx->d_val_xr.ensure(c[1] + c[0] + 1));  // + the resets resolved from Q items
      CK(ctx->d_val_cr.ensure(c[2] + c[0] + 1));  // + the releases
      CK(ctx->d_val_fnd.ensure(c[3] + c[1] + c[2] + 16));
    }
  }
  const uint32_t n_eq = c[0];
  // resolve releases / resets against the latest entry of their function on their stream
  const uint32_t* ord = nullptr;
  if (n_eq) {
    int rc = tl_sort(ctx, ctx->d_val_eq.ptr, 0, n_eq, n_eq, n_eq, &ord);
    if (rc) return rc;
    val_resolve_kernel<<<1, 1024, 0, st>>>(ctx->d_val_eq.ptr, ord, n_eq, ctx->d_val_xr.ptr, ctx->d_val_cr.ptr, T.cnt,
                                           c[1] + c[0], c[2] + c[0]);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  unsigned int c2[4];
  CK(cudaMemcpyAsync(c2, T.cnt, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  T.cap_f = c[3] + c[1] + c2[2] + 16;
  if (c2[2]) {  // leaks
    int rc = tl_sort(ctx, ctx->d_val_cr.ptr, 0, c2[2], c2[2], c2[2], &ord);
    if (rc) return rc;
    val_leak_kernel<<<std::max<uint32_t>(1, std::min<uint32_t>((c2[2] + 255) / 256, 4096)), 256, 0, st>>>(
        T, ctx->d_val_cr.ptr, ord, c2[2]);
    ctx->launches++;
  }
  if (c2[1]) {  // command lists
    int rc = tl_sort(ctx, ctx->d_val_xr.ptr, 0, c2[1], c2[1], c2[1], &ord);
    if (rc) return rc;
    val_cmdlist_kernel<<<std::max<uint32_t>(1, std::min<uint32_t>((c2[1] + 255) / 256, 4096)), 256, 0, st>>>(
        T, ctx->d_val_xr.ptr, ord, c2[1]);
    ctx->launches++;
  }
  CK(cudaGetLastError());
  unsigned int nf = 0;
  CK(cudaMemcpyAsync(&nf, T.cnt + 3, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ctx->val_findings.resize(nf);
  if (nf) CK(cudaMemcpy(ctx->val_findings.data(), ctx->d_val_fnd.ptr, nf * sizeof(hg_finding), cudaMemcpyDeviceToHost));
  ctx->val_ready = true;
  return HG_OK;
}

extern "C" {

int hg_set_validation_rules(hg_ctx* ctx, const hg_validation_rule* rules, uint32_t n_schemas) {
  if (!ctx || (n_schemas && !rules)) return HG_EARG;
  if (n_schemas != ctx->schemas.size()) return fail(ctx, HG_EARG, "one validation rule per registry schema");
  ctx->val_rules.assign(rules, rules + n_schemas);
  return HG_OK;
}

int hg_get_findings(hg_ctx* ctx, hg_finding* out, uint64_t cap, uint64_t* n) {
  if (!ctx || !n) return HG_EARG;
  if (!ctx->val_ready) return HG_ESTATE;
  *n = ctx->val_findings.size();
  if (!out) return HG_OK;
  if (cap < *n) return fail(ctx, HG_EARG, "findings buffer too small");
  std::copy(ctx->val_findings.begin(), ctx->val_findings.end(), out);
  return HG_OK;
}

}  // extern "C"
