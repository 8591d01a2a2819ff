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
// Kernel design: phase 1 in seg.cuh (segment walk / chain / decode), composition
// here, timeline ordering and formatting in timeline.cuh.
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

namespace {

// ---------------------------------------------------------------------------
// composition of segment summaries per stream (exact automaton from an empty stack)

constexpr int kComposeWarps = 4;
constexpr uint32_t kComposeFast = 128;  // stack positions per warp held in shared memory

// kBlock (single pass only): one warp per block of up to 32 consecutive ranges of a stream; exits
// that meet the block's empty stack stay pending and the block's stack becomes its summary, which
// the per-stream pass (kBlock = false) then composes -- 32x shorter sequential chains per stream.
struct ComposeBlocks {
  const uint32_t* stream;  // block -> stream
  const uint32_t* u0;      // block -> first unit (n_blocks + 1 entries)
  SegState* out;           // block summaries
  uint32_t n;
};

template <bool kBlock>
__global__ void __launch_bounds__(kComposeWarps * kWarp) compose_kernel(Params p, ComposeBlocks B) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  SmemRow* tab = p.n_fn <= kSmemFnMax ? reinterpret_cast<SmemRow*>(smem) : nullptr;
  const uint32_t cfast_off = p.n_fn <= kSmemFnMax ? ((uint32_t)sizeof(SmemRow) * p.n_fn + 15u) & ~15u : 0u;
  if (tab)
    for (uint32_t i = threadIdx.x; i < p.n_fn; i += blockDim.x) {
      SmemRow z; z.count = z.err = z.s0 = z.s1 = 0; z.mn = 0xFFFFFFFFu; z.mx = 0;
      tab[i] = z;
    }
  __syncthreads();
  HostFold hf;
  hf.small = false;
  hf.tab = tab;
  const uint32_t wid = blockIdx.x * kComposeWarps + warp;
  const uint32_t s = kBlock ? (wid < B.n ? B.stream[wid] : p.n_streams) : wid;
  uint32_t host = 0, orph = 0, trunc = 0, spans = 0;
  if (s < p.n_streams) {
    const uint32_t g0 = kBlock ? B.u0[wid] : p.stream_tile0[s];
    const uint32_t g1 = kBlock ? B.u0[wid + 1] : (s + 1 < p.n_streams) ? p.stream_tile0[s + 1] : p.n_tiles;
    // first failed tile (its summary is still composed) and the stack capacity
    uint32_t gerr = g1;
    unsigned long long need = 0;
    for (uint32_t g = g0 + lane; g < g1; g += kWarp) {
      if ((p.state[g].status & 3u) == TS_ERROR && g < gerr) gerr = g;
      need += p.state[g].pool_n_resid + (kBlock ? p.state[g].pool_n_pending : 0u);
    }
    gerr = __reduce_min_sync(0xffffffffu, gerr);
    #pragma unroll
    for (int d = 16; d; d >>= 1) need += __shfl_xor_sync(0xffffffffu, need, d);
    const uint32_t gend = gerr < g1 ? gerr + 1 : g1;
    unsigned long long sbase = 0;
    if (lane == 0 && need) sbase = atomicAdd(p.stack_used, need);
    sbase = __shfl_sync(0xffffffffu, sbase, 0);
    if (sbase + need <= p.stack_cap) {
      GStack gs;
      gs.base = p.stack_scratch + sbase;
      // the bottom kComposeFast positions in shared memory (call stacks are shallow; deeper ones spill)
      gs.fast = reinterpret_cast<SumEntry*>(smem + cfast_off) + warp * kComposeFast;
      gs.n_fast = kComposeFast;
      gs.n_pend = 0;
      gs.top = 0;
      bool res_done = false;
      for (uint32_t gb = g0; gb < gend; gb += kWarp) {
        uint32_t g = gb + lane;
        bool valid = g < gend;
        uint32_t np = valid ? p.state[g].pool_n_pending : 0;
        uint32_t nr = valid ? p.state[g].pool_n_resid : 0;
        unsigned long long poff = valid ? p.state[g].pool_off : 0;
        uint32_t c = np + nr, ein = c;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) { uint32_t v = __shfl_up_sync(0xffffffffu, ein, d); if ((int)lane >= d) ein += v; }
        const uint32_t T = __shfl_sync(0xffffffffu, ein, 31);
        const uint32_t ebase = ein - c;
        for (uint32_t r = 0; r < T; r += kWarp) {
          uint32_t e = r + lane;
          bool act = e < T;
          uint32_t owner = 0;
          #pragma unroll
          for (int step = 16; step; step >>= 1) {
            uint32_t cand = owner + step;
            uint32_t b = __shfl_sync(0xffffffffu, ebase, cand & 31);
            if (cand < 32 && b <= e) owner = cand;
          }
          uint32_t ob = __shfl_sync(0xffffffffu, ebase, owner);
          uint32_t onp = __shfl_sync(0xffffffffu, np, owner);
          unsigned long long opoff = __shfl_sync(0xffffffffu, poff, owner);
          uint32_t k = e - ob;
          SumEntry x;
          x.ts = 0; x.seq = 0; x.fn = -1; x.flags = 0; x.result = 0;
          if (act && opoff + k < p.pool_cap) x = p.pool[opoff + k];
          bool isX = act && k < onp;
          bool isE = act && k >= onp;
          bool paired, orphan;
          uint64_t ets;
          const RoundOut ro2 = round_resolve(gs, kBlock, isE, isX, x.fn, x.ts, x);
          paired = ro2.flags & 1u;
          orphan = (ro2.flags >> 1) & 1u;
          ets = ro2.ets;
          gs.n_pend = ro2.n_pend;
          gs.top = ro2.top;
          if (paired) {
            hf.fold(p, x.fn, x.ts - ets, (x.flags & 2u) != 0);
            host++;
            spans++;
          }
          if (p.tl_items)
            tl_emit(p, paired, x.ts, tl_klo(s, x.seq), ets, x.result, TL_HOST | (((x.flags >> 4) & 3u) << 4),
                    (uint32_t)x.fn);
          uint32_t bm = __ballot_sync(0xffffffffu, paired && (x.flags & 4u));
          if (bm && !res_done) {
            if ((int)lane == __ffs(bm) - 1)
              push_error(p, HG_ERR_RESULT, s, x.seq, 0, x.ts, 0, x.result ? x.result : ((x.flags & 8u) ? 0x7FF8000000000000ull : 0x7FF0000000000000ull));
            res_done = true;
          }
          if (orphan) { push_orphan(p, s, x.fn, x.ts, x.seq); orph++; }
        }
      }
      if (kBlock) {  // the block's stack (pending exits, then open entries) is its summary
        unsigned long long off = 0;
        if (lane == 0 && gs.top) off = atomicAdd(p.pool_used, (unsigned long long)gs.top);
        off = __shfl_sync(0xffffffffu, off, 0);
        if (off + gs.top <= p.pool_cap)
          for (uint32_t i = lane; i < gs.top; i += kWarp) p.pool[off + i] = gs.at(i);
        if (lane == 0) {
          SegState st;
          st.status = (p.epoch << 2) | TS_DONE;
          st.pool_n_pending = gs.n_pend;
          st.pool_off = off;
          st.pool_n_resid = gs.top - gs.n_pend;
          st.pad = 0;
          B.out[wid] = st;
        }
      }
      // open calls become truncated spans ending at the global last timestamp
      for (uint32_t ib = 0; !kBlock && ib < gs.top; ib += kWarp) {
        const uint32_t i = ib + lane;
        const bool on = i < gs.top;
        SumEntry en;
        en.ts = 0; en.fn = 0;
        if (on) {
          en = gs.at(i);
          hf.fold(p, en.fn, (p.last_ts_dev ? *p.last_ts : p.global_last_ts) - en.ts, false);
          trunc++;
          spans++;
        }
        if (p.tl_items)  // stacks in (str(hostname), pid, tid) order, innermost first (pipeline.py:230-238)
          tl_emit(p, on, ~0ull, (1ull << 63) | tl_klo(p.flush_rank ? p.flush_rank[s] : s, on ? gs.top - 1 - i : 0), en.ts, 0,
                  TL_HOST | TL_TRUNC | (1u << 4), (uint32_t)en.fn);
      }
    } else if (lane == 0) {
      atomicExch(p.watchdog, 2u);  // stack scratch exhausted (host grows and reruns)
    }
  }
  uint32_t a0 = __reduce_add_sync(0xffffffffu, host), a1 = __reduce_add_sync(0xffffffffu, orph),
           a2 = __reduce_add_sync(0xffffffffu, trunc), a3 = __reduce_add_sync(0xffffffffu, spans);
  if (lane == 0) {
    if (a0) atomicAdd(&p.stats[ST_HOST], (unsigned long long)a0);
    if (a1) atomicAdd(&p.stats[ST_ORPHANS], (unsigned long long)a1);
    if (a2) atomicAdd(&p.stats[ST_TRUNC], (unsigned long long)a2);
    if (a3 && s < p.n_streams) atomicAdd(&p.stream_spans[s], (unsigned long long)a3);
  }
  __syncthreads();
  if (tab) {
    for (uint32_t f = threadIdx.x; f < p.n_fn; f += blockDim.x) {
      SmemRow r = tab[f];
      if (!r.count) continue;
      unsigned long long* a = p.host_acc + 6ull * f;
      atomicAdd(&a[0], (unsigned long long)r.count);
      if (r.err) atomicAdd(&a[1], (unsigned long long)r.err);
      add_i128(&a[2], &a[3], (uint64_t)r.s0 | ((uint64_t)r.s1 << 32), 0);
      atomicMin(&a[4], (unsigned long long)r.mn);
      atomicMax(&a[5], (unsigned long long)r.mx);
    }
  }
}

__global__ void init_acc_kernel(unsigned long long* host_acc, uint32_t n_fn, unsigned long long* dev_acc, uint32_t n_dev,
                                unsigned long long* dev_wide) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_fn) {
    unsigned long long* a = host_acc + 6ull * i;
    a[0] = a[1] = a[2] = a[3] = 0; a[4] = ~0ull; a[5] = 0;
  }
  if (i < n_dev) {
    unsigned long long* a = dev_acc + 6ull * i;
    a[0] = a[1] = a[2] = a[3] = 0; a[4] = ~0ull; a[5] = 0;
    unsigned long long* w = dev_wide + 6ull * i;  // lock, count, min = INT128_MAX, max = INT128_MIN
    w[0] = w[1] = 0; w[2] = ~0ull; w[3] = 0x7FFFFFFFFFFFFFFFull; w[4] = 0; w[5] = 0x8000000000000000ull;
  }
}

}  // namespace

#include "ctx.h"

extern "C" {

int hg_abi_version(void) { return HG_ABI_VERSION; }

const char* hg_last_error(hg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int hg_create(const hg_config* cfg, hg_ctx** out) {
  if (!out) return HG_EARG;
  hg_ctx* ctx = new hg_ctx();
  if (cfg) ctx->cfg = *cfg;
  if (ctx->cfg.tile_bytes) ctx->seg_bytes = std::max<uint32_t>(256, ctx->cfg.tile_bytes);
  *out = ctx;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(ctx, HG_ECUDA, "no CUDA device available");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  for (auto& ev : ctx->ev) CK(cudaEventCreate(&ev));
  CK(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
  CK(cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->cfg.device));
  if (const char* e = getenv("HAPIGPU_PATH")) ctx->path_opt = atoi(e);
  return HG_OK;
}

void hg_destroy(hg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ingest_free(ctx);
  if (ctx->pin) cudaFreeHost(ctx->pin);
  ctx->pin = nullptr;
  ctx->d_schemas.release(); ctx->d_sid_map.release(); ctx->d_kinds.release(); ctx->d_field_role.release();
  ctx->d_data.release(); ctx->d_base.release(); ctx->d_size.release();
  ctx->d_tile_stream.release(); ctx->d_stream_tile0.release();
  ctx->d_state.release(); ctx->d_pool.release(); ctx->d_stack.release();
  ctx->d_host_acc.release(); ctx->d_dev_acc.release(); ctx->d_dev_wide.release(); ctx->d_counters.release();
  ctx->d_orphans.release(); ctx->d_errors.release(); ctx->d_stream_spans.release();
  ctx->d_keys.release(); ctx->d_vals.release(); ctx->d_name_len.release(); ctx->d_small.release();
  ctx->d_name_off.release(); ctx->d_arena.release(); ctx->d_desc.release();
  ctx->d_tl_items.release(); ctx->d_tl_rn.release(); ctx->d_tl_pres.release(); ctx->d_tl_rpre.release();
  ctx->d_ev_rn.release(); ctx->d_ev_seq.release();
  for (int k = 0; k < 2; k++) { ctx->d_tl_keys[k].release(); ctx->d_tl_idx[k].release(); ctx->d_tl_ro[k].release(); }
  ctx->d_tl_tcnt.release(); ctx->d_tl_tile0.release(); ctx->d_tl_split.release();
  ctx->d_tl_lens.release(); ctx->d_tl_stream_proc.release(); ctx->d_tl_offs.release(); ctx->d_tl_bsum.release();
  ctx->d_tl_fnq_off.release(); ctx->d_tl_sstr_off.release(); ctx->d_tl_fnq.release(); ctx->d_tl_sstr.release();
  ctx->d_tl_out.release(); ctx->d_tl_devpid.release(); ctx->d_tl_proc_first.release(); ctx->d_tl_th_state.release();
  ctx->d_tl_th_first.release(); ctx->d_tl_th_hi.release(); ctx->d_tl_th_lo.release();
  ctx->d_segw.release(); ctx->d_seginfo.release(); ctx->d_stream_nrec.release(); ctx->d_tl_rec_off.release();
  ctx->d_deep.release(); ctx->d_params.release();
  ctx->d_range_stream.release(); ctx->d_stream_range0.release(); ctx->d_rstate.release(); ctx->d_rseg.release();
  ctx->d_range_base.release(); ctx->d_vplan.release(); ctx->d_fdesc.release(); ctx->d_dplan.release();
  ctx->d_blk_stream.release(); ctx->d_blk_u0.release(); ctx->d_stream_blk0.release(); ctx->d_blk_state.release();
  for (auto& ev : ctx->ev) if (ev) cudaEventDestroy(ev);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int hg_set_registry(hg_ctx* ctx, const hg_schema* schemas, uint32_t n_schemas, const uint8_t* kinds, uint32_t n_kinds,
                    uint32_t n_functions) {
  if (!ctx || (n_schemas && !schemas)) return HG_EARG;
  ctx->deep_inline = false;
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
      if (d.role_kind[HG_ROLE_RESULT] == HG_KIND_I64) d.flags |= SF_RESULT_I64;
    }
    d.track = 0xFF;  // COUNTER_TRACKS (sinks.py:309-319)
    if (h.event_class == HG_CLASS_TELEMETRY) {
      static const int first[4] = {0, 3, 5, 7}, count[4] = {3, 2, 2, 2};
      if (h.counter_kind < 4 && h.counter_domain >= 0 && h.counter_domain < count[h.counter_kind])
        d.track = (uint8_t)(first[h.counter_kind] + h.counter_domain);
    }
    // var plan
    d.nvar = 0;
    {
      uint32_t nv = 0, lead = 0;
      bool ok = true;
      for (int r = 0; r < HG_NUM_ROLES; r++) { d.role_seg[r] = 0xFF; d.role_delta[r] = 0; }
      for (uint32_t f = 0; f < h.n_fields && ok; f++) {
        uint8_t k = kinds[h.kinds_offset + f];
        for (int r = 0; r < HG_NUM_ROLES; r++)
          if (h.role[r] == (int16_t)f) { d.role_seg[r] = (uint8_t)nv; d.role_delta[r] = (uint16_t)lead; }
        if (k >= HG_KIND_STRING) {
          if (nv == 4 || lead > 0xFFFF) { ok = false; break; }
          d.lead[nv] = (uint16_t)lead;
          d.vkind[nv] = k == HG_KIND_STRING ? 1 : 0;
          nv++;
          lead = 0;
        } else {
          lead += 8;
        }
      }
      if (ok && lead <= 0xFFFF) { d.lead[nv] = (uint16_t)lead; d.nvar = (uint8_t)nv; }
      else d.nvar = kNoPlan;
    }
    if (h.feed_error == 1) d.flags |= SF_FEED_ALWAYS;
    if (h.feed_error == 2) d.flags |= SF_FEED_TIMELINE;
    ctx->sid_map[h.id] = (int32_t)ctx->schemas.size();
    ctx->schemas.push_back(d);
  }
  if (n_functions >= (1u << 19) - 1) return fail(ctx, HG_EUNSUPPORTED, "more than 2^19-2 distinct functions");
  ctx->n_fn = n_functions;
  ctx->max_sid = n_schemas ? max_sid : 0;
  // single-variable-field payload plans for the range kernel's inline checks
  ctx->vplan.assign(ctx->sid_map.size(), 0u);
  for (uint32_t i = 0; i < n_schemas; i++) {
    const DSchema& d = ctx->schemas[ctx->sid_map[schemas[i].id]];
    if ((d.flags & SF_VAR) && d.nvar == 1 && d.lead[0] < 0x4000 && d.lead[1] < 0x4000)
      ctx->vplan[schemas[i].id] = VP_VALID | (d.vkind[0] ? VP_STR : 0u) | ((uint32_t)d.lead[1] << 14) | d.lead[0];
  }
  // compact descriptors: x = fn(20) | cls(3)<<20 | flags(8)<<23 (top bit = present); y = fixed_len | result field<<16
  ctx->desc.assign(ctx->sid_map.size(), make_uint2(0, 0));
  for (uint32_t i = 0; i < n_schemas; i++) {
    const DSchema& d = ctx->schemas[ctx->sid_map[schemas[i].id]];
    uint32_t fn = d.fn < 0 ? 0xFFFFFu : (uint32_t)d.fn;
    uint32_t flags = d.flags & 0x7Fu;
    // result field index (its byte offset / 8); for variable schemas only when every field
    // before it is fixed-size (the segment decoder then reads it without a field walk)
    uint32_t resf = (d.flags & SF_RESULT) ? (uint32_t)d.role[HG_ROLE_RESULT] : 0xFFu;
    if ((d.flags & SF_VAR) && (d.flags & SF_RESULT) && !(d.nvar != kNoPlan && d.role_seg[HG_ROLE_RESULT] == 0 &&
                                                         d.role_delta[HG_ROLE_RESULT] == 8u * resf))
      resf = 0xFFu;
    const bool dt = d.cls == HG_CLASS_DEVICE || d.cls == HG_CLASS_TELEMETRY;
    if ((d.flags & (SF_RESULT_F64 | SF_FEED_ALWAYS)) || ((d.flags & SF_RESULT) && resf > 5u) ||  // result within 64 B
        ((d.flags & SF_VAR) && !dt && !(ctx->vplan[schemas[i].id] & VP_VALID)))
      flags |= SF_NOINLINE;
    ctx->desc[schemas[i].id] = make_uint2((fn & 0xFFFFFu) | ((uint32_t)d.cls << 20) | (flags << 23) | D_PRESENT,
                                          (uint32_t)d.fixed_len | ((resf & 0xFFu) << 16) | ((uint32_t)d.counter_kind << 24));
  }
  // inline-record descriptors of the range kernel (fast.cuh fdesc), one per id plus a sentinel
  ctx->fdesc.assign(ctx->sid_map.size() + 1, make_uint4(M_FN | (FK_NEVER << 20), 1u, 0u, 0u));
  ctx->dplan.assign(ctx->sid_map.size() + 1, make_uint4(0u, 0u, 0u, 0u));
  for (uint32_t i = 0; i < n_schemas; i++) {
    const uint32_t id = schemas[i].id;
    const DSchema& d = ctx->schemas[ctx->sid_map[id]];
    const uint2 dd = ctx->desc[id];
    const uint32_t resf = (dd.y >> 16) & 0xFFu;
    const bool var = (d.flags & SF_VAR) != 0;
    const bool dt = d.cls == HG_CLASS_DEVICE || d.cls == HG_CLASS_TELEMETRY;
    const uint32_t vp = ctx->vplan[id];
    bool never = (d.flags & SF_FEED_ALWAYS) != 0;
    if (d.cls == HG_CLASS_EXIT && (d.flags & SF_RESULT) && ((d.flags & SF_RESULT_F64) || resf != 0)) never = true;
    if (var && !dt && !(vp & VP_VALID)) never = true;
    const uint32_t lo = d.fixed_len, hi = var ? kRInline - 16u : d.fixed_len;
    if (lo > kRInline - 16u) never = true;
    if (never) continue;
    const uint32_t kind = d.cls == HG_CLASS_ENTRY ? FK_ENTRY : d.cls == HG_CLASS_EXIT ? FK_EXIT : dt ? FK_DEFER : FK_PASS;
    uint32_t x = (dd.x & M_FN) | (kind << 20) | (result_kind(d.flags) << 26);
    if (d.cls == HG_CLASS_EXIT && (d.flags & SF_RESULT)) x |= FD_RES;
    if (d.cls == HG_CLASS_DEVICE) x |= FD_ISDEV;
    uint32_t z = 0;
    if (var && !dt) {
      x |= FD_VAR;
      if (vp & VP_STR) x |= FD_STR;
      z = (vp & 0x3FFFu) | (((vp >> 14) & 0x3FFFu) << 16);
    }
    ctx->fdesc[id] = make_uint4(x, lo | (hi << 16), z, 0u);
    // device-profiling records: two variable fields, start/end in the fixed prefix (fast.cuh dplan)
    if (d.cls == HG_CLASS_DEVICE && d.nvar == 2 && d.role[HG_ROLE_START] >= 0 && d.role[HG_ROLE_END] >= 0 &&
        d.role[HG_ROLE_NAME] >= 0 && d.role_seg[HG_ROLE_START] == 0 && d.role_seg[HG_ROLE_END] == 0 &&
        d.role_seg[HG_ROLE_NAME] < 2 && d.role_kind[HG_ROLE_NAME] >= HG_KIND_STRING &&
        d.role_delta[HG_ROLE_NAME] == d.lead[d.role_seg[HG_ROLE_NAME]] &&
        d.role_kind[HG_ROLE_START] != HG_KIND_F64 && d.role_kind[HG_ROLE_END] != HG_KIND_F64 &&
        d.role_kind[HG_ROLE_START] < HG_KIND_STRING && d.role_kind[HG_ROLE_END] < HG_KIND_STRING)
      ctx->dplan[id] = make_uint4(
          (uint32_t)d.lead[0] | ((uint32_t)d.lead[1] << 16),
          (uint32_t)d.lead[2] | ((uint32_t)d.role_seg[HG_ROLE_NAME] << 16) | ((uint32_t)d.vkind[0] << 17) |
              ((uint32_t)d.vkind[1] << 18) | ((d.role_kind[HG_ROLE_START] == HG_KIND_I64 ? 1u : 0u) << 19) |
              ((d.role_kind[HG_ROLE_END] == HG_KIND_I64 ? 1u : 0u) << 20) | (1u << 31),
          (uint32_t)d.role_delta[HG_ROLE_START] | ((uint32_t)d.role_delta[HG_ROLE_END] << 16), 0u);
  }
  ctx->has_dev = false;
  for (const DSchema& d : ctx->schemas) ctx->has_dev |= d.cls == HG_CLASS_DEVICE;
  ctx->fast_warps = 0;
  ctx->staged = false;
  cudaSetDevice(ctx->cfg.device);
  CK(ctx->d_schemas.ensure(std::max<size_t>(ctx->schemas.size(), 1)));
  CK(ctx->d_sid_map.ensure(ctx->sid_map.size()));
  CK(ctx->d_kinds.ensure(std::max<size_t>(n_kinds, 1)));
  CK(ctx->d_field_role.ensure(std::max<size_t>(n_kinds, 1)));
  if (!ctx->schemas.empty())
    CK(cudaMemcpy(ctx->d_schemas.ptr, ctx->schemas.data(), ctx->schemas.size() * sizeof(DSchema), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_sid_map.ptr, ctx->sid_map.data(), ctx->sid_map.size() * 4, cudaMemcpyHostToDevice));
  CK(ctx->d_desc.ensure(ctx->desc.size()));
  CK(cudaMemcpy(ctx->d_desc.ptr, ctx->desc.data(), ctx->desc.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(ctx->d_vplan.ensure(ctx->vplan.size()));
  CK(cudaMemcpy(ctx->d_vplan.ptr, ctx->vplan.data(), ctx->vplan.size() * 4, cudaMemcpyHostToDevice));
  CK(ctx->d_fdesc.ensure(ctx->fdesc.size()));
  CK(cudaMemcpy(ctx->d_fdesc.ptr, ctx->fdesc.data(), ctx->fdesc.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  CK(ctx->d_dplan.ensure(ctx->dplan.size()));
  CK(cudaMemcpy(ctx->d_dplan.ptr, ctx->dplan.data(), ctx->dplan.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  if (n_kinds) {
    CK(cudaMemcpy(ctx->d_kinds.ptr, kinds, n_kinds, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_field_role.ptr, ctx->field_role.data(), n_kinds, cudaMemcpyHostToDevice));
  }
  ctx->have_results = false;
  return HG_OK;
}

int hg_add_stream(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid, const void* data, uint64_t size) {
  if (!ctx || (size && !data)) return HG_EARG;
  HostStream hs{hostname ? hostname : "", pid, tid, (const uint8_t*)data, size, hostname == nullptr};
  hs.pid_none = pid == INT64_MIN;
  hs.tid_none = tid == INT64_MIN;
  ctx->streams.push_back(hs);
  ctx->staged = false;
  ctx->have_results = false;
  return HG_OK;
}

int hg_clear_streams(hg_ctx* ctx) {
  if (!ctx) return HG_EARG;
  ctx->flush_order = false;
  ctx->deep_inline = false;
  ctx->streams.clear();
  ctx->staged = false;
  ctx->have_results = false;
  return HG_OK;
}

static int build_ranges(hg_ctx* ctx);

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
  // exact-path segment size (unless configured): about three waves of seg_decode lanes (~384
  // resident per SM), a power of two in [2 KB, 8 KB] -- small traces get more, shorter lanes
  // (C5 x0.1: 3.1 -> 2.1 ms of phase 1 at 2 KB), big ones keep 8 KB (C5 x1: 15.7 vs 17.5 ms at 4 KB)
  if (!ctx->cfg.tile_bytes) {
    const uint64_t want = off / (3ull * 384 * (uint64_t)std::max(ctx->sm_count, 1));
    uint32_t sb = 2048;
    while (sb < 8192 && 2ull * sb <= want) sb *= 2;
    ctx->seg_bytes = sb;
  }
  // segments: stream-major, each stream cut into seg_bytes pieces from byte 16
  ctx->tile_stream.clear();
  ctx->stream_tile0.assign(ns, 0);
  for (uint32_t s = 0; s < ns; s++) {
    ctx->stream_tile0[s] = (uint32_t)ctx->tile_stream.size();
    const uint64_t sz = ctx->sizes[s];
    const uint32_t nt = sz > 16 ? (uint32_t)((sz - 16 + ctx->seg_bytes - 1) / ctx->seg_bytes) : 0;
    for (uint32_t t = 0; t < nt; t++) ctx->tile_stream.push_back(s);
  }
  return build_ranges(ctx);
}

// ranges for the single pass: one per resident lane, never crossing a stream; range_shift moves
// every cut point (the retry after a failed range speculation)
static int build_ranges(hg_ctx* ctx) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  uint32_t n_fd = 0, n_cd = 0;
  ctx->desc_mode = fast_desc_mode(ctx->max_sid, ctx->n_fn, ctx->has_dev, (uint32_t)ctx->smem_optin, n_fd, n_cd);
  uint32_t nw = kRMaxThreads / kWarp;
  while (nw > 1 && fast_smem_layout(ctx->n_fn, nw, n_fd, n_cd, ctx->has_dev).total > (uint32_t)ctx->smem_optin) nw--;
  ctx->fast_warps = nw;
  const uint64_t lanes = (uint64_t)std::max(ctx->sm_count, 1) * nw * kWarp;
  uint64_t payload = 0, max_pay = 0;
  for (uint32_t s = 0; s < ns; s++) {
    const uint64_t pay = ctx->sizes[s] > 16 ? ctx->sizes[s] - 16 : 0;
    payload += pay;
    max_pay = std::max(max_pay, pay);
  }
  auto count = [&](uint64_t R) {
    uint64_t c = 0;
    for (uint32_t s = 0; s < ns; s++) c += ctx->sizes[s] > 16 ? (ctx->sizes[s] - 16 + R - 1) / R : 0;
    return c;
  };
  uint64_t R = ctx->range_opt ? ctx->range_opt : std::max<uint64_t>(1024, (payload + lanes - 1) / lanes);
  R = (R + 15) & ~15ull;
  if (!ctx->range_opt && count(R) > lanes) {  // smallest R (16-byte steps) with at most one range per lane
    uint64_t lo = R / 16, hi = std::max<uint64_t>(R / 16, (max_pay + 15) / 16);
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (count(mid * 16) <= lanes) hi = mid; else lo = mid + 1;
    }
    R = lo * 16;
  }
  // compose_kernel resolves a stream's range summaries in order (one warp per stream): bound the
  // ranges per stream so a single huge stream does not serialise there
  if (!ctx->range_opt) {
    uint64_t max_per = 8192;
    if (const char* e = getenv("HAPIGPU_MAX_RANGES")) max_per = std::max<uint64_t>(1, strtoull(e, nullptr, 10));
    R = std::max<uint64_t>(R, ((max_pay + max_per - 1) / max_per + 15) & ~15ull);
  }
  R += ctx->range_shift;
  R = std::min<uint64_t>(R, 1ull << 28);
  ctx->range_bytes = (uint32_t)R;
  ctx->range_stream.clear();
  ctx->stream_range0.assign(ns, 0);
  for (uint32_t s = 0; s < ns; s++) {
    ctx->stream_range0[s] = (uint32_t)ctx->range_stream.size();
    const uint64_t nr = ctx->sizes[s] > 16 ? (ctx->sizes[s] - 16 + R - 1) / R : 0;
    for (uint64_t j = 0; j < nr; j++) ctx->range_stream.push_back(s);
  }
  ctx->n_ranges = (uint32_t)ctx->range_stream.size();
  ctx->max_rps = 0;
  for (uint32_t s = 0; s < ns; s++)
    ctx->max_rps = std::max<uint32_t>(ctx->max_rps, (s + 1 < ns ? ctx->stream_range0[s + 1] : ctx->n_ranges) - ctx->stream_range0[s]);
  // compose blocks: up to 32 consecutive ranges of one stream
  ctx->blk_stream.clear();
  ctx->blk_u0.clear();
  ctx->stream_blk0.assign(ns, 0);
  for (uint32_t s = 0; s < ns; s++) {
    ctx->stream_blk0[s] = (uint32_t)ctx->blk_stream.size();
    const uint32_t r0 = ctx->stream_range0[s];
    const uint32_t r1 = s + 1 < ns ? ctx->stream_range0[s + 1] : ctx->n_ranges;
    for (uint32_t r = r0; r < r1; r += kWarp) {
      ctx->blk_stream.push_back(s);
      ctx->blk_u0.push_back(r);
    }
  }
  ctx->n_blk = (uint32_t)ctx->blk_stream.size();
  ctx->blk_u0.push_back(ctx->n_ranges);
  return HG_OK;
}

static int upload_ranges(hg_ctx* ctx) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  const size_t nr = ctx->n_ranges;
  CK(ctx->d_range_stream.ensure(std::max<size_t>(nr, 1)));
  CK(ctx->d_stream_range0.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_rstate.ensure(std::max<size_t>(nr, 1)));
  CK(ctx->d_rseg.ensure(std::max<size_t>(nr, 1)));
  CK(ctx->d_range_base.ensure(std::max<size_t>(nr, 1)));
  if (nr) CK(cudaMemcpyAsync(ctx->d_range_stream.ptr, ctx->range_stream.data(), nr * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(upload(ctx->d_blk_stream, ctx->blk_stream, ctx->stream));
  CK(upload(ctx->d_blk_u0, ctx->blk_u0, ctx->stream));
  CK(upload(ctx->d_stream_blk0, ctx->stream_blk0, ctx->stream));
  CK(ctx->d_blk_state.ensure(std::max<uint32_t>(ctx->n_blk, 1)));
  if (ns) CK(cudaMemcpyAsync(ctx->d_stream_range0.ptr, ctx->stream_range0.data(), ns * 4, cudaMemcpyHostToDevice, ctx->stream));
  return HG_OK;
}

static int stage(hg_ctx* ctx) {
  cudaSetDevice(ctx->cfg.device);
  build_layout(ctx);
  const uint32_t ns = (uint32_t)ctx->streams.size();
  const size_t pad = kDataPad;
  CK(ctx->d_data.ensure(ctx->total_bytes + pad));
  CK(cudaMemsetAsync(ctx->d_data.ptr + ctx->total_bytes, 0, pad, ctx->stream));
  ctx->h2d_bytes = 0;
  int irc = ingest_streams(ctx);  // pinned / pageable / file / device sources (ingest.cu)
  if (irc) return irc;
  CK(ctx->d_base.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_size.ensure(std::max<uint32_t>(ns, 1)));
  if (ns) {
    CK(cudaMemcpyAsync(ctx->d_base.ptr, ctx->base.data(), ns * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_size.ptr, ctx->sizes.data(), ns * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  size_t nt = ctx->tile_stream.size();
  CK(ctx->d_tile_stream.ensure(std::max<size_t>(nt, 1)));
  CK(ctx->d_stream_tile0.ensure(std::max<uint32_t>(ns, 1)));
  if (nt) {
    CK(cudaMemcpyAsync(ctx->d_tile_stream.ptr, ctx->tile_stream.data(), nt * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ns) CK(cudaMemcpyAsync(ctx->d_stream_tile0.ptr, ctx->stream_tile0.data(), ns * 4, cudaMemcpyHostToDevice, ctx->stream));
  int rc = upload_ranges(ctx);
  if (rc) return rc;
  if (ctx->d_state.n < nt) {
    CK(ctx->d_state.ensure(nt));
    CK(cudaMemsetAsync(ctx->d_state.ptr, 0, nt * sizeof(SegState), ctx->stream));
    ctx->epoch = 0;
  }
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
  if (ctx->deep_cap == 0) ctx->deep_cap = 1 << 20;
  CK(ctx->d_deep.ensure(ctx->deep_cap));
  CK(ctx->d_segw.ensure(std::max<size_t>(nt, 1)));
  CK(ctx->d_seginfo.ensure(std::max<size_t>(nt, 1)));
  CK(ctx->d_stream_nrec.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_tl_rec_off.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_pool.ensure(ctx->pool_cap));
  CK(ctx->d_stack.ensure(ctx->stack_cap));
  CK(ctx->d_orphans.ensure(ctx->orphan_cap));
  CK(ctx->d_errors.ensure(ctx->error_cap));
  CK(ctx->d_host_acc.ensure(6ull * std::max<uint32_t>(ctx->n_fn, 1)));
  CK(ctx->d_dev_acc.ensure(6ull * ctx->row_cap));
  CK(ctx->d_dev_wide.ensure(6ull * ctx->row_cap));
  CK(ctx->d_counters.ensure(C_NUM));
  CK(ctx->d_stream_spans.ensure(std::max<uint32_t>(ns, 1)));
  CK(ctx->d_keys.ensure(ctx->dict_mask + 1));
  CK(ctx->d_vals.ensure(ctx->dict_mask + 1));
  CK(ctx->d_name_len.ensure(ctx->row_cap));
  CK(ctx->d_name_off.ensure(ctx->row_cap));
  CK(ctx->d_arena.ensure(ctx->arena_cap));
  return HG_OK;
}

Params make_params(hg_ctx* ctx) {
  Params p{};
  p.data = ctx->d_data.ptr;
  p.stream_base = ctx->d_base.ptr;
  p.stream_size = ctx->d_size.ptr;
  p.tile_stream = ctx->d_tile_stream.ptr;
  p.stream_tile0 = ctx->d_stream_tile0.ptr;
  p.n_tiles = (uint32_t)ctx->tile_stream.size();
  p.n_streams = (uint32_t)ctx->streams.size();
  p.schemas = ctx->d_schemas.ptr;
  p.sid_map = ctx->d_sid_map.ptr;
  p.desc = ctx->d_desc.ptr;
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
  p.dev_wide = ctx->d_dev_wide.ptr;
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
  p.tl_items = (ctx->want & (HG_WANT_TIMELINE | HG_WANT_TL_ITEMS)) ? ctx->d_tl_items.ptr : nullptr;
  p.tl_n = C + C_TL_N;
  p.tl_n2 = C + C_TL_N2;
  p.tl_comp_base = ctx->tl_comp_base;
  p.tl_cap = ctx->tl_cap;
  p.tl_rec_off = ctx->d_tl_rec_off.ptr;
  p.tl_ritems = ctx->tl_ranges ? ctx->d_tl_items.ptr : nullptr;
  p.tl_rcap = ctx->tl_rcap;
  p.tl_rn = ctx->tl_ranges ? ctx->d_tl_rn.ptr : nullptr;
  p.tl_pres = ctx->tl_ranges ? ctx->d_tl_pres.ptr : nullptr;
  p.ev_ritems = ctx->ev_ranges ? ctx->d_ev_items.ptr : nullptr;
  p.ev_rn = ctx->ev_ranges ? ctx->d_ev_rn.ptr : nullptr;
  p.seg_bytes = ctx->seg_bytes;
  p.deep = ctx->d_deep.ptr;
  p.deep_used = C + C_DEEP_USED;
  p.deep_cap = ctx->deep_cap;
  p.range_stream = ctx->d_range_stream.ptr;
  p.stream_range0 = ctx->d_stream_range0.ptr;
  p.n_ranges = ctx->n_ranges;
  p.range_bytes = ctx->range_bytes;
  p.rstate = ctx->d_rstate.ptr;
  p.range_base = ctx->d_range_base.ptr;
  p.anom = reinterpret_cast<uint32_t*>(C + C_ANOM);
  p.vplan = ctx->d_vplan.ptr;
  p.fdesc = ctx->d_fdesc.ptr;
  p.has_dev = ctx->has_dev ? 1u : 0u;
  p.prescan = 0;
  p.dplan = ctx->d_dplan.ptr;
  p.flush_rank = ctx->flush_order ? ctx->d_flush_rank.ptr : nullptr;
  return p;
}

// per-run resets shared by both phase-1 paths
int init_run(hg_ctx* ctx) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  ctx->epoch++;
  if (ctx->epoch >= (1u << 29)) {
    CK(cudaMemsetAsync(ctx->d_state.ptr, 0, ctx->d_state.n * sizeof(SegState), ctx->stream));
    ctx->epoch = 1;
  }
  CK(cudaMemsetAsync(ctx->d_counters.ptr, 0, C_NUM * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_stream_spans.ptr, 0, std::max<uint32_t>(ns, 1) * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_keys.ptr, 0, (ctx->dict_mask + 1) * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_vals.ptr, 0, (ctx->dict_mask + 1) * 4, ctx->stream));
  uint32_t nmax = std::max(ctx->n_fn, ctx->row_cap);
  init_acc_kernel<<<(nmax + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_host_acc.ptr, ctx->n_fn, ctx->d_dev_acc.ptr,
                                                                ctx->row_cap, ctx->d_dev_wide.ptr);
  ctx->launches = 1;
  return HG_OK;
}

// pinned host staging for device -> host result copies (pageable destinations would make every
// cudaMemcpyAsync a synchronous round trip)
static int pinned(hg_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->pin_cap) return HG_OK;
  if (ctx->pin) cudaFreeHost(ctx->pin);
  ctx->pin = nullptr;
  ctx->pin_cap = 0;
  const size_t cap = std::max<size_t>(bytes + (bytes >> 1), 1 << 16);
  CK(cudaHostAlloc(&ctx->pin, cap, cudaHostAllocDefault));
  ctx->pin_cap = cap;
  return HG_OK;
}

static int read_counters(hg_ctx* ctx) {
  int rc = pinned(ctx, C_NUM * 8);
  if (rc) return rc;
  CK(cudaMemcpyAsync(ctx->pin, ctx->d_counters.ptr, C_NUM * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->counters.assign(reinterpret_cast<const unsigned long long*>(ctx->pin),
                       reinterpret_cast<const unsigned long long*>(ctx->pin) + C_NUM);
  return HG_OK;
}

// timeline messages of the single pass: rcap slots per range (a record is at least 16 bytes),
// compose's messages after them (at most one per summary entry); false when they do not fit
static bool tl_range_buffers(hg_ctx* ctx) {
  const uint64_t rcap = ctx->range_bytes / 16ull + 2;
  const uint64_t base = (uint64_t)ctx->n_ranges * rcap;
  const uint64_t cap = base + ctx->pool_cap + 64;
  if (cap >= (1ull << 32)) return false;
  if (ctx->d_tl_items.ensure(cap) != cudaSuccess || ctx->d_tl_rn.ensure(std::max<uint32_t>(ctx->n_ranges, 1)) != cudaSuccess ||
      ctx->d_tl_pres.ensure(std::max<uint64_t>((uint64_t)ctx->n_ranges * kRLP, 1)) != cudaSuccess) {
    cudaGetLastError();  // (clear the allocation failure)
    return false;
  }
  ctx->tl_rcap = (uint32_t)rcap;
  ctx->tl_comp_base = base;
  ctx->tl_cap = cap;
  ctx->tl_ranges = true;
  return true;
}

// every record of the single pass for the event sinks: rcap slots per range
static bool ev_range_buffers(hg_ctx* ctx) {
  const uint64_t rcap = ctx->range_bytes / 16ull + 2;
  const uint64_t cap = (uint64_t)ctx->n_ranges * rcap;
  if (cap >= (1ull << 32)) return false;
  if (ctx->d_ev_items.ensure(std::max<uint64_t>(cap, 1)) != cudaSuccess ||
      ctx->d_ev_rn.ensure(std::max<uint32_t>(ctx->n_ranges, 1)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  ctx->tl_rcap = (uint32_t)rcap;
  ctx->ev_ranges = true;
  return true;
}

int hg_run_local(hg_ctx* ctx, uint32_t want) {
  if (!ctx) return HG_EARG;
  cudaSetDevice(ctx->cfg.device);
  ctx->want = want;
  ctx->have_results = false;
  ctx->merged = false;
  ctx->phase1_done = false;
  // the single pass serves tally, timeline and event runs (per-range lists of the timeline's
  // messages and / or of every record)
  const uint32_t tlw = want & (HG_WANT_TIMELINE | HG_WANT_TL_ITEMS);
  const uint32_t evw = want & (HG_WANT_EVENTS | HG_WANT_VALIDATE);
  bool fast = ctx->path_opt != 1 && !((tlw || evw) && getenv("HAPIGPU_TL_EXACT"));
  ctx->tl_ranges = false;
  ctx->ev_ranges = false;
  bool retried = false;
  for (int attempt = 0; attempt < 9; attempt++) {
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
    ctx->tl_ranges = false;
    ctx->ev_ranges = false;
    if (fast && tlw && !tl_range_buffers(ctx)) fast = false;  // too large: the exact path
    if (fast && evw && !ev_range_buffers(ctx)) fast = false;
    rc = fast ? launch_fast(ctx) : launch_phase1(ctx);
    if (rc) return rc;
    rc = read_counters(ctx);
    if (rc) return rc;
    ctx->h2d_bytes = h2d;
    bool grow = false;
    unsigned long long* C = ctx->counters.data();
    if (C[C_POOL_USED] > ctx->pool_cap || (fast && 2 * C[C_POOL_USED] > ctx->pool_cap)) {  // single pass: room for
      ctx->pool_cap = 2 * C[C_POOL_USED] + (C[C_POOL_USED] >> 2);                         // the block summaries
      ctx->stack_cap = ctx->pool_cap;
      grow = true;
    }
    if (C[C_N_ORPHANS] > ctx->orphan_cap) { ctx->orphan_cap = C[C_N_ORPHANS] * 2; grow = true; }
    if (C[C_DEEP_USED] > ctx->deep_cap) { ctx->deep_cap = C[C_DEEP_USED] * 2; grow = true; }
    // stacks overflowed the inline slots: a rerun (buffers grown) already takes the deep variant
    if (fast && grow && C[C_DEEP_USED] > 0) ctx->deep_inline = true;
    if ((uint32_t)C[C_N_ERRORS] > ctx->error_cap) { ctx->error_cap = (uint32_t)C[C_N_ERRORS] * 2; grow = true; }
    if ((uint32_t)C[C_OVERFLOW]) {
      ctx->row_cap *= 4; ctx->dict_mask = ctx->dict_mask * 4 + 3; ctx->arena_cap = std::max<uint64_t>(ctx->arena_cap * 4, C[C_ARENA_USED] * 2);
      grow = true;
    }
    if (!grow && fast && (uint32_t)ctx->counters[C_ANOM] && !retried && !ctx->range_opt &&
        !((uint32_t)ctx->counters[C_ANOM] & 6u)) {
      // a record-level or chain failure may be a wrong range speculation: move every cut point once
      retried = true;
      ctx->range_shift = 16u * 61u;
      int rr = build_ranges(ctx);
      if (!rr) rr = upload_ranges(ctx);
      ctx->range_shift = 0;
      if (rr) return rr;
      ctx->retries++;
      continue;
    }
    if (!grow && fast && (uint32_t)ctx->counters[C_ANOM]) {
      // the single pass met something it does not reproduce exactly: rerun the exact path
      if (ctx->path_opt == 2) return fail(ctx, HG_ESTATE, "single-pass path rejected the trace (HAPIGPU_PATH=2)");
      fast = false;
      ctx->fallbacks++;
      ctx->last_anom = (uint32_t)ctx->counters[C_ANOM];
      if (getenv("HAPIGPU_DEBUG")) fprintf(stderr, "hapigpu: single pass rejected (reasons 0x%x)\n", ctx->last_anom);
      continue;
    }
    if (!grow) break;
    if (attempt == 8) return fail(ctx, HG_ENOMEM, "scratch buffers kept overflowing");
  }
  ctx->last_path = fast ? 1 : 0;
  // stacks overflowed the inline slots: later runs keep them on the inline path
  if (fast && ctx->counters[C_DEEP_USED] > 0) ctx->deep_inline = true;
  if ((uint32_t)ctx->counters[C_WATCHDOG])
    return fail(ctx, HG_ECUDA, "tile look-back watchdog fired (engine bug)");

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

// cross-range / cross-segment composition and truncation (compose_kernel), queued on the stream
static int launch_compose(hg_ctx* ctx, uint64_t global_last_ts, bool last_ts_on_device) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  if (!ns) return HG_OK;
  Params p = make_params(ctx);
  p.global_last_ts = global_last_ts;
  p.last_ts_dev = last_ts_on_device ? 1u : 0u;
  if (ctx->last_path == 1) {  // summaries per range (fast.cuh)
    p.state = ctx->d_rseg.ptr;
    p.stream_tile0 = ctx->d_stream_range0.ptr;
    p.n_tiles = ctx->n_ranges;
  }
  CK(cudaMemsetAsync(p.stack_used, 0, 8, ctx->stream));
  // the tally accumulators already hold phase-1 spans; compose adds the rest
  size_t csmem = (ctx->n_fn <= kSmemFnMax ? ((sizeof(SmemRow) * ctx->n_fn + 15) & ~(size_t)15) : 0) +
                 sizeof(SumEntry) * kComposeFast * kComposeWarps;
  if (csmem != ctx->compose_smem) {
    CK(cudaFuncSetAttribute(compose_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(csmem, 1)));
    CK(cudaFuncSetAttribute(compose_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(csmem, 1)));
    ctx->compose_smem = csmem;
  }
  if (ctx->last_path == 1 && ctx->n_blk < ctx->n_ranges) {
    // blocks of 32 ranges first, then each stream over its block summaries
    ComposeBlocks B{ctx->d_blk_stream.ptr, ctx->d_blk_u0.ptr, ctx->d_blk_state.ptr, ctx->n_blk};
    compose_kernel<true><<<(ctx->n_blk + kComposeWarps - 1) / kComposeWarps, kComposeWarps * kWarp, csmem,
                           ctx->stream>>>(p, B);
    CK(cudaMemsetAsync(p.stack_used, 0, 8, ctx->stream));
    p.state = ctx->d_blk_state.ptr;
    p.stream_tile0 = ctx->d_stream_blk0.ptr;
    p.n_tiles = ctx->n_blk;
    ctx->launches++;
  }
  compose_kernel<false><<<(ns + kComposeWarps - 1) / kComposeWarps, kComposeWarps * kWarp, csmem, ctx->stream>>>(
      p, ComposeBlocks{nullptr, nullptr, nullptr, 0});
  CK(cudaGetLastError());
  ctx->launches++;
  return HG_OK;
}

static int collect_results(hg_ctx* ctx, uint64_t global_last_ts);

int hg_local_flags(hg_ctx* ctx, uint32_t* flags) {
  if (!ctx || !flags) return HG_EARG;
  if (!ctx->phase1_done) return HG_ESTATE;
  *flags = (uint32_t)ctx->counters[C_WIDE] ? HG_FLAG_WIDE_DEVICE : 0u;
  return HG_OK;
}

int hg_finish(hg_ctx* ctx, uint64_t global_last_ts) {
  if (!ctx || !ctx->phase1_done) return HG_ESTATE;
  cudaSetDevice(ctx->cfg.device);
  const uint32_t ns = (uint32_t)ctx->streams.size();
  for (int attempt = 0; attempt < 3; attempt++) {
    if (ns) {
      int lrc = launch_compose(ctx, global_last_ts, false);
      if (lrc) return lrc;
    }
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    int rc = read_counters(ctx);
    if (rc) return rc;
    if ((uint32_t)ctx->counters[C_WATCHDOG] == 1u) return fail(ctx, HG_ECUDA, "look-back watchdog fired (engine bug)");
    if ((uint32_t)ctx->counters[C_WATCHDOG] == 0u && ctx->counters[C_STACK_USED] <= ctx->stack_cap &&
        ctx->counters[C_N_ORPHANS] <= ctx->orphan_cap)
      break;
    return fail(ctx, HG_ENOMEM, "composition scratch overflow");  // TODO: rerun the whole pipeline with larger buffers
  }
  return collect_results(ctx, global_last_ts);
}

// results to the host (every copy into one pinned staging buffer, one synchronisation), timings,
// and the timeline / event / validation passes a run asked for
static int collect_results(hg_ctx* ctx, uint64_t global_last_ts) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  unsigned long long* C = ctx->counters.data();
  ctx->n_dev_rows = (uint32_t)std::min<unsigned long long>(C[C_N_ROWS], ctx->row_cap);
  ctx->d2h_bytes = C_NUM * 8;
  const uint64_t arena_used = std::min<uint64_t>(C[C_ARENA_USED], ctx->arena_cap);
  const uint64_t n_orph = std::min<uint64_t>(C[C_N_ORPHANS], ctx->orphan_cap);
  const uint32_t n_err = (uint32_t)std::min<unsigned long long>((uint32_t)C[C_N_ERRORS], ctx->error_cap);
  struct Part { void* dst; const void* src; size_t bytes; size_t at; };
  Part parts[9];
  int np = 0;
  size_t total = 0;
  auto part = [&](void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    parts[np++] = Part{dst, src, bytes, total};
    total += (bytes + 15) & ~(size_t)15;
  };
  ctx->host_acc.resize(6ull * ctx->n_fn);
  ctx->dev_acc.resize(6ull * ctx->n_dev_rows);
  ctx->name_off.resize(ctx->n_dev_rows);
  ctx->name_len.resize(ctx->n_dev_rows);
  ctx->arena.resize(arena_used);
  ctx->orphans.resize(n_orph);
  ctx->errors.resize(n_err);
  ctx->stream_spans.resize(ns);
  ctx->dev_wide.assign((uint32_t)ctx->counters[C_WIDE] ? 6ull * ctx->n_dev_rows : 0, 0);
  part(ctx->dev_wide.data(), ctx->d_dev_wide.ptr, ctx->dev_wide.size() * 8);
  part(ctx->host_acc.data(), ctx->d_host_acc.ptr, ctx->host_acc.size() * 8);
  part(ctx->dev_acc.data(), ctx->d_dev_acc.ptr, ctx->dev_acc.size() * 8);
  part(ctx->name_off.data(), ctx->d_name_off.ptr, ctx->n_dev_rows * 8ull);
  part(ctx->name_len.data(), ctx->d_name_len.ptr, ctx->n_dev_rows * 4ull);
  part(ctx->arena.data(), ctx->d_arena.ptr, arena_used);
  part(ctx->orphans.data(), ctx->d_orphans.ptr, n_orph * sizeof(hg_orphan));
  part(ctx->errors.data(), ctx->d_errors.ptr, n_err * sizeof(hg_trace_error));
  part(ctx->stream_spans.data(), ctx->d_stream_spans.ptr, ns * 8ull);
  {
    int prc = pinned(ctx, total);
    if (prc) return prc;
  }
  for (int i = 0; i < np; i++)
    CK(cudaMemcpyAsync(ctx->pin + parts[i].at, parts[i].src, parts[i].bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->ev[3], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < np; i++) memcpy(parts[i].dst, ctx->pin + parts[i].at, parts[i].bytes);
  ctx->d2h_bytes += ctx->host_acc.size() * 8 + ctx->dev_acc.size() * 8 + arena_used + n_orph * sizeof(hg_orphan) +
                    n_err * sizeof(hg_trace_error) + ns * 8 + ctx->n_dev_rows * 12;
  float k_ms = 0, t_ms = 0;
  if (ctx->last_path == 1 && ctx->n_ranges) {  // single pass: decode = range kernel, chain = verification
    cudaEventElapsedTime(&k_ms, ctx->ev[4], ctx->ev[5]);
    ctx->walk_ms = 0;
    cudaEventElapsedTime(&ctx->decode_ms, ctx->ev[4], ctx->ev[7]);
    cudaEventElapsedTime(&ctx->chain_ms, ctx->ev[7], ctx->ev[5]);
  } else if (!ctx->tile_stream.empty()) {
    cudaEventElapsedTime(&k_ms, ctx->ev[4], ctx->ev[5]);
    cudaEventElapsedTime(&ctx->walk_ms, ctx->ev[4], ctx->ev[6]);
    cudaEventElapsedTime(&ctx->chain_ms, ctx->ev[6], ctx->ev[7]);
    cudaEventElapsedTime(&ctx->decode_ms, ctx->ev[7], ctx->ev[5]);
  }
  cudaEventElapsedTime(&t_ms, ctx->ev[0], ctx->ev[3]);
  ctx->kernel_ms = k_ms;
  ctx->total_ms = t_ms;
  ctx->have_results = true;
  ctx->tl_ready = false;
  ctx->ev_ready = false;
  ctx->val_ready = false;
  if (!ctx->errors.empty()) return HG_TRACE_ERROR;
  if (ctx->want & HG_WANT_TIMELINE) {
    int rc = run_timeline(ctx, global_last_ts);
    if (rc) return rc;
  } else if (ctx->want & HG_WANT_TL_ITEMS) {
    int rc = run_timeline_order(ctx);
    if (rc) return rc;
  }
  if (ctx->want & (HG_WANT_EVENTS | HG_WANT_VALIDATE)) {
    int rc = run_events(ctx);
    if (rc) return rc;
  }
  if (ctx->want & HG_WANT_VALIDATE) return run_validation(ctx);
  return HG_OK;
}

// one rank, tally only, single pass: phase 1 and composition back to back -- compose reads the last
// timestamp fast_verify left on the device -- and ONE synchronisation for the counters.  Anything
// the single pass or the scratch sizes cannot vouch for is redone by the split path below.
static int run_fused(hg_ctx* ctx, uint32_t want, bool& done) {
  done = false;
  ctx->want = want;
  ctx->tl_ranges = false;  // (a tally run: no timeline messages; the last timeline run's buffers are stale)
  ctx->ev_ranges = false;
  ctx->have_results = false;
  ctx->merged = false;
  ctx->phase1_done = false;
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  uint64_t h2d = 0;
  if (!ctx->staged) {
    int rc = stage(ctx);
    if (rc) return rc;
    h2d = ctx->h2d_bytes;
  }
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  int rc = ensure_scratch(ctx, 0);
  if (!rc) rc = launch_fast(ctx);
  if (rc) return rc;
  ctx->last_path = 1;
  rc = launch_compose(ctx, 0, true);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  rc = read_counters(ctx);
  if (rc) return rc;
  ctx->h2d_bytes = h2d;
  const unsigned long long* C = ctx->counters.data();
  const bool clean = !(uint32_t)C[C_ANOM] && !(uint32_t)C[C_OVERFLOW] &&
                     !(uint32_t)C[C_WATCHDOG] && !(uint32_t)C[C_N_ERRORS] && 2 * C[C_POOL_USED] <= ctx->pool_cap &&
                     C[C_N_ORPHANS] <= ctx->orphan_cap && C[C_DEEP_USED] <= ctx->deep_cap &&
                     C[C_STACK_USED] <= ctx->stack_cap;
  if (C[C_DEEP_USED] > 0) ctx->deep_inline = true;  // later passes (the split path's too) keep stacks inline
  if (!clean) return HG_OK;  // not done: the split path reruns everything
  ctx->local_last_ts = C[C_LAST_TS];
  ctx->local_events = C[C_STATS + ST_EVENTS];
  ctx->phase1_done = true;
  done = true;
  return collect_results(ctx, ctx->local_last_ts);
}

int hg_run(hg_ctx* ctx, uint32_t want) {
  if (!ctx) return HG_EARG;
  cudaSetDevice(ctx->cfg.device);
  if (want == HG_WANT_TALLY && ctx->path_opt != 1 && !getenv("HAPIGPU_NO_FUSED")) {
    bool done = false;
    int rc = run_fused(ctx, want, done);
    if (rc || done) return rc;
  }
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
      if (!ctx->merged && !ctx->dev_wide.empty() && ctx->dev_wide[6ull * d + 1]) {  // spans beyond +-2^63 ns
        const unsigned long long* w = &ctx->dev_wide[6ull * d];
        const bool narrow = a[0] > w[1];  // some span of the row fit 64 bits
        const __int128 wmn = ((__int128)(int64_t)w[3] << 64) | w[2], wmx = ((__int128)(int64_t)w[5] << 64) | w[4];
        const __int128 nmn = mn, nmx = mx;
        const __int128 fmn = narrow && nmn < wmn ? nmn : wmn, fmx = narrow && nmx > wmx ? nmx : wmx;
        r.min_lo = (uint64_t)fmn; r.min_hi = (int64_t)(fmn >> 64);
        r.max_lo = (uint64_t)fmx; r.max_hi = (int64_t)(fmx >> 64);
      }
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

int hg_set_function_names(hg_ctx* ctx, const char* bytes, const uint64_t* offsets, const uint8_t* is_null,
                          uint32_t n) {
  if (!ctx || (n && !offsets)) return HG_EARG;
  ctx->fn_names.clear();
  ctx->fn_null.assign(n, 0);
  for (uint32_t i = 0; i < n; i++) {
    ctx->fn_names.emplace_back(bytes + offsets[i], bytes + offsets[i + 1]);
    if (is_null) ctx->fn_null[i] = is_null[i];
  }
  ctx->have_fn_names = true;
  return HG_OK;
}

int hg_timeline_size(hg_ctx* ctx, uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return HG_EARG;
  if (!ctx->tl_ready) return fail(ctx, HG_ESTATE, "no timeline: run with HG_WANT_TIMELINE first");
  *n_bytes = ctx->tl_size;
  return HG_OK;
}

int hg_get_timeline(hg_ctx* ctx, char* out, uint64_t cap) {
  if (!ctx || !out) return HG_EARG;
  if (!ctx->tl_ready) return fail(ctx, HG_ESTATE, "no timeline: run with HG_WANT_TIMELINE first");
  if (cap < ctx->tl_size) return fail(ctx, HG_EARG, "timeline buffer too small");
  cudaSetDevice(ctx->cfg.device);
  CK(cudaMemcpy(out, ctx->d_tl_out.ptr, ctx->tl_size, cudaMemcpyDeviceToHost));
  return HG_OK;
}

int hg_phase_timing(hg_ctx* ctx, float* walk_ms, float* chain_ms, float* decode_ms) {
  if (!ctx) return HG_EARG;
  if (walk_ms) *walk_ms = ctx->walk_ms;
  if (chain_ms) *chain_ms = ctx->chain_ms;
  if (decode_ms) *decode_ms = ctx->decode_ms;
  return HG_OK;
}

int hg_set_flush_order(hg_ctx* ctx, const uint32_t* rank, uint32_t n) {
  if (!ctx) return HG_EARG;
  if (!rank || !n) { ctx->flush_order = false; return HG_OK; }
  if (n != ctx->streams.size()) return fail(ctx, HG_EARG, "flush order: one rank per added stream");
  std::vector<uint32_t> r(rank, rank + n), inv(n, ~0u);
  for (uint32_t s = 0; s < n; s++) {
    if (r[s] >= n || inv[r[s]] != ~0u) return fail(ctx, HG_EARG, "flush order is not a permutation");
    inv[r[s]] = s;
  }
  cudaSetDevice(ctx->cfg.device);
  CK(upload(ctx->d_flush_rank, r, ctx->stream));
  CK(upload(ctx->d_flush_stream, inv, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->flush_order = true;
  return HG_OK;
}

int hg_set_timeline_device(hg_ctx* ctx, int32_t device_index) {
  if (!ctx) return HG_EARG;
  ctx->cfg.timeline_device_index = device_index;
  return HG_OK;
}

int hg_timeline_ms(hg_ctx* ctx, float* ms) {
  if (!ctx || !ms) return HG_EARG;
  *ms = ctx->tl_ms;
  return HG_OK;
}

int hg_device_tally(hg_ctx* ctx, void** host_rows, uint64_t* n_host_rows) {
  if (!ctx) return HG_EARG;
  if (host_rows) *host_rows = ctx->d_host_acc.ptr;
  if (n_host_rows) *n_host_rows = ctx->n_fn;
  return HG_OK;
}

int hg_set_option(hg_ctx* ctx, uint32_t key, uint64_t value) {
  if (!ctx) return HG_EARG;
  if (key == HG_OPT_PATH) {
    if (value > 2) return fail(ctx, HG_EARG, "path option: 0 auto, 1 exact, 2 single pass");
    ctx->path_opt = (int)value;
  } else if (key == HG_OPT_RANGE_BYTES) {
    if (value && (value < 16 || value > (1ull << 28))) return fail(ctx, HG_EARG, "range bytes out of [16, 2^28]");
    ctx->range_opt = (uint32_t)((value + 15) & ~15ull);
    ctx->staged = false;
  } else {
    return fail(ctx, HG_EARG, "unknown option");
  }
  return HG_OK;
}

int hg_last_path(hg_ctx* ctx, uint32_t* path, uint64_t* fallbacks, uint32_t* range_bytes) {
  if (!ctx) return HG_EARG;
  if (path) *path = (uint32_t)ctx->last_path;
  if (fallbacks) *fallbacks = ctx->fallbacks;
  if (range_bytes) *range_bytes = ctx->range_bytes;
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
