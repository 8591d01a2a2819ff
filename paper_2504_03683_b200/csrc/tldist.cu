// tldist.cu -- the timeline of a multi-rank run (collective (6) of SURVEY.md §8e; TimelineSink,
// sinks.py:341-418, whose object order is the global mux order of pipeline.py:68-114).
//
// Every rank decodes and pairs its own streams (HG_WANT_TL_ITEMS: the exact phase 1 emits the
// timeline messages, compose the cross-range and truncated spans, tl_sort orders them by mux key).
// hg_tl_export turns that sorted run into a rank-independent form: the stream field of every key
// becomes the stream's index in the whole trace (truncated spans: its global flush rank), and the
// device / telemetry messages, which print fields of their record, carry a copy of the record's
// payload.  Rank 0 receives the runs (NCCL on the caller's side) and hg_tl_import merges them --
// the same merge-path passes that merge a single GPU's stream runs (tl_sort_runs, one run per rank)
// -- and formats them with the whole trace's stream identities (timeline_from), so the bytes equal
// a single run over the whole trace.
#define HG_TLX_KERNELS
#include "ctx.h"

namespace {

__device__ __forceinline__ bool has_payload(const TlItem& it) {
  const uint32_t k = it.kind & 3u;
  return k == TL_DEVICE || k == TL_SAMPLE;
}

// payload length of every message (0 for host spans); the record header precedes the payload
__global__ void tlx_len_kernel(const TlItem* items, const uint32_t* order, uint32_t n, uint32_t* len) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const TlItem it = items[order[i]];
    len[i] = has_payload(it) ? ldu32(reinterpret_cast<const uint8_t*>(it.a) - 4) : 0u;
  }
}

// the sorted run with global stream keys; payloads copied to their offsets
__global__ void tlx_write_kernel(const TlItem* items, const uint32_t* order, uint32_t n, const uint64_t* off,
                                 const uint32_t* len, const uint32_t* smap, const uint32_t* fmap,
                                 const uint32_t* flush_stream, TlItem* out, uint8_t* pay) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    TlItem it = items[order[i]];
    const uint64_t trunc = it.klo >> 63, field = (it.klo >> 40) & 0x7FFFFFull, low = it.klo & ((1ull << 40) - 1);
    uint64_t g;
    if (trunc) {
      const uint32_t s = flush_stream ? flush_stream[field] : (uint32_t)field;
      g = fmap[s];
    } else {
      g = smap[field];
    }
    it.klo = (trunc << 63) | (g << 40) | low;
    if (has_payload(it)) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(it.a);
      uint8_t* dst = pay + off[i];
      for (uint32_t b = 0; b < len[i]; b++) dst[b] = src[b];
      it.a = off[i];
    }
    out[i] = it;
  }
}

// rank 0: payload offsets -> addresses in the concatenated payload buffer
__global__ void tlx_fix_kernel(TlItem* items, uint64_t n, const unsigned long long* run0, const uint64_t* pay0,
                               uint32_t runs, const uint8_t* pay) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    TlItem it = items[j];
    if (!has_payload(it)) continue;
    uint32_t lo = 0, hi = runs;  // last run starting at or before j
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (run0[mid] <= j) lo = mid;
      else hi = mid;
    }
    it.a = reinterpret_cast<uint64_t>(pay + pay0[lo] + it.a);
    items[j] = it;
  }
}

}  // namespace

extern "C" {

int hg_tl_export(hg_ctx* ctx, const uint32_t* stream_global, const uint32_t* flush_global, void* items, void* payload,
                 uint64_t* n_items, uint64_t* payload_bytes, uint64_t* n_device_spans) {
  if (!ctx || !n_items || !payload_bytes) return HG_EARG;
  if (!ctx->have_results || !ctx->tl_order) return fail(ctx, HG_ESTATE, "hg_tl_export needs a run with HG_WANT_TL_ITEMS");
  cudaSetDevice(ctx->cfg.device);
  cudaStream_t st = ctx->stream;
  const uint32_t n = ctx->tl_n, ns = (uint32_t)ctx->streams.size();
  if (n_device_spans) *n_device_spans = ctx->counters[C_STATS + ST_DEVICE];
  CK(ctx->d_tlx_len.ensure(std::max<uint32_t>(n, 1)));
  CK(ctx->d_tlx_off.ensure(std::max<uint32_t>(n, 1)));
  const uint32_t g = std::max<uint32_t>(1, std::min<uint32_t>((n + 255) / 256, (uint32_t)ctx->sm_count * 8));
  if (!items) {  // sizes
    uint64_t total = 0;
    if (n) {
      tlx_len_kernel<<<g, 256, 0, st>>>(ctx->d_tl_items.ptr, ctx->tl_order, n, ctx->d_tlx_len.ptr);
      int rc = tl_scan(ctx, ctx->d_tlx_len.ptr, n, ctx->d_tlx_off.ptr,
                       reinterpret_cast<uint64_t*>(ctx->d_counters.ptr + C_TL_TOTAL));
      if (rc) return rc;
      CK(cudaMemcpyAsync(&total, ctx->d_counters.ptr + C_TL_TOTAL, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      ctx->launches++;
    }
    *n_items = n;
    *payload_bytes = total;
    return HG_OK;
  }
  if (ns && (!stream_global || !flush_global)) return HG_EARG;
  std::vector<uint32_t> maps(stream_global, stream_global + ns);
  maps.insert(maps.end(), flush_global, flush_global + ns);
  CK(upload(ctx->d_tlx_map, maps, st));
  if (n) {
    tlx_write_kernel<<<g, 256, 0, st>>>(ctx->d_tl_items.ptr, ctx->tl_order, n, ctx->d_tlx_off.ptr, ctx->d_tlx_len.ptr,
                                        ctx->d_tlx_map.ptr, ctx->d_tlx_map.ptr + ns,
                                        ctx->flush_order ? ctx->d_flush_stream.ptr : nullptr,
                                        static_cast<TlItem*>(items), static_cast<uint8_t*>(payload));
    CK(cudaGetLastError());
    ctx->launches++;
  }
  CK(cudaStreamSynchronize(st));  // the buffers are consumed on another stream (the collective's)
  *n_items = n;
  return HG_OK;
}

int hg_tl_import(hg_ctx* ctx, void* items, uint64_t n_items, const uint64_t* run_start, const uint64_t* payload_start,
                 uint32_t n_runs, const void* payload, const char* const* hosts, const int64_t* pids, const int64_t* tids,
                 uint32_t n_streams, const uint32_t* flush_stream, uint64_t n_device_spans, uint64_t global_last_ts) {
  if (!ctx || (n_items && !items) || !run_start || !payload_start || !pids || !tids || (n_streams && !flush_stream))
    return HG_EARG;
  if (n_items >= (1ull << 32)) return fail(ctx, HG_EUNSUPPORTED, "timeline: more than 2^32 messages");
  cudaSetDevice(ctx->cfg.device);
  cudaStream_t st = ctx->stream;
  std::vector<unsigned long long> runs(run_start, run_start + n_runs);
  std::vector<uint64_t> pay0(payload_start, payload_start + n_runs);
  CK(upload(ctx->d_tlx_runs, runs, st));
  CK(upload(ctx->d_tlx_off, pay0, st));
  std::vector<uint32_t> fl(flush_stream, flush_stream + n_streams);
  CK(upload(ctx->d_tlx_flush, fl, st));
  TlItem* it = static_cast<TlItem*>(items);
  if (n_items) {
    const uint32_t g = std::max<uint32_t>(1, std::min<uint64_t>((n_items + 255) / 256, (uint64_t)ctx->sm_count * 8));
    tlx_fix_kernel<<<g, 256, 0, st>>>(it, n_items, ctx->d_tlx_runs.ptr, ctx->d_tlx_off.ptr, n_runs,
                                      static_cast<const uint8_t*>(payload));
    CK(cudaGetLastError());
    ctx->launches++;
  }
  TlSource S;
  S.items = it;
  S.nrec_slots = (uint32_t)n_items;
  S.N = (uint32_t)n_items;
  S.ncomp = 0;
  S.n = (uint32_t)n_items;
  S.rec_off = ctx->d_tlx_runs.ptr;
  S.n_runs = n_runs;
  for (uint32_t s = 0; s < n_streams; s++)
    S.streams.push_back(TlStreamName{hosts[s] ? hosts[s] : "", hosts[s] == nullptr, pids[s], pids[s] == INT64_MIN,
                                     tids[s], tids[s] == INT64_MIN});
  S.flush_stream = ctx->d_tlx_flush.ptr;
  S.n_dev = n_device_spans;
  return timeline_from(ctx, S, global_last_ts);
}

}  // extern "C"
