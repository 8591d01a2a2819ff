// merge.cu -- multi-GPU tally merge (aggregator.py:35-76 as two collectives over device memory).
//
// Every rank owns a disjoint set of streams.  After hg_finish its tally lives in
// d_host_acc (function rows) and d_dev_acc (device-name rows) on the GPU.  hg_merge_export writes
// them, together with IntervalStats and the per-stream span counts, into ONE caller-owned int64
// buffer in a rank-independent layout, so that a SUM all-reduce over its first region and a MAX
// all-reduce over its second region (NCCL, on the caller's side) ARE merge_tallies:
//
//   SUM region  [kMergeStats]            IntervalStats counters + ranks that met a trace error
//               [n_streams_global]       span count per global stream (span identities, sinks.py:240-242)
//               [R x 5]                  count, error_count, sum bits 0-31, sum bits 32-63, sum bits 64-127
//   MAX region  [R]                      ~key(min)   (MAX of ~x = ~MIN of x)
//               [R]                      key(max)
//
// R = n_fn + n_dev_global rows; key(u) = (int64)(u ^ 2^63), which orders host extrema (u64) by
// their unsigned value and device extrema (stored bias64) by their signed value.  The 128-bit sums
// travel as three limbs that stay below 2^63 for any rank count < 2^31, so the SUM is exact.
// hg_merge_import reads the reduced buffer back (host memory) and installs the merged rows and the
// global device-name list as this context's results (hg_get_tally / hg_get_device_names / hg_get_stats).
#include "ctx.h"

namespace {

constexpr uint32_t kMergeStats = 8;

__global__ void merge_export_kernel(const unsigned long long* host_acc, uint32_t n_fn,
                                    const unsigned long long* dev_acc, uint32_t n_dev_local,
                                    const uint32_t* dev_map, uint32_t n_dev_global,
                                    const unsigned long long* stats, uint32_t trace_error,
                                    const unsigned long long* spans, const uint32_t* stream_global,
                                    uint32_t n_streams_local, uint32_t n_streams_global, long long* dst) {
  const uint32_t R = n_fn + n_dev_global;
  long long* s_stats = dst;
  long long* s_spans = s_stats + kMergeStats;
  long long* s_rows = s_spans + n_streams_global;
  long long* m_min = s_rows + 5ull * R;
  long long* m_max = m_min + R;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  // neutral elements first (rows absent on this rank); then the local rows scatter over them
  for (uint32_t i = tid; i < kMergeStats; i += nt) s_stats[i] = i < ST_N ? (long long)stats[i] : (i == ST_N ? trace_error : 0);
  for (uint32_t i = tid; i < n_streams_global; i += nt) s_spans[i] = 0;
  for (uint32_t r = tid; r < n_fn + n_dev_global; r += nt) {
    for (int k = 0; k < 5; k++) s_rows[5ull * r + k] = 0;
    m_min[r] = ~0x7FFFFFFFFFFFFFFFll;  // ~INT64_MAX = INT64_MIN
    m_max[r] = (long long)0x8000000000000000ull;
  }
  __syncthreads();  // single CTA: see the launch
  for (uint32_t i = tid; i < n_streams_local; i += nt) s_spans[stream_global[i]] = (long long)spans[i];
  for (uint32_t r = tid; r < n_fn + n_dev_local; r += nt) {
    const unsigned long long* a = r < n_fn ? host_acc + 6ull * r : dev_acc + 6ull * (r - n_fn);
    if (!a[0]) continue;
    const uint32_t g = r < n_fn ? r : n_fn + dev_map[r - n_fn];
    long long* o = s_rows + 5ull * g;
    o[0] = (long long)a[0];
    o[1] = (long long)a[1];
    o[2] = (long long)(a[2] & 0xFFFFFFFFull);
    o[3] = (long long)(a[2] >> 32);
    o[4] = (long long)a[3];
    m_min[g] = ~(long long)(a[4] ^ 0x8000000000000000ull);
    m_max[g] = (long long)(a[5] ^ 0x8000000000000000ull);
  }
}

}  // namespace

extern "C" {

uint64_t hg_merge_size(uint32_t n_fn, uint32_t n_dev_global, uint32_t n_streams_global, uint64_t* sum_elems) {
  const uint64_t R = (uint64_t)n_fn + n_dev_global;
  if (sum_elems) *sum_elems = kMergeStats + n_streams_global + 5 * R;
  return kMergeStats + n_streams_global + 7 * R;
}

int hg_merge_export(hg_ctx* ctx, void* dst, const uint32_t* dev_map, uint32_t n_dev_local, uint32_t n_dev_global,
                    const uint32_t* stream_global, uint32_t n_streams_global) {
  if (!ctx || !dst) return HG_EARG;
  if (!ctx->have_results) return fail(ctx, HG_ESTATE, "hg_merge_export before hg_finish");
  if (n_dev_local != ctx->n_dev_rows) return fail(ctx, HG_EARG, "dev_map must cover every local device row");
  if ((uint32_t)ctx->counters[C_WIDE])
    return fail(ctx, HG_EUNSUPPORTED, "multi-rank merge of device spans beyond the signed 64-bit range");
  const uint32_t ns = (uint32_t)ctx->streams.size();
  for (uint32_t d = 0; d < n_dev_local; d++)
    if (dev_map[d] >= n_dev_global) return fail(ctx, HG_EARG, "dev_map entry out of range");
  for (uint32_t s = 0; s < ns; s++)
    if (!stream_global || stream_global[s] >= n_streams_global) return fail(ctx, HG_EARG, "stream_global out of range");
  cudaSetDevice(ctx->cfg.device);
  std::vector<uint32_t> maps(dev_map, dev_map + n_dev_local);
  maps.insert(maps.end(), stream_global, stream_global + ns);
  DBuf<uint32_t>& dm = ctx->d_merge_map;
  CK(upload(dm, maps, ctx->stream));
  unsigned long long* C = ctx->d_counters.ptr;
  merge_export_kernel<<<1, 1024, 0, ctx->stream>>>(ctx->d_host_acc.ptr, ctx->n_fn, ctx->d_dev_acc.ptr, n_dev_local,
                                                   dm.ptr, n_dev_global, C + C_STATS, ctx->errors.empty() ? 0u : 1u,
                                                   ctx->d_stream_spans.ptr, dm.ptr + n_dev_local, ns,
                                                   n_streams_global, static_cast<long long*>(dst));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));  // dst is consumed on another stream (the collective's)
  ctx->launches++;
  return HG_OK;
}

int hg_merge_import(hg_ctx* ctx, const void* src, uint32_t n_dev_global, uint32_t n_streams_global,
                    const char* names, const uint64_t* name_offsets) {
  if (!ctx || !src) return HG_EARG;
  if (!ctx->have_results) return fail(ctx, HG_ESTATE, "hg_merge_import before hg_finish");
  if (n_dev_global && (!names || !name_offsets)) return fail(ctx, HG_EARG, "device names required");
  const long long* b = static_cast<const long long*>(src);
  const uint32_t n_fn = ctx->n_fn, R = n_fn + n_dev_global;
  const long long* rows = b + kMergeStats + n_streams_global;
  const long long* mn = rows + 5ull * R;
  const long long* mx = mn + R;
  for (uint32_t i = 0; i < ST_N; i++) ctx->counters[C_STATS + i] = (unsigned long long)b[i];
  ctx->host_acc.assign(6ull * n_fn, 0);
  ctx->dev_acc.assign(6ull * n_dev_global, 0);
  for (uint32_t r = 0; r < R; r++) {
    const long long* o = rows + 5ull * r;
    unsigned long long* a = r < n_fn ? &ctx->host_acc[6ull * r] : &ctx->dev_acc[6ull * (r - n_fn)];
    if (!o[0]) continue;
    const unsigned __int128 lo = (unsigned __int128)(unsigned long long)o[2] +
                                 ((unsigned __int128)(unsigned long long)o[3] << 32);
    const __int128 sum = (__int128)lo + ((__int128)o[4] << 64);
    a[0] = (unsigned long long)o[0];
    a[1] = (unsigned long long)o[1];
    a[2] = (unsigned long long)sum;
    a[3] = (unsigned long long)(sum >> 64);
    a[4] = (unsigned long long)(~mn[r]) ^ 0x8000000000000000ull;
    a[5] = (unsigned long long)mx[r] ^ 0x8000000000000000ull;
  }
  ctx->n_dev_rows = n_dev_global;
  ctx->name_off.resize(n_dev_global);
  ctx->name_len.resize(n_dev_global);
  const uint64_t nb = n_dev_global ? name_offsets[n_dev_global] : 0;
  ctx->arena.assign(names, names + nb);
  for (uint32_t d = 0; d < n_dev_global; d++) {
    ctx->name_off[d] = name_offsets[d];
    ctx->name_len[d] = (uint32_t)(name_offsets[d + 1] - name_offsets[d]);
  }
  ctx->merged = true;
  return HG_OK;
}

}  // extern "C"
