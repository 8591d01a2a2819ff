// timeline.cu -- timeline ordering and JSON formatting on the GPU (timeline.cuh)
#define HG_TL_KERNELS
#include "ctx.h"

// stable order of message slots by mux key (khi, klo): items[0, nrec_slots) hold every stream's
// record-region run (stream s from rec_off[s]; empty slots have key ~0), items[nrec_slots, N) the
// ncomp messages compose appended (unsorted); n = messages in all.  The record-region runs are
// compacted, compose's messages sorted per tile, then all runs merged pairwise with merge-path
// passes -- the k-way merge of the reference's muxer (pipeline.py:68-114).  *order = item index
// of every message in mux order (a scratch buffer of the context, valid until the next sort).
int tl_sort_runs(hg_ctx* ctx, const TlItem* items, uint32_t nrec_slots, uint32_t N, uint32_t ncomp, uint32_t n,
                 const unsigned long long* rec_off, uint32_t ns, const uint32_t** order) {
  cudaStream_t st = ctx->stream;
  const uint32_t nrec = n - ncomp;
  const uint32_t n_rtiles = (nrec_slots + kSortTile - 1) / kSortTile;
  const uint32_t ntc = (ncomp + kSortTile - 1) / kSortTile;
  uint32_t R = ns + ntc;
  for (int k = 0; k < 2; k++) {
    CK(ctx->d_tl_keys[k].ensure(std::max<uint32_t>(n, 1)));
    CK(ctx->d_tl_idx[k].ensure(std::max<uint32_t>(n, 1)));
    CK(ctx->d_tl_ro[k].ensure(R + 2));
  }
  CK(ctx->d_tl_tcnt.ensure(n_rtiles + 2));
  CK(ctx->d_tl_tile0.ensure(R / 2 + 3));
  CK(ctx->d_tl_split.ensure(n / kSortTile + R / 2 + 3));
  if (n) {
    if (n_rtiles) {
      tl_count_kernel<<<n_rtiles, kSortThreads, 0, st>>>(items, nrec_slots, ctx->d_tl_tcnt.ptr);
      tl_small_scan_kernel<<<1, 1024, 0, st>>>(ctx->d_tl_tcnt.ptr, n_rtiles);
      ctx->launches += 2;
    }
    tl_compact_kernel<<<n_rtiles + std::max<uint32_t>(ntc, 1), kSortThreads, 0, st>>>(
        items, nrec_slots, N, ctx->d_tl_tcnt.ptr, n_rtiles, rec_off, ns, nrec, n,
        ctx->d_tl_keys[0].ptr, ctx->d_tl_idx[0].ptr, ctx->d_tl_ro[0].ptr);
    ctx->launches++;
    if (ntc) {
      tl_tilesort_kernel<<<ntc, kSortThreads, 0, st>>>(ctx->d_tl_keys[0].ptr, ctx->d_tl_idx[0].ptr, nrec, ncomp);
      ctx->launches++;
    }
    CK(cudaGetLastError());
  }
  return tl_merge_passes(ctx, R, n, order);
}

// the merge-path passes over the R sorted runs in d_tl_keys[0] / d_tl_idx[0] (run offsets in
// d_tl_ro[0]); returns the item index of every message in mux order
int tl_merge_passes(hg_ctx* ctx, uint32_t R, uint32_t n, const uint32_t** order) {
  cudaStream_t st = ctx->stream;
  int cur = 0;
  if (n) {
    while (R > 1) {
      const uint32_t P = (R + 1) / 2;
      const uint32_t tiles = n / kSortTile + P + 1;  // bound on the output tiles of the pass
      tl_pairs_kernel<<<1, 1024, 0, st>>>(ctx->d_tl_ro[cur].ptr, R, ctx->d_tl_tile0.ptr, ctx->d_tl_ro[cur ^ 1].ptr);
      tl_split_kernel<<<(tiles + 127) / 128, 128, 0, st>>>(ctx->d_tl_keys[cur].ptr, ctx->d_tl_ro[cur].ptr, R,
                                                           ctx->d_tl_tile0.ptr, ctx->d_tl_split.ptr);
      tl_merge_kernel<<<tiles, kSortThreads, 0, st>>>(ctx->d_tl_keys[cur].ptr, ctx->d_tl_idx[cur].ptr,
                                                      ctx->d_tl_keys[cur ^ 1].ptr, ctx->d_tl_idx[cur ^ 1].ptr,
                                                      ctx->d_tl_ro[cur].ptr, R, ctx->d_tl_tile0.ptr, ctx->d_tl_split.ptr);
      CK(cudaGetLastError());
      ctx->launches += 3;
      cur ^= 1;
      R = P;
    }
  }
  *order = ctx->d_tl_idx[cur].ptr;
  return HG_OK;
}

// the single pass's messages (per range) + compose's: keys of every range appended in range order
// (tl_range_compact_kernel), compose's tiles sorted, then the merge passes
int tl_sort_ranges(hg_ctx* ctx, const TlSource& S, uint32_t* n_out, const uint32_t** order) {
  cudaStream_t st = ctx->stream;
  const uint32_t nr = S.n_ranges, ns = S.n_runs, ncomp = S.ncomp;
  CK(ctx->d_tl_rpre.ensure(nr + 1));
  if (nr) CK(cudaMemcpyAsync(ctx->d_tl_rpre.ptr, S.rn, nr * 4ull, cudaMemcpyDeviceToDevice, st));
  tl_small_scan_kernel<<<1, 1024, 0, st>>>(ctx->d_tl_rpre.ptr, nr);  // exclusive; [nr] = the total
  uint32_t nrec = 0;
  CK(cudaMemcpyAsync(&nrec, ctx->d_tl_rpre.ptr + nr, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ctx->launches++;
  const uint64_t n64 = (uint64_t)nrec + ncomp;
  if (n64 >= (1ull << 32)) return fail(ctx, HG_EUNSUPPORTED, "timeline: more than 2^32 messages");
  const uint32_t n = (uint32_t)n64;
  const uint32_t ntc = (ncomp + kSortTile - 1) / kSortTile;
  const uint32_t R = ns + ntc;
  for (int k = 0; k < 2; k++) {
    CK(ctx->d_tl_keys[k].ensure(std::max<uint32_t>(n, 1)));
    CK(ctx->d_tl_idx[k].ensure(std::max<uint32_t>(n, 1)));
    CK(ctx->d_tl_ro[k].ensure(R + 2));
  }
  CK(ctx->d_tl_tile0.ensure(R / 2 + 3));
  CK(ctx->d_tl_split.ensure(n / kSortTile + R / 2 + 3));
  const uint32_t nrb = (nr + kSortThreads / 32 - 1) / (kSortThreads / 32);
  tl_range_compact_kernel<<<nrb + std::max<uint32_t>(ntc, 1), kSortThreads, 0, st>>>(
      const_cast<TlItem*>(S.items), nr, S.rcap, S.rn, ctx->d_tl_rpre.ptr, S.range_stream, S.range_base,
      S.stream_range0, ns, S.nrec_slots, ncomp, nrec, ctx->d_tl_keys[0].ptr, ctx->d_tl_idx[0].ptr, ctx->d_tl_ro[0].ptr);
  ctx->launches++;
  if (ntc) {
    tl_tilesort_kernel<<<ntc, kSortThreads, 0, st>>>(ctx->d_tl_keys[0].ptr, ctx->d_tl_idx[0].ptr, nrec, ncomp);
    ctx->launches++;
  }
  CK(cudaGetLastError());
  *n_out = n;
  return tl_merge_passes(ctx, R, n, order);
}

int tl_sort(hg_ctx* ctx, const TlItem* items, uint32_t nrec_slots, uint32_t N, uint32_t ncomp, uint32_t n,
            const uint32_t** order) {
  return tl_sort_runs(ctx, items, nrec_slots, N, ncomp, n, ctx->d_tl_rec_off.ptr, (uint32_t)ctx->streams.size(), order);
}

// exclusive scan of n u32 lengths into u64 offsets, *total (device) = the sum
int tl_scan(hg_ctx* ctx, const uint32_t* lens, uint32_t n, uint64_t* offs, uint64_t* total) {
  const uint32_t nsb = (n + kScanBlock - 1) / kScanBlock;
  CK(ctx->d_tl_bsum.ensure(std::max<uint32_t>(nsb, 1)));
  tl_scan1_kernel<<<nsb, kScanBlock, 0, ctx->stream>>>(lens, n, ctx->d_tl_bsum.ptr);
  tl_scan2_kernel<<<1, kScanBlock, 0, ctx->stream>>>(ctx->d_tl_bsum.ptr, nsb, total);
  tl_scan3_kernel<<<nsb, kScanBlock, 0, ctx->stream>>>(lens, n, ctx->d_tl_bsum.ptr, offs);
  ctx->launches += 3;
  return HG_OK;
}

// the context's own messages: the record region of every stream + compose's messages
static TlSource own_source(hg_ctx* ctx) {
  const unsigned long long* C = ctx->counters.data();
  TlSource S;
  if (ctx->tl_ranges) {  // the single pass's per-range messages (n: known after their scan)
    S.ranges = true;
    S.n_ranges = ctx->n_ranges;
    S.rcap = ctx->tl_rcap;
    S.rn = ctx->d_tl_rn.ptr;
    S.range_stream = ctx->d_range_stream.ptr;
    S.range_base = ctx->d_range_base.ptr;
    S.stream_range0 = ctx->d_stream_range0.ptr;
  }
  S.items = ctx->d_tl_items.ptr;
  S.nrec_slots = (uint32_t)ctx->tl_comp_base;
  S.N = (uint32_t)(ctx->tl_comp_base + C[C_TL_N2]);
  S.ncomp = (uint32_t)C[C_TL_N2];
  S.n = (uint32_t)(C[C_TL_N] + C[C_TL_N2]);  // messages; the sort moves the empty slots last
  S.rec_off = ctx->d_tl_rec_off.ptr;
  S.n_runs = (uint32_t)ctx->streams.size();
  for (const HostStream& hs : ctx->streams)
    S.streams.push_back(TlStreamName{hs.host, hs.host_none, hs.pid, hs.pid_none, hs.tid, hs.tid_none});
  S.flush_stream = ctx->flush_order ? ctx->d_flush_stream.ptr : nullptr;
  S.n_dev = C[C_STATS + ST_DEVICE];
  return S;
}

int run_timeline(hg_ctx* ctx, uint64_t global_last_ts) {
  ctx->tl_ready = false;
  const unsigned long long* C = ctx->counters.data();
  const uint64_t n_slots = ctx->tl_comp_base + C[C_TL_N2];
  if (n_slots > ctx->tl_cap || n_slots >= (1ull << 32))
    return fail(ctx, HG_ENOMEM, "timeline message buffer overflow");
  return timeline_from(ctx, own_source(ctx), global_last_ts);
}

// the messages of a context sorted by mux key only (a rank's share of a multi-rank timeline)
int run_timeline_order(hg_ctx* ctx) {
  ctx->tl_order = nullptr;
  const unsigned long long* C = ctx->counters.data();
  if (ctx->tl_comp_base + C[C_TL_N2] > ctx->tl_cap || ctx->tl_comp_base + C[C_TL_N2] >= (1ull << 32))
    return fail(ctx, HG_ENOMEM, "timeline message buffer overflow");
  const TlSource S = own_source(ctx);
  if (S.ranges) return tl_sort_ranges(ctx, S, &ctx->tl_n, &ctx->tl_order);
  ctx->tl_n = S.n;
  return tl_sort_runs(ctx, S.items, S.nrec_slots, S.N, S.ncomp, S.n, S.rec_off, S.n_runs, &ctx->tl_order);
}

// order, format and store the timeline JSON (TimelineSink.on_finish, sinks.py:414-418)
int timeline_from(hg_ctx* ctx, const TlSource& S, uint64_t global_last_ts) {
  ctx->tl_ready = false;
  if (!ctx->have_fn_names || ctx->fn_names.size() != ctx->n_fn)
    return fail(ctx, HG_ESTATE, "hg_set_function_names is required for the timeline");
  uint32_t n = S.n;
  const uint32_t ns = (uint32_t)S.streams.size();
  cudaStream_t st = ctx->stream;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  // host tables: quoted function names; per stream pid, tid, process name
  std::vector<char> fnq;
  std::vector<uint64_t> fnq_off(1, 0);
  for (uint32_t f = 0; f < ctx->n_fn; f++) {
    std::string q = ctx->fn_null[f] ? std::string("null") : json_quote(ctx->fn_names[f]);
    fnq.insert(fnq.end(), q.begin(), q.end());
    fnq_off.push_back(fnq.size());
  }
  const int64_t dev_pid = 9000000 + (int64_t)ctx->cfg.timeline_device_index;
  std::vector<char> sstr;
  std::vector<uint64_t> sstr_off(1, 0);
  std::vector<uint32_t> sproc(std::max<uint32_t>(ns, 1), 0);
  std::map<int64_t, uint32_t> proc_id;  // process_name metas are keyed by (pid, 0)
  for (uint32_t s = 0; s < ns; s++) {
    const TlStreamName& hs = S.streams[s];
    // None pid / tid (record sources): JSON null, "None" in the process name (sinks.py:367-369)
    std::string a = hs.pid_none ? std::string("null") : std::to_string(hs.pid);
    std::string b = hs.tid_none ? std::string("null") : std::to_string(hs.tid);
    std::string c = json_quote("Host " + (hs.host_none ? std::string("None") : hs.host) + " pid " +
                               (hs.pid_none ? std::string("None") : a));
    for (const std::string* x : {&a, &b, &c}) {
      sstr.insert(sstr.end(), x->begin(), x->end());
      sstr_off.push_back(sstr.size());
    }
    auto it = proc_id.find(hs.pid);
    if (it == proc_id.end()) it = proc_id.emplace(hs.pid, (uint32_t)proc_id.size()).first;
    sproc[s] = it->second;
  }
  auto dit = proc_id.find(dev_pid);
  const uint32_t dev_proc = dit != proc_id.end() ? dit->second : (uint32_t)proc_id.size();
  const uint32_t n_proc = (uint32_t)proc_id.size() + 1;
  std::string dps = std::to_string(dev_pid);
  std::vector<char> devpid(dps.begin(), dps.end());
  for (std::vector<char>* v : {&fnq, &sstr, &devpid}) v->insert(v->end(), 8, '\0');  // word-wise readers
  CK(upload(ctx->d_tl_fnq, fnq, st));
  CK(upload(ctx->d_tl_fnq_off, fnq_off, st));
  CK(upload(ctx->d_tl_sstr, sstr, st));
  CK(upload(ctx->d_tl_sstr_off, sstr_off, st));
  CK(upload(ctx->d_tl_stream_proc, sproc, st));
  CK(upload(ctx->d_tl_devpid, devpid, st));
  // sort by mux key: the streams' record slots are sorted runs; drop the empty slots, sort
  // compose's messages per tile, merge the runs pairwise
  const uint32_t* order = nullptr;
  {
    int rc = S.ranges ? tl_sort_ranges(ctx, S, &n, &order)
                      : tl_sort_runs(ctx, S.items, S.nrec_slots, S.N, S.ncomp, n, S.rec_off, S.n_runs, &order);
    if (rc) return rc;
  }
  // metadata first occurrences
  const uint64_t n_dev = S.n_dev;
  uint32_t th_size = 64;
  while (th_size < 2 * n_dev && th_size < (1u << 30)) th_size <<= 1;
  CK(ctx->d_tl_proc_first.ensure(n_proc));
  CK(ctx->d_tl_th_state.ensure(th_size));
  CK(ctx->d_tl_th_first.ensure(kThDirect + th_size));
  CK(ctx->d_tl_th_hi.ensure(th_size));
  CK(ctx->d_tl_th_lo.ensure(th_size));
  CK(cudaMemsetAsync(ctx->d_tl_proc_first.ptr, 0xFF, n_proc * 4, st));
  CK(cudaMemsetAsync(ctx->d_tl_th_state.ptr, 0, (size_t)th_size * 4, st));
  CK(cudaMemsetAsync(ctx->d_tl_th_first.ptr, 0xFF, (size_t)(kThDirect + th_size) * 4, st));
  CK(ctx->d_tl_lens.ensure(std::max<uint32_t>(n, 1)));
  CK(ctx->d_tl_offs.ensure(std::max<uint32_t>(n, 1)));
  TlTables T{};
  T.items = S.items;
  T.n = n;
  T.order = order;
  T.fnq = ctx->d_tl_fnq.ptr;
  T.fnq_off = ctx->d_tl_fnq_off.ptr;
  T.sstr = ctx->d_tl_sstr.ptr;
  T.sstr_off = ctx->d_tl_sstr_off.ptr;
  T.stream_proc = ctx->d_tl_stream_proc.ptr;
  T.dev_proc = dev_proc;
  T.dev_pid = ctx->d_tl_devpid.ptr;
  T.dev_pid_len = (uint32_t)dps.size();
  T.proc_first = ctx->d_tl_proc_first.ptr;
  T.th_state = ctx->d_tl_th_state.ptr;
  T.th_hi = ctx->d_tl_th_hi.ptr;
  T.th_lo = ctx->d_tl_th_lo.ptr;
  T.th_first = ctx->d_tl_th_first.ptr;
  T.th_mask = th_size - 1;
  T.th_overflow = reinterpret_cast<unsigned int*>(ctx->d_counters.ptr + C_TL_TH_OVF);
  T.schemas = ctx->d_schemas.ptr;
  T.sid_map = ctx->d_sid_map.ptr;
  T.kinds = ctx->d_kinds.ptr;
  T.max_sid = ctx->max_sid;
  T.last_ts = global_last_ts;
  T.flush_stream = S.flush_stream;
  T.lens = ctx->d_tl_lens.ptr;
  T.offs = ctx->d_tl_offs.ptr;
  uint64_t total = 0;
  if (n) {
    const uint32_t g = std::min<uint32_t>((n + kTlTile - 1) / kTlTile, (uint32_t)ctx->sm_count * HG_TL_LEN_MINB * 2);
    tl_len_kernel<<<g, kTlThreads, 0, st>>>(T);
    tl_meta_len_kernel<<<std::min<uint32_t>((n_proc + kThDirect + th_size + 255) / 256, (uint32_t)ctx->sm_count * 8), 256,
                         0, st>>>(T, n_proc, kThDirect + th_size);
    tl_scan(ctx, T.lens, n, T.offs, reinterpret_cast<uint64_t*>(ctx->d_counters.ptr + C_TL_TOTAL));
    CK(cudaGetLastError());
    ctx->launches += 2;
    unsigned long long tail[2] = {0, 0};
    CK(cudaMemcpyAsync(tail, ctx->d_counters.ptr + C_TL_TOTAL, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((uint32_t)tail[1]) return fail(ctx, HG_ENOMEM, "timeline thread-name table overflow");
    total = tail[0];
  }
  // "[" + body + "\n]"  (json.dump of a non-empty list, indent=1); "[]" when empty
  ctx->tl_size = n ? total + 3 : 2;
  CK(ctx->d_tl_out.ensure(ctx->tl_size + 32));
  T.out = ctx->d_tl_out.ptr;
  static const char open_close[4] = {'[', '\n', ']', 0};
  if (n) {
    CK(cudaMemcpyAsync(T.out, open_close, 1, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(T.out + 1 + total, open_close + 1, 2, cudaMemcpyHostToDevice, st));
    const uint32_t g = std::min<uint32_t>((n + kTlTile - 1) / kTlTile, (uint32_t)ctx->sm_count * HG_TL_WRITE_MINB);
    // staging: 1/16 above the tile's average bytes (about 4 standard deviations of a 128-object
    // tile), 16-byte granular; the kernel's 8 CTAs per SM fit while objects average below ~165 bytes
    const uint64_t avg_tile = (total + n - 1) / n * kTlTile;
    T.stage_cap = (uint32_t)std::min<uint64_t>(((avg_tile + avg_tile / 16) + 15) & ~15ull, 160u * 1024u);
    const size_t smem = tl_write_smem(T.stage_cap);
    CK(cudaFuncSetAttribute(tl_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    tl_write_kernel<<<g, kTlThreads, smem, st>>>(T);
    CK(cudaGetLastError());
    ctx->launches++;
  } else {
    static const char empty[2] = {'[', ']'};
    CK(cudaMemcpyAsync(T.out, empty, 2, cudaMemcpyHostToDevice, st));
  }
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  cudaEventElapsedTime(&ctx->tl_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->tl_ready = true;
  return HG_OK;
}

