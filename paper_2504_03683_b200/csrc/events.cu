// events.cu -- event sinks on the GPU: the muxer as an event-order service
// and PrettyPrintSink's text.
//
// Reference: mux_streams (pipeline.py:68-114) hands every record of every stream to the
// `consumes = "events"` sinks in heap order (ts, hostname, pid, tid, seq, stream); PrettyPrintSink
// (sinks.py:66-106) renders each as
//   HH:MM:SS.nnnnnnnnn - <hostname> - vpid: P, vtid: T - <schema>: { f: v, ... }
// with fmt_timestamp (sinks.py:43-46) and _fmt_value (sinks.py:49-59): addresses 0x%016x, strings
// json.dumps (ensure_ascii), blobs "[ b0, b1 ]", f64 repr(float), integers str().
//
// Pipeline (after an exact-path phase 1 whose SegInfo holds every verified segment start):
//   ev_index_kernel   one lane per segment walks its records: (ts, stream << 40 | seq, offset, sid)
//                     into the record region (stream s from rec_off[s]) -- every stream a sorted run
//   tl_sort           the timeline's k-way merge of the runs (timeline.cu): the mux order, since
//                     streams are indexed in (hostname, pid, tid) order and identities are distinct
//   ev_line<TC>       exact byte length of every line; tl_scan -> offsets
//   ev_line<TW>       each line written at its offset
#define HG_EV_KERNELS
#include "ctx.h"

namespace {

struct EvTables {
  const TlItem* items;
  const uint32_t* order;
  uint32_t n;
  const uint8_t* data;
  const int32_t* sid_map;
  const DSchema* schemas;
  const uint8_t* kinds;
  const char* spre;  const uint64_t* spre_off;   // per stream: " - host - vpid: P, vtid: T - "
  const char* sname; const uint64_t* sname_off;  // per schema (index): "name: "
  const char* fname; const uint64_t* fname_off;  // per field (kinds index): "name: "
  uint32_t* lens;
  const uint64_t* offs;
  char* out;
  uint32_t stage_cap;  // ev_write_kernel: staging bytes per tile
};

__global__ void __launch_bounds__(256) ev_index_kernel(const SegInfo* info, const uint32_t* tile_stream, uint32_t n_tiles,
                                                       const uint8_t* data, const uint64_t* stream_base,
                                                       const unsigned long long* rec_off, TlItem* items) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_tiles; g += gridDim.x * blockDim.x) {
    const SegInfo I = info[g];
    if ((I.flags & SI_DEAD) || !I.n) continue;
    const uint32_t s = tile_stream[g];
    const uint8_t* gb = data + stream_base[s];
    uint64_t o = I.entry;
    const uint64_t slot0 = rec_off[s] + I.base;
    for (uint32_t k = 0; k < I.n; k++) {
      const uint32_t sid = ldu32(gb + o);
      const uint64_t ts = ldu64(gb + o + 4);
      const uint32_t plen = ldu32(gb + o + 12);
      TlItem it;
      it.khi = ts; it.klo = tl_klo(s, I.base + k); it.a = stream_base[s] + o; it.b = 0; it.kind = 0; it.x = sid;
      items[slot0 + k] = it;
      o += 16ull + plen;
    }
  }
}

template <class W>
__device__ __forceinline__ void w_dec(W& w, uint64_t v) {
  if constexpr (W::kWrite) w.n += nf::fmt_u64(v, w.at());
  else w.s(nullptr, ndig(v));
}

template <class W>
__device__ __forceinline__ void w_2(W& w, uint32_t v) { w.c((char)('0' + v / 10)); w.c((char)('0' + v % 10)); }

// fmt_timestamp (sinks.py:43-46): HH:MM:SS.nnnnnnnnn of ns modulo one day
template <class W>
__device__ __forceinline__ void w_ts(W& w, uint64_t ns) {
  if constexpr (!W::kWrite) {
    w.s(nullptr, 18);
  } else {
    const uint64_t sec = ns / 1000000000ull;
    uint32_t frac = (uint32_t)(ns - sec * 1000000000ull);
    const uint32_t d = (uint32_t)(sec % 86400ull);
    w_2(w, d / 3600); w.c(':'); w_2(w, d % 3600 / 60); w.c(':'); w_2(w, d % 60); w.c('.');
    char* q = w.at();
    for (int i = 8; i >= 0; i--) { q[i] = (char)('0' + frac % 10); frac /= 10; }
    w.n += 9;
  }
}

// repr(float(value)) (sinks.py:57-58): nan / inf spelled as Python does
template <class W>
__device__ __forceinline__ void w_repr(W& w, uint64_t bits) {
  const uint64_t mag = bits & 0x7FFFFFFFFFFFFFFFull;
  if (mag > 0x7FF0000000000000ull) { w.lit("nan"); return; }
  if (mag == 0x7FF0000000000000ull) {
    if (bits >> 63) w.lit("-inf");
    else w.lit("inf");
    return;
  }
  char b[40];
  const int k = nf::fmt_double(__longlong_as_double((long long)bits), b);
  w.s(b, (uint32_t)k);
}

template <class W>
__device__ void ev_line(const EvTables& T, const TlItem& it, W& w) {
  const uint32_t s = (uint32_t)(it.klo >> 40);
  const int32_t si = T.sid_map[it.x];
  const DSchema& sc = T.schemas[si];
  w_ts(w, it.khi);
  w.s(T.spre + T.spre_off[s], (uint32_t)(T.spre_off[s + 1] - T.spre_off[s]));
  w.s(T.sname + T.sname_off[si], (uint32_t)(T.sname_off[si + 1] - T.sname_off[si]));
  if (!sc.nfields) {
    w.lit("{ }");
  } else {
    w.lit("{ ");
    const uint8_t* q = T.data + it.a + 16;
    for (uint32_t f = 0; f < sc.nfields; f++) {
      const uint32_t k = sc.kinds_off + f;
      if (f) w.lit(", ");
      w.s(T.fname + T.fname_off[k], (uint32_t)(T.fname_off[k + 1] - T.fname_off[k]));
      const uint8_t kind = T.kinds[k];
      if (kind == HG_KIND_STRING || kind == HG_KIND_BLOB) {
        const uint32_t len = ldu32(q);
        if (kind == HG_KIND_STRING) {
          json_str(w, q + 4, len);
        } else {  // "[ " + ", ".join(str(b)) + " ]": four bytes per load, a byte's digits by compares
          w.lit("[ ");
          for (uint32_t j = 0; j < len; j += 4) {
            const uint32_t word = ldu32(q + 4 + j);  // (the data array is padded past its last byte)
            const uint32_t m = len - j < 4u ? len - j : 4u;
            for (uint32_t k = 0; k < m; k++) {
              if (j + k) w.lit(", ");
              const uint32_t b = (word >> (8u * k)) & 255u;
              if constexpr (W::kWrite) {
                if (b >= 100u) w.c((char)('0' + b / 100u));
                if (b >= 10u) w.c((char)('0' + b / 10u % 10u));
                w.c((char)('0' + b % 10u));
              } else {
                w.s(nullptr, b >= 100u ? 3u : b >= 10u ? 2u : 1u);
              }
            }
          }
          w.lit(" ]");
        }
        q += 4 + len;
        continue;
      }
      const uint64_t v = ldu64(q);
      q += 8;
      if (kind == HG_KIND_U64) {
        w_dec(w, v);
      } else if (kind == HG_KIND_I64) {
        if ((int64_t)v < 0) { w.c('-'); w_dec(w, 0 - v); }
        else w_dec(w, v);
      } else if (kind == HG_KIND_ADDRESS) {  // f"0x{value:016x}"
        if constexpr (W::kWrite) {
          const char* hx = "0123456789abcdef";
          w.c('0'); w.c('x');
          char* d = w.at();
          for (int j = 15; j >= 0; j--) d[15 - j] = hx[(v >> (4 * j)) & 15];
          w.n += 16;
        } else {
          w.s(nullptr, 18);
        }
      } else {  // f64
        w_repr(w, v);
      }
    }
    w.lit(" }");
  }
  w.c('\n');
}

// Lines are formatted in CTA tiles of kEvTile consecutive mux positions, handed to the threads in
// schema order (a bitonic sort of (schema id, position) keys in shared memory): the lines of a
// schema run the same field loop, so a warp's lanes stay together (7 of 32 active otherwise).
constexpr uint32_t kEvTile = 128;

struct EvTile {
  TlItem it[kEvTile];
  uint32_t key[kEvTile];  // schema id << 7 | tile position, ~0 past the end
};

// gathers the tile's items (thread t: position t) and sorts the keys; returns this thread's position or ~0
__device__ __forceinline__ uint32_t ev_tile_sort(const EvTables& T, uint64_t i0, EvTile& S) {
  const uint32_t t = threadIdx.x;
  uint32_t key = 0xFFFFFFFFu;
  if (i0 + t < T.n) {
    const TlItem it = T.items[T.order[i0 + t]];
    S.it[t] = it;
    key = (it.x << 7) | t;
  }
  S.key[t] = key;
  __syncthreads();
  for (uint32_t k = 2; k <= kEvTile; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t u = t ^ j;
      if (u > t) {
        const uint32_t a = S.key[t], b = S.key[u];
        if ((a > b) == ((t & k) == 0)) { S.key[t] = b; S.key[u] = a; }
      }
      __syncthreads();
    }
  }
  const uint32_t q = S.key[t];
  return q == 0xFFFFFFFFu ? q : (q & (kEvTile - 1));
}

__global__ void __launch_bounds__(kEvTile, 8) ev_len_kernel(EvTables T) {
  __shared__ EvTile S;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kEvTile; i0 < T.n; i0 += (uint64_t)gridDim.x * kEvTile) {
    const uint32_t j = ev_tile_sort(T, i0, S);
    if (j != 0xFFFFFFFFu) {
      TC c{0};
      ev_line(T, S.it[j], c);
      T.lens[i0 + j] = (uint32_t)c.n;
    }
    __syncthreads();
  }
}

// a CTA formats its tile's lines into a shared staging buffer at their offsets and stores the
// tile's byte window with aligned 16-byte writes (tiles beyond the buffer write straight to HBM)
struct EvWriteSmem {
  EvTile g;
  uint64_t off[kEvTile];
  uint64_t o0, oend;
  __align__(16) char stage[16];  // stage_cap + 16 bytes (dynamic shared memory)
};

__global__ void __launch_bounds__(kEvTile, 8) ev_write_kernel(EvTables T) {
  extern __shared__ __align__(16) char ev_smem[];
  EvWriteSmem& S = *reinterpret_cast<EvWriteSmem*>(ev_smem);
  const uint32_t t = threadIdx.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kEvTile; i0 < T.n; i0 += (uint64_t)gridDim.x * kEvTile) {
    const uint64_t i = i0 + t, last = min((uint64_t)T.n, i0 + kEvTile) - 1;
    if (i <= last) {
      const uint64_t off = T.offs[i];
      S.off[t] = off;
      if (i == i0) S.o0 = off;
      if (i == last) S.oend = off + T.lens[i];
    }
    const uint32_t j = ev_tile_sort(T, i0, S.g);  // (its barriers publish off / o0 / oend)
    const uint64_t al = S.o0 & ~15ull, total = S.oend - al;
    const bool staged = total <= (uint64_t)T.stage_cap;
    if (j != 0xFFFFFFFFu) {
      const uint64_t off = S.off[j];
      TW w{staged ? S.stage + (off - al) : T.out + off, 0};
      ev_line(T, S.g.it[j], w);
    }
    __syncthreads();
    if (staged) {  // bytes [head, end) of the 16-byte aligned window at al
      char* gout = T.out + al;
      const uint32_t head = (uint32_t)(S.o0 - al), end = (uint32_t)total;
      const uint32_t full_end = end & ~15u;
      for (uint32_t b0 = 16u * t + (head ? 16u : 0u); b0 < full_end; b0 += 16u * kEvTile)
        *reinterpret_cast<uint4*>(gout + b0) = *reinterpret_cast<const uint4*>(S.stage + b0);
      if (t < 16) {  // the partial first and last chunks, a byte per thread
        if (head && head + t < 16u && head + t < end) gout[head + t] = S.stage[head + t];
        const uint32_t b = full_end + t;
        if (b < end && (b >= 16u || !head)) gout[b] = S.stage[b];
      }
    }
    __syncthreads();
  }
}

// (stream, record index) of every event in mux order
__global__ void ev_order_kernel(const TlItem* items, const uint32_t* order, uint32_t n, uint32_t* stream,
                                unsigned long long* seq) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t klo = items[order[i]].klo;
    stream[i] = (uint32_t)(klo >> 40);
    seq[i] = klo & ((1ull << 40) - 1);
  }
}

static std::string py_str_int(bool none, int64_t v) { return none ? std::string("None") : std::to_string(v); }

}  // namespace

// after hg_finish: order every record by the muxer's key and render PrettyPrintSink's lines
int run_events(hg_ctx* ctx) {
  ctx->ev_ready = false;
  if (ctx->last_path != 0 && !ctx->ev_ranges) return fail(ctx, HG_ESTATE, "event sinks: no record lists of the run");
  if (!ctx->have_schema_names) return fail(ctx, HG_ESTATE, "hg_set_schema_names is required for event sinks");
  cudaStream_t st = ctx->stream;
  const uint32_t ns = (uint32_t)ctx->streams.size();
  const uint64_t total = ctx->counters[C_STATS + ST_EVENTS];
  if (total >= (1ull << 32)) return fail(ctx, HG_EUNSUPPORTED, "event sinks: more than 2^32 records");
  const uint32_t n = (uint32_t)total;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  const uint32_t* order = nullptr;
  if (ctx->last_path == 1) {  // the single pass's per-range record lists: keys, then the merge passes
    TlSource S;
    S.ranges = true;
    S.items = ctx->d_ev_items.ptr;
    S.n_ranges = ctx->n_ranges;
    S.rcap = ctx->tl_rcap;
    S.rn = ctx->d_ev_rn.ptr;
    S.range_stream = ctx->d_range_stream.ptr;
    S.range_base = ctx->d_range_base.ptr;
    S.stream_range0 = ctx->d_stream_range0.ptr;
    S.nrec_slots = ctx->n_ranges * ctx->tl_rcap;
    S.n_runs = ns;
    uint32_t n2 = 0;
    int rc = tl_sort_ranges(ctx, S, &n2, &order);
    if (rc) return rc;
    if (n2 != n) return fail(ctx, HG_ECUDA, "event sinks: record lists do not cover the run (engine bug)");
  }
  if (ctx->last_path == 0) CK(ctx->d_ev_items.ensure(std::max<uint32_t>(n, 1)));
  const uint32_t nt = ctx->last_path == 0 ? (uint32_t)ctx->tile_stream.size() : 0u;
  if (nt) {
    ev_index_kernel<<<std::min<uint32_t>((nt + 255) / 256, (uint32_t)ctx->sm_count * 8), 256, 0, st>>>(
        ctx->d_seginfo.ptr, ctx->d_tile_stream.ptr, nt, ctx->d_data.ptr, ctx->d_base.ptr, ctx->d_tl_rec_off.ptr,
        ctx->d_ev_items.ptr);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  int rc = HG_OK;
  if (ctx->last_path == 0) {
    rc = tl_sort(ctx, ctx->d_ev_items.ptr, n, n, 0, n, &order);
    if (rc) return rc;
  }
  // host tables
  std::vector<char> spre, sname;
  std::vector<uint64_t> spre_off(1, 0), sname_off(1, 0);
  for (uint32_t s = 0; s < ns; s++) {
    const HostStream& hs = ctx->streams[s];
    std::string x = " - " + (hs.host_none ? std::string("None") : hs.host) + " - vpid: " +
                    py_str_int(hs.pid_none, hs.pid) + ", vtid: " + py_str_int(hs.tid_none, hs.tid) + " - ";
    spre.insert(spre.end(), x.begin(), x.end());
    spre_off.push_back(spre.size());
  }
  for (const std::string& nm : ctx->schema_names) {
    std::string x = nm + ": ";
    sname.insert(sname.end(), x.begin(), x.end());
    sname_off.push_back(sname.size());
  }
  std::vector<char> fname;
  std::vector<uint64_t> fname_off(1, 0);
  for (const std::string& nm : ctx->field_names) {
    std::string x = nm + ": ";
    fname.insert(fname.end(), x.begin(), x.end());
    fname_off.push_back(fname.size());
  }
  for (std::vector<char>* v : {&spre, &sname, &fname}) v->insert(v->end(), 8, '\0');  // word-wise readers
  CK(upload(ctx->d_ev_spre, spre, st));
  CK(upload(ctx->d_ev_spre_off, spre_off, st));
  CK(upload(ctx->d_ev_sname, sname, st));
  CK(upload(ctx->d_ev_sname_off, sname_off, st));
  CK(upload(ctx->d_ev_fname, fname, st));
  CK(upload(ctx->d_ev_fname_off, fname_off, st));
  CK(ctx->d_ev_lens.ensure(std::max<uint32_t>(n, 1)));
  CK(ctx->d_ev_offs.ensure(std::max<uint32_t>(n, 1)));
  EvTables T{};
  T.items = ctx->d_ev_items.ptr;
  T.order = order;
  T.n = n;
  T.data = ctx->d_data.ptr;
  T.sid_map = ctx->d_sid_map.ptr;
  T.schemas = ctx->d_schemas.ptr;
  T.kinds = ctx->d_kinds.ptr;
  T.spre = ctx->d_ev_spre.ptr; T.spre_off = ctx->d_ev_spre_off.ptr;
  T.sname = ctx->d_ev_sname.ptr; T.sname_off = ctx->d_ev_sname_off.ptr;
  T.fname = ctx->d_ev_fname.ptr; T.fname_off = ctx->d_ev_fname_off.ptr;
  T.lens = ctx->d_ev_lens.ptr;
  T.offs = ctx->d_ev_offs.ptr;
  uint64_t bytes = 0;
  if (n) {
    const uint32_t g = std::min<uint32_t>((n + kEvTile - 1) / kEvTile, (uint32_t)ctx->sm_count * 8);
    ev_len_kernel<<<g, kEvTile, 0, st>>>(T);
    rc = tl_scan(ctx, T.lens, n, ctx->d_ev_offs.ptr, reinterpret_cast<uint64_t*>(ctx->d_counters.ptr + C_TL_TOTAL));
    if (rc) return rc;
    ctx->launches++;
    unsigned long long tot = 0;
    CK(cudaMemcpyAsync(&tot, ctx->d_counters.ptr + C_TL_TOTAL, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bytes = tot;
    CK(ctx->d_ev_out.ensure(bytes + 32));
    T.out = ctx->d_ev_out.ptr;
    // staging: 1/16 above the tile's average bytes (16-byte granular)
    const uint64_t avg_tile = (bytes + n - 1) / n * kEvTile;
    T.stage_cap = (uint32_t)std::min<uint64_t>(((avg_tile + avg_tile / 16) + 15) & ~15ull, 160u * 1024u);
    const size_t smem = sizeof(EvWriteSmem) + T.stage_cap;
    CK(cudaFuncSetAttribute(ev_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint32_t gw = std::min<uint32_t>((n + kEvTile - 1) / kEvTile, (uint32_t)ctx->sm_count * 8);
    ev_write_kernel<<<gw, kEvTile, smem, st>>>(T);
    CK(cudaGetLastError());
    ctx->launches++;
  }
  ctx->ev_size = bytes;
  ctx->ev_order = order;
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  cudaEventElapsedTime(&ctx->ev_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->ev_ready = true;
  return HG_OK;
}

extern "C" {

int hg_set_schema_names(hg_ctx* ctx, const char* names, const uint64_t* offsets, uint32_t n_schemas,
                        const char* field_names, const uint64_t* field_offsets, uint32_t n_fields) {
  if (!ctx || (n_schemas && (!names || !offsets)) || (n_fields && (!field_names || !field_offsets))) return HG_EARG;
  if (n_schemas != ctx->schemas.size() || n_fields != ctx->kinds.size())
    return fail(ctx, HG_EARG, "schema / field name counts differ from the registry");
  ctx->schema_names.clear();
  ctx->field_names.clear();
  for (uint32_t i = 0; i < n_schemas; i++) ctx->schema_names.emplace_back(names + offsets[i], offsets[i + 1] - offsets[i]);
  for (uint32_t i = 0; i < n_fields; i++)
    ctx->field_names.emplace_back(field_names + field_offsets[i], field_offsets[i + 1] - field_offsets[i]);
  ctx->have_schema_names = true;
  return HG_OK;
}

int hg_events_size(hg_ctx* ctx, uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return HG_EARG;
  if (!ctx->ev_ready) return HG_ESTATE;
  *n_bytes = ctx->ev_size;
  return HG_OK;
}

int hg_get_events(hg_ctx* ctx, char* out, uint64_t cap) {
  if (!ctx || (!out && cap)) return HG_EARG;
  if (!ctx->ev_ready) return HG_ESTATE;
  if (cap < ctx->ev_size) return fail(ctx, HG_EARG, "event text buffer too small");
  if (ctx->ev_size) CK(cudaMemcpy(out, ctx->d_ev_out.ptr, ctx->ev_size, cudaMemcpyDeviceToHost));
  return HG_OK;
}

int hg_get_event_order(hg_ctx* ctx, uint32_t* stream, uint64_t* seq, uint64_t cap, uint64_t* n) {
  if (!ctx || !n) return HG_EARG;
  if (!ctx->ev_ready) return HG_ESTATE;
  const uint64_t total = ctx->counters[C_STATS + ST_EVENTS];
  *n = total;
  if (!stream && !seq) return HG_OK;
  if (cap < total) return fail(ctx, HG_EARG, "event order buffer too small");
  if (!total) return HG_OK;
  cudaSetDevice(ctx->cfg.device);
  CK(ctx->d_ev_lens.ensure(total));  // (scratch: the line lengths are no longer needed)
  CK(ctx->d_ev_seq.ensure(total));
  ev_order_kernel<<<std::min<uint64_t>((total + 255) / 256, (uint64_t)ctx->sm_count * 8), 256, 0, ctx->stream>>>(
      ctx->d_ev_items.ptr, ctx->ev_order, (uint32_t)total, ctx->d_ev_lens.ptr, ctx->d_ev_seq.ptr);
  CK(cudaGetLastError());
  std::vector<uint32_t> s32(total);
  std::vector<unsigned long long> s64(total);
  CK(cudaMemcpyAsync(s32.data(), ctx->d_ev_lens.ptr, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(s64.data(), ctx->d_ev_seq.ptr, total * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (uint64_t i = 0; i < total; i++) {
    if (stream) stream[i] = s32[i];
    if (seq) seq[i] = s64[i];
  }
  return HG_OK;
}

int hg_events_ms(hg_ctx* ctx, float* ms) {
  if (!ctx || !ms) return HG_EARG;
  *ms = ctx->ev_ms;
  return HG_OK;
}

}  // extern "C"
