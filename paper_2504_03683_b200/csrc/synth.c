/*
 * synth.c -- deterministic synthetic trace-stream generator (bench/test input).
 *
 * Emits one stream file in the reference's byte format
 * (/root/reference/pkg/docs/trace-format.md; encoder tracefile.py:106-145,
 * file header tracefile.py:275): [u32 magic][u32 version][u64 0] then records
 * [u32 schema_id][u64 ts][u32 payload_len][payload].  The call structure
 * follows SURVEY.md §8(d): random well-nested entry/exit pairs with a push
 * probability, a depth cap, optional call layering (top-layer APIs wrapping
 * lower-layer ones), nonzero results, device-profiling records after profiled
 * calls, annotations, and optional injected orphan/mismatched exits and
 * unclosed calls.  Fixture traces generated here are decoded by the
 * reference itself in tests/golden/make_golden.py, which pins this encoder.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../include/hapigpu.h"

typedef struct synth_params {
  uint64_t seed;
  uint64_t n_events;
  uint32_t max_depth;
  uint32_t pad0;
  uint64_t gap_lo, gap_hi;
  uint64_t ts0_hi;
  double push_p, err_p, prof_p, meta_p, orphan_p, mismatch_p;
  double zipf_s;
  uint32_t n_layers;
  int32_t close_at_end;
  int32_t meta_sid;
  uint64_t dev_off_hi;       /* device span start = record ts + U[0, dev_off_hi]          */
  int64_t dev_lo, dev_hi;    /* device span duration U[dev_lo, dev_hi] (negative: end < start) */
} synth_params;

typedef struct synth_fn {
  uint32_t entry_sid, exit_sid;
  int32_t prof_sid;   /* -1: not profiled */
  uint32_t layer;
  int32_t memcpy;     /* profiling name is a memcpy(X2Y) tag */
} synth_fn;

/* xoshiro256** */
typedef struct { uint64_t s[4]; } rng_t;
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t next64(rng_t* r) {
  uint64_t* s = r->s;
  uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
  return res;
}
static void seed_rng(rng_t* r, uint64_t seed) {
  for (int i = 0; i < 4; i++) {
    seed += 0x9E3779B97F4A7C15ull;
    uint64_t z = seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    r->s[i] = z ^ (z >> 31);
  }
}
static double unif(rng_t* r) { return (next64(r) >> 11) * (1.0 / 9007199254740992.0); }
static uint64_t range(rng_t* r, uint64_t lo, uint64_t hi) { return lo + (hi > lo ? next64(r) % (hi - lo + 1) : 0); }

typedef struct {
  uint8_t* out; uint64_t cap, len, events;
  int overflow;
} sink_t;

static void put(sink_t* k, const void* p, uint64_t n) {
  if (k->len + n > k->cap) { k->overflow = 1; return; }
  memcpy(k->out + k->len, p, n); k->len += n;
}
static void put32(sink_t* k, uint32_t v) { put(k, &v, 4); }
static void put64(sink_t* k, uint64_t v) { put(k, &v, 8); }

typedef struct {
  const hg_schema* by_id; uint32_t n_ids; const uint8_t* kinds;
  const char* const* names; uint32_t n_names;
} gen_reg;

static const char* MEMCPY_TAGS[4] = {"memcpy(H2D)", "memcpy(D2H)", "memcpy(D2D)", "memcpy(H2H)"};

/* payload for one record; special values per role.  ctx: 0 entry, 1 exit, 2 profiling, 3 meta */
static void emit(sink_t* k, rng_t* r, const gen_reg* G, uint32_t sid, uint64_t ts, uint64_t result,
                 uint64_t dev_start, uint64_t dev_end, const char* dev_name, int memcpy_kind) {
  const hg_schema* s = &G->by_id[sid];
  const uint8_t* kd = G->kinds + s->kinds_offset;
  uint8_t body[8192];
  uint64_t n = 0;
  for (int i = 0; i < s->n_fields; i++) {
    uint64_t v;
    int role = -1;
    for (int q = 0; q < HG_NUM_ROLES; q++) if (s->role[q] == i) role = q;
    switch (kd[i]) {
      case HG_KIND_U64: case HG_KIND_ADDRESS: case HG_KIND_I64: case HG_KIND_F64:
        if (role == HG_ROLE_RESULT) v = result;
        else if (role == HG_ROLE_START) v = dev_start;
        else if (role == HG_ROLE_END) v = dev_end;
        else if (role == HG_ROLE_TILE || role == HG_ROLE_ENGINE) v = next64(r) & 1;
        else if (kd[i] == HG_KIND_F64) { double x = unif(r); memcpy(&v, &x, 8); }
        else if (kd[i] == HG_KIND_I64) v = range(r, 0, 9);
        else v = next64(r) & ((1ull << 40) - 1);
        memcpy(body + n, &v, 8); n += 8;
        break;
      case HG_KIND_STRING: {
        const char* str;
        char tmp[32];
        if (role == HG_ROLE_NAME) str = dev_name;
        else if (role == HG_ROLE_CMDKIND) str = memcpy_kind ? "memcpy" : "kernel";
        else if (G->n_names) str = G->names[next64(r) % G->n_names];
        else { int l = (int)range(r, 0, 16); for (int j = 0; j < l; j++) tmp[j] = (char)range(r, 'a', 'z'); tmp[l] = 0; str = tmp; }
        uint32_t l = (uint32_t)strlen(str);
        if (l > 4096) l = 4096;
        memcpy(body + n, &l, 4); n += 4; memcpy(body + n, str, l); n += l;
        break;
      }
      default: {  /* blob: 0, 8 or 32 bytes */
        static const uint32_t L[3] = {0, 8, 32};
        uint32_t l = L[next64(r) % 3];
        memcpy(body + n, &l, 4); n += 4;
        for (uint32_t j = 0; j < l; j++) body[n + j] = (uint8_t)next64(r);
        n += l;
      }
    }
  }
  put32(k, sid); put64(k, ts); put32(k, (uint32_t)n); put(k, body, n);
  k->events++;
}

/* Zipf(s) over m items via inverse CDF on a precomputed table */
static uint32_t pick(rng_t* r, const double* cdf, uint32_t m) {
  double u = unif(r) * cdf[m - 1];
  uint32_t lo = 0, hi = m - 1;
  while (lo < hi) { uint32_t mid = (lo + hi) / 2; if (cdf[mid] < u) lo = mid + 1; else hi = mid; }
  return lo;
}

#define MAXFN 8192
#define MAXDEPTH 512

int synth_stream(const synth_params* P, const hg_schema* by_id, uint32_t n_ids, const uint8_t* kinds,
                 const synth_fn* fns, uint32_t n_fns, const char* const* names, uint32_t n_names,
                 uint8_t* out, uint64_t cap, uint64_t* out_len, uint64_t* out_events) {
  if (n_fns == 0 || n_fns > MAXFN) return -1;
  gen_reg G = {by_id, n_ids, kinds, names, n_names};
  sink_t k = {out, cap, 0, 0, 0};
  rng_t r;
  seed_rng(&r, P->seed);
  uint32_t nl = P->n_layers ? P->n_layers : 1;
  /* per-layer function lists + Zipf CDFs */
  static __thread uint32_t lay_fn[8][MAXFN];
  static __thread double lay_cdf[8][MAXFN];
  uint32_t lay_n[8] = {0};
  if (nl > 8) nl = 8;
  for (uint32_t f = 0; f < n_fns; f++) {
    uint32_t L = fns[f].layer < nl ? fns[f].layer : nl - 1;
    lay_fn[L][lay_n[L]++] = f;
  }
  for (uint32_t L = 0; L < nl; L++) {
    double acc = 0;
    for (uint32_t i = 0; i < lay_n[L]; i++) { acc += P->zipf_s > 0 ? 1.0 / pow((double)(i + 1), P->zipf_s) : 1.0; lay_cdf[L][i] = acc; }
  }
  uint32_t hdr[4] = {0x54485049u, 1u, 0u, 0u};
  put(&k, hdr, 16);
  uint64_t ts = range(&r, 0, P->ts0_hi);
  uint32_t stack[MAXDEPTH];
  uint32_t depth = 0;
  uint32_t maxd = P->max_depth < MAXDEPTH ? P->max_depth : MAXDEPTH;
  while (k.events < P->n_events && !k.overflow) {
    ts += range(&r, P->gap_lo, P->gap_hi);
    double u = unif(&r);
    if (P->meta_sid >= 0 && u < P->meta_p) {
      emit(&k, &r, &G, (uint32_t)P->meta_sid, ts, 0, 0, 0, "", 0);
      continue;
    }
    if (u < P->meta_p + P->orphan_p) {  /* stray exit */
      const synth_fn* f = &fns[next64(&r) % n_fns];
      emit(&k, &r, &G, f->exit_sid, ts, 0, 0, 0, "", 0);
      continue;
    }
    uint64_t remaining = P->n_events - k.events;
    int can_push = depth < maxd && remaining > (uint64_t)depth + 2;
    int do_push = depth == 0 ? can_push : (can_push && unif(&r) < P->push_p);
    if (!can_push && depth == 0) {  /* budget exhausted: pad with annotations or stop */
      if (P->meta_sid >= 0) emit(&k, &r, &G, (uint32_t)P->meta_sid, ts, 0, 0, 0, "", 0);
      else break;
      continue;
    }
    if (do_push) {
      uint32_t L = depth < nl ? depth : nl - 1;
      while (lay_n[L] == 0 && L > 0) L--;
      uint32_t fi = lay_fn[L][pick(&r, lay_cdf[L], lay_n[L])];
      stack[depth++] = fi;
      emit(&k, &r, &G, fns[fi].entry_sid, ts, 0, 0, 0, "", 0);
    } else {
      uint32_t fi = stack[depth - 1];
      if (P->mismatch_p > 0 && unif(&r) < P->mismatch_p) {  /* typed mismatch: orphan, no pop */
        uint32_t other = (fi + 1 + (uint32_t)(next64(&r) % (n_fns > 1 ? n_fns - 1 : 1))) % n_fns;
        emit(&k, &r, &G, fns[other].exit_sid, ts, 0, 0, 0, "", 0);
        continue;
      }
      depth--;
      uint64_t res = unif(&r) < P->err_p ? 3 : 0;
      emit(&k, &r, &G, fns[fi].exit_sid, ts, res, 0, 0, "", 0);
      if (fns[fi].prof_sid >= 0 && unif(&r) < P->prof_p && k.events < P->n_events) {
        ts += range(&r, P->gap_lo, P->gap_hi);
        uint64_t st = ts + range(&r, 0, P->dev_off_hi);
        int64_t dur = P->dev_lo + (int64_t)range(&r, 0, (uint64_t)(P->dev_hi - P->dev_lo));
        uint64_t en = st + (uint64_t)dur;
        const char* nm;
        int mc = fns[fi].memcpy;
        if (mc) nm = MEMCPY_TAGS[next64(&r) & 3];
        else nm = n_names ? names[next64(&r) % n_names] : "kernel";
        emit(&k, &r, &G, (uint32_t)fns[fi].prof_sid, ts, 0, st, en, nm, mc);
      }
    }
  }
  while (P->close_at_end && depth && !k.overflow) {
    ts += range(&r, P->gap_lo, P->gap_hi);
    uint32_t fi = stack[--depth];
    emit(&k, &r, &G, fns[fi].exit_sid, ts, unif(&r) < P->err_p ? 3 : 0, 0, 0, "", 0);
  }
  *out_len = k.len;
  *out_events = k.events;
  return k.overflow ? -2 : 0;
}

/* Telemetry sampler stream (sampler.py:98-128 shape): the 9 counters every
 * period_ns from start to until inclusive.  tel_sids in TELEMETRY_COUNTERS order. */
int synth_sampler(const uint32_t* tel_sids, uint64_t device, uint64_t start, uint64_t period, uint64_t until,
                  uint64_t seed, uint8_t* out, uint64_t cap, uint64_t* out_len, uint64_t* out_events) {
  sink_t k = {out, cap, 0, 0, 0};
  rng_t r;
  seed_rng(&r, seed);
  uint32_t hdr[4] = {0x54485049u, 1u, 0u, 0u};
  put(&k, hdr, 16);
  for (uint64_t t = start; t <= until && !k.overflow; t += period) {
    double util[4];
    for (int i = 0; i < 4; i++) util[i] = (next64(&r) & 1) ? 1.0 : 0.0;
    double tile0 = 25.0 + 90.0 * util[0] + 35.0 * util[2], tile1 = 25.0 + 90.0 * util[1] + 35.0 * util[3];
    double vals[9] = {tile0 + tile1 + 45.0, tile0, tile1, 1600.0, 1600.0, util[0], util[1], util[2], util[3]};
    for (int c = 0; c < 9; c++) {
      uint64_t vb; memcpy(&vb, &vals[c], 8);
      put32(&k, tel_sids[c]); put64(&k, t); put32(&k, 16); put64(&k, device); put64(&k, vb);
      k.events++;
    }
  }
  *out_len = k.len;
  *out_events = k.events;
  return k.overflow ? -2 : 0;
}

/* timestamp of the last record of an encoded stream (header walk), 0 if none */
uint64_t synth_last_ts(const uint8_t* data, uint64_t len) {
  uint64_t off = 16, last = 0;
  while (off + 16 <= len) {
    uint64_t ts;
    uint32_t plen;
    memcpy(&ts, data + off + 4, 8);
    memcpy(&plen, data + off + 12, 4);
    last = ts;
    off += 16 + (uint64_t)plen;
  }
  return last;
}
