/*
 * ztrc_writer.c -- native implementation of the reference's C writer binding (include/ztrc_writer.h;
 * reference declarations pkg/cinterpose/src/writer_binding.h:14-19, contract
 * pkg/docs/writer-binding.md:10-45, behaviour of the Python writer tracefile.py:222-441).
 *
 * Producer side of the pipeline the GPU engine analyses: every emitting thread owns a stream with
 * a single-producer / single-consumer ring of `buffer_capacity` record slots.  ztrc_emit encodes
 * the 16-byte record header in front of the caller's payload and enqueues without blocking; a full
 * ring drops the NEWEST record and counts it (_Ring.push / _Stream.emit_bytes, tracefile.py:231-266).
 * One drainer thread moves ring contents to the stream files every 2 ms (TraceWriter._drain_loop,
 * tracefile.py:394-397); a stream file is created with its 16-byte header on the first non-empty
 * flush (_Stream.flush_to_file, tracefile.py:268-275).  ztrc_close stops the drainer, flushes,
 * writes streams.json (TraceWriter.finalize, tracefile.py:405-441) and flips metadata.json's
 * "complete" flag.
 */
#define _GNU_SOURCE
#include "../../include/ztrc_writer.h"

#include <dirent.h>
#include <errno.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <time.h>
#include <unistd.h>

#define ZTRC_MAGIC 0x54485049u
#define ZTRC_VERSION 1u
#define ZTRC_INLINE 56u /* record bytes kept inside a slot; longer records live on the heap */

typedef struct {
  uint32_t len;
  uint8_t* heap;
  uint8_t inl[ZTRC_INLINE];
} slot_t;

struct ztrc_stream {
  int64_t pid, tid;
  uint64_t gen;                    /* open generation the stream belongs to */
  slot_t* slots;
  uint64_t cap;
  _Atomic uint64_t head, tail;     /* consumer / producer positions (records) */
  uint64_t enqueued, dropped;      /* producer-side counters (read after quiescence) */
  FILE* fh;
  char path[4096];
};

static struct {
  pthread_mutex_t lock;            /* guards the stream list and the open state */
  int open;
  uint64_t gen;
  char dir[3072];
  char host[256];
  uint64_t cap;
  ztrc_stream_t** streams;
  size_t n, alloc;
  pthread_t drainer;
  _Atomic int stop, paused;
} W = {PTHREAD_MUTEX_INITIALIZER, 0, 0, "", "", 0, NULL, 0, 0, 0, 0, 0};

static __thread ztrc_stream_t* tls_stream;
static __thread uint64_t tls_gen;
/* streams of closed traces: kept until the next ztrc_open so that a stale handle is refused
 * (its generation differs) instead of touching freed memory */
static ztrc_stream_t** G_old;
static size_t G_n;

uint64_t ztrc_clock_ns(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (uint64_t)t.tv_sec * 1000000000ull + (uint64_t)t.tv_nsec;
}

/* ------------------------------------------------------------------ drain */

static int flush_stream(ztrc_stream_t* s) {
  const uint64_t tail = atomic_load_explicit(&s->tail, memory_order_acquire);
  uint64_t head = atomic_load_explicit(&s->head, memory_order_relaxed);
  if (head == tail) return 0;
  if (!s->fh) {
    s->fh = fopen(s->path, "wb");
    if (!s->fh) return -1;
    const uint32_t hdr[4] = {ZTRC_MAGIC, ZTRC_VERSION, 0u, 0u};
    if (fwrite(hdr, 1, 16, s->fh) != 16) return -1;
  }
  int rc = 0;
  for (; head < tail; head++) {
    slot_t* sl = &s->slots[head % s->cap];
    const uint8_t* p = sl->heap ? sl->heap : sl->inl;
    if (fwrite(p, 1, sl->len, s->fh) != sl->len) rc = -1;
    free(sl->heap);
    sl->heap = NULL;
  }
  atomic_store_explicit(&s->head, head, memory_order_release);
  return rc;
}

static int drain_all(void) {
  int rc = 0;
  pthread_mutex_lock(&W.lock);
  for (size_t i = 0; i < W.n; i++)
    if (flush_stream(W.streams[i])) rc = -1;
  pthread_mutex_unlock(&W.lock);
  return rc;
}

static void* drain_loop(void* arg) {
  (void)arg;
  const struct timespec nap = {0, 2000000};
  while (!atomic_load(&W.stop)) {
    if (!atomic_load(&W.paused)) drain_all();
    nanosleep(&nap, NULL);
  }
  return NULL;
}

void ztrc_debug_pause_drainer(int paused) { atomic_store(&W.paused, paused ? 1 : 0); }
void ztrc_debug_drain(void) { drain_all(); }

/* ------------------------------------------------------------------ open / acquire / emit */

static int copy_file(const char* from, const char* to, char** text_out) {
  FILE* f = fopen(from, "rb");
  if (!f) return -1;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = malloc((size_t)n + 1);
  if (!buf || fread(buf, 1, (size_t)n, f) != (size_t)n) { fclose(f); free(buf); return -1; }
  fclose(f);
  buf[n] = 0;
  FILE* g = fopen(to, "wb");
  if (!g || fwrite(buf, 1, (size_t)n, g) != (size_t)n) { if (g) fclose(g); free(buf); return -1; }
  fclose(g);
  *text_out = buf;
  return 0;
}

static int dir_usable(const char* dir) {
  struct stat st;
  if (stat(dir, &st) != 0) return mkdir(dir, 0777) == 0 ? 0 : -1;  /* parents must exist */
  if (!S_ISDIR(st.st_mode)) return -1;
  DIR* d = opendir(dir);
  if (!d) return -1;
  struct dirent* e;
  int empty = 1;
  while ((e = readdir(d)))
    if (strcmp(e->d_name, ".") && strcmp(e->d_name, "..")) empty = 0;
  closedir(d);
  return empty ? 0 : -1;  /* TraceWriter refuses a non-empty directory (tracefile.py:309-312) */
}

int ztrc_open(const char* dir, const char* metadata_path, uint64_t buffer_capacity) {
  if (!dir || !metadata_path || buffer_capacity < 1) return -1;
  pthread_mutex_lock(&W.lock);
  if (W.open || strlen(dir) > 3000 || dir_usable(dir)) { pthread_mutex_unlock(&W.lock); return -1; }
  char dst[4096];
  snprintf(dst, sizeof dst, "%s/metadata.json", dir);
  char* text = NULL;
  if (copy_file(metadata_path, dst, &text)) { pthread_mutex_unlock(&W.lock); return -1; }
  const int incomplete = strstr(text, "\"complete\": false") != NULL;
  free(text);
  if (!incomplete) { unlink(dst); pthread_mutex_unlock(&W.lock); return -1; }
  for (size_t i = 0; i < G_n; i++) {
    free(G_old[i]->slots);
    free(G_old[i]);
  }
  G_n = 0;
  snprintf(W.dir, sizeof W.dir, "%s", dir);
  if (gethostname(W.host, sizeof W.host - 1)) snprintf(W.host, sizeof W.host, "localhost");
  W.cap = buffer_capacity;
  W.gen++;
  W.n = 0;
  atomic_store(&W.stop, 0);
  atomic_store(&W.paused, 0);
  if (pthread_create(&W.drainer, NULL, drain_loop, NULL)) { pthread_mutex_unlock(&W.lock); return -1; }
  W.open = 1;
  pthread_mutex_unlock(&W.lock);
  return 0;
}

ztrc_stream_t* ztrc_stream_acquire(void) {
  ztrc_stream_t* s = tls_stream;
  if (s && tls_gen == W.gen && W.open) return s;
  pthread_mutex_lock(&W.lock);
  if (!W.open) { pthread_mutex_unlock(&W.lock); return NULL; }
  s = calloc(1, sizeof *s);
  if (s) s->slots = calloc(W.cap, sizeof(slot_t));
  if (!s || !s->slots) { free(s); pthread_mutex_unlock(&W.lock); return NULL; }
  s->pid = (int64_t)getpid();
  s->tid = (int64_t)syscall(SYS_gettid);
  s->gen = W.gen;
  s->cap = W.cap;
  snprintf(s->path, sizeof s->path, "%s/stream_%lld_%lld.bin", W.dir, (long long)s->pid, (long long)s->tid);
  if (W.n == W.alloc) {
    W.alloc = W.alloc ? 2 * W.alloc : 16;
    W.streams = realloc(W.streams, W.alloc * sizeof *W.streams);
  }
  W.streams[W.n++] = s;
  tls_stream = s;
  tls_gen = W.gen;
  pthread_mutex_unlock(&W.lock);
  return s;
}

int ztrc_emit(ztrc_stream_t* s, uint32_t schema_id, uint64_t timestamp_ns, const uint8_t* payload,
              uint32_t payload_len) {
  if (!s || !W.open || s->gen != W.gen) return -1;
  const uint64_t tail = atomic_load_explicit(&s->tail, memory_order_relaxed);
  if (tail - atomic_load_explicit(&s->head, memory_order_acquire) >= s->cap) {
    s->dropped++;
    return 1;
  }
  slot_t* sl = &s->slots[tail % s->cap];
  const uint32_t len = 16u + payload_len;
  uint8_t* p = sl->inl;
  if (len > ZTRC_INLINE) {
    p = malloc(len);
    if (!p) { s->dropped++; return 1; }
  }
  memcpy(p, &schema_id, 4);
  memcpy(p + 4, &timestamp_ns, 8);
  memcpy(p + 12, &payload_len, 4);
  if (payload_len) memcpy(p + 16, payload, payload_len);
  sl->len = len;
  sl->heap = len > ZTRC_INLINE ? p : NULL;
  atomic_store_explicit(&s->tail, tail + 1, memory_order_release);
  s->enqueued++;
  return 0;
}

/* ------------------------------------------------------------------ close */

/* json.dumps(str) with ensure_ascii (json/encoder.py) of a UTF-8 hostname */
static void json_str(FILE* f, const char* s) {
  fputc('"', f);
  const unsigned char* p = (const unsigned char*)s;
  while (*p) {
    uint32_t c = *p, cp;
    int n = 1;
    if (c < 0x80) cp = c;
    else if (c < 0xE0) { cp = ((c & 0x1F) << 6) | (p[1] & 0x3F); n = 2; }
    else if (c < 0xF0) { cp = ((c & 0x0F) << 12) | ((p[1] & 0x3F) << 6) | (p[2] & 0x3F); n = 3; }
    else { cp = ((c & 0x07) << 18) | ((p[1] & 0x3F) << 12) | ((p[2] & 0x3F) << 6) | (p[3] & 0x3F); n = 4; }
    p += n;
    if (cp == '"') fputs("\\\"", f);
    else if (cp == '\\') fputs("\\\\", f);
    else if (cp == '\n') fputs("\\n", f);
    else if (cp == '\r') fputs("\\r", f);
    else if (cp == '\t') fputs("\\t", f);
    else if (cp == '\b') fputs("\\b", f);
    else if (cp == '\f') fputs("\\f", f);
    else if (cp >= 0x20 && cp < 0x7F) fputc((int)cp, f);
    else if (cp < 0x10000) fprintf(f, "\\u%04x", cp);
    else { cp -= 0x10000; fprintf(f, "\\u%04x\\u%04x", 0xD800 | (cp >> 10), 0xDC00 | (cp & 0x3FF)); }
  }
  fputc('"', f);
}

static int cmp_stream(const void* a, const void* b) {
  const ztrc_stream_t* x = *(ztrc_stream_t* const*)a;
  const ztrc_stream_t* y = *(ztrc_stream_t* const*)b;
  if (x->pid != y->pid) return x->pid < y->pid ? -1 : 1;
  return x->tid < y->tid ? -1 : (x->tid > y->tid);
}

static int flip_complete(void) {
  char path[4096 + 32];
  snprintf(path, sizeof path, "%s/metadata.json", W.dir);
  FILE* f = fopen(path, "rb");
  if (!f) return -1;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = malloc((size_t)n + 2);
  if (!buf || fread(buf, 1, (size_t)n, f) != (size_t)n) { fclose(f); free(buf); return -1; }
  fclose(f);
  buf[n] = 0;
  char* at = strstr(buf, "\"complete\": false");
  if (!at) { free(buf); return -1; }
  FILE* g = fopen(path, "wb");
  if (!g) { free(buf); return -1; }
  const size_t pre = (size_t)(at - buf), key = strlen("\"complete\": false");
  int rc = fwrite(buf, 1, pre, g) == pre && fputs("\"complete\": true", g) >= 0 &&
                   fwrite(at + key, 1, (size_t)n - pre - key, g) == (size_t)n - pre - key ? 0 : -1;
  if (fclose(g)) rc = -1;
  free(buf);
  return rc;
}

int ztrc_close(void) {
  pthread_mutex_lock(&W.lock);
  if (!W.open) { pthread_mutex_unlock(&W.lock); return -1; }
  W.open = 0;
  pthread_mutex_unlock(&W.lock);
  atomic_store(&W.stop, 1);
  pthread_join(W.drainer, NULL);
  int rc = drain_all();
  pthread_mutex_lock(&W.lock);
  qsort(W.streams, W.n, sizeof *W.streams, cmp_stream);  /* one host: (hostname, pid, tid) = (pid, tid) */
  char path[4096 + 32];
  snprintf(path, sizeof path, "%s/streams.json", W.dir);
  FILE* f = fopen(path, "wb");
  if (!f) rc = -1;
  size_t listed = 0;
  if (f) fputs("{\n \"streams\": [", f);
  for (size_t i = 0; i < W.n; i++) {
    ztrc_stream_t* s = W.streams[i];
    if (s->fh && fclose(s->fh)) rc = -1;
    s->fh = NULL;
    if (f && (s->enqueued || s->dropped)) {  /* acquired-but-silent streams are not listed */
      fputs(listed ? ",\n  {\n   \"hostname\": " : "\n  {\n   \"hostname\": ", f);
      json_str(f, W.host);
      fprintf(f, ",\n   \"pid\": %lld,\n   \"tid\": %lld,\n   \"event_count\": %llu,\n   \"dropped_count\": %llu,\n"
                 "   \"file\": \"stream_%lld_%lld.bin\"\n  }",
              (long long)s->pid, (long long)s->tid, (unsigned long long)s->enqueued, (unsigned long long)s->dropped,
              (long long)s->pid, (long long)s->tid);
      listed++;
    }
  }
  if (f) {
    fputs(listed ? "\n ]\n}" : "]\n}", f);
    if (fclose(f)) rc = -1;
  }
  if (!rc) rc = flip_complete();  /* on failure the trace stays marked incomplete */
  G_old = realloc(G_old, (G_n + W.n) * sizeof *G_old);
  for (size_t i = 0; i < W.n; i++) G_old[G_n++] = W.streams[i];
  W.n = 0;
  pthread_mutex_unlock(&W.lock);
  return rc;
}
