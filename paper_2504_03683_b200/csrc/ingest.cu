// ingest.cu -- stream bytes into HBM (the reference reads whole files,
// tracefile.py:489).
//
// Every stream lands at its 256-byte aligned offset of one device buffer (build_layout, engine.cu).
// Where its bytes come from decides how:
//   * pinned host memory (cudaHostAlloc / registered, e.g. a pinned torch tensor): one DMA;
//   * device memory on this GPU (a torch tensor, a GPUDirect-Storage buffer): one D2D copy, no PCIe;
//   * pageable host memory and stream FILES (hg_add_stream_file): a pipeline of host threads, each
//     owning two pinned staging buffers -- it fills one (pread of the file / memcpy of the pageable
//     bytes) while the copy engine drains the other into HBM, so disk / page-cache reads, host copies
//     and PCIe transfers overlap instead of serialising through the driver's pageable path.
// The file's 16-byte header has already been checked by the caller (tracefile.py:491-499 texts).
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <thread>

#include "ctx.h"

namespace {

constexpr uint64_t kChunk = 8ull << 20;  // bytes per staging buffer
constexpr int kMaxThreads = 8;

struct Piece {
  uint32_t s;
  uint64_t off, len;  // within the stream
};

struct Worker {
  cudaStream_t st = nullptr;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
};

}  // namespace

// pinned staging pool, created on first use and kept for the context's lifetime
struct IngestPool {
  Worker w[kMaxThreads];
  int n = 0;
};

static int pool_init(hg_ctx* ctx, int nthreads) {
  if (!ctx->ingest) ctx->ingest = new IngestPool();
  IngestPool& P = *ctx->ingest;
  for (int t = P.n; t < nthreads; t++) {
    Worker& W = P.w[t];
    CK(cudaStreamCreateWithFlags(&W.st, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
      CK(cudaHostAlloc(&W.buf[b], kChunk, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&W.ev[b], cudaEventDisableTiming));
    }
    P.n = t + 1;
  }
  return HG_OK;
}

void ingest_free(hg_ctx* ctx) {
  if (!ctx->ingest) return;
  IngestPool& P = *ctx->ingest;
  for (int t = 0; t < P.n; t++) {
    Worker& W = P.w[t];
    for (int b = 0; b < 2; b++) {
      if (W.ev[b]) cudaEventDestroy(W.ev[b]);
      if (W.buf[b]) cudaFreeHost(W.buf[b]);
    }
    if (W.st) cudaStreamDestroy(W.st);
  }
  delete ctx->ingest;
  ctx->ingest = nullptr;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// copy every stream into d_data at base[s]; blocks until the bytes are in HBM
int ingest_streams(hg_ctx* ctx) {
  const auto t0 = std::chrono::steady_clock::now();
  const uint32_t ns = (uint32_t)ctx->streams.size();
  IngestStats S{};
  std::vector<Piece> pieces;
  for (uint32_t s = 0; s < ns; s++) {
    const HostStream& hs = ctx->streams[s];
    if (!hs.size) continue;
    uint8_t* dst = ctx->d_data.ptr + ctx->base[s];
    if (hs.src == SRC_DEVICE) {
      CK(cudaMemcpyAsync(dst, hs.data, hs.size, cudaMemcpyDeviceToDevice, ctx->stream));
      S.device_bytes += hs.size;
    } else if (hs.src == SRC_HOST && is_pinned(hs.data)) {
      CK(cudaMemcpyAsync(dst, hs.data, hs.size, cudaMemcpyHostToDevice, ctx->stream));
      S.pinned_bytes += hs.size;
    } else {
      for (uint64_t o = 0; o < hs.size; o += kChunk) pieces.push_back(Piece{s, o, std::min(kChunk, hs.size - o)});
      (hs.src == SRC_FILE ? S.file_bytes : S.pageable_bytes) += hs.size;
    }
  }
  if (!pieces.empty()) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = (int)std::min<uint64_t>({(uint64_t)kMaxThreads, (uint64_t)hw, (uint64_t)pieces.size()});
    int rc = pool_init(ctx, nt);
    if (rc) return rc;
    std::atomic<size_t> next{0};
    std::atomic<int> bad{0};
    std::vector<std::string> errs(nt);
    auto work = [&](int t) {
      cudaSetDevice(ctx->cfg.device);
      Worker& W = ctx->ingest->w[t];
      int fd = -1;
      uint32_t fd_s = UINT32_MAX;
      int b = 0;
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= pieces.size() || bad.load()) break;
        const Piece& pc = pieces[i];
        const HostStream& hs = ctx->streams[pc.s];
        if (W.used[b] && cudaEventSynchronize(W.ev[b]) != cudaSuccess) { errs[t] = "staging event"; bad = 1; break; }
        uint8_t* buf = static_cast<uint8_t*>(W.buf[b]);
        if (hs.src == SRC_FILE) {
          if (fd_s != pc.s) {
            if (fd >= 0) close(fd);
            fd = open(hs.path.c_str(), O_RDONLY);
            fd_s = pc.s;
            if (fd < 0) { errs[t] = "cannot open " + hs.path; bad = 1; break; }
          }
          uint64_t got = 0;
          while (got < pc.len) {
            const ssize_t r = pread(fd, buf + got, pc.len - got, (off_t)(hs.file_off + pc.off + got));
            if (r <= 0) break;
            got += (uint64_t)r;
          }
          if (got != pc.len) { errs[t] = "short read of " + hs.path; bad = 1; break; }
        } else {
          memcpy(buf, hs.data + pc.off, pc.len);
        }
        if (cudaMemcpyAsync(ctx->d_data.ptr + ctx->base[pc.s] + pc.off, buf, pc.len, cudaMemcpyHostToDevice, W.st) !=
                cudaSuccess ||
            cudaEventRecord(W.ev[b], W.st) != cudaSuccess) {
          errs[t] = "staging copy";
          bad = 1;
          break;
        }
        W.used[b] = true;
        b ^= 1;
      }
      if (fd >= 0) close(fd);
      cudaStreamSynchronize(W.st);
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; t++) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (int t = 0; t < nt; t++) ctx->ingest->w[t].used[0] = ctx->ingest->w[t].used[1] = false;
    if (bad.load()) {
      for (auto& e : errs)
        if (!e.empty()) return fail(ctx, HG_EARG, "ingest: " + e);
      return fail(ctx, HG_ECUDA, "ingest failed");
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  S.ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  S.threads = ctx->ingest ? ctx->ingest->n : 0;
  ctx->ingest_stats = S;
  ctx->h2d_bytes = S.pinned_bytes + S.pageable_bytes + S.file_bytes;
  return HG_OK;
}

extern "C" {

int hg_add_stream_device(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid, const void* dptr, uint64_t size) {
  if (!ctx || (size && !dptr)) return HG_EARG;
  if (size) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, dptr) != cudaSuccess || a.type != cudaMemoryTypeDevice ||
        a.device != ctx->cfg.device) {
      cudaGetLastError();
      return fail(ctx, HG_EARG, "hg_add_stream_device: not device memory of this context's GPU");
    }
  }
  HostStream hs{hostname ? hostname : "", pid, tid, (const uint8_t*)dptr, size, hostname == nullptr};
  hs.pid_none = pid == INT64_MIN;
  hs.tid_none = tid == INT64_MIN;
  hs.src = SRC_DEVICE;
  ctx->streams.push_back(hs);
  ctx->staged = false;
  ctx->have_results = false;
  return HG_OK;
}

int hg_add_stream_file(hg_ctx* ctx, const char* hostname, int64_t pid, int64_t tid, const char* path, uint64_t offset,
                       uint64_t size) {
  if (!ctx || (size && !path)) return HG_EARG;
  HostStream hs{hostname ? hostname : "", pid, tid, nullptr, size, hostname == nullptr};
  hs.pid_none = pid == INT64_MIN;
  hs.tid_none = tid == INT64_MIN;
  hs.src = SRC_FILE;
  hs.path = path ? path : "";
  hs.file_off = offset;
  ctx->streams.push_back(hs);
  ctx->staged = false;
  ctx->have_results = false;
  return HG_OK;
}

int hg_ingest_stats(hg_ctx* ctx, uint64_t* pinned, uint64_t* pageable, uint64_t* file, uint64_t* device, float* ms,
                    uint32_t* threads) {
  if (!ctx) return HG_EARG;
  const IngestStats& S = ctx->ingest_stats;
  if (pinned) *pinned = S.pinned_bytes;
  if (pageable) *pageable = S.pageable_bytes;
  if (file) *file = S.file_bytes;
  if (device) *device = S.device_bytes;
  if (ms) *ms = S.ms;
  if (threads) *threads = (uint32_t)S.threads;
  return HG_OK;
}

}  // extern "C"
