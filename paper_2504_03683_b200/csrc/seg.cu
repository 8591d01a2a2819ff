// seg.cu -- the exact three-kernel phase 1 (seg.cuh): segment walk, chain, decode
#define HG_SEG_KERNELS
#include "ctx.h"

int launch_phase1(hg_ctx* ctx) {
  const uint32_t nt = (uint32_t)ctx->tile_stream.size();
  const uint32_t ns = (uint32_t)ctx->streams.size();
  int rc0 = init_run(ctx);
  if (rc0) return rc0;
  if (nt) {
    Params p = make_params(ctx);
    const size_t dsm = sizeof(uint2) * kSdescMax;
    CK(cudaEventRecord(ctx->ev[4], ctx->stream));
    const uint32_t gw = std::min<uint32_t>((nt + 255) / 256, (uint32_t)ctx->sm_count * 8);
    seg_walk_kernel<<<gw, 256, dsm, ctx->stream>>>(p, ctx->d_segw.ptr);
    CK(cudaEventRecord(ctx->ev[6], ctx->stream));
    seg_chain_kernel<<<(ns + 3) / 4, 128, dsm, ctx->stream>>>(p, ctx->d_segw.ptr, ctx->d_seginfo.ptr, ctx->d_stream_nrec.ptr);
    CK(cudaEventRecord(ctx->ev[7], ctx->stream));
    CK(cudaGetLastError());
    ctx->launches += 2;
    if (ctx->want & (HG_WANT_TIMELINE | HG_WANT_EVENTS | HG_WANT_VALIDATE | HG_WANT_TL_ITEMS)) {
      // timeline slots: one per record (segment decode), then compose's messages
      seg_rec_off_kernel<<<1, 1024, 0, ctx->stream>>>(ctx->d_stream_nrec.ptr, ns, ctx->d_tl_rec_off.ptr,
                                                      ctx->d_counters.ptr + C_REC_TOTAL);
      ctx->launches++;
      unsigned long long total = 0;
      CK(cudaMemcpyAsync(&total, ctx->d_counters.ptr + C_REC_TOTAL, 8, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      ctx->tl_comp_base = total;
      ctx->tl_cap = 2 * total + 64;  // compose adds at most one message per summary entry
      if (ctx->want & (HG_WANT_TIMELINE | HG_WANT_TL_ITEMS)) CK(ctx->d_tl_items.ensure(ctx->tl_cap));
      p = make_params(ctx);
    }
    const size_t smem = seg_smem_layout(ctx->n_fn).total;
    CK(cudaFuncSetAttribute(seg_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seg_decode_kernel, kSegThreads, smem));
    if (per_sm < 1) return fail(ctx, HG_ECUDA, "segment kernel does not fit on an SM");
    uint32_t grid = std::min<uint32_t>((uint32_t)(per_sm * ctx->sm_count), (nt + kSegThreads - 1) / kSegThreads);
    grid = std::max<uint32_t>(grid, 1);
    CK(ctx->d_params.ensure(1));
    CK(cudaMemcpyAsync(ctx->d_params.ptr, &p, sizeof(Params), cudaMemcpyHostToDevice, ctx->stream));
    seg_decode_kernel<<<grid, kSegThreads, smem, ctx->stream>>>(p, ctx->d_seginfo.ptr, ctx->d_params.ptr);
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[5], ctx->stream));
    ctx->launches++;
  }
  return HG_OK;
}

