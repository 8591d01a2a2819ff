// fast.cu -- the single pass over HBM (fast.cuh): launch of the range kernel, chain verification, orphan fix-up
#define HG_FAST_KERNELS
#include "ctx.h"

// the single pass (fast.cuh): range kernel, chain verification, orphan index fix-up
int launch_fast(hg_ctx* ctx) {
  const uint32_t ns = (uint32_t)ctx->streams.size();
  int rc = init_run(ctx);
  if (rc) return rc;
  if (!ctx->n_ranges) return HG_OK;
  Params p = make_params(ctx);
  p.state = ctx->d_rseg.ptr;
  const uint32_t nw = ctx->fast_warps;
  uint32_t n_fd = 0, n_cd = 0;
  const int sd = fast_desc_mode(ctx->max_sid, ctx->n_fn, ctx->has_dev, (uint32_t)ctx->smem_optin, n_fd, n_cd);
  const size_t smem = fast_smem_layout(ctx->n_fn, nw, n_fd, n_cd, ctx->has_dev).total;
  using K = void (*)(Params, const Params*);
#define HG_FK(m) fast_kernel<0, false, m>, fast_kernel<0, true, m>, fast_kernel<1, false, m>, fast_kernel<1, true, m>, \
                 fast_kernel<2, false, m>, fast_kernel<2, true, m>
  static const K kerns[24] = {HG_FK(0), HG_FK(1), HG_FK(2), HG_FK(3)};
#undef HG_FK
  const int mode = (p.tl_ritems ? 1 : 0) | (p.ev_ritems ? 2 : 0);
  const K kern = kerns[6 * mode + 2 * sd + (ctx->deep_inline ? 1 : 0)];
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const uint32_t per_cta = nw * kWarp;
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)ctx->sm_count, (ctx->n_ranges + per_cta - 1) / per_cta));
  p.prescan = 1;
  CK(ctx->d_params.ensure(1));
  CK(cudaMemcpyAsync(ctx->d_params.ptr, &p, sizeof(Params), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->ev[4], ctx->stream));
  {
    const uint32_t sgrid = std::max<uint32_t>(1, (ctx->n_ranges + 7) / 8);  // a warp per range (54 -> 46 us on C2)
    const size_t ssm = ctx->max_sid < (uint32_t)kSdescMax ? 8u * (ctx->max_sid + 1) : 0u;
    fast_scan_kernel<<<sgrid, 256, ssm, ctx->stream>>>(p);
  }
  kern<<<grid, per_cta, smem, ctx->stream>>>(p, ctx->d_params.ptr);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[7], ctx->stream));
  if (ctx->max_rps > 1024) fast_verify_kernel<512><<<ns, 512, 0, ctx->stream>>>(p, ctx->d_stream_nrec.ptr);
  else fast_verify_kernel<128><<<ns, 128, 0, ctx->stream>>>(p, ctx->d_stream_nrec.ptr);
  fast_orphan_fix_kernel<<<32, 256, 0, ctx->stream>>>(p);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[5], ctx->stream));
  ctx->launches += 4;
  return HG_OK;
}

