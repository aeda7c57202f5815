// transfer.cu -- host <-> device transfers of the canonical [z][y][x][19]
// layout (lbm_set_pdfs / lbm_get_pdfs / lbm_get_macroscopic).
#include <algorithm>

#include "context.h"

namespace lbm {

// Host <-> device transfers of the canonical layout, pipelined through two
// persistent staging buffers: chunk k's DMA (copy stream) overlaps the
// import / export kernel of chunk k +- 1 (compute stream); the event pairs
// hand each buffer back and forth.  Returns after both streams drained, so the
// caller's host buffer is free again.
constexpr size_t kStageBytes = (size_t)64 << 20;

lbm_status ensure_xstage(lbm_ctx *ctx, size_t plane_bytes)
{
    const size_t need = std::max(kStageBytes, plane_bytes);
    if (!ctx->xstream) {
        if (cudaStreamCreateWithFlags(&ctx->xstream, cudaStreamNonBlocking) != cudaSuccess)
            return ctx->fail(LBM_ERR_CUDA, "copy stream creation failed");
        for (int b = 0; b < 2; ++b)
            if (cudaEventCreateWithFlags(&ctx->xev_copy[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ctx->xev_kern[b], cudaEventDisableTiming) != cudaSuccess)
                return ctx->fail(LBM_ERR_CUDA, "copy event creation failed");
    }
    if (ctx->xstage_bytes >= need) return LBM_OK;
    for (int b = 0; b < 2; ++b)
        if (ctx->xstage[b]) {
            cudaFree(ctx->xstage[b]);
            ctx->xstage[b] = nullptr;
            ctx->device_bytes -= (int64_t)ctx->xstage_bytes;
        }
    ctx->xstage_bytes = 0;
    for (int b = 0; b < 2; ++b) {
        lbm_status st = dev_alloc(ctx, &ctx->xstage[b], need);
        if (st) return st;
    }
    ctx->xstage_bytes = need;
    return LBM_OK;
}

lbm_status transfer_chunks(lbm_ctx *ctx, double *host, bool to_device, int mode, double *rho, double *u)
{
    const int64_t on[3] = {ctx->dec.owned_hi[0] - ctx->dec.owned_lo[0], ctx->dec.owned_hi[1] - ctx->dec.owned_lo[1],
                           ctx->dec.owned_hi[2] - ctx->dec.owned_lo[2]};
    const int64_t plane_cells = on[0] * on[1];
    const size_t per_cell = mode == 0 ? Q * sizeof(double) : 4 * sizeof(double);
    lbm_status st = ensure_xstage(ctx, (size_t)plane_cells * Q * sizeof(double));
    if (st) return st;
    int64_t zc = (int64_t)(ctx->xstage_bytes / (plane_cells * per_cell));
    if (zc < 1) zc = 1;
    if (zc > on[2]) zc = on[2];
    const void *grid = ctx->grid[ctx->cur];
    // representation of the state in the grid (aux_kernels.cu rep_slot / read_state)
    const int rep = ctx->layout == LBM_LAYOUT_AA ? (to_device || ctx->aa_phase == 0 ? 1 : 2) : 0;
    if (to_device) ctx->aa_phase = 0;
    cudaStream_t cs = ctx->stream, xs = ctx->xstream;
    cudaError_t e = cudaSuccess;
    // the copy stream starts after everything already queued on the compute stream
    e = cudaEventRecord(ctx->xev_kern[0], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(xs, ctx->xev_kern[0], 0);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_kern[1], cs);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_copy[0], xs);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_copy[1], xs);
    int64_t k = 0;
    for (int64_t z0 = 0; z0 < on[2] && e == cudaSuccess; z0 += zc, ++k) {
        const int b = (int)(k & 1);
        double *stage = ctx->xstage[b];
        const int64_t nzc = std::min(zc, on[2] - z0);
        const size_t cells = (size_t)(nzc * plane_cells);
        if (to_device) {
            // buffer b is free once the import of chunk k - 2 has run
            e = cudaStreamWaitEvent(xs, ctx->xev_kern[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(stage, host + (size_t)z0 * plane_cells * Q, cells * Q * sizeof(double),
                                    cudaMemcpyHostToDevice, xs);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_copy[b], xs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ctx->xev_copy[b], 0);
            if (e == cudaSuccess)
                e = ctx->esize == 8 ? launch_import<double>(stage, z0, nzc, ctx->dec.owned_lo, on, ctx->dec.brick,
                                                            ctx->g, (double *)grid, rep, cs)
                                    : launch_import<float>(stage, z0, nzc, ctx->dec.owned_lo, on, ctx->dec.brick,
                                                           ctx->g, (float *)grid, rep, cs);
            ctx->launches += 1;
            if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_kern[b], cs);
        } else {
            // buffer b is free once the copy-out of chunk k - 2 has run
            e = cudaStreamWaitEvent(cs, ctx->xev_copy[b], 0);
            double *srho = stage, *su = stage + cells;
            if (e == cudaSuccess)
                e = ctx->esize == 8
                        ? launch_export<double>((const double *)grid, ctx->flags, z0, nzc, ctx->dec.owned_lo, on,
                                                ctx->dec.brick, ctx->g, stage, mode, srho, su, rep,
                                                (const double *)ctx->corr, cs)
                        : launch_export<float>((const float *)grid, ctx->flags, z0, nzc, ctx->dec.owned_lo, on,
                                               ctx->dec.brick, ctx->g, stage, mode, srho, su, rep,
                                               (const float *)ctx->corr, cs);
            ctx->launches += 1;
            if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_kern[b], cs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(xs, ctx->xev_kern[b], 0);
            if (e == cudaSuccess) {
                if (mode == 0) {
                    e = cudaMemcpyAsync(host + (size_t)z0 * plane_cells * Q, stage, cells * Q * sizeof(double),
                                        cudaMemcpyDeviceToHost, xs);
                } else {
                    if (rho)
                        e = cudaMemcpyAsync(rho + (size_t)z0 * plane_cells, srho, cells * sizeof(double),
                                            cudaMemcpyDeviceToHost, xs);
                    if (e == cudaSuccess && u)
                        e = cudaMemcpyAsync(u + (size_t)z0 * plane_cells * 3, su, cells * 3 * sizeof(double),
                                            cudaMemcpyDeviceToHost, xs);
                }
            }
            if (e == cudaSuccess) e = cudaEventRecord(ctx->xev_copy[b], xs);
        }
    }
    const cudaError_t e1 = cudaStreamSynchronize(xs), e2 = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = e1 != cudaSuccess ? e1 : e2;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "host/device transfer", __FILE__, __LINE__);
    return LBM_OK;
}

}  // namespace lbm
