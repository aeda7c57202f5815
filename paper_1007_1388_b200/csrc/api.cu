// api.cu -- the C ABI of include/lbm.h (argument validation, state rules,
// error reporting); the work is in setup.cu, step.cu and transfer.cu.
#include <algorithm>
#include <cstdlib>
#include <new>

#include "context.h"

namespace lbm {
thread_local std::string g_create_error;

// Before the host reads or replaces the state: drain both streams and, with the
// fused exchange, wait until the peers' last stores into this rank's grid have
// landed (quiesce, step.cu).
static lbm_status drain(lbm_ctx *ctx)
{
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->comm_stream));
    return quiesce(ctx);
}
}  // namespace lbm

// ===================================================================== C ABI
extern "C" {

LBM_API int32_t lbm_abi_version(void) { return LBM_ABI_VERSION; }

LBM_API void lbm_config_default(lbm_config *cfg)
{
    if (!cfg) return;
    std::memset(cfg, 0, sizeof *cfg);
    cfg->omega = 1.0 / 0.65;
    cfg->precision = LBM_FP64;
    cfg->device = -1;
    cfg->rank = 0;
    cfg->nranks = 1;
    cfg->exchange_mode = LBM_EXCHANGE_AUTO;
    cfg->overlap = 1;
    cfg->use_graphs = 1;
    cfg->layout = LBM_LAYOUT_AB;
}

LBM_API lbm_status lbm_create(const int64_t domain[3], const int32_t patch[3], double omega, int32_t precision,
                              lbm_ctx **out)
{
    if (!domain || !patch) {
        g_create_error = "domain/patch is NULL";
        if (out) *out = nullptr;
        return LBM_ERR_ARG;
    }
    lbm_config cfg;
    lbm_config_default(&cfg);
    for (int a = 0; a < 3; ++a) {
        cfg.domain[a] = domain[a];
        cfg.patch[a] = patch[a];
    }
    cfg.omega = omega;
    cfg.precision = precision;
    return create_impl(&cfg, out);
}

LBM_API lbm_status lbm_create_ex(const lbm_config *cfg, lbm_ctx **out) { return create_impl(cfg, out); }

LBM_API lbm_status lbm_destroy(lbm_ctx *ctx)
{
    destroy_ctx(ctx);
    return LBM_OK;
}

LBM_API lbm_status lbm_set_flags(lbm_ctx *ctx, const uint8_t *flags, const double *wall_u, int32_t nvel)
{
    CHECK_CTX(ctx);
    const char *m = validate_flags(ctx->dec, flags, wall_u, nvel);
    if (m[0]) return ctx->fail(LBM_ERR_ARG, m);
    if (ctx->layout == LBM_LAYOUT_AA && ctx->aa_phase != 0)
        return ctx->fail(LBM_ERR_STATE, "AA layout: set_flags is only valid after an even number of steps");
    lbm_status st = drain(ctx);
    if (st) return st;
    st = apply_flags(ctx, flags, wall_u, nvel);
    if (st) return st;
    return refresh_state(ctx);
}

LBM_API lbm_status lbm_get_flags(lbm_ctx *ctx, uint8_t *out)
{
    CHECK_CTX(ctx);
    if (!out) return ctx->fail(LBM_ERR_ARG, "flags_out is NULL");
    {
        lbm_status st = drain(ctx);
        if (st) return st;
    }
    const Decomp &d = ctx->dec;
    const Geom &g = ctx->g;
    std::vector<uint8_t> h((size_t)d.nlocal * g.fs);
    CK(cudaMemcpy(h.data(), ctx->flags, h.size(), cudaMemcpyDeviceToHost));
    const int64_t on[3] = {d.owned_hi[0] - d.owned_lo[0], d.owned_hi[1] - d.owned_lo[1], d.owned_hi[2] - d.owned_lo[2]};
    for (int64_t z = -1; z <= on[2]; ++z)
        for (int64_t y = -1; y <= on[1]; ++y)
            for (int64_t x = -1; x <= on[0]; ++x) {
                const int64_t c[3] = {x, y, z};
                int b[3], lc[3];
                for (int a = 0; a < 3; ++a) {
                    int64_t cc = std::min(std::max(c[a], (int64_t)0), on[a] - 1);
                    b[a] = (int)(cc / g.n[a]);
                    lc[a] = (int)(c[a] - (int64_t)b[a] * g.n[a]);
                }
                const int lp = (b[2] * d.brick[1] + b[1]) * d.brick[0] + b[0];
                const int64_t ci = flag_index(g, lc[0], lc[1], lc[2]);
                out[((z + 1) * (on[1] + 2) + (y + 1)) * (on[0] + 2) + (x + 1)] = h[(size_t)lp * g.fs + ci];
            }
    return LBM_OK;
}

LBM_API lbm_status lbm_set_pdfs(lbm_ctx *ctx, const double *f)
{
    CHECK_CTX(ctx);
    if (!f) return ctx->fail(LBM_ERR_ARG, "f is NULL");
    lbm_status st = drain(ctx);
    if (st) return st;
    st = transfer_chunks(ctx, const_cast<double *>(f), true, 0, nullptr, nullptr);
    if (st) return st;
    return refresh_state(ctx);
}

LBM_API lbm_status lbm_init_noise(lbm_ctx *ctx, uint64_t seed)
{
    CHECK_CTX(ctx);
    {
        lbm_status st = drain(ctx);
        if (st) return st;
    }
    const Decomp &d = ctx->dec;
    const int64_t on[3] = {d.owned_hi[0] - d.owned_lo[0], d.owned_hi[1] - d.owned_lo[1], d.owned_hi[2] - d.owned_lo[2]};
    cudaError_t e = ctx->esize == 8
                        ? launch_noise<double>((double *)ctx->grid[ctx->cur], seed, d.domain, d.owned_lo, on, d.brick,
                                               ctx->g, ctx->layout == LBM_LAYOUT_AA ? 1 : 0, ctx->stream)
                        : launch_noise<float>((float *)ctx->grid[ctx->cur], seed, d.domain, d.owned_lo, on, d.brick,
                                              ctx->g, ctx->layout == LBM_LAYOUT_AA ? 1 : 0, ctx->stream);
    ctx->aa_phase = 0;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "noise_kernel", __FILE__, __LINE__);
    ctx->launches += 1;
    return refresh_state(ctx);
}

LBM_API lbm_status lbm_step_async(lbm_ctx *ctx, int64_t nsteps)
{
    CHECK_CTX(ctx);
    if (nsteps < 0) return ctx->fail(LBM_ERR_ARG, "nsteps must be >= 0");
    return enqueue_steps(ctx, nsteps);
}

LBM_API lbm_status lbm_synchronize(lbm_ctx *ctx)
{
    CHECK_CTX(ctx);
    // lbm_step returns with the state globally quiescent: the peers' stores
    // into this rank's grid for every step done have landed.
    lbm_status st = drain(ctx);
    if (st) return st;
    if ((st = chk_report(ctx))) return st;
    if (ctx->timing) return flush_timing(ctx);
    return LBM_OK;
}

LBM_API lbm_status lbm_step(lbm_ctx *ctx, int64_t nsteps)
{
    lbm_status st = lbm_step_async(ctx, nsteps);
    if (st) return st;
    return lbm_synchronize(ctx);
}

LBM_API lbm_status lbm_get_pdfs(lbm_ctx *ctx, double *f_out)
{
    CHECK_CTX(ctx);
    if (!f_out) return ctx->fail(LBM_ERR_ARG, "f_out is NULL");
    lbm_status st = drain(ctx);
    if (st) return st;
    return transfer_chunks(ctx, f_out, false, 0, nullptr, nullptr);
}

LBM_API lbm_status lbm_get_pdfs_at(lbm_ctx *ctx, const int64_t *xyz, int64_t n, double *out)
{
    CHECK_CTX(ctx);
    if (n < 0 || (n > 0 && (!xyz || !out))) return ctx->fail(LBM_ERR_ARG, "bad sample arguments");
    if (n == 0) return LBM_OK;
    {
        lbm_status st = drain(ctx);
        if (st) return st;
    }
    std::vector<int64_t> loc((size_t)3 * n);
    for (int64_t k = 0; k < n; ++k)
        for (int a = 0; a < 3; ++a) {
            const int64_t c = xyz[3 * k + a];
            if (c < ctx->dec.owned_lo[a] || c >= ctx->dec.owned_hi[a])
                return ctx->fail(LBM_ERR_ARG, "sample cell outside the owned brick");
            loc[3 * k + a] = c - ctx->dec.owned_lo[a];
        }
    int64_t *dxyz = nullptr;
    double *dout = nullptr;
    lbm_status st = dev_alloc(ctx, &dxyz, loc.size() * sizeof(int64_t));
    if (st) return st;
    st = dev_alloc(ctx, &dout, (size_t)n * Q * sizeof(double));
    if (st) {
        cudaFree(dxyz);
        return st;
    }
    cudaError_t e = cudaMemcpyAsync(dxyz, loc.data(), loc.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess)
    {
        const int rep = ctx->layout == LBM_LAYOUT_AA ? (ctx->aa_phase == 0 ? 1 : 2) : 0;
        if (e == cudaSuccess)
            e = ctx->esize == 8 ? launch_gather<double>((const double *)ctx->grid[ctx->cur], ctx->flags, dxyz, n,
                                                        ctx->dec.brick, ctx->g, dout, rep, (const double *)ctx->corr,
                                                        ctx->stream)
                                : launch_gather<float>((const float *)ctx->grid[ctx->cur], ctx->flags, dxyz, n,
                                                       ctx->dec.brick, ctx->g, dout, rep, (const float *)ctx->corr,
                                                       ctx->stream);
    }
    ctx->launches += 1;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, dout, (size_t)n * Q * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(dxyz);
    cudaFree(dout);
    ctx->device_bytes -= (int64_t)(loc.size() * sizeof(int64_t) + (size_t)n * Q * sizeof(double));
    if (e != cudaSuccess) return ctx->cuda_fail(e, "gather", __FILE__, __LINE__);
    return LBM_OK;
}

LBM_API lbm_status lbm_get_macroscopic(lbm_ctx *ctx, double *rho_out, double *u_out)
{
    CHECK_CTX(ctx);
    {
        lbm_status st = drain(ctx);
        if (st) return st;
    }
    if (!rho_out && !u_out) return LBM_OK;
    return transfer_chunks(ctx, nullptr, false, 1, rho_out, u_out);
}

LBM_API lbm_status lbm_total_mass(lbm_ctx *ctx, double *mass_out)
{
    CHECK_CTX(ctx);
    if (!mass_out) return ctx->fail(LBM_ERR_ARG, "mass_out is NULL");
    lbm_status st = drain(ctx);
    if (st) return st;
    if (!ctx->d_mass && (st = dev_alloc(ctx, &ctx->d_mass, (size_t)(kMassBlocks + 1) * sizeof(double)))) return st;
    const Decomp &d = ctx->dec;
    const int64_t on[3] = {d.owned_hi[0] - d.owned_lo[0], d.owned_hi[1] - d.owned_lo[1], d.owned_hi[2] - d.owned_lo[2]};
    // representation of the state in the grid (aux_kernels.cu rep_slot / read_state)
    const int rep = ctx->layout == LBM_LAYOUT_AA ? (ctx->aa_phase == 0 ? 1 : 2) : 0;
    double *sum = ctx->d_mass + kMassBlocks;
    const cudaError_t e =
        ctx->esize == 8 ? launch_mass<double>((const double *)ctx->grid[ctx->cur], ctx->flags, d.owned_lo, on, d.brick,
                                              ctx->g, rep, (const double *)ctx->corr, ctx->d_mass, sum, ctx->stream)
                        : launch_mass<float>((const float *)ctx->grid[ctx->cur], ctx->flags, d.owned_lo, on, d.brick,
                                             ctx->g, rep, (const float *)ctx->corr, ctx->d_mass, sum, ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "mass_kernel", __FILE__, __LINE__);
    ctx->launches += 2;
    if (ctx->nccl) NK(ncclAllReduce(sum, sum, 1, ncclFloat64, ncclSum, ctx->nccl, ctx->stream));
    double dsum = 0.0;
    CK(cudaMemcpyAsync(&dsum, sum, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *mass_out = (double)ctx->fluid_global + dsum;  // rho0 = 1 per fluid cell + sum of delta rho
    return LBM_OK;
}

static void fill_info_decomp(const Decomp &d, int esize, const SegLists &segs, lbm_info *out)
{
    for (int a = 0; a < 3; ++a) {
        out->domain[a] = d.domain[a];
        out->patch[a] = d.patch[a];
        out->proc_grid[a] = d.proc[a];
        out->proc_coord[a] = d.coord[a];
        out->owned_lo[a] = d.owned_lo[a];
        out->owned_hi[a] = d.owned_hi[a];
    }
    out->precision = esize;
    out->rank = d.rank;
    out->nranks = d.nranks;
    out->patches_local = d.nlocal;
    out->patches_global = d.pgrid[0] * d.pgrid[1] * d.pgrid[2];
    std::vector<int> peers;
    int64_t remote = 0, local = 0;
    int msgs = 0;
    for (const Seg &s : segs.send) {
        if (s.peer != d.rank) {
            remote += (int64_t)s.nq * s.cells * esize;
            ++msgs;
            if (std::find(peers.begin(), peers.end(), s.peer) == peers.end()) peers.push_back(s.peer);
        } else {
            local += (int64_t)s.nq * s.cells * esize;
        }
    }
    for (const Seg &s : segs.local) local += (int64_t)s.nq * s.cells * esize;
    out->peers = (int32_t)peers.size();
    out->messages_remote = msgs;
    out->halo_bytes_remote_per_step = remote;
    out->halo_bytes_local_per_step = local;
}

LBM_API lbm_status lbm_get_info(lbm_ctx *ctx, lbm_info *out)
{
    if (!ctx || !out) return LBM_ERR_ARG;
    std::memset(out, 0, sizeof *out);
    fill_info_decomp(ctx->dec, ctx->esize, ctx->ex[EX_AB].segs, out);
    out->fluid_cells_local = ctx->fluid_local;
    out->fluid_cells_global = ctx->fluid_global;
    out->steps_done = ctx->steps;
    out->bytes_per_step_algorithmic = 2.0 * Q * ctx->esize * (double)ctx->fluid_local;
    out->kernel_launches = ctx->launches;
    out->device_bytes = ctx->device_bytes;
    for (int i = 0; i < LBM_NPHASES; ++i) {
        out->phase_ms[i] = ctx->phase_ms[i];
        out->phase_count[i] = ctx->phase_count[i];
    }
    out->row_pitch_elems = ctx->g.px;
    out->align_bytes = 32;  // rows start on 32-B sectors
    out->graphs_active = (ctx->graph[0] || ctx->graph[1]) ? 1 : 0;
    out->layout = ctx->layout;
    out->aa_phase = ctx->aa_phase;
    out->exchange_fused = ctx->direct ? 1 : 0;
    out->local_pull = 0;  // removed in round 2 (measured slower)
    out->local_direct = ctx->ldirect ? 1 : 0;
    out->overlap_active = (ctx->use_overlap && !ctx->direct) ? 1 : 0;
    int nr = 0;
    if (ctx->nccl && ncclCommCount(ctx->nccl, &nr) != ncclSuccess) nr = -1;
    out->nccl_ranks = nr;
    out->fused_peers = ctx->direct ? ctx->npeers_direct : 0;
    return LBM_OK;
}

LBM_API lbm_status lbm_set_timing(lbm_ctx *ctx, int32_t enable)
{
    CHECK_CTX(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    lbm_status st = flush_timing(ctx);
    if (st) return st;
    ctx->timing = enable != 0;
    for (int i = 0; i < LBM_NPHASES; ++i) {
        ctx->phase_ms[i] = 0;
        ctx->phase_count[i] = 0;
    }
    return LBM_OK;
}

LBM_API lbm_status lbm_get_stream(lbm_ctx *ctx, void **stream_out)
{
    if (!ctx || !stream_out) return LBM_ERR_ARG;
    *stream_out = (void *)ctx->stream;
    return LBM_OK;
}

LBM_API const char *lbm_last_error(const lbm_ctx *ctx)
{
    if (!ctx) return g_create_error.c_str();
    return ctx->err.c_str();
}

LBM_API lbm_status lbm_nccl_unique_id(void *out, int64_t nbytes)
{
    if (!out || nbytes < (int64_t)sizeof(ncclUniqueId)) return LBM_ERR_ARG;
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        g_create_error = std::string("ncclGetUniqueId failed: ") + ncclGetErrorString(r);
        return LBM_ERR_NCCL;
    }
    std::memcpy(out, &id, sizeof id);
    return LBM_OK;
}

LBM_API lbm_status lbm_plan(const lbm_config *cfg, lbm_info *info, lbm_msg *msgs, int32_t cap, int32_t *nmsgs)
{
    if (!cfg) return LBM_ERR_ARG;
    Decomp dec;
    const char *m = decompose(*cfg, dec);
    if (m[0]) {
        g_create_error = m;
        return LBM_ERR_ARG;
    }
    SegLists segs;
    build_segments(dec, segs);
    if (info) {
        std::memset(info, 0, sizeof *info);
        fill_info_decomp(dec, cfg->precision, segs, info);
    }
    int32_t k = 0;
    auto emit = [&](const Seg &s, int send) {
        if (s.peer == dec.rank && !dec.force_buffers) return;
        if (msgs && k < cap) {
            lbm_msg &o = msgs[k];
            o.peer = s.peer;
            o.send = send;
            o.patch_local = send ? s.send_patch : s.recv_patch;
            o.patch_remote = send ? s.recv_patch : s.send_patch;
            for (int a = 0; a < 3; ++a) o.dir[a] = s.d[a];
            o.nq = s.nq;
            o.cells = s.cells;
            o.offset = s.offset;
        }
        ++k;
    };
    for (const Seg &s : segs.send) emit(s, 1);
    for (const Seg &s : segs.recv) emit(s, 0);
    if (nmsgs) *nmsgs = k;
    return LBM_OK;
}

}  // extern "C"
