// step.cu -- one time step (the paper's Sweep) on a rank: sweep
// (fused pull + BB + collide, sweep.cu / sweep_aa.cu) and ghost exchange -- folded into the
// sweep as direct ghost stores (same GPU and, fused, NVLink stores into the
// peers' grids with one epoch handshake), or extract -> NCCL -> insert
// (P:287-313), shells first and overlapped with the interiors (the
// paper sums these times).  Step pairs are captured in CUDA graphs.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <new>

#include "context.h"

namespace lbm {

void fill_dir_offsets(const Geom &g, bool aa, int esize, DirOffsets &o)
{
    for (int i = 0; i < Q; ++i) {
        const int sl = aa ? OPPf(i) : i;
        const int64_t yz = EYf(i) * (int64_t)g.px + EZf(i) * g.plane;
        o.pull[i] = (sl * g.qs - EXf(i) - yz) * esize;
        o.gpull[i] = (sl * g.gq + (EXf(i) > 0 ? 0 : g.gside) - EYf(i) - EZf(i) * (int64_t)g.gy) * esize;
        o.slot[i] = i * g.qs * esize;
        o.oslot[i] = OPPf(i) * g.qs * esize;
        o.push[i] = (i * g.qs + EXf(i) + yz) * esize;
        o.gpush[i] = (i * g.gq + (EXf(i) < 0 ? 0 : g.gside) + EYf(i) + EZf(i) * (int64_t)g.gy) * esize;
        o.gwall[i] = (OPPf(i) * g.gq + (EXf(i) < 0 ? 0 : g.gside) + EYf(i) + EZf(i) * (int64_t)g.gy) * esize;
        o.wall[i] = (OPPf(i) * g.qs + EXf(i) + yz) * esize;
    }
}

Checker next_checker(lbm_ctx *ctx)
{
    Checker c = ctx->chk;
#ifdef LBM_CHECKED
    c.launch = (++ctx->chk_seq) << 32;
#endif
    return c;
}

lbm_status chk_alloc(lbm_ctx *ctx, size_t grid_bytes)
{
#ifdef LBM_CHECKED
    Checker &c = ctx->chk;
    c.esize = ctx->esize;
    if (const char *v = std::getenv("LBM_CHECKED_INJECT")) c.inject = std::atoi(v);
    c.elems = (int64_t)(grid_bytes / ctx->esize);
    for (int i = 0; i < 2; ++i) {
        c.lo[i] = (const char *)ctx->grid[i];
        c.hi[i] = ctx->grid[i] ? (const char *)ctx->grid[i] + grid_bytes : nullptr;
    }
    lbm_status st;
    if ((st = dev_alloc(ctx, &c.wr, 2 * (size_t)c.elems * sizeof(unsigned long long)))) return st;
    if ((st = dev_alloc(ctx, &c.rd, 2 * (size_t)c.elems * sizeof(unsigned long long)))) return st;
    if ((st = dev_alloc(ctx, &c.err, 3 * sizeof(unsigned long long)))) return st;
    CK(memset_sync(ctx, c.err, 0, 3 * sizeof(unsigned long long)));
    return chk_clear(ctx, ctx->stream);
#else
    (void)ctx;
    (void)grid_bytes;
    return LBM_OK;
#endif
}

lbm_status chk_clear(lbm_ctx *ctx, cudaStream_t s)
{
#ifdef LBM_CHECKED
    const size_t b = 2 * (size_t)ctx->chk.elems * sizeof(unsigned long long);
    CK(cudaMemsetAsync(ctx->chk.wr, 0, b, s));
    CK(cudaMemsetAsync(ctx->chk.rd, 0, b, s));
#else
    (void)ctx;
    (void)s;
#endif
    return LBM_OK;
}

lbm_status chk_report(lbm_ctx *ctx)
{
#ifdef LBM_CHECKED
    unsigned long long e[3] = {0, 0, 0};
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(e, ctx->chk.err, sizeof e, cudaMemcpyDeviceToHost));
    if (e[0] | e[1] | e[2]) {
        CK(cudaMemset(ctx->chk.err, 0, sizeof e));
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "checked build: %llu out-of-bounds or misaligned accesses, %llu elements written twice in "
                      "one step, %llu read/write races within a launch",
                      e[0], e[1], e[2]);
        return ctx->fail(LBM_ERR_INTERNAL, buf);
    }
#else
    (void)ctx;
#endif
    return LBM_OK;
}

template <typename real>
SweepArgs<real> sweep_args(lbm_ctx *ctx, const DevBoxes &b)
{
    SweepArgs<real> a;
    if (ctx->layout == LBM_LAYOUT_AA) {  // in place
        a.src = (const real *)ctx->grid[0];
        a.dst = (real *)ctx->grid[0];
    } else {
        a.src = (const real *)ctx->grid[ctx->cur];
        a.dst = (real *)ctx->grid[1 - ctx->cur];
    }
    a.kind = ctx->kind;
    a.corr = (const real *)ctx->corr;
    a.g = ctx->g;
    a.omega = (real)ctx->cfg.omega;
    a.tiles = b.desc;
    a.sidewall = ctx->sidewall;
    a.dnbr = ctx->ldirect ? (real *const *)ctx->d_dnbr : nullptr;
    a.dsti = ctx->layout == LBM_LAYOUT_AA ? 0 : 1 - ctx->cur;
    fill_dir_offsets(ctx->g, ctx->layout == LBM_LAYOUT_AA, (int)sizeof(real), a.off);
    a.chk = next_checker(ctx);
    return a;
}

lbm_status launch_sweep_set(lbm_ctx *ctx, const DevBoxes &b, cudaStream_t s)
{
    if (b.tiles == 0) return LBM_OK;
    cudaError_t e;
    if (ctx->layout == LBM_LAYOUT_AA) {
        const bool pull = ctx->aa_phase == 0;
        if (ctx->esize == 8)
            e = launch_sweep_aa<double>(sweep_args<double>(ctx, b), b.tiles, pull, ctx->sweep_variant, s);
        else
            e = launch_sweep_aa<float>(sweep_args<float>(ctx, b), b.tiles, pull, ctx->sweep_variant, s);
    } else if (ctx->esize == 8)
        e = launch_sweep<double>(sweep_args<double>(ctx, b), b.tiles, ctx->sweep_variant, s);
    else
        e = launch_sweep<float>(sweep_args<float>(ctx, b), b.tiles, ctx->sweep_variant, s);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "sweep_kernel launch", __FILE__, __LINE__);
    ctx->launches += 1;
    return LBM_OK;
}

lbm_status launch_copy(lbm_ctx *ctx, const DevSegs &d, void *grid_src, void *grid_dst, void *buf_src, void *buf_dst,
                       cudaStream_t s)
{
    if (d.n == 0 || d.max_elems == 0) return LBM_OK;
    cudaError_t e;
    if (ctx->esize == 8)
        e = launch_copy_segments<double>(d.segs, d.n, d.max_elems, (const double *)grid_src, (double *)grid_dst,
                                         (const double *)buf_src, (double *)buf_dst, ctx->flags, ctx->g, s);
    else
        e = launch_copy_segments<float>(d.segs, d.n, d.max_elems, (const float *)grid_src, (float *)grid_dst,
                                        (const float *)buf_src, (float *)buf_dst, ctx->flags, ctx->g, s);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "copy_segments launch", __FILE__, __LINE__);
    ctx->launches += (d.n + 65534) / 65535;
    return LBM_OK;
}

// Transport of the send buffers: grouped NCCL send/recv per peer.
// A self-peer (exchange_mode FORCE_BUFFERS / SELF_PEER on one GPU) goes through
// the same NCCL group when the context has a communicator (FORCE_BUFFERS: a
// one-rank communicator), else (SELF_PEER's state refresh) a device copy.
lbm_status transport(lbm_ctx *ctx, const ExSet &X, cudaStream_t s)
{
    const ncclDataType_t dt = ctx->esize == 8 ? ncclFloat64 : ncclFloat32;
    char *sb = (char *)ctx->sendbuf, *rb = (char *)ctx->recvbuf;
    if (!ctx->nccl) {
        for (const Peer &p : X.peers)
            if (p.rank == ctx->dec.rank && p.send_n > 0)
                CK(cudaMemcpyAsync(rb + p.recv_off * ctx->esize, sb + p.send_off * ctx->esize,
                                   p.send_n * ctx->esize, cudaMemcpyDeviceToDevice, s));
        return LBM_OK;
    }
    NK(ncclGroupStart());
    for (const Peer &p : X.peers) {
        if (p.send_n > 0) NK(ncclSend(sb + p.send_off * ctx->esize, (size_t)p.send_n, dt, p.rank, ctx->nccl, s));
        if (p.recv_n > 0) NK(ncclRecv(rb + p.recv_off * ctx->esize, (size_t)p.recv_n, dt, p.rank, ctx->nccl, s));
    }
    NK(ncclGroupEnd());
    return LBM_OK;
}

// Ghost refresh of grid `gi` (used after set_pdfs / init and inside the step).
// in_step: right after a sweep, whose direct stores (ldirect) already filled
// the same-GPU ghosts.
lbm_status exchange_seq(lbm_ctx *ctx, int gi, cudaStream_t s, TimingSlot *ts, int kind, bool in_step)
{
    void *grid = ctx->grid[gi];
    const ExSet &X = ctx->ex[kind];
    lbm_status st;
    // direct ghost stores: the sweep already filled the same-GPU ghosts
    const bool skip_local = in_step && ctx->ldirect;
    const bool work = (skip_local ? X.pack_remote.n : X.pack_all.n) > 0 || X.has_remote || X.unpack.n > 0;
    if (!work) return LBM_OK;  // single periodic-free patch: nothing to exchange
    if (ts) ts->exchange = true;
    if (ts) CK(cudaEventRecord(ts->ev[2], s));
    if ((st = launch_copy(ctx, skip_local ? X.pack_remote : X.pack_all, grid, grid, nullptr, ctx->sendbuf, s)))
        return st;
    if (ts) CK(cudaEventRecord(ts->ev[3], s));
    if (X.has_remote) {
        if ((st = transport(ctx, X, s))) return st;
    }
    if (ts) CK(cudaEventRecord(ts->ev[4], s));
    if ((st = launch_copy(ctx, X.unpack, nullptr, grid, ctx->recvbuf, nullptr, s))) return st;
    if (ts) CK(cudaEventRecord(ts->ev[5], s));
    return LBM_OK;
}

void fill_bb_offsets(const Geom &g, int mode, int esize, BbOffsets &o)
{
    for (int j = 0; j < Q; ++j) {
        const int xslot = mode == 0 ? j : OPPf(j), wslot = mode == 0 ? OPPf(j) : j;
        o.xs[j] = xslot * g.qs * esize;
        o.wm[j] = (wslot * g.qs + EXf(j) + EYf(j) * (int64_t)g.px + EZf(j) * g.plane) * esize;
        o.wg[j] = (wslot * g.gq + (EXf(j) < 0 ? 0 : g.gside) + EYf(j) + EZf(j) * (int64_t)g.gy) * esize;
    }
}

lbm_status launch_bb(lbm_ctx *ctx, int gi, int mode, cudaStream_t s, bool full)
{
    const BbEntry *list = full ? ctx->bb_full : ctx->bb_list;
    const int64_t n = full ? ctx->bb_full_n : ctx->bb_n;
    if (n == 0) return LBM_OK;
    BbOffsets o;
    fill_bb_offsets(ctx->g, mode, ctx->esize, o);
    cudaError_t e = ctx->esize == 8
                        ? launch_bb_list<double>((double *)ctx->grid[gi], ctx->flags, list, n,
                                                 (const double *)ctx->corr, ctx->g, mode, o, next_checker(ctx), s)
                        : launch_bb_list<float>((float *)ctx->grid[gi], ctx->flags, list, n,
                                                (const float *)ctx->corr, ctx->g, mode, o, next_checker(ctx), s);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "bounce-back list launch", __FILE__, __LINE__);
    ctx->launches += 1;
    return LBM_OK;
}

// After the state or the flags change: refresh the ghost layers of the current
// grid and park the store-side bounce-back values in the wall cells.
lbm_status refresh_state(lbm_ctx *ctx)
{
    // AB: ghost layers of the current grid.  AA (swapped state): half-exchange 1,
    // which is what the next PULL step gathers from the ghost layers.
    const bool aa = ctx->layout == LBM_LAYOUT_AA;
    lbm_status st = exchange_seq(ctx, ctx->cur, ctx->stream, nullptr, aa ? EX_AA1 : EX_AB, false);
    if (st) return st;
    if ((st = chk_clear(ctx, ctx->stream))) return st;
    if ((st = launch_bb(ctx, ctx->cur, aa ? 1 : 0, ctx->stream, true))) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    return chk_report(ctx);
}

lbm_status accumulate_slot(lbm_ctx *ctx, TimingSlot &ts)
{
    if (!ts.used) return LBM_OK;
    CK(cudaEventSynchronize(ts.ev[kEvPerSlot - 1]));
    auto el = [&](int a, int b) -> double {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ts.ev[a], ts.ev[b]);
        return (double)ms;
    };
    if (!ts.overlap) {
        ctx->phase_ms[PH_SWEEP] += el(0, ts.exchange ? 2 : kEvPerSlot - 1);
        ctx->phase_count[PH_SWEEP] += 1;
        if (ts.exchange) {
            ctx->phase_ms[PH_PACK] += el(2, 3);
            ctx->phase_ms[PH_NCCL] += el(3, 4);
            ctx->phase_ms[PH_UNPACK] += el(4, 5);
            ctx->phase_count[PH_PACK] += 1;
            ctx->phase_count[PH_NCCL] += 1;
            ctx->phase_count[PH_UNPACK] += 1;
        }
    } else {
        ctx->phase_ms[PH_SHELL] += el(0, 2);
        ctx->phase_ms[PH_PACK] += el(2, 3);
        ctx->phase_ms[PH_NCCL] += el(6, 7);
        ctx->phase_ms[PH_UNPACK] += el(7, 8);
        ctx->phase_ms[PH_INTERIOR] += el(3, 9);
        for (int p : {PH_SHELL, PH_PACK, PH_NCCL, PH_UNPACK, PH_INTERIOR}) ctx->phase_count[p] += 1;
    }
    ctx->phase_ms[PH_STEP] += el(0, kEvPerSlot - 1);
    ctx->phase_count[PH_STEP] += 1;
    ts.used = false;
    cudaGetLastError();
    return LBM_OK;
}

lbm_status flush_timing(lbm_ctx *ctx)
{
    for (int i = 0; i < kTimingSlots; ++i) {
        lbm_status st = accumulate_slot(ctx, ctx->slots[i]);
        if (st) return st;
    }
    return LBM_OK;
}

// Enqueue one time step grid[cur] -> grid[1-cur] and flip cur.
lbm_status enqueue_step(lbm_ctx *ctx)
{
    cudaStream_t s = ctx->stream;
    TimingSlot *ts = nullptr;
    lbm_status st;
    if (kChecked && (st = chk_clear(ctx, s))) return st;  // one step = one single-writer window
    if (ctx->timing) {
        ts = &ctx->slots[ctx->slot_next];
        ctx->slot_next = (ctx->slot_next + 1) % kTimingSlots;
        if ((st = accumulate_slot(ctx, *ts))) return st;
        ts->used = true;
        ts->overlap = ctx->use_overlap && !ctx->direct;
        ts->exchange = false;
        CK(cudaEventRecord(ts->ev[0], s));
    }
    // AB: grid[cur] -> grid[1-cur], exchange of the pulled PDFs.  AA: in place
    // on grid[0]; a PULL step is followed by half-exchange 2, a LOCAL step by 1.
    const bool aa = ctx->layout == LBM_LAYOUT_AA;
    const int dsti = aa ? 0 : 1 - ctx->cur;
    const int kind = aa ? (ctx->aa_phase == 0 ? EX_AA2 : EX_AA1) : EX_AB;
    const ExSet &X = ctx->ex[kind];
    void *dst = ctx->grid[dsti];
    // walls after the sweep (launch_bb_list): two grids store-side (0); AA: the
    // PULL fix-up (2) or LOCAL's store side (1)
    const int bb_mode = aa ? (ctx->aa_phase == 0 ? 2 : 1) : 0;
    if (ctx->direct) {
        // Fused exchange across GPUs.  C (high priority): wait for the peers' epoch,
        // sweep the shells facing remote neighbours with the fused kernel (NVLink
        // stores of the outgoing PDFs into the peers' ghost layers), publish the
        // epoch.  S, concurrently: the plain sweep of everything else.  Then S joins
        // C and copies the ghosts between same-GPU patches.
        cudaStream_t c = ctx->comm_stream;
        cudaEvent_t ev_start = ts ? ts->ev[10] : ctx->slots[0].ev[10];
        cudaEvent_t ev_shell = ts ? ts->ev[11] : ctx->slots[0].ev[11];
        CK(cudaEventRecord(ev_start, s));
        CK(cudaStreamWaitEvent(c, ev_start, 0));
        cudaError_t e = launch_wait_peers(ctx->d_inbox, ctx->d_peer_rank, ctx->npeers_direct, ctx->d_epoch,
                                          ctx->d_error, c);
        if (e != cudaSuccess) return ctx->cuda_fail(e, "wait_peers launch", __FILE__, __LINE__);
        ctx->launches += 1;
        const DevBoxes &bs = ctx->box_shell;
        if (bs.tiles > 0) {
            const bool pull = ctx->aa_phase == 0;  // AA: PULL after an even step count
            if (ctx->esize == 8) {
                SweepArgs<double> a = sweep_args<double>(ctx, bs);
                a.dnbr = (double *const *)ctx->d_dnbr;
                e = aa ? launch_sweep_aa<double>(a, bs.tiles, pull, ctx->sweep_variant, c)
                       : launch_sweep<double>(a, bs.tiles, ctx->sweep_variant, c);
            } else {
                SweepArgs<float> a = sweep_args<float>(ctx, bs);
                a.dnbr = (float *const *)ctx->d_dnbr;
                e = aa ? launch_sweep_aa<float>(a, bs.tiles, pull, ctx->sweep_variant, c)
                       : launch_sweep<float>(a, bs.tiles, ctx->sweep_variant, c);
            }
            if (e != cudaSuccess) return ctx->cuda_fail(e, "shell sweep launch", __FILE__, __LINE__);
            ctx->launches += 1;
        }
        e = launch_signal_peers(ctx->d_epoch, ctx->d_peer_inbox, ctx->npeers_direct, c);
        if (e != cudaSuccess) return ctx->cuda_fail(e, "signal_peers launch", __FILE__, __LINE__);
        ctx->launches += 1;
        CK(cudaEventRecord(ev_shell, c));
        if ((st = launch_sweep_set(ctx, ctx->box_interior, s))) return st;
        CK(cudaStreamWaitEvent(s, ev_shell, 0));
        if ((st = launch_bb(ctx, dsti, bb_mode, s))) return st;
        if (!ctx->ldirect && (st = launch_copy(ctx, X.local_copy, dst, dst, nullptr, nullptr, s))) return st;
    } else if (!ctx->use_overlap) {
        if ((st = launch_sweep_set(ctx, ctx->box_all, s))) return st;
        if ((st = launch_bb(ctx, dsti, bb_mode, s))) return st;
        if ((st = exchange_seq(ctx, dsti, s, ts, kind, true))) return st;
    } else {
        cudaStream_t c = ctx->comm_stream;
        // S: shells facing remote neighbours, then pack them.
        if ((st = launch_sweep_set(ctx, ctx->box_shell, s))) return st;
        if (ts) CK(cudaEventRecord(ts->ev[2], s));
        if ((st = launch_copy(ctx, X.pack_remote, dst, dst, nullptr, ctx->sendbuf, s))) return st;
        if (ts) CK(cudaEventRecord(ts->ev[3], s));
        CK(cudaEventRecord(ts ? ts->ev[10] : ctx->slots[0].ev[10], s));
        // C: transport + unpack while S sweeps the interiors.
        CK(cudaStreamWaitEvent(c, ts ? ts->ev[10] : ctx->slots[0].ev[10], 0));
        if (ts) CK(cudaEventRecord(ts->ev[6], c));
        if ((st = transport(ctx, X, c))) return st;
        if (ts) CK(cudaEventRecord(ts->ev[7], c));
        if ((st = launch_copy(ctx, X.unpack, nullptr, dst, ctx->recvbuf, nullptr, c))) return st;
        if (ts) CK(cudaEventRecord(ts->ev[8], c));
        CK(cudaEventRecord(ts ? ts->ev[11] : ctx->slots[0].ev[11], c));
        if ((st = launch_sweep_set(ctx, ctx->box_interior, s))) return st;
        if ((st = launch_bb(ctx, dsti, bb_mode, s))) return st;
        if (ts) CK(cudaEventRecord(ts->ev[9], s));
        if (!ctx->ldirect && (st = launch_copy(ctx, X.local_copy, dst, dst, nullptr, nullptr, s)))
            return st;
        CK(cudaStreamWaitEvent(s, ts ? ts->ev[11] : ctx->slots[0].ev[11], 0));
    }
    if (ts) CK(cudaEventRecord(ts->ev[kEvPerSlot - 1], s));
    if (aa)
        ctx->aa_phase ^= 1;
    else
        ctx->cur = dsti;
    ctx->steps += 1;
    return LBM_OK;
}

lbm_status ensure_graph(lbm_ctx *ctx)
{
    // AB: one graph per starting grid; AA: one graph, starting from the swapped phase.
    const int c = ctx->layout == LBM_LAYOUT_AA ? 0 : ctx->cur;
    if (ctx->graph[c]) return LBM_OK;
    cudaGraph_t graph = nullptr;
    const int64_t l0 = ctx->launches, s0 = ctx->steps;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    lbm_status st = enqueue_step(ctx);
    if (!st) st = enqueue_step(ctx);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (st) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (e != cudaSuccess) return ctx->cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
    ctx->graph_launches[c] = ctx->launches - l0;
    ctx->launches = l0;
    ctx->steps = s0;  // capture did not execute anything
    // cur flipped twice -> back to c
    e = cudaGraphInstantiate(&ctx->graph[c], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        ctx->graph[c] = nullptr;
        return ctx->cuda_fail(e, "cudaGraphInstantiate", __FILE__, __LINE__);
    }
    return LBM_OK;
}

lbm_status enqueue_steps(lbm_ctx *ctx, int64_t n)
{
    lbm_status st;
    const bool graphs = ctx->cfg.use_graphs && !ctx->timing && !kChecked;
    const bool aa = ctx->layout == LBM_LAYOUT_AA;
    while (n > 0) {
        if (graphs && n >= 2 && !(aa && ctx->aa_phase != 0)) {
            if ((st = ensure_graph(ctx))) return st;
            const int gidx = aa ? 0 : ctx->cur;
            CK(cudaGraphLaunch(ctx->graph[gidx], ctx->stream));
            ctx->launches += ctx->graph_launches[gidx];
            ctx->steps += 2;
            n -= 2;
        } else {
            if ((st = enqueue_step(ctx))) return st;
            n -= 1;
        }
    }
    return LBM_OK;
}

lbm_status quiesce(lbm_ctx *ctx)
{
    if (!ctx->direct || ctx->npeers_direct <= 0) return LBM_OK;
    cudaEvent_t ev = ctx->slots[0].ev[12];
    CK(cudaEventRecord(ev, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ev, 0));
    cudaError_t e = launch_wait_peers(ctx->d_inbox, ctx->d_peer_rank, ctx->npeers_direct, ctx->d_epoch,
                                      ctx->d_error, ctx->comm_stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "wait_peers launch", __FILE__, __LINE__);
    ctx->launches += 1;
    CK(cudaStreamSynchronize(ctx->comm_stream));
    CK(cudaStreamSynchronize(ctx->stream));
    int err = 0;
    CK(cudaMemcpy(&err, ctx->d_error, sizeof(int), cudaMemcpyDeviceToHost));
    if (err)
        return ctx->fail(LBM_ERR_INTERNAL,
                         "fused exchange: a peer GPU did not reach the step barrier within LBM_PEER_TIMEOUT_S "
                         "(default 120 s)");
    return LBM_OK;
}

}  // namespace lbm
