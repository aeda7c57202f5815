// setup.cu -- creating a rank's context: patch geometry (SoA with ghost shell,
// P:1095-1124), the sweep box lists, the static ghost-exchange plans (P:287-313,
// both sides derive identical offsets from lbm_plan), flags and the wall table
// (P:482-490), the fused-exchange setup (CUDA IPC of the peers' grids) and the
// direct ghost-store tables; destroy.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <new>

#include "context.h"

namespace lbm {

Geom make_geom(const int n[3], int esize)
{
    Geom g;
    for (int a = 0; a < 3; ++a) g.n[a] = n[a];
    const int se = 32 / esize;                  // elements per 32-B sector
    auto up = [](int64_t v, int64_t m) { return (v + m - 1) / m * m; };
    g.px = (int)up(n[0], se);                   // unpadded rows (= n0 when n0 fills whole sectors)
    g.py = n[1] + 2;
    g.plane = (int64_t)g.px * g.py;
    g.qs = up(g.plane * (n[2] + 2), 32);
    g.gyo = se;                                 // y = 0 on a sector boundary, y = -1 just before it
    g.gy = (int)up(g.gyo + n[1] + 1, se);
    g.gside = (int64_t)g.gy * (n[2] + 2);
    g.gq = 2 * g.gside;
    g.gbase = (int64_t)Q * g.qs;
    g.ps = up(g.gbase + (int64_t)Q * g.gq, 32);
    g.fxo = 4;                                  // even: a cell pair's kinds are one uchar2
    g.fpx = (int)up(g.fxo + n[0] + 1, 4);
    g.fplane = (int64_t)g.fpx * g.py;
    g.fs = g.fplane * (n[2] + 2);
    return g;
}

Box make_box(const lbm_ctx *ctx, int patch, const int lo[3], const int n[3])
{
    Box b;
    b.patch = patch;
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = lo[a];
        b.n[a] = n[a];
    }
    b.tiles_x = (n[0] + ctx->tile_x - 1) / ctx->tile_x;
    b.tiles_y = (n[1] + ctx->tile_y - 1) / ctx->tile_y;
    return b;
}

lbm_status upload_boxes(lbm_ctx *ctx, const std::vector<Box> &boxes, DevBoxes &out)
{
    std::vector<int4> tiles;
    for (const Box &b : boxes) {
        if (b.n[0] <= 0 || b.n[1] <= 0 || b.n[2] <= 0) continue;
        const int xend = b.lo[0] + b.n[0], yend = b.lo[1] + b.n[1];
        for (int z = b.lo[2]; z < b.lo[2] + b.n[2]; ++z)
            for (int ty = 0; ty < b.tiles_y; ++ty)
                for (int tx = 0; tx < b.tiles_x; ++tx)
                    tiles.push_back(make_int4(b.patch, ((b.lo[0] + tx * ctx->tile_x) << 16) | xend,
                                              ((b.lo[1] + ty * ctx->tile_y) << 16) | yend, z));
    }
    out.n = (int)boxes.size();
    out.tiles = (int64_t)tiles.size();
    if (tiles.empty()) return LBM_OK;
    lbm_status st = dev_alloc(ctx, &out.desc, tiles.size() * sizeof(int4));
    if (st) return st;
    CK(upload(ctx, out.desc, tiles.data(), tiles.size() * sizeof(int4)));
    return LBM_OK;
}

void release_boxes(lbm_ctx *ctx, DevBoxes &b)
{
    if (b.desc) {
        cudaFree(b.desc);
        ctx->device_bytes -= (int64_t)(b.tiles * sizeof(int4));
    }
    b = DevBoxes{};
}

lbm_status upload_segs(lbm_ctx *ctx, const std::vector<CopySeg> &v, DevSegs &out)
{
    out.n = (int)v.size();
    out.max_elems = 0;
    out.total_elems = 0;
    for (const CopySeg &s : v) {
        out.max_elems = std::max(out.max_elems, s.nelem);
        out.total_elems += s.nelem;
    }
    if (v.empty()) return LBM_OK;
    lbm_status st = dev_alloc(ctx, &out.segs, v.size() * sizeof(CopySeg));
    if (st) return st;
    CK(upload(ctx, out.segs, v.data(), v.size() * sizeof(CopySeg)));
    return LBM_OK;
}

CopySeg grid_to_x(const lbm_ctx *ctx, const Seg &s, bool to_buffer, int64_t buf_base)
{
    // Source: the sender's boundary layer (a local patch); destination: either
    // the receiver's ghost layer (local copy) or the send buffer.
    CopySeg c;
    std::memset(&c, 0, sizeof c);
    const int lsend = ctx->dec.global_to_local(s.send_patch);
    c.src_base = (int64_t)lsend * ctx->g.ps;
    c.src_is_buf = 0;
    for (int a = 0; a < 3; ++a) {
        c.src_lo[a] = s.send_lo[a];
        c.dst_lo[a] = s.recv_lo[a];
        c.size[a] = s.size[a];
    }
    c.nq = s.nq;
    for (int i = 0; i < 5; ++i) c.q[i] = i < s.nq ? s.q[i] : 0;
    c.cells = s.cells;
    c.nelem = (int64_t)s.nq * s.cells;
    if (to_buffer) {
        c.dst_is_buf = 1;
        c.dst_base = buf_base + s.offset;
    } else {
        const int lrecv = ctx->dec.global_to_local(s.recv_patch);
        c.dst_is_buf = 0;
        c.dst_base = (int64_t)lrecv * ctx->g.ps;
        c.dst_flag_base = (int64_t)lrecv * ctx->g.fs;
    }
    return c;
}

CopySeg buffer_to_grid(const lbm_ctx *ctx, const Seg &s, int64_t buf_base)
{
    CopySeg c;
    std::memset(&c, 0, sizeof c);
    const int lrecv = ctx->dec.global_to_local(s.recv_patch);
    c.src_is_buf = 1;
    c.src_base = buf_base + s.offset;
    c.dst_is_buf = 0;
    c.dst_base = (int64_t)lrecv * ctx->g.ps;
    c.dst_flag_base = (int64_t)lrecv * ctx->g.fs;
    for (int a = 0; a < 3; ++a) {
        c.dst_lo[a] = s.recv_lo[a];
        c.size[a] = s.size[a];
    }
    c.nq = s.nq;
    for (int i = 0; i < 5; ++i) c.q[i] = i < s.nq ? s.q[i] : 0;
    c.cells = s.cells;
    c.nelem = (int64_t)s.nq * s.cells;
    return c;
}

// Exchange plan of one kind: peers, message offsets, device copy descriptors.
lbm_status setup_exset(lbm_ctx *ctx, int kind, bool upload)
{
    ExSet &X = ctx->ex[kind];
    build_segments(ctx->dec, X.segs, kind);
    std::vector<Peer> peers;
    auto peer_of = [&](int r) -> Peer & {
        for (Peer &p : peers)
            if (p.rank == r) return p;
        peers.push_back(Peer{r, 0, 0, 0, 0});
        return peers.back();
    };
    for (const Seg &s : X.segs.send) peer_of(s.peer).send_n += (int64_t)s.nq * s.cells;
    for (const Seg &s : X.segs.recv) peer_of(s.peer).recv_n += (int64_t)s.nq * s.cells;
    std::sort(peers.begin(), peers.end(), [](const Peer &a, const Peer &b) { return a.rank < b.rank; });
    int64_t so = 0, ro = 0;
    for (Peer &p : peers) {
        p.send_off = so;
        p.recv_off = ro;
        so += p.send_n;
        ro += p.recv_n;
    }
    X.peers = peers;
    X.send_elems = so;
    X.recv_elems = ro;
    X.has_remote = so > 0 || ro > 0;
    X.has_nccl = false;
    for (const Peer &p : peers)
        if (p.rank != ctx->dec.rank) X.has_nccl = true;
    if (!upload) return LBM_OK;

    auto peer_send_off = [&](int r) {
        for (const Peer &p : peers)
            if (p.rank == r) return p.send_off;
        return (int64_t)0;
    };
    auto peer_recv_off = [&](int r) {
        for (const Peer &p : peers)
            if (p.rank == r) return p.recv_off;
        return (int64_t)0;
    };
    auto tag = [&](CopySeg c, const Seg &s) {
        c.mask = kind == EX_AA2 ? 2 : 0;
        for (int a = 0; a < 3; ++a) c.d[a] = s.d[a];
        return c;
    };
    std::vector<CopySeg> pack_all, pack_remote, local, unpack;
    for (const Seg &s : X.segs.send) {
        CopySeg c = tag(grid_to_x(ctx, s, true, peer_send_off(s.peer)), s);
        pack_all.push_back(c);
        pack_remote.push_back(c);
    }
    for (const Seg &s : X.segs.local) {
        CopySeg c = tag(grid_to_x(ctx, s, false, 0), s);
        pack_all.push_back(c);
        local.push_back(c);
    }
    for (const Seg &s : X.segs.recv) unpack.push_back(tag(buffer_to_grid(ctx, s, peer_recv_off(s.peer)), s));
    lbm_status st;
    if ((st = upload_segs(ctx, pack_all, X.pack_all))) return st;
    if ((st = upload_segs(ctx, pack_remote, X.pack_remote))) return st;
    if ((st = upload_segs(ctx, local, X.local_copy))) return st;
    if ((st = upload_segs(ctx, unpack, X.unpack))) return st;
    X.h_pack_all = pack_all;
    X.h_local = local;
    X.h_unpack = unpack;
    return LBM_OK;
}

// After set_flags: a grid-destination segment whose destination cells are all
// fluid needs no per-element flag check (mask 1).  The checks are half the DRAM
// reads of the copy kernel on strided x faces (profiles/r01_ncu_copy_*).
lbm_status update_seg_masks(lbm_ctx *ctx, const uint8_t *gflags)
{
    const Decomp &d = ctx->dec;
    const int64_t NX = d.domain[0], NY = d.domain[1], NZ = d.domain[2];
    auto all_fluid = [&](const CopySeg &c) {
        const int l = (int)(c.dst_base / ctx->g.ps);
        int pc[3];
        d.patch_coord(d.local_to_global(l), pc);
        for (int z = 0; z < c.size[2]; ++z)
            for (int y = 0; y < c.size[1]; ++y)
                for (int x = 0; x < c.size[0]; ++x) {
                    int64_t gc[3] = {(int64_t)pc[0] * d.patch[0] + c.dst_lo[0] + x,
                                     (int64_t)pc[1] * d.patch[1] + c.dst_lo[1] + y,
                                     (int64_t)pc[2] * d.patch[2] + c.dst_lo[2] + z};
                    const int64_t N[3] = {NX, NY, NZ};
                    for (int a = 0; a < 3; ++a)
                        if (d.periodic[a]) gc[a] = (gc[a] % N[a] + N[a]) % N[a];
                    if (gflags[((gc[2] + 1) * (NY + 2) + (gc[1] + 1)) * (NX + 2) + (gc[0] + 1)] != 0) return false;
                }
        return true;
    };
    for (int k = 0; k < 3; ++k) {
        ExSet &X = ctx->ex[k];
        if (k == EX_AA2) continue;  // its mask also involves the writer cells
        std::vector<CopySeg> *hv[3] = {&X.h_pack_all, &X.h_local, &X.h_unpack};
        DevSegs *dv[3] = {&X.pack_all, &X.local_copy, &X.unpack};
        for (int j = 0; j < 3; ++j) {
            std::vector<CopySeg> &v = *hv[j];
            if (v.empty() || !dv[j]->segs) continue;
            for (CopySeg &c : v)
                if (!c.dst_is_buf) c.mask = all_fluid(c) ? 1 : 0;
            CK(upload(ctx, dv[j]->segs, v.data(), v.size() * sizeof(CopySeg)));
        }
    }
    return LBM_OK;
}

// One bounce-back list (launch_bb_list_count / _write): the kind-1 cells, minus the
// links the two-grid sweep stores itself when sidewall is given.
static lbm_status build_list(lbm_ctx *ctx, const unsigned long long *sidewall, BbEntry **list, int64_t *len)
{
    if (*list) {
        cudaFree(*list);
        ctx->device_bytes -= *len * (int64_t)sizeof(BbEntry);
        *list = nullptr;
    }
    *len = 0;
    const int64_t total = (int64_t)ctx->dec.nlocal * ctx->g.fs;
    const int64_t nch = bb_list_chunks(total);
    int64_t *d_counts = nullptr;
    lbm_status st = dev_alloc(ctx, &d_counts, (size_t)std::max<int64_t>(nch, 1) * sizeof(int64_t));
    if (st) return st;
    std::vector<int64_t> counts((size_t)nch);
    cudaError_t e = launch_bb_list_count(ctx->kind, ctx->wmask, sidewall, total, ctx->g, d_counts, ctx->stream);
    if (e == cudaSuccess && nch > 0)
        e = cudaMemcpyAsync(counts.data(), d_counts, nch * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    int64_t n = 0;
    for (int64_t &c : counts) {
        const int64_t t = c;
        c = n;
        n += t;
    }
    if (e == cudaSuccess && n > 0 && !(st = dev_alloc(ctx, list, (size_t)n * sizeof(BbEntry)))) {
        *len = n;
        e = upload(ctx, d_counts, counts.data(), nch * sizeof(int64_t));
        if (e == cudaSuccess)
            e = launch_bb_list_write(ctx->kind, ctx->wmask, ctx->flags, sidewall, total, ctx->g, d_counts, *list,
                                     ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    }
    cudaFree(d_counts);
    ctx->device_bytes -= std::max<int64_t>(nch, 1) * (int64_t)sizeof(int64_t);
    if (st) return st;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "build bounce-back list", __FILE__, __LINE__);
    ctx->launches += 2;
    return LBM_OK;
}

lbm_status build_wall_lists(lbm_ctx *ctx)
{
    // The captured step graphs hold the old lists' pointers and lengths: drop them
    // (the next multi-step call re-captures).
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 2; ++i)
        if (ctx->graph[i]) {
            cudaGraphExecDestroy(ctx->graph[i]);
            ctx->graph[i] = nullptr;
        }
    // Patch sides that are a uniform wall: the sweeps' face lanes store the
    // bounce-back of the face's inner cells' links through it, the per-step list
    // leaves them out; the full list (every link) serves the fills after set_pdfs /
    // set_flags.
    lbm_status st;
    CK(launch_sidewall(ctx->flags, ctx->dec.nlocal, ctx->g, ctx->sidewall, ctx->stream));
    if ((st = build_list(ctx, nullptr, &ctx->bb_full, &ctx->bb_full_n))) return st;
    if ((st = build_list(ctx, ctx->sidewall, &ctx->bb_list, &ctx->bb_n))) return st;
    cudaError_t e = cudaSuccess;
    for (DevBoxes *b : {&ctx->box_all, &ctx->box_shell, &ctx->box_interior})
        if (e == cudaSuccess) e = launch_tile_solid(b->desc, b->tiles, ctx->kind, ctx->sidewall, ctx->g, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "build wall lists", __FILE__, __LINE__);
    ctx->launches += 4;
    return LBM_OK;
}

// Sweep boxes.  all: one box per local patch.  Overlap: for patches with
// remote segments, a shell on every side a remote segment touches (1 cell
// thick in y/z; SWEEP_BX thick in x so the shell rows stay coalesced) and the
// remaining interior box.  whole_x (fused exchange): a patch with a remote x
// side goes into the shell set whole -- an x slab splits every row between
// two concurrently running kernels, which cost 9 % at 256^3 fp64 on a 2x1x1
// process grid (row reads lose their DRAM page locality), while the fused
// exchange has no transfer to hide behind the interior sweep.
lbm_status build_boxes(lbm_ctx *ctx, bool whole_x)
{
    std::vector<Box> all, shell, interior;
    const int *n = ctx->g.n;
    const int zero[3] = {0, 0, 0};
    std::vector<int> side(6 * ctx->dec.nlocal, 0);
    for (const Seg &s : ctx->ex[EX_AB].segs.send) {
        const int l = ctx->dec.global_to_local(s.send_patch);
        // s.d is the direction from the receiver to this (sending) patch; the
        // sender's boundary layer is on side -s.d.
        for (int a = 0; a < 3; ++a) {
            if (s.d[a] == -1) side[6 * l + 2 * a + 1] = 1;  // high side of axis a
            if (s.d[a] == 1) side[6 * l + 2 * a + 0] = 1;   // low side
        }
    }
    for (int l = 0; l < ctx->dec.nlocal; ++l) {
        all.push_back(make_box(ctx, l, zero, n));
        bool any = false;
        for (int k = 0; k < 6; ++k) any = any || side[6 * l + k];
        if (!any) {
            interior.push_back(make_box(ctx, l, zero, n));
            continue;
        }
        if (whole_x && (side[6 * l] || side[6 * l + 1])) {
            shell.push_back(make_box(ctx, l, zero, n));
            continue;
        }
        int th[6];
        for (int a = 0; a < 3; ++a) {
            const int t = a == 0 ? ctx->tile_x : 1;
            th[2 * a] = side[6 * l + 2 * a] ? std::min(t, n[a]) : 0;
            th[2 * a + 1] = side[6 * l + 2 * a + 1] ? std::min(t, n[a] - th[2 * a]) : 0;
        }
        int lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = th[2 * a];
            hi[a] = n[a] - th[2 * a + 1];
        }
        // Every box starts on an even x (cell pairs) and a 16-cell boundary in x
        // (whole 64-B chunks for fp32): round the high-x shell start down.
        const int xa = 16;
        hi[0] = std::max(lo[0], hi[0] / xa * xa);
        // z slabs (full xy), then y slabs (full x, inner z), then x slabs (inner y, z)
        auto add = [&](int x0, int x1, int y0, int y1, int z0, int z1) {
            if (x1 <= x0 || y1 <= y0 || z1 <= z0) return;
            int blo[3] = {x0, y0, z0}, bn[3] = {x1 - x0, y1 - y0, z1 - z0};
            shell.push_back(make_box(ctx, l, blo, bn));
        };
        add(0, n[0], 0, n[1], 0, lo[2]);
        add(0, n[0], 0, n[1], hi[2], n[2]);
        add(0, n[0], 0, lo[1], lo[2], hi[2]);
        add(0, n[0], hi[1], n[1], lo[2], hi[2]);
        add(0, lo[0], lo[1], hi[1], lo[2], hi[2]);
        add(hi[0], n[0], lo[1], hi[1], lo[2], hi[2]);
        if (hi[0] > lo[0] && hi[1] > lo[1] && hi[2] > lo[2]) {
            int bn[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
            interior.push_back(make_box(ctx, l, lo, bn));
        }
    }
    for (DevBoxes *b : {&ctx->box_all, &ctx->box_shell, &ctx->box_interior}) release_boxes(ctx, *b);
    lbm_status st;
    if ((st = upload_boxes(ctx, all, ctx->box_all))) return st;
    if ((st = upload_boxes(ctx, shell, ctx->box_shell))) return st;
    if ((st = upload_boxes(ctx, interior, ctx->box_interior))) return st;
    if (ctx->flags_set && (st = build_wall_lists(ctx))) return st;
    return LBM_OK;
}

// Build the exchange plans, message buffers and sweep boxes.
lbm_status setup_exchange(lbm_ctx *ctx)
{
    const bool aa = ctx->layout == LBM_LAYOUT_AA;
    lbm_status st;
    if ((st = setup_exset(ctx, EX_AB, !aa))) return st;
    if ((st = setup_exset(ctx, EX_AA1, aa))) return st;
    if ((st = setup_exset(ctx, EX_AA2, aa))) return st;
    int64_t so = 0, ro = 0;
    for (int k = 0; k < 3; ++k) {
        so = std::max(so, ctx->ex[k].send_elems);
        ro = std::max(ro, ctx->ex[k].recv_elems);
    }
    ctx->has_remote = ctx->ex[EX_AB].has_remote;
    ctx->has_nccl = ctx->ex[EX_AB].has_nccl;
    if ((st = dev_alloc(ctx, &ctx->sendbuf, (size_t)so * ctx->esize))) return st;
    if ((st = dev_alloc(ctx, &ctx->recvbuf, (size_t)ro * ctx->esize))) return st;

    if ((st = build_boxes(ctx, false))) return st;
    // Shells first, transport overlapped with the interiors, whenever anything
    // goes through the buffers -- also a one-GPU FORCE_BUFFERS run, whose
    // self-peer messages travel through a one-rank NCCL communicator.
    ctx->use_overlap = ctx->cfg.overlap && ctx->has_remote;
    return LBM_OK;
}

lbm_status apply_flags(lbm_ctx *ctx, const uint8_t *flags, const double *wall_u, int nvel)
{
    const int64_t nx = ctx->dec.domain[0], ny = ctx->dec.domain[1], nz = ctx->dec.domain[2];
    const size_t total = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
    uint8_t *dflags = nullptr;
    lbm_status st = dev_alloc(ctx, &dflags, total);
    if (st) return st;
    cudaError_t e = upload(ctx, dflags, flags, total);
    if (e == cudaSuccess)
        e = launch_build_flags(dflags, ctx->dec.domain, ctx->dec.periodic, ctx->d_origin, ctx->dec.nlocal, ctx->g,
                               ctx->flags, ctx->kind, ctx->wmask, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(dflags);
    ctx->device_bytes -= (int64_t)total;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "build flags", __FILE__, __LINE__);
    ctx->launches += 2 * ((ctx->dec.nlocal + 65534) / 65535);
    // Wall correction table 6 w_i rho0 (e_i . u_w[k]) (R3, R9),
    // computed in double and rounded once to the storage precision.
    std::vector<double> cd((size_t)LBM_MAX_WALL_VELOCITIES * Q, 0.0);
    for (int k = 0; k < nvel; ++k)
        for (int i = 0; i < Q; ++i) {
            const double eu = EX(i) * wall_u[3 * k] + EY(i) * wall_u[3 * k + 1] + EZ(i) * wall_u[3 * k + 2];
            cd[(size_t)k * Q + i] = 6.0 * WQ(i) * 1.0 * eu;
        }
    if (ctx->esize == 8) {
        CK(upload(ctx, ctx->corr, cd.data(), cd.size() * sizeof(double)));
    } else {
        std::vector<float> cf(cd.begin(), cd.end());
        CK(upload(ctx, ctx->corr, cf.data(), cf.size() * sizeof(float)));
    }
    {
        lbm_status st2 = update_seg_masks(ctx, flags);
        if (st2) return st2;
    }
    // Fluid cell counts (MFLUPS counts fluid cells, R16).
    int64_t gl = 0, lo = 0;
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y) {
            const uint8_t *row = flags + ((z + 1) * (ny + 2) + (y + 1)) * (nx + 2) + 1;
            const bool zy_owned = z >= ctx->dec.owned_lo[2] && z < ctx->dec.owned_hi[2] && y >= ctx->dec.owned_lo[1] &&
                                  y < ctx->dec.owned_hi[1];
            for (int64_t x = 0; x < nx; ++x) {
                if (row[x] == 0) {
                    ++gl;
                    if (zy_owned && x >= ctx->dec.owned_lo[0] && x < ctx->dec.owned_hi[0]) ++lo;
                }
            }
        }
    ctx->fluid_global = gl;
    ctx->fluid_local = lo;
    ctx->flags_set = true;
    return build_wall_lists(ctx);
}

const char *validate_flags(const Decomp &dec, const uint8_t *flags, const double *wall_u, int nvel)
{
    static thread_local char msg[256];
    if (!flags) return "flags is NULL";
    if (nvel < 0 || nvel > LBM_MAX_WALL_VELOCITIES) return "nvel must be in [0, 254]";
    if (nvel > 0 && !wall_u) return "wall_u is NULL but nvel > 0";
    for (int k = 0; k < 3 * nvel; ++k)
        if (!std::isfinite(wall_u[k])) return "wall_u must be finite";
    const int64_t nx = dec.domain[0], ny = dec.domain[1], nz = dec.domain[2];
    for (int64_t z = -1; z <= nz; ++z)
        for (int64_t y = -1; y <= ny; ++y) {
            const uint8_t *row = flags + ((z + 1) * (ny + 2) + (y + 1)) * (nx + 2);
            const bool yz_shell = (!dec.periodic[1] && (y < 0 || y >= ny)) || (!dec.periodic[2] && (z < 0 || z >= nz));
            for (int64_t x = -1; x <= nx; ++x) {
                const uint8_t f = row[x + 1];
                const bool shell = yz_shell || (!dec.periodic[0] && (x < 0 || x >= nx));
                if (shell && f == LBM_FLUID) {
                    std::snprintf(msg, sizeof msg, "shell cell (%lld,%lld,%lld) on a non-periodic axis is fluid",
                                  (long long)x, (long long)y, (long long)z);
                    return msg;
                }
                if (f >= LBM_VELOCITY0 && f - LBM_VELOCITY0 >= nvel) {
                    std::snprintf(msg, sizeof msg, "cell (%lld,%lld,%lld) has velocity wall %d but nvel = %d",
                                  (long long)x, (long long)y, (long long)z, f - LBM_VELOCITY0, nvel);
                    return msg;
                }
            }
        }
    return "";
}

void destroy_ctx(lbm_ctx *ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    // Fused exchange: peers may still be storing into this rank's grid and inbox
    // (their last step); wait for them before freeing (best effort: a poisoned
    // context skips it, a dead peer times out).
    if (!ctx->poisoned) quiesce(ctx);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
    for (int i = 0; i < 2; ++i)
        if (ctx->graph[i]) cudaGraphExecDestroy(ctx->graph[i]);
    if (ctx->nccl) ncclCommDestroy(ctx->nccl);
    for (void *p : ctx->ipc_mapped) cudaIpcCloseMemHandle(p);
    for (void *p : {(void *)ctx->d_mass, (void *)ctx->d_dnbr, (void *)ctx->d_epoch, (void *)ctx->d_inbox,
                    (void *)ctx->d_peer_inbox, (void *)ctx->d_peer_rank, (void *)ctx->d_error})
        if (p) cudaFree(p);
    for (ExSet &X : ctx->ex)
        for (void *p : {(void *)X.pack_all.segs, (void *)X.pack_remote.segs, (void *)X.local_copy.segs,
                        (void *)X.unpack.segs})
            if (p) cudaFree(p);
    void *ptrs[] = {ctx->grid[0], ctx->grid[1], ctx->flags, ctx->kind, ctx->wmask, ctx->corr, ctx->d_origin, ctx->sendbuf,
                    ctx->recvbuf,
                    ctx->box_all.desc, ctx->box_shell.desc, ctx->box_interior.desc, ctx->bb_list, ctx->bb_full,
                    ctx->sidewall
#ifdef LBM_CHECKED
                    , ctx->chk.wr, ctx->chk.rd, ctx->chk.err
#endif
    };
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (ctx->events_created)
        for (auto &sl : ctx->slots)
            for (auto &ev : sl.ev) cudaEventDestroy(ev);
    for (int b = 0; b < 2; ++b) {
        if (ctx->xstage[b]) cudaFree(ctx->xstage[b]);
        if (ctx->xev_copy[b]) cudaEventDestroy(ctx->xev_copy[b]);
        if (ctx->xev_kern[b]) cudaEventDestroy(ctx->xev_kern[b]);
    }
    if (ctx->xstream) cudaStreamDestroy(ctx->xstream);
    if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    cudaGetLastError();
    delete ctx;
}

// Fused-exchange setup: neighbour pointer table, epoch / inbox buffers and,
// across GPUs, the CUDA IPC mapping of the peers' grids and inboxes (handles
// all-gathered over the NCCL communicator).  All ranks agree on the outcome.
lbm_status setup_direct(lbm_ctx *ctx)
{
    const Decomp &dec = ctx->dec;
    const int R = dec.nranks, me = dec.rank;
    lbm_status st;
    if ((st = dev_alloc(ctx, &ctx->d_epoch, sizeof(unsigned long long)))) return st;
    if ((st = dev_alloc(ctx, &ctx->d_inbox, (size_t)R * sizeof(unsigned long long)))) return st;
    if ((st = dev_alloc(ctx, &ctx->d_error, sizeof(int)))) return st;
    CK(memset_sync(ctx, ctx->d_epoch, 0, sizeof(unsigned long long)));
    CK(memset_sync(ctx, ctx->d_inbox, 0, (size_t)R * sizeof(unsigned long long)));
    CK(memset_sync(ctx, ctx->d_error, 0, sizeof(int)));
    // Remote peers of the exchange plan.  exchange_mode SELF_PEER (one GPU): this
    // rank is its own peer -- every neighbour patch is reached through the peer
    // table and the epoch handshake exactly as across GPUs, with its own grid and
    // inbox in place of IPC-mapped ones.
    const bool self = ctx->cfg.exchange_mode == LBM_EXCHANGE_SELF_PEER;
    std::vector<int> peers;
    for (const Peer &p : ctx->ex[EX_AB].peers)
        if (p.rank != me || self) peers.push_back(p.rank);
    if (peers.empty()) return LBM_OK;  // nothing crosses a GPU boundary: copy path
    std::vector<void *> peer_grid((size_t)R * 2, nullptr), peer_inbox((size_t)R, nullptr);
    if (self) {
        const bool aa = ctx->layout == LBM_LAYOUT_AA;
        peer_grid[(size_t)2 * me] = ctx->grid[0];
        peer_grid[(size_t)2 * me + 1] = ctx->grid[aa ? 0 : 1];
        peer_inbox[me] = ctx->d_inbox;
    } else {
        // all-gather {grid0, grid1, inbox} IPC handles
        const size_t hb = sizeof(cudaIpcMemHandle_t);
        std::vector<cudaIpcMemHandle_t> mine(3);
        // the AA layout has one grid: its handle travels in both slots, opened once
        const bool aa = ctx->layout == LBM_LAYOUT_AA;
        CK(cudaIpcGetMemHandle(&mine[0], ctx->grid[0]));
        CK(cudaIpcGetMemHandle(&mine[1], ctx->grid[aa ? 0 : 1]));
        CK(cudaIpcGetMemHandle(&mine[2], ctx->d_inbox));
        char *dbuf = nullptr;
        if ((st = dev_alloc(ctx, &dbuf, 3 * hb * (size_t)(R + 1)))) return st;
        CK(upload(ctx, dbuf, mine.data(), 3 * hb));
        NK(ncclAllGather(dbuf, dbuf + 3 * hb, 3 * hb, ncclUint8, ctx->nccl, ctx->stream));
        std::vector<cudaIpcMemHandle_t> all((size_t)3 * R);
        CK(cudaMemcpyAsync(all.data(), dbuf + 3 * hb, 3 * hb * R, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(dbuf);
        ctx->device_bytes -= (int64_t)(3 * hb * (size_t)(R + 1));
        int ok = 1;
        for (int r : peers) {
            for (int i = 0; i < 3 && ok; ++i) {
                if (aa && i == 1) {
                    peer_grid[(size_t)2 * r + 1] = peer_grid[(size_t)2 * r];
                    continue;
                }
                void *ptr = nullptr;
                if (cudaIpcOpenMemHandle(&ptr, all[(size_t)3 * r + i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    ok = 0;
                    break;
                }
                ctx->ipc_mapped.push_back(ptr);
                if (i < 2)
                    peer_grid[(size_t)2 * r + i] = ptr;
                else
                    peer_inbox[r] = ptr;
            }
        }
        // every rank must take the same path
        int *dok = nullptr;
        if ((st = dev_alloc(ctx, &dok, sizeof(int)))) return st;
        CK(upload(ctx, dok, &ok, sizeof(int)));
        NK(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, ctx->nccl, ctx->stream));
        CK(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(dok);
        ctx->device_bytes -= (int64_t)sizeof(int);
        if (!ok) return LBM_OK;  // stay on the NCCL exchange
    }
    // neighbour table
    const int nl = dec.nlocal;
    std::vector<void *> nbr((size_t)nl * NDIR * 2, nullptr);
    for (int l = 0; l < nl; ++l) {
        const int gpatch = dec.local_to_global(l);
        for (int k = 0; k < NDIR; ++k) {
            const int nbp = neighbour(dec, gpatch, kDirs[k].d);
            if (nbp < 0) continue;
            const int r = dec.owner(nbp);
            if (r == me && !self) continue;  // same-GPU neighbours: direct stores / ghost copies
            const int64_t off = (int64_t)dec.local_index_on_owner(nbp) * ctx->g.ps * ctx->esize;
            for (int i = 0; i < 2; ++i) {
                char *base = (char *)peer_grid[(size_t)2 * r + i];
                nbr[((size_t)l * NDIR + k) * 2 + i] = base + off;
            }
        }
    }
    ctx->h_nbr = nbr;
    std::vector<unsigned long long *> pin;
    std::vector<int> prank;
    for (int r : peers) {
        pin.push_back((unsigned long long *)peer_inbox[r] + me);
        prank.push_back(r);
    }
    ctx->npeers_direct = (int)peers.size();
    if (!peers.empty()) {
        if ((st = dev_alloc(ctx, &ctx->d_peer_inbox, pin.size() * sizeof(void *)))) return st;
        CK(upload(ctx, ctx->d_peer_inbox, pin.data(), pin.size() * sizeof(void *)));
        if ((st = dev_alloc(ctx, &ctx->d_peer_rank, prank.size() * sizeof(int)))) return st;
        CK(upload(ctx, ctx->d_peer_rank, prank.data(), prank.size() * sizeof(int)));
    }
    ctx->direct = true;
    return LBM_OK;
}

lbm_status create_impl(const lbm_config *cfg, lbm_ctx **out)
{
    if (!out) return LBM_ERR_ARG;
    *out = nullptr;
    if (!cfg) {
        g_create_error = "cfg is NULL";
        return LBM_ERR_ARG;
    }
    Decomp dec;
    const char *m = decompose(*cfg, dec);
    if (m[0]) {
        g_create_error = m;
        return LBM_ERR_ARG;
    }
    if (cfg->nranks > 1 && !cfg->nccl_unique_id) {
        g_create_error = "nccl_unique_id is required when nranks > 1";
        return LBM_ERR_ARG;
    }
    lbm_ctx *ctx = new (std::nothrow) lbm_ctx();
    if (!ctx) {
        g_create_error = "host allocation failed";
        return LBM_ERR_OOM;
    }
    ctx->cfg = *cfg;
    ctx->dec = dec;
    ctx->esize = cfg->precision;
    ctx->layout = cfg->layout;
    if (const char *a = std::getenv("LBM_SWEEP_VARIANT")) {  // occupancy alternative (tools/sweep_tune.py)
        const int v = std::atoi(a);
        if (v >= 0 && v < kSweepVariants) ctx->sweep_variant = v;
    }
    auto bail = [&](lbm_status st) {
        g_create_error = ctx->err.empty() ? "create failed" : ctx->err;
        destroy_ctx(ctx);
        return st;
    };
    // Device
    int dev = cfg->device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) {
            ctx->err = std::string("no CUDA device: ") + cudaGetErrorString(e);
            return bail(LBM_ERR_CUDA);
        }
    }
    ctx->device = dev;
    {
        cudaError_t e = cudaSetDevice(dev);
        cudaDeviceProp prop;
        if (e == cudaSuccess) e = cudaGetDeviceProperties(&prop, dev);
        if (e != cudaSuccess) {
            ctx->err = std::string("cannot use CUDA device: ") + cudaGetErrorString(e);
            cudaGetLastError();
            return bail(LBM_ERR_CUDA);
        }
        if (prop.major != 10 || prop.minor != 0) {
            ctx->err = "liblbm_b200 is built for sm_100a (B200); device " + std::to_string(dev) + " is " +
                       std::string(prop.name) + " (sm_" + std::to_string(prop.major) + std::to_string(prop.minor) + ")";
            return bail(LBM_ERR_CUDA);
        }
    }
    ctx->g = make_geom(dec.patch, ctx->esize);
    lbm_status st;
    // Streams and events
    if (cfg->stream) {
        ctx->stream = (cudaStream_t)cfg->stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            ctx->err = "cudaStreamCreate failed";
            return bail(LBM_ERR_CUDA);
        }
        ctx->own_stream = true;
    }
    {
        // The exchange stream gets the highest priority so the NCCL / unpack
        // blocks are scheduled ahead of the interior sweep they overlap with.
        int lo_prio = 0, hi_prio = 0;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        if (cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, hi_prio) != cudaSuccess) {
            ctx->err = "cudaStreamCreate failed";
            return bail(LBM_ERR_CUDA);
        }
    }
    for (auto &sl : ctx->slots)
        for (auto &ev : sl.ev)
            if (cudaEventCreate(&ev) != cudaSuccess) {
                ctx->err = "cudaEventCreate failed";
                return bail(LBM_ERR_CUDA);
            }
    ctx->events_created = true;
    // Memory budget check (clean OOM before the big allocations).
    const size_t grid_bytes = (size_t)dec.nlocal * ctx->g.ps * ctx->esize;
    const size_t flag_bytes = (size_t)dec.nlocal * ctx->g.fs;
    const int ngrids = ctx->layout == LBM_LAYOUT_AA ? 1 : 2;
    {
        size_t freeb = 0, totalb = 0;
        if (cudaMemGetInfo(&freeb, &totalb) == cudaSuccess && ngrids * grid_bytes + 2 * flag_bytes > freeb) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "need %.2f GB of device memory for the PDF grid(s) and flags, %.2f GB free",
                          ((double)ngrids * grid_bytes + 2.0 * flag_bytes) / 1e9, freeb / 1e9);
            ctx->err = buf;
            return bail(LBM_ERR_OOM);
        }
    }
    for (int i = 0; i < ngrids; ++i) {
        if ((st = dev_alloc(ctx, &ctx->grid[i], grid_bytes))) return bail(st);
        if (cudaMemsetAsync(ctx->grid[i], 0, grid_bytes, ctx->stream) != cudaSuccess) return bail(LBM_ERR_CUDA);
    }
    if ((st = chk_alloc(ctx, grid_bytes))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->sidewall, (size_t)dec.nlocal * sizeof(unsigned long long)))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->flags, flag_bytes))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->kind, flag_bytes))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->wmask, flag_bytes * sizeof(uint32_t)))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->corr, (size_t)LBM_MAX_WALL_VELOCITIES * Q * ctx->esize))) return bail(st);
    {
        std::vector<int> origin(3 * dec.nlocal);
        for (int l = 0; l < dec.nlocal; ++l) {
            int c[3];
            dec.patch_coord(dec.local_to_global(l), c);
            for (int a = 0; a < 3; ++a) origin[3 * l + a] = c[a] * dec.patch[a];
        }
        if ((st = dev_alloc(ctx, &ctx->d_origin, origin.size() * sizeof(int)))) return bail(st);
        if (upload(ctx, ctx->d_origin, origin.data(), origin.size() * sizeof(int)) !=
            cudaSuccess)
            return bail(LBM_ERR_CUDA);
    }
    {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
            ctx->num_sms = sms;
    }
    if ((st = setup_exchange(ctx))) return bail(st);
    // NCCL communicator (bootstrap id broadcast by the caller, e.g. torch.distributed).
    // One GPU with FORCE_BUFFERS: a one-rank communicator, so the self-peer
    // messages take the grouped ncclSend / ncclRecv path of P:287-313.
    if (cfg->nranks > 1 || (ctx->has_remote && cfg->exchange_mode == LBM_EXCHANGE_FORCE_BUFFERS)) {
        ncclUniqueId id;
        if (cfg->nranks > 1) {
            std::memcpy(&id, cfg->nccl_unique_id, sizeof id);
        } else if (ncclGetUniqueId(&id) != ncclSuccess) {
            ctx->err = "ncclGetUniqueId failed";
            return bail(LBM_ERR_NCCL);
        }
        ncclResult_t r = ncclCommInitRank(&ctx->nccl, cfg->nranks, id, cfg->rank);
        if (r != ncclSuccess) {
            ctx->nccl = nullptr;
            ctx->err = std::string("ncclCommInitRank failed: ") + ncclGetErrorString(r);
            return bail(LBM_ERR_NCCL);
        }
    }
    // Fused exchange across GPUs (and with exchange_mode SELF_PEER on one GPU)
    // unless the NCCL path is requested (exchange_mode FORCE_BUFFERS, or env
    // LBM_EXCHANGE=nccl).
    const bool aa = ctx->layout == LBM_LAYOUT_AA;
    {
        const char *ev = std::getenv("LBM_EXCHANGE");
        const bool want = cfg->exchange_mode != LBM_EXCHANGE_FORCE_BUFFERS && !(ev && std::string(ev) == "nccl");
        if (want && (st = setup_direct(ctx))) return bail(st);
    }
    {
        // Direct ghost stores by the x2 sweeps: face / edge cells write their
        // outgoing PDFs straight into the neighbour patches' ghost layers.
        // (1) same-GPU neighbours, replacing the ghost copies after the sweep
        //     (default; LBM_LOCAL_DIRECT=0 keeps the copies);
        // (2) with the fused exchange, the shells facing other GPUs store
        //     through the peer-mapped table.
        const char *ev = std::getenv("LBM_LOCAL_DIRECT");
        const bool on = ev ? std::string(ev) != "0" : true;
        const bool want_local = on && cfg->exchange_mode == LBM_EXCHANGE_AUTO && !ctx->ex[EX_AB].segs.local.empty();
        const bool want_shell = ctx->direct;
        if (want_local || want_shell) {
            std::vector<void *> tab = ctx->direct ? ctx->h_nbr : std::vector<void *>((size_t)dec.nlocal * NDIR * 2, nullptr);
            for (int l = 0; l < dec.nlocal && want_local; ++l) {
                const int gp = dec.local_to_global(l);
                for (int k = 0; k < NDIR; ++k) {
                    const int nbp = neighbour(dec, gp, kDirs[k].d);
                    if (nbp < 0 || dec.owner(nbp) != dec.rank) continue;
                    const int64_t off = (int64_t)dec.local_index_on_owner(nbp) * ctx->g.ps * ctx->esize;
                    for (int i = 0; i < 2; ++i)  // AA: one grid
                        tab[((size_t)l * NDIR + k) * 2 + i] = (char *)ctx->grid[aa ? 0 : i] + off;
                }
            }
            if ((st = dev_alloc(ctx, &ctx->d_dnbr, tab.size() * sizeof(void *)))) return bail(st);
            if (upload(ctx, ctx->d_dnbr, tab.data(), tab.size() * sizeof(void *)) != cudaSuccess)
                return bail(LBM_ERR_CUDA);
            ctx->ldirect = want_local;
        }
    }
    // fused exchange: patches with a remote x side are swept whole (build_boxes)
    if (ctx->direct && (st = build_boxes(ctx, true))) return bail(st);
    // Default geometry: closed no-slip box at rest (f~ = 0).
    {
        const int64_t nx = dec.domain[0], ny = dec.domain[1], nz = dec.domain[2];
        std::vector<uint8_t> fl((size_t)(nx + 2) * (ny + 2) * (nz + 2), 0);
        for (int64_t z = -1; z <= nz; ++z)
            for (int64_t y = -1; y <= ny; ++y)
                for (int64_t x = -1; x <= nx; ++x) {
                    const bool shell = x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz;
                    if (shell) fl[((z + 1) * (ny + 2) + (y + 1)) * (nx + 2) + (x + 1)] = LBM_NOSLIP;
                }
        if ((st = apply_flags(ctx, fl.data(), nullptr, 0))) return bail(st);
    }
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return bail(LBM_ERR_CUDA);
    *out = ctx;
    return LBM_OK;
}

}  // namespace lbm
