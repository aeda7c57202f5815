// runtime.cu -- patch runtime and C ABI (include/lbm.h) of the B200 solver.
//
// One process per GPU; each rank owns a brick of patches (the paper's
// Blocks) stored back to back in one SoA allocation per PDF grid
// (two grids).  A time step (the paper's Sweep) is:
//   sweep (fused pull + BB + collide, kernels.cu)  ->  ghost exchange
//   (extract = pack / local copy, transport = NCCL send/recv, insert = unpack;
//   P:287-313).  With overlap on, the patch shells facing remote
//   neighbours are swept first, packed and sent on a second stream while the
//   interiors are swept (the paper sums these times).  Steps are
//   captured pairwise (src/dst swap) in a CUDA graph and replayed.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "lbm_internal.h"

using namespace lbm;

namespace {

thread_local std::string g_create_error;

constexpr int kAlignDefault = 128;  // bytes; interior x = 0 of every row starts on this boundary
constexpr int kTimingSlots = 64;
enum Phase { PH_SWEEP = 0, PH_SHELL = 1, PH_INTERIOR = 2, PH_PACK = 3, PH_NCCL = 4, PH_UNPACK = 5, PH_STEP = 6 };
constexpr int kEvPerSlot = 14;

struct DevBoxes {
    Box *boxes = nullptr;
    int64_t *prefix = nullptr;
    int n = 0;
    int64_t tiles = 0;
};

struct DevSegs {
    CopySeg *segs = nullptr;
    int n = 0;
    int64_t max_elems = 0;
    int64_t total_elems = 0;
};

struct Peer {
    int rank;
    int64_t send_off, send_n, recv_off, recv_n;
};

// One exchange kind (EX_AB, EX_AA1, EX_AA2): segment lists, device copy
// descriptors and the per-peer message layout.
struct ExSet {
    SegLists segs;
    DevSegs pack_all;   // pack + local copies (non-overlapped step / ghost refresh)
    DevSegs pack_remote, local_copy, unpack;
    std::vector<CopySeg> h_pack_all, h_local, h_unpack;  // host copies (flag masks are refreshed)
    std::vector<Peer> peers;
    int64_t send_elems = 0, recv_elems = 0;
    bool has_remote = false;   // anything goes through buffers
    bool has_nccl = false;     // a peer other than this rank
};

struct TimingSlot {
    cudaEvent_t ev[kEvPerSlot];
    bool used = false;
    bool overlap = false;
    bool exchange = false;  // exchange phases were recorded (there was exchange work)
};

}  // namespace

struct lbm_ctx {
    lbm_config cfg;
    Decomp dec;
    Geom g;
    int esize = 8;
    int device = 0;
    int align = kAlignDefault;
    // SIMT sweep variants [fp32, fp64] measured best by tools/sweep_tune.py (profiles/r01_sweep_tune_*):
    // two cells per thread with 2-vector accesses (x2): fp32 4 blocks/SM, fp64 3 blocks/SM (128 threads);
    // env LBM_SWEEP_VARIANT.
    int sweep_variant[2] = {12, 13};
    int aa_variant[2] = {12, 13};  // AA kernels, two cells per thread (tools/sweep_tune.py --layout 1)
    int direct_variant[2] = {6, 5};  // AA kernels (tools/sweep_tune.py --layout 1): fp32 4 blocks/SM, fp64 2
    bool use_tma = false;           // TMA-staged sweep (sweep_tma.cu); env LBM_SWEEP_IMPL=tma|simt
    int tile_x = SWEEP_BX, tile_y = SWEEP_BY;
    int num_sms = 148;
    int tma_variant = 0;            // tile shape (sweep_tma.cu TmaShape); env LBM_TMA_SHAPE
    alignas(64) CUtensorMap tm_pdf[2];
    alignas(64) CUtensorMap tm_kind;
    alignas(64) CUtensorMap tm_flags;
    cudaStream_t stream = nullptr, comm_stream = nullptr;
    // host <-> device transfers (transfer_chunks): two staging buffers and a
    // copy stream, so the DMA of one chunk overlaps the kernel of the next
    double *xstage[2] = {nullptr, nullptr};
    size_t xstage_bytes = 0;
    cudaStream_t xstream = nullptr;
    cudaEvent_t xev_copy[2] = {}, xev_kern[2] = {};
    bool own_stream = false;
    void *grid[2] = {nullptr, nullptr};
    int cur = 0;
    uint8_t *flags = nullptr, *kind = nullptr;
    void *corr = nullptr;
    int *d_origin = nullptr;
    ExSet ex[3];               // indexed by ExKind
    // Fused exchange (sweep_direct.cu): the sweep stores outgoing PDFs straight
    // into neighbour ghost layers (local or CUDA-IPC-mapped peer memory).
    bool direct = false;
    void **d_nbr = nullptr;                 // [nlocal][18][2] neighbour patch bases
    unsigned long long *d_epoch = nullptr;
    unsigned long long *d_inbox = nullptr;  // [nranks] epochs published by the peers
    unsigned long long **d_peer_inbox = nullptr;
    int *d_peer_rank = nullptr;
    int *d_error = nullptr;
    int npeers_direct = 0;
    std::vector<void *> ipc_mapped;         // peer grids / inboxes opened with cudaIpcOpenMemHandle
    // Local pull (NEXT-2): face cells read same-GPU neighbour patches directly;
    // no ghost copies between local patches.
    bool lpull = false;
    void **d_lnbr = nullptr;                // [nlocal][18][2]
    // direct ghost stores by the x2 sweep (same-GPU and, with `direct`, peer patches)
    bool ldirect = false;                   // same-GPU neighbours: no ghost copies
    bool x2_shells = false;                 // fused exchange: shells swept by the x2 kernel
    void **d_dnbr = nullptr;                // [nlocal][18][2]
    std::vector<void *> h_nbr;              // setup_direct's peer-mapped table
    int layout = LBM_LAYOUT_AB;
    int aa_phase = 0;          // AA: 0 swapped (next step PULL), 1 streamed (next step LOCAL)
    void *sendbuf = nullptr, *recvbuf = nullptr;
    bool has_remote = false;   // anything goes through buffers
    bool has_nccl = false;     // a peer other than this rank
    ncclComm_t nccl = nullptr;
    DevBoxes box_all, box_shell, box_interior;
    bool use_overlap = false;
    int64_t fluid_local = 0, fluid_global = 0;
    bool flags_set = false;
    int64_t steps = 0, launches = 0;
    int64_t launches_per_step = 0;
    int64_t device_bytes = 0;
    std::string err;
    bool poisoned = false;
    bool timing = false;
    double phase_ms[LBM_NPHASES] = {0};
    int64_t phase_count[LBM_NPHASES] = {0};
    TimingSlot slots[kTimingSlots];
    int slot_next = 0;
    bool events_created = false;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int64_t graph_launches[2] = {0, 0};

    lbm_status fail(lbm_status st, const std::string &m)
    {
        err = m;
        if (st == LBM_ERR_CUDA || st == LBM_ERR_NCCL || st == LBM_ERR_INTERNAL) poisoned = true;
        return st;
    }
    lbm_status cuda_fail(cudaError_t e, const char *what, int line)
    {
        char buf[512];
        std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s [runtime.cu:%d]", cudaGetErrorName(e),
                      cudaGetErrorString(e), what, line);
        if (e == cudaErrorMemoryAllocation) {
            err = buf;
            return LBM_ERR_OOM;
        }
        return fail(LBM_ERR_CUDA, buf);
    }
    lbm_status nccl_fail(ncclResult_t r, const char *what, int line)
    {
        char buf[512];
        std::snprintf(buf, sizeof buf, "NCCL error %d (%s) in %s [runtime.cu:%d]", (int)r, ncclGetErrorString(r), what,
                      line);
        return fail(LBM_ERR_NCCL, buf);
    }
};

#define CK(call)                                                              \
    do {                                                                      \
        cudaError_t e_ = (call);                                              \
        if (e_ != cudaSuccess) return ctx->cuda_fail(e_, #call, __LINE__);    \
    } while (0)
#define NK(call)                                                              \
    do {                                                                      \
        ncclResult_t r_ = (call);                                             \
        if (r_ != ncclSuccess) return ctx->nccl_fail(r_, #call, __LINE__);    \
    } while (0)
#define CHECK_CTX(ctx)                                                        \
    do {                                                                      \
        if (!(ctx)) return LBM_ERR_ARG;                                       \
        if ((ctx)->poisoned) return LBM_ERR_STATE;                            \
        cudaError_t e_ = cudaSetDevice((ctx)->device);                        \
        if (e_ != cudaSuccess) return (ctx)->cuda_fail(e_, "cudaSetDevice", __LINE__); \
    } while (0)

namespace {

template <typename T>
lbm_status dev_alloc(lbm_ctx *ctx, T **p, size_t bytes)
{
    *p = nullptr;
    if (bytes == 0) return LBM_OK;
    cudaError_t e = cudaMalloc((void **)p, bytes);
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        char buf[256];
        std::snprintf(buf, sizeof buf, "cudaMalloc of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
        ctx->err = buf;
        return e == cudaErrorMemoryAllocation ? LBM_ERR_OOM : ctx->fail(LBM_ERR_CUDA, buf);
    }
    ctx->device_bytes += (int64_t)bytes;
    return LBM_OK;
}

Geom make_geom(const int n[3], int esize, int align)
{
    Geom g;
    for (int a = 0; a < 3; ++a) g.n[a] = n[a];
    const int ae = align / esize;             // elements per alignment unit
    g.xo = ae;                                // x = -1 sits right before the aligned x = 0
    // columns up to x = n + 1 must exist: the two-cells-per-thread kernels read
    // the phantom partner x0 + 1 = n of an odd row and its pull neighbour n + 1
    g.px = ((g.xo + n[0] + 2 + ae - 1) / ae) * ae;
    g.py = n[1] + 2;
    g.plane = (int64_t)g.px * g.py;
    g.qs = g.plane * (n[2] + 2);
    g.ps = (int64_t)Q * g.qs;
    g.fs = g.qs;
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
    std::vector<int64_t> prefix(boxes.size() + 1, 0);
    for (size_t i = 0; i < boxes.size(); ++i) {
        const Box &b = boxes[i];
        const int zc = (ctx->use_tma || ctx->layout == LBM_LAYOUT_AA)
                           ? 1
                           : sweep_cells_z(ctx->sweep_variant[ctx->esize == 8 ? 1 : 0]);
        int64_t t = (b.n[0] > 0 && b.n[1] > 0 && b.n[2] > 0)
                        ? (int64_t)b.tiles_x * b.tiles_y * ((b.n[2] + zc - 1) / zc)
                        : 0;
        prefix[i + 1] = prefix[i] + t;
    }
    out.n = (int)boxes.size();
    out.tiles = prefix.back();
    if (boxes.empty()) return LBM_OK;
    lbm_status st = dev_alloc(ctx, &out.boxes, boxes.size() * sizeof(Box));
    if (st) return st;
    st = dev_alloc(ctx, &out.prefix, prefix.size() * sizeof(int64_t));
    if (st) return st;
    CK(cudaMemcpy(out.boxes, boxes.data(), boxes.size() * sizeof(Box), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(out.prefix, prefix.data(), prefix.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    return LBM_OK;
}

void release_boxes(lbm_ctx *ctx, DevBoxes &b)
{
    if (b.boxes) {
        cudaFree(b.boxes);
        ctx->device_bytes -= (int64_t)(b.n * sizeof(Box));
    }
    if (b.prefix) {
        cudaFree(b.prefix);
        ctx->device_bytes -= (int64_t)((b.n + 1) * sizeof(int64_t));
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
    CK(cudaMemcpy(out.segs, v.data(), v.size() * sizeof(CopySeg), cudaMemcpyHostToDevice));
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
            CK(cudaMemcpy(dv[j]->segs, v.data(), v.size() * sizeof(CopySeg), cudaMemcpyHostToDevice));
        }
    }
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
        // Every tile must start on a 16-cell boundary in x (16-B aligned TMA
        // starts for the PDF, kind and flag maps, see sweep_tma.cu): round the
        // high-x shell start down.
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
    ctx->use_overlap = ctx->cfg.overlap && ctx->has_nccl;
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
    a.flags = ctx->flags;
    a.kind = ctx->kind;
    a.corr = (const real *)ctx->corr;
    a.g = ctx->g;
    a.omega = (real)ctx->cfg.omega;
    a.boxes = b.boxes;
    a.tile_prefix = b.prefix;
    a.nboxes = b.n;
    a.lnbr = ctx->lpull ? (const real *const *)ctx->d_lnbr : nullptr;
    a.srci = ctx->cur;
    a.dnbr = ctx->ldirect && ctx->layout == LBM_LAYOUT_AB ? (real *const *)ctx->d_dnbr : nullptr;
    a.dsti = 1 - ctx->cur;
    return a;
}

lbm_status launch_sweep_set(lbm_ctx *ctx, const DevBoxes &b, cudaStream_t s)
{
    if (b.tiles == 0) return LBM_OK;
    cudaError_t e;
    if (ctx->layout == LBM_LAYOUT_AA) {
        const bool pull = ctx->aa_phase == 0;
        if (ctx->esize == 8)
            e = launch_sweep_aa<double>(sweep_args<double>(ctx, b), b.tiles, pull, ctx->aa_variant[1], s);
        else
            e = launch_sweep_aa<float>(sweep_args<float>(ctx, b), b.tiles, pull, ctx->aa_variant[0], s);
    } else if (ctx->use_tma) {
        const CUtensorMap &pm = ctx->tm_pdf[ctx->cur];
        if (ctx->esize == 8)
            e = launch_sweep_tma<double>(pm, ctx->tm_kind, ctx->tm_flags, sweep_args<double>(ctx, b), b.tiles,
                                         ctx->num_sms, ctx->tma_variant, s);
        else
            e = launch_sweep_tma<float>(pm, ctx->tm_kind, ctx->tm_flags, sweep_args<float>(ctx, b), b.tiles,
                                        ctx->num_sms, ctx->tma_variant, s);
    } else if (ctx->esize == 8)
        e = launch_sweep<double>(sweep_args<double>(ctx, b), b.tiles, ctx->sweep_variant[1], s);
    else
        e = launch_sweep<float>(sweep_args<float>(ctx, b), b.tiles, ctx->sweep_variant[0], s);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "sweep_kernel launch", __LINE__);
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
    if (e != cudaSuccess) return ctx->cuda_fail(e, "copy_segments launch", __LINE__);
    ctx->launches += (d.n + 65534) / 65535;
    return LBM_OK;
}

// Transport of the send buffers: grouped NCCL send/recv per peer;
// a self-peer (exchange_mode FORCE_BUFFERS) is a device copy.
lbm_status transport(lbm_ctx *ctx, const ExSet &X, cudaStream_t s)
{
    const ncclDataType_t dt = ctx->esize == 8 ? ncclFloat64 : ncclFloat32;
    char *sb = (char *)ctx->sendbuf, *rb = (char *)ctx->recvbuf;
    for (const Peer &p : X.peers)
        if (p.rank == ctx->dec.rank && p.send_n > 0)
            CK(cudaMemcpyAsync(rb + p.recv_off * ctx->esize, sb + p.send_off * ctx->esize, p.send_n * ctx->esize,
                               cudaMemcpyDeviceToDevice, s));
    if (!X.has_nccl) return LBM_OK;
    NK(ncclGroupStart());
    for (const Peer &p : X.peers) {
        if (p.rank == ctx->dec.rank) continue;
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
    // local pull: same-GPU neighbours are read in place, only remote segments move
    const bool skip_local = ctx->lpull || (in_step && ctx->ldirect);
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

// After the state or the flags change: refresh the ghost layers of the current
// grid and park the store-side bounce-back values in the wall cells.
lbm_status refresh_state(lbm_ctx *ctx)
{
    // AB: ghost layers of the current grid.  AA (swapped state): half-exchange 1,
    // which is what the next PULL step gathers from the ghost layers.
    const bool aa = ctx->layout == LBM_LAYOUT_AA;
    lbm_status st = exchange_seq(ctx, ctx->cur, ctx->stream, nullptr, aa ? EX_AA1 : EX_AB, false);
    if (st) return st;
    cudaError_t e = ctx->esize == 8
                        ? launch_bb_fill<double>((double *)ctx->grid[ctx->cur], ctx->flags, ctx->kind,
                                                 (const double *)ctx->corr, ctx->dec.nlocal, ctx->g, aa ? 1 : 0,
                                                 ctx->stream)
                        : launch_bb_fill<float>((float *)ctx->grid[ctx->cur], ctx->flags, ctx->kind,
                                                (const float *)ctx->corr, ctx->dec.nlocal, ctx->g, aa ? 1 : 0,
                                                ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "bb_fill", __LINE__);
    ctx->launches += (ctx->dec.nlocal + 65534) / 65535;
    CK(cudaStreamSynchronize(ctx->stream));
    return LBM_OK;
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
        if (e != cudaSuccess) return ctx->cuda_fail(e, "wait_peers launch", __LINE__);
        ctx->launches += 1;
        const DevBoxes &bs = ctx->box_shell;
        if (bs.tiles > 0 && ctx->x2_shells) {
            if (ctx->esize == 8) {
                SweepArgs<double> a = sweep_args<double>(ctx, bs);
                a.dnbr = (double *const *)ctx->d_dnbr;
                e = launch_sweep<double>(a, bs.tiles, ctx->sweep_variant[1], c);
            } else {
                SweepArgs<float> a = sweep_args<float>(ctx, bs);
                a.dnbr = (float *const *)ctx->d_dnbr;
                e = launch_sweep<float>(a, bs.tiles, ctx->sweep_variant[0], c);
            }
            if (e != cudaSuccess) return ctx->cuda_fail(e, "shell sweep launch", __LINE__);
            ctx->launches += 1;
        } else if (bs.tiles > 0) {
            void **tab = ctx->ldirect ? ctx->d_dnbr : ctx->d_nbr;
            if (ctx->esize == 8) {
                DirectArgs<double> dx{(double *const *)tab, dsti};
                e = launch_sweep_direct<double>(sweep_args<double>(ctx, bs), dx, bs.tiles, ctx->direct_variant[1], c);
            } else {
                DirectArgs<float> dx{(float *const *)tab, dsti};
                e = launch_sweep_direct<float>(sweep_args<float>(ctx, bs), dx, bs.tiles, ctx->direct_variant[0], c);
            }
            if (e != cudaSuccess) return ctx->cuda_fail(e, "sweep_direct launch", __LINE__);
            ctx->launches += 1;
        }
        e = launch_signal_peers(ctx->d_epoch, ctx->d_peer_inbox, ctx->npeers_direct, c);
        if (e != cudaSuccess) return ctx->cuda_fail(e, "signal_peers launch", __LINE__);
        ctx->launches += 1;
        CK(cudaEventRecord(ev_shell, c));
        if ((st = launch_sweep_set(ctx, ctx->box_interior, s))) return st;
        CK(cudaStreamWaitEvent(s, ev_shell, 0));
        if (!ctx->ldirect && (st = launch_copy(ctx, X.local_copy, dst, dst, nullptr, nullptr, s))) return st;
    } else if (!ctx->use_overlap) {
        if ((st = launch_sweep_set(ctx, ctx->box_all, s))) return st;
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
        if (ts) CK(cudaEventRecord(ts->ev[9], s));
        if (!ctx->lpull && !ctx->ldirect && (st = launch_copy(ctx, X.local_copy, dst, dst, nullptr, nullptr, s)))
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
    if (e != cudaSuccess) return ctx->cuda_fail(e, "cudaStreamEndCapture", __LINE__);
    ctx->graph_launches[c] = ctx->launches - l0;
    ctx->launches = l0;
    ctx->steps = s0;  // capture did not execute anything
    // cur flipped twice -> back to c
    e = cudaGraphInstantiate(&ctx->graph[c], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        ctx->graph[c] = nullptr;
        return ctx->cuda_fail(e, "cudaGraphInstantiate", __LINE__);
    }
    return LBM_OK;
}

lbm_status enqueue_steps(lbm_ctx *ctx, int64_t n)
{
    lbm_status st;
    const bool graphs = ctx->cfg.use_graphs && !ctx->timing;
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

lbm_status apply_flags(lbm_ctx *ctx, const uint8_t *flags, const double *wall_u, int nvel)
{
    const int64_t nx = ctx->dec.domain[0], ny = ctx->dec.domain[1], nz = ctx->dec.domain[2];
    const size_t total = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
    uint8_t *dflags = nullptr;
    lbm_status st = dev_alloc(ctx, &dflags, total);
    if (st) return st;
    cudaError_t e = cudaMemcpy(dflags, flags, total, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = launch_build_flags(dflags, ctx->dec.domain, ctx->dec.periodic, ctx->d_origin, ctx->dec.nlocal, ctx->g,
                               ctx->flags, ctx->kind, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(dflags);
    ctx->device_bytes -= (int64_t)total;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "build flags", __LINE__);
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
        CK(cudaMemcpy(ctx->corr, cd.data(), cd.size() * sizeof(double), cudaMemcpyHostToDevice));
    } else {
        std::vector<float> cf(cd.begin(), cd.end());
        CK(cudaMemcpy(ctx->corr, cf.data(), cf.size() * sizeof(float), cudaMemcpyHostToDevice));
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
    return LBM_OK;
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
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
    for (int i = 0; i < 2; ++i)
        if (ctx->graph[i]) cudaGraphExecDestroy(ctx->graph[i]);
    if (ctx->nccl) ncclCommDestroy(ctx->nccl);
    for (void *p : ctx->ipc_mapped) cudaIpcCloseMemHandle(p);
    for (void *p : {(void *)ctx->d_lnbr, (void *)ctx->d_dnbr, (void *)ctx->d_nbr, (void *)ctx->d_epoch, (void *)ctx->d_inbox,
                    (void *)ctx->d_peer_inbox, (void *)ctx->d_peer_rank, (void *)ctx->d_error})
        if (p) cudaFree(p);
    for (ExSet &X : ctx->ex)
        for (void *p : {(void *)X.pack_all.segs, (void *)X.pack_remote.segs, (void *)X.local_copy.segs,
                        (void *)X.unpack.segs})
            if (p) cudaFree(p);
    void *ptrs[] = {ctx->grid[0], ctx->grid[1], ctx->flags, ctx->kind, ctx->corr, ctx->d_origin, ctx->sendbuf,
                    ctx->recvbuf,
                    ctx->box_all.boxes, ctx->box_all.prefix, ctx->box_shell.boxes, ctx->box_shell.prefix,
                    ctx->box_interior.boxes, ctx->box_interior.prefix};
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
    CK(cudaMemset(ctx->d_epoch, 0, sizeof(unsigned long long)));
    CK(cudaMemset(ctx->d_inbox, 0, (size_t)R * sizeof(unsigned long long)));
    CK(cudaMemset(ctx->d_error, 0, sizeof(int)));
    // Remote peers of the exchange plan.
    std::vector<int> peers;
    for (const Peer &p : ctx->ex[EX_AB].peers)
        if (p.rank != me) peers.push_back(p.rank);
    if (peers.empty()) return LBM_OK;  // nothing crosses a GPU boundary: copy path
    std::vector<void *> peer_grid((size_t)R * 2, nullptr), peer_inbox((size_t)R, nullptr);
    {
        // all-gather {grid0, grid1, inbox} IPC handles
        const size_t hb = sizeof(cudaIpcMemHandle_t);
        std::vector<cudaIpcMemHandle_t> mine(3);
        CK(cudaIpcGetMemHandle(&mine[0], ctx->grid[0]));
        CK(cudaIpcGetMemHandle(&mine[1], ctx->grid[1]));
        CK(cudaIpcGetMemHandle(&mine[2], ctx->d_inbox));
        char *dbuf = nullptr;
        if ((st = dev_alloc(ctx, &dbuf, 3 * hb * (size_t)(R + 1)))) return st;
        CK(cudaMemcpy(dbuf, mine.data(), 3 * hb, cudaMemcpyHostToDevice));
        NK(ncclAllGather(dbuf, dbuf + 3 * hb, 3 * hb, ncclUint8, ctx->nccl, ctx->stream));
        std::vector<cudaIpcMemHandle_t> all((size_t)3 * R);
        CK(cudaMemcpyAsync(all.data(), dbuf + 3 * hb, 3 * hb * R, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(dbuf);
        ctx->device_bytes -= (int64_t)(3 * hb * (size_t)(R + 1));
        int ok = 1;
        for (int r : peers) {
            for (int i = 0; i < 3 && ok; ++i) {
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
        CK(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
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
            if (r == me) continue;  // same-GPU neighbours: ghost copy after the sweep
            const int64_t off = (int64_t)dec.local_index_on_owner(nbp) * ctx->g.ps * ctx->esize;
            for (int i = 0; i < 2; ++i) {
                char *base = (char *)peer_grid[(size_t)2 * r + i];
                nbr[((size_t)l * NDIR + k) * 2 + i] = base + off;
            }
        }
    }
    ctx->h_nbr = nbr;
    if ((st = dev_alloc(ctx, &ctx->d_nbr, nbr.size() * sizeof(void *)))) return st;
    CK(cudaMemcpy(ctx->d_nbr, nbr.data(), nbr.size() * sizeof(void *), cudaMemcpyHostToDevice));
    std::vector<unsigned long long *> pin;
    std::vector<int> prank;
    for (int r : peers) {
        pin.push_back((unsigned long long *)peer_inbox[r] + me);
        prank.push_back(r);
    }
    ctx->npeers_direct = (int)peers.size();
    if (!peers.empty()) {
        if ((st = dev_alloc(ctx, &ctx->d_peer_inbox, pin.size() * sizeof(void *)))) return st;
        CK(cudaMemcpy(ctx->d_peer_inbox, pin.data(), pin.size() * sizeof(void *), cudaMemcpyHostToDevice));
        if ((st = dev_alloc(ctx, &ctx->d_peer_rank, prank.size() * sizeof(int)))) return st;
        CK(cudaMemcpy(ctx->d_peer_rank, prank.data(), prank.size() * sizeof(int), cudaMemcpyHostToDevice));
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
    if (const char *a = std::getenv("LBM_SWEEP_VARIANT")) {
        int v = std::atoi(a);
        if (v >= 0 && v < kSweepVariants) {
            ctx->sweep_variant[0] = ctx->sweep_variant[1] = v;
        }
        if ((v >= 0 && v < 8) || v >= 12) ctx->aa_variant[0] = ctx->aa_variant[1] = v;
        if (v >= 4 && v < 8) ctx->direct_variant[0] = ctx->direct_variant[1] = v;
    }
    if (const char *a = std::getenv("LBM_AA_VARIANT")) {  // AA kernels alone (12..15, kernels.cu launch_aa_x2)
        int v = std::atoi(a);
        if ((v >= 0 && v < 8) || (v >= 12 && v < kSweepVariants)) ctx->aa_variant[0] = ctx->aa_variant[1] = v;
    }
    if (const char *a = std::getenv("LBM_SWEEP_IMPL")) {
        if (std::string(a) == "simt") ctx->use_tma = false;
        if (std::string(a) == "tma") ctx->use_tma = true;
    }
    if (ctx->layout == LBM_LAYOUT_AA) ctx->use_tma = false;  // the AA kernels are SIMT
    if (const char *a = std::getenv("LBM_TMA_SHAPE")) {
        int v = std::atoi(a);
        if (v >= 0 && v <= 2) ctx->tma_variant = v;
    }
    if (ctx->use_tma) {
        if (ctx->esize == 8)
            tma_tile_shape<double>(ctx->tma_variant, &ctx->tile_x, &ctx->tile_y);
        else
            tma_tile_shape<float>(ctx->tma_variant, &ctx->tile_x, &ctx->tile_y);
    }
    if (const char *a = std::getenv("LBM_ALIGN_BYTES")) {
        int v = std::atoi(a);
        if (v >= ctx->esize && v <= 1024 && (v & (v - 1)) == 0) ctx->align = v;
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
            char buf[256];
            std::snprintf(buf, sizeof buf, "liblbm_b200 is built for sm_100a (B200); device %d is %s (sm_%d%d)", dev,
                          prop.name, prop.major, prop.minor);
            ctx->err = buf;
            return bail(LBM_ERR_CUDA);
        }
    }
    ctx->g = make_geom(dec.patch, ctx->esize, ctx->align);
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
    if ((st = dev_alloc(ctx, &ctx->flags, flag_bytes))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->kind, flag_bytes))) return bail(st);
    if ((st = dev_alloc(ctx, &ctx->corr, (size_t)LBM_MAX_WALL_VELOCITIES * Q * ctx->esize))) return bail(st);
    {
        std::vector<int> origin(3 * dec.nlocal);
        for (int l = 0; l < dec.nlocal; ++l) {
            int c[3];
            dec.patch_coord(dec.local_to_global(l), c);
            for (int a = 0; a < 3; ++a) origin[3 * l + a] = c[a] * dec.patch[a];
        }
        if ((st = dev_alloc(ctx, &ctx->d_origin, origin.size() * sizeof(int)))) return bail(st);
        if (cudaMemcpy(ctx->d_origin, origin.data(), origin.size() * sizeof(int), cudaMemcpyHostToDevice) !=
            cudaSuccess)
            return bail(LBM_ERR_CUDA);
    }
    {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
            ctx->num_sms = sms;
    }
    if (ctx->use_tma) {
        for (int i = 0; i < 2; ++i) {
            cudaError_t e = ctx->esize == 8
                                ? make_tma_maps<double>(ctx->grid[i], ctx->kind, ctx->flags, dec.nlocal, ctx->g,
                                                        ctx->tma_variant, &ctx->tm_pdf[i], &ctx->tm_kind, &ctx->tm_flags)
                                : make_tma_maps<float>(ctx->grid[i], ctx->kind, ctx->flags, dec.nlocal, ctx->g,
                                                       ctx->tma_variant, &ctx->tm_pdf[i], &ctx->tm_kind, &ctx->tm_flags);
            if (e != cudaSuccess) {
                ctx->err = "cuTensorMapEncodeTiled failed for the PDF / kind arrays";
                return bail(LBM_ERR_CUDA);
            }
        }
    }
    if ((st = setup_exchange(ctx))) return bail(st);
    // NCCL communicator (bootstrap id broadcast by the caller, e.g. torch.distributed)
    if (cfg->nranks > 1) {
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_unique_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&ctx->nccl, cfg->nranks, id, cfg->rank);
        if (r != ncclSuccess) {
            ctx->nccl = nullptr;
            ctx->err = std::string("ncclCommInitRank failed: ") + ncclGetErrorString(r);
            return bail(LBM_ERR_NCCL);
        }
    }
    {
        // Fused exchange for the two-grid layout unless the NCCL path is requested
        // (exchange_mode FORCE_BUFFERS, or env LBM_EXCHANGE=nccl).
        const char *ev = std::getenv("LBM_EXCHANGE");
        const bool want = ctx->layout == LBM_LAYOUT_AB && cfg->exchange_mode == LBM_EXCHANGE_AUTO &&
                          !(ev && std::string(ev) == "nccl");
        if (want && (st = setup_direct(ctx))) return bail(st);
    }
    {
        // Local pull for the SIMT two-grid sweep when same-GPU neighbours exist.
        // Opt-in: measured slower than the ghost copies on B200.
        const char *ev = std::getenv("LBM_LOCAL_PULL");
        const int v = ctx->sweep_variant[ctx->esize == 8 ? 1 : 0];
        const bool want = ctx->layout == LBM_LAYOUT_AB && !ctx->use_tma && !ctx->direct &&
                          cfg->exchange_mode == LBM_EXCHANGE_AUTO && v >= 4 && v < 8 &&
                          (ev && std::string(ev) == "1") && !ctx->ex[EX_AB].segs.local.empty();
        if (want) {
            std::vector<void *> tab((size_t)dec.nlocal * NDIR * 2, nullptr);
            for (int l = 0; l < dec.nlocal; ++l) {
                const int gp = dec.local_to_global(l);
                for (int k = 0; k < NDIR; ++k) {
                    const int nbp = neighbour(dec, gp, kDirs[k].d);
                    if (nbp < 0 || dec.owner(nbp) != dec.rank) continue;
                    const int64_t off = (int64_t)dec.local_index_on_owner(nbp) * ctx->g.ps * ctx->esize;
                    for (int i = 0; i < 2; ++i) tab[((size_t)l * NDIR + k) * 2 + i] = (char *)ctx->grid[i] + off;
                }
            }
            if ((st = dev_alloc(ctx, &ctx->d_lnbr, tab.size() * sizeof(void *)))) return bail(st);
            if (cudaMemcpy(ctx->d_lnbr, tab.data(), tab.size() * sizeof(void *), cudaMemcpyHostToDevice) !=
                cudaSuccess)
                return bail(LBM_ERR_CUDA);
            ctx->lpull = true;
        }
    }
    {
        // Direct ghost stores by the two-grid x2 sweep: face / edge cells write
        // their outgoing PDFs straight into the neighbour patches' ghost layers.
        // (1) same-GPU neighbours, replacing the ghost copies after the sweep
        //     (default; LBM_LOCAL_DIRECT=0 keeps the copies);
        // (2) with the fused exchange, the shells facing other GPUs are swept by
        //     the same kernel through the peer-mapped table instead of the
        //     one-cell sweep_direct_kernel (LBM_SHELL_KERNEL=onecell keeps it).
        const char *ev = std::getenv("LBM_LOCAL_DIRECT");
        const char *es = std::getenv("LBM_SHELL_KERNEL");
        const int v = ctx->sweep_variant[ctx->esize == 8 ? 1 : 0];
        const bool x2 = ctx->layout == LBM_LAYOUT_AB && !ctx->use_tma && cfg->exchange_mode == LBM_EXCHANGE_AUTO &&
                        v >= 12;
        const bool want_local = x2 && !ctx->lpull && !(ev && std::string(ev) == "0") &&
                                !ctx->ex[EX_AB].segs.local.empty();
        const bool want_shell = x2 && ctx->direct && !(es && std::string(es) == "onecell");
        if (want_local || want_shell) {
            std::vector<void *> tab = ctx->direct ? ctx->h_nbr : std::vector<void *>((size_t)dec.nlocal * NDIR * 2, nullptr);
            for (int l = 0; l < dec.nlocal && want_local; ++l) {
                const int gp = dec.local_to_global(l);
                for (int k = 0; k < NDIR; ++k) {
                    const int nbp = neighbour(dec, gp, kDirs[k].d);
                    if (nbp < 0 || dec.owner(nbp) != dec.rank) continue;
                    const int64_t off = (int64_t)dec.local_index_on_owner(nbp) * ctx->g.ps * ctx->esize;
                    for (int i = 0; i < 2; ++i) tab[((size_t)l * NDIR + k) * 2 + i] = (char *)ctx->grid[i] + off;
                }
            }
            if ((st = dev_alloc(ctx, &ctx->d_dnbr, tab.size() * sizeof(void *)))) return bail(st);
            if (cudaMemcpy(ctx->d_dnbr, tab.data(), tab.size() * sizeof(void *), cudaMemcpyHostToDevice) !=
                cudaSuccess)
                return bail(LBM_ERR_CUDA);
            ctx->ldirect = want_local;
            ctx->x2_shells = want_shell;
        }
    }
    if (ctx->direct) {
        // fused exchange: patches with a remote x side are swept whole (build_boxes);
        // LBM_XSHELL=slab keeps the SWEEP_BX-wide x slabs
        const char *ev = std::getenv("LBM_XSHELL");
        if (!(ev && std::string(ev) == "slab") && (st = build_boxes(ctx, true))) return bail(st);
    }
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
    // representation of the state in the grid (kernels.cu rep_slot / read_state)
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
    if (e != cudaSuccess) return ctx->cuda_fail(e, "host/device transfer", __LINE__);
    return LBM_OK;
}

}  // namespace

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
    CK(cudaStreamSynchronize(ctx->stream));
    lbm_status st = apply_flags(ctx, flags, wall_u, nvel);
    if (st) return st;
    return refresh_state(ctx);
}

LBM_API lbm_status lbm_get_flags(lbm_ctx *ctx, uint8_t *out)
{
    CHECK_CTX(ctx);
    if (!out) return ctx->fail(LBM_ERR_ARG, "flags_out is NULL");
    CK(cudaStreamSynchronize(ctx->stream));
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
                const int64_t ci = ((int64_t)(lc[2] + 1) * g.py + (lc[1] + 1)) * g.px + (lc[0] + g.xo);
                out[((z + 1) * (on[1] + 2) + (y + 1)) * (on[0] + 2) + (x + 1)] = h[(size_t)lp * g.fs + ci];
            }
    return LBM_OK;
}

LBM_API lbm_status lbm_set_pdfs(lbm_ctx *ctx, const double *f)
{
    CHECK_CTX(ctx);
    if (!f) return ctx->fail(LBM_ERR_ARG, "f is NULL");
    CK(cudaStreamSynchronize(ctx->stream));
    lbm_status st = transfer_chunks(ctx, const_cast<double *>(f), true, 0, nullptr, nullptr);
    if (st) return st;
    return refresh_state(ctx);
}

LBM_API lbm_status lbm_init_noise(lbm_ctx *ctx, uint64_t seed)
{
    CHECK_CTX(ctx);
    const Decomp &d = ctx->dec;
    const int64_t on[3] = {d.owned_hi[0] - d.owned_lo[0], d.owned_hi[1] - d.owned_lo[1], d.owned_hi[2] - d.owned_lo[2]};
    cudaError_t e = ctx->esize == 8
                        ? launch_noise<double>((double *)ctx->grid[ctx->cur], seed, d.domain, d.owned_lo, on, d.brick,
                                               ctx->g, ctx->layout == LBM_LAYOUT_AA ? 1 : 0, ctx->stream)
                        : launch_noise<float>((float *)ctx->grid[ctx->cur], seed, d.domain, d.owned_lo, on, d.brick,
                                              ctx->g, ctx->layout == LBM_LAYOUT_AA ? 1 : 0, ctx->stream);
    ctx->aa_phase = 0;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "noise_kernel", __LINE__);
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
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->comm_stream));
    if (ctx->d_error && ctx->npeers_direct > 0) {
        int err = 0;
        CK(cudaMemcpy(&err, ctx->d_error, sizeof(int), cudaMemcpyDeviceToHost));
        if (err) return ctx->fail(LBM_ERR_INTERNAL, "fused exchange: a peer GPU did not reach the step barrier");
    }
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
    CK(cudaStreamSynchronize(ctx->stream));
    return transfer_chunks(ctx, f_out, false, 0, nullptr, nullptr);
}

LBM_API lbm_status lbm_get_pdfs_at(lbm_ctx *ctx, const int64_t *xyz, int64_t n, double *out)
{
    CHECK_CTX(ctx);
    if (n < 0 || (n > 0 && (!xyz || !out))) return ctx->fail(LBM_ERR_ARG, "bad sample arguments");
    if (n == 0) return LBM_OK;
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
    if (e != cudaSuccess) return ctx->cuda_fail(e, "gather", __LINE__);
    return LBM_OK;
}

LBM_API lbm_status lbm_get_macroscopic(lbm_ctx *ctx, double *rho_out, double *u_out)
{
    CHECK_CTX(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    if (!rho_out && !u_out) return LBM_OK;
    return transfer_chunks(ctx, nullptr, false, 1, rho_out, u_out);
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
    out->align_bytes = ctx->align;
    out->graphs_active = (ctx->graph[0] || ctx->graph[1]) ? 1 : 0;
    out->layout = ctx->layout;
    out->aa_phase = ctx->aa_phase;
    out->exchange_fused = ctx->direct ? 1 : 0;
    out->local_pull = ctx->lpull ? 1 : 0;
    out->local_direct = ctx->ldirect ? 1 : 0;
    if (ctx->lpull) out->halo_bytes_local_per_step = 0;
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
