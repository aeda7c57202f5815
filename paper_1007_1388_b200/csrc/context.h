// context.h -- the per-rank runtime context and the helpers shared by the
// runtime's translation units (private; the product interface is include/lbm.h):
//   setup.cu     geometry, sweep boxes, exchange plans, flags, fused-exchange
//                setup, create / destroy
//   step.cu      one time step: sweep launches, ghost exchange, overlap,
//                timing, CUDA graphs
//   transfer.cu  host <-> device transfers of the canonical layout
//   api.cu       the C ABI
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "lbm_internal.h"

namespace lbm {

constexpr int kTimingSlots = 64;
enum Phase { PH_SWEEP = 0, PH_SHELL = 1, PH_INTERIOR = 2, PH_PACK = 3, PH_NCCL = 4, PH_UNPACK = 5, PH_STEP = 6 };
constexpr int kEvPerSlot = 14;

// A sweep's work list: one 16-B descriptor per 64 x 4-cell tile (one block),
// {patch, x0 << 16 | xend, y0 << 16 | yend, z}, built on the host from the boxes.
// A block decodes its tile with one load and no division or search.
struct DevBoxes {
    int4 *desc = nullptr;
    int n = 0;          // boxes
    int64_t tiles = 0;  // descriptors == blocks of one launch
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

// file name without directories, for error messages
inline const char *base_name(const char *path)
{
    const char *s = std::strrchr(path, '/');
    return s ? s + 1 : path;
}

}  // namespace lbm

using namespace lbm;

struct lbm_ctx {
    lbm_config cfg;
    Decomp dec;
    Geom g;
    int esize = 8;
    int device = 0;
    // x2 sweep occupancy (sweep.cu launch_sweep): 0 = measured best, 1 = the
    // alternative (env LBM_SWEEP_VARIANT, tools/sweep_tune.py)
    int sweep_variant = 0;
    int tile_x = SWEEP_BX, tile_y = SWEEP_BY;
    int num_sms = 148;
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
    uint32_t *wmask = nullptr;  // wall-neighbour masks of kind-1 cells (flag layout)
    Checker chk;                  // checked build only (kernels.cuh): shadow arrays of the grids
    unsigned long long chk_seq = 0;
    BbEntry *bb_list = nullptr;  // wall-adjacent fluid cells in memory order, per step (launch_bb_list)
    int64_t bb_n = 0;
    BbEntry *bb_full = nullptr;  // every wall link: the fills after set_pdfs / set_flags
    int64_t bb_full_n = 0;
    unsigned long long *sidewall = nullptr;  // [nlocal] uniform-wall sides (launch_sidewall)
    void *corr = nullptr;
    int *d_origin = nullptr;
    ExSet ex[3];               // indexed by ExKind
    // Fused exchange (handshake.cu): the sweep stores outgoing PDFs straight
    // into neighbour ghost layers (local or CUDA-IPC-mapped peer memory).
    bool direct = false;
    unsigned long long *d_epoch = nullptr;
    unsigned long long *d_inbox = nullptr;  // [nranks] epochs published by the peers
    unsigned long long **d_peer_inbox = nullptr;
    int *d_peer_rank = nullptr;
    int *d_error = nullptr;
    int npeers_direct = 0;
    std::vector<void *> ipc_mapped;         // peer grids / inboxes opened with cudaIpcOpenMemHandle
    // direct ghost stores by the x2 sweeps (same-GPU and, with `direct`, peer patches)
    bool ldirect = false;                   // same-GPU neighbours: no ghost copies
    void **d_dnbr = nullptr;                // [nlocal][18][2] neighbour patch bases per grid
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
    double *d_mass = nullptr;  // lbm_total_mass scratch: kMassBlocks partials + the sum
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
    lbm_status cuda_fail(cudaError_t e, const char *what, const char *file, int line)
    {
        char buf[512];
        std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s [%s:%d]", cudaGetErrorName(e),
                      cudaGetErrorString(e), what, base_name(file), line);
        if (e == cudaErrorMemoryAllocation) {
            err = buf;
            return LBM_ERR_OOM;
        }
        return fail(LBM_ERR_CUDA, buf);
    }
    lbm_status nccl_fail(ncclResult_t r, const char *what, const char *file, int line)
    {
        char buf[512];
        std::snprintf(buf, sizeof buf, "NCCL error %d (%s) in %s [%s:%d]", (int)r, ncclGetErrorString(r), what,
                      base_name(file), line);
        return fail(LBM_ERR_NCCL, buf);
    }
};

#define CK(call)                                                              \
    do {                                                                      \
        cudaError_t e_ = (call);                                              \
        if (e_ != cudaSuccess) return ctx->cuda_fail(e_, #call, __FILE__, __LINE__);    \
    } while (0)
#define NK(call)                                                              \
    do {                                                                      \
        ncclResult_t r_ = (call);                                             \
        if (r_ != ncclSuccess) return ctx->nccl_fail(r_, #call, __FILE__, __LINE__);    \
    } while (0)
#define CHECK_CTX(ctx)                                                        \
    do {                                                                      \
        if (!(ctx)) return LBM_ERR_ARG;                                       \
        if ((ctx)->poisoned) return LBM_ERR_STATE;                            \
        cudaError_t e_ = cudaSetDevice((ctx)->device);                        \
        if (e_ != cudaSuccess) return (ctx)->cuda_fail(e_, "cudaSetDevice", __FILE__, __LINE__); \
    } while (0)

namespace lbm {

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

// Host -> device uploads and memsets ordered with the ctx stream.  A plain
// cudaMemcpy from pageable host memory may return before its DMA has landed,
// and cudaMemset on device memory is asynchronous -- both on the legacy stream,
// which the library's non-blocking streams do not wait for: a kernel launched
// right after could read the buffer half written (seen: lid-plane flags).
inline cudaError_t upload(lbm_ctx *ctx, void *dst, const void *src, size_t bytes)
{
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    return e;
}

inline cudaError_t memset_sync(lbm_ctx *ctx, void *dst, int value, size_t bytes)
{
    cudaError_t e = cudaMemsetAsync(dst, value, bytes, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    return e;
}

extern thread_local std::string g_create_error;  // api.cu: lbm_last_error(NULL)

Geom make_geom(const int n[3], int esize);

Box make_box(const lbm_ctx *ctx, int patch, const int lo[3], const int n[3]);

lbm_status upload_boxes(lbm_ctx *ctx, const std::vector<Box> &boxes, DevBoxes &out);
// After the flags change (or the boxes are rebuilt): the bounce-back list and the
// tiles' non-fluid bits.
lbm_status build_wall_lists(lbm_ctx *ctx);
// Checked build (kernels.cuh Checker): the checker of the next launch (fresh
// launch sequence), clearing the shadows at a step boundary, and the report
// (LBM_ERR_INTERNAL with the counts if anything was flagged).  No-ops otherwise.
Checker next_checker(lbm_ctx *ctx);
lbm_status chk_alloc(lbm_ctx *ctx, size_t grid_bytes);
lbm_status chk_clear(lbm_ctx *ctx, cudaStream_t s);
lbm_status chk_report(lbm_ctx *ctx);
#ifdef LBM_CHECKED
constexpr bool kChecked = true;
#else
constexpr bool kChecked = false;
#endif
// The bounce-back list kernel on grid gi (mode: aux_kernels.cu bb_list_kernel);
// full: every link (after set_pdfs / set_flags), else the per-step list.
lbm_status launch_bb(lbm_ctx *ctx, int gi, int mode, cudaStream_t s, bool full = false);

void release_boxes(lbm_ctx *ctx, DevBoxes &b);

lbm_status upload_segs(lbm_ctx *ctx, const std::vector<CopySeg> &v, DevSegs &out);

CopySeg grid_to_x(const lbm_ctx *ctx, const Seg &s, bool to_buffer, int64_t buf_base);

CopySeg buffer_to_grid(const lbm_ctx *ctx, const Seg &s, int64_t buf_base);

lbm_status setup_exset(lbm_ctx *ctx, int kind, bool upload);

lbm_status update_seg_masks(lbm_ctx *ctx, const uint8_t *gflags);

lbm_status build_boxes(lbm_ctx *ctx, bool whole_x);

lbm_status setup_exchange(lbm_ctx *ctx);

lbm_status apply_flags(lbm_ctx *ctx, const uint8_t *flags, const double *wall_u, int nvel);

const char *validate_flags(const Decomp &dec, const uint8_t *flags, const double *wall_u, int nvel);

void destroy_ctx(lbm_ctx *ctx);

lbm_status setup_direct(lbm_ctx *ctx);

lbm_status create_impl(const lbm_config *cfg, lbm_ctx **out);

lbm_status launch_sweep_set(lbm_ctx *ctx, const DevBoxes &b, cudaStream_t s);

lbm_status launch_copy(lbm_ctx *ctx, const DevSegs &d, void *grid_src, void *grid_dst, void *buf_src, void *buf_dst,
                       cudaStream_t s);

lbm_status transport(lbm_ctx *ctx, const ExSet &X, cudaStream_t s);

lbm_status exchange_seq(lbm_ctx *ctx, int gi, cudaStream_t s, TimingSlot *ts, int kind, bool in_step);

lbm_status refresh_state(lbm_ctx *ctx);

lbm_status accumulate_slot(lbm_ctx *ctx, TimingSlot &ts);

lbm_status flush_timing(lbm_ctx *ctx);

lbm_status enqueue_step(lbm_ctx *ctx);

lbm_status ensure_graph(lbm_ctx *ctx);

lbm_status enqueue_steps(lbm_ctx *ctx, int64_t n);

// Fused exchange: wait until every peer has finished storing into this rank's
// memory for the steps done so far (peers' epoch >= own epoch), then drain
// both streams.  No-op without peers.
lbm_status quiesce(lbm_ctx *ctx);

lbm_status transfer_chunks(lbm_ctx *ctx, double *host, bool to_device, int mode, double *rho, double *u);

}  // namespace lbm
