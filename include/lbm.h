/*
 * lbm.h -- C ABI of the B200-native D3Q19 LBGK patch solver (the hot path of
 * Feichtinger et al., "A Flexible Patch-Based Lattice Boltzmann
 * Parallelization Approach for Heterogeneous GPU-CPU Clusters", arXiv:1007.1388).
 *
 * Citations: P:n = PAPER.md line n (section / equation named alongside).
 *
 * What the library computes (one time step, lbm_step):
 *   For every FLUID cell x of the lattice (D3Q19, 19 PDFs per cell)
 *     pull      p_i = f~_i(x - e_i)                       x - e_i fluid
 *               p_i = f~_opp(i)(x)                        no-slip wall
 *               p_i = f~_opp(i)(x) + 6 w_i rho0 e_i.u_w    moving wall    (R3)
 *     moments   drho = sum p_i ;  u = sum e_i p_i / rho0
 *     collide   f~_i(x) <- p_i - omega (p_i - f~eq_i(drho, u))           (eq:lbm P:410-415)
 *               f~eq_i = w_i [drho + rho0 (3 e_i.u + 4.5 (e_i.u)^2 - 1.5 u.u)]  (eq:feq P:416-425)
 *   with centred PDFs f~_i = f_i - w_i rho0, rho0 = 1, two PDF
 *   grids or one (AA pattern), then the ghost layers of every patch
 *   (the paper's Block) are refreshed: 5 PDFs per face cell, 1 PDF
 *   per edge cell, no corners.  By default the sweep
 *   itself stores those PDFs into the neighbour patches' ghost layers: plain
 *   stores on the same GPU, NVLink stores into the peer's CUDA-IPC-mapped grid
 *   across GPUs (one epoch handshake per step); alternatively pack -> NCCL
 *   send/recv -> unpack.
 *
 * Direction order (ABI, R2):
 *   i : 0      1  2  3  4  5  6   7      8      9      10     11     12     13     14     15     16     17     18
 *   e : (000) +x -x +y -y +z -z (++0) (--0) (+-0) (-+0) (+0+) (-0-) (+0-) (-0+) (0++) (0--) (0+-) (0-+)
 *   w : 1/3 | 1/18 x 6 | 1/36 x 12 ;  opp(i) = i+1 for odd i, i-1 for even i > 0.
 *
 * Conventions common to every entry point:
 *   * Host pointers are caller-owned, read or written only during the call,
 *     never retained.  Device memory, streams and the NCCL communicator are
 *     owned by the lbm_ctx and released by lbm_destroy.
 *   * A ctx is not thread-safe; use one per host thread / rank.
 *   * Arguments are validated before any side effect; a violation returns
 *     LBM_ERR_ARG and leaves the state unchanged.  A CUDA or NCCL failure
 *     poisons the ctx: later calls return LBM_ERR_STATE and only
 *     lbm_destroy / lbm_last_error remain valid.
 *   * Coordinates are global lattice cells (x fastest); the lattice interior
 *     is [0,nx) x [0,ny) x [0,nz); the one-cell shell is -1 and n.
 *   * Canonical PDF arrays are double [z][y][x][19] (centred f~, the
 *     post-collision state stored at its own cell, R6) over this rank's
 *     owned brick [owned_lo, owned_hi); non-fluid cells read back as 0.
 *   * No CPU fallback: every step of the update runs in the library's sm_100a
 *     kernels; on a machine without a usable B200 lbm_create fails with
 *     LBM_ERR_CUDA.
 */
#ifndef LBM_B200_H
#define LBM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define LBM_API __attribute__((visibility("default")))
#else
#define LBM_API
#endif

#define LBM_Q 19
#define LBM_ABI_VERSION 1
#define LBM_NCCL_ID_BYTES 128
#define LBM_MAX_WALL_VELOCITIES 254
#define LBM_NPHASES 8

typedef struct lbm_ctx lbm_ctx;

typedef enum {
    LBM_OK = 0,
    LBM_ERR_ARG = 1,      /* invalid argument; nothing changed                */
    LBM_ERR_STATE = 2,    /* ctx poisoned by an earlier CUDA/NCCL failure, or
                             call not valid in the current state              */
    LBM_ERR_OOM = 3,      /* device (or pinned host) allocation failed        */
    LBM_ERR_CUDA = 4,     /* CUDA runtime/driver error (message in last_error) */
    LBM_ERR_NCCL = 5,     /* NCCL error                                        */
    LBM_ERR_INTERNAL = 6
} lbm_status;

typedef enum { LBM_FP32 = 4, LBM_FP64 = 8 } lbm_precision; /* storage AND arithmetic (R15) */

/* Cell flags (D2 of SURVEY): 0 fluid, 1 no-slip wall,
 * 2 + k: wall moving with velocity wall_u[k] (k < nvel <= 254).              */
enum { LBM_FLUID = 0, LBM_NOSLIP = 1, LBM_VELOCITY0 = 2 };

/* PDF storage layout (north_star (a)).                   */
enum {
    LBM_LAYOUT_AB = 0, /* two PDF grids, pull from src, write dst, swap        */
    LBM_LAYOUT_AA = 1  /* one PDF grid, AA pattern: alternating in-place PULL / LOCAL
                          steps, half the memory; results equal LBM_LAYOUT_AB bitwise
                          after every even step count                               */
};

/* Exchange transport for neighbouring patches.                               */
enum {
    LBM_EXCHANGE_AUTO = 0,        /* direct ghost stores by the sweep (same GPU and, over
                                     NVLink, other GPUs); env LBM_EXCHANGE=nccl: NCCL  */
    LBM_EXCHANGE_FORCE_BUFFERS = 1, /* every neighbour patch, same-GPU ones included, goes
                                     pack -> buffer -> grouped ncclSend/ncclRecv -> unpack
                                     (P:287-313), shells first and overlapped with the
                                     interiors when overlap = 1; on one GPU through a
                                     one-rank communicator (the NCCL path, tested there) */
    LBM_EXCHANGE_SELF_PEER = 2     /* nranks == 1 only: every neighbour patch is reached as
                                     if on another GPU that is this one -- remote shells
                                     on the comm stream with direct stores through the
                                     peer table, one epoch handshake per step (the fused
                                     multi-GPU path, tested on one GPU)              */
};

/* Extended creation parameters (lbm_config_default fills the defaults).     */
typedef struct {
    int64_t domain[3];      /* global interior lattice (nx, ny, nz) > 0                         */
    int32_t patch[3];       /* patch (= paper Block) size; divides domain per axis    */
    double omega;           /* 1/tau, 0 < omega < 2 (nu = (1/omega - 1/2)/3)          */
    int32_t precision;      /* LBM_FP32 or LBM_FP64                                              */
    int32_t periodic[3];    /* 1 = periodic axis (ghosts wrap), 0 = walls in the one-cell shell  */
    int32_t device;         /* CUDA device ordinal; -1 = the calling thread's current device    */
    int32_t rank, nranks;   /* this process's rank among nranks (one process per GPU)          */
    int32_t proc_grid[3];   /* ranks per axis, product == nranks; {0,0,0} = default:
                               1 -> 1x1x1, 2 -> 1x1x2, 4 -> 1x2x2, 8 -> 2x2x2, else 1x1xN       */
    const void *nccl_unique_id; /* LBM_NCCL_ID_BYTES from lbm_nccl_unique_id on rank 0,
                                   same bytes on every rank; required iff nranks > 1            */
    int32_t exchange_mode;  /* LBM_EXCHANGE_*                                                    */
    int32_t overlap;        /* NCCL exchange: 1 = sweep patch shells first, exchange on a second
                               stream while the interiors are swept; 0 = sequential.  (The
                               fused exchange always sweeps remote shells on its own stream.) */
    int32_t use_graphs;     /* 1 = capture the step pair in a CUDA graph and replay it          */
    void *stream;           /* cudaStream_t for all compute launches; NULL = library-owned      */
    int32_t layout;         /* LBM_LAYOUT_AB or LBM_LAYOUT_AA                                    */
} lbm_config;

/* Per-ctx information (lbm_get_info).                                         */
typedef struct {
    int64_t domain[3];
    int32_t patch[3];
    int32_t precision;
    int32_t rank, nranks;
    int32_t proc_grid[3], proc_coord[3];
    int64_t owned_lo[3], owned_hi[3];      /* this rank's brick of cells                    */
    int32_t patches_local, patches_global;
    int32_t peers;                         /* distinct remote ranks exchanged with per step */
    int32_t messages_remote;               /* remote (patch, direction) segments sent/step  */
    int64_t fluid_cells_local, fluid_cells_global;  /* valid after lbm_set_flags          */
    int64_t steps_done;
    double bytes_per_step_algorithmic;     /* 2 * 19 * sizeof(real) * fluid_cells_local   */
    int64_t halo_bytes_remote_per_step;    /* bytes this rank sends to other ranks / step   */
    int64_t halo_bytes_local_per_step;     /* bytes exchanged between same-GPU patches / step
                                              (direct stores or copies)                     */
    int64_t kernel_launches;               /* cumulative library kernel launches            */
    int64_t device_bytes;                  /* device memory held by the ctx                 */
    /* Phase timing (lbm_set_timing): accumulated milliseconds and event counts.
       0 sweep (whole patches)  1 sweep_shell  2 sweep_interior  3 pack+local copy
       4 nccl  5 unpack  6 step total  7 reserved                                        */
    double phase_ms[LBM_NPHASES];
    int64_t phase_count[LBM_NPHASES];
    int64_t row_pitch_elems;               /* PDF row pitch: n_x rounded up to a 32-B sector
                                              (x ghosts live in compact side columns)       */
    int32_t align_bytes;                   /* alignment of every row start (32)             */
    int32_t graphs_active;
    int32_t layout;                        /* LBM_LAYOUT_*                                  */
    int32_t aa_phase;                      /* AA: 0 swapped (even step count), 1 streamed   */
    int32_t exchange_fused;                /* 1: the sweep stores outgoing PDFs straight into
                                              neighbour ghost layers (same GPU: plain stores,
                                              other GPUs: NVLink stores to CUDA-IPC-mapped
                                              memory, one epoch handshake per step);
                                              0: pack -> NCCL / copy -> unpack             */
    int32_t local_pull;                    /* always 0 (the round-1 local-pull sweep was
                                              measured slower and removed)                 */
    int32_t local_direct;                  /* 1: the sweep stores the outgoing PDFs of face /
                                              edge cells straight into same-GPU neighbour
                                              patches' ghost layers (no ghost copies)     */
    int32_t overlap_active;                /* 1: buffered exchange with shells first and the
                                              transport overlapped with the interior sweep */
    int32_t nccl_ranks;                    /* size of the ctx's NCCL communicator (0: none;
                                              1: one-GPU FORCE_BUFFERS self-peer messages)  */
    int32_t fused_peers;                   /* peers of the fused exchange's epoch handshake
                                              (SELF_PEER on one GPU: 1, this rank)          */
    int32_t reserved0;
} lbm_info;

/* One remote message of the static exchange plan (lbm_plan, host-only).      */
typedef struct {
    int32_t peer;            /* other rank                                               */
    int32_t send;            /* 1 = this rank sends, 0 = this rank receives              */
    int32_t patch_local;     /* global id of this rank's patch (sender or receiver)      */
    int32_t patch_remote;    /* global id of the peer's patch                            */
    int32_t dir[3];          /* direction from the receiving patch to the sending patch  */
    int32_t nq;              /* PDFs per cell: 5 (face) or 1 (edge)                      */
    int64_t cells;           /* cells in the segment                                     */
    int64_t offset;          /* element offset of the segment inside the peer message   */
} lbm_msg;

/* Library / ABI version (== LBM_ABI_VERSION).                                 */
LBM_API int32_t lbm_abi_version(void);

/* Fill *cfg with defaults: single rank, device -1, exchange AUTO, overlap 1,
 * graphs 1, not periodic, omega 1/0.65, fp64.  domain/patch must be set.     */
LBM_API void lbm_config_default(lbm_config *cfg);

/* North-star minimal form (BASELINE.json): single GPU (current device),
 * non-periodic, one rank.  domain[3] > 0, patch[3] divides domain,
 * 0 < omega < 2, precision in {LBM_FP32, LBM_FP64}.  On success *out is a
 * ctx holding a closed no-slip box at rest (f~ = 0), valid for lbm_step.  */
LBM_API lbm_status lbm_create(const int64_t domain[3], const int32_t patch[3], double omega,
                              int32_t precision, lbm_ctx **out);

/* Extended form (periodic axes, device choice, multi-rank over NCCL).        */
LBM_API lbm_status lbm_create_ex(const lbm_config *cfg, lbm_ctx **out);

/* Frees every resource of ctx; NULL-safe; valid on a poisoned ctx.           */
LBM_API lbm_status lbm_destroy(lbm_ctx *ctx);

/* Cell flags for the WHOLE global lattice incl. its one-cell shell:
 * (LBM_LAYOUT_AA: only valid after an even number of steps since the last
 * set_pdfs / init_noise, else LBM_ERR_STATE.)
 * uint8 [(nz+2)][(ny+2)][(nx+2)], x fastest (every rank passes the same
 * array).  wall_u: nvel x 3 doubles, velocity of flag 2 + k (may be NULL when
 * nvel == 0).  Shell cells on non-periodic axes must be non-fluid, and every
 * flag >= 2 must satisfy flag - 2 < nvel, else LBM_ERR_ARG.  On periodic axes
 * the shell entries are ignored (ghosts wrap).  The PDF state is kept.      */
LBM_API lbm_status lbm_set_flags(lbm_ctx *ctx, const uint8_t *flags, const double *wall_u, int32_t nvel);

/* Read back the flags of this rank's owned brick plus its one-cell shell as
 * stored on the device: uint8 [(hz-lz+2)][(hy-ly+2)][(hx-lx+2)].           */
LBM_API lbm_status lbm_get_flags(lbm_ctx *ctx, uint8_t *flags_out);

/* Set the state: canonical double [z][y][x][19] over the owned brick
 * (converted to the ctx precision on the device), then refresh ghosts.       */
LBM_API lbm_status lbm_set_pdfs(lbm_ctx *ctx, const double *f);

/* Set the state to the seeded dyadic noise of paper_1007_1388_b200/inputs.py
 * (f~ = k / 2^20, k = splitmix64-derived in [-1024, 1024], counter-based over
 * the global (cell, i) index), drawn on the device; then refresh ghosts.     */
LBM_API lbm_status lbm_init_noise(lbm_ctx *ctx, uint64_t seed);

/* Advance nsteps time steps (nsteps >= 0).  Returns after the work is done
 * (synchronous).                                                              */
LBM_API lbm_status lbm_step(lbm_ctx *ctx, int64_t nsteps);

/* Enqueue nsteps time steps on the ctx stream and return immediately;
 * lbm_synchronize waits for them.                                            */
LBM_API lbm_status lbm_step_async(lbm_ctx *ctx, int64_t nsteps);
LBM_API lbm_status lbm_synchronize(lbm_ctx *ctx);

/* Canonical PDFs of the owned brick -> f_out (double [z][y][x][19]).       */
LBM_API lbm_status lbm_get_pdfs(lbm_ctx *ctx, double *f_out);

/* PDFs at n explicit global cells (xyz[3*k .. 3*k+2], owned by this rank)
 * -> out[19*k .. 19*k+18].  Cells outside the owned brick: LBM_ERR_ARG.     */
LBM_API lbm_status lbm_get_pdfs_at(lbm_ctx *ctx, const int64_t *xyz, int64_t n, double *out);

/* Macroscopic fields of the owned brick: rho = rho0 + sum f~_i,
 * u = sum e_i f~_i / rho0 at fluid cells; rho = 0, u = 0 at non-fluid cells.
 * rho_out: double [z][y][x]; u_out: double [z][y][x][3].  Either may be NULL. */
LBM_API lbm_status lbm_get_macroscopic(lbm_ctx *ctx, double *rho_out, double *u_out);

/* Total mass of the whole lattice: sum over all fluid cells of rho = rho0 +
 * sum_i f~_i (conserved by the collision and the bounce-back,
 * SURVEY V6), computed on the device in fp64 (deterministic on each rank) and
 * summed over the ranks with one NCCL all-reduce -- a collective: every rank
 * must call it.  Off the hot path (reads the whole state).  mass_out: caller-
 * owned double, the same value on every rank.                                */
LBM_API lbm_status lbm_total_mass(lbm_ctx *ctx, double *mass_out);

LBM_API lbm_status lbm_get_info(lbm_ctx *ctx, lbm_info *out);

/* Enable (1) / disable (0) per-phase CUDA-event timing inside lbm_step;
 * enabling also resets the accumulated phase_ms / phase_count.               */
LBM_API lbm_status lbm_set_timing(lbm_ctx *ctx, int32_t enable);

/* The cudaStream_t all compute kernels are launched on.                      */
LBM_API lbm_status lbm_get_stream(lbm_ctx *ctx, void **stream_out);

/* Message of the last failing call on ctx (ctx == NULL: last create error);
 * valid until the next call on that ctx.  Never NULL.                        */
LBM_API const char *lbm_last_error(const lbm_ctx *ctx);

/* ncclGetUniqueId into out (nbytes >= LBM_NCCL_ID_BYTES); call on rank 0 and
 * broadcast the bytes to the other ranks (e.g. with torch.distributed).     */
LBM_API lbm_status lbm_nccl_unique_id(void *out, int64_t nbytes);

/* Host-only (no GPU, no CUDA calls): the static decomposition and remote
 * exchange plan this rank would use for cfg.  info receives the decomposition
 * fields of lbm_info (domain, patch, proc grid/coord, owned box, patch counts,
 * peers, messages_remote, halo bytes for cfg->precision); msgs (capacity cap,
 * may be NULL) receives the remote messages, sends then receives, each in the
 * canonical (receiving patch id, direction) order; *nmsgs = total count.     */
LBM_API lbm_status lbm_plan(const lbm_config *cfg, lbm_info *info, lbm_msg *msgs, int32_t cap,
                            int32_t *nmsgs);

#ifdef __cplusplus
}
#endif
#endif /* LBM_B200_H */
