// kernels.cuh -- launch wrappers of the sm_100a kernels (sweep.cu, sweep_aa.cu, aux_kernels.cu, handshake.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "lbm_internal.h"

namespace lbm {

// Sweep launch configuration: BX threads along x (one warp-row = 32 cells),
// BY rows along y per block.
constexpr int SWEEP_BX = 64;
constexpr int SWEEP_BY = 4;

// Per-direction byte offsets, uniform over a launch and filled on the host
// (fill_dir_offsets), so that each of a thread's 38 pull addresses and 19 store
// addresses is its base pointer plus a kernel-parameter constant -- one 64-bit
// add -- instead of a per-thread multiply / shift chain (the integer address
// arithmetic was 45 % of the fp32 sweep's instructions, profiles/r02_*).
//   pull[i]  : p_i of the pair's first cell: slot(i) * qs - e_i . (1, px, plane),
//              relative to the cell's element in slice 0 (slot(i) = i two-grid,
//              opp(i) AA PULL); the second cell's value is one element further;
//   gpull[i] : e_ix != 0, the x-ghost column element it pulls instead at a row
//              end: slot(i) * gq + (e_ix > 0 ? 0 : gside) - e_iy - e_iz * gy,
//              relative to the cell's ghost-column base (side 0, q 0, (y, z));
//   slot[i]  : i * qs (slot i at the cell);
//   oslot[i] : opp(i) * qs (AA LOCAL's stores; a separate table so that ptxas
//              re-derives the store addresses instead of keeping the 19 load
//              addresses live through the collision);
//   push[i]  : AA PULL scatter target x + e_i in slot i: i * qs + e_i . (1, px, plane);
//   gpush[i] : e_ix != 0, the x-ghost column target of a row-end scatter:
//              i * gq + (e_ix < 0 ? 0 : gside) + e_iy + e_iz * gy;
//   gwall[i] : e_ix != 0, the half-way bounce-back slot of the x-ghost wall
//              cell x + e_i: opp(i) * gq + (e_ix < 0 ? 0 : gside) + e_iy + e_iz * gy;
//   wall[i]  : the same slot of a wall cell x + e_i in the main slices (a y / z
//              ghost row or plane): opp(i) * qs + e_i . (1, px, plane).
struct DirOffsets {
    int64_t pull[Q], gpull[Q], slot[Q], oslot[Q], push[Q], gpush[Q], gwall[Q], wall[Q];
};
void fill_dir_offsets(const Geom &g, bool aa, int esize, DirOffsets &o);

// Checked build (make checked, -DLBM_CHECKED; tools/check_cases.py): every
// global load / store of the sweeps, the direct ghost stores and the bounce-back
// list is checked to lie inside the PDF grid allocations, and shadow arrays
// record per element the last writer and reader (id = launch sequence << 32 |
// thread + 1) over one time step.  Counted errors: [0] an access outside the
// grids or misaligned, [1] an element written twice in one step (the
// single-writer claim), [2] an element read by one thread and written by
// another in the same launch (a race of the in-place AA kernels).  The
// product build carries an empty Checker.
#ifdef LBM_CHECKED
struct Checker {
    const char *lo[2] = {nullptr, nullptr}, *hi[2] = {nullptr, nullptr};
    unsigned long long *wr = nullptr, *rd = nullptr;  // [2][elems]
    unsigned long long *err = nullptr;                  // [3]
    int64_t elems = 0;                                  // elements per grid
    int esize = 8;
    int inject = 0;  // LBM_CHECKED_INJECT=1: the bounce-back list stores twice (the checker's negative control)
    unsigned long long launch = 0;
};
#else
struct Checker {};
#endif

template <typename real>
struct SweepArgs {
    const real *src;
    real *dst;
    const uint8_t *kind;    // [patch][fs] 0 fluid (all neighbours fluid), 1 fluid next to a wall, 2 non-fluid
    const real *corr;       // [nvel][19]: 6 w_i rho0 (e_i . u_w[k]) rounded to real
    Geom g;
    real omega;
    const int4 *tiles;      // device: one descriptor per block (context.h DevBoxes)
    const unsigned long long *sidewall = nullptr;  // [patch] uniform-wall sides (launch_sidewall), two grids
    // Direct ghost stores: [nlocal][18][2] base of the neighbour patch (same GPU,
    // or peer-mapped) in grid i, null where the copy path serves it.  Face / edge
    // cells store their outgoing PDFs into that patch's ghost cells of grid dsti.
    // dnbr == nullptr disables them.
    real *const *dnbr = nullptr;
    int dsti = 0;
    DirOffsets off;
    Checker chk;
};

// The 18 neighbour directions in the plan's order (plan.cpp kDirs).
__host__ __device__ constexpr int ndir(int k, int a)
{
    constexpr int t[NDIR][3] = {{0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {1, 0, -1}, {0, 1, -1}, {-1, -1, 0},
                                {0, -1, 0},  {1, -1, 0},  {-1, 0, 0}, {1, 0, 0},  {-1, 1, 0}, {0, 1, 0},
                                {1, 1, 0},   {0, -1, 1},  {-1, 0, 1}, {0, 0, 1},  {1, 0, 1},  {0, 1, 1}};
    return t[k][a];
}

// Does direction q travel into the neighbour at d (e_q[a] == d[a] on every
// axis where d is non-zero)?  5 q per face, 1 per edge.
__host__ __device__ constexpr bool outgoing(int q, int k)
{
    return q != 0 && (ndir(k, 0) == 0 || EXf(q) == ndir(k, 0)) && (ndir(k, 1) == 0 || EYf(q) == ndir(k, 1)) &&
           (ndir(k, 2) == 0 || EZf(q) == ndir(k, 2));
}

// Two-grid sweep (sweep.cu): two cells per thread along x, 2-vector accesses;
// variant 0: default occupancy (fp64 3, fp32 4 blocks of 128 threads per SM),
// 1: the alternative (fp64 2, fp32 5).
template <typename real>
cudaError_t launch_sweep(const SweepArgs<real> &a, int64_t total_tiles, int variant, cudaStream_t s);
constexpr int kSweepVariants = 2;

// Fused-exchange handshake (handshake.cu).
cudaError_t launch_wait_peers(const unsigned long long *inbox, const int *peer_rank, int npeers,
                              const unsigned long long *epoch, int *error, cudaStream_t s);
cudaError_t launch_signal_peers(unsigned long long *epoch, unsigned long long *const *peer_inbox, int npeers,
                                cudaStream_t s);

// Total mass: sum of delta rho over the owned fluid cells into *out (fp64,
// deterministic; partial: kMassBlocks doubles of scratch).
constexpr int kMassBlocks = 1024, kMassThreads = 256;
template <typename real>
cudaError_t launch_mass(const real *grid, const uint8_t *flags, const int64_t owned_lo[3], const int64_t on[3],
                        const int brick[3], const Geom &g, int rep, const real *corr, double *partial, double *out,
                        cudaStream_t s);

template <typename real>
cudaError_t launch_copy_segments(const CopySeg *segs, int nseg, int64_t max_elems, const real *grid_src,
                                 real *grid_dst, const real *buf_src, real *buf_dst, const uint8_t *flags,
                                 const Geom &g, cudaStream_t s);

// Half-way bounce-back over the list of wall-adjacent fluid cells (modes in
// aux_kernels.cu bb_list_kernel: 0 two-grid store side, 1 AA LOCAL store side /
// swapped state, 2 AA PULL fix-up), after every sweep and once after the state
// or the flags are set.  One entry per cell, in ascending memory order: its
// position, wall mask (bit j: x + e_j is non-fluid) and
// vinfo = bits j of the moving walls | their shared velocity index << 24
// (kBbMixed: the walls move differently -- read each wall's flag).
struct BbEntry {
    uint64_t pos;  // patch << 45 | z << 30 | y << 15 | x (bb_pos)
    uint32_t mask, vinfo;
};
__host__ __device__ constexpr uint64_t bb_pos(int patch, int x, int y, int z)
{
    return (uint64_t)patch << 45 | (uint64_t)z << 30 | (uint64_t)y << 15 | (uint64_t)x;
}
// Byte offsets of a wall link x -> w = x + e_j in the bounce-back list kernel,
// uniform over a launch (filled on the host per mode, fill_bb_offsets): xs[j]
// the slot of x it reads or writes (relative to x's element in slice 0), wm[j]
// the slot of w when w lies in the main slices (same base), wg[j] when w is an
// x ghost (relative to x's ghost-column base, ghost_base).
struct BbOffsets {
    int64_t xs[Q], wm[Q], wg[Q];
};
void fill_bb_offsets(const Geom &g, int mode, int esize, BbOffsets &o);
constexpr uint32_t kBbMixed = 255;
template <typename real>
cudaError_t launch_bb_list(real *grid, const uint8_t *flags, const BbEntry *list, int64_t n, const real *corr,
                           const Geom &g, int mode, const BbOffsets &o, const Checker &ck, cudaStream_t s);
// Building the list (kind == 1 cells of all `total` flag-layout elements): per-chunk
// counts (bb_list_chunks(total) of them), then, with their exclusive scan, the entries.
int64_t bb_list_chunks(int64_t total);
// sidewall (launch_sidewall; null: every link) drops the links of the inner face
// cells of uniform-wall sides from the list: the two-grid sweep stores those itself.
cudaError_t launch_bb_list_count(const uint8_t *kind, const uint32_t *wmask, const unsigned long long *sidewall,
                                 int64_t total, const Geom &g, int64_t *counts, cudaStream_t s);
cudaError_t launch_bb_list_write(const uint8_t *kind, const uint32_t *wmask, const uint8_t *flags,
                                 const unsigned long long *sidewall, int64_t total, const Geom &g,
                                 const int64_t *offsets, BbEntry *list, cudaStream_t s);
// Per local patch, bits s = 2 axis + (0 low, 1 high): that side is a uniform wall --
// every ghost cell the side's inner face cells (the other two coordinates in
// [1, n - 2]) link to, i.e. the ghost layer's part over the face, carries one
// non-fluid flag, kept in bits 8 + 8 s .. 15 + 8 s.
cudaError_t launch_sidewall(const uint8_t *flags, int nlocal, const Geom &g, unsigned long long *sidewall,
                            cudaStream_t s);
__host__ __device__ constexpr int side_flag(unsigned long long sw, int side) { return (int)((sw >> (8 + 8 * side)) & 0xff); }
// Tile bits: 31 of the patch field, the tile holds a non-fluid cell; 30 / 29, its
// patch's -x / +x side is a uniform wall (sidewall; null: none), whose flag goes
// to bits 16-23 / 24-31 of the z field.
cudaError_t launch_tile_solid(int4 *tiles, int64_t n, const uint8_t *kind, const unsigned long long *sidewall,
                              const Geom &g, cudaStream_t s);

// AA-pattern in-place sweeps (sweep_aa.cu): pull = true -> PULL kernel, else LOCAL;
// variant as launch_sweep.
template <typename real>
cudaError_t launch_sweep_aa(const SweepArgs<real> &a, int64_t total_tiles, bool pull, int variant, cudaStream_t s);

// Build per-patch flags (incl. ghosts, periodic wrap) from the global flag
// array (device copy, (nz+2)(ny+2)(nx+2)), then the per-cell kind and the
// wall-neighbour masks of kind-1 cells.
cudaError_t launch_build_flags(const uint8_t *global, const int64_t domain[3], const int periodic[3],
                               const int *patch_origin /*3 per local patch*/, int nlocal, const Geom &g,
                               uint8_t *flags, uint8_t *kind, uint32_t *wmask, cudaStream_t s);

// Import / export between the canonical double [z][y][x][19] layout of a
// range of owned z-planes and the patch grids.  rep: 0 two-grid, 1 AA
// swapped, 2 AA streamed (export / gather only).
template <typename real>
cudaError_t launch_import(const double *canon, int64_t z0, int64_t nz_chunk, const int64_t owned_lo[3],
                          const int64_t owned_n[3], const int brick[3], const Geom &g, real *grid, int rep,
                          cudaStream_t s);
template <typename real>
cudaError_t launch_export(const real *grid, const uint8_t *flags, int64_t z0, int64_t nz_chunk,
                          const int64_t owned_lo[3], const int64_t owned_n[3], const int brick[3],
                          const Geom &g, double *canon, int mode /*0 pdfs, 1 macroscopic*/, double *rho,
                          double *u, int rep, const real *corr, cudaStream_t s);
template <typename real>
cudaError_t launch_noise(real *grid, uint64_t seed, const int64_t domain[3], const int64_t owned_lo[3],
                         const int64_t owned_n[3], const int brick[3], const Geom &g, int rep, cudaStream_t s);
template <typename real>
cudaError_t launch_gather(const real *grid, const uint8_t *flags, const int64_t *xyz_local /*3 per cell*/,
                          int64_t n, const int brick[3], const Geom &g, double *out, int rep, const real *corr,
                          cudaStream_t s);

}  // namespace lbm
