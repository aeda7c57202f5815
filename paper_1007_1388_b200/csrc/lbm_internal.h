// lbm_internal.h -- internal definitions of the B200 D3Q19 patch solver.
// Product code: shares nothing with oracle/ (own direction table, own layouts).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "lbm.h"

namespace lbm {

constexpr int Q = 19;

// Frozen D3Q19 order (include/lbm.h, R2).  Opposites are i, i+1.
// P:403-405 (D3Q19), P:441-442 (weights 1/3, 1/18, 1/36).  Stored as bit
// masks so that host and device code fold them at compile time.
//   i : 0 | 1 2 3 4 5 6 | 7 8 9 10 11 12 13 14 15 16 17 18
constexpr unsigned kXP = (1u << 1) | (1u << 7) | (1u << 9) | (1u << 11) | (1u << 13);
constexpr unsigned kXM = (1u << 2) | (1u << 8) | (1u << 10) | (1u << 12) | (1u << 14);
constexpr unsigned kYP = (1u << 3) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 17);
constexpr unsigned kYM = (1u << 4) | (1u << 8) | (1u << 9) | (1u << 16) | (1u << 18);
constexpr unsigned kZP = (1u << 5) | (1u << 11) | (1u << 14) | (1u << 15) | (1u << 18);
constexpr unsigned kZM = (1u << 6) | (1u << 12) | (1u << 13) | (1u << 16) | (1u << 17);
__host__ __device__ constexpr int EXf(int i) { return (int)((kXP >> i) & 1u) - (int)((kXM >> i) & 1u); }
__host__ __device__ constexpr int EYf(int i) { return (int)((kYP >> i) & 1u) - (int)((kYM >> i) & 1u); }
__host__ __device__ constexpr int EZf(int i) { return (int)((kZP >> i) & 1u) - (int)((kZM >> i) & 1u); }
__host__ __device__ constexpr int OPPf(int i) { return i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1); }
__host__ __device__ constexpr double Wf(int i) { return i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0); }
#define EX(i) ::lbm::EXf(i)
#define EY(i) ::lbm::EYf(i)
#define EZ(i) ::lbm::EZf(i)
#define OPP(i) ::lbm::OPPf(i)
#define WQ(i) ::lbm::Wf(i)

// The 18 patch-neighbour directions (6 faces + 12 edges; D3Q19 has no corner
// velocities, so corner ghosts are never read).  Fixed order = ABI of the
// exchange plan: lexicographic over (dz, dy, dx) in {-1,0,1}^3 minus the
// centre and the 8 corners.
constexpr int NDIR = 18;
struct Dir3 { int d[3]; };

// Patch geometry shared by every patch of a ctx (all patches have one size).
// PDF storage of one patch (elements, back to back; patches back to back):
//   main q-slices  [q][z = -1..n2][y = -1..n1][x = 0..n0-1]: rows of exactly
//                  n0 cells (px = n0 rounded up to a 32-B sector, = n0 for
//                  every BASELINE size) with the y / z ghost rows and planes;
//   x-ghost columns [q][side][z = -1..n2][y = -1..n1] (side 0: x = -1,
//                  side 1: x = n0), y = 0 on a sector boundary.
// Unpadded rows stream better than rows padded for an in-row x ghost (the
// access pattern's own ceiling drops 5-7 % at 256^3 and 17 % for 64^3 patches,
// profiles/r01_stream_ceiling_*compact.log), and a patch's x faces become
// y-contiguous runs for the exchange.
// Flags and cell kinds (uint8) keep an in-row x ghost: [z][y][x = -1..n0],
// row pitch fpx, x = 0 at offset fxo (even, so a cell pair is one uchar2).
struct Geom {
    int n[3];        // patch interior size
    int px, py;      // PDF row pitch (elements), rows per plane (n1 + 2)
    int64_t plane;   // px * py
    int64_t qs;      // elements per main q-slice (plane * (n2 + 2), rounded up to 32)
    int gy, gyo;     // x-ghost column: pitch per z plane, offset of y = 0
    int64_t gside;   // gy * (n2 + 2): one x-ghost column (one side, one q)
    int64_t gq;      // 2 * gside: both sides of one q
    int64_t gbase;   // Q * qs: start of the x-ghost columns in a patch
    int64_t ps;      // elements per patch (main + ghosts, rounded up to 32)
    int fpx, fxo;    // flag row pitch, offset of x = 0 in a flag row
    int64_t fplane;  // fpx * py
    int64_t fs;      // flag bytes per patch = fplane * (n2 + 2)
};

#ifndef __CUDACC__
#define LBM_HD inline
#else
#define LBM_HD __host__ __device__ __forceinline__
#endif
// element of interior cell (x, y, z), 0 <= x < n0, -1 <= y <= n1, -1 <= z <= n2, in a main q-slice
LBM_HD int64_t main_index(const Geom &g, int x, int y, int z)
{
    return ((int64_t)(z + 1) * g.py + (y + 1)) * (int64_t)g.px + x;
}
// element of x-ghost cell (side 0: x = -1, 1: x = n0) of direction q, relative to the patch base
LBM_HD int64_t ghost_index(const Geom &g, int q, int side, int y, int z)
{
    return g.gbase + (int64_t)q * g.gq + side * g.gside + (int64_t)(z + 1) * g.gy + (y + g.gyo);
}
// element of PDF q of any cell -1 <= x, y, z <= n, relative to the patch base
LBM_HD int64_t pdf_index(const Geom &g, int q, int x, int y, int z)
{
    if (x < 0) return ghost_index(g, q, 0, y, z);
    if (x >= g.n[0]) return ghost_index(g, q, 1, y, z);
    return (int64_t)q * g.qs + main_index(g, x, y, z);
}
// flag / kind byte of cell (x, y, z), relative to the patch's flag base
LBM_HD int64_t flag_index(const Geom &g, int x, int y, int z)
{
    return ((int64_t)(z + 1) * g.py + (y + 1)) * (int64_t)g.fpx + (x + g.fxo);
}

// Sweep box: cells [lo, lo + n) of local patch `patch`.
struct Box {
    int patch;
    int lo[3];
    int n[3];
    int tiles_x, tiles_y;
};

// Copy segment of the ghost exchange (pack, local copy or unpack).
// src/dst are either a PDF grid region (cells lo..lo+size of local patch at
// element base) or a linear buffer at element base.  Element order inside a
// segment: q-list major, then cells x fastest.
struct CopySeg {
    int64_t src_base, dst_base;
    int64_t dst_flag_base;          // flag offset of the destination patch (grid destinations)
    int32_t mask;                   // 0: write grid destinations only into fluid cells;
                                    // 1: every destination cell is fluid (no check);
                                    // 2: AA half-exchange 2 -- additionally the writer cell
                                    //    y - e_q must be fluid and inside the sender (see plan.cpp)
    int32_t d[3];                   // direction from the receiving patch to the sending patch
    int32_t src_is_buf, dst_is_buf;
    int32_t src_lo[3], dst_lo[3], size[3];
    int32_t nq;
    int32_t q[5];
    int64_t cells;
    int64_t nelem;
};

// Host-only decomposition (no CUDA): plan.cpp.
struct Seg {
    int recv_patch, send_patch;   // global patch ids
    int dir;                      // direction index (0..17) from receiver to sender
    int d[3];
    int nq, q[5];
    int size[3];
    int recv_lo[3];               // ghost region in the receiving patch (local coords)
    int send_lo[3];               // boundary region in the sending patch
    int64_t cells;
    int peer;                     // other rank (remote) or own rank
    int64_t offset;               // element offset inside the peer message
};

struct Decomp {
    int64_t domain[3];
    int patch[3];
    int pgrid[3];        // patches per axis (global)
    int proc[3];         // ranks per axis
    int coord[3];        // this rank's coordinate
    int brick[3];        // patches per rank per axis
    int rank, nranks;
    int periodic[3];
    int force_buffers;
    int64_t owned_lo[3], owned_hi[3];
    int nlocal;                   // local patches
    // local patch l <-> global id; local order = brick-local z, y, x
    int local_to_global(int l) const;
    int global_to_local(int g) const;   // -1 if not owned
    int local_index_on_owner(int g) const;  // storage index of g on its owning rank
    int owner(int g) const;
    void patch_coord(int g, int c[3]) const;
    int patch_id(const int c[3]) const;
};

// Returns an error message (empty on success).
const char *decompose(const lbm_config &cfg, Decomp &dec);
// Build the segment lists: local copies, sends and receives (sorted per peer
// in the canonical (receiving patch, dir) order, offsets filled in).
struct SegLists {
    std::vector<Seg> local;   // same-rank ghost copies (exchange_mode AUTO)
    std::vector<Seg> send;    // grouped by peer (ascending), canonical order inside
    std::vector<Seg> recv;
};
// Exchange kinds (d = direction from the receiving patch to the sending patch):
//   EX_AB : two-grid pull.  sender boundary layer -> receiver ghost layer,
//           slots q with e_q[a] = -d[a] (the PDFs the receiver's cells pull).
//   EX_AA1: AA half-exchange 1 (after the local step).  Same regions, slots
//           e_q[a] = +d[a] (swapped post-collision values the receiver's next
//           pull step gathers from its ghost layer).
//   EX_AA2: AA half-exchange 2 (after the pull step).  sender GHOST layer ->
//           receiver BOUNDARY layer, slots e_q[a] = -d[a] (what the sender's
//           cells scattered into their ghost layer belongs to the receiver).
enum ExKind { EX_AB = 0, EX_AA1 = 1, EX_AA2 = 2 };
void build_segments(const Decomp &dec, SegLists &out, int kind = EX_AB);
// Neighbour patch of global patch g in direction d (periodic wrap), or -1.
int neighbour(const Decomp &dec, int g, const int d[3]);
extern const Dir3 kDirs[NDIR];

}  // namespace lbm
