// sweep_common.cuh -- device helpers shared by the sweep kernels (sweep.cu,
// sweep_aa.cu) and the auxiliary kernels (aux_kernels.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace lbm {

// shift of the y / z neighbour of direction i inside a main q-slice (x is handled
// separately: the x neighbours of the row ends live in the x-ghost columns)
__device__ __forceinline__ int64_t yz_shift(const Geom &g, int i)
{
    return EY(i) * (int64_t)g.px + EZ(i) * g.plane;
}

// shift of neighbour x + e_i in the flag / kind layout (has an in-row x ghost)
__device__ __forceinline__ int64_t flag_shift(const Geom &g, int i)
{
    return EX(i) + EY(i) * (int64_t)g.fpx + EZ(i) * g.fplane;
}

// Locate the box and the cell pair of this block / thread: tiles of 64 x 4 cells
// of one z plane (two cells per thread along x), the box found by a binary
// search over the tile prefix sums.
struct PairCoord {
    int patch, x0, y, z, xend;
    bool valid;
};

template <typename real>
__device__ __forceinline__ PairCoord locate_pair(const SweepArgs<real> &a)
{
    const int64_t b = blockIdx.x;
    int lo = 0, hi = a.nboxes;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a.tile_prefix[mid] <= b) lo = mid; else hi = mid;
    }
    const Box &bx = a.boxes[lo];
    int t = (int)(b - a.tile_prefix[lo]);
    const int tiles_x = bx.tiles_x, tiles_y = bx.tiles_y;
    const int tx = t % tiles_x;
    t /= tiles_x;
    const int ty = t % tiles_y;
    const int tz = t / tiles_y;
    PairCoord c;
    c.patch = bx.patch;
    c.x0 = bx.lo[0] + tx * SWEEP_BX + 2 * (int)threadIdx.x;
    c.y = bx.lo[1] + ty * SWEEP_BY + (int)threadIdx.y;
    c.z = bx.lo[2] + tz;
    c.xend = bx.lo[0] + bx.n[0];
    c.valid = c.x0 < c.xend && c.y < bx.lo[1] + bx.n[1];
    return c;
}

// two cells per thread along x: the 2-vector type of the storage precision
template <typename real> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

}  // namespace lbm
