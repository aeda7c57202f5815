// sweep_common.cuh -- device helpers shared by the sweep kernels (sweep.cu,
// sweep_aa.cu) and the auxiliary kernels (aux_kernels.cu).
#pragma once

#include <cstdint>
#include <type_traits>

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

// The cell pair of this thread: the block's 64 x 4-cell tile of one z plane
// from its descriptor (one 16-B load, context.h DevBoxes; bit 31 of the patch
// field: the tile holds a non-fluid cell), two cells per thread along x.
struct PairCoord {
    int patch, x0, y, z, xend;
    bool valid;
    bool solid;  // the tile holds a non-fluid cell (launch_tile_solid)
};

template <typename real>
__device__ __forceinline__ PairCoord locate_pair(const SweepArgs<real> &a)
{
    const int4 t = __ldg(a.tiles + blockIdx.x);
    PairCoord c;
    c.patch = t.x & 0x7fffffff;
    c.solid = t.x < 0;
    c.x0 = (int)((unsigned)t.y >> 16) + 2 * (int)threadIdx.x;
    c.xend = t.y & 0xffff;
    c.y = (int)((unsigned)t.z >> 16) + (int)threadIdx.y;
    c.z = t.w;
    c.valid = c.x0 < c.xend && c.y < (t.z & 0xffff);
    return c;
}

// base pointer + byte offset (DirOffsets)
template <typename T, typename B>
__device__ __forceinline__ T *at(B *base, int64_t off)
{
    using C = typename std::conditional<std::is_const<B>::value || std::is_const<T>::value, const char, char>::type;
    return reinterpret_cast<T *>(reinterpret_cast<C *>(base) + off);
}

// x-ghost column base of cell row (y, z): side 0, q 0 (add DirOffsets gpull / gpush)
template <typename real>
__device__ __forceinline__ real *ghost_base(const Geom &g, real *P, int y, int z)
{
    return P + g.gbase + (int64_t)(z + 1) * g.gy + (y + g.gyo);
}

// two cells per thread along x: the 2-vector type of the storage precision
template <typename real> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

}  // namespace lbm
