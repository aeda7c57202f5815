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
    bool solid;       // the tile holds a non-fluid cell (launch_tile_solid)
    bool xlo, xhi;    // the patch's -x / +x side is a uniform wall (launch_sidewall) ...
    int flo, fhi;     // ... with this flag
};

template <typename real>
__device__ __forceinline__ PairCoord locate_pair(const SweepArgs<real> &a)
{
    const int4 t = __ldg(a.tiles + blockIdx.x);
    PairCoord c;
    c.patch = t.x & 0x1fffffff;
    c.solid = t.x < 0;
    c.xlo = (t.x >> 30) & 1;
    c.xhi = (t.x >> 29) & 1;
    c.flo = (t.w >> 16) & 0xff;
    c.fhi = (int)((unsigned)t.w >> 24);
    c.x0 = (int)((unsigned)t.y >> 16) + 2 * (int)threadIdx.x;
    c.xend = t.y & 0xffff;
    c.y = (int)((unsigned)t.z >> 16) + (int)threadIdx.y;
    c.z = t.w & 0xffff;
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

// Global loads / stores of PDF values (kernels.cuh Checker): plain __ldg / store
// in the product build, checked and recorded in the checked build.
#ifdef LBM_CHECKED
// out of line in the checked build: inlined at every access it made ptxas take minutes
static __device__ __noinline__ void ck_access(const Checker &c, const void *p, int bytes, bool write)
#else
__device__ __forceinline__ void ck_access(const Checker &c, const void *p, int bytes, bool write)
#endif
{
#ifdef LBM_CHECKED
    const char *cp = static_cast<const char *>(p);
    int gi = -1;
    for (int k = 0; k < 2; ++k)
        if (c.lo[k] && cp >= c.lo[k] && cp + bytes <= c.hi[k]) gi = k;
    if (gi < 0 || ((uintptr_t)cp % (uintptr_t)bytes) != 0) {
        atomicAdd(c.err + 0, 1ull);
        return;
    }
    const int64_t e0 = (int64_t)((cp - c.lo[gi]) / c.esize);
    const unsigned long long tid =
        (unsigned long long)blockIdx.x * blockDim.x * blockDim.y + threadIdx.y * blockDim.x + threadIdx.x + 1;
    const unsigned long long id = c.launch | tid;
    for (int k = 0; k < bytes / c.esize; ++k) {
        const int64_t e = gi * c.elems + e0 + k;
        if (write) {
            if (atomicExch(c.wr + e, id) != 0ull) atomicAdd(c.err + 1, 1ull);
            const unsigned long long r = atomicAdd(c.rd + e, 0ull);
            if (r != 0ull && (r >> 32) == (id >> 32) && r != id) atomicAdd(c.err + 2, 1ull);
        } else {
            atomicExch(c.rd + e, id);
            const unsigned long long w = atomicAdd(c.wr + e, 0ull);
            if (w != 0ull && (w >> 32) == (id >> 32) && w != id) atomicAdd(c.err + 2, 1ull);
        }
    }
#else
    (void)c;
    (void)p;
    (void)bytes;
    (void)write;
#endif
}
template <typename T>
__device__ __forceinline__ T gld(const Checker &c, const T *p)
{
    ck_access(c, p, (int)sizeof(T), false);
    return __ldg(p);
}
template <typename T>
__device__ __forceinline__ void gst(const Checker &c, T *p, const T &v)
{
    ck_access(c, p, (int)sizeof(T), true);
    *p = v;
}

// two cells per thread along x: the 2-vector type of the storage precision
template <typename real> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

}  // namespace lbm
