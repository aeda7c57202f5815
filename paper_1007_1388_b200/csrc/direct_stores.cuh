// direct_stores.cuh -- direct ghost stores of a cell pair, shared by the
// two-grid x2 sweep (sweep.cu: slot q of the neighbour's ghost copy, read by its
// next pull) and the AA LOCAL step (sweep_aa.cu: slot opp(q), gathered by the
// neighbour's next PULL; OPPSLOT).
#pragma once

#include <cstdint>
#include <utility>

#include "kernels.cuh"
#include "sweep_common.cuh"

namespace lbm {

// Neighbour patch kd of `patch` in the destination grid (null: none / copy path).
template <typename real>
__device__ __forceinline__ real *direct_ptr(const SweepArgs<real> &a, int patch, int kd)
{
    return (real *)__ldg(reinterpret_cast<const unsigned long long *>(a.dnbr + ((int64_t)patch * NDIR + kd) * 2 +
                                                                      a.dsti));
}

// Stores toward neighbour KD of the cells of the pair that lie on that side
// (on0 / on1): each PDF q travelling into the neighbour (5 per face, 1 per edge,
// P:331-337) goes into the neighbour's ghost cell at the same global position.
// A y / z face lands in a ghost row / plane of the neighbour's main slices (the
// pair stays a 2-vector); an x face or an x edge lands in the neighbour's
// x-ghost column (side 0 of the +x neighbour, side 1 of the -x neighbour).
template <typename real, int KD, bool OPPSLOT>
__device__ __forceinline__ void direct_dir_x2(const Geom &g, const Checker &ck, real *nb, int x0, int y, int z, bool on0,
                                              bool on1, const real *p0, const real *p1)
{
    using V2 = typename Vec2<real>::T;
    constexpr int ddx = ndir(KD, 0), ddy = ndir(KD, 1), ddz = ndir(KD, 2);
    if ((!on0 && !on1) || !nb) return;
    const int ty = y - ddy * g.n[1], tz = z - ddz * g.n[2];
    if constexpr (ddx != 0) {
        // exactly one cell of the pair lies on the x face
        real *gc = nb + ghost_index(g, 0, ddx > 0 ? 0 : 1, ty, tz);
        const real *pv = on0 ? p0 : p1;
#pragma unroll
        for (int q = 1; q < Q; ++q)
            if (outgoing(q, KD)) gst(ck, gc + (OPPSLOT ? OPP(q) : q) * g.gq, pv[q]);
    } else {
        real *gb = nb + main_index(g, x0, ty, tz);
#pragma unroll
        for (int q = 1; q < Q; ++q) {
            if (!outgoing(q, KD)) continue;
            const int64_t sl = (OPPSLOT ? OPP(q) : q) * g.qs;
            if (on0 && on1) {  // same x as the pair: aligned 2-vector
                V2 w;
                w.x = p0[q];
                w.y = p1[q];
                gst(ck, reinterpret_cast<V2 *>(gb + sl), w);
            } else {
                if (on0) gst(ck, gb + sl, p0[q]);
                if (on1) gst(ck, gb + sl + 1, p1[q]);
            }
        }
    }
}

template <typename real, int KD, bool OPPSLOT>
__device__ __forceinline__ void direct_dir_x2_on(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool c0,
                                                 bool c1, const real *p0, const real *p1)
{
    constexpr int ddx = ndir(KD, 0), ddy = ndir(KD, 1), ddz = ndir(KD, 2);
    const int n0 = a.g.n[0], n1 = a.g.n[1], n2 = a.g.n[2];
    const bool yz = (ddy == 0 || (ddy > 0 ? y == n1 - 1 : y == 0)) && (ddz == 0 || (ddz > 0 ? z == n2 - 1 : z == 0));
    bool on0 = c0 && yz, on1 = c1 && yz;
    if (ddx < 0) {
        on0 = on0 && x0 == 0;
        on1 = false;  // x0 + 1 > 0
    } else if (ddx > 0) {
        on0 = on0 && x0 == n0 - 1;
        on1 = on1 && x0 + 1 == n0 - 1;
    }
    if (on0 || on1) direct_dir_x2<real, KD, OPPSLOT>(a.g, a.chk, direct_ptr(a, patch, KD), x0, y, z, on0, on1, p0, p1);
}

template <typename real, bool OPPSLOT, int... KD>
__device__ __forceinline__ void direct_dirs_x2(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool c0,
                                               bool c1, const real *p0, const real *p1,
                                               std::integer_sequence<int, KD...>)
{
    (direct_dir_x2_on<real, KD, OPPSLOT>(a, patch, x0, y, z, c0, c1, p0, p1), ...);
}

// Direct ghost stores of a cell pair (x0, x0 + 1) -- the pack / copy / unpack of
// P:331-337 folded into the sweep: a fluid cell on a patch face or edge stores
// each PDF that travels into the neighbour at d (5 per face, 1 per edge) into
// that neighbour's ghost cell at the same global position, in the grid the
// neighbour pulls from next step.  c0 / c1: the cell is fluid and in the box.
// Warps off the y / z faces (y, z are warp-uniform) only handle the x faces,
// whose neighbour pointer (nb_x) the kernel loaded up front with the PDFs, so
// no dependent load sits at the end of the thread.
static_assert(ndir(8, 0) == -1 && ndir(8, 1) == 0 && ndir(8, 2) == 0, "plan order: kd 8 = -x");
static_assert(ndir(9, 0) == 1 && ndir(9, 1) == 0 && ndir(9, 2) == 0, "plan order: kd 9 = +x");

template <typename real, bool OPPSLOT = false>
__device__ __forceinline__ void direct_stores_x2(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool c0,
                                                 bool c1, const real *p0, const real *p1, real *nb_x)
{
    const Geom &g = a.g;
    const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
    const bool yzf = y == 0 || y == n1 - 1 || z == 0 || z == n2 - 1;
    if (!yzf) {
        const bool hi0 = c0 && x0 == n0 - 1, hi1 = c1 && x0 + 1 == n0 - 1;
        if (x0 == 0) {
            direct_dir_x2<real, 8, OPPSLOT>(g, a.chk, nb_x, x0, y, z, c0, false, p0, p1);
            if (hi0 || hi1) direct_dir_x2<real, 9, OPPSLOT>(g, a.chk, direct_ptr(a, patch, 9), x0, y, z, hi0, hi1, p0, p1);
        } else {
            direct_dir_x2<real, 9, OPPSLOT>(g, a.chk, nb_x, x0, y, z, hi0, hi1, p0, p1);
        }
        return;
    }
    direct_dirs_x2<real, OPPSLOT>(a, patch, x0, y, z, c0, c1, p0, p1, std::make_integer_sequence<int, NDIR>{});
}

}  // namespace lbm
