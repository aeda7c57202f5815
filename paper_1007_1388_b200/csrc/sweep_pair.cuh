// sweep_pair.cuh -- the pull of a cell pair (x0, x0 + 1), shared by the two-grid
// sweep (sweep.cu) and the AA PULL step (sweep_aa.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "sweep_common.cuh"

namespace lbm {

// Pull: p_i = src_slot(i)(x - e_i) for both cells of the pair, with
// slot(i) = i (two grids) or opp(i) (AA PULL, swapped representation).
// Branch-free: when x - e_i is a wall cell, its slot already holds the
// half-way bounce-back value (store-side bounce-back, sweep.cu).  The 9
// directions with e_x = 0 are aligned 2-vector loads; the 10 with e_x != 0 are
// scalar loads, from the row or -- for a row-end cell, whose x neighbour lives
// in the x-ghost column -- from the ghost column (two predicated loads per
// value: measured 1-2 % faster than one load from a selected address, and
// 5-6 % faster than a ghost-load branch after the row loads,
// profiles/r02_ab_pull_ghost.jsonl).  All 38 loads are issued before any is
// consumed.  The phantom partner of an odd row end reads in-bounds garbage
// that is never used.
template <typename real, bool AA>
__device__ __forceinline__ void pull_pair(const Geom &g, const real *P, int64_t c, int x0, int y, int z, real (&p0)[Q],
                                          real (&p1)[Q])
{
    using V2 = typename Vec2<real>::T;
    const int n0 = g.n[0];
    const bool lo0 = x0 == 0, hi0 = x0 + 1 == n0, hi1 = x0 + 2 == n0;
    const real *G = P + g.gbase + (int64_t)(z + 1) * g.gy + (y + g.gyo);
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int sl = AA ? OPP(i) : i;
        const real *s = P + (int64_t)sl * g.qs + c - yz_shift(g, i);
        if (EX(i) == 0) {
            const V2 v = __ldg(reinterpret_cast<const V2 *>(s));
            p0[i] = v.x;
            p1[i] = v.y;
        } else {
            const real *gs = G + (int64_t)sl * g.gq + (EX(i) > 0 ? 0 : g.gside) - EY(i) - EZ(i) * (int64_t)g.gy;
            if (EX(i) > 0) {
                p0[i] = (lo0 ? __ldg(gs) : __ldg(s - 1));
                p1[i] = __ldg(s);
            } else {
                p0[i] = (hi0 ? __ldg(gs) : __ldg(s + 1));
                p1[i] = (hi1 ? __ldg(gs) : __ldg(s + 2));
            }
        }
    }
}

}  // namespace lbm
