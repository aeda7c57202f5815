// sweep_pair.cuh -- the pull of a cell pair (x0, x0 + 1), shared by the two-grid
// sweep (sweep.cu) and the AA PULL step (sweep_aa.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "sweep_common.cuh"

namespace lbm {

// Pull: p_i = src_slot(i)(x - e_i) for both cells of the pair, with
// slot(i) = i (two grids) or opp(i) (AA PULL, swapped representation).
// Branch-free for the row: when x - e_i is a wall cell, its slot already holds
// the half-way bounce-back value (store-side bounce-back, sweep.cu).  The 9
// directions with e_x = 0 are aligned 2-vector loads; the 10 with e_x != 0 are
// scalar loads from the row.  All 38 are issued before any is consumed.  A
// row-end cell's x neighbour lives in the x-ghost column: the row load of that
// lane (in-bounds: the previous / next row or the row padding) is replaced by
// a ghost-column load in a branch that only warps holding a row end enter --
// per-lane address selects on every warp cost the issue-bound fp32 sweep 16 %.
template <typename real, bool AA>
__device__ __forceinline__ void pull_pair(const Geom &g, const real *P, int64_t c, int x0, int y, int z, real (&p0)[Q],
                                          real (&p1)[Q])
{
    using V2 = typename Vec2<real>::T;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int sl = AA ? OPP(i) : i;
        const real *s = P + (int64_t)sl * g.qs + c - yz_shift(g, i);
        if (EX(i) == 0) {
            const V2 v = __ldg(reinterpret_cast<const V2 *>(s));
            p0[i] = v.x;
            p1[i] = v.y;
        } else if (EX(i) > 0) {  // pull from x - 1
            p0[i] = __ldg(s - 1);
            p1[i] = __ldg(s);
        } else {  // pull from x + 1
            p0[i] = __ldg(s + 1);
            p1[i] = __ldg(s + 2);
        }
    }
    const int n0 = g.n[0];
    const bool lo0 = x0 == 0;       // x0 - 1 is the -x ghost
    const bool hi0 = x0 + 1 == n0;  // x0 + 1 is the +x ghost (odd n0)
    const bool hi1 = x0 + 2 == n0;  // x0 + 2 is the +x ghost
    if (lo0 || hi0 || hi1) {
        const real *G = P + g.gbase + (int64_t)(z + 1) * g.gy + (y + g.gyo);  // ghost column (q 0, side 0) at (y, z)
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (EX(i) == 0) continue;
            const int sl = AA ? OPP(i) : i;
            const real *gs = G + (int64_t)sl * g.gq + (EX(i) > 0 ? 0 : g.gside) - EY(i) - EZ(i) * (int64_t)g.gy;
            if (EX(i) > 0) {
                if (lo0) p0[i] = __ldg(gs);
            } else {
                if (hi0) p0[i] = __ldg(gs);
                if (hi1) p1[i] = __ldg(gs);
            }
        }
    }
}

}  // namespace lbm
