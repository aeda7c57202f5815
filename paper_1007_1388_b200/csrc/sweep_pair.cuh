// sweep_pair.cuh -- the pull of a cell pair (x0, x0 + 1), shared by the two-grid
// sweep (sweep.cu) and the AA PULL step (sweep_aa.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "sweep_common.cuh"

namespace lbm {

// Pull: p_i = src_slot(i)(x - e_i) for both cells of the pair, with
// slot(i) = i (two grids) or opp(i) (AA PULL, swapped representation), encoded
// in the offset table (kernels.cuh DirOffsets).  C: the first cell's element in
// slice 0; G: its x-ghost column base (ghost_base).
// Branch-free: when x - e_i is a wall cell, its slot already holds the
// half-way bounce-back value (store-side bounce-back, sweep.cu).  The 9
// directions with e_x = 0 are aligned 2-vector loads; the 10 with e_x != 0 are
// scalar loads, from the row or -- for a row-end cell, whose x neighbour lives
// in the x-ghost column -- from the ghost column: one load from a selected
// address (with the uniform offset tables 7 % faster in fp64 than two
// predicated loads, which ptxas issues after the 2-vector loads; 5-6 % faster
// than a ghost-load branch after the row loads).  All 38 loads are issued
// before any is consumed.
template <typename real>
__device__ __forceinline__ void pull_pair(const DirOffsets &o, const Checker &ck, const real *C, const real *G,
                                          bool lo0, bool hi0, bool hi1, bool has1, real (&p0)[Q], real (&p1)[Q])
{
    using V2 = typename Vec2<real>::T;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const real *s = at<const real>(C, o.pull[i]);
        if (EX(i) == 0) {
            const V2 v = gld(ck, reinterpret_cast<const V2 *>(s));
            p0[i] = v.x;
            p1[i] = v.y;
        } else {
            const real *gs = at<const real>(G, o.gpull[i]);
            // the phantom partner of an odd row end (!has1) re-reads the first
            // cell's value instead of a slot another thread of an in-place (AA)
            // sweep may be writing
            const real *s1 = has1 ? s + 1 : s;
            if (EX(i) > 0) {
                p0[i] = gld(ck, lo0 ? gs : s);
                p1[i] = gld(ck, s1);
            } else {
                p0[i] = gld(ck, hi0 ? gs : s);
                p1[i] = gld(ck, hi1 ? gs : s1);
            }
        }
    }
}

}  // namespace lbm
