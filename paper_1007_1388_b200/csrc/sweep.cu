// sweep.cu -- the two-grid sweep kernel of the D3Q19 LBGK patch solver (sm_100a).
//
// The hot loop is the fused pull stream + bounce-back + BGK collide update of
// eq:lbm / eq:feq with centred PDFs, pull streaming
// from two grids and half-way bounce-back with a moving-wall term
// (P:482-490).  SoA layout: one q-slice per direction with rows of
// exactly n_x cells, the x neighbours of the row ends in compact x-ghost columns
// (lbm_internal.h Geom).  The kernel is HBM-bound: 19 loads + 19 stores of
// sizeof(real) per fluid cell, no data reuse across directions
// (each src element is pulled by exactly one cell), so the design goal is
// enough independent loads in flight per SM and fully coalesced, sector-aligned
// stores: two cells per thread along x, 2-vector loads for the 9 directions
// with e_x = 0 and 2-vector stores for all 19, optionally storing the outgoing
// PDFs of patch-face cells straight into neighbour ghost layers.
#include <cstdint>
#include <utility>

#include "collide.cuh"
#include "direct_stores.cuh"
#include "kernels.cuh"
#include "sweep_common.cuh"
#include "sweep_pair.cuh"

namespace lbm {

// Store-side bounce-back (two-grid): f_j(x) leaving toward the wall w = x + e_j
// comes back to x next step as direction opp(j) (R3); park it, plus
// the moving-wall term of the delivered direction opp(j), in w's slot opp(j),
// so the next step's pull of x is branch-free.  m: wall-neighbour mask of x.
template <typename real>
__device__ __forceinline__ void store_bb_ab(const SweepArgs<real> &a, real *D, const uint8_t *fl, int x, int y,
                                            int z, uint32_t m, const real *p)
{
#pragma unroll
    for (int j = 1; j < Q; ++j) {
        if (!((m >> j) & 1u)) continue;
        real v = p[j];
        const uint8_t f = fl[flag_shift(a.g, j)];
        if (f >= 2) v += a.corr[(f - 2) * Q + OPP(j)];
        D[pdf_index(a.g, OPP(j), x + EX(j), y + EY(j), z + EZ(j))] = v;
    }
}

// One thread = the cell pair (x0, x0 + 1) of one row; block (32, 4) threads =
// 64 x 4 cells of one z plane.  A pair of fluid cells stores 2-vectors; a pair
// containing a non-fluid cell stores scalars (a wall cell's slots hold
// store-side bounce-back values of its neighbours and must not be
// overwritten).  Only lanes next to a wall run the bounce-back stores; keeping
// that tail small matters because a warp whose row reaches a wall runs it for
// every lane's instruction stream.
template <typename real, int MINB, bool DIRECT>
__global__ void __launch_bounds__(32 * SWEEP_BY, MINB) sweep_x2_kernel(const SweepArgs<real> a)
{
    using V2 = typename Vec2<real>::T;
    const PairCoord pc = locate_pair(a);
    if (!pc.valid) return;
    const int x0 = pc.x0, y = pc.y, z = pc.z;
    const bool has1 = x0 + 1 < pc.xend;
    const Geom &g = a.g;
    const int64_t c = main_index(g, x0, y, z);
    const int64_t fc = (int64_t)pc.patch * g.fs + flag_index(g, x0, y, z);
    const uchar2 kk = *reinterpret_cast<const uchar2 *>(a.kind + fc);
    const uint8_t k0 = kk.x, k1 = has1 ? kk.y : (uint8_t)2;
    // x-face neighbour of this pair for the direct ghost stores: -x if x0 == 0,
    // else +x (the +x one of a pair on both faces, n0 <= 2, loads late)
    real *nb_x = nullptr;
    if (DIRECT && (x0 == 0 || x0 + 1 >= g.n[0] - 1)) nb_x = direct_ptr(a, pc.patch, x0 == 0 ? 8 : 9);
    real p0[Q], p1[Q];
    pull_pair<real, false>(g, a.src + (int64_t)pc.patch * g.ps, c, x0, y, z, p0, p1);
    if (k0 == 2 && k1 == 2) return;
    const uint32_t m0 = k0 == 1 ? a.wmask[fc] : 0u;
    const uint32_t m1 = k1 == 1 ? a.wmask[fc + 1] : 0u;
    collide_bgk<real>(p0, a.omega);
    collide_bgk<real>(p1, a.omega);
    real *d = a.dst + (int64_t)pc.patch * g.ps + c;
    if (k0 != 2 && k1 != 2) {
        // both cells fluid (the common case): aligned 2-vector stores
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            V2 w;
            w.x = p0[i];
            w.y = p1[i];
            *reinterpret_cast<V2 *>(d + i * g.qs) = w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (k0 != 2) d[i * g.qs] = p0[i];
            if (k1 != 2) d[i * g.qs + 1] = p1[i];
        }
    }
    if (m0 | m1) {
        // a wall next to a cell of the pair: coordinates re-decoded from the tile
        // descriptor (L1 hit) rather than kept live through the collision
        const PairCoord q = locate_pair(a);
        const int64_t fq = (int64_t)q.patch * g.fs + flag_index(g, q.x0, q.y, q.z);
        real *D = a.dst + (int64_t)q.patch * g.ps;
        if (m0) store_bb_ab<real>(a, D, a.flags + fq, q.x0, q.y, q.z, m0, p0);
        if (m1) store_bb_ab<real>(a, D, a.flags + fq + 1, q.x0 + 1, q.y, q.z, m1, p1);
    }
    if (DIRECT) direct_stores_x2<real>(a, pc.patch, x0, y, z, k0 != 2, k1 != 2, p0, p1, nb_x);
}

template <typename real>
cudaError_t launch_sweep(const SweepArgs<real> &a, int64_t total_tiles, int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    dim3 block(32, SWEEP_BY, 1);
    const unsigned grid = (unsigned)total_tiles;
    // min blocks of 128 threads per SM: fp64 3 / 2, fp32 4 / 5 (variant 0 / 1)
    constexpr int M0 = sizeof(real) == 8 ? 3 : 4, M1 = sizeof(real) == 8 ? 2 : 5;
    if (a.dnbr) {
        if (variant == 1) sweep_x2_kernel<real, M1, true><<<grid, block, 0, s>>>(a);
        else sweep_x2_kernel<real, M0, true><<<grid, block, 0, s>>>(a);
    } else {
        if (variant == 1) sweep_x2_kernel<real, M1, false><<<grid, block, 0, s>>>(a);
        else sweep_x2_kernel<real, M0, false><<<grid, block, 0, s>>>(a);
    }
    return cudaGetLastError();
}

template cudaError_t launch_sweep<float>(const SweepArgs<float> &, int64_t, int, cudaStream_t);
template cudaError_t launch_sweep<double>(const SweepArgs<double> &, int64_t, int, cudaStream_t);

}  // namespace lbm
