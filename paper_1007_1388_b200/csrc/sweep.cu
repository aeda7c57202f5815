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

// The bounce-back through a uniform-wall y (A = 1) or z (A = 2) face of a cell pair
// on it: c the pair's coordinate along A, o its other inner coordinate (z / y);
// in0 / in1: the cell is fluid and off the face's x rim.  d: the pair's first
// cell in the destination grid.  Both sides when the patch is one cell thick.
template <typename real, int A>
__device__ __forceinline__ void face_wall_stores(const SweepArgs<real> &a, real *d, unsigned long long sw, int c,
                                                 int o, bool in0, bool in1, const real *p0, const real *p1)
{
    using V2 = typename Vec2<real>::T;
    const Geom &g = a.g;
    const int B = A == 1 ? 2 : 1;  // the other coordinate's axis
    if (o < 1 || o > g.n[B] - 2 || !(in0 | in1)) return;
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
        const int side = 2 * A + hi;
        if (c != (hi ? g.n[A] - 1 : 0) || !((sw >> side) & 1ull)) continue;
        const int s = hi ? 1 : -1;
        const int f = side_flag(sw, side);
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            if ((A == 1 ? EY(j) : EZ(j)) != s) continue;  // links through this face only
            real v0 = p0[j], v1 = p1[j];
            if (f >= 2) {
                const real cj = __ldg(a.corr + (f - 2) * Q + OPP(j));
                v0 += cj;
                v1 += cj;
            }
            real *t = at<real>(d, a.off.wall[j]);
            if (EX(j) == 0 && in0 && in1) {
                V2 w;
                w.x = v0;
                w.y = v1;
                gst(a.chk, reinterpret_cast<V2 *>(t), w);
            } else {
                if (in0) gst(a.chk, t, v0);
                if (in1) gst(a.chk, t + 1, v1);
            }
        }
    }
}

// One thread = the cell pair (x0, x0 + 1) of one row; block (32, 4) threads =
// 64 x 4 cells of one z plane.  The sweep carries no wall logic: the pull is
// branch-free because the wall slots it reads already hold the half-way
// bounce-back values, which the bounce-back list kernel (aux_kernels.cu
// bb_list_kernel, store side) writes after every sweep for the few
// wall-adjacent cells.  (With the walls in the sweep, the per-cell kind load,
// the dependent wall-mask load and the bounce-back tail of the wall lanes --
// half the warps of a 256^3 cavity hold an x-wall lane -- cost 10 % (fp64) and
// 23 % (fp32) of the step, profiles/r02_wall_path_ab.jsonl.)  Only tiles that
// hold a non-fluid cell read the cells' kinds, so non-fluid cells are neither
// updated nor stored; a pair of fluid cells stores 2-vectors.
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
    uint8_t k0 = 0, k1 = has1 ? 0 : 2;  // 2: non-fluid (or the phantom partner of an odd row end)
    if (pc.solid) {
        const uchar2 kk =
            *reinterpret_cast<const uchar2 *>(a.kind + (int64_t)pc.patch * g.fs + flag_index(g, x0, y, z));
        k0 = kk.x;
        if (has1) k1 = kk.y;
    }
    // x-face neighbour of this pair for the direct ghost stores: -x if x0 == 0,
    // else +x (the +x one of a pair on both faces, n0 <= 2, loads late)
    real *nb_x = nullptr;
    if (DIRECT && (x0 == 0 || x0 + 1 >= g.n[0] - 1)) nb_x = direct_ptr(a, pc.patch, x0 == 0 ? 8 : 9);
    const real *P = a.src + (int64_t)pc.patch * g.ps;
    real p0[Q], p1[Q];
    pull_pair<real>(a.off, a.chk, P + c, ghost_base(g, P, y, z), x0 == 0, x0 + 1 == g.n[0], x0 + 2 == g.n[0], has1,
                    p0, p1);
    if (k0 == 2 && k1 == 2) return;
    collide_pair(p0, p1, a.omega);
    real *d = a.dst + (int64_t)pc.patch * g.ps + c;
    if (k0 != 2 && k1 != 2) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            V2 w;
            w.x = p0[i];
            w.y = p1[i];
            gst(a.chk, at<V2>(d, a.off.slot[i]), w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (k0 != 2) gst(a.chk, at<real>(d, a.off.slot[i]), p0[i]);
            if (k1 != 2) gst(a.chk, at<real>(d, a.off.slot[i]) + 1, p1[i]);
        }
    }
    if (DIRECT) direct_stores_x2<real>(a, pc.patch, x0, y, z, k0 != 2, k1 != 2, p0, p1, nb_x);
    // Uniform-wall sides (launch_sidewall): the half-way bounce-back of the
    // links through such a face, which the per-step list leaves out, stored by the
    // face cells themselves -- every link of an inner face cell through the face
    // leads into the ghost layer over it, so no wall lookup is needed.  x: the
    // row-end lanes, into the compact ghost column; y / z: whole face rows /
    // planes (warp-uniform), into the ghost rows / planes of the main slices.
    if (y >= 1 && y <= g.n[1] - 2 && z >= 1 && z <= g.n[2] - 2 && (pc.xlo || pc.xhi)) {
        const bool lo = pc.xlo && x0 == 0 && k0 != 2;
        const bool hi0 = pc.xhi && x0 == g.n[0] - 1 && k0 != 2, hi1 = pc.xhi && x0 + 1 == g.n[0] - 1 && k1 != 2;
        if (lo | hi0 | hi1) {
            real *G = ghost_base(g, a.dst + (int64_t)pc.patch * g.ps, y, z);
#pragma unroll
            for (int j = 1; j < Q; ++j) {
                if (EX(j) == 0 || (EX(j) < 0 ? !lo : !(hi0 | hi1))) continue;
                real v = EX(j) < 0 || hi0 ? p0[j] : p1[j];
                const int f = EX(j) < 0 ? pc.flo : pc.fhi;  // the side's wall flag: >= 2 moves
                if (f >= 2) v += __ldg(a.corr + (f - 2) * Q + OPP(j));
                gst(a.chk, at<real>(G, a.off.gwall[j]), v);
            }
        }
    }
    if (a.sidewall && (y == 0 || y == g.n[1] - 1 || z == 0 || z == g.n[2] - 1)) {
        const unsigned long long sw = __ldg(a.sidewall + pc.patch);
        const bool in0 = k0 != 2 && x0 >= 1 && x0 <= g.n[0] - 2, in1 = k1 != 2 && x0 + 1 <= g.n[0] - 2;
        face_wall_stores<real, 1>(a, d, sw, y, z, in0, in1, p0, p1);
        face_wall_stores<real, 2>(a, d, sw, z, y, in0, in1, p0, p1);
    }
}

template <typename real, int MINB>
cudaError_t launch_x2(const SweepArgs<real> &a, unsigned grid, cudaStream_t s)
{
    const dim3 block(32, SWEEP_BY, 1);
    if (a.dnbr) sweep_x2_kernel<real, MINB, true><<<grid, block, 0, s>>>(a);
    else sweep_x2_kernel<real, MINB, false><<<grid, block, 0, s>>>(a);
    return cudaGetLastError();
}

template <typename real>
cudaError_t launch_sweep(const SweepArgs<real> &a, int64_t total_tiles, int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)total_tiles;
    // min blocks of 128 threads per SM (variant 0 / 1): fp64 3 / 2, fp32 5 / 4
    constexpr int M0 = sizeof(real) == 8 ? 3 : 5, M1 = sizeof(real) == 8 ? 2 : 4;
    return variant == 1 ? launch_x2<real, M1>(a, grid, s) : launch_x2<real, M0>(a, grid, s);
}

template cudaError_t launch_sweep<float>(const SweepArgs<float> &, int64_t, int, cudaStream_t);
template cudaError_t launch_sweep<double>(const SweepArgs<double> &, int64_t, int, cudaStream_t);

}  // namespace lbm
