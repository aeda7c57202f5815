// sweep_aa.cu -- AA-pattern in-place sweep kernels (one PDF array; north_star
// (a)): the update of sweep.cu in alternating PULL /
// LOCAL steps.
//
// With S_i(x) the post-collision state of the two-grid scheme:
//   swapped  representation (after an even step count): A[x][opp(i)] = S_i(x)
//   streamed representation (after an odd step count):  A[x][i] = p_i(x), the
//                                                        value x pulls next
// PULL  (swapped -> streamed): p_i = A[x - e_i][opp(i)]; collide; write out_i to
//       A[x + e_i][i], or -- x + e_i a wall -- its bounce-back
//       out_i + 6 w rho0 e_opp(i).u_w to A[x][opp(i)] (R3).
// LOCAL (streamed -> swapped): p_i = A[x][i]; collide; A[x][opp(i)] = out_i, and
//       for walls w = x + e_j the store-side bounce-back A[w][j] = out_j + corr,
//       which the next PULL gathers branch-free (both bounce-back parts: the
//       uniform-wall side stores below and the bounce-back list, aux_kernels.cu).
// Every slot has exactly one writer per step and is read only by it, so both
// kernels run in place without races; the results equal the two-grid scheme
// bitwise after every even step count.
//
// Two cells per thread along x (cf. sweep_x2_kernel): LOCAL reads and writes
// only its own cells, so all 19 loads and 19 stores are aligned 2-vectors; PULL
// vectorises the 9 gathers and scatters with e_x = 0, and its row-end cells
// gather from / scatter into the x-ghost columns.  Every pair of fluid cells
// takes a straight-line scatter: per-direction wall redirect tests cost PULL
// +41 % instructions (1.05 -> 0.88 ms at 256^3 fp64, round 1,
// profiles/r01_ncu_aa_*), and the walls' dependent mask loads and bounce-back
// tails a further 10-20 % (round 2) -- both now live in the bounce-back list
// kernel that runs after each AA step (sweep_aa_x2_kernel below).
//
// Direct ghost stores (the AA pattern's two half-exchanges folded into the
// sweep):
//   LOCAL: a fluid cell on a patch face / edge stores out_q, for each q that
//          travels into the neighbour, into the neighbour's ghost copy of the
//          cell at slot opp(q) -- what the neighbour's next PULL gathers there
//          (the two-grid store pattern, direct_stores.cuh with OPPSLOT);
//   PULL:  a fluid cell x whose scatter target x + e_q lies in a neighbour patch
//          (and is fluid) stores out_q into that cell of the neighbour, slot q --
//          what the neighbour's next LOCAL reads.  Only fluid writers store: the
//          writer mask of half-exchange 2 holds by construction.
// Every slot keeps exactly one writer per step, so this races with nothing.
#include <cstdint>

#include "collide.cuh"
#include "direct_stores.cuh"
#include "kernels.cuh"
#include "sweep_common.cuh"
#include "sweep_pair.cuh"

namespace lbm {

// (oz, oy, ox) + 1 in base 3 -> neighbour direction kd of the plan order, -1: none
__constant__ int8_t c_kd27[27] = {-1, 0,  -1, 1,  2,  3,  -1, 4,  -1, 5,  6,  7,  8, -1,
                                  9,  10, 11, 12, -1, 13, -1, 14, 15, 16, -1, 17, -1};

// PULL of one cell on a y / z face: every scatter target x + e_q outside the
// patch goes into the neighbour patch holding it.  A wall target receives the
// value too (never read there: the bounce-back list's fix-up takes it from this
// patch's own ghost copy, which the straight scatter also wrote).
template <typename real>
__device__ __forceinline__ void aa_pull_direct(const SweepArgs<real> &a, int patch, int x, int y, int z, const real *p)
{
    const Geom &g = a.g;
    const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        const int dx = x + EX(q), dy = y + EY(q), dz = z + EZ(q);
        const int ox = dx < 0 ? -1 : (dx >= n0 ? 1 : 0);
        const int oy = dy < 0 ? -1 : (dy >= n1 ? 1 : 0);
        const int oz = dz < 0 ? -1 : (dz >= n2 ? 1 : 0);
        if ((ox | oy | oz) == 0) continue;  // target inside the patch
        const int kd = c_kd27[(oz + 1) * 9 + (oy + 1) * 3 + (ox + 1)];
        real *nb = direct_ptr(a, patch, kd);
        if (!nb) continue;
        gst(a.chk, nb + pdf_index(g, q, dx - ox * n0, dy - oy * n1, dz - oz * n2), p[q]);
    }
}

// PULL, a cell on the x face S (-1 / +1) and on no y / z face: its scatter
// targets x + e_q with e_qx = S are the x neighbour's cells
// (x + S - S n0, y + e_qy, z + e_qz); y +- 1, z +- 1 stay inside the patch.
template <typename real, int S>
__device__ __forceinline__ void aa_pull_xface(const SweepArgs<real> &a, real *nb, int x, int y, int z, const real *p)
{
    if (!nb) return;
    const Geom &g = a.g;
    real *row = nb + main_index(g, x + S - S * g.n[0], y, z);
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (EXf(q) != S) continue;
        gst(a.chk, row + q * g.qs + yz_shift(g, q), p[q]);
    }
}

// A pair (x0, x0 + 1): only cells on a patch face do anything.  nb_x: the x
// neighbour of the pair's x-face cell (-x if x0 == 0, else +x), loaded up front.
template <typename real, bool PULL>
__device__ __forceinline__ void aa_direct_pair(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool has1,
                                               uint8_t k0, uint8_t k1, const real *p0, const real *p1, real *nb_x)
{
    if (!PULL) {
        direct_stores_x2<real, true>(a, patch, x0, y, z, k0 != 2, has1 && k1 != 2, p0, p1, nb_x);
        return;
    }
    const Geom &g = a.g;
    const int n0 = g.n[0];
    const bool yzf = y == 0 || y == g.n[1] - 1 || z == 0 || z == g.n[2] - 1;  // warp-uniform
    if (yzf) {
        if (k0 != 2) aa_pull_direct<real>(a, patch, x0, y, z, p0);
        if (has1 && k1 != 2) aa_pull_direct<real>(a, patch, x0 + 1, y, z, p1);
        return;
    }
    if (x0 == 0) {
        if (k0 != 2) aa_pull_xface<real, -1>(a, nb_x, x0, y, z, p0);
        if (n0 == 1 && k0 != 2) aa_pull_xface<real, 1>(a, direct_ptr(a, patch, 9), x0, y, z, p0);
        if (n0 == 2 && has1 && k1 != 2) aa_pull_xface<real, 1>(a, direct_ptr(a, patch, 9), x0 + 1, y, z, p1);
    } else {
        if (x0 == n0 - 1 && k0 != 2) aa_pull_xface<real, 1>(a, nb_x, x0, y, z, p0);
        if (has1 && x0 + 1 == n0 - 1 && k1 != 2) aa_pull_xface<real, 1>(a, nb_x, x0 + 1, y, z, p1);
    }
}

// Uniform-wall patch sides (launch_sidewall; cf. sweep.cu): the half-way
// bounce-back of the links of a side's inner face cells through it, which the
// per-step list leaves out, stored by the cells themselves from registers --
// PULL: out_i + corr into the cell's own slot opp(i) (the list's fix-up, mode 2);
// LOCAL: out_j + corr into the wall slot j of the ghost cell x + e_j (mode 1).
// cin0 / cin1: the cell is fluid.
template <typename real, bool PULL>
__device__ __forceinline__ void aa_side_wall_stores(const SweepArgs<real> &a, const PairCoord &pc, real *P, real *A,
                                                    bool cin0, bool cin1, const real *p0, const real *p1)
{
    const Geom &g = a.g;
    const int x0 = pc.x0, y = pc.y, z = pc.z;
    // x sides: the row-end lanes (side bits and flags in the tile descriptor)
    if (y >= 1 && y <= g.n[1] - 2 && z >= 1 && z <= g.n[2] - 2 && (pc.xlo || pc.xhi)) {
        const bool lo = pc.xlo && x0 == 0 && cin0;
        const bool hi0 = pc.xhi && x0 == g.n[0] - 1 && cin0, hi1 = pc.xhi && x0 + 1 == g.n[0] - 1 && cin1;
        if (lo | hi0 | hi1) {
            real *G = ghost_base(g, P, y, z);
#pragma unroll
            for (int i = 1; i < Q; ++i) {
                if (EX(i) == 0 || (EX(i) < 0 ? !lo : !(hi0 | hi1))) continue;
                const bool c1 = EX(i) > 0 && hi1;  // the wall-side cell is the pair's second
                real v = c1 ? p1[i] : p0[i];
                const int f = EX(i) < 0 ? pc.flo : pc.fhi;
                if (f >= 2) v += __ldg(a.corr + (f - 2) * Q + OPP(i));
                real *t = PULL ? at<real>(A, a.off.oslot[i]) + (c1 ? 1 : 0) : at<real>(G, a.off.gpush[i]);
                gst(a.chk, t, v);
            }
        }
    }
    // y / z sides: whole face rows / planes (warp-uniform)
    if (!(y == 0 || y == g.n[1] - 1 || z == 0 || z == g.n[2] - 1)) return;
    const unsigned long long sw = __ldg(a.sidewall + pc.patch);
    const bool xin0 = cin0 && x0 >= 1 && x0 <= g.n[0] - 2, xin1 = cin1 && x0 + 1 <= g.n[0] - 2;
#pragma unroll
    for (int side = 2; side < 6; ++side) {  // both sides of a one-cell-thick patch
        const int A_ = side / 2, hi = side & 1;
        const int c = A_ == 1 ? y : z, o = A_ == 1 ? z : y, no = A_ == 1 ? g.n[2] : g.n[1];
        if (o < 1 || o > no - 2 || !(xin0 | xin1)) continue;
        if (c != (hi ? g.n[A_] - 1 : 0) || !((sw >> side) & 1ull)) continue;
        const int s = hi ? 1 : -1;
        const int f = side_flag(sw, side);
#pragma unroll
        for (int i = 1; i < Q; ++i) {
            if ((A_ == 1 ? EY(i) : EZ(i)) != s) continue;
            real v0 = p0[i], v1 = p1[i];
            if (f >= 2) {
                const real ci = __ldg(a.corr + (f - 2) * Q + OPP(i));
                v0 += ci;
                v1 += ci;
            }
            real *t = PULL ? at<real>(A, a.off.oslot[i]) : at<real>(A, a.off.push[i]);
            if (xin0) gst(a.chk, t, v0);
            if (xin1) gst(a.chk, t + 1, v1);
        }
    }
}

// As the two-grid sweep, the AA kernels carry no wall logic: PULL scatters every
// out_i to x + e_i, a wall cell included, and the bounce-back list's PULL fix-up
// (aux_kernels.cu bb_list_kernel, mode 2) then moves out_i + corr from the wall's
// slot i into A[x][opp(i)]; after LOCAL, its store-side mode (1) parks
// out_j + corr in the wall slots A[x + e_j][j] that the next PULL gathers.  The
// only reader of a wall slot written by the blind scatter is the fix-up, and
// the only reader of A[x][opp(i)] is x's next LOCAL.  Only tiles holding a
// non-fluid cell read the cells' kinds.
template <typename real, bool PULL, int MINB, bool DIRECT>
__global__ void __launch_bounds__(32 * SWEEP_BY, MINB) sweep_aa_x2_kernel(const SweepArgs<real> a)
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
    real *nb_x = nullptr;  // x-face neighbour for the direct ghost stores, loaded with the PDFs
    if (DIRECT && (x0 == 0 || x0 + 1 >= g.n[0] - 1)) nb_x = direct_ptr(a, pc.patch, x0 == 0 ? 8 : 9);
    real *P = a.dst + (int64_t)pc.patch * g.ps;  // in place
    real *A = P + c;
    real p0[Q], p1[Q];
    if (PULL) {
        pull_pair<real>(a.off, a.chk, A, ghost_base(g, (const real *)P, y, z), x0 == 0, x0 + 1 == g.n[0],
                        x0 + 2 == g.n[0], has1, p0, p1);
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const V2 v = gld(a.chk, at<const V2>(A, a.off.slot[i]));
            p0[i] = v.x;
            p1[i] = v.y;
        }
    }
    if (k0 == 2 && k1 == 2) return;
    collide_pair(p0, p1, a.omega);
    const bool both = k0 != 2 && k1 != 2;
    if (PULL) {
        if (both) {
            // straight-line scatter to x + e_i; a row-end target lives in the
            // x-ghost column, stored in a branch only warps holding a row end take
            const bool lo0 = x0 == 0, hi1 = x0 + 2 == g.n[0];
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                real *t = at<real>(A, a.off.push[i]);  // target of the first cell
                if (EX(i) == 0) {
                    V2 w;
                    w.x = p0[i];
                    w.y = p1[i];
                    gst(a.chk, reinterpret_cast<V2 *>(t), w);
                } else if (EX(i) > 0) {  // to x + 1
                    gst(a.chk, t, p0[i]);
                    if (!hi1) gst(a.chk, t + 1, p1[i]);
                } else {  // to x - 1
                    if (!lo0) gst(a.chk, t, p0[i]);
                    gst(a.chk, t + 1, p1[i]);
                }
            }
            // (the inner cells of a uniform-wall x side skip it: aa_side_wall_stores
            // redirects those links, and the next LOCAL rewrites the wall slot)
            const bool inner = y >= 1 && y <= g.n[1] - 2 && z >= 1 && z <= g.n[2] - 2;
            const bool glo = lo0 && !(pc.xlo && inner), ghi = hi1 && !(pc.xhi && inner);
            if (glo || ghi) {
                real *G = ghost_base(g, P, y, z);
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    if (EX(i) == 0) continue;
                    real *gt = at<real>(G, a.off.gpush[i]);
                    if (EX(i) > 0 && ghi) gst(a.chk, gt, p1[i]);
                    if (EX(i) < 0 && glo) gst(a.chk, gt, p0[i]);
                }
            }
        } else {
            // one cell of the pair is non-fluid (or the phantom of an odd row end)
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                if (k0 != 2) gst(a.chk, P + pdf_index(g, i, x0 + EX(i), y + EY(i), z + EZ(i)), p0[i]);
                if (k1 != 2) gst(a.chk, P + pdf_index(g, i, x0 + 1 + EX(i), y + EY(i), z + EZ(i)), p1[i]);
            }
        }
    } else if (both) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            V2 w;
            w.x = p0[i];
            w.y = p1[i];
            gst(a.chk, at<V2>(A, a.off.oslot[i]), w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (k0 != 2) gst(a.chk, at<real>(A, a.off.oslot[i]), p0[i]);
            if (k1 != 2) gst(a.chk, at<real>(A, a.off.oslot[i]) + 1, p1[i]);
        }
    }
    if (DIRECT) aa_direct_pair<real, PULL>(a, pc.patch, x0, y, z, has1, k0, k1, p0, p1, nb_x);
    if (a.sidewall) aa_side_wall_stores<real, PULL>(a, pc, P, A, k0 != 2, k1 != 2, p0, p1);
}

template <typename real>
cudaError_t launch_sweep_aa(const SweepArgs<real> &a, int64_t total_tiles, bool pull, int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    dim3 block(32, SWEEP_BY, 1);
    const unsigned grid = (unsigned)total_tiles;
    // min blocks of 128 threads per SM (variant 0 / 1): fp64 3 / 2, fp32 5 / 4
    constexpr int M0 = sizeof(real) == 8 ? 3 : 5, M1 = sizeof(real) == 8 ? 2 : 4;
    const bool m1 = variant == 1;
    if (a.dnbr) {
        if (pull) {
            if (m1) sweep_aa_x2_kernel<real, true, M1, true><<<grid, block, 0, s>>>(a);
            else sweep_aa_x2_kernel<real, true, M0, true><<<grid, block, 0, s>>>(a);
        } else {
            if (m1) sweep_aa_x2_kernel<real, false, M1, true><<<grid, block, 0, s>>>(a);
            else sweep_aa_x2_kernel<real, false, M0, true><<<grid, block, 0, s>>>(a);
        }
    } else if (pull) {
        if (m1) sweep_aa_x2_kernel<real, true, M1, false><<<grid, block, 0, s>>>(a);
        else sweep_aa_x2_kernel<real, true, M0, false><<<grid, block, 0, s>>>(a);
    } else {
        if (m1) sweep_aa_x2_kernel<real, false, M1, false><<<grid, block, 0, s>>>(a);
        else sweep_aa_x2_kernel<real, false, M0, false><<<grid, block, 0, s>>>(a);
    }
    return cudaGetLastError();
}

template cudaError_t launch_sweep_aa<float>(const SweepArgs<float> &, int64_t, bool, int, cudaStream_t);
template cudaError_t launch_sweep_aa<double>(const SweepArgs<double> &, int64_t, bool, int, cudaStream_t);

}  // namespace lbm
