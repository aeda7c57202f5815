// sweep_aa.cu -- AA-pattern in-place sweep kernels (one PDF array; north_star
// (a)): the update of sweep.cu in alternating PULL /
// LOCAL steps.
#include <cstdint>

#include "collide.cuh"
#include "kernels.cuh"
#include "direct_stores.cuh"
#include "sweep_common.cuh"

namespace lbm {

// ------------------------------------------------------------------ AA pattern
// One PDF array, two alternating in-place kernels (north_star (a)).
// With S_i(x) the post-collision state of the two-grid scheme:
//   swapped  representation (after an even step count): A[x][opp(i)] = S_i(x)
//   streamed representation (after an odd step count):  A[x][i] = p_i(x), the
//                                                        value x pulls next
// PULL  (swapped -> streamed): p_i = A[x - e_i][opp(i)]; collide; write out_i to
//       A[x + e_i][i], or -- x + e_i a wall -- its bounce-back
//       out_i + 6 w rho0 e_opp(i).u_w to A[x][opp(i)] (R3).
// LOCAL (streamed -> swapped): p_i = A[x][i]; collide; A[x][opp(i)] = out_i, and
//       for walls w = x + e_j the store-side bounce-back A[w][j] = out_j + corr,
//       which the next PULL gathers branch-free.
// Every slot has exactly one writer per step and is read only by it, so both
// kernels run in place without races; the results equal the two-grid scheme
// bitwise after every even step count.
template <typename real, bool PULL, int MINB, int STCS>
__global__ void __launch_bounds__(SWEEP_BX *SWEEP_BY, MINB) sweep_aa_kernel(const SweepArgs<real> a)
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
    const int x = bx.lo[0] + tx * SWEEP_BX + (int)threadIdx.x;
    const int y = bx.lo[1] + ty * SWEEP_BY + (int)threadIdx.y;
    const int z = bx.lo[2] + tz;
    if (x >= bx.lo[0] + bx.n[0] || y >= bx.lo[1] + bx.n[1]) return;

    const Geom &g = a.g;
    const int64_t qs = g.qs;
    const int64_t cell = cell_index(g, x, y, z);
    const int64_t pbase = (int64_t)bx.patch * g.ps + cell;
    const int64_t fbase = (int64_t)bx.patch * g.fs + cell;
    const uint8_t k = a.kind[fbase];
    real *A = a.dst + pbase;  // in place: src == dst
    real p[Q];
    if (PULL) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            p[i] = ld_stream((const real *)A + OPP(i) * qs - sh);
        }
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) p[i] = ld_stream((const real *)A + i * qs);
    }
    if (k == 2) return;
    uint8_t nbf[Q];
    if (k == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
            nbf[j] = a.flags[fbase + sh];  // flag of x + e_j
        }
    }
    collide_bgk<real>(p, a.omega);
    if (PULL) {
        st_stream<real, STCS>(A, p[0]);
#pragma unroll
        for (int i = 1; i < Q; ++i) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            if (k == 1 && nbf[i] != 0) {
                real v = p[i];
                if (nbf[i] >= 2) v += a.corr[(nbf[i] - 2) * Q + OPP(i)];
                A[OPP(i) * qs] = v;
            } else {
                st_stream<real, STCS>(A + i * qs + sh, p[i]);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) st_stream<real, STCS>(A + OPP(i) * qs, p[i]);
        if (k == 1) {
#pragma unroll
            for (int j = 1; j < Q; ++j) {
                if (nbf[j] != 0) {
                    const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                    real v = p[j];
                    if (nbf[j] >= 2) v += a.corr[(nbf[j] - 2) * Q + OPP(j)];
                    A[j * qs + sh] = v;
                }
            }
        }
    }
}

// AA-pattern kernels with two cells per thread along x (cf. sweep_x2_kernel):
// LOCAL reads and writes only its own cells, so all 19 loads and 19 stores are
// aligned 2-vectors; PULL vectorises the 9 gathers and scatters with e_x = 0.
// A pair whose cells differ in kind (non-fluid, or a bounce-back redirect for
// that direction) falls back to scalar accesses.  Pairs with no wall next to
// either cell (kind 0, the common case) take a straight-line store path: the
// per-direction redirect tests cost PULL +41 % instructions over the two-grid
// sweep in this latency-bound kernel (1.05 -> 0.88 ms at 256^3 fp64,
// profiles/r01_ncu_aa_*).  Realigning the 10 e_x != 0 scatters into 2-vectors
// with warp shuffles was measured slower (tools/stream_ceiling.cu mode 3: the
// ceiling gains 1.6 %, the kernel loses more to the shuffles).
// ------------------------------------------------- direct ghost stores (AA)
// The AA pattern's two half-exchanges folded into the
// sweep, as sweep.cu does for the two-grid layout:
//   LOCAL: a fluid cell g on a patch face / edge stores out_q, for each q that
//          travels into the neighbour, into the neighbour's ghost copy of g at
//          slot opp(q) -- what the neighbour's next PULL gathers there (the
//          two-grid store pattern, direct_stores.cuh with OPPSLOT);
//   PULL:  a fluid cell x whose scatter target x + e_q lies in a neighbour patch
//          (and is fluid) stores out_q into that cell of the neighbour, slot q --
//          what the neighbour's next LOCAL reads.  Only fluid writers store:
//          the writer mask of half-exchange 2 holds by construction.
// Every slot keeps exactly one writer per step, so this races with nothing.

// (oz, oy, ox) + 1 in base 3 -> neighbour direction kd of the plan order, -1: none
__constant__ int8_t c_kd27[27] = {-1, 0,  -1, 1,  2,  3,  -1, 4,  -1, 5,  6,  7,  8, -1,
                                  9,  10, 11, 12, -1, 13, -1, 14, 15, 16, -1, 17, -1};

template <typename real>
__device__ __forceinline__ void aa_pull_direct(const SweepArgs<real> &a, int patch, int x, int y, int z, uint8_t k,
                                               const uint8_t *f, const real *p)
{
    const Geom &g = a.g;
    const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        const int dx = x + EX(q), dy = y + EY(q), dz = z + EZ(q);
        const int ox = dx < 0 ? -1 : (dx >= n0 ? 1 : 0);
        const int oy = dy < 0 ? -1 : (dy >= n1 ? 1 : 0);
        const int oz = dz < 0 ? -1 : (dz >= n2 ? 1 : 0);
        if ((ox | oy | oz) == 0) continue;   // target inside the patch
        if (k == 1 && f[q] != 0) continue;   // wall target: the bounce-back stays at x
        const int kd = c_kd27[(oz + 1) * 9 + (oy + 1) * 3 + (ox + 1)];
        real *nb = direct_ptr(a, patch, kd);
        if (!nb) continue;
        nb[q * g.qs + cell_index(g, dx - ox * n0, dy - oy * n1, dz - oz * n2)] = p[q];
    }
}

// PULL, a cell on the x face S (-1 / +1) and on no y / z face: its scatter
// targets x + e_q with e_qx = S are the x neighbour's cells
// (x + S - S n0, y + e_qy, z + e_qz); y +- 1, z +- 1 stay inside the patch.
template <typename real, int S>
__device__ __forceinline__ void aa_pull_xface(const SweepArgs<real> &a, real *nb, int x, int y, int z, uint8_t k,
                                              const uint8_t *f, const real *p)
{
    if (!nb) return;
    const Geom &g = a.g;
    real *row = nb + cell_index(g, x + S - S * g.n[0], y, z);
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (EXf(q) != S) continue;
        if (k == 1 && f[q] != 0) continue;  // wall target: the bounce-back stays at x
        row[q * g.qs + EYf(q) * (int64_t)g.px + EZf(q) * g.plane] = p[q];
    }
}

// A pair (x0, x0 + 1): only cells on a patch face do anything.  nb_x: the x
// neighbour of the pair's x-face cell (-x if x0 == 0, else +x), loaded up front.
// LOCAL stores like the two-grid sweep (direct_stores.cuh), into slot opp(q).
template <typename real, bool PULL>
__device__ __forceinline__ void aa_direct_pair(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool has1,
                                               uint8_t k0, uint8_t k1, const uint8_t *f0, const uint8_t *f1,
                                               const real *p0, const real *p1, real *nb_x)
{
    if (!PULL) {
        direct_stores_x2<real, true>(a, patch, x0, y, z, k0 != 2, has1 && k1 != 2, p0, p1, nb_x);
        return;
    }
    const Geom &g = a.g;
    const int n0 = g.n[0];
    const bool yzf = y == 0 || y == g.n[1] - 1 || z == 0 || z == g.n[2] - 1;  // warp-uniform
    if (yzf) {
        if (k0 != 2) aa_pull_direct<real>(a, patch, x0, y, z, k0, f0, p0);
        if (has1 && k1 != 2) aa_pull_direct<real>(a, patch, x0 + 1, y, z, k1, f1, p1);
        return;
    }
    if (x0 == 0) {
        if (k0 != 2) aa_pull_xface<real, -1>(a, nb_x, x0, y, z, k0, f0, p0);
        if (n0 == 1 && k0 != 2) aa_pull_xface<real, 1>(a, direct_ptr(a, patch, 9), x0, y, z, k0, f0, p0);
        if (n0 == 2 && has1 && k1 != 2) aa_pull_xface<real, 1>(a, direct_ptr(a, patch, 9), x0 + 1, y, z, k1, f1, p1);
    } else {
        if (x0 == n0 - 1 && k0 != 2) aa_pull_xface<real, 1>(a, nb_x, x0, y, z, k0, f0, p0);
        if (has1 && x0 + 1 == n0 - 1 && k1 != 2) aa_pull_xface<real, 1>(a, nb_x, x0 + 1, y, z, k1, f1, p1);
    }
}

template <typename real, bool PULL, int MINB, bool DIRECT>
__global__ void __launch_bounds__(32 * SWEEP_BY, MINB) sweep_aa_x2_kernel(const SweepArgs<real> a)
{
    using V2 = typename Vec2<real>::T;
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
    const int x0 = bx.lo[0] + tx * SWEEP_BX + 2 * (int)threadIdx.x;
    const int y = bx.lo[1] + ty * SWEEP_BY + (int)threadIdx.y;
    const int z = bx.lo[2] + tz;
    const int xend = bx.lo[0] + bx.n[0];
    if (x0 >= xend || y >= bx.lo[1] + bx.n[1]) return;
    const bool has1 = x0 + 1 < xend;

    const Geom &g = a.g;
    const int64_t qs = g.qs;
    const int64_t cell = cell_index(g, x0, y, z);
    const int64_t pbase = (int64_t)bx.patch * g.ps + cell;
    const int64_t fbase = (int64_t)bx.patch * g.fs + cell;
    const uint8_t k0 = a.kind[fbase];
    const uint8_t k1 = has1 ? a.kind[fbase + 1] : (uint8_t)2;
    real *nb_x = nullptr;  // x-face neighbour for the direct ghost stores, loaded with the PDFs
    if (DIRECT && (x0 == 0 || x0 + 1 >= g.n[0] - 1)) nb_x = direct_ptr(a, bx.patch, x0 == 0 ? 8 : 9);
    real *A = a.dst + pbase;  // in place
    real p0[Q], p1[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        if (PULL) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            const real *src = A + OPP(i) * qs - sh;
            if (EX(i) == 0) {
                const V2 v = __ldg(reinterpret_cast<const V2 *>(src));
                p0[i] = v.x;
                p1[i] = v.y;
            } else {
                p0[i] = __ldg(src);
                p1[i] = __ldg(src + 1);
            }
        } else {
            const V2 v = __ldg(reinterpret_cast<const V2 *>(A + i * qs));
            p0[i] = v.x;
            p1[i] = v.y;
        }
    }
    if (k0 == 2 && k1 == 2) return;
    uint8_t f0[Q], f1[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) f0[j] = f1[j] = 0;
    if (k0 == 1 || k1 == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
            if (k0 == 1) f0[j] = a.flags[fbase + sh];
            if (k1 == 1) f1[j] = a.flags[fbase + 1 + sh];
        }
    }
    collide_bgk<real>(p0, a.omega);
    collide_bgk<real>(p1, a.omega);
    const bool both = k0 != 2 && k1 != 2;
    if (PULL && k0 == 0 && k1 == 0) {
        // no wall next to either cell (the common case): straight-line scatter
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            if (EX(i) == 0) {
                V2 w;
                w.x = p0[i];
                w.y = p1[i];
                *reinterpret_cast<V2 *>(A + i * qs + sh) = w;
            } else {
                A[i * qs + sh] = p0[i];
                A[i * qs + sh + 1] = p1[i];
            }
        }
    } else if (PULL) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            const bool r0 = f0[i] != 0, r1 = f1[i] != 0;  // x + e_i is a wall: bounce back into x
            if (EX(i) == 0 && both && !r0 && !r1) {
                V2 w;
                w.x = p0[i];
                w.y = p1[i];
                *reinterpret_cast<V2 *>(A + i * qs + sh) = w;
                continue;
            }
            if (k0 != 2) {
                if (r0) {
                    real v = p0[i];
                    if (f0[i] >= 2) v += a.corr[(f0[i] - 2) * Q + OPP(i)];
                    A[OPP(i) * qs] = v;
                } else {
                    A[i * qs + sh] = p0[i];
                }
            }
            if (k1 != 2) {
                if (r1) {
                    real v = p1[i];
                    if (f1[i] >= 2) v += a.corr[(f1[i] - 2) * Q + OPP(i)];
                    A[OPP(i) * qs + 1] = v;
                } else {
                    A[i * qs + sh + 1] = p1[i];
                }
            }
        }
    } else {
        if (both) {
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                V2 w;
                w.x = p0[i];
                w.y = p1[i];
                *reinterpret_cast<V2 *>(A + OPP(i) * qs) = w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                if (k0 != 2) A[OPP(i) * qs] = p0[i];
                if (k1 != 2) A[OPP(i) * qs + 1] = p1[i];
            }
        }
        if (k0 == 1 || k1 == 1) {
            // store-side bounce-back into wall slots (see sweep_aa_kernel)
#pragma unroll
            for (int j = 1; j < Q; ++j) {
                const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                if (f0[j] != 0) {
                    real v = p0[j];
                    if (f0[j] >= 2) v += a.corr[(f0[j] - 2) * Q + OPP(j)];
                    A[j * qs + sh] = v;
                }
                if (f1[j] != 0) {
                    real v = p1[j];
                    if (f1[j] >= 2) v += a.corr[(f1[j] - 2) * Q + OPP(j)];
                    A[j * qs + sh + 1] = v;
                }
            }
        }
    }
    if (DIRECT) aa_direct_pair<real, PULL>(a, bx.patch, x0, y, z, has1, k0, k1, f0, f1, p0, p1, nb_x);
}

template <typename real>
static void launch_aa_x2(const SweepArgs<real> &a, unsigned grid, bool pull, int variant, cudaStream_t s)
{
    dim3 block(32, SWEEP_BY, 1);
    constexpr int M0 = sizeof(real) == 8 ? 2 : 4, M1 = sizeof(real) == 8 ? 3 : 5;
    // 12 / 14: min blocks M0; 13 / 15: M1; a.dnbr: with direct ghost stores
    const bool m1 = variant == 13 || variant == 15;
    if (a.dnbr) {
        if (pull) {
            if (m1) sweep_aa_x2_kernel<real, true, M1, true><<<grid, block, 0, s>>>(a);
            else sweep_aa_x2_kernel<real, true, M0, true><<<grid, block, 0, s>>>(a);
        } else {
            if (m1) sweep_aa_x2_kernel<real, false, M1, true><<<grid, block, 0, s>>>(a);
            else sweep_aa_x2_kernel<real, false, M0, true><<<grid, block, 0, s>>>(a);
        }
        return;
    }
    if (pull) {
        if (m1) sweep_aa_x2_kernel<real, true, M1, false><<<grid, block, 0, s>>>(a);
        else sweep_aa_x2_kernel<real, true, M0, false><<<grid, block, 0, s>>>(a);
    } else {
        if (m1) sweep_aa_x2_kernel<real, false, M1, false><<<grid, block, 0, s>>>(a);
        else sweep_aa_x2_kernel<real, false, M0, false><<<grid, block, 0, s>>>(a);
    }
}

template <typename real>
cudaError_t launch_sweep_aa(const SweepArgs<real> &a, int64_t total_tiles, bool pull, int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    dim3 block(SWEEP_BX, SWEEP_BY, 1);
    const unsigned grid = (unsigned)total_tiles;
    if (variant >= 12) {
        launch_aa_x2<real>(a, grid, pull, variant, s);
        return cudaGetLastError();
    }
    const int v = variant & 7;  // min blocks / store hint as for the two-grid sweep
    if (pull) {
        switch (v) {
        case 4: sweep_aa_kernel<real, true, 3, 0><<<grid, block, 0, s>>>(a); break;
        case 5: sweep_aa_kernel<real, true, 3, 1><<<grid, block, 0, s>>>(a); break;
        case 6: sweep_aa_kernel<real, true, 4, 0><<<grid, block, 0, s>>>(a); break;
        case 7: sweep_aa_kernel<real, true, 4, 1><<<grid, block, 0, s>>>(a); break;
        default: sweep_aa_kernel<real, true, 2, 0><<<grid, block, 0, s>>>(a); break;
        }
    } else {
        switch (v) {
        case 4: sweep_aa_kernel<real, false, 3, 0><<<grid, block, 0, s>>>(a); break;
        case 5: sweep_aa_kernel<real, false, 3, 1><<<grid, block, 0, s>>>(a); break;
        case 6: sweep_aa_kernel<real, false, 4, 0><<<grid, block, 0, s>>>(a); break;
        case 7: sweep_aa_kernel<real, false, 4, 1><<<grid, block, 0, s>>>(a); break;
        default: sweep_aa_kernel<real, false, 2, 0><<<grid, block, 0, s>>>(a); break;
        }
    }
    return cudaGetLastError();
}

template cudaError_t launch_sweep_aa<float>(const SweepArgs<float> &, int64_t, bool, int, cudaStream_t);
template cudaError_t launch_sweep_aa<double>(const SweepArgs<double> &, int64_t, bool, int, cudaStream_t);

}  // namespace lbm
