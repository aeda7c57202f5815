// sweep.cu -- the two-grid sweep kernels of the D3Q19 LBGK patch solver (sm_100a).
//
// The hot loop is the fused pull stream + bounce-back + BGK collide update of
// eq:lbm / eq:feq with centred PDFs, pull streaming
// from two grids and half-way bounce-back with a moving-wall term
// (P:482-490).  SoA layout: one q-slice per direction, rows
// padded so interior x = 0 is aligned.  The kernel is HBM-bound:
// 19 loads + 19 stores of sizeof(real) per fluid cell, no data
// reuse across directions (each src element is pulled by exactly one cell), so
// there is nothing to stage in shared memory; the design goal is enough
// independent loads in flight per SM and fully coalesced, sector-aligned
// stores.  Default: sweep_x2_kernel (two cells per thread), optionally storing
// the outgoing PDFs of patch-face cells straight into neighbour ghost layers.
#include <cstdint>
#include <utility>

#include "collide.cuh"
#include "kernels.cuh"
#include "direct_stores.cuh"
#include "sweep_common.cuh"

namespace lbm {

template <typename real, int MINB, int STCS, int ZC>
__global__ void __launch_bounds__(SWEEP_BX *SWEEP_BY, MINB) sweep_kernel(const SweepArgs<real> a)
{
    // Locate this block's box (binary search over the tile prefix sums).
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
    const int z0 = bx.lo[2] + tz * ZC;
    if (x >= bx.lo[0] + bx.n[0] || y >= bx.lo[1] + bx.n[1]) return;
    const int zend = bx.lo[2] + bx.n[2];

    const Geom &g = a.g;
    const int64_t qs = g.qs;
    const int64_t cell0 = cell_index(g, x, y, z0);
    const int64_t pbase0 = (int64_t)bx.patch * g.ps + cell0;
    const int64_t fbase0 = (int64_t)bx.patch * g.fs + cell0;
    // ZC cells per thread along z (ZC = 2 doubles the independent loads in flight).
    uint8_t k[ZC];
    real p[ZC][Q];
#pragma unroll
    for (int c = 0; c < ZC; ++c) k[c] = (z0 + c < zend) ? a.kind[fbase0 + c * g.plane] : (uint8_t)2;
    // Pull: p_i = src_i(x - e_i), branch-free.  When x - e_i is a
    // wall cell, its slot i already holds the half-way bounce-back value
    // f_opp(i)(x) + 6 w_i rho0 e_i.u_w (R3), written there by x's
    // own update of the previous step (store-side bounce-back below) or by
    // bb_fill after the state was set.  Issued for every cell in the box
    // together with the kind byte (one DRAM round trip per cell).
#pragma unroll
    for (int c = 0; c < ZC; ++c) {
        if (c > 0 && z0 + c >= zend) break;
        const real *s = a.src + pbase0 + c * g.plane;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            p[c][i] = ld_stream(s + i * qs - sh);
        }
    }
#pragma unroll
    for (int c = 0; c < ZC; ++c) {
        if (k[c] == 2) continue;  // non-fluid (or beyond the box): never updated (R13)
        const int64_t fbase = fbase0 + c * g.plane;
        uint8_t nbf[Q];
        if (k[c] == 1) {
#pragma unroll
            for (int j = 1; j < Q; ++j) {
                const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                nbf[j] = a.flags[fbase + sh];  // flag of x + e_j
            }
        }
        collide_bgk<real>(p[c], a.omega);
        real *d = a.dst + pbase0 + c * g.plane;
#pragma unroll
        for (int i = 0; i < Q; ++i) st_stream<real, STCS>(d + i * qs, p[c][i]);
        if (k[c] == 1) {
            // Store-side bounce-back: f_j(x) leaving toward the wall w = x + e_j comes
            // back to x next step as direction opp(j); park it (plus the moving-wall
            // term of the delivered direction opp(j)) in w's slot opp(j).
#pragma unroll
            for (int j = 1; j < Q; ++j) {
                if (nbf[j] != 0) {
                    const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                    real v = p[c][j];
                    if (nbf[j] >= 2) v += a.corr[(nbf[j] - 2) * Q + OPP(j)];
                    d[OPP(j) * qs + sh] = v;
                }
            }
        }
    }
}

// Sweep with two cells per thread along x: the 9 directions with e_x = 0 are
// pulled with aligned 2-vector loads (float2 / double2) and all 19 outputs are
// written with 2-vector stores, so every fp32 warp instruction moves 256 B like
// the one-cell fp64 sweep
// (fp32 with one cell per thread sustains 5.45 TB/s of DRAM traffic vs 6.04 for
// fp64, profiles/r01_ncu_*).  A pair containing a non-fluid cell stores
// scalars: a wall cell's slots hold store-side bounce-back values of its
// neighbours and must not be overwritten.  Block (32, 4) threads = 64 x 4 cells.


template <typename real, int MINB, int STCS, bool DIRECT>
__global__ void __launch_bounds__(32 * SWEEP_BY, MINB) sweep_x2_kernel(const SweepArgs<real> a)
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
    const int64_t cell = cell_index(g, x0, y, z);  // even element index (x0 + xo even)
    const int64_t pbase = (int64_t)bx.patch * g.ps + cell;
    const int64_t fbase = (int64_t)bx.patch * g.fs + cell;
    uint8_t k0 = a.kind[fbase];
    uint8_t k1 = has1 ? a.kind[fbase + 1] : (uint8_t)2;
    // x-face neighbour of this pair for the direct ghost stores: -x if x0 == 0,
    // else +x (the +x one of a pair on both faces, n0 <= 2, loads late)
    real *nb_x = nullptr;
    if (DIRECT && (x0 == 0 || x0 + 1 >= g.n[0] - 1)) nb_x = direct_ptr(a, bx.patch, x0 == 0 ? 8 : 9);
    const real *s = a.src + pbase;
    real p0[Q], p1[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
        if (EX(i) == 0) {
            const V2 v = __ldg(reinterpret_cast<const V2 *>(s + i * qs - sh));
            p0[i] = v.x;
            p1[i] = v.y;
        } else {
            p0[i] = __ldg(s + i * qs - sh);
            p1[i] = __ldg(s + i * qs - sh + 1);
        }
    }
    if (k0 == 2 && k1 == 2) return;
    uint8_t f0[Q], f1[Q];
    if (k0 == 1 || k1 == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
            f0[j] = k0 == 1 ? a.flags[fbase + sh] : (uint8_t)0;
            f1[j] = k1 == 1 ? a.flags[fbase + 1 + sh] : (uint8_t)0;
        }
    }
    collide_bgk<real>(p0, a.omega);
    collide_bgk<real>(p1, a.omega);
    real *d = a.dst + pbase;
    if (k0 != 2 && k1 != 2) {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            V2 *dp = reinterpret_cast<V2 *>(d + i * qs);
            if (STCS)
                {
                V2 w;
                w.x = p0[i];
                w.y = p1[i];
                __stcs(dp, w);
            }
            else
                {
                V2 w;
                w.x = p0[i];
                w.y = p1[i];
                *dp = w;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (k0 != 2) d[i * qs] = p0[i];
            if (k1 != 2) d[i * qs + 1] = p1[i];
        }
    }
    // store-side bounce-back (sweep_kernel above)
    if (k0 == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j)
            if (f0[j] != 0) {
                const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                real v = p0[j];
                if (f0[j] >= 2) v += a.corr[(f0[j] - 2) * Q + OPP(j)];
                d[OPP(j) * qs + sh] = v;
            }
    }
    if (k1 == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j)
            if (f1[j] != 0) {
                const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                real v = p1[j];
                if (f1[j] >= 2) v += a.corr[(f1[j] - 2) * Q + OPP(j)];
                d[OPP(j) * qs + sh + 1] = v;
            }
    }
    if (DIRECT) direct_stores_x2<real>(a, bx.patch, x0, y, z, k0 != 2, k1 != 2, p0, p1, nb_x);
}

template <typename real>
static bool launch_x2(const SweepArgs<real> &a, unsigned grid, int variant, cudaStream_t s)
{
    dim3 block(32, SWEEP_BY, 1);
    // min blocks of 128 threads: fp32 4 / 5, fp64 2 / 3 (38 live doubles per thread)
    constexpr int M0 = sizeof(real) == 8 ? 2 : 4, M1 = sizeof(real) == 8 ? 3 : 5;
    if (a.dnbr) {
        switch (variant) {
        case 12: sweep_x2_kernel<real, M0, 0, true><<<grid, block, 0, s>>>(a); break;
        default: sweep_x2_kernel<real, M1, 0, true><<<grid, block, 0, s>>>(a); break;
        }
        return true;
    }
    switch (variant) {
    case 12: sweep_x2_kernel<real, M0, 0, false><<<grid, block, 0, s>>>(a); break;
    case 13: sweep_x2_kernel<real, M1, 0, false><<<grid, block, 0, s>>>(a); break;
    case 14: sweep_x2_kernel<real, M0, 1, false><<<grid, block, 0, s>>>(a); break;
    default: sweep_x2_kernel<real, M1, 1, false><<<grid, block, 0, s>>>(a); break;
    }
    return true;
}

// 27 -> 18 neighbour-direction index (plan.cpp kDirs order; -1: centre / corner).
__constant__ int8_t c_dir27[27] = {-1, 0,  -1, 1,  2,  3,  -1, 4,  -1, 5,  6,  7,  8, -1,
                                   9,  10, 11, 12, -1, 13, -1, 14, 15, 16, -1, 17, -1};

// Two-grid sweep whose face cells pull across patch boundaries straight from
// the same-GPU neighbour patch: no ghost copy between
// local patches.  A source cell x - e_i outside the patch belongs to the
// neighbour in direction (ox, oy, oz) and sits at (x - e_i) - (ox, oy, oz) * n
// in its coordinates.  Wall sources keep the store-side bounce-back value of the
// patch's own ghost layer; remote neighbours keep the exchanged ghosts.
template <typename real, int MINB, int STCS>
__global__ void __launch_bounds__(SWEEP_BX *SWEEP_BY, MINB) sweep_lp_kernel(const SweepArgs<real> a)
{
    const int64_t b = blockIdx.x;
    int lo = 0, hi = a.nboxes;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a.tile_prefix[mid] <= b) lo = mid; else hi = mid;
    }
    const Box &bx = a.boxes[lo];
    // The tile's patch neighbours, indexed by (oz+1)*9 + (oy+1)*3 + (ox+1).
    __shared__ const real *tab[27];
    const int tid = threadIdx.y * SWEEP_BX + threadIdx.x;
    if (tid < 27) {
        const int kd = c_dir27[tid];
        tab[tid] = kd < 0 ? nullptr : a.lnbr[((int64_t)bx.patch * NDIR + kd) * 2 + a.srci];
    }
    __syncthreads();
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
    const real *s = a.src + pbase;
    const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
    // y / z faces are uniform over a warp (32 consecutive x of one row); an x face
    // is one lane, whose e_x != 0 directions are redirected by predication.
    const bool xlo = x == 0, xhi = x == n0 - 1;
    const int oyl = y == 0 ? -1 : 0, oyh = y == n1 - 1 ? 1 : 0;
    const int ozl = z == 0 ? -1 : 0, ozh = z == n2 - 1 ? 1 : 0;
    real p[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
        const real *addr = s + i * qs - sh;
        const int ox = EX(i) == 1 ? (xlo ? -1 : 0) : (EX(i) == -1 ? (xhi ? 1 : 0) : 0);
        const int oy = EY(i) == 1 ? oyl : (EY(i) == -1 ? oyh : 0);
        const int oz = EZ(i) == 1 ? ozl : (EZ(i) == -1 ? ozh : 0);
        if (ox | oy | oz) {
            const real *nb = tab[(oz + 1) * 9 + (oy + 1) * 3 + (ox + 1)];
            if (nb && (k == 0 || a.flags[fbase - sh] == 0))
                addr = nb + i * qs + cell_index(g, x - EX(i) - ox * n0, y - EY(i) - oy * n1, z - EZ(i) - oz * n2);
        }
        p[i] = ld_stream(addr);
    }
    if (k == 2) return;
    uint8_t nbf[Q];
    if (k == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
            nbf[j] = a.flags[fbase + sh];
        }
    }
    collide_bgk<real>(p, a.omega);
    real *d = a.dst + pbase;
#pragma unroll
    for (int i = 0; i < Q; ++i) st_stream<real, STCS>(d + i * qs, p[i]);
    if (k == 1) {
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            if (nbf[j] != 0) {
                const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
                real v = p[j];
                if (nbf[j] >= 2) v += a.corr[(nbf[j] - 2) * Q + OPP(j)];
                d[OPP(j) * qs + sh] = v;
            }
        }
    }
}

// variant 0..7 = 2 * m + stcs: min blocks per SM = m + 1, stcs = evict-first
// stores, one cell per thread; 8..11: two cells per thread along z.
template <typename real>
cudaError_t launch_sweep(const SweepArgs<real> &a, int64_t total_tiles, int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    dim3 block(SWEEP_BX, SWEEP_BY, 1);
    const unsigned grid = (unsigned)total_tiles;
    if (variant >= 12 && launch_x2<real>(a, grid, variant, s)) return cudaGetLastError();
    if (a.lnbr && variant >= 4 && variant < 8) {
        switch (variant) {
        case 4: sweep_lp_kernel<real, 3, 0><<<grid, block, 0, s>>>(a); break;
        case 5: sweep_lp_kernel<real, 3, 1><<<grid, block, 0, s>>>(a); break;
        case 6: sweep_lp_kernel<real, 4, 0><<<grid, block, 0, s>>>(a); break;
        default: sweep_lp_kernel<real, 4, 1><<<grid, block, 0, s>>>(a); break;
        }
        return cudaGetLastError();
    }
    switch (variant) {
    case 0: sweep_kernel<real, 1, 0, 1><<<grid, block, 0, s>>>(a); break;
    case 1: sweep_kernel<real, 1, 1, 1><<<grid, block, 0, s>>>(a); break;
    case 2: sweep_kernel<real, 2, 0, 1><<<grid, block, 0, s>>>(a); break;
    case 3: sweep_kernel<real, 2, 1, 1><<<grid, block, 0, s>>>(a); break;
    case 4: sweep_kernel<real, 3, 0, 1><<<grid, block, 0, s>>>(a); break;
    case 5: sweep_kernel<real, 3, 1, 1><<<grid, block, 0, s>>>(a); break;
    case 6: sweep_kernel<real, 4, 0, 1><<<grid, block, 0, s>>>(a); break;
    case 7: sweep_kernel<real, 4, 1, 1><<<grid, block, 0, s>>>(a); break;
    case 8: sweep_kernel<real, 2, 0, 2><<<grid, block, 0, s>>>(a); break;
    case 9: sweep_kernel<real, 2, 1, 2><<<grid, block, 0, s>>>(a); break;
    case 10: sweep_kernel<real, 3, 0, 2><<<grid, block, 0, s>>>(a); break;
    case 11: sweep_kernel<real, 3, 1, 2><<<grid, block, 0, s>>>(a); break;
    default: sweep_kernel<real, 3, 1, 1><<<grid, block, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

template cudaError_t launch_sweep<float>(const SweepArgs<float> &, int64_t, int, cudaStream_t);
template cudaError_t launch_sweep<double>(const SweepArgs<double> &, int64_t, int, cudaStream_t);

}  // namespace lbm
