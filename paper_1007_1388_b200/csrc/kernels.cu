// kernels.cu -- sm_100a kernels of the D3Q19 LBGK patch solver.
//
// The hot loop is sweep_kernel: the fused pull stream + bounce-back + BGK
// collide update of eq:lbm / eq:feq with centred PDFs,
// pull streaming from two grids and half-way bounce-back with a
// moving-wall term.  SoA layout: one q-slice per
// direction, rows padded so interior x = 0 is aligned.  The
// kernel is HBM-bound: 19 loads + 19 stores of sizeof(real) per fluid cell
// (P:1075-1082), no data reuse across directions (each src element is pulled
// by exactly one cell), so there is nothing to stage in shared memory; the
// design goal is enough independent loads in flight per SM and fully
// coalesced, sector-aligned stores.
#include <cstdint>
#include <utility>

#include "collide.cuh"
#include "kernels.cuh"

namespace lbm {

__device__ __forceinline__ int64_t cell_index(const Geom &g, int x, int y, int z)
{
    return ((int64_t)(z + 1) * g.py + (y + 1)) * (int64_t)g.px + (x + g.xo);
}

template <typename real>
__device__ __forceinline__ real ld_stream(const real *p)
{
    return __ldg(p);
}

template <typename real, int STCS>
__device__ __forceinline__ void st_stream(real *p, real v)
{
    if (STCS)
        __stcs(p, v);  // evict-first: dst is not re-read in this sweep
    else
        *p = v;
}

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
template <typename real> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

// Direct ghost stores of a cell pair (x0, x0 + 1) -- the pack / copy / unpack of
// P:331-337 folded into the sweep: a fluid cell on a patch face or edge stores
// each PDF that travels into the neighbour at d (5 per face, 1 per edge) into
// that neighbour's ghost cell at the same global position, in the grid the
// neighbour pulls from next step.  c0 / c1: the cell is fluid and in the box.
// A ghost column (x = -1, or x = n when sector-aligned) shares its 32-B sector
// only with row padding, which nothing reads: storing the whole sector (value +
// zeros) spares L2 the DRAM fill of a partially written sector -- strided
// 4 / 8-B column stores otherwise cost a read-modify-write each.
template <typename real>
__device__ __forceinline__ void st_ghost_sector(real *sector, bool last, real v)
{
    if constexpr (sizeof(real) == 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (last) b.w = v; else a.x = v;
        reinterpret_cast<float4 *>(sector)[0] = a;
        reinterpret_cast<float4 *>(sector)[1] = b;
    } else {
        double2 a = make_double2(0.0, 0.0), b = a;
        if (last) b.y = v; else a.x = v;
        reinterpret_cast<double2 *>(sector)[0] = a;
        reinterpret_cast<double2 *>(sector)[1] = b;
    }
}

// Direct stores toward neighbour kd (compile-time after unrolling) of a cell
// pair whose cells are on that side (on0 / on1).
template <typename real>
__device__ __forceinline__ real *direct_ptr(const SweepArgs<real> &a, int patch, int kd)
{
    return (real *)__ldg(reinterpret_cast<const unsigned long long *>(a.dnbr + ((int64_t)patch * NDIR + kd) * 2 +
                                                                      a.dsti));
}

template <typename real, int KD>
__device__ __forceinline__ void direct_dir_x2(const SweepArgs<real> &a, real *nb, int x0, int y, int z, bool on0,
                                              bool on1, const real *p0, const real *p1)
{
    using V2 = typename Vec2<real>::T;
    constexpr int ddx = ndir(KD, 0), ddy = ndir(KD, 1), ddz = ndir(KD, 2);
    if ((!on0 && !on1) || !nb) return;
    const Geom &g = a.g;
    const int64_t qs = g.qs;
    const int n0 = g.n[0];
    real *gb = nb + cell_index(g, x0 - ddx * n0, y - ddy * g.n[1], z - ddz * g.n[2]);
    if constexpr (ddx != 0) {
        constexpr int SE = 32 / (int)sizeof(real);  // elements per 32-B sector
        // ghost column x = -1 (ddx > 0) ends a sector; x = n0 (ddx < 0) may start one
        const bool whole = ddx > 0 ? (g.xo >= SE && g.xo % SE == 0)
                                   : ((g.xo + n0) % SE == 0 && g.xo + n0 + SE <= g.px);
        if (whole) {
            // exactly one cell of the pair lies on the x face (x0 == 0 for ddx < 0;
            // x0 or x0 + 1 == n0 - 1 for ddx > 0)
            const real *pv = on0 ? p0 : p1;
            real *gs = gb + (on0 ? 0 : 1) - (ddx > 0 ? SE - 1 : 0);
#pragma unroll
            for (int q = 1; q < Q; ++q)
                if (outgoing(q, KD)) st_ghost_sector<real>(gs + q * qs, ddx > 0, pv[q]);
            return;
        }
    }
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        if (!outgoing(q, KD)) continue;
        if (ddx == 0 && on0 && on1) {  // same x as the pair: aligned 2-vector
            V2 w;
            w.x = p0[q];
            w.y = p1[q];
            *reinterpret_cast<V2 *>(gb + q * qs) = w;
        } else {
            if (on0) gb[q * qs] = p0[q];
            if (on1) gb[q * qs + 1] = p1[q];
        }
    }
}

template <typename real, int KD>
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
    if (on0 || on1) direct_dir_x2<real, KD>(a, direct_ptr(a, patch, KD), x0, y, z, on0, on1, p0, p1);
}

template <typename real, int... KD>
__device__ __forceinline__ void direct_dirs_x2(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool c0,
                                               bool c1, const real *p0, const real *p1,
                                               std::integer_sequence<int, KD...>)
{
    (direct_dir_x2_on<real, KD>(a, patch, x0, y, z, c0, c1, p0, p1), ...);
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

template <typename real>
__device__ __forceinline__ void direct_stores_x2(const SweepArgs<real> &a, int patch, int x0, int y, int z, bool c0,
                                                 bool c1, const real *p0, const real *p1, real *nb_x)
{
    const Geom &g = a.g;
    const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
    const bool yzf = y == 0 || y == n1 - 1 || z == 0 || z == n2 - 1;
    if (!yzf) {
        const bool hi0 = c0 && x0 == n0 - 1, hi1 = c1 && x0 + 1 == n0 - 1;
        if (x0 == 0) {
            direct_dir_x2<real, 8>(a, nb_x, x0, y, z, c0, false, p0, p1);
            if (hi0 || hi1) direct_dir_x2<real, 9>(a, direct_ptr(a, patch, 9), x0, y, z, hi0, hi1, p0, p1);
        } else {
            direct_dir_x2<real, 9>(a, nb_x, x0, y, z, hi0, hi1, p0, p1);
        }
        return;
    }
    direct_dirs_x2<real>(a, patch, x0, y, z, c0, c1, p0, p1, std::make_integer_sequence<int, NDIR>{});
}

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
    // store-side bounce-back (kernels.cu sweep_kernel)
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
template <typename real, bool PULL, int MINB>
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
        if (k0 != 1 && k1 != 1) return;
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

template <typename real>
static void launch_aa_x2(const SweepArgs<real> &a, unsigned grid, bool pull, int variant, cudaStream_t s)
{
    dim3 block(32, SWEEP_BY, 1);
    constexpr int M0 = sizeof(real) == 8 ? 2 : 4, M1 = sizeof(real) == 8 ? 3 : 5;
    // 12 / 14: min blocks M0; 13 / 15: M1
    const bool m1 = variant == 13 || variant == 15;
    if (pull) {
        if (m1) sweep_aa_x2_kernel<real, true, M1><<<grid, block, 0, s>>>(a);
        else sweep_aa_x2_kernel<real, true, M0><<<grid, block, 0, s>>>(a);
    } else {
        if (m1) sweep_aa_x2_kernel<real, false, M1><<<grid, block, 0, s>>>(a);
        else sweep_aa_x2_kernel<real, false, M0><<<grid, block, 0, s>>>(a);
    }
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

template <typename real>
static void launch_aa_x2(const SweepArgs<real> &a, unsigned grid, bool pull, int variant, cudaStream_t s);

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

// ---------------------------------------------------------------- ghost exchange copies
// Non-fluid destination cells are skipped: their PDF slots hold the store-side
// bounce-back values written by the receiving patch itself.
template <typename real>
__global__ void __launch_bounds__(256) copy_segments_kernel(const CopySeg *segs, const real *grid_src,
                                                            real *grid_dst, const real *buf_src,
                                                            real *buf_dst, const uint8_t *flags, const Geom g)
{
    const CopySeg &sg = segs[blockIdx.y];
    // 32-bit element decomposition (a segment has < 2^31 elements).
    const int nelem = (int)sg.nelem, cells = (int)sg.cells;
    const int s0 = sg.size[0], s1 = sg.size[1];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nelem; e += gridDim.x * blockDim.x) {
        const int qi = e / cells;
        const int c = e - qi * cells;
        const int r = c / s0;
        const int cx = c - r * s0;
        const int cz = r / s1;
        const int cy = r - cz * s1;
        const int q = sg.q[qi];
        real v;
        if (sg.src_is_buf)
            v = buf_src[sg.src_base + e];
        else
            v = grid_src[sg.src_base + q * g.qs +
                         cell_index(g, sg.src_lo[0] + cx, sg.src_lo[1] + cy, sg.src_lo[2] + cz)];
        if (sg.dst_is_buf) {
            buf_dst[sg.dst_base + e] = v;
        } else {
            const int y[3] = {sg.dst_lo[0] + cx, sg.dst_lo[1] + cy, sg.dst_lo[2] + cz};
            const int64_t ci = cell_index(g, y[0], y[1], y[2]);
            bool ok = sg.mask == 1 || flags[sg.dst_flag_base + ci] == 0;  // mask 1: all destinations fluid
            if (sg.mask == 2 && ok) {
                // AA half-exchange 2: the value was scattered by the sender's cell
                // w = y - e_q; only entries whose writer is a fluid cell of the
                // sender (not another patch's ghost) are delivered.
                const int w[3] = {y[0] - EX(q), y[1] - EY(q), y[2] - EZ(q)};
                for (int a2 = 0; a2 < 3; ++a2)
                    if (sg.d[a2] == 0 && (w[a2] < 0 || w[a2] >= g.n[a2])) ok = false;
                if (ok) ok = flags[sg.dst_flag_base + cell_index(g, w[0], w[1], w[2])] == 0;
            }
            if (ok) grid_dst[sg.dst_base + q * g.qs + ci] = v;
        }
    }
}

template <typename real>
cudaError_t launch_copy_segments(const CopySeg *segs, int nseg, int64_t max_elems, const real *grid_src,
                                 real *grid_dst, const real *buf_src, real *buf_dst, const uint8_t *flags,
                                 const Geom &g, cudaStream_t s)
{
    if (nseg <= 0 || max_elems <= 0) return cudaSuccess;
    int64_t bx = (max_elems + 255) / 256;
    if (bx > 1024) bx = 1024;
    for (int off = 0; off < nseg; off += 65535) {
        int n = nseg - off < 65535 ? nseg - off : 65535;
        dim3 grid((unsigned)bx, (unsigned)n, 1);
        copy_segments_kernel<real><<<grid, 256, 0, s>>>(segs + off, grid_src, grid_dst, buf_src, buf_dst, flags, g);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- flags
__global__ void build_flags_kernel(const uint8_t *global, int64_t nx, int64_t ny, int64_t nz, int p0, int p1,
                                   int p2, const int *origin, const Geom g, uint8_t *flags)
{
    const int lp = blockIdx.y;
    const int64_t total = g.fs;
    const int periodic[3] = {p0, p1, p2};
    const int64_t n[3] = {nx, ny, nz};
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int col = (int)(e % g.px);
        const int64_t r = e / g.px;
        const int row = (int)(r % g.py);
        const int pl = (int)(r / g.py);
        const int lc[3] = {col - g.xo, row - 1, pl - 1};
        uint8_t v = 1;
        if (lc[0] >= -1 && lc[0] <= g.n[0]) {
            int64_t c[3];
            bool ok = true;
            for (int ax = 0; ax < 3; ++ax) {
                c[ax] = origin[3 * lp + ax] + lc[ax];
                if (periodic[ax]) c[ax] = (c[ax] + n[ax]) % n[ax];
                if (c[ax] < -1 || c[ax] > n[ax]) ok = false;
            }
            if (ok) v = global[((c[2] + 1) * (ny + 2) + (c[1] + 1)) * (nx + 2) + (c[0] + 1)];
        }
        flags[(int64_t)lp * g.fs + e] = v;
    }
}

// kind: 2 = non-fluid (or ghost / padding), 1 = fluid with a non-fluid
// neighbour among the 18 (needs the flag-driven path), 0 = fluid with only
// fluid neighbours (pure pull).
__global__ void build_kind_kernel(const Geom g, const uint8_t *flags, uint8_t *kind)
{
    const int lp = blockIdx.y;
    const int64_t total = g.fs;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int col = (int)(e % g.px);
        const int64_t r = e / g.px;
        const int row = (int)(r % g.py);
        const int pl = (int)(r / g.py);
        const int x = col - g.xo, y = row - 1, z = pl - 1;
        const uint8_t *f = flags + (int64_t)lp * g.fs;
        uint8_t kd = 2;
        if (x >= 0 && x < g.n[0] && y >= 0 && y < g.n[1] && z >= 0 && z < g.n[2] && f[e] == 0) {
            kd = 0;
            for (int i = 1; i < Q; ++i) {
                const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
                if (f[e - sh] != 0) kd = 1;
            }
        }
        kind[(int64_t)lp * g.fs + e] = kd;
    }
}

cudaError_t launch_build_flags(const uint8_t *global, const int64_t domain[3], const int periodic[3],
                               const int *patch_origin, int nlocal, const Geom &g, uint8_t *flags,
                               uint8_t *kind, cudaStream_t s)
{
    int64_t bx = (g.fs + 255) / 256;
    if (bx > 4096) bx = 4096;
    for (int off = 0; off < nlocal; off += 65535) {
        int n = nlocal - off < 65535 ? nlocal - off : 65535;
        dim3 grid((unsigned)bx, (unsigned)n);
        build_flags_kernel<<<grid, 256, 0, s>>>(global, domain[0], domain[1], domain[2], periodic[0], periodic[1],
                                                periodic[2], patch_origin + 3 * off, g, flags + (int64_t)off * g.fs);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    for (int off = 0; off < nlocal; off += 65535) {
        int n = nlocal - off < 65535 ? nlocal - off : 65535;
        dim3 grid((unsigned)bx, (unsigned)n);
        build_kind_kernel<<<grid, 256, 0, s>>>(g, flags + (int64_t)off * g.fs, kind + (int64_t)off * g.fs);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- import / export
struct OwnedMap {
    int64_t lo[3];
    int64_t n[3];
    int brick[3];
};

__device__ __forceinline__ void owned_to_patch(const Geom &g, const int brick[3], int64_t ox, int64_t oy,
                                               int64_t oz, int &lp, int &lx, int &ly, int &lz)
{
    const int bx = (int)(ox / g.n[0]), by = (int)(oy / g.n[1]), bz = (int)(oz / g.n[2]);
    lx = (int)(ox - (int64_t)bx * g.n[0]);
    ly = (int)(oy - (int64_t)by * g.n[1]);
    lz = (int)(oz - (int64_t)bz * g.n[2]);
    lp = (bz * brick[1] + by) * brick[0] + bx;
}

// rep: 0 = two-grid (slot i holds f_i), 1 = AA swapped (slot opp(i) holds f_i),
//      2 = AA streamed (export only: f_i(x) = A[x + e_i][i], or at a wall
//          x + e_i the bounced value A[x][opp(i)] minus its wall term).
__device__ __forceinline__ int rep_slot(int rep, int i) { return rep == 1 ? OPP(i) : i; }

template <typename real>
__device__ __forceinline__ double read_state(const real *gp, const uint8_t *fp, const real *corr, const Geom &g,
                                             int rep, int i)
{
    if (rep != 2) return (double)gp[rep_slot(rep, i) * g.qs];
    const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
    const uint8_t f = fp[sh];
    if (i == 0 || f == 0) return (double)gp[i * g.qs + sh];
    real v = gp[OPP(i) * g.qs];
    if (f >= 2) v -= corr[(f - 2) * Q + OPP(i)];
    return (double)v;
}

template <typename real>
__global__ void import_kernel(const double *canon, int64_t z0, int64_t ncells, int64_t nx, int64_t ny,
                              int b0, int b1, int b2, const Geom g, real *grid, const int rep)
{
    const int brick[3] = {b0, b1, b2};
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ox = c % nx;
        const int64_t r = c / nx;
        const int64_t oy = r % ny;
        const int64_t oz = z0 + r / ny;
        int lp, lx, ly, lz;
        owned_to_patch(g, brick, ox, oy, oz, lp, lx, ly, lz);
        real *gp = grid + (int64_t)lp * g.ps + cell_index(g, lx, ly, lz);
#pragma unroll
        for (int q = 0; q < Q; ++q) gp[rep_slot(rep, q) * g.qs] = (real)canon[c * Q + q];
    }
}

template <typename real>
__global__ void export_kernel(const real *grid, const uint8_t *flags, int64_t z0, int64_t ncells, int64_t nx,
                              int64_t ny, int b0, int b1, int b2, const Geom g, int mode, double *canon,
                              double *rho, double *u, const int rep, const real *corr)
{
    const int brick[3] = {b0, b1, b2};
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ox = c % nx;
        const int64_t r = c / nx;
        const int64_t oy = r % ny;
        const int64_t oz = z0 + r / ny;
        int lp, lx, ly, lz;
        owned_to_patch(g, brick, ox, oy, oz, lp, lx, ly, lz);
        const int64_t ci = cell_index(g, lx, ly, lz);
        const uint8_t *fp = flags + (int64_t)lp * g.fs + ci;
        const bool fluid = fp[0] == 0;
        const real *gp = grid + (int64_t)lp * g.ps + ci;
        if (mode == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) canon[c * Q + q] = fluid ? read_state(gp, fp, corr, g, rep, q) : 0.0;
        } else {
            // Macroscopic export: rho = rho0 + sum f~, u = sum e f~ / rho0.
            double s = 0, jx = 0, jy = 0, jz = 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const double v = fluid ? read_state(gp, fp, corr, g, rep, q) : 0.0;
                s += v;
                jx += EX(q) * v;
                jy += EY(q) * v;
                jz += EZ(q) * v;
            }
            if (rho) rho[c] = fluid ? 1.0 + s : 0.0;
            if (u) {
                u[3 * c] = fluid ? jx : 0.0;
                u[3 * c + 1] = fluid ? jy : 0.0;
                u[3 * c + 2] = fluid ? jz : 0.0;
            }
        }
    }
}

template <typename real>
cudaError_t launch_import(const double *canon, int64_t z0, int64_t nz_chunk, const int64_t owned_lo[3],
                          const int64_t owned_n[3], const int brick[3], const Geom &g, real *grid, int rep,
                          cudaStream_t s)
{
    (void)owned_lo;
    const int64_t ncells = owned_n[0] * owned_n[1] * nz_chunk;
    if (ncells <= 0) return cudaSuccess;
    int64_t nb = (ncells + 255) / 256;
    if (nb > 8192) nb = 8192;
    import_kernel<real><<<(unsigned)nb, 256, 0, s>>>(canon, z0, ncells, owned_n[0], owned_n[1], brick[0],
                                                    brick[1], brick[2], g, grid, rep);
    return cudaGetLastError();
}

template <typename real>
cudaError_t launch_export(const real *grid, const uint8_t *flags, int64_t z0, int64_t nz_chunk,
                          const int64_t owned_lo[3], const int64_t owned_n[3], const int brick[3],
                          const Geom &g, double *canon, int mode, double *rho, double *u, int rep,
                          const real *corr, cudaStream_t s)
{
    (void)owned_lo;
    const int64_t ncells = owned_n[0] * owned_n[1] * nz_chunk;
    if (ncells <= 0) return cudaSuccess;
    int64_t nb = (ncells + 255) / 256;
    if (nb > 8192) nb = 8192;
    export_kernel<real><<<(unsigned)nb, 256, 0, s>>>(grid, flags, z0, ncells, owned_n[0], owned_n[1], brick[0],
                                                    brick[1], brick[2], g, mode, canon, rho, u, rep, corr);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- seeded noise (input generator)
// Same counter-based generator as paper_1007_1388_b200/inputs.py (not part of
// the method): k = splitmix64(global_index * 19 + q + seed * golden) % 2049 - 1024.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename real>
__global__ void noise_kernel(real *grid, uint64_t seed, int64_t NX, int64_t NY, int64_t lox, int64_t loy,
                             int64_t loz, int64_t nx, int64_t ny, int64_t ncells, int b0, int b1, int b2,
                             const Geom g, const int rep)
{
    const int brick[3] = {b0, b1, b2};
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ox = c % nx;
        const int64_t r = c / nx;
        const int64_t oy = r % ny;
        const int64_t oz = r / ny;
        int lp, lx, ly, lz;
        owned_to_patch(g, brick, ox, oy, oz, lp, lx, ly, lz);
        const uint64_t gi = (uint64_t)(((loz + oz) * NY + (loy + oy)) * NX + (lox + ox));
        real *gp = grid + (int64_t)lp * g.ps + cell_index(g, lx, ly, lz);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t key = gi * 19ull + (uint64_t)q + seed * 0x9E3779B97F4A7C15ull;
            const int64_t k = (int64_t)(splitmix64(key) % 2049ull) - 1024;
            gp[rep_slot(rep, q) * g.qs] = (real)((double)k * (1.0 / 1048576.0));
        }
    }
}

template <typename real>
cudaError_t launch_noise(real *grid, uint64_t seed, const int64_t domain[3], const int64_t owned_lo[3],
                         const int64_t owned_n[3], const int brick[3], const Geom &g, int rep, cudaStream_t s)
{
    const int64_t ncells = owned_n[0] * owned_n[1] * owned_n[2];
    int64_t nb = (ncells + 255) / 256;
    if (nb > 16384) nb = 16384;
    noise_kernel<real><<<(unsigned)nb, 256, 0, s>>>(grid, seed, domain[0], domain[1], owned_lo[0], owned_lo[1],
                                                   owned_lo[2], owned_n[0], owned_n[1], ncells, brick[0], brick[1],
                                                   brick[2], g, rep);
    return cudaGetLastError();
}

template <typename real>
__global__ void gather_kernel(const real *grid, const uint8_t *flags, const int64_t *xyz, int64_t n, int b0,
                              int b1, int b2, const Geom g, double *out, const int rep, const real *corr)
{
    const int brick[3] = {b0, b1, b2};
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        int lp, lx, ly, lz;
        owned_to_patch(g, brick, xyz[3 * c], xyz[3 * c + 1], xyz[3 * c + 2], lp, lx, ly, lz);
        const int64_t ci = cell_index(g, lx, ly, lz);
        const uint8_t *fp = flags + (int64_t)lp * g.fs + ci;
        const bool fluid = fp[0] == 0;
        const real *gp = grid + (int64_t)lp * g.ps + ci;
        for (int q = 0; q < Q; ++q) out[c * Q + q] = fluid ? read_state(gp, fp, corr, g, rep, q) : 0.0;
    }
}

template <typename real>
cudaError_t launch_gather(const real *grid, const uint8_t *flags, const int64_t *xyz_local, int64_t n,
                          const int brick[3], const Geom &g, double *out, int rep, const real *corr, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    int64_t nb = (n + 127) / 128;
    if (nb > 4096) nb = 4096;
    gather_kernel<real><<<(unsigned)nb, 128, 0, s>>>(grid, flags, xyz_local, n, brick[0], brick[1], brick[2], g, out,
                                                     rep, corr);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- bounce-back fill
// Writes, for the current state, the store-side bounce-back values of every
// wall-adjacent fluid cell x into its wall neighbours: grid_opp(j)(x + e_j) =
// grid_j(x) + corr.  Needed once after the state or the flags are set; every
// later step maintains them inside the sweep.
// aa = 0: two-grid state (wall slot opp(j) <- S_j(x)); aa = 1: AA swapped
// state (S_j(x) = A[x][opp(j)], wall slot j, as the LOCAL kernel writes it).
template <typename real>
__global__ void bb_fill_kernel(real *grid, const uint8_t *flags, const uint8_t *kind, const real *corr,
                               const Geom g, const int aa)
{
    const int lp = blockIdx.y;
    real *gp = grid + (int64_t)lp * g.ps;
    const uint8_t *fp = flags + (int64_t)lp * g.fs;
    const uint8_t *kp = kind + (int64_t)lp * g.fs;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < g.fs; e += (int64_t)gridDim.x * blockDim.x) {
        if (kp[e] != 1) continue;
        for (int j = 1; j < Q; ++j) {
            const int64_t sh = EX(j) + EY(j) * (int64_t)g.px + EZ(j) * g.plane;
            const uint8_t f = fp[e + sh];
            if (f == 0) continue;
            real v = gp[(aa ? OPP(j) : j) * g.qs + e];
            if (f >= 2) v += corr[(f - 2) * Q + OPP(j)];
            gp[(aa ? j : OPP(j)) * g.qs + e + sh] = v;
        }
    }
}

template <typename real>
cudaError_t launch_bb_fill(real *grid, const uint8_t *flags, const uint8_t *kind, const real *corr, int nlocal,
                           const Geom &g, int aa, cudaStream_t s)
{
    int64_t bx = (g.fs + 255) / 256;
    if (bx > 2048) bx = 2048;
    for (int off = 0; off < nlocal; off += 65535) {
        int n = nlocal - off < 65535 ? nlocal - off : 65535;
        dim3 grid_dim((unsigned)bx, (unsigned)n);
        bb_fill_kernel<real><<<grid_dim, 256, 0, s>>>(grid + (int64_t)off * g.ps, flags + (int64_t)off * g.fs,
                                                      kind + (int64_t)off * g.fs, corr, g, aa);
    }
    return cudaGetLastError();
}

#define LBM_INSTANTIATE(real)                                                                                   \
    template cudaError_t launch_sweep<real>(const SweepArgs<real> &, int64_t, int, cudaStream_t);               \
    template cudaError_t launch_sweep_aa<real>(const SweepArgs<real> &, int64_t, bool, int, cudaStream_t);      \
    template cudaError_t launch_copy_segments<real>(const CopySeg *, int, int64_t, const real *, real *,        \
                                                    const real *, real *, const uint8_t *, const Geom &,       \
                                                    cudaStream_t);                                             \
    template cudaError_t launch_bb_fill<real>(real *, const uint8_t *, const uint8_t *, const real *, int,      \
                                              const Geom &, int, cudaStream_t);                                \
    template cudaError_t launch_import<real>(const double *, int64_t, int64_t, const int64_t *, const int64_t *, \
                                             const int *, const Geom &, real *, int, cudaStream_t);            \
    template cudaError_t launch_export<real>(const real *, const uint8_t *, int64_t, int64_t, const int64_t *,  \
                                             const int64_t *, const int *, const Geom &, double *, int,        \
                                             double *, double *, int, const real *, cudaStream_t);             \
    template cudaError_t launch_noise<real>(real *, uint64_t, const int64_t *, const int64_t *, const int64_t *, \
                                            const int *, const Geom &, int, cudaStream_t);                     \
    template cudaError_t launch_gather<real>(const real *, const uint8_t *, const int64_t *, int64_t,            \
                                             const int *, const Geom &, double *, int, const real *,           \
                                             cudaStream_t);

LBM_INSTANTIATE(float)
LBM_INSTANTIATE(double)

}  // namespace lbm
