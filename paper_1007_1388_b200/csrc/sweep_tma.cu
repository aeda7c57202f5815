// sweep_tma.cu -- TMA-staged, warp-specialised persistent sweep (sm_100a).
//
// Same update as sweep_kernel (sweep.cu): branch-free pull +
// BGK collide (eq:lbm / eq:feq) on centred PDFs, with
// half-way bounce-back applied on the store side (see sweep.cu).
// What differs is how the pull neighbourhood reaches the SM: the pull of
// direction i for a tile of TX x TY cells of one z-plane is the TX x TY box of
// q-slice i shifted by -e_i, so a producer warp issues 19
// cp.async.bulk.tensor loads (one 4-D tensor map over [19 * patches][z][y][x])
// plus one for the tile's cell kinds and one for its 3-plane flag
// neighbourhood, into a STAGES-deep shared-memory ring guarded by mbarriers.
// The bytes in flight per SM are then bounded by shared memory (~215 KB)
// instead of by the register file, which is what limits the SIMT sweep.
// Consumer warps read their 19 values with conflict-free LDS, release the
// stage, collide and store with coalesced STG.
//
// Measured on this B200 (tools/tma_probe.cu): a tiled TMA load whose innermost
// start offset is not 16-B aligned raises cudaErrorIllegalInstruction, and the
// bulk engine reads DRAM in 64-B chunks.  So the 9 directions with e_ix = 0 load
// exactly the tile's aligned rows (box TX wide), and the 10 with e_ix = +-1 load
// one 64-B chunk more (box TX + C wide, C = 64 B / sizeof(real)): from x0 - C
// for e_ix = +1 (pull from x - 1), from x0 for e_ix = -1 (pull from x + 1).
// That is exactly the chunks a SIMT warp touches; one box of TX + 2A with A =
// 16 B for all 19 directions read +25 % (profiles/r01_ncu_sweep_tma*).  Every
// tile starts at a multiple of 16 cells in x.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "collide.cuh"
#include "kernels.cuh"

namespace lbm {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

constexpr int align128(int b) { return (b + 127) / 128 * 128; }

}  // namespace

template <typename real, int TX, int TY, int STAGES, int CPS>
struct TmaCfg {
    static constexpr int TT = TX * TY;                       // cells per tile = consumer threads
    static constexpr int THREADS = TT + 32;                  // + producer warp
    static constexpr int C = 64 / (int)sizeof(real);         // one 64-B chunk (elements)
    static constexpr int BWS = TX + C;                       // box width of the e_x != 0 directions
    static constexpr int BOX_BYTES = align128(BWS * TY * (int)sizeof(real));  // 128-B aligned slots
    static constexpr int BOX_STRIDE = BOX_BYTES / (int)sizeof(real);
    static constexpr int FW = TX + 32;                       // flag box width (bytes, 16-B halo each side)
    static constexpr int FPLANE = FW * (TY + 2);
    static constexpr int KIND_OFF = Q * BOX_BYTES;
    static constexpr int FLAG_OFF = KIND_OFF + align128(TT);
    static constexpr int STAGE_STRIDE = FLAG_OFF + align128(3 * FPLANE);
    static constexpr int TX_BYTES = (9 * TX + 10 * BWS) * TY * (int)sizeof(real) + TT + 3 * FPLANE;  // per stage
    static constexpr int BAR_OFF = STAGES * STAGE_STRIDE;
    static constexpr int SMEM = BAR_OFF + STAGES * (16 + 32);
    static_assert(TX % 16 == 0 && TX % C == 0, "tile x must keep 64-B aligned TMA starts");
    static_assert(SMEM <= 232448 / CPS - 1024, "shared memory budget");
};

// Tile metadata written by the producer for each stage.
struct TileMeta {
    int patch, x0, y0, z;
    int xend, yend, pad0, pad1;
};

template <typename real, int TX, int TY, int STAGES, int CPS>
__global__ void __launch_bounds__(TmaCfg<real, TX, TY, STAGES, CPS>::THREADS, CPS)
    sweep_tma_kernel(const __grid_constant__ CUtensorMap tm_pdf, const __grid_constant__ CUtensorMap tm_pdfs,
                     const __grid_constant__ CUtensorMap tm_kind, const __grid_constant__ CUtensorMap tm_flags,
                     const SweepArgs<real> a, const int64_t total_tiles)
{
    using C = TmaCfg<real, TX, TY, STAGES, CPS>;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full = (uint64_t *)(smem + C::BAR_OFF);
    uint64_t *empty = full + STAGES;
    TileMeta *meta = (TileMeta *)(empty + STAGES);

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::TT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    const Geom &g = a.g;
    if (tid < 32) {
        // ---------------- producer warp (one lane issues all TMA traffic)
        if (tid == 0) {
            prefetch_tmap(&tm_pdf);
            prefetch_tmap(&tm_pdfs);
            prefetch_tmap(&tm_kind);
            prefetch_tmap(&tm_flags);
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x;; t += gridDim.x) {
                mbar_wait(&empty[stage], phase ^ 1);
                TileMeta m;
                if (t >= total_tiles) {
                    m.patch = -1;
                    meta[stage] = m;
                    mbar_arrive(&full[stage]);  // sentinel: no bytes expected
                    break;
                }
                int lo = 0, hi = a.nboxes;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (a.tile_prefix[mid] <= t) lo = mid; else hi = mid;
                }
                const Box bx = a.boxes[lo];
                int r = (int)(t - a.tile_prefix[lo]);
                const int tx = r % bx.tiles_x;
                r /= bx.tiles_x;
                const int ty = r % bx.tiles_y;
                const int tz = r / bx.tiles_y;
                m.patch = bx.patch;
                m.x0 = bx.lo[0] + tx * TX;
                m.y0 = bx.lo[1] + ty * TY;
                m.z = bx.lo[2] + tz;
                m.xend = bx.lo[0] + bx.n[0];
                m.yend = bx.lo[1] + bx.n[1];
                meta[stage] = m;
                unsigned char *sb = smem + stage * C::STAGE_STRIDE;
                mbar_arrive_expect_tx(&full[stage], (uint32_t)C::TX_BYTES);
                // Pull boxes of q-slice i, rows y0 - ey, plane z - ez (padded coordinates:
                // interior x = 0 is column xo, y = 0 row 1, z = 0 plane 1).
                const int cx = m.x0 + g.xo, cy = m.y0 + 1, cz = m.z + 1, cq = m.patch * Q;
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    if (EX(i) == 0)
                        tma_load_4d(sb + i * C::BOX_BYTES, &tm_pdf, cx, cy - EY(i), cz - EZ(i), cq + i, &full[stage]);
                    else
                        tma_load_4d(sb + i * C::BOX_BYTES, &tm_pdfs, EX(i) > 0 ? cx - C::C : cx, cy - EY(i),
                                    cz - EZ(i), cq + i, &full[stage]);
                }
                tma_load_4d(sb + C::KIND_OFF, &tm_kind, cx, cy, cz, m.patch, &full[stage]);
                tma_load_4d(sb + C::FLAG_OFF, &tm_flags, cx - 16, cy - 1, cz - 1, m.patch, &full[stage]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // ---------------- consumer warps: one cell per thread
    const int c = tid - 32;
    const int cxl = c % TX, cyl = c / TX;
    const real omega = a.omega;
    const int64_t qs = g.qs;
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
        mbar_wait(&full[stage], phase);
        const TileMeta m = meta[stage];
        if (m.patch < 0) break;
        const int sbase = stage * C::STAGE_STRIDE;
        const real *box = reinterpret_cast<const real *>(smem + sbase);
        real p[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i)
            p[i] = EX(i) == 0 ? box[i * C::BOX_STRIDE + cyl * TX + cxl]
                              : box[i * C::BOX_STRIDE + cyl * C::BWS + cxl + (EX(i) > 0 ? C::C - 1 : 1)];
        const uint8_t k = smem[sbase + C::KIND_OFF + c];
        uint8_t nbf[Q];
        if (k == 1) {
            // flags of x + e_j from the tile's 3-plane flag neighbourhood
            const unsigned char *fb = smem + sbase + C::FLAG_OFF;
#pragma unroll
            for (int j = 1; j < Q; ++j)
                nbf[j] = fb[(1 + EZ(j)) * C::FPLANE + (cyl + 1 + EY(j)) * C::FW + cxl + 16 + EX(j)];
        }
        mbar_arrive(&empty[stage]);  // release: the LDS above are performed before the stage is reused
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }
        const int x = m.x0 + cxl, y = m.y0 + cyl;
        if (x >= m.xend || y >= m.yend || k == 2) continue;  // outside the box or non-fluid (R13)
        collide_bgk<real>(p, omega);
        const int64_t cell = ((int64_t)(m.z + 1) * g.py + (y + 1)) * (int64_t)g.px + (x + g.xo);
        real *d = a.dst + (int64_t)m.patch * g.ps + cell;
#pragma unroll
        for (int i = 0; i < Q; ++i) d[i * qs] = p[i];
        if (k == 1) {
            // Store-side half-way bounce-back (R3): park f_j(x) (+ moving-wall
            // term of the delivered direction opp(j)) in slot opp(j) of the wall x + e_j.
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
}

// ------------------------------------------------------------------ host side
// Shape variants (tile x, tile y, stages) per precision; index = LBM_TMA_SHAPE.
template <typename real, int V>
struct TmaShape;
template <>
struct TmaShape<double, 0> { static constexpr int TX = 64, TY = 4, ST = 5, CPS = 1; };
template <>
struct TmaShape<double, 1> { static constexpr int TX = 128, TY = 2, ST = 5, CPS = 1; };
template <>
struct TmaShape<double, 2> { static constexpr int TX = 64, TY = 4, ST = 2, CPS = 2; };
template <>
struct TmaShape<float, 0> { static constexpr int TX = 128, TY = 2, ST = 9, CPS = 1; };
template <>
struct TmaShape<float, 1> { static constexpr int TX = 128, TY = 2, ST = 4, CPS = 2; };
template <>
struct TmaShape<float, 2> { static constexpr int TX = 64, TY = 4, ST = 4, CPS = 2; };

template <typename real>
void tma_tile_shape(int variant, int *tx, int *ty)
{
    switch (variant) {
    case 1: *tx = TmaShape<real, 1>::TX; *ty = TmaShape<real, 1>::TY; break;
    case 2: *tx = TmaShape<real, 2>::TX; *ty = TmaShape<real, 2>::TY; break;
    default: *tx = TmaShape<real, 0>::TX; *ty = TmaShape<real, 0>::TY; break;
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

static cudaError_t encode4(CUtensorMap *map, CUtensorMapDataType dt, int esize, const void *base, const Geom &g,
                           cuuint64_t d3, cuuint32_t b0, cuuint32_t b1, cuuint32_t b2)
{
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[4] = {(cuuint64_t)g.px, (cuuint64_t)g.py, (cuuint64_t)(g.n[2] + 2), d3};
    cuuint64_t strides[3] = {(cuuint64_t)g.px * esize, (cuuint64_t)g.plane * esize, (cuuint64_t)g.qs * esize};
    cuuint32_t box[4] = {b0, b1, b2, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    // L2 promotion: none by default (256-B promotion of the short box rows
    // raised DRAM reads by 25 %, profiles/r01_ncu_sweep_tma*); env LBM_TMA_PROMO=0..3.
    static int promo = -1;
    if (promo < 0) {
        const char *e = std::getenv("LBM_TMA_PROMO");
        promo = e ? std::atoi(e) : 0;
        if (promo < 0 || promo > 3) promo = 0;
    }
    const CUtensorMapL2promotion pr[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    CUresult r = enc(map, dt, 4, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, pr[promo], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Maps: PDFs [19 * nlocal][nz + 2][py][px] (boxes TX x TY and (TX + C) x TY,
// C = 64 B / sizeof(real)), kinds and flags [nlocal][nz + 2][py][px] bytes
// (boxes TX x TY and (TX + 32) x (TY + 2) x 3).
template <typename real>
cudaError_t make_tma_maps(const void *grid, const uint8_t *kind, const uint8_t *flags, int nlocal, const Geom &g,
                          int variant, CUtensorMap *pdf_map, CUtensorMap *pdfs_map, CUtensorMap *kind_map,
                          CUtensorMap *flag_map)
{
    int TX, TY;
    tma_tile_shape<real>(variant, &TX, &TY);
    const int Cw = 64 / (int)sizeof(real);
    const CUtensorMapDataType dt = sizeof(real) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cudaError_t e = encode4(pdf_map, dt, (int)sizeof(real), grid, g, (cuuint64_t)Q * nlocal, TX, TY, 1);
    if (e != cudaSuccess) return e;
    e = encode4(pdfs_map, dt, (int)sizeof(real), grid, g, (cuuint64_t)Q * nlocal, TX + Cw, TY, 1);
    if (e != cudaSuccess) return e;
    if (kind_map) {
        e = encode4(kind_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, kind, g, nlocal, TX, TY, 1);
        if (e != cudaSuccess) return e;
    }
    if (flag_map) e = encode4(flag_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, flags, g, nlocal, TX + 32, TY + 2, 3);
    return e;
}

template <typename real, int V>
static cudaError_t launch_v(const CUtensorMap &pm, const CUtensorMap &psm, const CUtensorMap &km,
                            const CUtensorMap &fm, const SweepArgs<real> &a, int64_t total_tiles, int num_sms,
                            cudaStream_t s)
{
    constexpr int TX = TmaShape<real, V>::TX, TY = TmaShape<real, V>::TY, ST = TmaShape<real, V>::ST;
    constexpr int CPS = TmaShape<real, V>::CPS;
    using C = TmaCfg<real, TX, TY, ST, CPS>;
    // per launch (cheap, and correct for whichever device is current)
    cudaError_t e = cudaFuncSetAttribute(sweep_tma_kernel<real, TX, TY, ST, CPS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)num_sms * CPS;
    if (grid > total_tiles) grid = total_tiles;
    sweep_tma_kernel<real, TX, TY, ST, CPS><<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(pm, psm, km, fm, a,
                                                                                       total_tiles);
    return cudaGetLastError();
}

template <typename real>
cudaError_t launch_sweep_tma(const CUtensorMap &pdf_map, const CUtensorMap &pdfs_map, const CUtensorMap &kind_map,
                             const CUtensorMap &flag_map, const SweepArgs<real> &a, int64_t total_tiles, int num_sms,
                             int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    switch (variant) {
    case 1: return launch_v<real, 1>(pdf_map, pdfs_map, kind_map, flag_map, a, total_tiles, num_sms, s);
    case 2: return launch_v<real, 2>(pdf_map, pdfs_map, kind_map, flag_map, a, total_tiles, num_sms, s);
    default: return launch_v<real, 0>(pdf_map, pdfs_map, kind_map, flag_map, a, total_tiles, num_sms, s);
    }
}

template void tma_tile_shape<float>(int, int *, int *);
template void tma_tile_shape<double>(int, int *, int *);
template cudaError_t make_tma_maps<float>(const void *, const uint8_t *, const uint8_t *, int, const Geom &, int,
                                          CUtensorMap *, CUtensorMap *, CUtensorMap *, CUtensorMap *);
template cudaError_t make_tma_maps<double>(const void *, const uint8_t *, const uint8_t *, int, const Geom &, int,
                                           CUtensorMap *, CUtensorMap *, CUtensorMap *, CUtensorMap *);
template cudaError_t launch_sweep_tma<float>(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                                             const CUtensorMap &, const SweepArgs<float> &, int64_t, int, int,
                                             cudaStream_t);
template cudaError_t launch_sweep_tma<double>(const CUtensorMap &, const CUtensorMap &, const CUtensorMap &,
                                              const CUtensorMap &, const SweepArgs<double> &, int64_t, int, int,
                                              cudaStream_t);

}  // namespace lbm
