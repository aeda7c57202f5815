// aux_kernels.cu -- the non-sweep kernels: ghost-exchange copies (pack /
// local copy / unpack), flags and cell kinds, canonical import /
// export and macroscopic moments, the seeded noise initialiser, the
// sampled gather and the store-side bounce-back fill.
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "sweep_common.cuh"

namespace lbm {

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
            v = grid_src[sg.src_base + pdf_index(g, q, sg.src_lo[0] + cx, sg.src_lo[1] + cy, sg.src_lo[2] + cz)];
        if (sg.dst_is_buf) {
            buf_dst[sg.dst_base + e] = v;
        } else {
            const int y[3] = {sg.dst_lo[0] + cx, sg.dst_lo[1] + cy, sg.dst_lo[2] + cz};
            bool ok = sg.mask == 1 || flags[sg.dst_flag_base + flag_index(g, y[0], y[1], y[2])] == 0;  // mask 1: all destinations fluid
            if (sg.mask == 2 && ok) {
                // AA half-exchange 2: the value was scattered by the sender's cell
                // w = y - e_q; only entries whose writer is a fluid cell of the sender
                // (not another patch's ghost) are delivered.
                const int w[3] = {y[0] - EX(q), y[1] - EY(q), y[2] - EZ(q)};
                for (int a2 = 0; a2 < 3; ++a2)
                    if (sg.d[a2] == 0 && (w[a2] < 0 || w[a2] >= g.n[a2])) ok = false;
                if (ok) ok = flags[sg.dst_flag_base + flag_index(g, w[0], w[1], w[2])] == 0;
            }
            if (ok) grid_dst[sg.dst_base + pdf_index(g, q, y[0], y[1], y[2])] = v;
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
        const int col = (int)(e % g.fpx);
        const int64_t r = e / g.fpx;
        const int row = (int)(r % g.py);
        const int pl = (int)(r / g.py);
        const int lc[3] = {col - g.fxo, row - 1, pl - 1};
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
// fluid neighbours (pure pull).  wmask (kind-1 cells): bit j set if x + e_j is
// non-fluid -- one 32-bit word instead of 18 flag bytes for the sweep's
// store-side bounce-back.
__global__ void build_kind_kernel(const Geom g, const uint8_t *flags, uint8_t *kind, uint32_t *wmask)
{
    const int lp = blockIdx.y;
    const int64_t total = g.fs;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int col = (int)(e % g.fpx);
        const int64_t r = e / g.fpx;
        const int row = (int)(r % g.py);
        const int pl = (int)(r / g.py);
        const int x = col - g.fxo, y = row - 1, z = pl - 1;
        const uint8_t *f = flags + (int64_t)lp * g.fs;
        uint8_t kd = 2;
        uint32_t m = 0;
        if (x >= 0 && x < g.n[0] && y >= 0 && y < g.n[1] && z >= 0 && z < g.n[2] && f[e] == 0) {
            for (int j = 1; j < Q; ++j)
                if (f[e + flag_shift(g, j)] != 0) m |= 1u << j;
            kd = m ? 1 : 0;
        }
        kind[(int64_t)lp * g.fs + e] = kd;
        wmask[(int64_t)lp * g.fs + e] = m;
    }
}

cudaError_t launch_build_flags(const uint8_t *global, const int64_t domain[3], const int periodic[3],
                               const int *patch_origin, int nlocal, const Geom &g, uint8_t *flags,
                               uint8_t *kind, uint32_t *wmask, cudaStream_t s)
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
        build_kind_kernel<<<grid, 256, 0, s>>>(g, flags + (int64_t)off * g.fs, kind + (int64_t)off * g.fs,
                                               wmask + (int64_t)off * g.fs);
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

// PDF i of the state at cell (x, y, z) of a patch (gp: patch base, fp: the
// cell's flag byte)
template <typename real>
__device__ __forceinline__ double read_state(const real *gp, const uint8_t *fp, const real *corr, const Geom &g,
                                             int rep, int i, int x, int y, int z)
{
    if (rep != 2) return (double)gp[pdf_index(g, rep_slot(rep, i), x, y, z)];
    const uint8_t f = fp[flag_shift(g, i)];
    if (i == 0 || f == 0) return (double)gp[pdf_index(g, i, x + EX(i), y + EY(i), z + EZ(i))];
    real v = gp[pdf_index(g, OPP(i), x, y, z)];
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
        real *gp = grid + (int64_t)lp * g.ps;
#pragma unroll
        for (int q = 0; q < Q; ++q) gp[pdf_index(g, rep_slot(rep, q), lx, ly, lz)] = (real)canon[c * Q + q];
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
        const uint8_t *fp = flags + (int64_t)lp * g.fs + flag_index(g, lx, ly, lz);
        const bool fluid = fp[0] == 0;
        const real *gp = grid + (int64_t)lp * g.ps;
        if (mode == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) canon[c * Q + q] = fluid ? read_state(gp, fp, corr, g, rep, q, lx, ly, lz) : 0.0;
        } else {
            // Macroscopic export: rho = rho0 + sum f~, u = sum e f~ / rho0.
            double s = 0, jx = 0, jy = 0, jz = 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const double v = fluid ? read_state(gp, fp, corr, g, rep, q, lx, ly, lz) : 0.0;
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

// ---------------------------------------------------------------- total mass
// sum of delta rho = sum_i f~_i over the owned fluid cells in fp64,
// deterministic: a fixed grid of kMassBlocks blocks, each thread summing its cells
// in order, a tree per block into partial[b], then one block summing the
// partials in order (lbm_total_mass; off the hot path).
template <typename real>
__global__ void __launch_bounds__(kMassThreads) mass_kernel(const real *grid, const uint8_t *flags, int64_t ncells,
                                                            int64_t nx, int64_t ny, int b0, int b1, int b2,
                                                            const Geom g, const int rep, const real *corr,
                                                            double *partial)
{
    const int brick[3] = {b0, b1, b2};
    double s = 0.0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ox = c % nx;
        const int64_t r = c / nx;
        const int64_t oy = r % ny;
        const int64_t oz = r / ny;
        int lp, lx, ly, lz;
        owned_to_patch(g, brick, ox, oy, oz, lp, lx, ly, lz);
        const uint8_t *fp = flags + (int64_t)lp * g.fs + flag_index(g, lx, ly, lz);
        if (fp[0] != 0) continue;
        const real *gp = grid + (int64_t)lp * g.ps;
        double cs = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) cs += read_state(gp, fp, corr, g, rep, q, lx, ly, lz);
        s += cs;
    }
    __shared__ double sh[kMassThreads];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kMassThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(kMassThreads) mass_finish_kernel(const double *partial, double *out)
{
    __shared__ double sh[kMassThreads];
    double s = 0.0;
    for (int b = threadIdx.x; b < kMassBlocks; b += kMassThreads) s += partial[b];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = kMassThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

template <typename real>
cudaError_t launch_mass(const real *grid, const uint8_t *flags, const int64_t owned_lo[3], const int64_t on[3],
                        const int brick[3], const Geom &g, int rep, const real *corr, double *partial, double *out,
                        cudaStream_t s)
{
    (void)owned_lo;
    const int64_t ncells = on[0] * on[1] * on[2];
    mass_kernel<real><<<kMassBlocks, kMassThreads, 0, s>>>(grid, flags, ncells, on[0], on[1], brick[0], brick[1],
                                                          brick[2], g, rep, corr, partial);
    mass_finish_kernel<<<1, kMassThreads, 0, s>>>(partial, out);
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
        real *gp = grid + (int64_t)lp * g.ps;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t key = gi * 19ull + (uint64_t)q + seed * 0x9E3779B97F4A7C15ull;
            const int64_t k = (int64_t)(splitmix64(key) % 2049ull) - 1024;
            gp[pdf_index(g, rep_slot(rep, q), lx, ly, lz)] = (real)((double)k * (1.0 / 1048576.0));
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
        const uint8_t *fp = flags + (int64_t)lp * g.fs + flag_index(g, lx, ly, lz);
        const bool fluid = fp[0] == 0;
        const real *gp = grid + (int64_t)lp * g.ps;
        for (int q = 0; q < Q; ++q) out[c * Q + q] = fluid ? read_state(gp, fp, corr, g, rep, q, lx, ly, lz) : 0.0;
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
// Half-way bounce-back (R3) as a list kernel over the wall-adjacent
// fluid cells x (the bounce-back list, bb_list_build_kernel) and their wall
// links w = x + e_j, with corr = 6 w rho0 e_opp(j).u_w of w's velocity:
//   mode 0 (two grids, after every sweep and once after set_pdfs / set_flags):
//          grid_opp(j)(w) = grid_j(x) + corr -- store side, so that the next
//          step's pull of x from w is branch-free;
//   mode 1 (AA, after LOCAL and once after set_pdfs / set_flags, swapped state
//          S_j(x) = A[x][opp(j)]): A[w][j] = A[x][opp(j)] + corr;
//   mode 2 (AA, after PULL, whose straight scatter put out_j(x) into the wall
//          slot A[w][j]): A[x][opp(j)] = A[w][j] + corr -- the PULL bounce-back.
// The sweeps themselves carry no wall logic.  Each target slot has exactly one
// writer (x = w - e_j), so entries are independent.
template <typename real, int mode>
__global__ void __launch_bounds__(256) bb_list_kernel(real *grid, const uint8_t *flags, const BbEntry *list, int64_t n,
                                                      const real *corr, const Geom g, const BbOffsets o,
                                                      const Checker ck)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const BbEntry en = list[t];
        const int lp = (int)(en.pos >> 45);
        const int z = (int)((en.pos >> 30) & 0x7fff), y = (int)((en.pos >> 15) & 0x7fff), x = (int)(en.pos & 0x7fff);
        real *gp = grid + (int64_t)lp * g.ps;
        real *C = gp + main_index(g, x, y, z);
        real *G = ghost_base(g, gp, y, z);
        const bool xlo = x == 0, xhi = x == g.n[0] - 1;
        const uint32_t vel = en.vinfo >> 24;
        // all link values first, then the stores: no slot is both read and
        // written by this kernel (reads: fluid slots in modes 0 / 1, wall slots in
        // mode 2; writes: the other kind), so the loads are independent,
        // non-coherent and in flight together instead of one memory latency per link
        real v[Q];
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            if (!((en.mask >> j) & 1u)) continue;
            const bool cross = (EX(j) < 0 && xlo) || (EX(j) > 0 && xhi);  // w is an x ghost
            const real *src = mode == 2 ? (cross ? at<real>(G, o.wg[j]) : at<real>(C, o.wm[j])) : at<real>(C, o.xs[j]);
            v[j] = gld(ck, src);
            if ((en.vinfo >> j) & 1u) {  // moving wall: its velocity is shared (vel) or read from its flag
                const int k = vel != kBbMixed
                                  ? (int)vel
                                  : __ldg(flags + (int64_t)lp * g.fs + flag_index(g, x + EX(j), y + EY(j), z + EZ(j))) - 2;
                v[j] += __ldg(corr + k * Q + OPP(j));
            }
        }
#pragma unroll
        for (int j = 1; j < Q; ++j) {
            if (!((en.mask >> j) & 1u)) continue;
            const bool cross = (EX(j) < 0 && xlo) || (EX(j) > 0 && xhi);
            real *dst = mode == 2 ? at<real>(C, o.xs[j]) : (cross ? at<real>(G, o.wg[j]) : at<real>(C, o.wm[j]));
            gst(ck, dst, v[j]);
#ifdef LBM_CHECKED
            if (ck.inject) gst(ck, dst, v[j]);
#endif
        }
    }
}

template <typename real>
cudaError_t launch_bb_list(real *grid, const uint8_t *flags, const BbEntry *list, int64_t n, const real *corr,
                           const Geom &g, int mode, const BbOffsets &o, const Checker &ck, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (mode == 2) bb_list_kernel<real, 2><<<(unsigned)blocks, 256, 0, s>>>(grid, flags, list, n, corr, g, o, ck);
    else if (mode == 1) bb_list_kernel<real, 1><<<(unsigned)blocks, 256, 0, s>>>(grid, flags, list, n, corr, g, o, ck);
    else bb_list_kernel<real, 0><<<(unsigned)blocks, 256, 0, s>>>(grid, flags, list, n, corr, g, o, ck);
    return cudaGetLastError();
}

// The bounce-back list: the kind-1 cells of every local patch in ascending
// flag-layout order (deterministic), each with its wall mask and which of its
// walls move (and their shared velocity), so the list kernel reads one 16-B
// entry per cell instead of a mask word and up to 18 flag bytes.  Pass 0
// counts per chunk, the host scans the counts, pass 1 writes each chunk's
// entries at its offset in order.
constexpr int kBbChunk = 256 * 8;
// The wall mask of list entry i (0: not an entry): kind-1 cells, minus the links
// of the inner face cells of uniform-wall sides, which the two-grid sweep stores
// itself (sidewall_kernel).
__device__ __forceinline__ uint32_t bb_entry_mask(const uint8_t *kind, const uint32_t *wmask,
                                                  const unsigned long long *sidewall, const Geom &g, int64_t i)
{
    if (kind[i] != 1) return 0u;
    uint32_t m = wmask[i];
    if (sidewall) {
        const int64_t lp = i / g.fs, e = i - lp * g.fs;
        const int64_t r = e / g.fpx;
        const int p[3] = {(int)(e % g.fpx) - g.fxo, (int)(r % g.py) - 1, (int)(r / g.py) - 1};
        const unsigned long long sw = sidewall[lp];
        constexpr unsigned lo_bits[3] = {kXM, kYM, kZM}, hi_bits[3] = {kXP, kYP, kZP};
        for (int a = 0; a < 3; ++a) {
            const int b = (a + 1) % 3, c = (a + 2) % 3;
            const bool inner = p[b] >= 1 && p[b] <= g.n[b] - 2 && p[c] >= 1 && p[c] <= g.n[c] - 2;
            if (!inner) continue;
            if (((sw >> (2 * a)) & 1ull) && p[a] == 0) m &= ~lo_bits[a];
            if (((sw >> (2 * a + 1)) & 1ull) && p[a] == g.n[a] - 1) m &= ~hi_bits[a];
        }
    }
    return m;
}

__global__ void bb_list_build_kernel(const uint8_t *kind, const uint32_t *wmask, const uint8_t *flags,
                                     const unsigned long long *sidewall, int64_t total, const Geom g, int64_t *counts,
                                     BbEntry *list)
{
    __shared__ int warp_tot[8];
    const int64_t base = (int64_t)blockIdx.x * kBbChunk + (int64_t)threadIdx.x * 8;
    int mine = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) mine += (base + k < total && bb_entry_mask(kind, wmask, sidewall, g, base + k)) ? 1 : 0;
    // block-exclusive scan of the per-thread counts (thread order = index order)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int before = 0, tot = 0;
    for (int i = 0; i < 8; ++i) {
        if (i < w) before += warp_tot[i];
        tot += warp_tot[i];
    }
    if (!list) {
        if (threadIdx.x == 0) counts[blockIdx.x] = tot;
        return;
    }
    int64_t pos = counts[blockIdx.x] + before + incl - mine;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = base + k;
        const uint32_t m = i < total ? bb_entry_mask(kind, wmask, sidewall, g, i) : 0u;
        if (!m) continue;
        BbEntry en;
        const int64_t lp = i / g.fs, e = i - lp * g.fs;
        const int64_t r = e / g.fpx;
        en.pos = bb_pos((int)lp, (int)(e % g.fpx) - g.fxo, (int)(r % g.py) - 1, (int)(r / g.py) - 1);
        en.mask = m;
        uint32_t vm = 0, vel = kBbMixed + 1;  // kBbMixed + 1: no moving wall yet
        for (int j = 1; j < Q; ++j) {
            if (!((en.mask >> j) & 1u)) continue;
            const uint8_t f = flags[i + flag_shift(g, j)];
            if (f < 2) continue;
            vm |= 1u << j;
            const uint32_t kv = f - 2u;
            vel = vel == kBbMixed + 1 ? kv : (vel == kv ? vel : kBbMixed);
        }
        en.vinfo = vm | ((vel > kBbMixed ? 0u : vel) << 24);
        list[pos++] = en;
    }
}

cudaError_t launch_bb_list_count(const uint8_t *kind, const uint32_t *wmask, const unsigned long long *sidewall,
                                 int64_t total, const Geom &g, int64_t *counts, cudaStream_t s)
{
    const int64_t blocks = (total + kBbChunk - 1) / kBbChunk;
    if (blocks > 0)
        bb_list_build_kernel<<<(unsigned)blocks, 256, 0, s>>>(kind, wmask, nullptr, sidewall, total, g, counts, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_bb_list_write(const uint8_t *kind, const uint32_t *wmask, const uint8_t *flags,
                                 const unsigned long long *sidewall, int64_t total, const Geom &g,
                                 const int64_t *offsets, BbEntry *list, cudaStream_t s)
{
    const int64_t blocks = (total + kBbChunk - 1) / kBbChunk;
    if (blocks > 0)
        bb_list_build_kernel<<<(unsigned)blocks, 256, 0, s>>>(kind, wmask, flags, sidewall, total, g,
                                                              (int64_t *)offsets, list);
    return cudaGetLastError();
}

int64_t bb_list_chunks(int64_t total) { return (total + kBbChunk - 1) / kBbChunk; }

// Tile bits (sweep_common.cuh locate_pair): bit 31 of the patch field, the tile
// holds a non-fluid cell -- only those tiles read the cells' kinds; bits 30 / 29,
// the patch's -x / +x side is a uniform wall (sidewall) -- the two-grid sweep stores
// the x links' bounce-back of that face's inner cells from its row-end lanes --
// with the wall's flag in bits 16-23 / 24-31 of the z field.  One block per tile.
__global__ void tile_solid_kernel(int4 *tiles, int64_t n, const uint8_t *kind, const unsigned long long *sidewall,
                                  const Geom g)
{
    for (int64_t b = blockIdx.x; b < n; b += gridDim.x) {
        const int4 t = tiles[b];
        const int patch = t.x & 0x1fffffff, z = t.w & 0xffff;
        const int x0 = (int)((unsigned)t.y >> 16), xend = t.y & 0xffff;
        const int y0 = (int)((unsigned)t.z >> 16), yend = t.z & 0xffff;
        const int x = x0 + (int)(threadIdx.x % SWEEP_BX), y = y0 + (int)(threadIdx.x / SWEEP_BX);
        const bool solid = x < xend && y < yend && kind[(int64_t)patch * g.fs + flag_index(g, x, y, z)] == 2;
        const int any = __syncthreads_or(solid);
        if (threadIdx.x == 0) {
            const unsigned long long sw = sidewall ? sidewall[patch] : 0ull;
            tiles[b].x = patch | (any ? (int)0x80000000u : 0) | (int)((sw & 1u) << 30) | (int)((sw & 2u) << 28);
            tiles[b].w = z | side_flag(sw, 0) << 16 | side_flag(sw, 1) << 24;
        }
        __syncthreads();
    }
}

// Per local patch and side s = 2 a + (0 low, 1 high): is the ghost layer's part over
// the face (the other two coordinates in [0, n - 1]) one non-fluid flag?  The inner
// face cells (those coordinates in [1, n - 2]) link only there.  One block per
// (patch, side); sidewall zeroed before.
__global__ void sidewall_kernel(const uint8_t *flags, const Geom g, unsigned long long *sidewall)
{
    const int lp = blockIdx.x, side = blockIdx.y;
    const uint8_t *f = flags + (int64_t)lp * g.fs;
    const int a = side / 2, b = (a + 1) % 3, c = (a + 2) % 3;
    const int nb = g.n[b], nc = g.n[c];
    int p[3];
    p[a] = side % 2 ? g.n[a] : -1;
    p[b] = 0;
    p[c] = 0;
    const uint8_t f0 = f[flag_index(g, p[0], p[1], p[2])];
    int ok = f0 != 0 && nb >= 3 && nc >= 3;
    for (int k = threadIdx.x; k < nb * nc && ok; k += blockDim.x) {
        p[b] = k % nb;
        p[c] = k / nb;
        ok &= f[flag_index(g, p[0], p[1], p[2])] == f0;
    }
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0 && ok) atomicOr(sidewall + lp, 1ull << side | (unsigned long long)f0 << (8 + 8 * side));
}

cudaError_t launch_sidewall(const uint8_t *flags, int nlocal, const Geom &g, unsigned long long *sidewall,
                            cudaStream_t s)
{
    if (nlocal <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(sidewall, 0, (size_t)nlocal * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    sidewall_kernel<<<dim3((unsigned)nlocal, 6), 256, 0, s>>>(flags, g, sidewall);
    return cudaGetLastError();
}

cudaError_t launch_tile_solid(int4 *tiles, int64_t n, const uint8_t *kind, const unsigned long long *sidewall,
                              const Geom &g, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>(n, 148 * 64);
    tile_solid_kernel<<<(unsigned)blocks, SWEEP_BX * SWEEP_BY, 0, s>>>(tiles, n, kind, sidewall, g);
    return cudaGetLastError();
}

#define LBM_INSTANTIATE(real)                                                                                   \
    template cudaError_t launch_copy_segments<real>(const CopySeg *, int, int64_t, const real *, real *,        \
                                                    const real *, real *, const uint8_t *, const Geom &,       \
                                                    cudaStream_t);                                             \
    template cudaError_t launch_bb_list<real>(real *, const uint8_t *, const BbEntry *, int64_t, const real *,  \
                                              const Geom &, int, const BbOffsets &, const Checker &,           \
                                              cudaStream_t);                                                   \
    template cudaError_t launch_import<real>(const double *, int64_t, int64_t, const int64_t *, const int64_t *, \
                                             const int *, const Geom &, real *, int, cudaStream_t);            \
    template cudaError_t launch_export<real>(const real *, const uint8_t *, int64_t, int64_t, const int64_t *,  \
                                             const int64_t *, const int *, const Geom &, double *, int,        \
                                             double *, double *, int, const real *, cudaStream_t);             \
    template cudaError_t launch_noise<real>(real *, uint64_t, const int64_t *, const int64_t *, const int64_t *, \
                                            const int *, const Geom &, int, cudaStream_t);                     \
    template cudaError_t launch_mass<real>(const real *, const uint8_t *, const int64_t *, const int64_t *,       \
                                           const int *, const Geom &, int, const real *, double *, double *,   \
                                           cudaStream_t);                                                      \
    template cudaError_t launch_gather<real>(const real *, const uint8_t *, const int64_t *, int64_t,            \
                                             const int *, const Geom &, double *, int, const real *,           \
                                             cudaStream_t);

LBM_INSTANTIATE(float)
LBM_INSTANTIATE(double)

}  // namespace lbm
