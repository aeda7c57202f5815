// sweep_direct.cu -- the two-grid sweep fused with the ghost exchange (sm_100a).
//
// The paper extracts boundary PDFs into buffers after the kernel, moves them
// (cudaMemcpy + MPI) and inserts them into the neighbour's ghost layer before
// its next kernel.  Here the sweep does all three in one
// pass: a fluid cell x on a patch face (or edge) stores each outgoing PDF f_q(x)
// -- the 5 (face) or 1 (edge) directions whose e_q points into the neighbour --
// both into its own patch and straight into the neighbour patch's ghost layer
// of the next step's source grid on the other GPU: NVLink stores into its
// CUDA-IPC-mapped grid.  The fused kernel sweeps only the shells that face
// remote neighbours, on the high-priority stream, concurrently with the plain
// sweep of the interiors, so the transfer overlaps the compute.  There is no
// pack, no NCCL and no unpack on the hot path.
//
// Cross-GPU ordering (one handshake per step): after the sweep, a one-thread
// kernel fences at system scope, bumps this rank's epoch and publishes it with
// a system-scope release store into each peer's inbox.  The next step starts
// with wait_peers_kernel, which acquires until every peer's epoch has caught
// up -- i.e. the peers have finished reading the grid this rank is about to
// overwrite and have finished writing the ghosts it is about to read.  Bounded
// wait (120 s by default, LBM_PEER_TIMEOUT_S): it reports an error instead of
// hanging.  Only the shell
// sweeps touch ghost layers (read or remote write), so only they are ordered
// by the handshake; the interior sweep never waits for a peer.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "collide.cuh"
#include "kernels.cuh"

namespace lbm {

namespace {

__device__ __forceinline__ int64_t cidx(const Geom &g, int x, int y, int z)
{
    return ((int64_t)(z + 1) * g.py + (y + 1)) * (int64_t)g.px + (x + g.xo);
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace

template <typename real, int MINB, int STCS>
__global__ void __launch_bounds__(SWEEP_BX *SWEEP_BY, MINB)
    sweep_direct_kernel(const SweepArgs<real> a, const DirectArgs<real> dx)
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
    const Geom &g = a.g;
    const int64_t qs = g.qs;

    if (x < bx.lo[0] + bx.n[0] && y < bx.lo[1] + bx.n[1]) {
        const int64_t cell = cidx(g, x, y, z);
        const int64_t pbase = (int64_t)bx.patch * g.ps + cell;
        const int64_t fbase = (int64_t)bx.patch * g.fs + cell;
        const uint8_t k = a.kind[fbase];
        const real *s = a.src + pbase;
        real p[Q];
        // branch-free pull (wall slots hold the store-side bounce-back)
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t sh = EX(i) + EY(i) * (int64_t)g.px + EZ(i) * g.plane;
            p[i] = __ldg(s + i * qs - sh);
        }
        if (k != 2) {
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
            for (int i = 0; i < Q; ++i) {
                if (STCS)
                    __stcs(d + i * qs, p[i]);
                else
                    d[i * qs] = p[i];
            }
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
            // Fused exchange: outgoing PDFs of face / edge cells go straight into the
            // neighbour patch's ghost cell (same global cell) of the next source grid.
            const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
            if (x == 0 || x == n0 - 1 || y == 0 || y == n1 - 1 || z == 0 || z == n2 - 1) {
                real *const *tab = dx.nbr + (int64_t)bx.patch * (NDIR * 2);
#pragma unroll
                for (int kd = 0; kd < NDIR; ++kd) {
                    const int ddx = ndir(kd, 0), ddy = ndir(kd, 1), ddz = ndir(kd, 2);
                    const bool on = (ddx == 0 || (ddx > 0 ? x == n0 - 1 : x == 0)) &&
                                    (ddy == 0 || (ddy > 0 ? y == n1 - 1 : y == 0)) &&
                                    (ddz == 0 || (ddz > 0 ? z == n2 - 1 : z == 0));
                    if (!on) continue;
                    real *nb = tab[kd * 2 + dx.dsti];
                    if (!nb) continue;
                    const int64_t gc = cidx(g, x - ddx * n0, y - ddy * n1, z - ddz * n2);
#pragma unroll
                    for (int q = 1; q < Q; ++q)
                        if (outgoing(q, kd)) nb[q * qs + gc] = p[q];
                }
            }
        }
    }
}

// Publish this rank's step completion to its peers: runs after the sweep on the
// same stream, so every store of the sweep (local and NVLink peer stores) is
// performed before the system-scope fence and the release store of the epoch.
__global__ void signal_peers_kernel(unsigned long long *epoch, unsigned long long *const *peer_inbox, int npeers)
{
    if (threadIdx.x != 0) return;
    __threadfence_system();
    const unsigned long long e = *epoch + 1;
    *epoch = e;
    for (int i = 0; i < npeers; ++i) st_release_sys(peer_inbox[i], e);
}

// Wait until every peer has finished the step this rank just finished.
__device__ __forceinline__ unsigned long long globaltimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Bounded by wall time (timeout_ns, env LBM_PEER_TIMEOUT_S, default 120 s): a
// peer that never arrives (its process died) is reported through *error and
// lbm_synchronize instead of hanging the GPU; a peer that is merely late (host
// work between its steps) is waited for.
__global__ void wait_peers_kernel(const unsigned long long *inbox, const int *peer_rank, int npeers,
                                  const unsigned long long *epoch, int *error, unsigned long long timeout_ns)
{
    const int i = threadIdx.x;
    if (i >= npeers) return;
    const unsigned long long target = *epoch;
    const unsigned long long *slot = inbox + peer_rank[i];
    if (ld_acquire_sys(slot) >= target) return;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(slot) < target) {
        __nanosleep(256);
        if (globaltimer_ns() - t0 > timeout_ns) {
            atomicExch(error, 1);
            return;
        }
    }
}

template <typename real>
cudaError_t launch_sweep_direct(const SweepArgs<real> &a, const DirectArgs<real> &dx, int64_t total_tiles,
                                int variant, cudaStream_t s)
{
    if (total_tiles <= 0) return cudaSuccess;
    dim3 block(SWEEP_BX, SWEEP_BY, 1);
    const unsigned grid = (unsigned)total_tiles;
    switch (variant) {
    case 4: sweep_direct_kernel<real, 3, 0><<<grid, block, 0, s>>>(a, dx); break;
    case 5: sweep_direct_kernel<real, 3, 1><<<grid, block, 0, s>>>(a, dx); break;
    case 7: sweep_direct_kernel<real, 4, 1><<<grid, block, 0, s>>>(a, dx); break;
    default: sweep_direct_kernel<real, 4, 0><<<grid, block, 0, s>>>(a, dx); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_signal_peers(unsigned long long *epoch, unsigned long long *const *peer_inbox, int npeers,
                                cudaStream_t s)
{
    if (npeers <= 0) return cudaSuccess;
    signal_peers_kernel<<<1, 32, 0, s>>>(epoch, peer_inbox, npeers);
    return cudaGetLastError();
}

cudaError_t launch_wait_peers(const unsigned long long *inbox, const int *peer_rank, int npeers,
                              const unsigned long long *epoch, int *error, cudaStream_t s)
{
    if (npeers <= 0) return cudaSuccess;
    static unsigned long long timeout_ns = 0;
    if (!timeout_ns) {
        const char *e = std::getenv("LBM_PEER_TIMEOUT_S");
        const double sec = e ? std::atof(e) : 120.0;
        timeout_ns = (unsigned long long)((sec > 0 ? sec : 120.0) * 1e9);
    }
    wait_peers_kernel<<<1, 32, 0, s>>>(inbox, peer_rank, npeers, epoch, error, timeout_ns);
    return cudaGetLastError();
}

template cudaError_t launch_sweep_direct<float>(const SweepArgs<float> &, const DirectArgs<float> &, int64_t, int,
                                                cudaStream_t);
template cudaError_t launch_sweep_direct<double>(const SweepArgs<double> &, const DirectArgs<double> &, int64_t, int,
                                                 cudaStream_t);

}  // namespace lbm
