// handshake.cu -- the cross-GPU step handshake of the fused exchange (sm_100a).
//
// The paper extracts boundary PDFs into buffers after the kernel, moves them
// (cudaMemcpy + MPI) and inserts them into the neighbour's ghost layer before
// its next kernel.  With the fused exchange the x2 sweep
// (sweep.cu / sweep_aa.cu, DIRECT) does all three in one pass: a fluid cell on a
// patch face stores each outgoing PDF straight into the neighbour patch's ghost
// layer, on another GPU through its CUDA-IPC-mapped grid (NVLink stores).  The
// shells that face remote neighbours are swept on the high-priority stream,
// concurrently with the plain sweep of the interiors.
//
// Cross-GPU ordering (one handshake per step): after the shell sweep, a
// one-thread kernel fences at system scope, bumps this rank's epoch and
// publishes it with a system-scope release store into each peer's inbox.  The
// next step starts with wait_peers_kernel, which acquires until every peer's
// epoch has caught up -- i.e. the peers have finished reading the grid this rank
// is about to overwrite and have finished writing the ghosts it is about to
// read.  Bounded wait (120 s by default, LBM_PEER_TIMEOUT_S): it reports an error
// instead of hanging.  A periodic self-neighbour through the same mechanism
// (exchange_mode SELF_PEER, one GPU) waits on its own previous signal, which
// precedes it in stream order, so nothing ever spins on a concurrent kernel.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

namespace lbm {

namespace {

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

}  // namespace lbm
