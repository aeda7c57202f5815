// stream_ceiling.cu -- bandwidth ceiling of the sweep's access pattern on this GPU.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/stream_ceiling tools/stream_ceiling.cu
//   build/stream_ceiling [n=256] [patches=1]
// patches > 1: that many n^3 patches, each with its own ghost shell (the
// patch-heavy layout), z of the grid running over patch * n + z.
// Streams 19 q-slices in and 19 out over an n^3 lattice with the sweep's
// padded layout (row pitch roundup(xo + n + 2, 128 B)), two cells per thread,
// no arithmetic: (a) aligned copy, (b) pull-shifted reads (x - e_i per slice).
// Reports algorithmic GB/s = 2 * 19 * elem * n^3 / time.  Also a plain 1-D copy.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

constexpr int Q = 19;
__constant__ int cEX[Q] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
__constant__ int cEY[Q] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
__constant__ int cEZ[Q] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};

// SHIFT 0: aligned; 1: pull-shifted reads (x - e_i); 2: pull-shifted reads and
// push-shifted writes (x + e_i, the AA PULL step's scatter); 3: as 2, but the
// e_x != 0 scatters realigned through warp shuffles into 2-vector stores.
template <typename T, int SHIFT>
__global__ void __launch_bounds__(128, 3) stream_kernel(const T *__restrict__ src, T *__restrict__ dst, int n,
                                                        int px, long long plane, long long qs, int xo)
{
    const int x0 = blockIdx.x * 64 + 2 * threadIdx.x;
    const int y = blockIdx.y * 4 + threadIdx.y;
    const int z = blockIdx.z % n;
    const long long pbase = (long long)(blockIdx.z / n) * Q * qs;
    if (x0 >= n || y >= n) return;
    const long long cell = pbase + ((long long)(z + 1) * (n + 2) + (y + 1)) * px + x0 + xo;
    T a[Q], b[Q];
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const long long sh = SHIFT ? (cEX[i] + cEY[i] * (long long)px + cEZ[i] * plane) : 0;
        if (SHIFT == 4 && cEX[i] != 0) {
            // aligned pair at x0 (row shifted in y / z only) + the neighbour lane's element
            const T *row = src + cell + i * qs - (sh - cEX[i]);
            const V2 v = __ldg(reinterpret_cast<const V2 *>(row));
            const int lane = threadIdx.x;
            if (cEX[i] > 0) {  // need (x0 - 1, x0): (lane - 1's .y, my .x)
                T up = __shfl_up_sync(0xffffffffu, v.y, 1);
                if (lane == 0) up = __ldg(row - 1);
                a[i] = up;
                b[i] = v.x;
            } else {           // need (x0 + 1, x0 + 2): (my .y, lane + 1's .x)
                T dn = __shfl_down_sync(0xffffffffu, v.x, 1);
                if (lane == 31) dn = __ldg(row + 2);
                a[i] = v.y;
                b[i] = dn;
            }
        } else if (!SHIFT || cEX[i] == 0) {
            const V2 v = __ldg(reinterpret_cast<const V2 *>(src + cell + i * qs - sh));
            a[i] = v.x;
            b[i] = v.y;
        } else {
            a[i] = __ldg(src + cell + i * qs - sh);
            b[i] = __ldg(src + cell + i * qs - sh + 1);
        }
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const long long sh = (SHIFT == 2 || SHIFT == 3) ? (cEX[i] + cEY[i] * (long long)px + cEZ[i] * plane) : 0;
        if (SHIFT == 3 && cEX[i] != 0) {
            // pair (x0, x0 + 1) of the destination row: e_x = +1 -> (b of lane - 1, a);
            // e_x = -1 -> (b, a of lane + 1); edge lanes store their stray element alone
            const int lane = threadIdx.x;
            using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
            T *row = dst + cell + i * qs + (sh - cEX[i]);
            if (cEX[i] > 0) {
                const T up = __shfl_up_sync(0xffffffffu, b[i], 1);
                if (lane > 0) {
                    V2 w; w.x = up; w.y = a[i];
                    *reinterpret_cast<V2 *>(row) = w;
                } else {
                    row[1] = a[i];
                }
                if (lane == 31) row[2] = b[i];
            } else {
                const T dn = __shfl_down_sync(0xffffffffu, a[i], 1);
                if (lane < 31) {
                    V2 w; w.x = b[i]; w.y = dn;
                    *reinterpret_cast<V2 *>(row) = w;
                } else {
                    row[0] = b[i];
                }
                if (lane == 0) row[-1] = a[i];
            }
        } else {
            dst[cell + i * qs + sh] = a[i];
            dst[cell + i * qs + sh + 1] = b[i];
        }
    }
}

// fp32, four cells per thread: float4 for the 9 directions with e_x = 0, four
// scalar loads for the pull-shifted ones; float4 stores.  Block (16, 8) = 64 x 8.
template <bool SHIFT>
__global__ void __launch_bounds__(128, 4) stream4_kernel(const float *__restrict__ src, float *__restrict__ dst, int n,
                                                         int px, long long plane, long long qs, int xo)
{
    const int x0 = blockIdx.x * 64 + 4 * threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int z = blockIdx.z % n;
    const long long pbase = (long long)(blockIdx.z / n) * Q * qs;
    if (x0 >= n || y >= n) return;
    const long long cell = pbase + ((long long)(z + 1) * (n + 2) + (y + 1)) * px + x0 + xo;
    float4 v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const long long sh = SHIFT ? (cEX[i] + cEY[i] * (long long)px + cEZ[i] * plane) : 0;
        const float *s = src + cell + i * qs - sh;
        if (!SHIFT || cEX[i] == 0) {
            v[i] = __ldg(reinterpret_cast<const float4 *>(s));
        } else {
            v[i].x = __ldg(s); v[i].y = __ldg(s + 1); v[i].z = __ldg(s + 2); v[i].w = __ldg(s + 3);
        }
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) *reinterpret_cast<float4 *>(dst + cell + i * qs) = v[i];
}

void run4(int n, int P)
{
    const int ae = 32, xo = ae;
    const int px = ((xo + n + 2 + ae - 1) / ae) * ae;
    const long long plane = (long long)px * (n + 2), qs = plane * (n + 2);
    const size_t bytes = (size_t)P * Q * qs * sizeof(float);
    float *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    dim3 grid((n + 63) / 64, (n + 7) / 8, n * P), block(16, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double alg = 2.0 * Q * sizeof(float) * (double)n * n * n * P;
    for (int shift = 0; shift < 2; ++shift) {
        for (int w = 0; w < 5; ++w)
            shift ? stream4_kernel<true><<<grid, block>>>(a, b, n, px, plane, qs, xo)
                  : stream4_kernel<false><<<grid, block>>>(a, b, n, px, plane, qs, xo);
        const int reps = 50;
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r)
            shift ? stream4_kernel<true><<<grid, block>>>(r & 1 ? b : a, r & 1 ? a : b, n, px, plane, qs, xo)
                  : stream4_kernel<false><<<grid, block>>>(r & 1 ? b : a, r & 1 ? a : b, n, px, plane, qs, xo);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("elem=4 n=%d patches=%d four cells/thread %s: %.3f ms/launch, %.1f GB/s algorithmic\n", n, P,
               shift ? "pull-shifted" : "aligned", ms / reps, alg / (ms / reps * 1e-3) / 1e9);
    }
    cudaFree(a);
    cudaFree(b);
}

// Patch layout with the x-ghost columns moved out of the rows (a design study for
// the patch-heavy configuration): rows hold exactly the n interior cells (aligned,
// pitch n, no x padding), and each patch keeps two compact arrays g[side][5 q][z][y]
// for its x ghosts.  The pull of the 10 e_x != 0 directions takes the row values
// and, for the cell on the patch's x face, the compact ghost; every cell on an x
// face also writes its 5 outgoing values into the compact array (the neighbour's
// ghost).  Two cells per thread, block (32, 4) = 64 x 4.
template <typename T>
__global__ void __launch_bounds__(128, 3) stream_compact_kernel(const T *__restrict__ src, T *__restrict__ dst,
                                                               const T *__restrict__ gsrc, T *__restrict__ gdst,
                                                               int n, long long plane, long long qs)
{
    const int x0 = blockIdx.x * 64 + 2 * threadIdx.x;
    const int y = blockIdx.y * 4 + threadIdx.y;
    const int z = blockIdx.z % n;
    const long long p = blockIdx.z / n;
    if (x0 >= n || y >= n) return;
    const long long pbase = p * Q * qs;
    const long long cell = pbase + ((long long)(z + 1) * (n + 2) + (y + 1)) * n + x0;  // rows: pitch n
    const long long gplane = (long long)(n + 2) * (n + 2);                              // [z][y] with halo
    const long long gbase = p * 2 * 5 * gplane;                                          // [side][5][z][y]
    T a[Q], b[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const long long sh = cEY[i] * (long long)n + cEZ[i] * plane;  // y / z shift only
        const T *row = src + cell + i * qs - sh;
        if (cEX[i] == 0) {
            a[i] = __ldg(row);
            b[i] = __ldg(row + 1);
        } else if (cEX[i] > 0) {  // pull from x - 1
            const long long gi = gbase + (0 * 5 + (i % 5)) * gplane + (long long)(z + 1 - cEZ[i]) * (n + 2) + (y + 1 - cEY[i]);
            a[i] = x0 == 0 ? __ldg(gsrc + gi) : __ldg(row - 1);
            b[i] = __ldg(row);
        } else {                  // pull from x + 1
            const long long gi = gbase + (1 * 5 + (i % 5)) * gplane + (long long)(z + 1 - cEZ[i]) * (n + 2) + (y + 1 - cEY[i]);
            a[i] = __ldg(row + 1);
            b[i] = x0 + 2 >= n ? __ldg(gsrc + gi) : __ldg(row + 2);
        }
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        dst[cell + i * qs] = a[i];
        dst[cell + i * qs + 1] = b[i];
    }
    // x-face cells write their 5 outgoing values into the compact ghost arrays
    if (x0 == 0 || x0 + 2 >= n) {
        const long long go = (long long)(z + 1) * (n + 2) + (y + 1);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (x0 == 0) gdst[gbase + (1 * 5 + k) * gplane + go] = a[2 * k + 2];
            if (x0 + 2 >= n) gdst[gbase + (0 * 5 + k) * gplane + go] = b[2 * k + 1];
        }
    }
}

template <typename T>
void run_compact(int n, int P)
{
    const long long plane = (long long)n * (n + 2), qs = plane * (n + 2);
    const size_t bytes = (size_t)P * Q * qs * sizeof(T);
    const size_t gbytes = (size_t)P * 2 * 5 * (n + 2) * (n + 2) * sizeof(T);
    T *a, *b, *ga, *gb;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&ga, gbytes);
    cudaMalloc(&gb, gbytes);
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    cudaMemset(ga, 0, gbytes);
    cudaMemset(gb, 0, gbytes);
    dim3 grid((n + 63) / 64, (n + 3) / 4, n * P), block(32, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double alg = 2.0 * Q * sizeof(T) * (double)n * n * n * P;
    for (int w = 0; w < 5; ++w) stream_compact_kernel<T><<<grid, block>>>(a, b, ga, gb, n, plane, qs);
    const int reps = 50;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
        stream_compact_kernel<T><<<grid, block>>>(r & 1 ? b : a, r & 1 ? a : b, r & 1 ? gb : ga, r & 1 ? ga : gb, n,
                                                  plane, qs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("elem=%zu n=%d patches=%d pull-shifted, compact x ghosts (rows unpadded): %.3f ms/launch, %.1f GB/s algorithmic\n",
           sizeof(T), n, P, ms / reps, alg / (ms / reps * 1e-3) / 1e9);
    cudaFree(a);
    cudaFree(b);
    cudaFree(ga);
    cudaFree(gb);
}

// Layout variant: x = -1 stored in the previous row's tail slot (x = 0 at offset 0,
// pitch roundup(n + 2, 128 B)), i.e. half the row padding of the default layout.
template <typename T>
void run_xo0(int n, int P)
{
    const int ae = 128 / sizeof(T), xo = 0;
    const int px = ((n + 2 + ae - 1) / ae) * ae;
    const long long plane = (long long)px * (n + 2), qs = plane * (n + 2);
    const size_t elems = (size_t)P * Q * qs + 2 * px;
    T *a0, *b0;
    cudaMalloc(&a0, elems * sizeof(T));
    cudaMalloc(&b0, elems * sizeof(T));
    cudaMemset(a0, 0, elems * sizeof(T));
    cudaMemset(b0, 0, elems * sizeof(T));
    T *a = a0 + px, *b = b0 + px;  // room for x = -1 of the very first row
    dim3 grid((n + 63) / 64, (n + 3) / 4, n * P), block(32, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double alg = 2.0 * Q * sizeof(T) * (double)n * n * n * P;
    for (int w = 0; w < 5; ++w) stream_kernel<T, 1><<<grid, block>>>(a, b, n, px, plane, qs, xo);
    const int reps = 50;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) stream_kernel<T, 1><<<grid, block>>>(r & 1 ? b : a, r & 1 ? a : b, n, px, plane, qs, xo);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("elem=%zu n=%d patches=%d pull-shifted, x = -1 in the previous row (pitch %d): %.3f ms/launch, %.1f GB/s algorithmic\n",
           sizeof(T), n, P, px, ms / reps, alg / (ms / reps * 1e-3) / 1e9);
    cudaFree(a0);
    cudaFree(b0);
}

template <typename T>
__global__ void copy1d(const T *__restrict__ s, T *__restrict__ d, long long n)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        d[i] = s[i];
}

template <typename T>
void run(int n, int P)
{
    const int ae = 128 / sizeof(T), xo = ae;
    const int px = ((xo + n + 2 + ae - 1) / ae) * ae;
    const long long plane = (long long)px * (n + 2), qs = plane * (n + 2);
    const size_t bytes = (size_t)P * Q * qs * sizeof(T);
    T *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    dim3 grid((n + 63) / 64, (n + 3) / 4, n * P), block(32, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double alg = 2.0 * Q * sizeof(T) * (double)n * n * n * P;
    auto launch = [&](int shift, T *s, T *d) {
        switch (shift) {
        case 0: stream_kernel<T, 0><<<grid, block>>>(s, d, n, px, plane, qs, xo); break;
        case 1: stream_kernel<T, 1><<<grid, block>>>(s, d, n, px, plane, qs, xo); break;
        case 2: stream_kernel<T, 2><<<grid, block>>>(s, d, n, px, plane, qs, xo); break;
        case 3: stream_kernel<T, 3><<<grid, block>>>(s, d, n, px, plane, qs, xo); break;
        default: stream_kernel<T, 4><<<grid, block>>>(s, d, n, px, plane, qs, xo); break;
        }
    };
    const char *names[5] = {"aligned 19-in/19-out", "pull-shifted 19-in/19-out", "pull reads + push-shifted writes",
                            "pull reads + push writes, shuffle-aligned",
                            "pull-shifted, 2-vector loads + shuffles for e_x != 0"};
    for (int shift = 0; shift < 5; ++shift) {
        for (int w = 0; w < 5; ++w) launch(shift, a, b);
        const int reps = 50;
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch(shift, r & 1 ? b : a, r & 1 ? a : b);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("elem=%zu n=%d patches=%d %s: %.3f ms/launch, %.1f GB/s algorithmic\n", sizeof(T), n, P,
               names[shift], ms / reps, alg / (ms / reps * 1e-3) / 1e9);
    }
    const long long ne = (long long)(bytes / sizeof(T));
    for (int w = 0; w < 3; ++w) copy1d<T><<<148 * 8, 256>>>(a, b, ne);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) copy1d<T><<<148 * 8, 256>>>(r & 1 ? b : a, r & 1 ? a : b, ne);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("elem=%zu plain 1-D copy of %.2f GB: %.1f GB/s (read+write)\n", sizeof(T), bytes / 1e9,
           2.0 * bytes / (ms / 20 * 1e-3) / 1e9);
    cudaFree(a);
    cudaFree(b);
}

int main(int argc, char **argv)
{
    const int n = argc > 1 ? atoi(argv[1]) : 256;
    const int P = argc > 2 ? atoi(argv[2]) : 1;
    run<double>(n, P);
    run<float>(n, P);
    run4(n, P);
    if (P > 1) {
        run_compact<double>(n, P);
        run_compact<float>(n, P);
    }
    run_xo0<double>(n, P);
    run_xo0<float>(n, P);
    return 0;
}
