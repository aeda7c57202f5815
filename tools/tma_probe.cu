// tma_probe.cu -- standalone probe of cp.async.bulk.tensor constraints on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/tma_probe tools/tma_probe.cu -lcuda
//   build/tma_probe <box_w> <box_h> <elem_bytes 1|4|8> <rank 2|4> <dtype u|f>
// Loads one box at a shifted coordinate into shared memory and checks it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int rank, int c0, int c1, unsigned bytes,
                      unsigned char *out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes));
        if (rank == 2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(smem_u32(sm)),
                "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(smem_u32(&bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
                "%5}], [%6];" ::"r"(smem_u32(sm)),
                "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(1), "r"(2), "r"(smem_u32(&bar))
                : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(&bar)));
    }
    __syncthreads();
    for (unsigned i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char **argv)
{
    const int bw = atoi(argv[1]), bh = atoi(argv[2]), es = atoi(argv[3]), rank = atoi(argv[4]);
    const char dt = argv[5][0];
    const int W = 256, H = 16, D2 = 4, D3 = 4;
    std::vector<unsigned char> host((size_t)W * H * D2 * D3 * es);
    for (size_t i = 0; i < host.size(); ++i) host[i] = (unsigned char)(i * 7 + 3);
    void *dev;
    unsigned char *out;
    cudaMalloc(&dev, host.size());
    cudaMalloc(&out, 1 << 20);
    cudaMemcpy(dev, host.data(), host.size(), cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    CUtensorMapDataType t = es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                            : es == 4 ? (dt == 'f' ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT32)
                                      : (dt == 'f' ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_INT64);
    alignas(64) CUtensorMap map;
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)D2, (cuuint64_t)D3};
    cuuint64_t str[3] = {(cuuint64_t)W * es, (cuuint64_t)W * H * es, (cuuint64_t)W * H * D2 * es};
    cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)bh, 1, 1};
    cuuint32_t est[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, t, rank, dev, dims, str, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("box %dx%d es=%d rank=%d %c: ENCODE FAILED %d\n", bw, bh, es, rank, dt, (int)r);
        return 0;
    }
    const unsigned bytes = (unsigned)(bw * bh * es);
    const int c0 = argc > 6 ? atoi(argv[6]) : 3, c1 = 1;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    probe<<<1, 128, 65536>>>(map, rank, c0, c1, bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("box %dx%d es=%d rank=%d %c c0=%d: RUN FAILED %s\n", bw, bh, es, rank, dt, c0, cudaGetErrorName(e));
        return 0;
    }
    std::vector<unsigned char> got(bytes);
    cudaMemcpy(got.data(), out, bytes, cudaMemcpyDeviceToHost);
    size_t base = rank == 2 ? 0 : ((size_t)2 * W * H * D2 + (size_t)1 * W * H) * es;
    int bad = 0;
    for (int y = 0; y < bh; ++y)
        for (int x = 0; x < bw * es; ++x) {
            size_t gi = base + ((size_t)(c1 + y) * W) * es + (size_t)c0 * es + x;
            if (got[(size_t)y * bw * es + x] != host[gi]) ++bad;
        }
    printf("box %dx%d es=%d rank=%d %c c0=%d: %s (%d bad)\n", bw, bh, es, rank, dt, c0, bad ? "WRONG" : "ok", bad);
    return 0;
}
