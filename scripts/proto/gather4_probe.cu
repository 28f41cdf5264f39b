// Feasibility probe: TMA tile::gather4 of 4 arbitrary rows of a [d][64] fp64 array into shared
// memory (sm_100a).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o g4 gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, const int* rows, int nq, double* out) {
    __shared__ __align__(128) double buf[4 * 64];
    __shared__ __align__(8) uint64_t bar;
    for (int q = 0; q < nq; q++) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(4 * 64 * 8) : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(rows[4 * q + 0]), "r"(rows[4 * q + 1]),
                "r"(rows[4 * q + 2]), "r"(rows[4 * q + 3]), "r"(smem_u32(&bar))
                : "memory");
        }
        __syncthreads();
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        }
        for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) out[q * 256 + i] = buf[i];
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar)));
        __syncthreads();
    }
}

int main() {
    const int d = 100000, K = 64;
    std::vector<double> h((size_t)d * K);
    for (size_t i = 0; i < h.size(); i++) h[i] = (double)i;  // element (r, c) = r*64 + c
    double* dW; cudaMalloc(&dW, h.size() * 8); cudaMemcpy(dW, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap tmap;
    cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)d};
    cuuint64_t gstride[1] = {(cuuint64_t)K * 8};
    cuuint32_t box[2] = {(cuuint32_t)K, 1};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dW, gdim, gstride, box, estride,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    int hrows[8] = {5, 99999, 0, 31337, 7, 7, 50000, 12};
    int* drows; cudaMalloc(&drows, sizeof(hrows)); cudaMemcpy(drows, hrows, sizeof(hrows), cudaMemcpyHostToDevice);
    double* dout; cudaMalloc(&dout, 2 * 256 * 8);
    probe<<<1, 128>>>(tmap, drows, 2, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<double> o(512);
    cudaMemcpy(o.data(), dout, 512 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int q = 0; q < 2; q++)
        for (int j = 0; j < 4; j++)
            for (int c = 0; c < K; c++) {
                double want = (double)hrows[4 * q + j] * K + c;
                if (o[q * 256 + j * K + c] != want) bad++;
            }
    printf("gather4 mismatches: %d of 512\n", bad);
    return bad != 0;
}
