// Development microbenchmark: throughput of global fp64 / fp32 atomic adds (RED) into an
// L2-resident array at random addresses (the dense bin's accumulation).  nvcc -O3
// -gencode arch=compute_100a,code=sm_100a tools/ubench_red.cu -o /tmp/ubench_red
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}
template <typename T>
__global__ void k_red(T *acc, uint32_t mask, int iters) {
    uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; i++) {
        x = mix(x + 0x9e3779b9u);
        atomicAdd(acc + (x & mask), (T)1e-3);
    }
}
int main() {
    for (int lg : {20, 23, 26}) {   // 8 MB, 64 MB, 512 MB of doubles
        size_t n = (size_t)1 << lg;
        double *d; float *f;
        cudaMalloc(&d, n * 8); cudaMalloc(&f, n * 4);
        cudaMemset(d, 0, n * 8); cudaMemset(f, 0, n * 4);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        int blocks = 148 * 8, threads = 512, iters = 256;
        k_red<double><<<blocks, threads>>>(d, (uint32_t)(n - 1), 8);
        cudaEventRecord(a);
        k_red<double><<<blocks, threads>>>(d, (uint32_t)(n - 1), iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters;
        printf("fp64 RED, %zu MB array: %.1f G ops/s\n", n * 8 >> 20, ops / ms / 1e6);
        cudaEventRecord(a);
        k_red<float><<<blocks, threads>>>(f, (uint32_t)(n - 1), iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("fp32 RED, %zu MB array: %.1f G ops/s\n", n * 4 >> 20, ops / ms / 1e6);
        cudaFree(d); cudaFree(f);
    }
    return 0;
}
