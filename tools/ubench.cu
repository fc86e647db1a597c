// Microbenchmarks of the shared-memory primitives the SpGEMM accumulator can use
// (sm_100a).  Reports products/cycle/SM-equivalents for each insert flavour.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CAP = 4096;
constexpr int ITERS = 4096;

__device__ __forceinline__ unsigned hash_slot(unsigned x) { return (x * 0x9E3779B1u) >> 20; }

template <int MODE>
__global__ void kbench(float *out, unsigned seed, long long *cyc) {
    __shared__ float vals[CAP];
    __shared__ int keys[CAP];
    for (int i = threadIdx.x; i < CAP; i += blockDim.x) { vals[i] = 0; keys[i] = i; }
    __syncthreads();
    unsigned x = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 97u);
    long long t0 = clock64();
    float acc = 0;
    for (int it = 0; it < ITERS; it++) {
        x = x * 1664525u + 1013904223u;
        unsigned s = hash_slot(x);
        if (MODE == 0) {            // float atomicAdd (CAS loop on sm_100)
            atomicAdd(&vals[s], 1.0f);
        } else if (MODE == 1) {     // int atomicAdd (native ATOMS.ADD)
            atomicAdd(&keys[s], (int)(x & 3u) + 1);
        } else if (MODE == 2) {     // plain LDS + FADD + STS (racy; for throughput only)
            vals[s] += 1.0f;
        } else if (MODE == 3) {     // match_any on the slot + plain RMW
            unsigned m = __match_any_sync(0xffffffffu, s);
            if ((__ffs(m) - 1) == (threadIdx.x & 31)) vals[s] += (float)__popc(m);
        } else if (MODE == 4) {     // LDS probe of key + plain RMW
            int k = keys[s];
            if (k == (int)s) vals[s] += 1.0f;
        } else if (MODE == 5) {     // int CAS
            atomicCAS(&keys[s], (int)s, (int)s);
        } else if (MODE == 6) {     // 64-bit int atomicAdd (fixed-point accumulator)
            atomicAdd(reinterpret_cast<unsigned long long *>(vals) + (s >> 1),
                      (unsigned long long)(x & 0xffff) + 1ull);
        }
    }
    long long t1 = clock64();
    __syncthreads();
    for (int i = threadIdx.x; i < CAP; i += blockDim.x) acc += vals[i] + keys[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 148;
    const int NT = 512, PER_SM = 3;
    const int grid = sms * PER_SM;
    float *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * grid * NT);
    cudaMalloc(&cyc, sizeof(long long) * grid);
    const char *names[] = {"float atomicAdd smem (CAS loop)", "int atomicAdd smem (ATOMS.ADD)",
                           "plain LDS+FADD+STS", "match_any + leader RMW", "LDS key probe + RMW",
                           "int atomicCAS smem", "u64 atomicAdd smem"};
    for (int mode = 0; mode < 7; mode++) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: kbench<0><<<grid, NT>>>(out, 1, cyc); break;
                case 1: kbench<1><<<grid, NT>>>(out, 1, cyc); break;
                case 2: kbench<2><<<grid, NT>>>(out, 1, cyc); break;
                case 3: kbench<3><<<grid, NT>>>(out, 1, cyc); break;
                case 4: kbench<4><<<grid, NT>>>(out, 1, cyc); break;
                case 5: kbench<5><<<grid, NT>>>(out, 1, cyc); break;
                case 6: kbench<6><<<grid, NT>>>(out, 1, cyc); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)grid * NT * ITERS;
        double per_sm_cycle = ops / (ms * 1e-3) / sms / 1.965e9;
        printf("%-36s %8.3f ms  %.3e lane-ops/s  %.2f lane-ops/cycle/SM\n", names[mode], ms, ops / (ms * 1e-3),
               per_sm_cycle);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
