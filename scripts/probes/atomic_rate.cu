// L2 atomic throughput probe: random red.global.add.u32 into a counter table
// of a given size (feasibility of per-record global histogram atomics).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; return x ^ (x >> 33);
}

__global__ void k_red(unsigned* table, uint32_t mask, uint64_t per_thread, uint64_t seed) {
    uint64_t s = seed ^ (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x);
    for (uint64_t i = 0; i < per_thread; ++i) {
        s = mix(s + i);
        atomicAdd(&table[s & mask], 1u);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (uint32_t bits : {8u, 16u, 20u, 24u}) {
        const uint32_t n = 1u << bits;
        unsigned* t;
        cudaMalloc(&t, size_t(n) * 4);
        cudaMemset(t, 0, size_t(n) * 4);
        const int blocks = sms * 8, threads = 256;
        const uint64_t per = 2048;
        k_red<<<blocks, threads>>>(t, n - 1, 16, 1);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_red<<<blocks, threads>>>(t, n - 1, per, 7);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = double(blocks) * threads * per;
        printf("table 2^%u u32 (%6.1f MB): %.1f G atomics/s\n", bits, n * 4.0 / 1e6, ops / (ms * 1e6));
        cudaFree(t);
    }
    return 0;
}
