// PCIe probe: device<->pinned-host bandwidth by DMA (cudaMemcpyAsync) vs by
// kernels reading / writing mapped pinned host memory (zero-copy), 8 GiB.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_copy(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = size_t(8) << 30;
    uint8_t *d = nullptr, *h = nullptr;
    cudaMalloc(&d, bytes);
    cudaMallocHost(&h, bytes);
    cudaMemset(d, 1, bytes);
    for (size_t i = 0; i < bytes; i += 4096) h[i] = 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto f) {
        f();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s %7.2f GB/s (%s)\n", name, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run("DMA H2D", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); });
    run("DMA D2H", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); });
    for (int g : {148, 296, 592, 1184}) {
        char nm[64];
        snprintf(nm, sizeof nm, "kernel D2H (zero-copy stores) g=%d", g);
        run(nm, [&] { k_copy<<<g, 256>>>((uint4*)h, (const uint4*)d, bytes / 16); });
        snprintf(nm, sizeof nm, "kernel H2D (zero-copy loads) g=%d", g);
        run(nm, [&] { k_copy<<<g, 256>>>((uint4*)d, (const uint4*)h, bytes / 16); });
    }
    return 0;
}
