// Pure HBM read bandwidth (the histogram pass's ceiling): stream a large
// buffer with 16-B non-allocating loads, fold into a checksum.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int UNROLL>
__global__ void k_read(const uint4* __restrict__ p, uint64_t n16, unsigned* out) {
    uint32_t acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * stride < n16; i += UNROLL * stride) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p + i + u * stride));
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) acc ^= p[i].x;
    if (acc == 0x12345678u) atomicAdd(out, 1u);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t bytes = 32ull << 30;
    uint4* p;
    unsigned* out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int bpsm : {2, 4, 8}) {
        for (int pass = 0; pass < 2; ++pass) {
            cudaEventRecord(a);
            k_read<8><<<sms * bpsm, 256>>>(p, bytes / 16, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (pass) printf("read 32 GiB, %d CTAs/SM x 256 thr, unroll 8: %.0f GB/s\n", bpsm, bytes / (ms * 1e6));
        }
    }
    cudaEventRecord(a);
    cudaMemcpy(p, p + (bytes / 32), bytes / 2, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("copy 16 GiB (read+write): %.0f GB/s\n", bytes / (ms * 1e6));
    return 0;
}
