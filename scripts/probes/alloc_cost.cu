// Probe: cost of allocating / freeing the host drop-in's device buffers
// (2 x 64 GiB at C5), and whether an allocation overlaps an in-flight H2D.
//   nvcc -O2 -o scripts/probes/alloc_cost scripts/probes/alloc_cost.cu && scripts/probes/alloc_cost
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x) do { cudaError_t e = (x); if (e) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    const size_t G = size_t(1) << 30, B = 64 * G;
    void *a = nullptr, *b = nullptr;
    CK(cudaFree(0));
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        CK(cudaMalloc(&a, B));
        double t1 = now();
        CK(cudaMalloc(&b, B));
        double t2 = now();
        CK(cudaFree(a));
        double t3 = now();
        CK(cudaFree(b));
        double t4 = now();
        std::printf("cudaMalloc 64GiB %.1f ms, again %.1f ms; cudaFree %.1f ms, %.1f ms\n", t1 - t0, t2 - t1, t3 - t2, t4 - t3);
    }
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        CK(cudaMallocAsync(&a, B, st));
        CK(cudaMallocAsync(&b, B, st));
        CK(cudaStreamSynchronize(st));
        double t1 = now();
        CK(cudaMemsetAsync(a, 0, B, st));
        CK(cudaMemsetAsync(b, 0, B, st));
        CK(cudaStreamSynchronize(st));
        double t2 = now();
        CK(cudaFreeAsync(a, st));
        CK(cudaFreeAsync(b, st));
        CK(cudaStreamSynchronize(st));
        double t3 = now();
        std::printf("cudaMallocAsync 2x64GiB %.1f ms (+first-touch memset %.1f ms); cudaFreeAsync+sync %.1f ms\n",
                    t1 - t0, t2 - t1, t3 - t2);
    }
    // allocation while a 16 GiB H2D copy is in flight
    void* h = nullptr;
    CK(cudaMallocHost(&h, 16 * G));
    CK(cudaMalloc(&a, 16 * G));
    double t0 = now();
    CK(cudaMemcpyAsync(a, h, 16 * G, cudaMemcpyHostToDevice, st));
    double t1 = now();
    CK(cudaMalloc(&b, B));
    double t2 = now();
    CK(cudaStreamSynchronize(st));
    double t3 = now();
    std::printf("H2D 16GiB alone-ish: issue %.1f ms; cudaMalloc 64GiB during it %.1f ms; copy done at %.1f ms\n",
                t1 - t0, t2 - t1, t3 - t0);
    CK(cudaFree(b));
    t0 = now();
    CK(cudaMemcpyAsync(a, h, 16 * G, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    std::printf("H2D 16GiB alone %.1f ms\n", now() - t0);
    return 0;
}
