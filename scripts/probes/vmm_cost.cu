// Probe: virtual-memory-management (cuMem*) cost of mapping / unmapping the
// host drop-in's device buffers, and whether unmapping one range waits for
// a D2H copy still reading another range.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o scripts/probes/vmm_cost scripts/probes/vmm_cost.cu && scripts/probes/vmm_cost
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x) do { auto e = (x); if (e) { std::printf("%s: error %d\n", #x, int(e)); return 1; } } while (0)
template <typename T> static T entry(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
    return reinterpret_cast<T>(p);
}
int main() {
    CK(cudaFree(0));
    auto pCreate = entry<decltype(&cuMemCreate)>("cuMemCreate");
    auto pReserve = entry<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
    auto pMap = entry<decltype(&cuMemMap)>("cuMemMap");
    auto pAccess = entry<decltype(&cuMemSetAccess)>("cuMemSetAccess");
    auto pUnmap = entry<decltype(&cuMemUnmap)>("cuMemUnmap");
    auto pRelease = entry<decltype(&cuMemRelease)>("cuMemRelease");
    auto pFree = entry<decltype(&cuMemAddressFree)>("cuMemAddressFree");
    auto pGran = entry<decltype(&cuMemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gran = 0;
    CK(pGran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t G = size_t(1) << 30, B = 64 * G, CH = 4 * G;
    std::printf("granularity %zu\n", gran);
    auto map = [&](CUdeviceptr& va, std::vector<CUmemGenericAllocationHandle>& hs, size_t chunk) -> int {
        CK(pReserve(&va, B, 0, 0, 0));
        for (size_t o = 0; o < B; o += chunk) {
            CUmemGenericAllocationHandle h;
            CK(pCreate(&h, chunk, &prop, 0));
            CK(pMap(va + o, chunk, 0, h, 0));
            hs.push_back(h);
        }
        CUmemAccessDesc ad = {};
        ad.location = prop.location;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CK(pAccess(va, B, &ad, 1));
        return 0;
    };
    auto unmap = [&](CUdeviceptr va, std::vector<CUmemGenericAllocationHandle>& hs, size_t chunk) -> int {
        for (size_t i = 0; i < hs.size(); ++i) {
            CK(pUnmap(va + i * chunk, chunk));
            CK(pRelease(hs[i]));
        }
        CK(pFree(va, B));
        hs.clear();
        return 0;
    };
    for (size_t chunk : {B, CH}) {
        CUdeviceptr va;
        std::vector<CUmemGenericAllocationHandle> hs;
        double t0 = now();
        if (map(va, hs, chunk)) return 1;
        double t1 = now();
        CK(cudaMemset(reinterpret_cast<void*>(va), 0, B));
        CK(cudaDeviceSynchronize());
        double t2 = now();
        if (unmap(va, hs, chunk)) return 1;
        double t3 = now();
        std::printf("VMM 64GiB in %zu-GiB chunks: map %.1f ms, first-touch memset %.1f ms, unmap+release %.1f ms\n",
                    chunk >> 30, t1 - t0, t2 - t1, t3 - t2);
    }
    // unmap B while a D2H copy from A is in flight
    CUdeviceptr va, vb;
    std::vector<CUmemGenericAllocationHandle> ha, hb;
    if (map(va, ha, CH) || map(vb, hb, CH)) return 1;
    CK(cudaMemset(reinterpret_cast<void*>(vb), 0, B));
    void* h = nullptr;
    CK(cudaMallocHost(&h, 16 * G));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaDeviceSynchronize());
    double t0 = now();
    CK(cudaMemcpyAsync(h, reinterpret_cast<void*>(va), 16 * G, cudaMemcpyDeviceToHost, st));
    double t1 = now();
    if (unmap(vb, hb, CH)) return 1;
    double t2 = now();
    CK(cudaStreamSynchronize(st));
    double t3 = now();
    std::printf("unmap of B during a 16 GiB D2H from A: unmap took %.1f ms (issued at %.1f), copy done at %.1f ms\n",
                t2 - t1, t1 - t0, t3 - t0);
    // cudaFree of a cudaMalloc'd buffer during the same kind of copy
    void* c = nullptr;
    CK(cudaMalloc(&c, B));
    CK(cudaMemset(c, 0, B));
    CK(cudaDeviceSynchronize());
    t0 = now();
    CK(cudaMemcpyAsync(h, reinterpret_cast<void*>(va), 16 * G, cudaMemcpyDeviceToHost, st));
    t1 = now();
    CK(cudaFree(c));
    t2 = now();
    CK(cudaStreamSynchronize(st));
    t3 = now();
    std::printf("cudaFree of 64 GiB during a 16 GiB D2H: free returned after %.1f ms, copy done at %.1f ms\n", t2 - t1, t3 - t0);
    return 0;
}
