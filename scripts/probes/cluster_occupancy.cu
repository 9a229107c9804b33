// How many thread-block clusters of a given size can be co-resident on this
// GPU for a 512-thread CTA with a given dynamic shared-memory footprint
// (feasibility probe for a cluster-wide local sort).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (p) p[blockIdx.x] = s[0];
}

int main() {
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    for (int smem : {100 << 10, 150 << 10, 200 << 10, 220 << 10}) {
        cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int cl : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cl * 64);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cl;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
            printf("smem %3d KB cluster %2d: max active clusters %3d (%3d CTAs) %s\n", smem >> 10, cl, n,
                   n * cl, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
