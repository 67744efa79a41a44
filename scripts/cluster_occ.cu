// How many thread-block clusters of size 1/2/4/8 can be co-resident with one 512-thread CTA of
// 227 KB dynamic shared memory per SM (the byte-floor stream kernel's footprint)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int *p) {
    extern __shared__ int s[];
    if (p) p[threadIdx.x] = s[threadIdx.x];
}
int main() {
    const size_t smem = 227 * 1024;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 256);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
