// How many clusters of 2 / 4 / 8 CTAs (1 CTA per SM, ~226 KB smem) fit on this B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kern(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
    const int smem = 226 * 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    printf("{\"cluster_occupancy\": [");
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148 * 4);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        printf("%s{\"cluster\": %d, \"max_active_clusters\": %d, \"ctas\": %d, \"err\": \"%s\"}", cs == 1 ? "" : ", ", cs, n, n * cs, cudaGetErrorString(e));
    }
    printf("]}\n");
}
