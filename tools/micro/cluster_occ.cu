// How many thread-block clusters of a 512-thread, ~200 KB-smem CTA can be
// co-resident on this GPU (diagnostics for the split-K reduction design).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) dummy(int* p) {
    extern __shared__ int s[];
    if (p) p[0] = s[0];
}
int main() {
    int smems[] = {130 * 1024, 196 * 1024, 220 * 1024};
    for (int smem : smems) {
        cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int c : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(c * 16, 1, 1);
            cfg.blockDim = dim3(512, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = c;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
            printf("smem %3d KB cluster %2d: max active clusters %3d -> %3d CTAs %s\n", smem / 1024, c, n,
                   n * c, e ? cudaGetErrorString(e) : "");
        }
    }
    return 0;
}
