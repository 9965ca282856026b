// How many clusters of n CTAs (512 threads, ~162 KB smem each) can be resident at once
// on this GPU (cudaOccupancyMaxActiveClusters). Dev tool.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[threadIdx.x]; }
int main() {
    const int smems[] = {162 * 1024, 100 * 1024, 60 * 1024};
    for (int smem : smems) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int n = 2; n <= 16; ++n) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(n, 8);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = n; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr; cfg.numAttrs = 1;
            int c = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&c, k, &cfg);
            printf("smem %3d KB cluster %2d: max active clusters %d (%s)\n", smem / 1024, n, c, cudaGetErrorString(e));
        }
    }
    return 0;
}
