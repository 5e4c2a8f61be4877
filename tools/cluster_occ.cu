// tools/cluster_occ.cu — how many clusters of a pass-B-like CTA (256 threads,
// one CTA per SM by shared memory) the B200 keeps resident at once, per cluster
// size: cudaOccupancyMaxActiveClusters, i.e. how many SMs a clustered launch
// can actually use (GPC fragmentation).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_cluster_occ tools/cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(1, 1, 1) dummy1(double* p) { extern __shared__ double s[]; if (p) p[0] = s[0]; }
__global__ void dummy(double* p) { extern __shared__ double s[]; if (p) p[0] = s[0]; }

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    printf("SMs %d\n", prop.multiProcessorCount);
    const int smems[] = {64 * 1024, 100 * 1024, 160 * 1024, 226 * 1024};
    for (int sm : smems) {
        cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs * 64);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
            printf("smem %3d KB cluster %2d: max active clusters %4d -> %4d CTAs (%s)\n", sm / 1024, cs, n,
                   n * cs, cudaGetErrorString(e));
        }
    }
    return 0;
}
