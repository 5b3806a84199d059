// Co-resident thread-block clusters on this GPU for one ~200 KB, 288-thread
// CTA per SM, by cluster size (cudaOccupancyMaxActiveClusters).
// nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occ cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
    const size_t bytes = 200 * 1024;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cl = 1; cl <= 16; cl *= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl * sms);
        cfg.blockDim = dim3(288);
        cfg.dynamicSmemBytes = bytes;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cluster %2d: %3d co-resident clusters = %3d SMs of %d (%s)\n", cl, n, n * cl, sms, cudaGetErrorString(e));
    }
    return 0;
}
