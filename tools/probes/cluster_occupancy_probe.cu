// How many thread-block clusters of size 2 / 4 / 8 can be co-resident on this GPU for a
// persistent kernel with ~200 KB of shared memory per CTA (one CTA per SM)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cop cluster_occupancy_probe.cu && /tmp/cop
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* p) {
    extern __shared__ int s[];
    if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    printf("SMs %d\n", nsm);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = cs, attr.val.clusterDim.y = 1, attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster size %2d: max active clusters %3d -> %3d SMs busy (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
