// Does a cooperative launch accept a cluster dimension, and how many 2-CTA clusters of a
// 225 KB-smem kernel can be co-resident?  nvcc -gencode arch=compute_100a,code=sm_100a -o coop_cluster_test coop_cluster_test.cu
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void k(int* out) {
    extern __shared__ int sm[];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    sm[0] = r;
    if (threadIdx.x == 0) out[blockIdx.x] = r;
}
int main() {
    int* out;
    cudaMalloc(&out, 148 * 4);
    const int smem = 225 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cl : {1, 2, 4}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148, 1, 1);
        cfg.blockDim = dim3(320, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        int nclu = -1;
        cudaError_t eo = cudaOccupancyMaxActiveClusters(&nclu, k, &cfg);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, out);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("cluster %d: max active clusters %d (%s), coop+cluster launch: %s / %s\n", cl, nclu, cudaGetErrorString(eo),
               cudaGetErrorString(e), cudaGetErrorString(e2));
        cudaGetLastError();
    }
    return 0;
}
