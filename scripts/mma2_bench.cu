// Microbenchmark: back-to-back tcgen05.mma issue rate for a CTA pair (cta_group::2, M=256) vs
// one CTA (cta_group::1, M=128), bf16, N=256, operands in 128-byte-swizzled shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma2_bench mma2_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

template <int CG>
__global__ void __launch_bounds__(128, 1) mma_kernel(int n_mma, int per_commit, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;          // 128 rows x 64 k  (16 KB)
    uint8_t* sB = smem + 16384;  // 256/CG rows x 64 k
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if ((threadIdx.x >> 5) == 1) {
        if (CG == 2) tmem_alloc_cg2(tslot, 256);
        else tmem_alloc(tslot, 256);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const bool leader = CG == 1 || cluster_ctarank() == 0;
    const int warp_u = __shfl_sync(0xffffffff, int(threadIdx.x >> 5), 0);
    if (warp_u == 1 && leader) {
        constexpr uint32_t idesc = umma_idesc_bf16(128 * CG, 256);
        const uint64_t ad = umma_desc_sw128(sA), bd = umma_desc_sw128(sB);
        uint32_t ph = 0;
        const long long t0 = clock64();
        int c = 0;
        for (int i = 0; i < n_mma; ++i) {
            if (elect_one()) {
                if (CG == 2) umma_bf16_cg2(tmem, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i > 0);
                else umma_bf16(tmem, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i > 0);
            }
            __syncwarp();
            if (++c == per_commit) {
                c = 0;
                if (elect_one()) {
                    if (CG == 2) umma_commit_cg2(bar);
                    else umma_commit(bar);
                }
                __syncwarp();
                mbar_wait(bar, ph);
                ph ^= 1;
            }
        }
        const long long t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    if (CG == 2 && !leader) {
        // the leader's commits also arrive on this CTA's barrier: consume the phases
        uint32_t ph = 0;
        if (threadIdx.x == 32)
            for (int i = 0; i < n_mma / per_commit; ++i) {
                mbar_wait(bar, ph);
                ph ^= 1;
            }
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    if ((threadIdx.x >> 5) == 1) {
        if (CG == 2) tmem_dealloc_cg2(tmem, 256);
        else tmem_dealloc(tmem, 256);
    }
}

template <int CG>
void run(int grid) {
    unsigned long long* out;
    cudaMalloc(&out, 1024 * 8);
    cudaMemset(out, 0, 1024 * 8);
    const int smem = 16384 + 32768 + 1024 + 64;
    cudaFuncSetAttribute(mma_kernel<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid * CG);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = CG;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    const int n = 4096, per = 64;
    for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, mma_kernel<CG>, n, per, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, out, 1024 * 8, cudaMemcpyDeviceToHost);
    printf("cta_group::%d M=%d N=256 units=%3d: %7.1f cycles per MMA (%s)\n", CG, 128 * CG, grid, double(h[0]) / n,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
    run<1>(1);
    run<2>(1);
    run<1>(148);
    run<2>(74);
    return 0;
}
