// Microbenchmark: issue-to-completion cost of back-to-back tcgen05.mma (bf16, M=128, K=16) from
// one thread, operands in 128-byte-swizzled shared memory, as a function of N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) mma_kernel(int n_mma, int per_commit, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sA = smem;                 // 128 rows x 64 k  (16 KB)
    uint8_t* sB = smem + 16384;         // N rows x 64 k
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 256 * 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if ((threadIdx.x >> 5) == 1) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int warp_u = __shfl_sync(0xffffffff, int(threadIdx.x >> 5), 0);  // provably warp-uniform
    if (warp_u == 1) {  // whole warp runs the loop; one elected lane issues
        constexpr uint32_t idesc = umma_idesc_bf16(128, N);
        const uint64_t ad = umma_desc_sw128(sA), bd = umma_desc_sw128(sB);
        uint32_t ph = 0;
        const long long t0 = clock64();
        int c = 0;
        for (int i = 0; i < n_mma; ++i) {
            // n_acc independent accumulators (TMEM column offsets), round robin
            const int a = i & (NACC - 1);
            if (elect_one()) umma_bf16(tmem + a * N, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i >= NACC);
            if (++c == per_commit) {
                c = 0;
                if (elect_one()) umma_commit(bar);
                mbar_wait(bar, ph);
                ph ^= 1;
            }
        }
        const long long t1 = clock64();
        if (threadIdx.x == 32) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 1) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 8);
    const int smem = 16384 + 256 * 128 + 1024 + 64;
#define CFG(n, a) cudaFuncSetAttribute(mma_kernel<n, a>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
    CFG(64, 1); CFG(128, 1); CFG(256, 1); CFG(64, 2); CFG(128, 2); CFG(256, 2); CFG(64, 4); CFG(128, 4);
    for (int nacc : {1, 2, 4})
    for (int per : {4, 16, 1024})
        for (int n : {64, 128, 256}) {
            if (n * nacc > 512) continue;
            unsigned long long c = 0;
            for (int rep = 0; rep < 2; ++rep) {
#define RUN(nn, aa) if (n == nn && nacc == aa) mma_kernel<nn, aa><<<1, 128, smem>>>(1024, per, out)
                RUN(64, 1); RUN(128, 1); RUN(256, 1); RUN(64, 2); RUN(128, 2); RUN(256, 2); RUN(64, 4); RUN(128, 4);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
            }
            printf("N=%3d acc=%d commit+wait every %4d MMAs: %7.1f cycles per MMA (ideal %d)\n", n, nacc, per, c / 1024.0, 128 * n / 256);
        }
    return 0;
}
