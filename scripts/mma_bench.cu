// Microbenchmark: issue-to-completion cost of back-to-back tcgen05.mma (bf16, M=128, K=16) from
// one thread, operands in 128-byte-swizzled shared memory, as a function of N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

// TS = 1: A operand from TMEM (tcgen05.mma [d], [a_tmem], b_desc, ...), columns 256.. of the
// allocation hold the A tile (garbage values: only the issue rate is measured).
PI0B_DEV void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

template <int M, int N, int NACC, int TS>
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
        constexpr uint32_t idesc = umma_idesc_bf16(M, N);
        const uint64_t ad = umma_desc_sw128(sA), bd = umma_desc_sw128(sB);
        uint32_t ph = 0;
        const long long t0 = clock64();
        int c = 0;
        for (int i = 0; i < n_mma; ++i) {
            // n_acc independent accumulators (TMEM column offsets), round robin
            const int a = i & (NACC - 1);
            if (TS) {
                if (elect_one()) umma_bf16_ts(tmem + a * N, tmem + 256 + 8 * (i & 3), bd + 2 * (i & 3), idesc, i >= NACC);
            } else {
                if (elect_one()) umma_bf16(tmem + a * N, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i >= NACC);
            }
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

template <int M, int N, int TS>
static void run(int per, void* outp) {
    unsigned long long* out = (unsigned long long*)outp;
    const int smem = 16384 + 256 * 128 + 1024 + 64;
    cudaFuncSetAttribute(mma_kernel<M, N, 1, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
        mma_kernel<M, N, 1, TS><<<1, 128, smem>>>(1024, per, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            exit(1);
        }
        cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    }
    printf("M=%3d N=%3d %s commit+wait every %4d MMAs: %7.1f cycles per MMA\n", M, N, TS ? "A:TMEM" : "A:smem", per, c / 1024.0);
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 8);
    for (int per : {4, 1024}) {
        run<128, 64, 0>(per, out); run<128, 128, 0>(per, out); run<128, 256, 0>(per, out);
        run<64, 64, 0>(per, out); run<64, 128, 0>(per, out); run<64, 256, 0>(per, out);
        run<128, 64, 1>(per, out); run<128, 128, 1>(per, out); run<128, 256, 1>(per, out);
        run<64, 64, 1>(per, out); run<64, 128, 1>(per, out); run<64, 256, 1>(per, out);
    }
    return 0;
}
