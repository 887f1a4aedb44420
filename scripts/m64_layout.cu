// Probe: where does tcgen05.mma (cta_group::1, kind::f16) with M = 64 put the rows of D in TMEM?
// A[64 x 16] has row r = (r + 1), B[N=64 x 16] = ones -> D[r][n] = 16 (r + 1).  Every warp of a
// 128-thread CTA reads its lane quarter (32x32b.x4, columns 0..3) and reports which value each
// lane holds.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o m64_layout m64_layout.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

__global__ void probe(float* out) {
    __shared__ __align__(1024) uint8_t sA[16384];
    __shared__ __align__(1024) uint8_t sB[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // SW128 K-major: row r at r * 128 bytes, 16-byte chunk c at (c ^ (r & 7)); K = 16 -> chunks 0, 1
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        const int c = k / 8, e = k % 8;
        const __nv_bfloat16 va = __float2bfloat16(k < 16 ? float(r + 1) : 0.f);
        const __nv_bfloat16 vb = __float2bfloat16(k < 16 ? 1.f : 0.f);
        reinterpret_cast<__nv_bfloat16*>(sA + r * 128 + ((c ^ (r & 7)) << 4))[e] = va;
        reinterpret_cast<__nv_bfloat16*>(sB + r * 128 + ((c ^ (r & 7)) << 4))[e] = vb;
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) tmem_alloc(&tslot, 64);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        if (elect_one()) {
            umma_bf16(tmem, umma_desc_sw128(sA), umma_desc_sw128(sB), umma_idesc_bf16(64, 64), 0);
            umma_commit(&bar);
        }
        __syncwarp();
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    float4 v;
    tmem_ld4(tmem + (uint32_t(warp * 32) << 16), v);
    out[(warp * 32 + lane) * 4 + 0] = v.x;
    out[(warp * 32 + lane) * 4 + 1] = v.y;
    out[(warp * 32 + lane) * 4 + 2] = v.z;
    out[(warp * 32 + lane) * 4 + 3] = v.w;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 64);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 4 * 4);
    cudaMemset(d, 0, 128 * 16);
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[512];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("%s\n", cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) {
        const float v = h[l * 4];
        printf("lane %3d: col0 %7.1f -> row %s%d\n", l, v, v == 0 ? "(none) " : "", v == 0 ? -1 : int(v / 16.f + 0.5f) - 1);
    }
    return 0;
}
