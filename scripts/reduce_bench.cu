// Microbenchmark: cost of adding split-K partial tiles [64 x 128] fp32 (32 KB) into a shared
// fp32 target from N CTAs (N / 8 partials per target tile), until globally visible.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o reduce_bench reduce_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

PI0B_DEV void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(m)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1)
        : "memory");
}

// mode 0: red.v4 from registers; 1: TMA reduce, 4 SW128 boxes of 8 KB; 2: TMA reduce, one
// 32 KB box (no swizzle); 3: plain st.v4 into a private workspace slice.
__global__ void __launch_bounds__(256, 1) red_kernel(const __grid_constant__ CUtensorMap m4, const __grid_constant__ CUtensorMap m1,
                                                     float* target, float* ws, int mode, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int tile = blockIdx.x % 8;
    const int tid = threadIdx.x;
    // every thread holds 32 values (128 threads x 32 cols x ... ): rows r = tid & 63, cols half = tid >> 6
    const int r = tid & 63, q = tid >> 6;  // q in 0..3 -> 32 columns each
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = float(j + r) * 1e-3f;
    __syncthreads();
    const long long t0 = clock64();
    if (mode == 0) {
        float* dst = target + r * 1024 + tile * 128 + q * 32;
#pragma unroll
        for (int j = 0; j < 8; ++j) red_add_v4_f32(dst + 4 * j, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        __threadfence();
        __syncthreads();
    } else if (mode == 4 || mode == 5) {
        // coalesced: warp w -> rows 8w..8w+7, lane -> 4 consecutive columns (512 B per row)
        const int w = tid >> 5, lane = tid & 31;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float* dst = (mode == 4 ? target + (8 * w + i) * 1024 + tile * 128
                                    : ws + (size_t)blockIdx.x * 8192 + (8 * w + i) * 128) + lane * 4;
            if (mode == 4) red_add_v4_f32(dst, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            else *reinterpret_cast<float4*>(dst) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        __threadfence();
        __syncthreads();
    } else if (mode == 1 || mode == 2) {
        if (mode == 1) {
            uint8_t* box = smem + q * 8192 + r * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(box + ((j ^ (r & 7)) << 4)) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
            float* row = reinterpret_cast<float*>(smem) + r * 128 + q * 32;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = (j + r) & 7;  // rotate chunks: conflict-free across the warp's rows
                *reinterpret_cast<float4*>(row + 4 * jj) = make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            if (mode == 1)
                for (int b = 0; b < 4; ++b) tma_reduce_add_2d(&m4, smem + b * 8192, tile * 128 + 32 * b, 0);
            else
                tma_reduce_add_2d(&m1, smem, tile * 128, 0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            __threadfence();
        }
        __syncthreads();
    } else {
        float* dst = ws + (size_t)blockIdx.x * 8192 + r * 128 + q * 32;
#pragma unroll
        for (int j = 0; j < 8; ++j) *reinterpret_cast<float4*>(dst + 4 * j) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        __threadfence();
        __syncthreads();
    }
    if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    float *target, *ws;
    cudaMalloc(&target, 64 * 1024 * 4);
    cudaMalloc(&ws, 148ll * 8192 * 4);
    cudaMemset(target, 0, 64 * 1024 * 4);
    void* fn;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
    CUtensorMap m4, m1;
    cuuint64_t dims[2] = {1024, 64};
    cuuint64_t strides[1] = {4096};
    cuuint32_t es[2] = {1, 1};
    cuuint32_t b4[2] = {32, 64}, b1[2] = {128, 64};
    enc(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, target, dims, strides, b4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, target, dims, strides, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* names[] = {"red.v4 from registers", "TMA reduce 4x8KB SW128", "TMA reduce 1x32KB", "plain st.v4 (no add)",
                           "red.v4 coalesced", "st.v4 coalesced"};
    for (int mode = 0; mode < 6; ++mode)
        for (int n : {8, 32, 128, 148}) {
            double best = 1e30, med = 0;
            for (int rep = 0; rep < 3; ++rep) {
                red_kernel<<<n, 256, 40 * 1024>>>(m4, m1, target, ws, mode, out);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("%s: %s\n", names[mode], cudaGetErrorString(e));
                    return 1;
                }
                std::vector<unsigned long long> h(n);
                cudaMemcpy(h.data(), out, n * 8, cudaMemcpyDeviceToHost);
                unsigned long long mx = 0, sum = 0;
                for (auto v : h) {
                    mx = v > mx ? v : mx;
                    sum += v;
                }
                best = std::min(best, mx / (clk * 1e-3));
                med = sum / double(n) / (clk * 1e-3);
            }
            printf("%-26s ctas=%3d (%2d partials/tile): max %6.2f us  mean %6.2f us per CTA (32 KB each)\n", names[mode], n,
                   n / 8, best, med);
        }
    return 0;
}
