// Microbenchmark: per-SM TMA tile-load throughput and latency on B200 (16 KB bf16 tiles,
// 128-byte swizzle), as a function of ring depth, CTA count and L2 residency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bench tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap m, int tiles, int depth,
                                                     int rows_total, int l2_rows, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 8 * 16384);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        unsigned long long lat = 0;
        long long issue_t[8];
        int issued = 0;
        for (int i = 0; i < tiles; ++i) {
            // keep `depth` loads in flight
            while (issued < tiles && issued < i + depth) {
                const int s = issued % 8;
                mbar_arrive_expect_tx(&full[s], 16384);
                int row = l2_rows ? (issued * 128) % l2_rows : ((blockIdx.x * tiles + issued) * 128) % rows_total;
                issue_t[s] = clock64();
                tma_load_2d(smem + s * 16384, &m, &full[s], 0, row, kEvictFirst);
                ++issued;
            }
            const int s = i % 8;
            mbar_wait(&full[s], (i / 8) & 1);
            lat += clock64() - issue_t[s];
        }
        const long long t1 = clock64();
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = lat / tiles;
    }
}

int main() {
    const long long rows = 1ll << 22;  // 4M rows x 64 bf16 = 512 MB
    void* buf;
    cudaMalloc(&buf, rows * 128);
    cudaMemset(buf, 0, rows * 128);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
    CUtensorMap m;
    cuuint64_t dims[2] = {64, cuuint64_t(rows)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 2048);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 16);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("tiles of 16 KB; GB/s per SM and mean issue->landed latency (us)\n");
    for (int l2 : {0, 1}) {
        for (int ctas : {1, 20, 148}) {
            for (int depth : {1, 2, 4, 8}) {
                const int tiles = 256;
                tma_kernel<<<ctas, 128, 8 * 16384 + 2048>>>(m, tiles, depth, int(rows), l2 ? 2048 : 0, out);
                cudaDeviceSynchronize();
                tma_kernel<<<ctas, 128, 8 * 16384 + 2048>>>(m, tiles, depth, int(rows), l2 ? 2048 : 0, out);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<unsigned long long> h(ctas * 2);
                cudaMemcpy(h.data(), out, ctas * 16, cudaMemcpyDeviceToHost);
                double cyc = 0, lat = 0;
                for (int c = 0; c < ctas; ++c) {
                    cyc += h[c * 2];
                    lat += h[c * 2 + 1];
                }
                cyc /= ctas;
                lat /= ctas;
                const double us = cyc / (clk * 1e-3);
                printf("%s ctas=%3d depth=%d: %7.1f GB/s/SM (%7.1f GB/s total)  latency %6.3f us %s\n", l2 ? "L2 " : "HBM",
                       ctas, depth, tiles * 16384.0 / (us * 1e3), ctas * tiles * 16384.0 / (us * 1e3),
                       lat / (clk * 1e-3), e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
