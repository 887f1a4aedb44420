// Per-SM TMA ingest vs box size: each CTA streams `tiles` tiles of 32 KB (bf16, 128-byte swizzle,
// 64 columns x 256 rows) from an L2-resident 8 MB tensor, issued as boxes of 32 / 64 / 128 / 256
// rows, `depth` tiles in flight.  grid = 1 / 32 / 148 CTAs.  Prints GB/s per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_box_bench tma_box_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdint.h>
#include "../paper_2510_26742_b200/csrc/ptx.cuh"
using namespace pi0b;

__global__ void __launch_bounds__(64, 1) kern(const __grid_constant__ CUtensorMap m, int tiles, int depth, int box_rows,
                                               int rows_total, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 6 * 32768);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 6; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        auto issue = [&](int i) {
            const int s = i % depth;
            mbar_arrive_expect_tx(&full[s], 32768);
            const int row0 = ((blockIdx.x * 977 + i * 256) % (rows_total - 256));
            for (int r = 0; r < 256; r += box_rows)
                tma_load_2d(smem + s * 32768 + r * 128, &m, &full[s], 0, row0 + r, kEvictLast);
        };
        for (int i = 0; i < depth && i < tiles; ++i) issue(i);
        for (int i = 0; i < tiles; ++i) {
            mbar_wait(&full[i % depth], (i / depth) & 1);
            if (i + depth < tiles) issue(i + depth);
        }
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x] = t1 - t0;
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

int main() {
    const int rows = 65536;  // 64 cols x 65536 rows bf16 = 8 MB
    void* buf;
    cudaMalloc(&buf, size_t(rows) * 128);
    cudaMemset(buf, 1, size_t(rows) * 128);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
    for (int box : {32, 64, 128, 256}) {
        CUtensorMap m;
        cuuint64_t dims[2] = {64, cuuint64_t(rows)};
        cuuint64_t str[1] = {128};
        cuuint32_t bx[2] = {64, cuuint32_t(box)};
        cuuint32_t es[2] = {1, 1};
        enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int grid : {1, 32, 148})
            for (int depth : {2, 6}) {
                const int tiles = 64;
                for (int rep = 0; rep < 2; ++rep)
                    kern<<<grid, 64, 6 * 32768 + 1024>>>(m, tiles, depth, box, rows, out);
                cudaDeviceSynchronize();
                unsigned long long h[148];
                cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
                double mx = 0;
                for (int b = 0; b < grid; ++b) mx = h[b] > mx ? h[b] : mx;
                printf("box %3d rows  grid %3d  depth %d: %6.1f GB/s per SM (slowest CTA)  %s\n", box, grid, depth,
                       tiles * 32768.0 / mx, cudaGetErrorString(cudaGetLastError()));
            }
    }
}
