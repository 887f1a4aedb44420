// GEMM epilogue store patterns: how long does one CTA take to write its 128-row x 128-column bf16
// output tile (rows `ld` bytes apart, like ve.qkv's 6912 B) when every CTA of a 148-CTA grid does
// it at once?  Each thread holds one row's 64 columns (the tcgen05.ld 32x32b layout: 8 warps,
// warp w rows 32 (w % 4) + lane, column half w / 4).
//   0 per-thread row pieces: 8 x 16-byte st.global per thread (a warp instruction = 32 rows)
//   1 staged in shared memory (bf16, swizzled), then coalesced: a warp instruction = 2 rows x 256 B
//   2 staged, then one 256-byte cp.async.bulk per row (128 threads)
//   3 staged, then one 2D TMA tensor store of the whole tile (one thread)
//   4 no stores (baseline: launch + fill + register work)
// Kernel time by CUDA events over 200 back-to-back launches; also the per-CTA issue span.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/esb scripts/epi_store_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(uint8_t* out, int ld, unsigned long long* ts, const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(1024) uint8_t tile[];  // [128 rows][256 B], 16-byte pieces swizzled by row
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = (warp & 3) * 32 + lane, half = warp >> 2;
    float v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = float(row * 64 + j + blockIdx.x);
    __syncthreads();
    const unsigned long long t0 = gt();
    uint8_t* base = out + (size_t)blockIdx.x * 128 * ld;  // this CTA's tile: rows ld apart
    if (MODE == 0) {
        uint4* dst = reinterpret_cast<uint4*>(base + (size_t)row * ld + half * 128);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            dst[q] = make_uint4(pack(v[8 * q], v[8 * q + 1]), pack(v[8 * q + 2], v[8 * q + 3]), pack(v[8 * q + 4], v[8 * q + 5]),
                                pack(v[8 * q + 6], v[8 * q + 7]));
    } else if (MODE >= 1 && MODE <= 3) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int piece = half * 8 + q;  // 16 pieces of 16 B per 256-byte row
            const int sp = MODE == 3 ? piece : (piece ^ (row & 15));
            *reinterpret_cast<uint4*>(tile + row * 256 + sp * 16) =
                make_uint4(pack(v[8 * q], v[8 * q + 1]), pack(v[8 * q + 2], v[8 * q + 3]), pack(v[8 * q + 4], v[8 * q + 5]),
                           pack(v[8 * q + 6], v[8 * q + 7]));
        }
        if (MODE == 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (MODE == 1) {
            for (int e = threadIdx.x; e < 128 * 16; e += 256) {
                const int r = e >> 4, pc = e & 15;
                *reinterpret_cast<uint4*>(base + (size_t)r * ld + pc * 16) = *reinterpret_cast<const uint4*>(tile + r * 256 + ((pc ^ (r & 15)) * 16));
            }
        } else if (MODE == 2) {
            if (threadIdx.x < 128) {  // (unswizzled rows would be needed for a straight bulk copy: timing only)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;" ::"l"(base + (size_t)threadIdx.x * ld),
                             "r"((uint32_t)__cvta_generic_to_shared(tile + threadIdx.x * 256)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        } else {
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm), "r"(0),
                             "r"(int(blockIdx.x) * 128), "r"((uint32_t)__cvta_generic_to_shared(tile)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        }
    } else {
        if (v[row & 63] == -1.f) base[row] = 1;  // keep v alive
    }
    __syncthreads();
    const unsigned long long t1 = gt();
    if (threadIdx.x == 0) {
        ts[blockIdx.x * 2] = t0;
        ts[blockIdx.x * 2 + 1] = t1;
    }
}

template <int MODE>
void run(const char* name, uint8_t* out, int ld, unsigned long long* ts, const CUtensorMap& tm, int grid) {
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 20; ++i) k<MODE><<<grid, 256, 200 * 1024>>>(out, ld, ts, tm);
    cudaEventRecord(a);
    for (int i = 0; i < 200; ++i) k<MODE><<<grid, 256, 200 * 1024>>>(out, ld, ts, tm);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2 * 148];
    cudaMemcpy(h, ts, grid * 16, cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (int i = 0; i < grid; ++i) {
        const double d = (h[2 * i + 1] - h[2 * i]) * 1e-3;
        sum += d;
        mx = d > mx ? d : mx;
    }
    printf("%-34s grid %3d: %.2f us/launch, per-CTA issue span mean %.2f max %.2f us (%s)\n", name, grid, ms * 1e3 / 200, sum / grid,
           mx, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int ld = 6912;
    uint8_t* out;
    unsigned long long* ts;
    cudaMalloc(&out, (size_t)148 * 128 * ld);
    cudaMalloc(&ts, 148 * 16);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, 148 * 128};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map: %d\n", int(r));
    for (int grid : {108, 148}) {
        run<4>("no stores", out, ld, ts, tm, grid);
        run<0>("per-thread rows (8 x 16 B)", out, ld, ts, tm, grid);
        run<1>("staged, coalesced 2 rows x 256 B", out, ld, ts, tm, grid);
        run<2>("staged, bulk copy per row", out, ld, ts, tm, grid);
        run<3>("staged, one TMA tensor store", out, ld, ts, tm, grid);
    }
}
