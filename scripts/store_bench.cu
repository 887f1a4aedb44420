// How fast can one CTA write a 128-row x 512-byte output tile (64 KB, rows 4 KB apart) to global
// memory?  256 threads, coalesced 16-byte stores (plain / .cs / .cg) vs one 64 KB bulk store from
// shared memory.  Per-CTA globaltimer spans; grid = 32 or 128 CTAs.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int MODE>
__global__ void k(uint4* out, unsigned long long* ts) {
    extern __shared__ __align__(128) uint4 tile[];
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) tile[i] = make_uint4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    const unsigned long long t0 = gt();
    uint4* base = out + (size_t)blockIdx.x * 128 * 256;  // 128 rows x 4096 B per CTA
    if (MODE < 3) {
        for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
            const int r = e >> 5, q = e & 31;
            uint4 v = tile[e];
            uint4* dst = base + r * 256 + q;
            if (MODE == 0) *dst = v;
            else if (MODE == 1) __stcs(dst, v);
            else __stcg(dst, v);
        }
    } else {
        if (threadIdx.x < 128) {  // one 512-byte bulk store per row
            const int r = threadIdx.x;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(base + r * 256),
                         "r"((uint32_t)__cvta_generic_to_shared(tile + r * 32)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
    __syncthreads();
    const unsigned long long t1 = gt();
    if (threadIdx.x == 0) { ts[blockIdx.x * 2] = t0; ts[blockIdx.x * 2 + 1] = t1; }
}
int main() {
    uint4* out; unsigned long long* ts;
    cudaMalloc(&out, 148ull * 128 * 4096);
    cudaMalloc(&ts, 148 * 2 * 8);
    unsigned long long h[296];
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const char* names[] = {"st.global", "st.global.cs", "st.global.cg", "bulk store"};
    for (int grid : {32, 128}) for (int m = 0; m < 4; ++m) {
        for (int rep = 0; rep < 3; ++rep) {
            if (m == 0) k<0><<<grid, 256, 65536>>>(out, ts);
            if (m == 1) k<1><<<grid, 256, 65536>>>(out, ts);
            if (m == 2) k<2><<<grid, 256, 65536>>>(out, ts);
            if (m == 3) k<3><<<grid, 256, 65536>>>(out, ts);
        }
        cudaDeviceSynchronize();
        cudaMemcpy(h, ts, grid * 16, cudaMemcpyDeviceToHost);
        double mx = 0, sum = 0;
        for (int b = 0; b < grid; ++b) { double d = (h[2 * b + 1] - h[2 * b]) * 1e-3; sum += d; if (d > mx) mx = d; }
        printf("grid %3d %-13s per-CTA 64 KB: mean %.2f us, max %.2f us  (%s)\n", grid, names[m], sum / grid, mx,
               cudaGetErrorString(cudaGetLastError()));
    }
}
