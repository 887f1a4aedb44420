// DSMEM push bandwidth: every CTA of a cluster (1 CTA per SM, 148 CTAs) pushes B bytes into each
// peer's shared memory with st.async (256 threads, 16 B each, completing on the peer's mbarrier),
// then waits for the B * (C - 1) bytes pushed into it.  Per-CTA time from start to all received
// (globaltimer).  Compared with 256 threads cp.async-loading the same bytes from L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o dsmem_bench dsmem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void st_async4(uint32_t addr, uint4 v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(addr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ uint32_t crank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cnum() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

template <int MODE>  // 0: DSMEM push, 1: L2 cp.async load
__global__ void k(int bytes, const uint4* src, unsigned long long* ts) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t C = cnum(), me = crank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    cluster_sync_all();
    if (threadIdx.x == 0 && MODE == 0) mbar_arrive_expect_tx(&bar, uint32_t(bytes) * (C - 1));
    cluster_sync_all();
    const unsigned long long t0 = gt();
    if (MODE == 0) {
        for (uint32_t p = 1; p < C; ++p) {
            const uint32_t peer = (me + p) % C;
            const uint32_t base = mapa(smem_u32(sm + (p - 1) * bytes), peer), rb = mapa(smem_u32(&bar), peer);
            for (int o = threadIdx.x * 16; o < bytes; o += blockDim.x * 16)
                st_async4(base + o, make_uint4(o, p, me, 1), rb);
        }
        mbar_wait(&bar, 0);
    } else {
        const uint8_t* s = reinterpret_cast<const uint8_t*>(src) + (size_t)(blockIdx.x % 8) * bytes * 4;
        const int total = bytes * (C - 1);
        for (int o = threadIdx.x * 16; o < total; o += blockDim.x * 16) cp_async16(sm + o, s + o, true);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    }
    const unsigned long long t1 = gt();
    if (threadIdx.x == 0) ts[blockIdx.x] = t1 - t0;
    cluster_sync_all();
}

template <int MODE>
void run(int C, int bytes, const uint4* src, unsigned long long* d) {
    const int smem = bytes * (C - 1) + 1024;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148 / C * C);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = C;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    for (int it = 0; it < 3; ++it) cudaLaunchKernelEx(&cfg, k<MODE>, bytes, src, d);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148);
    cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
    const int n = 148 / C * C;
    double mx = 0, sum = 0;
    for (int i = 0; i < n; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        sum += h[i];
    }
    const double recv = double(bytes) * (C - 1);
    printf("%s cluster %d: %6d B to each peer (%6.0f KB in per CTA): mean %6.2f us max %6.2f us -> %6.1f GB/s per SM (%s)\n",
           MODE == 0 ? "DSMEM push" : "L2 cp.async", C, bytes, recv / 1024, sum / n / 1e3, mx / 1e3, recv / (sum / n),
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    uint4* src;
    cudaMalloc(&src, 64 << 20);
    cudaMemset(src, 1, 64 << 20);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    for (int C : {2, 4, 8})
        for (int b : {8192, 16384, 32768}) {
            if (b * (C - 1) > 200 * 1024) continue;
            run<0>(C, b, src, d);
            run<1>(C, b, src, d);
        }
}
