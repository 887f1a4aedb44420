// Microbenchmark: staging the fp32 residual stream y [64 x 1024] (L2-resident, 256 KB) into
// shared memory in 16 KB k-blocks, all 148 CTAs at once (2-CTA clusters) while a background warp
// per CTA streams weights from HBM (the megakernel's ae.ffn situation).
//   mode 0: per-thread coalesced cp.async (the megakernel today)
//   mode 1: one TMA 2-D box per k-block, local
//   mode 2: TMA multicast: CTA rank r loads k-blocks k % 2 == r for both CTAs of its cluster
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mcast_bench mcast_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

constexpr int kD = 4;            // fp32 ring slots (16 KB)
constexpr int kWS = 5;           // weight ring slots (16 KB)
constexpr int kKB = 16;          // k-blocks per pass
PI0B_DEV void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
PI0B_DEV void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
PI0B_DEV void arrive_remote(uint64_t* bar, uint32_t rank) {
    const uint32_t a = mapa_shared(smem_u32(bar), rank);
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}

__global__ void __launch_bounds__(288, 1) stage_kernel(const __grid_constant__ CUtensorMap ty, const float* y, const uint8_t* w,
                                                       long long wbytes, int mode, int stream, int reps,
                                                       unsigned long long* out, float* sink, volatile int* stop) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sF = smem;
    uint8_t* sW = smem + kD * 16384;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sW + kWS * 16384);
    uint64_t* full = bars;          // [kD]
    uint64_t* empty = bars + 8;     // [kD]
    uint64_t* wfull = bars + 16;    // [kWS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const uint32_t rank = cluster_ctarank();
    if (tid == 0) {
        for (int i = 0; i < kD; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], mode == 2 ? 2 : 1);
        }
        for (int i = 0; i < kWS; ++i) mbar_init(&wfull[i], 32);
        fence_barrier_init();
    }
    cluster_sync_all();
    if (warp == 8) {
      if (stream) {
        const uint8_t* base = w + (long long)blockIdx.x * wbytes;
        const long long n = wbytes / 16384;
        for (long long t = 0; t < n; ++t) {
            if (*stop) break;
            const int s = int(t % kWS);
            if (t >= kWS) mbar_wait(&wfull[s], uint32_t(((t / kWS) & 1) ^ 1));
            for (int u = 0; u < 32; ++u) cp_async16(sW + s * 16384 + u * 512 + lane * 16, base + t * 16384 + u * 512 + lane * 16, true);
            cp_async_arrive_noinc(&wfull[s]);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
      }
    } else {
    {   // let the stream ramp up
        const long long t0 = clock64();
        while (clock64() - t0 < 40000) {
        }
    }
    float acc = 0.f;
    long long t0 = 0;
    const int total = reps * kKB;
    // issue k-block i (global index over all passes) into slot i % kD
    auto issue = [&](int i) {
        if (i >= total) {
            if (mode == 0 || mode == 3) cp_async_commit();
            return;
        }
        const int s = i % kD, kb = i % kKB;
        if (mode == 0 || mode == 3) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = tid + 256 * u;
                cp_async16(sF + s * 16384 + q * 16, y + (size_t)(mode == 3 ? blockIdx.x : 0) * 65536 + (size_t)(q >> 4) * 1024 + kb * 64 + (q & 15) * 4, true);
            }
            cp_async_commit();
        } else if (tid == 0) {
            // wait until the slot's previous use was consumed (by both CTAs for multicast)
            if (i >= kD) mbar_wait(&empty[s], uint32_t(((i / kD) & 1) ^ 1));
            mbar_arrive_expect_tx(&full[s], 16384);
            if (mode == 1) tma_load_2d(sF + s * 16384, &ty, &full[s], kb * 64, 0, kEvictNormal);
            else if ((kb & 1) == int(rank)) tma_load_2d_mc(sF + s * 16384, &ty, &full[s], kb * 64, 0, 0x3);
        }
    };
    for (int i = 0; i < kD - 1; ++i) issue(i);
    for (int i = 0; i < total; ++i) {
        if (i == kKB) t0 = clock64();  // skip the first pass (ramp)
        issue(i + kD - 1);
        const int s = i % kD;
        if (mode == 0 || mode == 3) {
            cp_async_wait<kD - 1>();
            named_bar_sync(1, 256);
        } else {
            mbar_wait(&full[s], uint32_t((i / kD) & 1));
        }
        // consume: every thread reads 64 B of the slot
        const float4* f = reinterpret_cast<const float4*>(sF + s * 16384);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float4 v = f[tid + 256 * u];
            acc += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        }
        named_bar_sync(1, 256);
        if (mode != 0 && mode != 3 && tid == 0) {
            mbar_arrive(&empty[s]);
            if (mode == 2) arrive_remote(&empty[s], rank ^ 1u);
        }
    }
    const long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    sink[blockIdx.x * 256 + tid] = acc;
    named_bar_sync(1, 256);
    if (tid == 0) *stop = 1;
    }
    // keep the partner's multicast targets alive until both are done
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                   const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int G = 148;
    const long long wbytes = 128ll << 20;
    float* y;
    cudaMalloc(&y, 148ll * 64 * 1024 * 4);
    cudaMemset(y, 0, 148ll * 64 * 1024 * 4);
    uint8_t* w;
    cudaMalloc(&w, wbytes * G);
    unsigned long long* out;
    cudaMalloc(&out, G * 8);
    float* sink;
    cudaMalloc(&sink, G * 256 * 4);
    int* stop;
    cudaMalloc(&stop, 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap ty;
    cuuint64_t dims[2] = {1024, 64}, strides[1] = {1024 * 4};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(&ty, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es,
                                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", int(r));
        return 1;
    }
    const int smem = (kD + kWS) * 16384 + 1024 + 512;
    cudaFuncSetAttribute(stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* names[] = {"cp.async coalesced", "TMA box local", "TMA multicast x2", "cp.async, y per CTA"};
    const int reps = 20;
    for (int stream = 0; stream < 2; ++stream)
        for (int mode = 0; mode < 4; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(stop, 0, 4);
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(G);
                cfg.blockDim = dim3(288);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 2;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, stage_kernel, ty, (const float*)y, (const uint8_t*)w, wbytes, mode, stream, reps, out, sink,
                                   (volatile int*)stop);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<unsigned long long> h(G);
                cudaMemcpy(h.data(), out, G * 8, cudaMemcpyDeviceToHost);
                double m = 0, mx = 0;
                for (auto v : h) {
                    m += v;
                    mx = v > mx ? v : mx;
                }
                m /= G;
                const double ns = m / (clk * 1e-6) / ((reps - 1) * kKB);
                if (rep == 1)
                    printf("stream=%d %-20s %7.1f ns per 16 KB k-block (%5.1f GB/s per SM, max CTA %7.1f ns) %s\n", stream,
                           names[mode], ns, 16384 / ns, mx / (clk * 1e-6) / ((reps - 1) * kKB), e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    return 0;
}
