// Megakernel residual updates: how long until a split-K partial tile (64 rows x 128 fp32 = 32 KB,
// in shared memory) has been added into the fp32 residual stream and published?  128 producer
// CTAs (one per SM), 16 of them per 128-column block (16-way split-K), plus one watcher CTA that
// polls the phase counter.
//   0 per-thread rows: 128 threads, red.global.add.v4.f32 (the megakernel's kEpiRed today)
//   1 bulk reduce: 64 threads, one cp.reduce.async.bulk .add.f32 of 512 B per row, wait_group 0
//   2 bulk reduce, 64 rows issued by one thread
//   3 as 1 + fence.proxy.async.global before the release
// Each CTA: bar.sync, then thread 0 red.release.gpu on the counter.  Reported: producer span
// (start -> release issued), watcher span (start -> counter complete), and a checksum.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bulkred_bench scripts/bulkred_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kProducers = 128;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(float* y, unsigned* ctr, const unsigned long long* go, unsigned long long* ts) {
    extern __shared__ __align__(1024) float tile[];  // [64 rows][128]
    const int tid = threadIdx.x;
    if (blockIdx.x == kProducers) {  // watcher
        if (tid == 0) {
            while (*(volatile const unsigned long long*)go == 0) {
            }
            const unsigned long long t0 = gt();
            while (ld_acquire(ctr) < kProducers) {
            }
            ts[2 * kProducers] = t0;
            ts[2 * kProducers + 1] = gt();
        }
        return;
    }
    for (int i = tid; i < 64 * 128; i += 256) tile[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        if (blockIdx.x == 0) *(volatile unsigned long long*)go = 1;
        while (*(volatile const unsigned long long*)go == 0) {
        }
    }
    __syncthreads();
    const unsigned long long t0 = gt();
    const int blk = blockIdx.x % 8;  // 8 column blocks of 128 -> 16 producers each
    float* ybase = y + blk * 128;    // y is [64][1024]
    if (MODE == 0) {
        if (tid < 128) {
            const int r = tid & 63, h = tid >> 6;
            float* dst = ybase + r * 1024 + h * 64;
            const float* src = tile + r * 128 + h * 64;
#pragma unroll 1
            for (int q = 0; q < 16; ++q)
                asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + 4 * q), "f"(src[4 * q]), "f"(src[4 * q + 1]),
                             "f"(src[4 * q + 2]), "f"(src[4 * q + 3]) : "memory");
        }
    } else if (MODE == 1 || MODE == 3) {
        if (tid < 64) {
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;" ::"l"(ybase + tid * 1024),
                         "r"((uint32_t)__cvta_generic_to_shared(tile + tid * 128)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            if (MODE == 3) asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    } else {
        if (tid == 0) {
            for (int r = 0; r < 64; ++r)
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;" ::"l"(ybase + r * 1024),
                             "r"((uint32_t)__cvta_generic_to_shared(tile + r * 128)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        ts[2 * blockIdx.x] = t0;
        ts[2 * blockIdx.x + 1] = gt();
    }
}

template <int MODE>
void run(const char* name) {
    float* y;
    unsigned* ctr;
    unsigned long long *go, *ts;
    cudaMalloc(&y, 64 * 1024 * 4);
    cudaMalloc(&ctr, 4);
    cudaMalloc(&go, 8);
    cudaMalloc(&ts, (2 * kProducers + 2) * 8);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    std::vector<double> prod, watch;
    bool ok = true;
    for (int it = 0; it < 20; ++it) {
        cudaMemset(y, 0, 64 * 1024 * 4);
        cudaMemset(ctr, 0, 4);
        cudaMemset(go, 0, 8);
        k<MODE><<<kProducers + 1, 256, 200 * 1024>>>(y, ctr, go, ts);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(2 * kProducers + 2);
        cudaMemcpy(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<float> hy(64 * 1024);
        cudaMemcpy(hy.data(), y, hy.size() * 4, cudaMemcpyDeviceToHost);
        for (float v : hy) ok &= v == 16.0f;
        double mx = 0;
        for (int b = 0; b < kProducers; ++b) mx = std::max(mx, (h[2 * b + 1] - h[2 * b]) * 1e-3);
        if (it >= 5) {
            prod.push_back(mx);
            watch.push_back((h[2 * kProducers + 1] - h[2 * kProducers]) * 1e-3);
        }
    }
    auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    printf("%-40s producer max span %.2f us, watcher %.2f us, sums %s (%s)\n", name, med(prod), med(watch), ok ? "ok" : "WRONG",
           cudaGetErrorString(cudaGetLastError()));
}

#include <algorithm>
int main() {
    run<0>("per-thread rows, red.add.v4");
    run<1>("bulk reduce, 64 threads x 512 B");
    run<2>("bulk reduce, one thread x 64 rows");
    run<3>("bulk reduce + fence.proxy.async.global");
    run<0>("per-thread rows, red.add.v4 (again)");
}
