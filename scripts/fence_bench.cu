// Microbenchmark: latency of publishing a flag (fence + atomic) from one warp while another warp
// of the same CTA streams weights with cp.async (or TMA), vs an idle SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fence_bench fence_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

PI0B_DEV void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// mode: 0 fence.sc.gpu + atom; 1 fence.acq_rel.gpu + atom; 2 red.release.gpu only; 3 atom.acq_rel only
__global__ void __launch_bounds__(128, 1) fence_kernel(const uint8_t* src, long long bytes, int stream, int mode,
                                                       unsigned* flag, float* sink, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 4 * 16384);
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        done = 0;
        for (int i = 0; i < 4; ++i) mbar_init(&full[i], 32);
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (!stream) return;
        const uint8_t* base = src + (long long)blockIdx.x * bytes;
        const long long n = bytes / 16384;
        for (long long t = 0; t < n && !done; ++t) {
            const int s = int(t & 3);
            if (t >= 4) mbar_wait(&full[s], ((t - 4) >> 2) & 1);
            for (int u = 0; u < 32; ++u) cp_async16(smem + s * 16384 + (lane + 32 * u) * 16, base + t * 16384 + (lane + 32 * u) * 16, true);
            cp_async_arrive_noinc(&full[s]);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == 2) {
        // let the stream ramp up
        const long long t0 = clock64();
        while (clock64() - t0 < 20000) {
        }
        unsigned long long acc = 0;
        const int reps = 32;
        for (int r = 0; r < reps; ++r) {
            if (lane == 0) sink[blockIdx.x * 32 + r] = float(r);  // a store to publish
            __syncwarp();
            const long long a = clock64();
            if (lane == 0) {
                unsigned* f = flag + blockIdx.x * 32;
                if (mode == 0) {
                    __threadfence();
                    atomicAdd(f, 1u);
                } else if (mode == 1) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    atomicAdd(f, 1u);
                } else if (mode == 2) {
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(f) : "memory");
                } else {
                    unsigned old;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(f) : "memory");
                }
            }
            __syncwarp();
            acc += clock64() - a;
        }
        if (lane == 0) {
            out[blockIdx.x] = acc / reps;
            done = 1;
        }
    }
}

int main() {
    const long long bytes = 64ll << 20;
    uint8_t* src;
    cudaMalloc(&src, bytes * 148);
    unsigned* flag;
    cudaMalloc(&flag, 148 * 32 * 4);
    float* sink;
    cudaMalloc(&sink, 148 * 32 * 4);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8);
    cudaFuncSetAttribute(fence_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 2048);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* names[] = {"fence.sc.gpu + atomicAdd", "fence.acq_rel.gpu + atomicAdd", "red.release.gpu", "atom.acq_rel.gpu"};
    for (int ctas : {1, 148})
        for (int stream : {0, 1})
            for (int mode = 0; mode < 4; ++mode) {
                fence_kernel<<<ctas, 128, 4 * 16384 + 2048>>>(src, bytes / 64, stream, mode, flag, sink, out);
                fence_kernel<<<ctas, 128, 4 * 16384 + 2048>>>(src, bytes / 64, stream, mode, flag, sink, out);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<unsigned long long> h(ctas);
                cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
                double m = 0;
                for (auto v : h) m += v;
                m /= ctas;
                printf("ctas=%3d stream=%d %-32s %7.3f us %s\n", ctas, stream, names[mode], m / (clk * 1e-3),
                       e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
