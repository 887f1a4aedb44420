// Microbenchmark: latency of dependent global loads (L2-resident) issued by one warp while another
// warp of the same CTA streams 16 KB weight tiles from HBM (cp.async ring, or TMA ring), and the
// issue time of a 16 KB cp.async tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o colat_bench colat_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

PI0B_DEV void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// stream: 0 none, 1 cp.async ring (depth tiles), 2 TMA ring (depth tiles)
__global__ void __launch_bounds__(256, 1) colat(const __grid_constant__ CUtensorMap m, const uint8_t* wsrc, long long wbytes,
                                                int stream, int depth, const unsigned* chain, unsigned* sink,
                                                unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 8 * 16384);
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        done = 0;
        for (int i = 0; i < 8; ++i) mbar_init(&full[i], stream == 1 ? 32 : 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (stream == 0) return;
        const uint8_t* base = wsrc + (long long)blockIdx.x * wbytes;
        const long long n = wbytes / 16384;
        long long issue_cyc = 0, issued = 0;
        for (long long t = 0; t < n && !done; ++t) {
            const int s = int(t % depth);
            if (t >= depth) mbar_wait(&full[s], ((t - depth) / depth) & 1);
            const long long a = clock64();
            if (stream == 1) {
                for (int u = 0; u < 32; ++u)
                    cp_async16(smem + s * 16384 + (lane + 32 * u) * 16, base + t * 16384 + (lane + 32 * u) * 16, true);
                cp_async_arrive_noinc(&full[s]);
            } else if (lane == 0) {
                mbar_arrive_expect_tx(&full[s], 16384);
                tma_load_2d(smem + s * 16384, &m, &full[s], 0, int(((long long)blockIdx.x * n + t) * 128 % (1 << 22)), kEvictFirst);
            }
            issue_cyc += clock64() - a;
            ++issued;
        }
        if (lane == 0) out[blockIdx.x * 4 + 2] = issued ? issue_cyc / issued : 0;
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == 4) {
        const long long t0 = clock64();
        while (clock64() - t0 < 40000) {
        }
        // pointer chase through an L2-resident table (distinct lines)
        unsigned idx = blockIdx.x * 64 + lane;
        const long long a = clock64();
        const int reps = 64;
        for (int r = 0; r < reps; ++r) idx = __ldcg(chain + idx);
        const long long b = clock64();
        if (lane == 0) {
            out[blockIdx.x * 4] = (b - a) / reps;
            sink[blockIdx.x] = idx;
            done = 1;
        }
    }
}

int main() {
    const long long wbytes = 32ll << 20;
    uint8_t* w;
    cudaMalloc(&w, wbytes * 148);
    const int nchain = 1 << 20;
    std::vector<unsigned> h(nchain);
    for (int i = 0; i < nchain; ++i) h[i] = (unsigned)((i * 2654435761u + 12345u) % nchain) & ~31u;  // lines 128 B apart
    unsigned* chain;
    cudaMalloc(&chain, nchain * 4);
    cudaMemcpy(chain, h.data(), nchain * 4, cudaMemcpyHostToDevice);
    unsigned* sink;
    cudaMalloc(&sink, 148 * 4);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 32);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
    CUtensorMap m;
    cuuint64_t dims[2] = {64, 1ull << 22};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(colat, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 2048);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* sn[] = {"no stream", "cp.async ring", "TMA ring"};
    for (int ctas : {1, 148})
        for (int stream : {0, 1, 2})
            for (int depth : {2, 5, 8}) {
                if (stream == 0 && depth != 2) continue;
                colat<<<ctas, 256, 8 * 16384 + 2048>>>(m, w, wbytes, stream, depth, chain, sink, out);
                colat<<<ctas, 256, 8 * 16384 + 2048>>>(m, w, wbytes, stream, depth, chain, sink, out);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<unsigned long long> o(ctas * 4);
                cudaMemcpy(o.data(), out, ctas * 32, cudaMemcpyDeviceToHost);
                double lat = 0, iss = 0;
                for (int c = 0; c < ctas; ++c) {
                    lat += o[c * 4];
                    iss += o[c * 4 + 2];
                }
                printf("ctas=%3d %-14s depth=%d: dependent L2 load %6.3f us, tile issue %6.3f us %s\n", ctas, sn[stream],
                       depth, lat / ctas / (clk * 1e-3), iss / ctas / (clk * 1e-3), e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
