// Microbenchmark: end-to-end publish latency between two SMs while every SM streams weights
// from HBM in the background (the megakernel's situation).  CTA i and CTA i + G/2 ping-pong:
// each side writes 8 KB of data with 256 threads, bar.sync, one thread publishes a flag; the
// partner polls the flag (relaxed + acquire fence), checks the data, and answers.  Reported:
// half the round trip (= data write + publish + detection), averaged over rounds and pairs.
//   background stream  0: none   1: warp-wide cp.async 16 B (megakernel)   2: cp.async.bulk 16 KB
//   publish            0: red.release.gpu   1: fence.acq_rel.gpu + red.relaxed   2: st.release.gpu flag
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o publish_bench publish_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "../paper_2510_26742_b200/csrc/ptx.cuh"

using namespace pi0b;

PI0B_DEV void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
PI0B_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
PI0B_DEV unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kSlots = 5, kSlot = 16384;

__global__ void __launch_bounds__(288, 1) pp_kernel(const uint8_t* w, long long wbytes, int stream, int pub,
                                                    unsigned* flags, uint4* data, int rounds, unsigned long long* out,
                                                    volatile int* stop, int dmode) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSlots * kSlot);
    uint64_t* empty = full + 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, half = G / 2;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&full[i], stream == 1 ? 32 : 1);
            mbar_init(&empty[i], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 8) {
        // background weight stream; a consumer lane frees each slot as soon as it lands
        if (!stream) return;
        const uint8_t* base = w + (long long)blockIdx.x * wbytes;
        const long long n = wbytes / kSlot;
        for (long long t = 0; t < n; ++t) {
            if (*stop) break;
            const int s = int(t % kSlots);
            const uint32_t ph = uint32_t((t / kSlots) & 1);
            if (t >= kSlots) {
                mbar_wait(&full[s], ph ^ 1);  // landed (we are also the consumer)
            }
            if (stream == 1) {
                for (int u = 0; u < kSlot / 512; ++u)
                    cp_async16(smem + s * kSlot + u * 512 + lane * 16, base + t * kSlot + u * 512 + lane * 16, true);
                cp_async_arrive_noinc(&full[s]);
            } else {
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[s], kSlot);
                    bulk_g2s(smem + s * kSlot, base + t * kSlot, kSlot, &full[s], kEvictFirst);
                }
                __syncwarp();
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }
    // warps 0..7: ping-pong
    const int me = blockIdx.x, partner = me < half ? me + half : me - half;
    const bool initiator = me < half;
    const int tid = threadIdx.x;
    {   // let the stream ramp up
        const long long t0 = clock64();
        while (clock64() - t0 < 40000) {
        }
    }
    unsigned* myflag = flags + me * 32;
    unsigned* pflag = flags + partner * 32;
    uint4* mydata = data + (size_t)me * 512;
    const uint4* pdata = data + (size_t)partner * 512;
    unsigned long long t_begin = 0;
    int bad = 0;
    for (int r = 0; r < rounds; ++r) {
        if (!(initiator && r == 0)) {
            // wait for the partner's round r (initiator: r-1 answered)
            const unsigned target = initiator ? unsigned(r) : unsigned(r + 1);
            if (tid == 0) {
                if (pub >= 10) {
                    while (ld_acquire(pflag) < target) {
                    }
                } else {
                    while (ld_relaxed(pflag) < target) {
                    }
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
            }
            named_bar_sync(1, 256);
            if (dmode == 0) {
                const uint4 v = __ldcg(pdata + tid * 2);
                if (v.x != target) ++bad;
            }
        }
        if (initiator && r == 1 && tid == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        }
        const unsigned tag = initiator ? unsigned(r + 1) : unsigned(r + 1);
        if (dmode != 1) {
            mydata[tid * 2] = make_uint4(tag, tag, tag, tag);
            mydata[tid * 2 + 1] = make_uint4(tag, tag, tag, tag);
        }
        named_bar_sync(1, 256);
        if (tid == 0) {
            if (pub == 0 || pub == 10) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myflag) : "memory");
            } else if (pub == 1) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(myflag) : "memory");
            } else {
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(myflag), "r"(unsigned(r + 1)) : "memory");
            }
        }
    }
    if (initiator && tid == 0) {
        // wait for the last answer
        while (ld_relaxed(pflag) < unsigned(rounds)) {
        }
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        out[me] = (t_end - t_begin) / (2ull * (rounds - 1));
        out[G + me] = bad;
    }
    named_bar_sync(1, 256);
    if (tid == 0 && initiator) *stop = 1;
}

int main(int argc, char** argv) {
    const int s_lo = argc > 1 ? atoi(argv[1]) : 0, s_hi = argc > 2 ? atoi(argv[2]) : 2;
    const int G = 148;
    const long long wbytes = 256ll << 20;  // per CTA (never exhausted within the rounds)
    uint8_t* w;
    if (cudaMalloc(&w, wbytes * G) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    unsigned* flags;
    uint4* data;
    unsigned long long* out;
    int* stop;
    cudaMalloc(&flags, G * 32 * 4);
    cudaMalloc(&data, (size_t)G * 512 * 16);
    cudaMalloc(&out, 2 * G * 8);
    cudaMalloc(&stop, 4);
    const int smem = kSlots * kSlot + 1024 + 256;
    cudaFuncSetAttribute(pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* sn[] = {"none", "cp.async", "bulk"};
    const char* pn[] = {"red.release", "fence+red", "st.release"};
    const int rounds = 200;
    const char* dn[] = {"write+read 8KB", "flag only", "write only"};
    for (int dmode = 0; dmode < 3; ++dmode)
    for (int stream = s_lo; stream <= s_hi; ++stream)
        for (int pub : {0, 10}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(flags, 0, G * 32 * 4);
                cudaMemset(data, 0, (size_t)G * 512 * 16);
                cudaMemset(stop, 0, 4);
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                pp_kernel<<<G, 288, smem>>>(w, wbytes, stream, pub, flags, data, rounds, out, stop, dmode);
                cudaEventRecord(b);
                cudaError_t e = cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                std::vector<unsigned long long> h(2 * G);
                cudaMemcpy(h.data(), out, 2 * G * 8, cudaMemcpyDeviceToHost);
                double m = 0, mx = 0;
                unsigned long long bad = 0;
                for (int i = 0; i < G / 2; ++i) {
                    m += h[i];
                    mx = h[i] > mx ? h[i] : mx;
                    bad += h[G + i];
                }
                m /= (G / 2);
                if (rep == 1)
                    printf("%-15s stream=%-8s publish=%-12s one-way %6.3f us (max pair %6.3f)  kernel %.3f ms  HBM %.0f GB/s  bad=%llu %s\n",
                           dn[dmode], sn[stream], pub == 10 ? "red.rel/ld.acq" : pn[pub], m * 1e-3, mx * 1e-3, ms, 0.0, bad, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    return 0;
}
