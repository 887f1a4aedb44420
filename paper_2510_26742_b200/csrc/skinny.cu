// Small-M ("skinny") tcgen05 GEMM for the action expert: M <= 64 activation rows against a
// large weight, HBM-bound on the weight stream (32 MAC/byte at M = 64).
//
// Replaces the reference's fp64 matmul + epilogue (proj/src/tensor.cpp:49-67,
// proj/src/evaluate.cpp:160-223) for ae.qkv / ae.proj / ae.ffn / ae.down / ae.head /
// ae.action_proj / ae.action_out / ae.state_proj (proj/src/builder.cpp:291-363).
//
// Swap-AB: the weight tile is the 128-row MMA operand (TMEM lane = output feature) and the
// activations are the N = 64 operand, so no MMA row is wasted and the activation tile is
// only 8 KB per 64-wide k-block.  A cluster of CL CTAs splits K; the fp32 partial tiles are
// reduced through distributed shared memory (each CTA owns 64/CL feature pairs), so there is
// no global atomic, workspace or arrival counter on the critical path.  Weight tiles for the
// first pipeline stages are requested before griddepcontrol.wait, i.e. they stream while
// the previous kernel drains (programmatic dependent launch).
//
// Feature pairs (f, f + 64) of a 128-row tile are co-owned, which is what the two paired
// epilogues need, given the packing of csrc/kernels_misc.cu:
//   * RoPE  (ae.qkv): packed tile = [first-half cols 64u..64u+63 | their partners +128] of a
//     256-wide head, so (j, j + 128) rotate together (proj/src/tensor.cpp:150-178);
//   * gate  (ae.ffn): packed tile = [up 64t..64t+63 | gate 64t..64t+63] (up * gelu(gate)).
#include "gemm.cuh"
#include "ptx.cuh"

namespace pi0b {

namespace {

constexpr int kSkBN = 128;   // weight rows (output features) per tile = UMMA M
constexpr int kSkRows = 64;  // activation rows = UMMA N
constexpr int kSkStages = 8;
constexpr int kSkWBytes = kSkBN * 64 * 2;
constexpr int kSkXBytes = kSkRows * 64 * 2;
constexpr int kSkStage = kSkWBytes + kSkXBytes;
constexpr int kSkXLd = 68;  // exchange row stride (floats): conflict-free float4 stores
constexpr int kSkThreads = 192;
constexpr int kSkSmem = kSkStages * kSkStage + 1024 /*bars + vectors*/ + 1024 /*align*/;

PI0B_DEV uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// Logical output column of packed tile-local feature f of tile `tile` under the RoPE permutation.
PI0B_DEV int rope_col(int tile, int f) {
    const int p = tile * kSkBN + f;
    const int h = p >> 8, w = p & 255;
    const int u = w >> 7, part = (w & 127) >> 6, l = w & 63;
    return (h << 8) + part * 128 + u * 64 + l;
}

}  // namespace

template <int MODE>
__global__ void __launch_bounds__(kSkThreads, 1)
    skinny_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                  const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSkStages * kSkStage);
    uint64_t* empty = full + kSkStages;
    uint64_t* accum_full = empty + kSkStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_full + 1);
    float* sm_rs = reinterpret_cast<float*>(smem + kSkStages * kSkStage + 256);  // [64]
    float* sm_ss = sm_rs + 64;                                                     // [64] (+1 for row -1)
    float* sm_vec = sm_ss + 68;                                                    // [128]
    float* xch = reinterpret_cast<float*>(smem);  // [128][kSkXLd] partials, aliases the ring

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int CL = int(cluster_nctarank());
    const int crank = int(cluster_ctarank());
    const int tile = blockIdx.x / CL;
    const int KB = (p.K + 63) / 64;
    const int per = (KB + CL - 1) / CL;
    const int kb0 = crank * per;
    const int nkb = max(0, min(KB, kb0 + per) - kb0);
    const int perm = p.rope_cols > 0 ? 2 : (MODE == kModeGate ? 1 : 0);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < kSkStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 64);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // weights first (independent of the producer kernel), then activations
            const int pre = min(nkb, kSkStages);
            for (int i = 0; i < pre; ++i) {
                mbar_arrive_expect_tx(&full[i], kSkStage);
                tma_load_2d(smem + i * kSkStage, &tmW, &full[i], (kb0 + i) * 64, tile * kSkBN, kEvictFirst);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i)
                tma_load_2d(smem + i * kSkStage + kSkWBytes, &tmX, &full[i], (kb0 + i) * 64, 0, kEvictLast);
            for (int i = pre; i < nkb; ++i) {
                const int s = i % kSkStages;
                mbar_wait(&empty[s], ((i / kSkStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], kSkStage);
                tma_load_2d(smem + s * kSkStage, &tmW, &full[s], (kb0 + i) * 64, tile * kSkBN, kEvictFirst);
                tma_load_2d(smem + s * kSkStage + kSkWBytes, &tmX, &full[s], (kb0 + i) * 64, 0, kEvictLast);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(kSkBN, kSkRows);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % kSkStages;
                mbar_wait(&full[s], (i / kSkStages) & 1);
                tc_fence_after();
                const uint64_t ad = umma_desc_sw128(smem + s * kSkStage);
                const uint64_t bd = umma_desc_sw128(smem + s * kSkStage + kSkWBytes);
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
                umma_commit(&empty[s]);
            }
            umma_commit(accum_full);
        }
        __syncwarp();
    } else {
        // ---- epilogue part 1: stage per-row / per-feature vectors, drain TMEM to smem
        const int et = threadIdx.x - 64;
        const int q = warp & 3;
        pdl_wait();
        if (et < 64) {
            float rs = 1.f;
            if ((p.flags & kFlagRowScale) && et < p.M) rs = 1.0f / sqrtf(p.row_stats[et] * p.inv_width + p.eps);
            sm_rs[et] = rs;
            sm_ss[et] = 0.f;
        }
        if (et == 64) sm_ss[64] = 0.f;
        {
            const float* vec = MODE == kModeSiluTable ? p.table_row : ((p.flags & kFlagBias) ? p.bias : nullptr);
            const int col = perm == 2 && tile * kSkBN < p.rope_cols ? rope_col(tile, et) : tile * kSkBN + et;
            sm_vec[et] = (vec && col < p.N) ? vec[col] : 0.f;
        }
        mbar_wait(accum_full, 0);
        tc_fence_after();
        float v0[32], v1[32];
        const uint32_t ta = tmem + (uint32_t(q * 32) << 16);
        tmem_ld32(ta, v0);
        tmem_ld32(ta + 32, v1);
        if (nkb == 0) {  // an empty K slice contributes zero (TMEM was never written)
#pragma unroll
            for (int j = 0; j < 32; ++j) v0[j] = v1[j] = 0.f;
        }
        float* xr = xch + (q * 32 + lane) * kSkXLd;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            *reinterpret_cast<float4*>(xr + j) = make_float4(v0[j], v0[j + 1], v0[j + 2], v0[j + 3]);
            *reinterpret_cast<float4*>(xr + 32 + j) = make_float4(v1[j], v1[j + 1], v1[j + 2], v1[j + 3]);
        }
        pdl_launch_dependents();
    }

    cluster_sync_all();

    if (warp >= 2) {
        // ---- epilogue part 2: this CTA owns feature pairs [crank*P, (crank+1)*P); one item =
        // (pair, 4 rows): all peer partials are fetched with 16-byte DSMEM loads before use.
        const int et = threadIdx.x - 64;
        const int P = 64 / CL;
        const int i0 = crank * P;
        const bool rope = perm == 2 && tile * kSkBN < p.rope_cols && MODE == kModeBf16;
        const uint32_t xbase = smem_u32(xch);
        for (int idx = et; idx < P * (kSkRows / 4); idx += 128) {
            const int i = i0 + idx % P;
            const int r0 = (idx / P) * 4;
            if (r0 >= p.M) continue;
            float4 pa[8], pb[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                if (s < CL) {
                    const uint32_t base = mapa_shared(xbase, uint32_t(s));
                    pa[s] = ld_dsmem_f32x4(base + uint32_t((i * kSkXLd + r0) * 4));
                    pb[s] = ld_dsmem_f32x4(base + uint32_t(((i + 64) * kSkXLd + r0) * 4));
                }
            }
            float a4[4] = {0.f, 0.f, 0.f, 0.f}, b4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                if (s < CL) {
                    a4[0] += pa[s].x; a4[1] += pa[s].y; a4[2] += pa[s].z; a4[3] += pa[s].w;
                    b4[0] += pb[s].x; b4[1] += pb[s].y; b4[2] += pb[s].z; b4[3] += pb[s].w;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = r0 + u;
                if (r >= p.M) break;
                const float a = a4[u], b = b4[u];
                const float rs = sm_rs[r];
                if constexpr (MODE == kModeGate) {
                    const int col = tile * 64 + i;
                    if (col < p.N / 2) {
                        const float g = (a * rs) * gelu_tanh(b * rs);
                        reinterpret_cast<__nv_bfloat16*>(p.out)[(long long)r * p.ldo + col] = __float2bfloat16_rn(g);
                    }
                } else if constexpr (MODE == kModeBf16) {
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo;
                    float xa = a * rs + sm_vec[i], xb = b * rs + sm_vec[i + 64];
                    if (rope) {
                        const int ca = rope_col(tile, i);
                        const float2 t = reinterpret_cast<const float2*>(p.rope_cs)[(long long)(p.rope_pos0 + r) * 128 + (ca & 255)];
                        o[ca] = __float2bfloat16_rn(xa * t.x - xb * t.y);
                        o[ca + 128] = __float2bfloat16_rn(xa * t.y + xb * t.x);
                    } else {
                        if (p.flags & kFlagGelu) {
                            xa = gelu_tanh(xa);
                            xb = gelu_tanh(xb);
                        }
                        const int fa = tile * kSkBN + i;
                        if (fa < p.N) o[fa] = __float2bfloat16_rn(xa);
                        if (fa + 64 < p.N) o[fa + 64] = __float2bfloat16_rn(xb);
                    }
                } else if constexpr (MODE == kModeSiluTable) {
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo;
                    const int fa = tile * kSkBN + i;
                    if (fa < p.N) o[fa] = __float2bfloat16_rn(silu_f(a + sm_vec[i]));
                    if (fa + 64 < p.N) o[fa + 64] = __float2bfloat16_rn(silu_f(b + sm_vec[i + 64]));
                } else {
                    // kModeResid / kModeF32Store: fp32 stream + bf16 shadow + row sum of squares
                    const int fa = tile * kSkBN + i;
                    float* h = reinterpret_cast<float*>(p.out) + (long long)r * p.ldo;
                    __nv_bfloat16* hb = reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob;
                    float ss = 0.f;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const int f = fa + half * 64;
                        if (f >= p.N) continue;
                        const float z = (half ? b : a) * rs + sm_vec[i + half * 64];
                        const float x = MODE == kModeResid ? h[f] + p.resid_scale * z : z;
                        h[f] = x;
                        if (p.outb) hb[f] = __float2bfloat16_rn(x);
                        ss += x * x;
                        if (MODE == kModeF32Store && p.row0_src && r == 0) {
                            const float x0 = p.row0_src[f];
                            h[f - p.ldo] = x0;
                            if (p.outb) hb[f - p.ldob] = __float2bfloat16_rn(x0);
                            atomicAdd(&sm_ss[64], x0 * x0);
                        }
                    }
                    if (p.out_stats) atomicAdd(&sm_ss[r], ss);
                }
            }
        }
        if constexpr (MODE == kModeResid || MODE == kModeF32Store) {
            named_bar_sync(1, 128);
            if (p.out_stats) {
                if (et < p.M) atomicAdd(p.out_stats + et, sm_ss[et]);
                if (MODE == kModeF32Store && p.row0_src && et == 64) atomicAdd(p.out_stats - 1, sm_ss[64]);
            }
        }
    }

    cluster_sync_all();  // peers may still be reading this CTA's partials
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 64);
}

// ------------------------------------------------------------------ host side

cudaError_t skinny_configure() {
    cudaError_t e = cudaSuccess;
    auto set = [&](const void* fn) {
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSkSmem);
    };
    set(reinterpret_cast<const void*>(skinny_kernel<kModeBf16>));
    set(reinterpret_cast<const void*>(skinny_kernel<kModeGate>));
    set(reinterpret_cast<const void*>(skinny_kernel<kModeF32Store>));
    set(reinterpret_cast<const void*>(skinny_kernel<kModeResid>));
    set(reinterpret_cast<const void*>(skinny_kernel<kModeSiluTable>));
    return e;
}

int skinny_tiles(int n_packed) { return (n_packed + kSkBN - 1) / kSkBN; }

// cluster = K-split factor (1..8).  pdl = launch with programmatic stream serialization.
cudaError_t launch_skinny(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p, int n_packed,
                          int cluster, bool pdl, cudaStream_t stream) {
    if (p.M > kSkRows || cluster < 1 || cluster > 8 || (64 % cluster)) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(skinny_tiles(n_packed) * cluster, 1, 1);
    cfg.blockDim = dim3(kSkThreads, 1, 1);
    cfg.dynamicSmemBytes = kSkSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    switch (p.mode) {
        case kModeBf16: return cudaLaunchKernelEx(&cfg, skinny_kernel<kModeBf16>, tw, tx, p);
        case kModeGate: return cudaLaunchKernelEx(&cfg, skinny_kernel<kModeGate>, tw, tx, p);
        case kModeF32Store: return cudaLaunchKernelEx(&cfg, skinny_kernel<kModeF32Store>, tw, tx, p);
        case kModeResid: return cudaLaunchKernelEx(&cfg, skinny_kernel<kModeResid>, tw, tx, p);
        case kModeSiluTable: return cudaLaunchKernelEx(&cfg, skinny_kernel<kModeSiluTable>, tw, tx, p);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
