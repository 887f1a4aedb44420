// tcgen05 / TMEM / TMA GEMM with the reference's fused epilogues.
//
// Replaces the reference's fp64 `matmul` + `apply_epilogue` pair
// (proj/src/tensor.cpp:49-67, proj/src/evaluate.cpp:160-223, 268-275) for every
// Gemm / FusedGatedGemm node of the fused pi0 graph (proj/src/builder.cpp:197-367).
//
// Structure (one CTA = one 128 x BN output tile, optionally one K-split of it):
//   warp 0      TMA producer: A tile [128 x 64] and W tile [BN x 64] per stage,
//               128-byte swizzle, mbarrier complete_tx.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16),
//               tcgen05.commit releases smem stages and finally signals the epilogue.
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused scalar ops ->
//               global (bf16 rows, or the fp32 residual stream + bf16 shadow + row
//               sum-of-squares for the next RmsScale).
// Split-K: partials are reduced with red.global.add.f32 (into the residual stream
// itself for kModeResid, else into a self-cleaning fp32 workspace); the last CTA of
// a tile (arrival counter) runs the epilogue.
#include "gemm.cuh"
#include "ptx.cuh"

namespace pi0b {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kGemmThreads = 64 + 8 * 32;  // TMA warp, MMA warp, 8 epilogue warps

template <int BN, int STAGES>
struct GemmCfg {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int BAR_BYTES = 256;
    static constexpr int SMEM = STAGES * STAGE_BYTES + BAR_BYTES + BN * 4 + 1024;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

namespace {

PI0B_DEV void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32], int nvalid) {
    if (nvalid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            uint4 u;
            u.x = pack_bf16(v[j + 0], v[j + 1]);
            u.y = pack_bf16(v[j + 2], v[j + 3]);
            u.z = pack_bf16(v[j + 4], v[j + 5]);
            u.w = pack_bf16(v[j + 6], v[j + 7]);
            *reinterpret_cast<uint4*>(dst + j) = u;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) dst[j] = __float2bfloat16_rn(v[j]);
    }
}

PI0B_DEV void store_f32x32(float* dst, const float (&v)[32], int nvalid) {
    if (nvalid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) dst[j] = v[j];
    }
}

PI0B_DEV void load_f32x32(const float* src, float (&v)[32], int nvalid, bool cg) {
    if (nvalid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            const float4 f = cg ? __ldcg(reinterpret_cast<const float4*>(src + j)) : *reinterpret_cast<const float4*>(src + j);
            v[j] = f.x; v[j + 1] = f.y; v[j + 2] = f.z; v[j + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = j < nvalid ? (cg ? __ldcg(src + j) : src[j]) : 0.f;
    }
}

// Read 32 fp32 split-K partial sums of one row from the workspace and clear them.
PI0B_DEV void ws_take32(float* src, float (&v)[32], int nvalid) {
    load_f32x32(src, v, nvalid, true);
    if (nvalid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) __stcg(reinterpret_cast<float4*>(src + j), make_float4(0.f, 0.f, 0.f, 0.f));
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) __stcg(src + j, 0.f);
    }
}

PI0B_DEV void ws_add32(float* dst, const float (&v)[32], int nvalid) {
    if (nvalid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) red_add_v4_f32(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) red_add_f32(dst + j, v[j]);
    }
}

PI0B_DEV float sumsq32(const float (&v)[32], int nvalid) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) s += j < nvalid ? v[j] * v[j] : 0.f;
    return s;
}

}  // namespace

// MODE is a GemmMode; each instantiation carries only its own epilogue so the code a
// CTA executes once (cold instruction cache) stays small.
template <int BN, int STAGES, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
    using Cfg = GemmCfg<BN, STAGES>;
    constexpr bool kPaired = MODE == kModeGate || (MODE == kModeBf16 && BN == 256);
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* accum_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_full + 1);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    float* sm_vec = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::BAR_BYTES);

    const int warp = __shfl_sync(0xffffffff, int(threadIdx.x >> 5), 0);  // warp-uniform (see below)
    const int lane = threadIdx.x & 31;
    const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
    const int KB = (p.K + BK - 1) / BK;
    const int kb0 = split * p.kb_per_split;
    const int kb1 = min(KB, kb0 + p.kb_per_split);
    const int nkb = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                const int kc = (kb0 + i) * BK;
                tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kc, m_tile * BM, kEvictLast);
                tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kc, n_tile * BN, kEvictNormal);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // Warp-uniform loop, one elected lane issues: tcgen05.mma from a divergent single-lane
        // branch costs ~270 instead of ~128 issue cycles per N=256 MMA (scripts/mma_bench.cu).
        {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint64_t ad = umma_desc_sw128(sA + s * Cfg::A_BYTES);
                const uint64_t bd = umma_desc_sw128(sB + s * Cfg::B_BYTES);
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
                    umma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(accum_full);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue (8 warps)
        // Warp w may only touch TMEM lanes [32*(w%4), +32): two warps share each lane
        // quarter and split the tile's columns (hsel).
        const int q = warp & 3;
        const int hsel = (warp - 2) >> 2;
        const int etid = threadIdx.x - 64;  // 0..255
        const int row_in_tile = q * 32 + lane;
        const int r = m_tile * BM + row_in_tile;
        const bool valid = r < p.M;
        const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
        const int n0 = n_tile * BN;
        const bool split_k = p.splits > 1;

        // Stage the per-column vector (bias or SiluBias table row), zero-padded, while the
        // mainloop runs; prefetch the row scale.
        const float* vec = MODE == kModeSiluTable ? p.table_row : ((p.flags & kFlagBias) ? p.bias : nullptr);
        for (int c = etid; c < BN; c += 256) sm_vec[c] = (vec && n0 + c < p.N) ? vec[n0 + c] : 0.f;
        float rs = 1.0f;
        if ((p.flags & kFlagRowScale) && valid) rs = 1.0f / sqrtf(p.row_stats[r] * p.inv_width + p.eps);
        named_bar_sync(1, 256);

        mbar_wait(accum_full, 0);
        tc_fence_after();

        constexpr int NC = BN / 32;                 // 32-column chunks in the tile
        constexpr int NP = NC / 2;                  // (c, c + NP) pairs
        const int c_begin = kPaired ? hsel * (NP / 2) : hsel * (NC / 2);
        const int c_end = kPaired ? c_begin + NP / 2 : c_begin + NC / 2;
        bool from_ws = false;

        if (split_k) {
            // Partial sums -> global; the last-arriving CTA of the tile finishes.
#pragma unroll 1
            for (int c = hsel * (NC / 2); c < (hsel + 1) * (NC / 2); ++c) {
                float v[32];
                tmem_ld32(trow + c * 32, v);
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (!valid || nv <= 0) continue;
                if (MODE == kModeResid) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        v[j] = p.resid_scale * (v[j] * rs + (split == 0 ? sm_vec[c * 32 + j] : 0.f));
                    ws_add32(reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0, v, nv);
                } else {
                    ws_add32(p.ws + (long long)r * p.N + col0, v, nv);
                }
            }
            __threadfence();
            named_bar_sync(1, 256);
            if (etid == 0) {
                const int tile = m_tile * gridDim.y + n_tile;
                const int prev = atomicAdd(&p.counters[tile], 1);
                const int last = prev == p.splits - 1;
                if (last) atomicExch(&p.counters[tile], 0);
                *last_flag = last;
            }
            named_bar_sync(1, 256);
            if (!*last_flag) goto epilogue_done;
            __threadfence();
            from_ws = true;
        }

        if constexpr (MODE == kModeResid) {
            // h += scale*(rs*z + b) in place (already accumulated when split), bf16 shadow, row stats.
            float ss = 0.f;
#pragma unroll 1
            for (int c = c_begin; c < c_end; ++c) {
                float v[32], h[32];
                if (!from_ws) tmem_ld32(trow + c * 32, v);
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (!valid || nv <= 0) continue;
                float* hp = reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0;
                load_f32x32(hp, h, nv, from_ws);
                if (!from_ws) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) h[j] += p.resid_scale * (v[j] * rs + sm_vec[c * 32 + j]);
                    store_f32x32(hp, h, nv);
                }
                ss += sumsq32(h, nv);
                if (p.outb)
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob + col0, h, nv);
            }
            if (valid && p.out_stats) atomicAdd(p.out_stats + r, ss);
        } else if constexpr (kPaired) {
            // Gate: tile columns [0, BN/2) are up, [BN/2, BN) the matching gate columns.
            // RoPE (BN == 256, one head per tile): pairs (j, j+128), proj/src/tensor.cpp:150-178.
            const bool rope = MODE == kModeBf16 && (p.flags & kFlagRope) && n0 < p.rope_cols;
            const float2* cs = reinterpret_cast<const float2*>(p.rope_cs) + (long long)(p.rope_pos0 + r) * 128;
#pragma unroll 1
            for (int c = c_begin; c < c_end; ++c) {
                float a[32], b[32];
                if (from_ws) {
                    if (valid) {
                        ws_take32(p.ws + (long long)r * p.N + n0 + c * 32, a, 32);
                        ws_take32(p.ws + (long long)r * p.N + n0 + (c + NP) * 32, b, 32);
                    }
                } else {
                    tmem_ld32(trow + c * 32, a);
                    tmem_ld32(trow + (c + NP) * 32, b);
                }
                if (!valid) continue;
                if (MODE == kModeGate) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) a[j] = (a[j] * rs) * gelu_tanh(b[j] * rs);
                    const int ocol0 = n_tile * (BN / 2) + c * 32;
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + ocol0, a,
                                  min(32, p.N / 2 - ocol0));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        a[j] = a[j] * rs + sm_vec[c * 32 + j];
                        b[j] = b[j] * rs + sm_vec[(c + NP) * 32 + j];
                    }
                    if (rope) {
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            const float4 t = *reinterpret_cast<const float4*>(cs + c * 32 + j);
                            const float x0 = a[j], y0 = b[j], x1 = a[j + 1], y1 = b[j + 1];
                            a[j] = x0 * t.x - y0 * t.y;
                            b[j] = x0 * t.y + y0 * t.x;
                            a[j + 1] = x1 * t.z - y1 * t.w;
                            b[j + 1] = x1 * t.w + y1 * t.z;
                        }
                    }
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + n0;
                    store_bf16x32(o + c * 32, a, min(32, p.N - (n0 + c * 32)));
                    store_bf16x32(o + (c + NP) * 32, b, min(32, p.N - (n0 + (c + NP) * 32)));
                }
            }
        } else {
            // kModeBf16 (BN < 256) / kModeF32Store / kModeSiluTable, 32 columns at a time.
            float ss = 0.f;
#pragma unroll 1
            for (int c = c_begin; c < c_end; ++c) {
                float v[32];
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (from_ws) {
                    if (valid && nv > 0) ws_take32(p.ws + (long long)r * p.N + col0, v, nv);
                } else {
                    tmem_ld32(trow + c * 32, v);
                }
                if (!valid || nv <= 0) continue;
                if constexpr (MODE == kModeSiluTable) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = silu_f(v[j] + sm_vec[c * 32 + j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = v[j] * rs + sm_vec[c * 32 + j];
                    if (MODE == kModeBf16 && (p.flags & kFlagGelu)) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
                    }
                }
                if constexpr (MODE == kModeF32Store) {
                    store_f32x32(reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0, v, nv);
                    ss += sumsq32(v, nv);
                    if (p.outb)
                        store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob + col0, v, nv);
                } else {
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + col0, v, nv);
                }
            }
            if constexpr (MODE == kModeF32Store) {
                if (valid && p.out_stats) atomicAdd(p.out_stats + r, ss);
                // Optional extra row -1 (the state token of ae.suffix,
                // proj/src/builder.cpp:311-312), written by the first tile row.
                if (p.row0_src && m_tile == 0 && row_in_tile == 0) {
                    float* o = reinterpret_cast<float*>(p.out) - p.ldo;
                    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.outb) - p.ldob;
                    float s0 = 0.f;
                    for (int j = n0 + c_begin * 32; j < min(n0 + c_end * 32, p.N); ++j) {
                        const float x = p.row0_src[j];
                        o[j] = x;
                        if (p.outb) ob[j] = __float2bfloat16_rn(x);
                        s0 += x * x;
                    }
                    if (p.out_stats) atomicAdd(p.out_stats - 1, s0);
                }
            }
        }
    epilogue_done:;
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, Cfg::TMEM_COLS);
}

// ------------------------------------------------------------------ host side

template <int BN, int STAGES, int MODE>
static cudaError_t configure_t() {
    return cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmCfg<BN, STAGES>::SMEM);
}

template <int BN, int STAGES>
static cudaError_t configure_bn() {
    cudaError_t e = configure_t<BN, STAGES, kModeBf16>();
    if (e == cudaSuccess) e = configure_t<BN, STAGES, kModeF32Store>();
    if (e == cudaSuccess) e = configure_t<BN, STAGES, kModeResid>();
    if (e == cudaSuccess) e = configure_t<BN, STAGES, kModeSiluTable>();
    return e;
}

// Must run once per device before any launch (not capturable).
cudaError_t gemm_configure() {
    cudaError_t e = configure_bn<256, 4>();
    if (e == cudaSuccess) e = configure_t<256, 4, kModeGate>();
    if (e == cudaSuccess) e = configure_bn<128, 6>();
    if (e == cudaSuccess) e = configure_bn<64, 8>();
    return e;
}

template <int BN, int STAGES, int MODE>
static cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, dim3 grid,
                            cudaStream_t stream) {
    gemm_tc_kernel<BN, STAGES, MODE><<<grid, kGemmThreads, GemmCfg<BN, STAGES>::SMEM, stream>>>(ta, tb, p);
    return cudaGetLastError();
}

template <int BN, int STAGES>
static cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, dim3 grid,
                             cudaStream_t stream) {
    switch (p.mode) {
        case kModeBf16: return launch_t<BN, STAGES, kModeBf16>(ta, tb, p, grid, stream);
        case kModeF32Store: return launch_t<BN, STAGES, kModeF32Store>(ta, tb, p, grid, stream);
        case kModeResid: return launch_t<BN, STAGES, kModeResid>(ta, tb, p, grid, stream);
        case kModeSiluTable: return launch_t<BN, STAGES, kModeSiluTable>(ta, tb, p, grid, stream);
        case kModeGate:
            if constexpr (BN == 256) return launch_t<BN, STAGES, kModeGate>(ta, tb, p, grid, stream);
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gemm(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                        cudaStream_t stream) {
    if ((p.flags & kFlagRope) && bn != 256) return cudaErrorInvalidValue;
    const dim3 grid((p.M + BM - 1) / BM, (p.N + bn - 1) / bn, p.splits);
    switch (bn) {
        case 256: return launch_bn<256, 4>(ta, tb, p, grid, stream);
        case 128: return launch_bn<128, 6>(ta, tb, p, grid, stream);
        case 64: return launch_bn<64, 8>(ta, tb, p, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
