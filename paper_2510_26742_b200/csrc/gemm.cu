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
constexpr int kGemmThreads = 192;

template <int BN, int STAGES>
struct GemmCfg {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
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

// Read 32 fp32 split-K partial sums of one row from the workspace and clear them.
PI0B_DEV void ws_take32(float* src, float (&v)[32], int nvalid) {
    if (nvalid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float4 f = __ldcg(reinterpret_cast<const float4*>(src + j));
            v[j] = f.x; v[j + 1] = f.y; v[j + 2] = f.z; v[j + 3] = f.w;
            __stcg(reinterpret_cast<float4*>(src + j), make_float4(0.f, 0.f, 0.f, 0.f));
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j < nvalid) {
                v[j] = __ldcg(src + j);
                __stcg(src + j, 0.f);
            } else {
                v[j] = 0.f;
            }
        }
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

}  // namespace

template <int BN, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
    using Cfg = GemmCfg<BN, STAGES>;
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

    const int warp = threadIdx.x >> 5;
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
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint64_t ad = umma_desc_sw128(sA + s * Cfg::A_BYTES);
                const uint64_t bd = umma_desc_sw128(sB + s * Cfg::B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
                umma_commit(&empty[s]);
            }
            umma_commit(accum_full);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;
        const int row_in_tile = q * 32 + lane;
        const int r = m_tile * BM + row_in_tile;
        const bool valid = r < p.M;
        const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
        const int n0 = n_tile * BN;
        const int etid = threadIdx.x - 64;  // 0..127

        mbar_wait(accum_full, 0);
        tc_fence_after();

        const bool split_k = p.splits > 1;
        const bool resid = p.mode == kModeResid;
        float rs = 1.0f;
        if ((p.flags & kFlagRowScale) && valid)
            rs = 1.0f / sqrtf(p.row_stats[r] * p.inv_width + p.eps);

        if (split_k) {
            // Partial sums -> global; the last-arriving CTA of the tile finishes.
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                float v[32];
                tmem_ld32(trow + c * 32, v);
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (valid && nv > 0) {
                    if (resid) {
                        float* dst = reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            float b = 0.f;
                            if ((p.flags & kFlagBias) && split == 0 && j < nv) b = p.bias[col0 + j];
                            v[j] = p.resid_scale * (v[j] * rs + b);
                        }
                        ws_add32(dst, v, nv);
                    } else {
                        ws_add32(p.ws + (long long)r * p.N + col0, v, nv);
                    }
                }
            }
            __threadfence();
            named_bar_sync(1, 128);
            if (etid == 0) {
                const int tile = m_tile * gridDim.y + n_tile;
                const int prev = atomicAdd(&p.counters[tile], 1);
                const int last = prev == p.splits - 1;
                if (last) atomicExch(&p.counters[tile], 0);
                *last_flag = last;
            }
            named_bar_sync(1, 128);
            if (!*last_flag) goto epilogue_done;
            __threadfence();
        }

        if (resid) {
            // h += scale*(rs*z + b) (already accumulated when split), bf16 shadow, row stats.
            float ss = 0.f;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                float v[32];
                if (!split_k) tmem_ld32(trow + c * 32, v);
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (!valid || nv <= 0) continue;
                float* h = reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (j < nv) {
                        float x;
                        if (split_k) {
                            x = __ldcg(h + j);
                        } else {
                            float b = (p.flags & kFlagBias) ? p.bias[col0 + j] : 0.f;
                            x = h[j] + p.resid_scale * (v[j] * rs + b);
                            h[j] = x;
                        }
                        v[j] = x;
                        ss += x * x;
                    }
                }
                if (p.outb)
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob + col0, v, nv);
            }
            if (valid && p.out_stats) atomicAdd(p.out_stats + r, ss);
        } else if (p.mode == kModeGate) {
            // Tile columns [0, BN/2) are up, [BN/2, BN) the matching gate columns.
            constexpr int H = BN / 2;
#pragma unroll 1
            for (int c = 0; c < H / 32; ++c) {
                float u[32], g[32];
                const int ocol0 = n_tile * H + c * 32;
                const int nv = min(32, p.N / 2 - ocol0);
                if (split_k) {
                    if (valid) {
                        ws_take32(p.ws + (long long)r * p.N + n0 + c * 32, u, 32);
                        ws_take32(p.ws + (long long)r * p.N + n0 + H + c * 32, g, 32);
                    }
                } else {
                    tmem_ld32(trow + c * 32, u);
                    tmem_ld32(trow + H + c * 32, g);
                }
                if (!valid || nv <= 0) continue;
#pragma unroll
                for (int j = 0; j < 32; ++j) u[j] = (u[j] * rs) * gelu_tanh(g[j] * rs);
                store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + ocol0, u, nv);
            }
        } else if ((p.flags & kFlagRope) && n0 < p.rope_cols) {
            // RoPE, half-split pairing (j, j+128) inside each 256-wide head
            // (proj/src/tensor.cpp:150-178). BN == 256 so a tile is exactly one head.
            const float2* cs = reinterpret_cast<const float2*>(p.rope_cs) + (long long)(p.rope_pos0 + r) * 128;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float a[32], b[32];
                if (split_k) {
                    if (valid) {
                        ws_take32(p.ws + (long long)r * p.N + n0 + c * 32, a, 32);
                        ws_take32(p.ws + (long long)r * p.N + n0 + 128 + c * 32, b, 32);
                    }
                } else {
                    tmem_ld32(trow + c * 32, a);
                    tmem_ld32(trow + 128 + c * 32, b);
                }
                if (!valid) continue;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    float x = a[j] * rs, y = b[j] * rs;
                    if (p.flags & kFlagBias) {
                        x += p.bias[n0 + c * 32 + j];
                        y += p.bias[n0 + 128 + c * 32 + j];
                    }
                    const float2 t = cs[c * 32 + j];
                    a[j] = x * t.x - y * t.y;
                    b[j] = x * t.y + y * t.x;
                }
                __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + n0;
                store_bf16x32(o + c * 32, a, 32);
                store_bf16x32(o + 128 + c * 32, b, 32);
            }
        } else {
            // kModeBf16 / kModeF32Store / kModeSiluTable, 32 columns at a time.
            float ss = 0.f;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                float v[32];
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (split_k) {
                    if (valid && nv > 0) ws_take32(p.ws + (long long)r * p.N + col0, v, nv);
                } else {
                    tmem_ld32(trow + c * 32, v);
                }
                if (!valid || nv <= 0) continue;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    float x = v[j];
                    if (j < nv) {
                        if (p.mode == kModeSiluTable) {
                            x = silu_f(x + p.table_row[col0 + j]);
                        } else {
                            x *= rs;
                            if (p.flags & kFlagBias) x += p.bias[col0 + j];
                            if (p.flags & kFlagGelu) x = gelu_tanh(x);
                        }
                    }
                    v[j] = x;
                }
                if (p.mode == kModeF32Store) {
                    float* o = reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (j < nv) {
                            o[j] = v[j];
                            ss += v[j] * v[j];
                        }
                    }
                    if (p.outb)
                        store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob + col0, v, nv);
                } else {
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + col0, v, nv);
                }
            }
            if (p.mode == kModeF32Store) {
                if (valid && p.out_stats) atomicAdd(p.out_stats + r, ss);
                // Optional extra row -1 (the state token of ae.suffix,
                // proj/src/builder.cpp:311-312), written by the first tile row.
                if (p.row0_src && m_tile == 0 && row_in_tile == 0) {
                    float* o = reinterpret_cast<float*>(p.out) - p.ldo;
                    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.outb) - p.ldob;
                    float s0 = 0.f;
                    for (int j = n0; j < min(n0 + BN, p.N); ++j) {
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

template <int BN, int STAGES>
static cudaError_t configure_t() {
    return cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmCfg<BN, STAGES>::SMEM);
}

template <int BN, int STAGES>
static cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                                 int m_tiles, int n_tiles, cudaStream_t stream) {
    dim3 grid(m_tiles, n_tiles, p.splits);
    gemm_tc_kernel<BN, STAGES><<<grid, kGemmThreads, GemmCfg<BN, STAGES>::SMEM, stream>>>(ta, tb, p);
    return cudaGetLastError();
}

// Must run once per device before any launch (not capturable).
cudaError_t gemm_configure() {
    cudaError_t e = configure_t<256, 4>();
    if (e == cudaSuccess) e = configure_t<128, 6>();
    if (e == cudaSuccess) e = configure_t<64, 8>();
    return e;
}

cudaError_t launch_gemm(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                        cudaStream_t stream) {
    const int m_tiles = (p.M + BM - 1) / BM;
    const int n_tiles = (p.N + bn - 1) / bn;
    switch (bn) {
        case 256: return launch_gemm_t<256, 4>(ta, tb, p, m_tiles, n_tiles, stream);
        case 128: return launch_gemm_t<128, 6>(ta, tb, p, m_tiles, n_tiles, stream);
        case 64: return launch_gemm_t<64, 8>(ta, tb, p, m_tiles, n_tiles, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
