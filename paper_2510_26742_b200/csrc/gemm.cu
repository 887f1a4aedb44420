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
// Split-K: grid.z = the K-splits of a tile, launched as ONE thread-block cluster; after the
// mainloop each CTA parks the fp32 partials of the 32-column chunks it does not own in its own
// (now idle) pipeline shared memory, and the owner of each chunk pulls the peers' partials over
// DSMEM and runs the epilogue -- no global workspace, no atomics, no second pass.
// PDL: the next launch's prologue and first weight tiles overlap this kernel's tail
// (griddepcontrol.wait guards every read of the previous kernel's outputs).
#include "gemm.cuh"
#include "ptx.cuh"

namespace pi0b {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kGemmThreads = 64 + 8 * 32;  // TMA warp, MMA warp, 8 epilogue warps
static bool g_gemm_pdl = true;             // launch with programmatic stream serialization

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

PI0B_DEV void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
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

    if (threadIdx.x == 0) pdl_launch_dependents();
    const int S = p.splits;  // cluster size along K (grid.z)

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            // Weight tiles never depend on the previous kernel: issue the first ring's worth
            // before waiting for it (PDL), then the activation tiles.
            const int pre = min(STAGES, nkb);
            for (int i = 0; i < pre; ++i) {
                mbar_arrive_expect_tx(&full[i], Cfg::STAGE_BYTES);
                tma_load_2d(sB + i * Cfg::B_BYTES, &tmB, &full[i], (kb0 + i) * BK, n_tile * BN, kEvictNormal);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i)
                tma_load_2d(sA + i * Cfg::A_BYTES, &tmA, &full[i], (kb0 + i) * BK, m_tile * BM, kEvictLast);
            for (int i = pre; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                const int kc = (kb0 + i) * BK;
                tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kc, m_tile * BM, kEvictLast);
                tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kc, n_tile * BN, kEvictNormal);
            }
        }
        __syncwarp();
        if (S > 1) {
            cluster_sync_all();
            cluster_sync_all();
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
        if (S > 1) {
            cluster_sync_all();
            cluster_sync_all();
        }
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

        // Stage the per-column vector (bias or SiluBias table row), zero-padded, while the
        // mainloop runs; then wait for the previous kernel (PDL) before reading its outputs.
        const float* vec = MODE == kModeSiluTable ? p.table_row : ((p.flags & kFlagBias) ? p.bias : nullptr);
        for (int c = etid; c < BN; c += 256) sm_vec[c] = (vec && n0 + c < p.N) ? vec[n0 + c] : 0.f;
        pdl_wait();
        float rs = 1.0f;
        if ((p.flags & kFlagRowScale) && valid) rs = 1.0f / sqrtf(p.row_stats[r] * p.inv_width + p.eps);
        named_bar_sync(1, 256);

        mbar_wait(accum_full, 0);
        tc_fence_after();

        constexpr int NC = BN / 32;                 // 32-column chunks in the tile
        constexpr int NP = NC / 2;                  // (c, c + NP) pairs
        constexpr int NU = kPaired ? NP : NC;       // epilogue units: chunks, or chunk pairs
        // Split-K: unit u belongs to cluster rank u % S.  Chunk c of row r is parked at
        // stage + c*16 KB + r*128 B, 16-byte pieces XOR-swizzled by r (conflict-free).
        const int rank = split;
        const uint32_t srow = smem_u32(smem) + row_in_tile * 128;
        const int sw = row_in_tile & 7;
        if (S > 1) {
#pragma unroll 1
            for (int c = hsel * (NC / 2); c < (hsel + 1) * (NC / 2); ++c) {
                if ((kPaired ? c % NP : c) % S == rank) continue;
                float v[32];
                tmem_ld32(trow + c * 32, v);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    st_shared_v4(srow + c * 16384 + ((j ^ sw) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            cluster_sync_all();
        }
        // The full K sum of chunk c for this thread's row: own accumulator + the peers' partials.
        auto acc32 = [&](int c, float(&v)[32]) {
            tmem_ld32(trow + c * 32, v);
            if (S > 1) {
#pragma unroll 1
                for (int k = 0; k < S; ++k) {
                    if (k == rank) continue;
                    const uint32_t ra = mapa_shared(srow + c * 16384, k);
                    float4 f[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) f[j] = ld_dsmem_f32x4(ra + ((j ^ sw) << 4));
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        v[4 * j] += f[j].x;
                        v[4 * j + 1] += f[j].y;
                        v[4 * j + 2] += f[j].z;
                        v[4 * j + 3] += f[j].w;
                    }
                }
            }
        };
        const int u_first = S > 1 ? rank + S * hsel : hsel * (NU / 2);
        const int u_step = S > 1 ? 2 * S : 1;
        const int u_end = S > 1 ? NU : u_first + NU / 2;

        if constexpr (MODE == kModeResid) {
            // h += scale*(rs*z + b) in place, bf16 shadow, row stats.
            float ss = 0.f;
#pragma unroll 1
            for (int c = u_first; c < u_end; c += u_step) {
                float v[32], h[32];
                acc32(c, v);
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                if (!valid || nv <= 0) continue;
                float* hp = reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0;
                load_f32x32(hp, h, nv, false);
#pragma unroll
                for (int j = 0; j < 32; ++j) h[j] += p.resid_scale * (v[j] * rs + sm_vec[c * 32 + j]);
                store_f32x32(hp, h, nv);
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
            for (int c = u_first; c < u_end; c += u_step) {
                float a[32], b[32];
                acc32(c, a);
                acc32(c + NP, b);
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
            for (int c = u_first; c < u_end; c += u_step) {
                float v[32];
                const int col0 = n0 + c * 32;
                const int nv = min(32, p.N - col0);
                acc32(c, v);
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
                // proj/src/builder.cpp:311-312), written by the first tile row of rank 0.
                if (p.row0_src && m_tile == 0 && row_in_tile == 0 && rank == 0) {
                    float* o = reinterpret_cast<float*>(p.out) - p.ldo;
                    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.outb) - p.ldob;
                    float s0 = 0.f;
                    for (int j = n0 + hsel * (BN / 2); j < min(n0 + (hsel + 1) * (BN / 2), p.N); ++j) {
                        const float x = p.row0_src[j];
                        o[j] = x;
                        if (p.outb) ob[j] = __float2bfloat16_rn(x);
                        s0 += x * x;
                    }
                    if (p.out_stats) atomicAdd(p.out_stats - 1, s0);
                }
            }
        }
        // Peers may still be reading this CTA's parked partials.
        if (S > 1) cluster_sync_all();
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
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kGemmThreads, 1, 1);
    cfg.dynamicSmemBytes = GemmCfg<BN, STAGES>::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.splits > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = p.splits;
        ++na;
    }
    if (g_gemm_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, STAGES, MODE>, ta, tb, p);
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

void gemm_set_pdl(bool on) { g_gemm_pdl = on; }

// How many clusters of `splits` CTAs of this GEMM configuration fit on the device at once
// (clusters are confined to a GPC, so this is below num_sms / splits).
int gemm_max_active_clusters(int bn, int splits) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1, 1, splits);
    cfg.blockDim = dim3(kGemmThreads, 1, 1);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = splits;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaErrorInvalidValue;
    switch (bn) {
        case 256:
            cfg.dynamicSmemBytes = GemmCfg<256, 4>::SMEM;
            e = cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<256, 4, kModeBf16>, &cfg);
            break;
        case 128:
            cfg.dynamicSmemBytes = GemmCfg<128, 6>::SMEM;
            e = cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<128, 6, kModeBf16>, &cfg);
            break;
        case 64:
            cfg.dynamicSmemBytes = GemmCfg<64, 8>::SMEM;
            e = cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<64, 8, kModeBf16>, &cfg);
            break;
    }
    return e == cudaSuccess ? n : 0;
}

cudaError_t launch_gemm(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                        cudaStream_t stream) {
    if ((p.flags & kFlagRope) && bn != 256) return cudaErrorInvalidValue;
    if (p.splits < 1 || p.splits > kGemmMaxSplits) return cudaErrorInvalidValue;
    const dim3 grid((p.M + BM - 1) / BM, (p.N + bn - 1) / bn, p.splits);
    switch (bn) {
        case 256: return launch_bn<256, 4>(ta, tb, p, grid, stream);
        case 128: return launch_bn<128, 6>(ta, tb, p, grid, stream);
        case 64: return launch_bn<64, 8>(ta, tb, p, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
