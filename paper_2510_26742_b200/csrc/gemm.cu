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
#include "ktrace.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace pi0b {

// Timeline instrumentation (variant builds only, -DPI0B_GEMM_TRACE; scripts/gemm_trace.py): 16
// globaltimer stamps per CTA into the buffer set by pi0b_gemm_trace_buffer().
#ifdef PI0B_GEMM_TRACE
__device__ unsigned long long* g_gm_trace;
#define GM_STAMP(i)                                                                                      \
    do {                                                                                                 \
        if (g_gm_trace) {                                                                                \
            unsigned long long t_;                                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
            g_gm_trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + (i)] = t_; \
        }                                                                                                \
    } while (0)
extern "C" int pi0b_gemm_trace_buffer(unsigned long long* p) {
    return int(cudaMemcpyToSymbol(g_gm_trace, &p, sizeof(p)));
}
#else
#define GM_STAMP(i) \
    do {            \
    } while (0)
#endif

constexpr int BM = 128;
#ifndef PI0B_PAIR_STAGES
#define PI0B_PAIR_STAGES 7
#endif
constexpr int kPairStages = PI0B_PAIR_STAGES;  // smem ring depth of the CTA-pair GEMM (32 KB stages)
constexpr int BK = 64;
constexpr int kGemmThreads = 64 + 8 * 32;  // TMA warp, MMA warp, 8 epilogue warps
static bool g_gemm_pdl = true;             // launch with programmatic stream serialization

// MT: 128-row m-tiles per CTA sharing every weight tile (MT = 2: a 256 x BN CTA tile, two
// accumulators in TMEM, half the L2 -> SM weight traffic per FLOP of MT = 1).
// CG: CTAs per MMA (CG = 2: a CTA pair runs one 256 x BN tile with tcgen05 cta_group::2; each
// CTA stages its own 128 A rows and half of the BN weight rows, so the shared-memory operand
// traffic per MMA halves -- a single-CTA M=128 MMA fed by TMA is shared-memory-bandwidth bound
// at ~55% of the tensor pipe).
template <int BN, int STAGES, int MT = 1, int CG = 1>
struct GemmCfg {
    static constexpr int A_TILE = BM * BK * 2;
    static constexpr int A_BYTES = MT * A_TILE;
    static constexpr int B_BYTES = (BN / CG) * BK * 2;
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
template <int BN, int STAGES, int MODE, int MT = 1, int CG = 1>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
    using Cfg = GemmCfg<BN, STAGES, MT, CG>;
    static_assert(CG == 1 || (MT == 1 && BN == 256), "CTA-pair tiles are 256 x 256");
    // accumulator buffers: double-buffered when two fit in TMEM's 512 columns
    constexpr int NBUF = 2 * MT * Cfg::TMEM_COLS <= 512 ? 2 : 1;
    // chunk pairs (c, c + NP): gated FFN (up | gate), RoPE heads (bn 256, or bn 128 over
    // kPermRope-packed weights); bn 256 bf16 GEMMs without RoPE take the same path and simply
    // write both chunks in place
    const bool kPaired = MODE == kModeGate || (MODE == kModeBf16 && (BN == 256 || (BN == 128 && (p.flags & kFlagRopePacked))));
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* accum_full = empty + STAGES;   // [2] (double-buffered accumulator when persistent)
    uint64_t* accum_empty = accum_full + 2;  // [2]
    // split-K push combine: peers_free completes when every peer's pipeline smem is drained (and its
    // recv_full armed); recv_full when the peers' partials of this CTA's chunks have landed
    uint64_t* peers_free = accum_empty + 2;
    uint64_t* recv_full = peers_free + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_full + 1);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    float* sm_vec = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::BAR_BYTES);

    const int warp = __shfl_sync(0xffffffff, int(threadIdx.x >> 5), 0);  // warp-uniform (see below)
    const int lane = threadIdx.x & 31;
    KT_SMEM;
    KT_START();
    if (threadIdx.x == 0) GM_STAMP(0);
    // Persistent mode (p.persist, no split-K): CTA b walks tiles b, b + grid, ... (m fastest, so
    // CTAs running together share weight tiles in L2) with the accumulator double-buffered in
    // TMEM: the epilogue of tile j overlaps the mainloop of tile j + 1.
    const bool persist = p.persist != 0;
    // CG = 2: the pair (blockIdx.x / 2) owns a 256-row tile; this CTA its rows rank * 128 + ..
    const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = crank == 0;
    const int gm = (p.M + MT * CG * BM - 1) / (MT * CG * BM);
    const int n_tiles = persist ? gm * ((p.N + BN - 1) / BN) : 1;
    const int t_first = persist ? int(blockIdx.x) / CG : 0, t_step = persist ? int(gridDim.x) / CG : 1;
    auto tile_mn = [&](int t, int& m, int& n) {
        if (persist) {
            m = t % gm;
            n = t / gm;
        } else {
            m = blockIdx.x / CG;
            n = blockIdx.y;
        }
    };
    const int split = blockIdx.z;
    const int KB = (p.K + BK - 1) / BK;
    const int kb0 = split * p.kb_per_split;
    const int kb1 = min(KB, kb0 + p.kb_per_split);
    const int nkb = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        // CG = 2: the leader's full[s] collects both CTAs' TMA bytes (and one arrival each), its
        // accum_empty[b] both CTAs' epilogue arrivals
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], CG);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&accum_full[b], 1);
            mbar_init(&accum_empty[b], CG);
        }
        mbar_init(peers_free, p.splits > 1 ? p.splits - 1 : 1);
        mbar_init(recv_full, 1);
        fence_barrier_init();
    }
    __syncwarp();  // warp 0 reconverged before the (.aligned) block barrier
    const int tmem_cols = (persist ? NBUF : 1) * MT * Cfg::TMEM_COLS;
    if (warp == 1) {
        if constexpr (CG == 2) tmem_alloc_cg2(tmem_slot, tmem_cols);
        else tmem_alloc(tmem_slot, tmem_cols);
    }
    tc_fence_before();
    // Peer barriers initialised before any remote arrive.  CTA pair (CG = 2): a full cluster
    // barrier.  Split-K cluster (grid.z = p.splits > 1): the arrive (release) here, the matching
    // wait (acquire) just before each thread's first cluster access (split_wait below), so the
    // barrier costs nothing on the critical path.
    if constexpr (CG == 2) {
        cluster_sync_all();
    } else {
        // (fence_barrier_init above is the release of the inits; the arrive itself can be relaxed)
        if (p.splits > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
        __syncthreads();
    }
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) GM_STAMP(1);

    if (threadIdx.x == 0) pdl_launch_dependents();
    const int S = p.splits;  // cluster size along K (grid.z)
    // split-K combine by st.async pushes into the peers' drained pipeline smem (see the epilogue)
    const bool push = S > 1 && S * (BN / 32) * 16384 <= STAGES * Cfg::STAGE_BYTES;
    // the other half of the split-K init barrier: exactly once per thread, before its first
    // remote mbarrier arrive / DSMEM access / cluster barrier
    auto split_wait = [&]() {
        if (CG == 1 && S > 1) cluster_wait_acquire();
    };
    // Staged epilogue: a single-tile CTA (no persistence, no CTA pair / multi-tile) writes its
    // finished 32-column chunks as fp32 into the drained pipeline smem (past the split-K receive
    // slots) and then copies them out with whole-warp, row-contiguous stores -- per-thread row
    // stores (32 rows x 16 B per warp instruction) cost ~1.5 us per 32 KB tile
    // (DESIGN.md 5).  Chunk c of the tile lives at stage_off + c * 16 KB, [128 rows][128 B],
    // 16-byte pieces XOR-swizzled by row.
    constexpr int NCH = BN / 32;
    const int stage_off = S > 1 ? S * NCH * 16384 : 0;
    const bool staged = !kPaired && !persist && MT == 1 && CG == 1 && (S == 1 || push) &&
                        stage_off + NCH * 16384 <= STAGES * Cfg::STAGE_BYTES &&
                        MODE == kModeResid;
    // bf16-output tiles (ve.qkv, ve.fc1): staged as bf16 in the drained pipeline smem, then written
    // as whole rows (a warp = 2 rows x 256 B at bn 128): per-thread row pieces (32 rows per warp
    // store) cost ~2 us per 32 KB tile inside the GEMM, a third of a small GEMM's time.
    constexpr int PR = BN / 8;                       // 16-byte pieces per staged bf16 row
    constexpr int PSW = PR < 16 ? PR - 1 : 15;       // piece swizzle mask (by row)
    const bool staged16 = MODE == kModeBf16 && !kPaired && !persist && MT == 1 && CG == 1 && S == 1 &&
                          (p.flags & kFlagStageBf16) && 128 * PR * 16 <= STAGES * Cfg::STAGE_BYTES;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int g = 0;  // k-blocks issued by this CTA (ring position across tiles)
            for (int t = t_first; t < n_tiles; t += t_step) {
                int m_tile, n_tile;
                tile_mn(t, m_tile, n_tile);
                int i0 = 0;
                // CG = 2: this CTA's A rows / weight rows within the pair tile, and the leader's
                // full barrier (shared::cluster address) that both CTAs' copies complete on
                const int arow = CG == 2 ? (m_tile * 2 + int(crank)) * BM : 0;
                const int brow = n_tile * BN + int(crank) * (BN / CG);
                auto arm = [&](int s) {
                    if constexpr (CG == 2) {
                        if (leader) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
                        else mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&full[s]), 0));
                    } else {
                        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
                    }
                };
                auto load_b = [&](int s, int kc) {
                    if constexpr (CG == 2) tma_load_2d_cg2(sB + s * Cfg::B_BYTES, &tmB, mapa_shared(smem_u32(&full[s]), 0), kc, brow, kEvictNormal);
                    else tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kc, brow, kEvictNormal);
                };
                auto load_a = [&](int s, int kc) {
                    if constexpr (CG == 2) {
                        tma_load_2d_cg2(sA + s * Cfg::A_BYTES, &tmA, mapa_shared(smem_u32(&full[s]), 0), kc, arow, kEvictLast);
                    } else {
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
                            tma_load_2d(sA + s * Cfg::A_BYTES + mt * Cfg::A_TILE, &tmA, &full[s], kc, (m_tile * MT + mt) * BM,
                                        kEvictLast);
                    }
                };
                if (g == 0) {
                    // Weight tiles never depend on the previous kernel: issue the first ring's
                    // worth before waiting for it (PDL), then the activation tiles.
                    const int pre = min(STAGES, nkb);
                    for (int i = 0; i < pre; ++i) {
                        arm(i);
                        load_b(i, (kb0 + i) * BK);
                    }
                    pdl_wait();
                    KT_DEP();
                    GM_STAMP(2);
                    for (int i = 0; i < pre; ++i) load_a(i, (kb0 + i) * BK);
                    i0 = pre;
                    g = pre;
                }
                for (int i = i0; i < nkb; ++i, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    if (g >= STAGES) mbar_wait(&empty[s], ph ^ 1);
                    arm(s);
                    const int kc = (kb0 + i) * BK;
                    load_a(s, kc);
                    load_b(s, kc);
                }
            }
        }
        __syncwarp();
        split_wait();
        if (S > 1 && !push) {
            cluster_sync_all();
            cluster_sync_all();
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // Warp-uniform loop, one elected lane issues: tcgen05.mma from a divergent single-lane
        // branch costs ~270 instead of ~128 issue cycles per N=256 MMA (scripts/mma_bench.cu).
        if (leader) {  // CG = 2: only the leader CTA issues (for both)
            constexpr uint32_t idesc = umma_idesc_bf16(BM * CG, BN);
            int g = 0, j = 0;
            for (int t = t_first; t < n_tiles; t += t_step, ++j) {
                const int b = j % NBUF;
                if (j >= NBUF) {  // the epilogue of tile j - NBUF has drained this accumulator
                    mbar_wait(&accum_empty[b], ((j / NBUF) & 1) ^ 1);
                    tc_fence_after();
                }
                const uint32_t dt = tmem + uint32_t(b * MT * BN);
                for (int i = 0; i < nkb; ++i, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = (g / STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    if (lane == 0 && i == 0 && j == 0) GM_STAMP(3);
                    tc_fence_after();
                    const uint64_t ad = umma_desc_sw128(sA + s * Cfg::A_BYTES);
                    const uint64_t bd = umma_desc_sw128(sB + s * Cfg::B_BYTES);
                    if (elect_one()) {
                        if constexpr (CG == 2) {
#pragma unroll
                            for (int k = 0; k < BK / 16; ++k) umma_bf16_cg2(dt, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
                            umma_commit_cg2(&empty[s]);
                        } else {
#pragma unroll
                            for (int k = 0; k < BK / 16; ++k)
#pragma unroll
                                for (int mt = 0; mt < MT; ++mt)
                                    umma_bf16(dt + mt * BN, ad + ((mt * Cfg::A_TILE) >> 4) + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
                            umma_commit(&empty[s]);
                        }
                    }
                    __syncwarp();
                }
                if (elect_one()) {
                    if constexpr (CG == 2) umma_commit_cg2(&accum_full[b]);
                    else umma_commit(&accum_full[b]);
                }
                __syncwarp();
            }
        }
        __syncwarp();
        split_wait();
        if (S > 1 && !push) {
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
        int j = 0;
        for (int t = t_first; t < n_tiles; t += t_step, ++j) {
        int m_big, n_tile;
        tile_mn(t, m_big, n_tile);
        const uint32_t acc_base = uint32_t((j % NBUF) * MT * BN);
        if (MT > 1) mbar_wait(&accum_full[j % NBUF], (j / NBUF) & 1);
#pragma unroll 1
        for (int mt = 0; mt < MT; ++mt) {
        const int m_tile = CG == 2 ? m_big * 2 + int(crank) : m_big * MT + mt;
        const int r = m_tile * BM + row_in_tile;
        const bool valid = r < p.M;
        const uint32_t trow = tmem + (uint32_t(q * 32) << 16) + acc_base + uint32_t(mt * BN);
        const int n0 = n_tile * BN;

        // Stage the per-column vector (bias or SiluBias table row), zero-padded, while the
        // mainloop runs; then wait for the previous kernel (PDL) before reading its outputs.
        const float* vec = MODE == kModeSiluTable ? p.table_row : ((p.flags & kFlagBias) ? p.bias : nullptr);
        for (int c = etid; c < BN; c += 256) sm_vec[c] = (vec && n0 + c < p.N) ? vec[n0 + c] : 0.f;
        pdl_wait();
        float rs = 1.0f;
        if ((p.flags & kFlagRowScale) && valid) rs = 1.0f / sqrtf(p.row_stats[r] * p.inv_width + p.eps);
        constexpr int NC = BN / 32;                 // 32-column chunks in the tile
        constexpr int NP = NC / 2;                  // (c, c + NP) pairs
        const int NU = kPaired ? NP : NC;           // epilogue units: chunks, or chunk pairs
        // Split-K: unit u belongs to cluster rank u % S.
        const int rank = split;
        const int u_first = S > 1 ? rank + S * hsel : hsel * (NU / 2);
        const int u_step = S > 1 ? 2 * S : 1;
        const int u_end = S > 1 ? NU : u_first + NU / 2;
        // Residual base of this thread's first unit (the previous kernel's output, independent
        // of the accumulator): loaded now so its L2 latency overlaps the mainloop.
        float hpre[32];
        if constexpr (MODE == kModeResid) {
            const int col0 = n0 + u_first * 32;
            if (valid && u_first < u_end && col0 < p.N)
                load_f32x32(reinterpret_cast<const float*>(p.out) + (long long)r * p.ldo + col0, hpre, min(32, p.N - col0),
                            false);
        }
        named_bar_sync(1, 256);

        // Instruction-cache warm-up: the epilogue runs once per launch, mostly straight-line code
        // that is cold every time (~60 ns per 128-byte line on first execution), so a
        // single-tile CTA first runs it "dry" while its mainloop is still going -- the same
        // instructions on whatever TMEM / shared memory holds, with every global or shared store,
        // atomic, DSMEM push and barrier skipped -- and the real pass then runs from the cache.
        const bool warm = (p.flags & kFlagWarmEpi) && !persist && MT == 1 && CG == 1 && (S == 1 || push);
#pragma unroll 1
        for (int pass = warm ? 0 : 1; pass < 2; ++pass) {
        const bool dry = pass == 0;
        if (!dry) {
            if (MT == 1) mbar_wait(&accum_full[j % NBUF], (j / NBUF) & 1);
            tc_fence_after();
            if (etid == 0 && j == 0) GM_STAMP(4);
            split_wait();  // (S > 1 implies one tile per CTA: once)
        }
        // Split-K combine, push form (S * NC chunks of 16 KB fit in the drained pipeline smem):
        // as soon as its own MMAs are done a CTA arms its receive barrier and tells the peers its
        // pipeline smem is free; once all peers are free it st.asyncs the partials of the chunks
        // it does not own straight from TMEM into the owners' smem (slot [sender rank][chunk],
        // 128 B per row, 16-byte pieces XOR-swizzled by row), then waits for its own chunks'
        // partials -- no cluster-wide barrier and no remote loads on the critical path.
        // Otherwise (larger splits) the chunks are parked locally and pulled over DSMEM.
        const uint32_t srow = smem_u32(smem) + row_in_tile * 128;
        const int sw = row_in_tile & 7;
        auto owner_of = [&](int c) { return (kPaired ? c % NP : c) % S; };
        if (S > 1 && push) {
            if (etid == 0 && !dry) {
                int owned = 0;
                for (int c = 0; c < NC; ++c) owned += owner_of(c) == rank;
                mbar_arrive_expect_tx(recv_full, uint32_t((S - 1) * owned * 16384));
                for (int k = 0; k < S; ++k)
                    if (k != rank) mbar_arrive_cluster(mapa_shared(smem_u32(peers_free), uint32_t(k)));
            }
            if (!dry) mbar_wait_cluster(peers_free, 0);
#pragma unroll 1
            for (int c = hsel * (NC / 2); c < (hsel + 1) * (NC / 2); ++c) {
                const int own = owner_of(c);
                if (own == rank) continue;
                float v[32];
                tmem_ld32(trow + c * 32, v);
                const uint32_t dst = mapa_shared(srow + uint32_t((rank * NC + c) * 16384), uint32_t(own));
                const uint32_t bar = mapa_shared(smem_u32(recv_full), uint32_t(own));
                if (!dry) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        st_async_v4(dst + ((j ^ sw) << 4), make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]), bar);
                }
            }
            if (!dry) {
                if (etid == 0 && j == 0) GM_STAMP(5);
                mbar_wait_cluster(recv_full, 0);
                if (etid == 0 && j == 0) GM_STAMP(6);
            }
        } else if (S > 1) {
#pragma unroll 1
            for (int c = hsel * (NC / 2); c < (hsel + 1) * (NC / 2); ++c) {
                if (owner_of(c) == rank) continue;
                float v[32];
                tmem_ld32(trow + c * 32, v);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    st_shared_v4(srow + c * 16384 + ((j ^ sw) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            if (etid == 0 && j == 0) GM_STAMP(5);
            cluster_sync_all();
            if (etid == 0 && j == 0) GM_STAMP(6);
        }
        // The full K sum of chunk c for this thread's row: own accumulator + the peers' partials.
        auto acc32 = [&](int c, float(&v)[32]) {
            tmem_ld32(trow + c * 32, v);
            if (S > 1) {
#pragma unroll 1
                for (int k = 0; k < S; ++k) {
                    if (k == rank) continue;
                    float4 f[8];
                    if (push) {
                        const float4* src = reinterpret_cast<const float4*>(smem + (k * NC + c) * 16384 + row_in_tile * 128);
#pragma unroll
                        for (int j = 0; j < 8; ++j) f[j] = src[j ^ sw];
                    } else {
                        const uint32_t ra = mapa_shared(srow + c * 16384, k);
#pragma unroll
                        for (int j = 0; j < 8; ++j) f[j] = ld_dsmem_f32x4(ra + ((j ^ sw) << 4));
                    }
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
        const uint32_t sstage = smem_u32(smem) + uint32_t(stage_off) + row_in_tile * 128;
        auto stage32 = [&](int c, const float(&v)[32]) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
                st_shared_v4(sstage + c * 16384 + ((jj ^ sw) << 4), v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
        };
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
                if (c == u_first) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) h[j] = hpre[j];
                } else {
                    load_f32x32(hp, h, nv, false);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) h[j] += p.resid_scale * (v[j] * rs + sm_vec[c * 32 + j]);
                ss += sumsq32(h, nv);
                if (dry) continue;
                if (staged) {
                    stage32(c, h);
                    continue;
                }
                store_f32x32(hp, h, nv);
                if (p.outb)
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob + col0, h, nv);
            }
            if (valid && p.out_stats && !dry) atomicAdd(p.out_stats + r, ss);
        } else if (kPaired) {
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
                    for (int j = 0; j < 32; ++j) a[j] = (a[j] * rs) * gelu_fast(b[j] * rs);
                    const int ocol0 = n_tile * (BN / 2) + c * 32;
                    if (!dry) store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + ocol0, a,
                                  min(32, p.N / 2 - ocol0));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        a[j] = a[j] * rs + sm_vec[c * 32 + j];
                        b[j] = b[j] * rs + sm_vec[(c + NP) * 32 + j];
                    }
                    if (p.flags & kFlagGelu) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            a[j] = gelu_fast(a[j]);
                            b[j] = gelu_fast(b[j]);
                        }
                    }
                    // packed bn = 128 head tile: features at head * 256 + 64 * half + 32 c + j,
                    // partners 128 further (kernels_misc.cu packed_row, kPermRope)
                    const bool packed = BN == 128 && rope && (p.flags & kFlagRopePacked);
                    const int j0 = packed ? ((n0 >> 7) & 1) * 64 + c * 32 : c * 32;  // rope table column
                    if (rope) {
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            const float4 t = *reinterpret_cast<const float4*>(cs + j0 + j);
                            const float x0 = a[j], y0 = b[j], x1 = a[j + 1], y1 = b[j + 1];
                            a[j] = x0 * t.x - y0 * t.y;
                            b[j] = x0 * t.y + y0 * t.x;
                            a[j + 1] = x1 * t.z - y1 * t.w;
                            b[j + 1] = x1 * t.w + y1 * t.z;
                        }
                    }
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo;
                    if (dry) continue;
                    if (packed) {
                        const int f = (n0 >> 8) * 256 + j0;
                        store_bf16x32(o + f, a, 32);
                        store_bf16x32(o + f + 128, b, 32);
                    } else {
                        store_bf16x32(o + n0 + c * 32, a, min(32, p.N - (n0 + c * 32)));
                        store_bf16x32(o + n0 + (c + NP) * 32, b, min(32, p.N - (n0 + (c + NP) * 32)));
                    }
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
                if (etid == 0 && j == 0 && !dry && c == u_first) GM_STAMP(10);
                if (!valid || nv <= 0) continue;
                if constexpr (MODE == kModeSiluTable) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = silu_f(v[j] + sm_vec[c * 32 + j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = v[j] * rs + sm_vec[c * 32 + j];
                    if (MODE == kModeBf16 && (p.flags & kFlagGelu)) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
                    }
                }
                if (dry) continue;
                if constexpr (MODE == kModeF32Store) {
                    store_f32x32(reinterpret_cast<float*>(p.out) + (long long)r * p.ldo + col0, v, nv);
                    ss += sumsq32(v, nv);
                    if (p.outb)
                        store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)r * p.ldob + col0, v, nv);
                } else if (staged) {
                    stage32(c, v);
                } else if (staged16) {
                    const uint32_t srow16 = smem_u32(smem) + row_in_tile * (PR * 16);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int pc = c * 4 + q;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(srow16 + ((pc ^ (row_in_tile & PSW)) << 4)),
                                     "r"(pack_bf16(v[8 * q], v[8 * q + 1])), "r"(pack_bf16(v[8 * q + 2], v[8 * q + 3])),
                                     "r"(pack_bf16(v[8 * q + 4], v[8 * q + 5])), "r"(pack_bf16(v[8 * q + 6], v[8 * q + 7]))
                                     : "memory");
                    }
                } else {
                    store_bf16x32(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)r * p.ldo + col0, v, nv);
                }
                if (etid == 0 && j == 0 && c == u_first) GM_STAMP(11);
            }
            if (etid == 0 && j == 0 && !dry) GM_STAMP(12);
            if constexpr (MODE == kModeF32Store) {
                if (valid && p.out_stats && !dry) atomicAdd(p.out_stats + r, ss);
                // Optional extra row -1 (the state token of ae.suffix,
                // proj/src/builder.cpp:311-312), written by the first tile row of rank 0.
                if (p.row0_src && m_tile == 0 && row_in_tile == 0 && rank == 0 && !dry) {
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
        if (staged16) {
            named_bar_sync(1, 256);
            __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(p.out);
#pragma unroll 2
            for (int e = etid; e < 128 * PR; e += 256) {
                const int row = e / PR, pc = e % PR;
                const int gr = m_tile * BM + row, col = n0 + pc * 8;
                if (gr >= p.M || col >= p.N || dry) continue;
                const uint4 u = *reinterpret_cast<const uint4*>(smem + row * (PR * 16) + ((pc ^ (row & PSW)) << 4));
                if (col + 8 <= p.N) {
                    *reinterpret_cast<uint4*>(ob + (long long)gr * p.ldo + col) = u;
                } else {
                    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&u);
                    for (int k = 0; k < 8 && col + k < p.N; ++k) ob[(long long)gr * p.ldo + col + k] = hv[k];
                }
            }
        }
        if (staged) {
            // coalesced copy-out of the staged chunks this CTA owns (split-K: c % S == rank):
            // piece e = (row, 16-byte piece q) of chunk c; a warp writes 4 rows x 128 B (fp32) /
            // 4 rows x 64 B (bf16), each row segment contiguous in global memory
            named_bar_sync(1, 256);
            const uint8_t* sbase = smem + stage_off;
#pragma unroll 1
            for (int c = S > 1 ? rank : 0; c < NCH; c += S > 1 ? S : 1) {
                const int colc = n0 + c * 32;
#pragma unroll 2
                for (int e = etid; e < 128 * 8; e += 256) {
                    const int row = e >> 3, qq = e & 7;
                    const int gr = m_tile * BM + row, col = colc + qq * 4;
                    if (gr >= p.M || col >= p.N || dry) continue;
                    const float4 f = *reinterpret_cast<const float4*>(sbase + c * 16384 + row * 128 + ((qq ^ (row & 7)) << 4));
                    const uint2 b = make_uint2(pack_bf16(f.x, f.y), pack_bf16(f.z, f.w));
                    if (col + 4 <= p.N) {
                        if constexpr (MODE == kModeResid) {
                            *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + (long long)gr * p.ldo + col) = f;
                            if (p.outb) *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.outb) + (long long)gr * p.ldob + col) = b;
                        } else {
                            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)gr * p.ldo + col) = b;
                        }
                    } else {
                        const float fv[4] = {f.x, f.y, f.z, f.w};
                        for (int k = 0; k < 4 && col + k < p.N; ++k) {
                            if constexpr (MODE == kModeResid) {
                                reinterpret_cast<float*>(p.out)[(long long)gr * p.ldo + col + k] = fv[k];
                                if (p.outb) reinterpret_cast<__nv_bfloat16*>(p.outb)[(long long)gr * p.ldob + col + k] = __float2bfloat16_rn(fv[k]);
                            } else {
                                reinterpret_cast<__nv_bfloat16*>(p.out)[(long long)gr * p.ldo + col + k] = __float2bfloat16_rn(fv[k]);
                            }
                        }
                    }
                }
            }
        }
        }  // pass
        if (etid == 0 && j == 0) GM_STAMP(7);
        // Pull form: peers may still be reading this CTA's parked partials.  Push form: every
        // st.async into this CTA has landed (recv_full); the exit barrier below keeps senders alive.
        if (S > 1 && !push) cluster_sync_all();
        if (etid == 0 && j == 0) GM_STAMP(8);
        named_bar_sync(1, 256);  // sm_vec free for the next (sub-)tile
        }
        // accumulator drained (CG = 2: both CTAs arrive on the leader's barrier)
        tc_fence_before();
        named_bar_sync(1, 256);
        if (etid == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&accum_empty[j % NBUF]), 0));
            else mbar_arrive(&accum_empty[j % NBUF]);
        }
        }
    }

    tc_fence_before();
    if constexpr (CG == 2) {
        cluster_sync_all();  // the leader's MMAs into the peer's TMEM are complete
        if (warp == 1) tmem_dealloc_cg2(tmem, tmem_cols);
    } else {
        // Push form needs no exit barrier: every CTA waited for all pushes into its own smem
        // (recv_full) before its epilogue, and nothing ever reads a peer's smem.
        __syncthreads();
        if (warp == 1) tmem_dealloc(tmem, tmem_cols);
    }
    KT_END((1ull << 62) | (static_cast<unsigned long long>(p.N & 0xffff) << 40) |
           (static_cast<unsigned long long>(p.K & 0xffff) << 24) |
           ((reinterpret_cast<uintptr_t>(p.out_stats) ^ reinterpret_cast<uintptr_t>(p.row_stats) ^
             reinterpret_cast<uintptr_t>(p.out)) >> 4 & 0xffffff));
    if (threadIdx.x == 0) GM_STAMP(9);
}

// ------------------------------------------------------------------ host side

template <int BN, int STAGES, int MODE, int MT = 1, int CG = 1>
static cudaError_t configure_t() {
    return cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, MODE, MT, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                GemmCfg<BN, STAGES, MT, CG>::SMEM);
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
    if (e == cudaSuccess) e = configure_t<256, 3, kModeGate, 2>();
    if (e == cudaSuccess) e = configure_t<256, 3, kModeBf16, 2>();
    if (e == cudaSuccess) e = configure_t<256, 3, kModeResid, 2>();
    if (e == cudaSuccess) e = configure_t<256, kPairStages, kModeGate, 1, 2>();
    if (e == cudaSuccess) e = configure_t<256, kPairStages, kModeBf16, 1, 2>();
    if (e == cudaSuccess) e = configure_t<256, kPairStages, kModeResid, 1, 2>();
    if (e == cudaSuccess) e = configure_bn<128, 6>();
    if (e == cudaSuccess) e = configure_bn<64, 8>();
    return e;
}

template <int BN, int STAGES, int MODE, int MT = 1, int CG = 1>
static cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, dim3 grid,
                            cudaStream_t stream) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kGemmThreads, 1, 1);
    cfg.dynamicSmemBytes = GemmCfg<BN, STAGES, MT, CG>::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.splits > 1 || CG > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CG;
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
    return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, STAGES, MODE, MT, CG>, ta, tb, p);
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
KT_SETTER(ktrace_set_gemm)

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
    if ((p.flags & kFlagRope) && bn != 256 && !(bn == 128 && (p.flags & kFlagRopePacked))) return cudaErrorInvalidValue;
    if (p.splits < 1 || p.splits > kGemmMaxSplits) return cudaErrorInvalidValue;
    const int mt = p.mt > 1 ? p.mt : 1, cg = p.cg > 1 ? p.cg : 1;
    if (p.persist && p.splits != 1) return cudaErrorInvalidValue;
    static const int warm = [] { const char* e = getenv("PI0B_GEMM_WARM"); return e ? atoi(e) : 1; }();
    GemmParams q = p;
    if (warm) q.flags |= kFlagWarmEpi;
    static const int stage16 = [] { const char* e = getenv("PI0B_GEMM_STAGE_BF16"); return e ? atoi(e) : 1; }();
    if (stage16) q.flags |= kFlagStageBf16;
    if (mt > 1 && (mt != 2 || bn != 256 || p.splits != 1)) return cudaErrorInvalidValue;
    if (cg > 1 && (cg != 2 || mt != 1 || bn != 256 || p.splits != 1)) return cudaErrorInvalidValue;
    dim3 grid((p.M + mt * cg * BM - 1) / (mt * cg * BM), (p.N + bn - 1) / bn, p.splits);
    if (p.persist) {
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        unsigned slots = unsigned(sms / cg);
        if (cg == 2) {  // co-resident CTA pairs (clusters are placed within a GPC)
            static int pairs = -1;
            if (pairs < 0) {
                cudaLaunchConfig_t c{};
                c.gridDim = dim3(2, 1, 1);
                c.blockDim = dim3(kGemmThreads, 1, 1);
                c.dynamicSmemBytes = GemmCfg<256, kPairStages, 1, 2>::SMEM;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeClusterDimension;
                a[0].val.clusterDim.x = 2;
                a[0].val.clusterDim.y = 1;
                a[0].val.clusterDim.z = 1;
                c.attrs = a;
                c.numAttrs = 1;
                int n = 0;
                if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<256, kPairStages, kModeGate, 1, 2>, &c) != cudaSuccess) n = 0;
                pairs = n;
                if (getenv("PI0B_GEMM_DEBUG")) fprintf(stderr, "pi0b: %d co-resident GEMM CTA pairs\n", n);
            }
            if (pairs > 0) slots = std::min(slots, unsigned(pairs));
        }
        grid = dim3(std::min<unsigned>(grid.x * grid.y, slots), 1, 1);
    }
    grid.x *= cg;  // CTA pairs: cluster (2, 1, 1)
    if (cg == 2) {
        switch (p.mode) {
            case kModeGate: return launch_t<256, kPairStages, kModeGate, 1, 2>(ta, tb, q, grid, stream);
            case kModeBf16: return launch_t<256, kPairStages, kModeBf16, 1, 2>(ta, tb, q, grid, stream);
            case kModeResid: return launch_t<256, kPairStages, kModeResid, 1, 2>(ta, tb, q, grid, stream);
            default: return cudaErrorInvalidValue;
        }
    }
    if (mt == 2) {
        switch (p.mode) {
            case kModeGate: return launch_t<256, 3, kModeGate, 2>(ta, tb, q, grid, stream);
            case kModeBf16: return launch_t<256, 3, kModeBf16, 2>(ta, tb, q, grid, stream);
            case kModeResid: return launch_t<256, 3, kModeResid, 2>(ta, tb, q, grid, stream);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (bn) {
        case 256: return launch_bn<256, 4>(ta, tb, q, grid, stream);
        case 128: return launch_bn<128, 6>(ta, tb, q, grid, stream);
        case 64: return launch_bn<64, 8>(ta, tb, q, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
