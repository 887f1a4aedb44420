// tcgen05 flash attention: S = Q K^T and O += P V on the 5th-gen tensor cores with both
// accumulators in TMEM; the online softmax runs out of TMEM with two threads per query row (eight
// softmax warps: warps w and w + 4 share TMEM lane quarter w % 4 and split each 64-key tile), and
// P goes back through shared memory as the A operand of the PV MMA.
//
// Semantics are the reference `Evaluator::attention` (proj/src/evaluate.cpp:225-252): per head
// softmax(Q_h K_{h%kvh}^T / sqrt(d)) V, no mask, keys = rows of [segment 0 ; segment 1]
// (ae.kcat / ae.vcat, proj/src/builder.cpp:321-329).  MQA q-heads of one kv group are stacked
// as query rows; a CTA owns 128 stacked rows.  The running maximum is only moved (and O in
// TMEM rescaled) when it grows by more than 2^8, so O is almost never touched between tiles.
//
// Warps 0-7: softmax + epilogue (row R = 32 (w % 4) + lane, key half / O column half w / 4).
// Warp 8: TMEM allocator + single-thread MMA issuer.  Warp 9: TMA producer for Q, K and V.
// Shared-memory operand layouts are the 128-byte-swizzle UMMA layouts (1024-byte aligned
// regions, 16-byte chunk c of row r at (c ^ (r & 7))):
//   Q  [128 rows x DK]   K-major, one 16 KB region per 64 columns of d      (TMA, 32-row boxes)
//   K  [64 keys  x DK]   K-major B operand of QK^T (N = keys), 8 KB per 64 d (TMA)
//   V  [64 keys  x DV]   same bytes, consumed MN-major as B of PV (N = d)    (TMA)
//   P  [128 rows x 64]   K-major A operand of PV                             (st.shared)
// Key tiles are fetched as 32-row TMA boxes so a tile may straddle the two key segments.
// Key splits (grid.y = S, one (1, S, 1) cluster per q tile): split y owns rows [y 128/S, +128/S)
// of the tile; the other splits push their normalised partials and (max, sum) into its drained
// K ring with st.async (complete_tx on its receive barrier), and it combines them.
// The output tile is staged in shared memory and written with coalesced 16-byte stores.
#include "attention.cuh"
#include "ktrace.cuh"
#include "ptx.cuh"

#include <math.h>

#include <cstdlib>

namespace pi0b {

namespace {

constexpr int kFaRows = 128;
constexpr int kFaKeys = 64;

PI0B_DEV uint64_t desc_kmajor(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t(saddr) >> 4) & 0x3FFFull;
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// MN-major SW128: 64-element MN atoms `lbo` bytes apart, 8-row K groups 1024 bytes apart.
PI0B_DEV uint64_t desc_mnmajor(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t(saddr) >> 4) & 0x3FFFull;
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

PI0B_DEV void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

PI0B_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace

// Timeline instrumentation (variant builds only, -DPI0B_FA_TRACE; scripts/fa_trace.py): 16
// globaltimer stamps per CTA into the buffer set by pi0b_fa_trace_buffer().
#ifdef PI0B_FA_TRACE
__device__ unsigned long long* g_fa_trace;
#define FA_STAMP(i)                                                                                      \
    do {                                                                                                 \
        if (g_fa_trace) {                                                                                \
            unsigned long long t_;                                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
            g_fa_trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + (i)] = t_; \
        }                                                                                                \
    } while (0)
extern "C" int pi0b_fa_trace_buffer(unsigned long long* p) {
    return int(cudaMemcpyToSymbol(g_fa_trace, &p, sizeof(p)));
}
#else
#define FA_STAMP(i) \
    do {            \
    } while (0)
#endif

// D = real head dim, DK = QK contraction (D padded to 16), DV = PV width (D padded to 64),
// KK / KV = key / value ring depths, NQ = softmax threads per query row (each takes KEYS / NQ keys
// of a tile and DV / NQ output columns; 4 x 32 NQ softmax warps, then the MMA and TMA warps).
template <int D, int DK, int DV, int KK, int KV, int KEYS, int NQ>
struct FaCfg {
    static constexpr int SOFT = 128 * NQ;           // softmax / epilogue threads
    static constexpr int THREADS = SOFT + 64;
    static constexpr int MMA_WARP = SOFT / 32, TMA_WARP = MMA_WARP + 1;
    // row-max / row-sum exchange between a row's NQ threads: double-buffered by tile parity at
    // NQ = 2; NQ = 4 single-buffered (shared memory is full) with a second barrier per exchange
    static constexpr int XBUF = NQ == 2 ? 2 : 1;
    static constexpr int QA = (DK + 63) / 64;  // 64-col regions of Q / K
    static constexpr int VA = DV / 64;         // 64-col regions of V
    static constexpr int Q_BYTES = QA * kFaRows * 128;
    static constexpr int K_BYTES = QA * KEYS * 128;
    static constexpr int V_BYTES = VA * KEYS * 128;
    static constexpr int PR = KEYS / 64;                // 64-key regions of a P buffer
    static constexpr int P_BYTES = PR * kFaRows * 128;  // one P buffer; two are allocated
    static constexpr int XCH_BYTES = XBUF * NQ * kFaRows * 4;  // [XBUF][NQ parts][128 rows]
    static constexpr int SMEM = Q_BYTES + KK * K_BYTES + KV * V_BYTES + 2 * P_BYTES + XCH_BYTES + 256;
    static constexpr int TMEM_S = 0;  // two KEYS-column S buffers
    static constexpr int TMEM_O = 2 * KEYS;
    static constexpr int TMEM_COLS = 2 * KEYS + DV <= 256 ? 256 : 512;
    static_assert(2 * KEYS + DV <= 512, "TMEM columns");
    static_assert(KEYS == 64 || KEYS == 128, "key tile");
    static constexpr int ROW_BYTES = DV * 2;  // staged bf16 output row
    static_assert(Q_BYTES >= kFaRows * ROW_BYTES, "output staging fits the Q region");
    // (each thread's S part is read in 32-column TMEM loads)
    static_assert((NQ == 2 || NQ == 4) && (DV / NQ) % 32 == 0 && (KEYS / NQ) % 32 == 0, "softmax split");
};

template <int D, int DK, int DV, int KK, int KV, int KEYS, int NQ>
__global__ void __launch_bounds__(128 * NQ + 64, 1) fattn_kernel(const __grid_constant__ FaMaps maps, const AttnParams p) {
    using C = FaCfg<D, DK, DV, KK, KV, KEYS, NQ>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::Q_BYTES;
    uint8_t* sV = sK + KK * C::K_BYTES;
    uint8_t* sP = sV + KV * C::V_BYTES;
    float* xch = reinterpret_cast<float*>(sP + 2 * C::P_BYTES);  // [XBUF][NQ][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * C::P_BYTES + C::XCH_BYTES);
    uint64_t* k_full = bars;            // [KK]
    uint64_t* k_empty = k_full + KK;    // [KK]
    uint64_t* v_full = k_empty + KK;    // [KV]
    uint64_t* v_empty = v_full + KV;    // [KV]
    uint64_t* s_full = v_empty + KV;    // [2]
    uint64_t* s_free = s_full + 2;      // [2]
    uint64_t* p_full = s_free + 2;      // [2] per P buffer
    uint64_t* o_done = p_full + 2;      // [2] PV of tile t done (buffer t & 1 free again)
    uint64_t* q_full = o_done + 2;      // Q tiles landed (TMA)
    uint64_t* q_ready = q_full + 1;     // Q padding columns cleared (D % 16 != 0)
    uint64_t* peers_free = q_ready + 1; // key splits: every peer's K ring drained and armed
    uint64_t* recv_full = peers_free + 1;  // key splits: the peers' partials of this CTA's rows landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_full + 1);

    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffff, tid >> 5, 0), lane = tid & 31;
    KT_SMEM;
    KT_START();
    if (tid == 0) FA_STAMP(0);
    const int qt = blockIdx.x, grp = blockIdx.z;
    const int hpg = p.heads / p.kv_heads;
    const int grows = hpg * p.q_rows;
    const int kvh = grp;
    const int total = p.rows0 + p.rows1;
    const int pad0 = p.rows0_valid > 0 ? p.rows0_valid : p.rows0;  // first padding key of segment 0
    // Key split (grid.y = S, launched as a (1, S, 1) cluster): this CTA takes key tiles
    // [t0, t0 + ntiles) and finalises rows [y * 128 / S, (y + 1) * 128 / S) of the q tile.
    const int S = gridDim.y, y = int(blockIdx.y);
    const int ntiles_all = (total + KEYS - 1) / KEYS;
    const int tps = (ntiles_all + S - 1) / S;
    const int t0 = y * tps;
    const int ntiles = max(0, min(ntiles_all, t0 + tps) - t0);
    const int own_rows = kFaRows / S;

    if (tid == 0) {
        if (smem_u32(smem) & 1023u) __trap();  // SW128 operand regions need 1024-byte alignment
        for (int s = 0; s < KK; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < KV; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_free[s], C::SOFT);
            mbar_init(&p_full[s], C::SOFT);
            mbar_init(&o_done[s], 1);
        }
        mbar_init(q_full, 1);
        mbar_init(q_ready, 128);
        mbar_init(peers_free, S > 1 ? S - 1 : 1);
        mbar_init(recv_full, 1);
        fence_barrier_init();
    }
    if (warp == C::MMA_WARP) tmem_alloc(tmem_slot, C::TMEM_COLS);
    if (tid == 0) pdl_launch_dependents();
    __syncwarp();  // warp 0 reconverged after thread 0's set-up before the (.aligned) block barrier
    tc_fence_before();
    __syncthreads();  // (key splits touch no peer barrier or shared memory: one cluster barrier in the combine)
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) FA_STAMP(2);

    if (warp == C::TMA_WARP) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            pdl_wait();  // Q, K, V are the previous kernel's outputs
            KT_DEP();
            FA_STAMP(1);
            // Q: 32-row boxes (q_rows % 32 == 0, so a box never straddles two stacked heads)
            int qbytes = 0;
            for (int b = 0; b < kFaRows / 32; ++b)
                if (qt * kFaRows + b * 32 < grows) qbytes += 32 * 128 * C::QA;
            mbar_arrive_expect_tx(q_full, uint32_t(qbytes));
            for (int b = 0; b < kFaRows / 32; ++b) {
                const int g0 = qt * kFaRows + b * 32;
                if (g0 >= grows) break;
                const int head = kvh + p.kv_heads * (g0 / p.q_rows), row0 = g0 % p.q_rows;
                for (int a = 0; a < C::QA; ++a)
                    tma_load_2d(sQ + a * (kFaRows * 128) + b * 32 * 128, &maps.q, q_full, head * D + a * 64, row0,
                                kEvictNormal);
            }
            auto load_rows = [&](bool is_v, uint8_t* dst_tile, int t, int regions) {
                uint64_t* bar = is_v ? &v_full[t % KV] : &k_full[t % KK];
                if (maps.kv_box == 64) {
                    // one key segment: 64-key boxes per region (8 KB boxes: ~85 GB/s of TMA ingest
                    // per SM against ~60 for 32-row boxes; rows past the segment are zero-filled)
                    const CUtensorMap* m = is_v ? &maps.v0 : &maps.k0;
                    for (int b = 0; b < KEYS / 64; ++b)
                        for (int a = 0; a < regions; ++a)
                            tma_load_2d(dst_tile + a * (KEYS * 128) + b * 64 * 128, m, bar, kvh * D + a * 64,
                                        (t0 + t) * KEYS + b * 64, kEvictLast);
                    return;
                }
                // 32-key boxes; each box lies in one key segment (or fully OOB -> zeros)
                for (int half = 0; half < KEYS / 32; ++half) {
                    const int j = (t0 + t) * KEYS + half * 32;
                    const bool seg0 = j < p.rows0;
                    const CUtensorMap* m = seg0 ? (is_v ? &maps.v0 : &maps.k0) : (is_v ? &maps.v1 : &maps.k1);
                    const int row = seg0 ? j : j - p.rows0;
                    for (int a = 0; a < regions; ++a)
                        tma_load_2d(dst_tile + a * (KEYS * 128) + half * 32 * 128, m, bar, kvh * D + a * 64, row, kEvictLast);
                }
            };
            FA_STAMP(10);
            for (int t = 0; t < ntiles; ++t) {
                mbar_wait(&k_empty[t % KK], ((t / KK) & 1) ^ 1);
                mbar_arrive_expect_tx(&k_full[t % KK], C::K_BYTES);
                load_rows(false, sK + (t % KK) * C::K_BYTES, t, C::QA);
                mbar_wait(&v_empty[t % KV], ((t / KV) & 1) ^ 1);
                mbar_arrive_expect_tx(&v_full[t % KV], C::V_BYTES);
                load_rows(true, sV + (t % KV) * C::V_BYTES, t, C::VA);
            }
        }
        __syncwarp();
    } else if (warp == C::MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        {  // warp-uniform loop; one elected lane issues (see gemm.cu)
            constexpr uint32_t idesc_qk = umma_idesc_bf16(kFaRows, KEYS);
            constexpr uint32_t idesc_pv = umma_idesc_bf16(kFaRows, DV) | (1u << 16);  // B (V) MN-major
            const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV), p0 = smem_u32(sP);
            mbar_wait(q_ready, 0);
            auto issue_qk = [&](int t) {
                const int st = t % KK, sb = t & 1;
                mbar_wait(&k_full[st], (t / KK) & 1);
                if (t >= 2) mbar_wait(&s_free[sb], ((t - 2) >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < DK / 16; ++kk) {
                    const uint64_t a = desc_kmajor(q0 + (kk >> 2) * (kFaRows * 128) + (kk & 3) * 32);
                    const uint64_t b = desc_kmajor(k0 + st * C::K_BYTES + (kk >> 2) * (KEYS * 128) + (kk & 3) * 32);
                    if (elect_one()) umma_bf16(tmem + C::TMEM_S + sb * KEYS, a, b, idesc_qk, kk > 0);
                }
                if (elect_one()) {
                    umma_commit(&s_full[sb]);
                    umma_commit(&k_empty[st]);
                }
                __syncwarp();
            };
            if (ntiles > 0) issue_qk(0);
            if (lane == 0) FA_STAMP(11);
            for (int t = 0; t < ntiles; ++t) {
                if (t + 1 < ntiles) issue_qk(t + 1);
                const int sv = t % KV;
                mbar_wait(&v_full[sv], (t / KV) & 1);
                mbar_wait(&p_full[t & 1], (t >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < KEYS / 16; ++kk) {
                    const uint64_t a = desc_kmajor(p0 + (t & 1) * C::P_BYTES + (kk >> 2) * (kFaRows * 128) + (kk & 3) * 32);
                    const uint64_t b = desc_mnmajor(v0 + sv * C::V_BYTES + kk * 2048, KEYS * 128);
                    if (elect_one()) umma_bf16(tmem + C::TMEM_O, a, b, idesc_pv, (t | kk) > 0);
                }
                if (elect_one()) {
                    umma_commit(&o_done[t & 1]);
                    umma_commit(&v_empty[sv]);
                }
                __syncwarp();
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax + epilogue
        const int qd = warp & 3, hf = warp >> 2;  // TMEM lane quarter; key / O-column part (of NQ)
        const int r = qd * 32 + lane;
        const int g = qt * kFaRows + r;
        const bool row_ok = g < grows;
        const uint32_t trow = tmem + (uint32_t(qd * 32) << 16);
        const uint32_t pair_bar = 1 + qd;  // named barrier of the row's NQ warps qd, qd + 4, ..
        mbar_wait(q_full, 0);  // (also orders every thread after the producer's pdl_wait)
        if (hf == 0) {
            // Q columns D..DK of the last region belong to the next head (or are OOB zeros): clear
            // them so the QK contraction over DK = D rounded up to 16 sees only this head.
            if constexpr (D % 64 != 0 && D < DK) {
                constexpr int a = D / 64, c0 = (D % 64) / 8, c1 = (DK - 64 * a + 7) / 8;
#pragma unroll
                for (int c = c0; c < c1; ++c)
                    *reinterpret_cast<uint4*>(sQ + a * (kFaRows * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = make_uint4(0u, 0u, 0u, 0u);
                fence_proxy_async();
            }
            mbar_arrive(q_ready);
        }
        float m_ref = -INFINITY, l = 0.f;
        for (int t = 0; t < ntiles; ++t) {
            const int sb = t & 1;
            mbar_wait(&s_full[sb], (t >> 1) & 1);
            if (tid == 0 && t == 0) FA_STAMP(3);
            tc_fence_after();
            constexpr int KH = KEYS / NQ;  // keys of this thread's part of the tile
            float sv[KH];
#pragma unroll
            for (int i = 0; i < KH / 32; ++i)
                tmem_ld32(trow + C::TMEM_S + sb * KEYS + hf * KH + i * 32, *reinterpret_cast<float(*)[32]>(sv + i * 32));
            tc_fence_before();
            mbar_arrive(&s_free[sb]);
            const int kbase = (t0 + t) * KEYS + hf * KH;
            float mx = -INFINITY;
            // keys past the end, and the padding keys [pad0, rows0) of segment 0, are masked; a
            // tile that has neither (the common case) takes the unmasked loop
            if (kbase + KH <= total && (kbase + KH <= pad0 || kbase >= p.rows0)) {
#pragma unroll
                for (int j = 0; j < KH; ++j) {
                    sv[j] *= p.scale_log2;
                    mx = fmaxf(mx, sv[j]);
                }
            } else {
                const int end = total - kbase, lo = pad0 - kbase, hi = p.rows0 - kbase;
#pragma unroll
                for (int j = 0; j < KH; ++j) {
                    sv[j] = j < end && (j < lo || j >= hi) ? sv[j] * p.scale_log2 : -INFINITY;
                    mx = fmaxf(mx, sv[j]);
                }
            }
            // row max over the NQ key parts (the row's other threads are in warps w +- 4 ..)
            const int xb0 = C::XBUF == 2 ? sb * NQ : 0;
            xch[(xb0 + hf) * kFaRows + r] = mx;
            named_bar_sync(pair_bar, NQ * 32);
#pragma unroll
            for (int h = 0; h < NQ; ++h) mx = fmaxf(mx, xch[(xb0 + h) * kFaRows + r]);
            if (C::XBUF == 1) named_bar_sync(pair_bar, NQ * 32);  // all read before the next write
            // P is double-buffered: buffer t & 1 is free once PV(t - 2) is done; O may only be
            // rescaled once PV(t - 1) is done (rare: lazy rescale).  Both threads of a row make
            // the same decisions (same maxima).
            float factor = 1.f;
            const bool grow = mx > m_ref + 8.f;
            if (grow) {
                factor = exp2f(m_ref - mx);  // 0 on the first tile
                m_ref = mx;
                l *= factor;
            }
            const bool rescale = t > 0 && __any_sync(0xffffffff, grow);
            if (rescale) {
                mbar_wait(&o_done[(t - 1) & 1], ((t - 1) >> 1) & 1);
                tc_fence_after();
            } else if (t >= 2) {
                mbar_wait(&o_done[t & 1], ((t - 2) >> 1) & 1);
            }
            if (rescale) {
#pragma unroll 1
                for (int c = 0; c < DV / (32 * NQ); ++c) {
                    float o[32];
                    tmem_ld32(trow + C::TMEM_O + hf * (DV / NQ) + c * 32, o);
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] *= factor;
                    tmem_st32(trow + C::TMEM_O + hf * (DV / NQ) + c * 32, o);
                }
            }
            float ls = 0.f;
            uint32_t pk[KH / 2];
#pragma unroll
            for (int j = 0; j < KH; j += 2) {
                const float a0 = ex2_fast(sv[j] - m_ref), a1 = ex2_fast(sv[j + 1] - m_ref);
                ls += a0 + a1;
                pk[j / 2] = pack_bf16(a0, a1);
            }
            l += ls;
            // P [128 rows x KEYS] as KEYS / 64 regions of [128 rows x 128 B]; this thread's keys
            // [hf KH, +KH) are 16-byte chunks kq = hf KH / 8 + c (region kq / 8, chunk kq % 8)
#pragma unroll
            for (int c = 0; c < KH / 8; ++c) {
                const int kq = hf * (KH / 8) + c;
                *reinterpret_cast<uint4*>(sP + sb * C::P_BYTES + (kq >> 3) * (kFaRows * 128) + r * 128 + (((kq & 7) ^ (r & 7)) << 4)) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            }
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&p_full[sb]);
        }
        if (tid == 0) FA_STAMP(4);
        // row sum over the NQ parts (XBUF 2: the slot of a tile two back is free, see the max
        // exchange; XBUF 1: the last max exchange ended with a barrier)
        {
            const int xb0 = C::XBUF == 2 ? (ntiles & 1) * NQ : 0;
            xch[(xb0 + hf) * kFaRows + r] = l;
            named_bar_sync(pair_bar, NQ * 32);
            l = 0.f;
#pragma unroll
            for (int h = 0; h < NQ; ++h) l += xch[(xb0 + h) * kFaRows + r];
        }
        if (ntiles > 0) mbar_wait(&o_done[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
        tc_fence_after();
        if (tid == 0) FA_STAMP(5);
        // This thread's output columns: [hf * DV / NQ, (hf + 1) * DV / NQ) of row r, as 16-byte
        // chunks q of the staged row (bf16, row r at r * ROW_BYTES, chunk q at (q ^ (r & 7))).
        constexpr int HC = DV / NQ / 8;  // chunks per row part
        auto stage_row = [&](int row, const float* o, int c32, float scale) {
            uint8_t* srow = sQ + row * C::ROW_BYTES;
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
                const int q = hf * HC + (c32 * 32 + j) / 8;
                *reinterpret_cast<uint4*>(srow + ((q ^ (row & 7)) << 4)) =
                    make_uint4(pack_bf16(o[j] * scale, o[j + 1] * scale), pack_bf16(o[j + 2] * scale, o[j + 3] * scale),
                               pack_bf16(o[j + 4] * scale, o[j + 5] * scale), pack_bf16(o[j + 6] * scale, o[j + 7] * scale));
            }
        };
        int row_lo = 0, row_hi = kFaRows;  // rows this CTA writes out
        if (S == 1) {
            const float il = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
            for (int c = 0; c < DV / (32 * NQ); ++c) {
                float o[32];
                if (ntiles > 0) tmem_ld32(trow + C::TMEM_O + hf * (DV / NQ) + c * 32, o);
                else
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] = 0.f;
                stage_row(r, o, c, il);
            }
        } else {
            // ---------------- key-split combine through L2
            // Every split stages the normalised partial rows it does not own (bf16) and their
            // (max, sum) in its drained V ring, one contiguous block per owner, and writes the
            // blocks to the global workspace with coalesced stores; after one cluster barrier
            // (release / acquire: the blocks are visible) each split copies the blocks of its own
            // rows into its drained K ring and combines them.  Block = own_rows rows of ROW_BYTES
            // (16-byte chunk q of local row i at q ^ (i & 7)) followed by own_rows (max, sum)
            // pairs.  (Pushing the same blocks into the owners' smem with DSMEM bulk copies took
            // ~4.6 us at S = 4 -- scripts/fa_trace.py, round 2 -- against ~1 us through L2.)
            row_lo = y * own_rows;
            row_hi = row_lo + own_rows;
            const int blk = own_rows * (C::ROW_BYTES + 8);
            auto slot_of = [&](int sender, int owner_rank) { return sender < owner_rank ? sender : sender - 1; };
            uint8_t* wsb = static_cast<uint8_t*>(p.ws) + size_t(blockIdx.z * gridDim.x + blockIdx.x) * S * S * blk;
            const int owner = r / own_rows, lrow = r - owner * own_rows;
            // TMEM reads stay warp-converged (tcgen05.ld is .sync.aligned; with 8+ splits a warp
            // spans two owners): every thread stages its normalised partial, into the outgoing
            // block of its row's owner or, for its own rows, into the idle half of the Q region.
            const float il = l > 0.f ? 1.f / l : 0.f;
            uint8_t* ob = owner != y ? sV + slot_of(owner, y) * blk                              // outgoing
                                     : sQ + (row_lo < kFaRows / 2 ? kFaRows / 2 : 0) * C::ROW_BYTES;  // own
#pragma unroll 1
            for (int c = 0; c < DV / (32 * NQ); ++c) {
                float o[32];
                if (ntiles > 0) tmem_ld32(trow + C::TMEM_O + hf * (DV / NQ) + c * 32, o);
                else
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] = 0.f;  // a split without keys never reads TMEM
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    const int q = hf * HC + (c * 32 + j) / 8;
                    *reinterpret_cast<uint4*>(ob + lrow * C::ROW_BYTES + ((q ^ (lrow & 7)) << 4)) =
                        make_uint4(pack_bf16(o[j] * il, o[j + 1] * il), pack_bf16(o[j + 2] * il, o[j + 3] * il),
                                   pack_bf16(o[j + 4] * il, o[j + 5] * il), pack_bf16(o[j + 6] * il, o[j + 7] * il));
                }
            }
            if (hf == 0)  // (max, sum) of every row: into the outgoing block, or for own rows into sP + 2 KB
                (owner != y ? reinterpret_cast<float2*>(ob + own_rows * C::ROW_BYTES) : reinterpret_cast<float2*>(sP + 2048))[lrow] =
                    make_float2(l > 0.f ? m_ref : -INFINITY, l);
            named_bar_sync(6, C::SOFT);
            if (tid == 0) FA_STAMP(14);
            // outgoing blocks -> workspace [tile][sender][owner]
            for (int k = 0; k < S; ++k) {
                if (k == y) continue;
                const uint4* src = reinterpret_cast<const uint4*>(sV + slot_of(k, y) * blk);
                uint4* dst = reinterpret_cast<uint4*>(wsb + size_t(y * S + k) * blk);
                for (int e = tid; e < blk / 16; e += C::SOFT) dst[e] = src[e];
            }
            if (tid == 0) FA_STAMP(7);
            cluster_sync_all();  // (warps 8 and 9 arrive at the end of their roles)
            if (tid == 0) FA_STAMP(15);
            // incoming blocks of this split's rows -> the drained K ring
            for (int k = 0; k < S; ++k) {
                if (k == y) continue;
                const uint8_t* src = wsb + size_t(k * S + y) * blk;
                uint8_t* dst = sK + slot_of(k, y) * blk;
                for (int e = tid; e < blk / 16; e += C::SOFT) cp_async16(dst + e * 16, src + e * 16, true);
            }
            cp_async_commit();
            cp_async_wait<0>();
            named_bar_sync(6, C::SOFT);
            // o = sum_j w_j O_j / sum_j w_j over the S normalised partials, w_j = l_j 2^(m_j - M),
            // spread over all softmax threads (own_rows rows x DV columns; a per-row-thread combine
            // leaves the work to the warps of one sub-partition)
            if (tid < own_rows * min(C::SOFT / own_rows, DV / 8)) {
                constexpr int DVC = DV / 8;                       // 16-byte chunks per row
                const int segs = min(C::SOFT / own_rows, DVC);    // threads per row
                const int cps = DVC / segs;                       // chunks per thread
                const int lr = tid / segs, c0 = (tid % segs) * cps;
                const float2* ml_own = reinterpret_cast<const float2*>(sP + 2048);
                auto ml_of = [&](int k) {
                    return k == y ? ml_own[lr] : reinterpret_cast<const float2*>(sK + slot_of(k, y) * blk + own_rows * C::ROW_BYTES)[lr];
                };
                float M = -INFINITY;
                for (int k = 0; k < S; ++k) M = fmaxf(M, ml_of(k).x);
                float wk[8], den = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    wk[k] = 0.f;
                    if (k < S) {
                        const float2 v = ml_of(k);
                        wk[k] = v.y > 0.f ? v.y * exp2f(v.x - M) : 0.f;
                        den += wk[k];
                    }
                }
                const float iden = den > 0.f ? 1.f / den : 0.f;
                const uint8_t* own_src = sQ + (row_lo < kFaRows / 2 ? kFaRows / 2 : 0) * C::ROW_BYTES;
                const int rr = row_lo + lr;  // tile row of the output
#pragma unroll 1
                for (int cc = 0; cc < cps; ++cc) {
                    const int q = c0 + cc;
                    float o[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[e] = 0.f;
#pragma unroll 1
                    for (int k = 0; k < S; ++k) {
                        const uint8_t* src = (k == y ? own_src : sK + slot_of(k, y) * blk) + lr * C::ROW_BYTES;
                        const uint4 u = *reinterpret_cast<const uint4*>(src + ((q ^ (lr & 7)) << 4));
                        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            o[2 * e] += wk[k] * __uint_as_float(w4[e] << 16);
                            o[2 * e + 1] += wk[k] * __uint_as_float(w4[e] & 0xffff0000u);
                        }
                    }
                    *reinterpret_cast<uint4*>(sQ + rr * C::ROW_BYTES + ((q ^ (rr & 7)) << 4)) =
                        make_uint4(pack_bf16(o[0] * iden, o[1] * iden), pack_bf16(o[2] * iden, o[3] * iden),
                                   pack_bf16(o[4] * iden, o[5] * iden), pack_bf16(o[6] * iden, o[7] * iden));
                }
                if (tid == 0) FA_STAMP(8);
            }
        }
        if (tid == 0) FA_STAMP(6);
        // coalesced copy-out of the staged rows [row_lo, row_hi): D bf16 of each row.  Each row's
        // global address (stacked head -> head, row) is computed once, into a table in the P
        // buffers (free: every PV MMA is done), so the copy loop has no integer divisions.
        __nv_bfloat16** rowptr = reinterpret_cast<__nv_bfloat16**>(sP);
        if (tid < kFaRows) {
            const int gg = qt * kFaRows + tid;
            rowptr[tid] = gg < grows ? p.out + (long long)(gg % p.q_rows) * p.ldo + (kvh + p.kv_heads * (gg / p.q_rows)) * D
                                     : nullptr;
        }
        named_bar_sync(5, C::SOFT);
        if (tid == 0) FA_STAMP(12);
        constexpr int CPR = (D * 2 + 15) / 16;  // 16-byte chunks per output row
        if constexpr (CPR == 32) {  // D = 256: one row per warp and iteration, lane = chunk
            for (int rr = row_lo + warp; rr < row_hi; rr += C::SOFT / 32) {
                __nv_bfloat16* orow = rowptr[rr];
                if (!orow) continue;
                const uint4 v = *reinterpret_cast<const uint4*>(sQ + rr * C::ROW_BYTES + ((lane ^ (rr & 7)) << 4));
                *reinterpret_cast<uint4*>(orow + lane * 8) = v;
            }
        } else {
            const int n = (row_hi - row_lo) * CPR;
            for (int e = tid; e < n; e += C::SOFT) {
                const int rr = row_lo + e / CPR, q = e - (e / CPR) * CPR;
                __nv_bfloat16* orow = rowptr[rr];
                if (!orow) continue;
                const uint4 v = *reinterpret_cast<const uint4*>(sQ + rr * C::ROW_BYTES + ((q ^ (rr & 7)) << 4));
                *reinterpret_cast<uint4*>(orow + q * 8) = v;
            }
        }
        if (tid == 0) FA_STAMP(13);
        (void)row_ok;
    }
    // Key splits: the MMA and TMA warps take part in the softmax warps' cluster barrier (the
    // workspace exchange above); nothing crosses CTAs after it.
    tc_fence_before();
    if (S > 1 && warp >= C::MMA_WARP) cluster_sync_all();
    __syncthreads();
    if (tid == 0) FA_STAMP(9);
    KT_END((2ull << 62) | (static_cast<unsigned long long>(D) << 40) | (reinterpret_cast<uintptr_t>(p.out) >> 4 & 0xffffff));
    if (warp == C::MMA_WARP) tmem_dealloc(tmem, C::TMEM_COLS);
}

CUtensorMap make_tmap_bf16(const void* base, long long rows, long long cols, long long ld, int box_rows);

namespace {
template <int D, int DK, int DV, int KK, int KV, int KEYS, int NQ>
cudaError_t fa_configure_t() {
    return cudaFuncSetAttribute(fattn_kernel<D, DK, DV, KK, KV, KEYS, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                FaCfg<D, DK, DV, KK, KV, KEYS, NQ>::SMEM);
}
}  // namespace

cudaError_t fattn_configure() {
    cudaError_t e = fa_configure_t<72, 80, 128, 3, 3, 64, 2>();
    if (e == cudaSuccess) e = fa_configure_t<72, 80, 128, 2, 2, 128, 2>();
    if (e == cudaSuccess) e = fa_configure_t<72, 80, 128, 2, 2, 128, 4>();
    if (e == cudaSuccess) e = fa_configure_t<256, 256, 256, 2, 2, 64, 2>();
    return e;
}

// d = 72 (SigLIP): 128-key tiles by default -- the QK^T MMA costs the same ~86 cycles at N = 64
// and N = 128, so a 128-key tile halves its issue time per key and the per-tile softmax
// exchanges (PI0B_FA72_KEYS=64: the 64-key tiles with 3-deep rings).  d = 256 keeps 64-key tiles
// (a 128-key tile does not fit shared memory next to its 64 KB Q tile).
static int fa72_keys() {
    static const int k = [] {
        const char* e = std::getenv("PI0B_FA72_KEYS");
        return e && std::atoi(e) == 64 ? 64 : 128;
    }();
    return k;
}
// d = 72, 128-key tiles: softmax threads per query row (PI0B_FA72_NQ, 2 or 4).
static int fa72_nq() {
    static const int k = [] {
        const char* e = std::getenv("PI0B_FA72_NQ");
        return e && std::atoi(e) == 2 ? 2 : 4;
    }();
    return k;
}

// Tensor maps for one attention launch (built once at plan time).
FaMaps make_fattn_maps(const AttnParams& p, int head_dim) {
    FaMaps m;
    m.q = make_tmap_bf16(p.q, p.q_rows, (long long)p.heads * head_dim, p.ldq, 32);
    const long long width = (long long)p.kv_heads * head_dim;
    const bool one_seg = p.rows1 == 0 || !p.k1;
    m.kv_box = one_seg ? 64 : 32;
    m.k0 = make_tmap_bf16(p.k0, p.rows0, width, p.ld0, m.kv_box);
    m.v0 = make_tmap_bf16(p.v0, p.rows0, width, p.ld0, m.kv_box);
    const bool has1 = p.rows1 > 0 && p.k1;
    m.k1 = make_tmap_bf16(has1 ? p.k1 : p.k0, has1 ? p.rows1 : p.rows0, width, has1 ? p.ld1 : p.ld0, 32);
    m.v1 = make_tmap_bf16(has1 ? p.v1 : p.v0, has1 ? p.rows1 : p.rows0, width, has1 ? p.ld1 : p.ld0, 32);
    return m;
}

static bool g_fa_pdl = true;
void fattn_set_pdl(bool on) { g_fa_pdl = on; }

template <int D, int DK, int DV, int KK, int KV, int KEYS, int NQ>
static cudaError_t fa_launch_t(const FaMaps& maps, const AttnParams& p, dim3 grid, cudaStream_t stream) {
    using C = FaCfg<D, DK, DV, KK, KV, KEYS, NQ>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (g_fa_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (grid.y > 1) {  // key splits of one q tile form a cluster (co-scheduled; one cluster barrier)
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = grid.y;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fattn_kernel<D, DK, DV, KK, KV, KEYS, NQ>, maps, p);
}

// grid = (stacked q tiles of 128, key splits (p.kv_splits: 1, 2, 4 or 8), kv groups).
cudaError_t launch_fattn(int head_dim, const FaMaps& maps, const AttnParams& p, cudaStream_t stream) {
    const int grows = (p.heads / p.kv_heads) * p.q_rows;
    const int S = p.kv_splits > 1 ? p.kv_splits : 1;
    if (S != 1 && S != 2 && S != 4 && S != 8) return cudaErrorInvalidValue;
    const dim3 grid((grows + kFaRows - 1) / kFaRows, S, p.kv_heads);
    // 32-key boxes may not straddle the two key segments; one segment is read in 64-row boxes
    // whose rows past the segment are zero-filled (and masked), so its length is free
    if ((p.rows1 > 0 && (p.rows0 % 32)) || (p.rows1 % 32) || (p.q_rows % 32)) return cudaErrorInvalidValue;
    switch (head_dim) {
        case 72:
            if (fa72_keys() == 64) return fa_launch_t<72, 80, 128, 3, 3, 64, 2>(maps, p, grid, stream);
            return fa72_nq() == 4 ? fa_launch_t<72, 80, 128, 2, 2, 128, 4>(maps, p, grid, stream)
                                  : fa_launch_t<72, 80, 128, 2, 2, 128, 2>(maps, p, grid, stream);
        case 256: return fa_launch_t<256, 256, 256, 2, 2, 64, 2>(maps, p, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

KT_SETTER(ktrace_set_fattn)

}  // namespace pi0b
