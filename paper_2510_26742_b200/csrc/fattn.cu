// tcgen05 flash attention: S = Q K^T and O += P V on the 5th-gen tensor cores with both
// accumulators in TMEM; the online softmax runs one query row per thread straight out of
// TMEM (no shuffles), and P goes back through shared memory as the A operand of the PV MMA.
//
// Semantics are the reference `Evaluator::attention` (proj/src/evaluate.cpp:225-252): per head
// softmax(Q_h K_{h%kvh}^T / sqrt(d)) V, no mask, keys = rows of [segment 0 ; segment 1]
// (ae.kcat / ae.vcat, proj/src/builder.cpp:321-329).  MQA q-heads of one kv group are stacked
// as query rows; a CTA owns 128 stacked rows.  The running maximum is only moved (and O in
// TMEM rescaled) when it grows by more than 2^8, so O is almost never touched between tiles.
//
// Warps 0-3: softmax + epilogue, thread t = query row t = TMEM lane t (they also stage Q).
// Warp 4: TMEM allocator + single-thread MMA issuer.  Warp 5: TMA producer for K and V.
// Shared-memory operand layouts are the 128-byte-swizzle UMMA layouts (1024-byte aligned
// regions, 16-byte chunk c of row r at (c ^ (r & 7))):
//   Q  [128 rows x DK]   K-major, one 16 KB region per 64 columns of d      (cp.async)
//   K  [64 keys  x DK]   K-major B operand of QK^T (N = keys), 8 KB per 64 d (TMA)
//   V  [64 keys  x DV]   same bytes, consumed MN-major as B of PV (N = d)    (TMA)
//   P  [128 rows x 64]   K-major A operand of PV                             (st.shared)
// Key tiles are fetched as 32-row TMA boxes so a tile may straddle the two key segments.
#include "attention.cuh"
#include "ptx.cuh"

#include <math.h>

namespace pi0b {

namespace {

constexpr int kFaRows = 128;
constexpr int kFaKeys = 64;
constexpr int kFaThreads = 192;

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

struct FaMaps {
    CUtensorMap k0, v0, k1, v1;  // [rows, kv_heads*D] bf16, box {64 cols, 32 rows}, 128B swizzle
};

// D = real head dim, DK = QK contraction (D padded to 16), DV = PV width (D padded to 64),
// KK / KV = key / value ring depths.
template <int D, int DK, int DV, int KK, int KV>
struct FaCfg {
    static constexpr int QA = (DK + 63) / 64;  // 64-col regions of Q / K
    static constexpr int VA = DV / 64;         // 64-col regions of V
    static constexpr int Q_BYTES = QA * kFaRows * 128;
    static constexpr int K_BYTES = QA * kFaKeys * 128;
    static constexpr int V_BYTES = VA * kFaKeys * 128;
    static constexpr int P_BYTES = kFaRows * 128;  // one P buffer; two are allocated
    static constexpr int SMEM = Q_BYTES + KK * K_BYTES + KV * V_BYTES + 2 * P_BYTES + 256 + 1024;
    static constexpr int TMEM_S = 0;  // two 64-column S buffers
    static constexpr int TMEM_O = 128;
    static constexpr int TMEM_COLS = 128 + DV <= 256 ? 256 : 512;
};

template <int D, int DK, int DV, int KK, int KV>
__global__ void __launch_bounds__(kFaThreads, 1) fattn_kernel(const __grid_constant__ FaMaps maps, const AttnParams p) {
    using C = FaCfg<D, DK, DV, KK, KV>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::Q_BYTES;
    uint8_t* sV = sK + KK * C::K_BYTES;
    uint8_t* sP = sV + KV * C::V_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * C::P_BYTES);
    uint64_t* k_full = bars;            // [KK]
    uint64_t* k_empty = k_full + KK;    // [KK]
    uint64_t* v_full = k_empty + KK;    // [KV]
    uint64_t* v_empty = v_full + KV;    // [KV]
    uint64_t* s_full = v_empty + KV;    // [2]
    uint64_t* s_free = s_full + 2;      // [2]
    uint64_t* p_full = s_free + 2;      // [2] per P buffer
    uint64_t* o_done = p_full + 2;      // [2] PV of tile t done (buffer t & 1 free again)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffff, tid >> 5, 0), lane = tid & 31;
    const int qt = blockIdx.x, grp = blockIdx.z;
    const int hpg = p.heads / p.kv_heads;
    const int grows = hpg * p.q_rows;
    const int kvh = grp;
    const int total = p.rows0 + p.rows1;
    // Key split (grid.y = S, launched as a (1, S, 1) cluster): this CTA takes key tiles
    // [t0, t0 + ntiles); the partial outputs are combined over DSMEM at the end.
    const int S = gridDim.y;
    const int ntiles_all = (total + kFaKeys - 1) / kFaKeys;
    const int tps = (ntiles_all + S - 1) / S;
    const int t0 = int(blockIdx.y) * tps;
    const int ntiles = max(0, min(ntiles_all, t0 + tps) - t0);

    if (tid == 0) {
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
            mbar_init(&s_free[s], 128);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&p_full[s], 128);
            mbar_init(&o_done[s], 1);
        }
        fence_barrier_init();
    }
    if (warp == 4) tmem_alloc(tmem_slot, C::TMEM_COLS);
    if (tid == 0) pdl_launch_dependents();
    pdl_wait();  // every input (Q, K, V) is the previous kernel's output
    if (warp < 4) {
        // Q: thread r stages its own stacked row (DK/8 chunks) into the swizzled layout
        const int r = tid, g = qt * kFaRows + r;
        const __nv_bfloat16* qrow = p.q;
        const bool row_ok = g < grows;
        if (row_ok) qrow = p.q + (long long)(g % p.q_rows) * p.ldq + (kvh + p.kv_heads * (g / p.q_rows)) * D;
#pragma unroll
        for (int c = 0; c < DK / 8; ++c) {
            const bool ok = row_ok && c * 8 < D;
            cp_async16(sQ + (c >> 3) * (kFaRows * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4), ok ? qrow + c * 8 : p.q,
                       ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        fence_proxy_async();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 5) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            auto load_rows = [&](bool is_v, uint8_t* dst_tile, int t, int regions) {
                // two 32-key boxes per region; each box lies in one key segment (or fully OOB -> zeros)
                for (int half = 0; half < 2; ++half) {
                    const int j = (t0 + t) * kFaKeys + half * 32;
                    const bool seg0 = j < p.rows0;
                    const CUtensorMap* m = seg0 ? (is_v ? &maps.v0 : &maps.k0) : (is_v ? &maps.v1 : &maps.k1);
                    const int row = seg0 ? j : j - p.rows0;
                    for (int a = 0; a < regions; ++a)
                        tma_load_2d(dst_tile + a * (kFaKeys * 128) + half * 32 * 128, m,
                                    is_v ? &v_full[t % KV] : &k_full[t % KK], kvh * D + a * 64, row, kEvictLast);
                }
            };
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
    } else if (warp == 4) {
        // ------------------------------------------------------------ MMA issuer
        {  // warp-uniform loop; one elected lane issues (see gemm.cu)
            constexpr uint32_t idesc_qk = umma_idesc_bf16(kFaRows, kFaKeys);
            constexpr uint32_t idesc_pv = umma_idesc_bf16(kFaRows, DV) | (1u << 16);  // B (V) MN-major
            const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV), p0 = smem_u32(sP);
            auto issue_qk = [&](int t) {
                const int st = t % KK, sb = t & 1;
                mbar_wait(&k_full[st], (t / KK) & 1);
                if (t >= 2) mbar_wait(&s_free[sb], ((t - 2) >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < DK / 16; ++kk) {
                    const uint64_t a = desc_kmajor(q0 + (kk >> 2) * (kFaRows * 128) + (kk & 3) * 32);
                    const uint64_t b = desc_kmajor(k0 + st * C::K_BYTES + (kk >> 2) * (kFaKeys * 128) + (kk & 3) * 32);
                    if (elect_one()) umma_bf16(tmem + C::TMEM_S + sb * 64, a, b, idesc_qk, kk > 0);
                }
                if (elect_one()) {
                    umma_commit(&s_full[sb]);
                    umma_commit(&k_empty[st]);
                }
                __syncwarp();
            };
            if (ntiles > 0) issue_qk(0);
            for (int t = 0; t < ntiles; ++t) {
                if (t + 1 < ntiles) issue_qk(t + 1);
                const int sv = t % KV;
                mbar_wait(&v_full[sv], (t / KV) & 1);
                mbar_wait(&p_full[t & 1], (t >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kFaKeys / 16; ++kk) {
                    const uint64_t a = desc_kmajor(p0 + (t & 1) * C::P_BYTES + kk * 32);
                    const uint64_t b = desc_mnmajor(v0 + sv * C::V_BYTES + kk * 2048, kFaKeys * 128);
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
        const int r = tid;
        const int g = qt * kFaRows + r;
        const bool row_ok = g < grows;
        const uint32_t trow = tmem + (uint32_t(warp * 32) << 16);
        float m_ref = -INFINITY, l = 0.f;
        for (int t = 0; t < ntiles; ++t) {
            const int sb = t & 1;
            mbar_wait(&s_full[sb], (t >> 1) & 1);
            tc_fence_after();
            float s0[32], s1[32];
            tmem_ld32(trow + C::TMEM_S + sb * 64, s0);
            tmem_ld32(trow + C::TMEM_S + sb * 64 + 32, s1);
            tc_fence_before();
            mbar_arrive(&s_free[sb]);
            const int kbase = (t0 + t) * kFaKeys;
            float mx = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                s0[j] = kbase + j < total ? s0[j] * p.scale_log2 : -INFINITY;
                s1[j] = kbase + 32 + j < total ? s1[j] * p.scale_log2 : -INFINITY;
                mx = fmaxf(mx, fmaxf(s0[j], s1[j]));
            }
            // P is double-buffered: buffer t & 1 is free once PV(t - 2) is done; O may only be
            // rescaled once PV(t - 1) is done (rare: lazy rescale)
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
                for (int c = 0; c < DV / 32; ++c) {
                    float o[32];
                    tmem_ld32(trow + C::TMEM_O + c * 32, o);
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] *= factor;
                    tmem_st32(trow + C::TMEM_O + c * 32, o);
                }
            }
            float ls = 0.f;
            uint32_t pk[32];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const float a0 = ex2_fast(s0[j] - m_ref), a1 = ex2_fast(s0[j + 1] - m_ref);
                const float b0 = ex2_fast(s1[j] - m_ref), b1 = ex2_fast(s1[j + 1] - m_ref);
                ls += a0 + a1 + b0 + b1;
                pk[j / 2] = pack_bf16(a0, a1);
                pk[16 + j / 2] = pack_bf16(b0, b1);
            }
            l += ls;
            uint8_t* prow = sP + (t & 1) * C::P_BYTES + r * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&p_full[t & 1]);
        }
        // epilogue: O / l -> bf16
        if (ntiles > 0) mbar_wait(&o_done[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
        tc_fence_after();
        const float il = l > 0.f ? 1.f / l : 0.f;
        if (S > 1) {
            // park this split's normalised partial (bf16, row r at r * DV * 2, 16-byte chunks
            // swizzled by r & 7) in the now idle K ring, (m, l) in the P buffers
            uint8_t* prow = sK + r * (DV * 2);
#pragma unroll 1
            for (int c = 0; c < DV / 32; ++c) {
                float o[32];
                if (ntiles > 0) tmem_ld32(trow + C::TMEM_O + c * 32, o);
                else
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] = 0.f;
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    uint4 u;
                    u.x = pack_bf16(o[j] * il, o[j + 1] * il);
                    u.y = pack_bf16(o[j + 2] * il, o[j + 3] * il);
                    u.z = pack_bf16(o[j + 4] * il, o[j + 5] * il);
                    u.w = pack_bf16(o[j + 6] * il, o[j + 7] * il);
                    *reinterpret_cast<uint4*>(prow + ((((c * 32 + j) >> 3) ^ (r & 7)) << 4)) = u;
                }
            }
            reinterpret_cast<float2*>(sP)[r] = make_float2(l > 0.f ? m_ref : -INFINITY, l);
        }
        __nv_bfloat16* orow = p.out;
        if (row_ok) orow = p.out + (long long)(g % p.q_rows) * p.ldo + (kvh + p.kv_heads * (g / p.q_rows)) * D;
#pragma unroll 1
        for (int c = 0; c < (S > 1 ? 0 : DV / 32); ++c) {
            float o[32];
            tmem_ld32(trow + C::TMEM_O + c * 32, o);
            if (row_ok) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    if (c * 32 + j < D) {
                        uint4 u;
                        u.x = pack_bf16(o[j] * il, o[j + 1] * il);
                        u.y = pack_bf16(o[j + 2] * il, o[j + 3] * il);
                        u.z = pack_bf16(o[j + 4] * il, o[j + 5] * il);
                        u.w = pack_bf16(o[j + 6] * il, o[j + 7] * il);
                        *reinterpret_cast<uint4*>(orow + c * 32 + j) = u;
                    }
                }
            }
        }
    }
    if (S > 1) {
        // Combine the S key splits of this q tile: CTA y of the cluster finalises rows
        // [y * 128 / S, (y + 1) * 128 / S): o = sum_j w_j O_j / sum_j w_j, w_j = l_j 2^(m_j - M),
        // reading the peers' parked partials over DSMEM.
        cluster_sync_all();
        const int rows = kFaRows / S, r0 = int(blockIdx.y) * rows;
        float* wts = reinterpret_cast<float*>(sQ);  // [rows][S] normalised weights (Q is idle)
        for (int i = tid; i < rows; i += kFaThreads) {
            const int r = r0 + i;
            float m[8], l[8], M = -INFINITY, den = 0.f;
            for (int j = 0; j < S; ++j) {
                const float4 v = ld_dsmem_f32x4(mapa_shared(smem_u32(sP) + (r & ~1) * 8, j));
                m[j] = (r & 1) ? v.z : v.x;
                l[j] = (r & 1) ? v.w : v.y;
                M = fmaxf(M, m[j]);
            }
            for (int j = 0; j < S; ++j) {
                const float w = l[j] > 0.f ? l[j] * exp2f(m[j] - M) : 0.f;
                m[j] = w;
                den += w;
            }
            for (int j = 0; j < S; ++j) wts[i * S + j] = den > 0.f ? m[j] / den : 0.f;
        }
        __syncthreads();
        constexpr int CH = DV / 8;  // 16-byte chunks per row
        for (int it = tid; it < rows * CH; it += kFaThreads) {
            const int i = it / CH, c = it % CH, r = r0 + i;
            const int g = qt * kFaRows + r;
            if (g >= grows || c * 8 >= D) continue;
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            const uint32_t off = smem_u32(sK) + r * (DV * 2) + ((c ^ (r & 7)) << 4);
            for (int j = 0; j < S; ++j) {
                const float w = wts[i * S + j];
                const float4 v = ld_dsmem_f32x4(mapa_shared(off, j));
                const uint32_t u[4] = {__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    acc[2 * e] += w * __uint_as_float(u[e] << 16);
                    acc[2 * e + 1] += w * __uint_as_float(u[e] & 0xffff0000u);
                }
            }
            __nv_bfloat16* orow = p.out + (long long)(g % p.q_rows) * p.ldo + (kvh + p.kv_heads * (g / p.q_rows)) * D;
            uint4 o;
            o.x = pack_bf16(acc[0], acc[1]);
            o.y = pack_bf16(acc[2], acc[3]);
            o.z = pack_bf16(acc[4], acc[5]);
            o.w = pack_bf16(acc[6], acc[7]);
            *reinterpret_cast<uint4*>(orow + c * 8) = o;
        }
        cluster_sync_all();  // peers are done reading this CTA's parked partial
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) tmem_dealloc(tmem, C::TMEM_COLS);
}

CUtensorMap make_tmap_bf16(const void* base, long long rows, long long cols, long long ld, int box_rows);

namespace {
template <int D, int DK, int DV, int KK, int KV>
cudaError_t fa_configure_t() {
    return cudaFuncSetAttribute(fattn_kernel<D, DK, DV, KK, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                FaCfg<D, DK, DV, KK, KV>::SMEM);
}
}  // namespace

cudaError_t fattn_configure() {
    cudaError_t e = fa_configure_t<72, 80, 128, 3, 3>();
    if (e == cudaSuccess) e = fa_configure_t<256, 256, 256, 2, 2>();
    return e;
}

// Tensor maps for one attention launch (built once at plan time).
FaMaps make_fattn_maps(const AttnParams& p, int head_dim) {
    FaMaps m;
    const long long width = (long long)p.kv_heads * head_dim;
    m.k0 = make_tmap_bf16(p.k0, p.rows0, width, p.ld0, 32);
    m.v0 = make_tmap_bf16(p.v0, p.rows0, width, p.ld0, 32);
    const bool has1 = p.rows1 > 0 && p.k1;
    m.k1 = make_tmap_bf16(has1 ? p.k1 : p.k0, has1 ? p.rows1 : p.rows0, width, has1 ? p.ld1 : p.ld0, 32);
    m.v1 = make_tmap_bf16(has1 ? p.v1 : p.v0, has1 ? p.rows1 : p.rows0, width, has1 ? p.ld1 : p.ld0, 32);
    return m;
}

static bool g_fa_pdl = true;
void fattn_set_pdl(bool on) { g_fa_pdl = on; }

template <int D, int DK, int DV, int KK, int KV>
static cudaError_t fa_launch_t(const FaMaps& maps, const AttnParams& p, dim3 grid, cudaStream_t stream) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kFaThreads, 1, 1);
    cfg.dynamicSmemBytes = FaCfg<D, DK, DV, KK, KV>::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (g_fa_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (grid.y > 1) {  // key splits of one q tile form a cluster (DSMEM combine)
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = grid.y;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fattn_kernel<D, DK, DV, KK, KV>, maps, p);
}

// grid = (stacked q tiles of 128, key splits (p.kv_splits: 1, 2, 4 or 8), kv groups).
cudaError_t launch_fattn(int head_dim, const FaMaps& maps, const AttnParams& p, cudaStream_t stream) {
    const int grows = (p.heads / p.kv_heads) * p.q_rows;
    const int S = p.kv_splits > 1 ? p.kv_splits : 1;
    if (S != 1 && S != 2 && S != 4 && S != 8) return cudaErrorInvalidValue;
    const dim3 grid((grows + kFaRows - 1) / kFaRows, S, p.kv_heads);
    if ((p.rows0 % 32) || (p.rows1 % 32)) return cudaErrorInvalidValue;
    switch (head_dim) {
        case 72: return fa_launch_t<72, 80, 128, 3, 3>(maps, p, grid, stream);
        case 256: return fa_launch_t<256, 256, 256, 2, 2>(maps, p, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
