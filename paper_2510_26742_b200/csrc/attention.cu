// Flash-style attention (online softmax, fp32 statistics) for the three attention
// nodes of the fused pi0 graph:
//   ve.attn  16 heads x d72 MHA, q = kv = views*256 (joint over all views),
//   llm.attn 8 q-heads / 1 kv-head x d256 (MQA), q = kv = prefix,
//   ae.attn  8 q-heads / 1 kv-head x d256, q = 64 suffix rows, kv = [LLM KV_l ; own KV].
// Reference semantics: proj/src/evaluate.cpp:225-252 (no mask, scale 1/sqrt(d),
// softmax with max subtraction, proj/src/tensor.cpp:95-112).
//
// MQA is computed with all q-heads of a kv-group stacked as extra query rows, so the
// single K/V head is loaded once per 64-row tile.  Long key ranges can be split
// (flash-decoding): partial (O, m, l) go to an fp32 workspace and the last CTA of
// the query tile merges them.
//
// The QK^T and PV products use warp-level mma.sync m16n8k16 (bf16 in, fp32 accumulate).
#include "attention.cuh"
#include "ptx.cuh"

#include <math.h>

namespace pi0b {

constexpr int kAttnThreads = 128;
constexpr int kAttnQT = 64;
constexpr int kMaxSplits = 8;

constexpr int kKvStages = 3;   // key/value tiles in flight (prefetch distance 2)

template <int HD, int HDP, int KVT>
struct AttnCfg {
    static constexpr int LDS = HDP + 8;  // padded smem row (elements)
    static constexpr int SMEM = (kAttnQT + 2 * kKvStages * KVT) * LDS * 2;
};

template <int HD, int HDP, int KVT>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(const AttnParams p) {
    using Cfg = AttnCfg<HD, HDP, KVT>;
    constexpr int LDS = Cfg::LDS;
    constexpr int CH = HDP / 8;   // 16-byte chunks per padded row
    constexpr int CHV = HD / 8;   // chunks holding real data
    constexpr int NT = HD / 8;    // output n-tiles
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
    __nv_bfloat16* sK = sQ + kAttnQT * LDS;
    __nv_bfloat16* sV = sK + kKvStages * KVT * LDS;
    __shared__ int last_flag;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qt = blockIdx.x, split = blockIdx.y, grp = blockIdx.z;
    const int hpg = p.heads / p.kv_heads;
    const int grows = hpg * p.q_rows;
    const int kvh = grp;

    // ---- Q tile (stacked rows g -> (head, token))
    for (int idx = tid; idx < kAttnQT * CH; idx += kAttnThreads) {
        const int rr = idx / CH, ch = idx % CH;
        const int g = qt * kAttnQT + rr;
        const bool ok = g < grows && ch < CHV;
        const __nv_bfloat16* src = p.q;
        if (ok) {
            const int hh = g / p.q_rows, i = g % p.q_rows;
            const int h = kvh + p.kv_heads * hh;
            src = p.q + (long long)i * p.ldq + h * HD + ch * 8;
        }
        cp_async16(sQ + rr * LDS + ch * 8, src, ok);
    }

    const int total = p.rows0 + p.rows1;
    const int kv_begin = split * p.kv_per_split;
    const int kv_end = min(total, kv_begin + p.kv_per_split);
    const int ntiles = (kv_end - kv_begin + KVT - 1) / KVT;

    auto load_kv = [&](int t, int buf) {
        const int base = kv_begin + t * KVT;
        __nv_bfloat16* dk = sK + buf * KVT * LDS;
        __nv_bfloat16* dv = sV + buf * KVT * LDS;
        for (int idx = tid; idx < KVT * CH; idx += kAttnThreads) {
            const int rr = idx / CH, ch = idx % CH;
            const int j = base + rr;
            const bool ok = j < kv_end && ch < CHV;
            const __nv_bfloat16* ks = p.k0;
            const __nv_bfloat16* vs = p.v0;
            if (ok) {
                if (j < p.rows0) {
                    const long long off = (long long)j * p.ld0 + kvh * HD + ch * 8;
                    ks = p.k0 + off;
                    vs = p.v0 + off;
                } else {
                    const long long off = (long long)(j - p.rows0) * p.ld1 + kvh * HD + ch * 8;
                    ks = p.k1 + off;
                    vs = p.v1 + off;
                }
            }
            cp_async16(dk + rr * LDS + ch * 8, ks, ok);
            cp_async16(dv + rr * LDS + ch * 8, vs, ok);
        }
    };

    // Q and the first kKvStages-1 key/value tiles go out immediately; one commit group per tile.
#pragma unroll
    for (int t = 0; t < kKvStages - 1; ++t) {
        if (t < ntiles) load_kv(t, t);
        cp_async_commit();
    }

    float o[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const int g4 = lane >> 2, t4 = lane & 3;

    for (int t = 0; t < ntiles; ++t) {
        if (t + kKvStages - 1 < ntiles) load_kv(t + kKvStages - 1, (t + kKvStages - 1) % kKvStages);
        cp_async_commit();
        cp_async_wait<kKvStages - 1>();
        __syncthreads();
        const __nv_bfloat16* cK = sK + (t % kKvStages) * KVT * LDS;
        const __nv_bfloat16* cV = sV + (t % kKvStages) * KVT * LDS;

        float s[KVT / 8][4];
#pragma unroll
        for (int i = 0; i < KVT / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HDP / 16; ++ks) {
            uint32_t a[4];
            ldmatrix_x4(a, sQ + (warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + ks * 16 +
                               (lane >> 4) * 8);
#pragma unroll
            for (int n2 = 0; n2 < KVT / 16; ++n2) {
                uint32_t b[4];
                ldmatrix_x4(b, cK + (n2 * 16 + (lane & 7) + (lane >> 4) * 8) * LDS + ks * 16 +
                                   ((lane >> 3) & 1) * 8);
                mma_bf16_16816(s[2 * n2], a, b[0], b[1]);
                mma_bf16_16816(s[2 * n2 + 1], a, b[2], b[3]);
            }
        }
        // scale (log2 domain) + mask the ragged tail
        const int kbase = kv_begin + t * KVT;
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int n = 0; n < KVT / 8; ++n) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int j = kbase + n * 8 + 2 * t4 + (c & 1);
                float x = s[n][c] * p.scale_log2;
                if (j >= kv_end) x = -INFINITY;
                s[n][c] = x;
            }
            mx0 = fmaxf(mx0, fmaxf(s[n][0], s[n][1]));
            mx1 = fmaxf(mx1, fmaxf(s[n][2], s[n][3]));
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
        m0 = mn0;
        m1 = mn1;
        l0 *= c0;
        l1 *= c1;
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            o[i][0] *= c0; o[i][1] *= c0;
            o[i][2] *= c1; o[i][3] *= c1;
        }
#pragma unroll
        for (int n = 0; n < KVT / 8; ++n) {
            s[n][0] = exp2f(s[n][0] - m0);
            s[n][1] = exp2f(s[n][1] - m0);
            s[n][2] = exp2f(s[n][2] - m1);
            s[n][3] = exp2f(s[n][3] - m1);
            l0 += s[n][0] + s[n][1];
            l1 += s[n][2] + s[n][3];
        }
        // O += P V
#pragma unroll
        for (int kc = 0; kc < KVT / 16; ++kc) {
            uint32_t a[4];
            a[0] = pack_bf16(s[2 * kc][0], s[2 * kc][1]);
            a[1] = pack_bf16(s[2 * kc][2], s[2 * kc][3]);
            a[2] = pack_bf16(s[2 * kc + 1][0], s[2 * kc + 1][1]);
            a[3] = pack_bf16(s[2 * kc + 1][2], s[2 * kc + 1][3]);
            const __nv_bfloat16* vrow = cV + (kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS;
#pragma unroll
            for (int n2 = 0; n2 < NT / 2; ++n2) {
                uint32_t b[4];
                ldmatrix_x4_trans(b, vrow + n2 * 16 + (lane >> 4) * 8);
                mma_bf16_16816(o[2 * n2], a, b[0], b[1]);
                mma_bf16_16816(o[2 * n2 + 1], a, b[2], b[3]);
            }
            if constexpr (NT & 1) {
                uint32_t b[2];
                ldmatrix_x2_trans(b, vrow + (NT - 1) * 8);
                mma_bf16_16816(o[NT - 1], a, b[0], b[1]);
            }
        }
        __syncthreads();
    }

    l0 += __shfl_xor_sync(0xffffffff, l0, 1);
    l0 += __shfl_xor_sync(0xffffffff, l0, 2);
    l1 += __shfl_xor_sync(0xffffffff, l1, 1);
    l1 += __shfl_xor_sync(0xffffffff, l1, 2);
    const float il0 = l0 > 0.f ? 1.f / l0 : 0.f;
    const float il1 = l1 > 0.f ? 1.f / l1 : 0.f;
    const int rA = qt * kAttnQT + warp * 16 + g4;  // stacked row of (c0, c1)
    const int rB = rA + 8;                          // stacked row of (c2, c3)

    auto out_ptr = [&](int g) -> __nv_bfloat16* {
        const int hh = g / p.q_rows, i = g % p.q_rows;
        const int h = kvh + p.kv_heads * hh;
        return p.out + (long long)i * p.ldo + h * HD;
    };

    if (p.kv_splits == 1) {
        if (rA < grows) {
            __nv_bfloat16* dst = out_ptr(rA);
#pragma unroll
            for (int n = 0; n < NT; ++n)
                *reinterpret_cast<uint32_t*>(dst + n * 8 + 2 * t4) = pack_bf16(o[n][0] * il0, o[n][1] * il0);
        }
        if (rB < grows) {
            __nv_bfloat16* dst = out_ptr(rB);
#pragma unroll
            for (int n = 0; n < NT; ++n)
                *reinterpret_cast<uint32_t*>(dst + n * 8 + 2 * t4) = pack_bf16(o[n][2] * il1, o[n][3] * il1);
        }
        return;
    }

    // ---- split-KV: write normalised partial + (m, l); last CTA merges
    const long long rows_pad = (long long)gridDim.x * kAttnQT;
    const long long slab = ((long long)split * gridDim.z + grp) * rows_pad;
    {
        float* wa = p.ws_o + (slab + rA) * HD;
        float* wb = p.ws_o + (slab + rB) * HD;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            *reinterpret_cast<float2*>(wa + n * 8 + 2 * t4) = make_float2(o[n][0] * il0, o[n][1] * il0);
            *reinterpret_cast<float2*>(wb + n * 8 + 2 * t4) = make_float2(o[n][2] * il1, o[n][3] * il1);
        }
        if (t4 == 0) {
            *reinterpret_cast<float2*>(p.ws_ml + (slab + rA) * 2) = make_float2(m0, l0);
            *reinterpret_cast<float2*>(p.ws_ml + (slab + rB) * 2) = make_float2(m1, l1);
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        int* ctr = p.counters + grp * gridDim.x + qt;
        const int prev = atomicAdd(ctr, 1);
        last_flag = prev == p.kv_splits - 1;
        if (last_flag) atomicExch(ctr, 0);
    }
    __syncthreads();
    if (!last_flag) return;
    __threadfence();
    // Merge: per stacked row, weights w_s = l_s 2^(m_s - M) / sum (threads 0..63), then all
    // threads sweep (row, d-pair) items with the split loads of 8 rows in flight.
    __shared__ float wts[kAttnQT][kMaxSplits];
    if (tid < kAttnQT) {
        const int g = qt * kAttnQT + tid;
        float M = -INFINITY;
        for (int s2 = 0; s2 < p.kv_splits; ++s2)
            M = fmaxf(M, __ldcg(p.ws_ml + (((long long)s2 * gridDim.z + grp) * rows_pad + g) * 2));
        float W = 0.f;
        for (int s2 = 0; s2 < p.kv_splits; ++s2) {
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + ((long long)s2 * gridDim.z + grp) * rows_pad + g);
            const float w = ml.y > 0.f ? ml.y * exp2f(ml.x - M) : 0.f;
            wts[tid][s2] = w;
            W += w;
        }
        const float iw = W > 0.f ? 1.f / W : 0.f;
        for (int s2 = 0; s2 < p.kv_splits; ++s2) wts[tid][s2] *= iw;
    }
    __syncthreads();
    constexpr int PAIRS = HD / 2;
    const int S = p.kv_splits;
    for (int pr = tid; pr < PAIRS; pr += kAttnThreads) {
        const int d = pr * 2;
#pragma unroll 1
        for (int rr = 0; rr < kAttnQT; rr += 4) {
            float2 ov[4][kMaxSplits];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int g = min(qt * kAttnQT + rr + u, grows - 1);
#pragma unroll
                for (int s2 = 0; s2 < kMaxSplits; ++s2)
                    if (s2 < S)
                        ov[u][s2] = __ldcg(reinterpret_cast<const float2*>(
                            p.ws_o + (((long long)s2 * gridDim.z + grp) * rows_pad + g) * HD + d));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int g = qt * kAttnQT + rr + u;
                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                for (int s2 = 0; s2 < kMaxSplits; ++s2)
                    if (s2 < S) {
                        a0 += wts[rr + u][s2] * ov[u][s2].x;
                        a1 += wts[rr + u][s2] * ov[u][s2].y;
                    }
                if (g < grows) *reinterpret_cast<uint32_t*>(out_ptr(g) + d) = pack_bf16(a0, a1);
            }
        }
    }
}

template <int HD, int HDP, int KVT>
static cudaError_t launch_attn_t(const AttnParams& p, int q_tiles, cudaStream_t stream) {
    dim3 grid(q_tiles, p.kv_splits, p.kv_heads);
    attn_kernel<HD, HDP, KVT><<<grid, kAttnThreads, AttnCfg<HD, HDP, KVT>::SMEM, stream>>>(p);
    return cudaGetLastError();
}

// Must run once per device before any launch (not capturable).
cudaError_t attn_configure() {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<72, 80, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnCfg<72, 80, 64>::SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(attn_kernel<256, 256, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 AttnCfg<256, 256, 32>::SMEM);
    return e;
}

int attn_key_tile(int head_dim) { return head_dim == 72 ? 64 : 32; }
int attn_query_tile() { return kAttnQT; }

cudaError_t launch_attention(int head_dim, const AttnParams& p, cudaStream_t stream) {
    const int grows = (p.heads / p.kv_heads) * p.q_rows;
    const int q_tiles = (grows + kAttnQT - 1) / kAttnQT;
    switch (head_dim) {
        case 72: return launch_attn_t<72, 80, 64>(p, q_tiles, stream);
        case 256: return launch_attn_t<256, 256, 32>(p, q_tiles, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pi0b
