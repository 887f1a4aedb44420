// The action-expert megakernel: all flow steps of the pi0 action expert in one persistent
// launch (one CTA per SM).  See aemk.cuh for the task model.
//
// Replaces, for the AE half of the fused graph (proj/src/builder.cpp:291-363), the reference's
// demand-driven fp64 evaluation (proj/src/evaluate.cpp:254-349): matmul + apply_epilogue for
// every ae.* GEMM instance, Evaluator::attention for ae.attn over [LLM KV_l ; own KV]
// (ae.kcat / ae.vcat), the RmsStats nodes, the ae.suffix concat and the ae.act_rows slice.
//
// Warp roles (320 threads):
//   warp 0      weight producer: walks the CTA's task list and TMA-streams every GEMM task's
//               [128 features x 64 k] bf16 weight tiles into a 6-stage ring.  It never waits
//               on a dependency, only on free ring slots, so it runs ahead across barriers.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer.  GEMM: D[128 x 128] +=
//               X[128 x 64] * W^T, X = the 64 activation rows (rows 64..127 of the A tile are
//               don't-care and never read back).  Attention: S = Q K^T (N = 64 keys) and
//               O = P V (N = 256) for one head pair (128 stacked query rows) and one key block.
//   warps 2..9  workers: dependency waits, activation staging (TMA, or fp32 -> bf16 with the
//               row sums of squares of the RmsScale), epilogues from TMEM, softmax, the
//               TMA reduce-add of split-K partials into the fp32 residual stream, signalling.
//
// Split-K partials (ae.proj, ae.down, ae.action_out) and the per-key-block attention outputs
// are combined in L2 by cp.reduce.async.bulk.tensor (add.f32) — no workspace, no extra pass.
// Attention key blocks share the row maximum through an atomicMax rendezvous so that their
// exp-sums and P V products are directly additive.
#include "aemk.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <queue>
#include <stdexcept>
#include <string>
#include <vector>

namespace pi0b {

namespace {

constexpr int kAeThreads = 320;
constexpr int kWorkers = 256;
constexpr int kWSt = 4;
constexpr int kWTile = 128 * 64 * 2;  // 16 KB: 128 weight rows x 64 k
constexpr int kXSt = 4;
constexpr int kXTile = 64 * 128;      // 8 KB: 64 activation rows x 64 k (bf16, SW128)
constexpr int kFSt = 4;
constexpr int kFTile = 16384;         // 64 rows x 64 fp32 as two SW128 boxes of 32 columns
constexpr int kOffW = 0;
constexpr int kOffU = kWSt * kWTile;                // union region, 160 KB
constexpr int kOffX = kOffU;                        // GEMM: X ring (+1 pad slot)
constexpr int kOffF = kOffU + (kXSt + 1) * kXTile;  // GEMM: fp32 staging ring
constexpr int kOffE = kOffF + kFSt * kFTile;        // GEMM: fp32 epilogue tile (32 KB)
constexpr int kOffQ = kOffU;                        // ATTN: Q  [128 x 256] bf16, 4 x 16 KB
constexpr int kOffK = kOffU + 65536;                // ATTN: K  [64 x 256], 4 x 8 KB
constexpr int kOffV = kOffU + 98304;                // ATTN: V  [64 x 256], 4 x 8 KB
constexpr int kOffP = kOffK;                        // ATTN: P  [128 x 64] (reuses K)
constexpr int kOffAux = kOffU + 163840;
constexpr int kAeSmem = kOffAux + 1024 + 1024;      // + aux + alignment slack
static_assert(kOffE + 32768 <= kOffAux, "GEMM union overflow");
static_assert(kAeSmem <= 232448, "shared memory budget");
static_assert(kWSt <= 8 && kXSt <= 4 && kFSt <= 4, "barrier slots");

constexpr uint32_t kTAcc = 0, kTS = 128, kTO = 256;  // TMEM columns (512 allocated)

PI0B_DEV unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
PI0B_DEV unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
PI0B_DEV void red_release_add_u32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PI0B_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
PI0B_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
PI0B_DEV void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(m)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1)
        : "memory");
}
PI0B_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
PI0B_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Spin until a counter reaches `target` (relaxed polling, one acquire fence at the end); a
// broken schedule traps (~4 s) instead of hanging the GPU.
PI0B_DEV void wait_counter(const unsigned* c, unsigned target) {
    if (ld_relaxed_u32(c) < target) {
        const long long t0 = clock64();
        while (ld_relaxed_u32(c) < target) {
            if (clock64() - t0 > (1ll << 33)) __trap();
        }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
PI0B_DEV unsigned atom_add_acqrel_u32(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
PI0B_DEV void st_relaxed_u32(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Order-preserving float <-> unsigned key (atomicMax on the key == max on the float).
PI0B_DEV unsigned fkey(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
PI0B_DEV float fdecode(unsigned k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k); }

PI0B_DEV uint64_t desc_mn(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t(saddr) >> 4) & 0x3FFFull;
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}

PI0B_DEV void adv(int& slot, uint32_t& ph, int n, int stages) {
    slot += n;
    while (slot >= stages) {
        slot -= stages;
        ph ^= 1u;
    }
}

PI0B_DEV AeTask load_task(const AeTask* t) {
    const uint4* s = reinterpret_cast<const uint4*>(t);
    uint4 a = __ldg(s), b = __ldg(s + 1);
    AeTask r;
    uint4* d = reinterpret_cast<uint4*>(&r);
    d[0] = a;
    d[1] = b;
    return r;
}

PI0B_DEV uint32_t pack2(float a, float b) { return pack_bf16(a, b); }

PI0B_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace

__global__ void __launch_bounds__(kAeThreads, 1) aemk_kernel(const AeParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint8_t* sW = smem + kOffW;
    uint8_t* sU = smem + kOffU;
    uint8_t* sX = smem + kOffX;
    uint8_t* sF = smem + kOffF;
    uint8_t* sE = smem + kOffE;
    uint8_t* sQ = smem + kOffQ;
    uint8_t* sK = smem + kOffK;
    uint8_t* sV = smem + kOffV;
    uint8_t* sP = smem + kOffP;
    uint64_t* mb = reinterpret_cast<uint64_t*>(smem + kOffAux);
    uint64_t* w_full = mb;           // [kWSt <= 8]
    uint64_t* w_empty = mb + 8;      // [kWSt]
    uint64_t* x_full = mb + 16;      // [kXSt <= 4]
    uint64_t* x_empty = mb + 20;     // [kXSt]
    uint64_t* f_full = mb + 24;      // [kFSt <= 4]
    uint64_t* acc_full = mb + 28;
    uint64_t* acc_empty = mb + 29;
    uint64_t* q_full = mb + 30;
    uint64_t* k_full = mb + 31;
    uint64_t* v_full = mb + 32;
    uint64_t* s_full = mb + 33;
    uint64_t* p_full = mb + 34;
    uint64_t* o_done = mb + 35;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mb + 40);
    float* sm_rs = reinterpret_cast<float*>(smem + kOffAux + 512);  // [64]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const AeTask* my = p.tasks + size_t(blockIdx.x) * p.task_stride;
    const CUtensorMap* maps = reinterpret_cast<const CUtensorMap*>(p.maps);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 36; ++i) mbar_init(&mb[i], 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================================================================ weight producer
        if (lane == 0) {
            int ws = 0;
            uint32_t wph = 0;
            unsigned issued = 0;  // weight tiles issued so far
            const unsigned cap = unsigned(max(1, min(p.w_inflight, kWSt)));
            for (int i = 0;; ++i) {
                const AeTask t = load_task(my + i);
                if (t.kind == kAeEnd || t.phase >= p.limit_phase) break;
                if (t.kind != kAeGemm) continue;
                unsigned long long* tr = p.trace ? p.trace + (size_t(blockIdx.x) * p.task_stride + i) * 8 : nullptr;
                const CUtensorMap* wm = maps + t.wmap;
                for (int k = 0; k < t.nkb; ++k) {
                    mbar_wait(&w_empty[ws], wph ^ 1);
                    if (issued >= cap) {  // at most `cap` tiles in flight: keeps the memory queues short
                        const unsigned o = issued - cap;
                        mbar_wait(&w_full[o % kWSt], (o / kWSt) & 1);
                    }
                    if (tr && k == 0) tr[4] = gtimer();
                    mbar_arrive_expect_tx(&w_full[ws], kWTile);
                    tma_load_2d(sW + ws * kWTile, wm, &w_full[ws], (t.kb0 + k) * 64, t.tile * 128, kEvictFirst);
                    adv(ws, wph, 1, kWSt);
                    ++issued;
                }
                if (tr) tr[5] = gtimer();
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        if (lane == 0) {
            int ws = 0, xs = 0;
            uint32_t wph = 0, xph = 0, gidx = 0, aidx = 0;
            constexpr uint32_t idesc_g = umma_idesc_bf16(128, 128);
            constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64);
            constexpr uint32_t idesc_o = umma_idesc_bf16(128, 256) | (1u << 16);  // B (V) MN-major
            for (int i = 0;; ++i) {
                const AeTask t = load_task(my + i);
                if (t.kind == kAeEnd || t.phase >= p.limit_phase) break;
                if (t.kind == kAeGemm) {
                    unsigned long long* tr = p.trace ? p.trace + (size_t(blockIdx.x) * p.task_stride + i) * 8 : nullptr;
                    mbar_wait(acc_empty, (gidx & 1) ^ 1);
                    tc_fence_after();
                    for (int k = 0; k < t.nkb; ++k) {
                        mbar_wait(&w_full[ws], wph);
                        if (tr && k == t.nkb - 1) tr[6] = gtimer();
                        mbar_wait(&x_full[xs], xph);
                        tc_fence_after();
                        const uint64_t ad = umma_desc_sw128(sX + xs * kXTile);
                        const uint64_t bd = umma_desc_sw128(sW + ws * kWTile);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_bf16(tmem + kTAcc, ad + 2 * kk, bd + 2 * kk, idesc_g, (k | kk) != 0);
                        umma_commit(&w_empty[ws]);
                        umma_commit(&x_empty[xs]);
                        adv(ws, wph, 1, kWSt);
                        adv(xs, xph, 1, kXSt);
                    }
                    umma_commit(acc_full);
                    if (tr) tr[7] = gtimer();
                    ++gidx;
                } else if (t.kind == kAeAttn) {
                    const uint32_t ph = aidx & 1;
                    mbar_wait(q_full, ph);
                    mbar_wait(k_full, ph);
                    tc_fence_after();
                    const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK), v0 = smem_u32(sV), p0 = smem_u32(sP);
#pragma unroll
                    for (int kk = 0; kk < 16; ++kk) {
                        const uint64_t a = umma_desc_sw128(sQ + (kk >> 2) * 16384 + (kk & 3) * 32);
                        const uint64_t b = umma_desc_sw128(sK + (kk >> 2) * 8192 + (kk & 3) * 32);
                        umma_bf16(tmem + kTS, a, b, idesc_s, kk > 0);
                    }
                    umma_commit(s_full);
                    mbar_wait(p_full, ph);
                    mbar_wait(v_full, ph);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t a = umma_desc_sw128(sP + kk * 32);
                        const uint64_t b = desc_mn(v0 + kk * 2048, 8192);
                        umma_bf16(tmem + kTO, a, b, idesc_o, kk > 0);
                    }
                    umma_commit(o_done);
                    (void)q0;
                    (void)k0;
                    (void)p0;
                    ++aidx;
                }
            }
        }
        __syncwarp();
    } else {
        // ================================================================ workers
        const int wtid = threadIdx.x - 64;
        const int wq = warp & 3;                      // TMEM lane quarter of this warp
        const bool drainer = wq < 2;                  // warps 4, 5, 8, 9: TMEM lanes 0..63
        const int drow = wq * 32 + lane;              // drainer: activation row
        const int dhalf = warp >= 8 ? 1 : 0;          // drainer: column half
        const bool softmax = warp >= 4 && warp < 8;   // TMEM lanes 0..127 (stacked query rows)
        const int srow = wq * 32 + lane;
        const uint32_t tlane = uint32_t(wq * 32) << 16;
        int xs = 0, fs = 0;
        uint32_t xph = 0, fph = 0, gidx = 0, aidx = 0;
        // staging geometry: thread -> (row r, 16-column quarter q) of a 64 x 64 k-block
        const int sr = wtid >> 2, sq = wtid & 3;

        for (int i = 0;; ++i) {
            const AeTask t = load_task(my + i);
            if (t.kind == kAeEnd || t.phase >= p.limit_phase) break;
            unsigned long long* tr = p.trace ? p.trace + (size_t(blockIdx.x) * p.task_stride + i) * 8 : nullptr;
            if (tr && wtid == 0) tr[0] = gtimer();
            if (t.wait_cnt) {
                if (wtid == 0) {
                    wait_counter(p.mbox + size_t(blockIdx.x) * p.n_bars + t.wait_bar, 1u);
                    fence_proxy_async_global();
                }
                named_bar_sync(1, kWorkers);
            }
            if (tr && wtid == 0) tr[1] = gtimer();

            if (t.kind == kAeGemm) {
                // -------------------------------------------------- activation staging
                const CUtensorMap* xm = maps + t.xmap;
                if (t.xsrc == kXBf16) {
                    if (wtid == 0) {
                        int s = xs;
                        uint32_t ph = xph;
                        for (int k = 0; k < t.nkb; ++k) {
                            mbar_wait(&x_empty[s], ph ^ 1);
                            mbar_arrive_expect_tx(&x_full[s], kXTile);
                            tma_load_2d(sX + s * kXTile, xm, &x_full[s], (t.kb0 + k) * 64, 0, kEvictLast);
                            adv(s, ph, 1, kXSt);
                        }
                    }
                    adv(xs, xph, t.nkb, kXSt);
                } else if (t.xsrc == kXY || t.xsrc == kXO) {
                    float ss = 0.f;
                    if (wtid == 0) {
                        int s = fs;
                        uint32_t ph = fph;
                        for (int k = 0; k < t.nkb && k < kFSt; ++k) {
                            mbar_arrive_expect_tx(&f_full[s], kFTile);
                            tma_load_2d(sF + s * kFTile, xm, &f_full[s], (t.kb0 + k) * 64, 0, kEvictLast);
                            tma_load_2d(sF + s * kFTile + 8192, xm, &f_full[s], (t.kb0 + k) * 64 + 32, 0, kEvictLast);
                            adv(s, ph, 1, kFSt);
                        }
                    }
                    for (int k = 0; k < t.nkb; ++k) {
                        float scale = 1.f;
                        if (t.xsrc == kXO) {
                            const int head = ((t.kb0 + k) * 64) >> 8;
                            const float l = __ldcg(p.lacc[t.par] + head * 64 + sr);
                            scale = l > 0.f ? 1.f / l : 0.f;
                        }
                        mbar_wait(&f_full[fs], fph);
                        mbar_wait(&x_empty[xs], xph ^ 1);
                        const uint8_t* src = sF + fs * kFTile + (sq >> 1) * 8192 + sr * 128;
                        float v[16];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int c = (sq & 1) * 4 + j;
                            const float4 f = *reinterpret_cast<const float4*>(src + ((c ^ (sr & 7)) << 4));
                            v[4 * j] = f.x * scale;
                            v[4 * j + 1] = f.y * scale;
                            v[4 * j + 2] = f.z * scale;
                            v[4 * j + 3] = f.w * scale;
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) ss += v[j] * v[j];
                        uint8_t* dst = sX + xs * kXTile + sr * 128;
                        const uint4 u0 = make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
                        const uint4 u1 = make_uint4(pack2(v[8], v[9]), pack2(v[10], v[11]), pack2(v[12], v[13]),
                                                    pack2(v[14], v[15]));
                        *reinterpret_cast<uint4*>(dst + (((2 * sq) ^ (sr & 7)) << 4)) = u0;
                        *reinterpret_cast<uint4*>(dst + (((2 * sq + 1) ^ (sr & 7)) << 4)) = u1;
                        fence_proxy_async_smem();
                        named_bar_sync(1, kWorkers);
                        if (wtid == 0) {
                            mbar_arrive(&x_full[xs]);
                            if (k + kFSt < t.nkb) {
                                const int kb = t.kb0 + k + kFSt;
                                mbar_arrive_expect_tx(&f_full[fs], kFTile);
                                tma_load_2d(sF + fs * kFTile, xm, &f_full[fs], kb * 64, 0, kEvictLast);
                                tma_load_2d(sF + fs * kFTile + 8192, xm, &f_full[fs], kb * 64 + 32, 0, kEvictLast);
                            }
                        }
                        adv(fs, fph, 1, kFSt);
                        adv(xs, xph, 1, kXSt);
                    }
                    if (t.xsrc == kXY) {
                        ss += __shfl_xor_sync(0xffffffff, ss, 1);
                        ss += __shfl_xor_sync(0xffffffff, ss, 2);
                        if (sq == 0) sm_rs[sr] = 1.0f / sqrtf(ss * p.inv_width + p.eps);
                    }
                } else {  // kXRows: Euler state (ae.action_proj) or robot state (ae.state_proj), K <= 64
                    const bool init = t.epi == kEpiInit;
                    const float* src = init ? p.state : p.a;
                    const int rows = init ? 1 : p.chunk, cols = init ? p.state_dim : p.act_dim;
                    const int ld = init ? p.state_dim : p.lda;
                    mbar_wait(&x_empty[xs], xph ^ 1);
                    float v[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int c = sq * 16 + j;
                        v[j] = (sr < rows && c < cols) ? __ldcg(src + sr * ld + c) : 0.f;
                    }
                    uint8_t* dst = sX + xs * kXTile + sr * 128;
                    *reinterpret_cast<uint4*>(dst + (((2 * sq) ^ (sr & 7)) << 4)) =
                        make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
                    *reinterpret_cast<uint4*>(dst + (((2 * sq + 1) ^ (sr & 7)) << 4)) =
                        make_uint4(pack2(v[8], v[9]), pack2(v[10], v[11]), pack2(v[12], v[13]), pack2(v[14], v[15]));
                    fence_proxy_async_smem();
                    named_bar_sync(1, kWorkers);
                    if (wtid == 0) mbar_arrive(&x_full[xs]);
                    adv(xs, xph, 1, kXSt);
                }
                // FFN tasks recycle the attention accumulators of their layer parity (read by
                // this layer's ae.proj, which completed before any ae.ffn task started).
                if (t.epi == kEpiGate) {
                    const int parts = t.aux >> 8, part = t.aux & 255;
                    const int n4 = (64 * p.q_width) / 4;
                    float4* o4 = reinterpret_cast<float4*>(p.oacc[t.par]);
                    const int per = (n4 + parts - 1) / parts;
                    for (int j = part * per + wtid; j < min(n4, (part + 1) * per); j += kWorkers)
                        __stcg(o4 + j, make_float4(0.f, 0.f, 0.f, 0.f));
                    if (part == 0)
                        for (int j = wtid; j < p.heads * 64; j += kWorkers) {
                            p.lacc[t.par][j] = 0.f;
                            p.mmax[t.par][j] = 0u;
                        }
                }
                named_bar_sync(1, kWorkers);  // sm_rs complete
                if (tr && wtid == 0) tr[2] = gtimer();

                // -------------------------------------------------- epilogue
                mbar_wait(acc_full, gidx & 1);
                tc_fence_after();
                if (drainer) {
                    const int r = drow;
                    const uint32_t ta = tmem + kTAcc + tlane;
                    if (t.epi == kEpiRed) {
#pragma unroll 1
                        for (int cc = 0; cc < 2; ++cc) {
                            float v[32];
                            const int col0 = dhalf * 64 + cc * 32;
                            tmem_ld32(ta + col0, v);
                            uint8_t* box = sE + (col0 >> 5) * 8192 + r * 128;
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                *reinterpret_cast<float4*>(box + ((j ^ (r & 7)) << 4)) =
                                    make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        }
                        fence_proxy_async_smem();
                    } else if (t.epi == kEpiQkv || t.epi == kEpiGate) {
                        float a[32], b[32];
                        const int c0 = dhalf * 32;
                        tmem_ld32(ta + c0, a);
                        tmem_ld32(ta + 64 + c0, b);
                        const float rs = sm_rs[r];
                        if (t.epi == kEpiGate) {
                            __nv_bfloat16* o = p.g + (size_t)r * p.mlp + t.tile * 64 + c0;
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                float gg[8];
#pragma unroll
                                for (int u = 0; u < 8; ++u) gg[u] = (a[j + u] * rs) * gelu_tanh(b[j + u] * rs);
                                *reinterpret_cast<uint4*>(o + j) = make_uint4(pack2(gg[0], gg[1]), pack2(gg[2], gg[3]),
                                                                              pack2(gg[4], gg[5]), pack2(gg[6], gg[7]));
                            }
                        } else {
                            const int f0 = t.tile * 128;
                            __nv_bfloat16* orow = p.qkv + (size_t)r * p.n_qkv;
                            float xa[32], xb[32];
                            int ca;
                            if (f0 < p.rope_cols) {
                                // packed tile = [first halves w in [64u, 64u+64) | partners + 128]
                                const int hd = f0 >> 8, u = (f0 & 255) >> 7;
                                const int w0 = u * 64 + c0;
                                ca = hd * 256 + w0;
                                const float2* cs = reinterpret_cast<const float2*>(p.rope_cs) +
                                                   (size_t)(p.rope_pos0 + r) * 128 + w0;
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    const float2 t2 = cs[j];
                                    const float x = a[j] * rs, y = b[j] * rs;
                                    xa[j] = x * t2.x - y * t2.y;
                                    xb[j] = x * t2.y + y * t2.x;
                                }
                                __nv_bfloat16* o1 = orow + ca;
                                __nv_bfloat16* o2 = orow + ca + 128;
#pragma unroll
                                for (int j = 0; j < 32; j += 8) {
                                    *reinterpret_cast<uint4*>(o1 + j) = make_uint4(
                                        pack2(xa[j], xa[j + 1]), pack2(xa[j + 2], xa[j + 3]), pack2(xa[j + 4], xa[j + 5]),
                                        pack2(xa[j + 6], xa[j + 7]));
                                    *reinterpret_cast<uint4*>(o2 + j) = make_uint4(
                                        pack2(xb[j], xb[j + 1]), pack2(xb[j + 2], xb[j + 3]), pack2(xb[j + 4], xb[j + 5]),
                                        pack2(xb[j + 6], xb[j + 7]));
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    xa[j] = a[j] * rs;
                                    xb[j] = b[j] * rs;
                                }
                                __nv_bfloat16* o1 = orow + f0 + c0;
                                __nv_bfloat16* o2 = orow + f0 + 64 + c0;
#pragma unroll
                                for (int j = 0; j < 32; j += 8) {
                                    *reinterpret_cast<uint4*>(o1 + j) = make_uint4(
                                        pack2(xa[j], xa[j + 1]), pack2(xa[j + 2], xa[j + 3]), pack2(xa[j + 4], xa[j + 5]),
                                        pack2(xa[j + 6], xa[j + 7]));
                                    *reinterpret_cast<uint4*>(o2 + j) = make_uint4(
                                        pack2(xb[j], xb[j + 1]), pack2(xb[j + 2], xb[j + 3]), pack2(xb[j + 4], xb[j + 5]),
                                        pack2(xb[j + 6], xb[j + 7]));
                                }
                            }
                        }
                    } else if (t.epi == kEpiSilu) {
                        // ae.action_proj: silu(a W + T[step]); and the ae.suffix reset of this
                        // tile's columns of the residual stream: y = [st ; b_out] (builder.cpp:311-312)
#pragma unroll 1
                        for (int cc = 0; cc < 2; ++cc) {
                            float v[32];
                            const int col0 = t.tile * 128 + dhalf * 64 + cc * 32;
                            tmem_ld32(ta + dhalf * 64 + cc * 32, v);
                            const float* tr = p.table + (size_t)t.step * p.width + col0;
                            if (r < p.chunk) {
                                __nv_bfloat16* o = p.ap + (size_t)r * p.width + col0;
#pragma unroll
                                for (int j = 0; j < 32; j += 2)
                                    *reinterpret_cast<uint32_t*>(o + j) =
                                        pack2(silu_f(v[j] + tr[j]), silu_f(v[j + 1] + tr[j + 1]));
                            }
                            const float* src = r == 0 ? p.st : p.b_out;
                            float* yrow = p.y + (size_t)r * p.width + col0;
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<float4*>(yrow + j) = __ldcg(reinterpret_cast<const float4*>(src + col0 + j));
                        }
                    } else if (t.epi == kEpiHead) {
                        float v[32];
                        tmem_ld32(ta, v);  // warp-uniform: tcgen05.ld is .sync.aligned
                        if (dhalf == 0 && r < p.chunk) {
                            const float rs = sm_rs[r];
                            float* arow = p.a + (size_t)r * p.lda;
#pragma unroll
                            for (int c = 0; c < 32; ++c)
                                if (c < p.act_dim) arow[c] += p.euler * (v[c] * rs + p.b_head[c]);
                        }
                    } else if (t.epi == kEpiInit) {
#pragma unroll 1
                        for (int cc = 0; cc < 2; ++cc) {
                            float v[32];
                            const int col0 = t.tile * 128 + dhalf * 64 + cc * 32;
                            tmem_ld32(ta + dhalf * 64 + cc * 32, v);
                            if (r == 0)
                                for (int j = 0; j < 32; ++j)
                                    if (col0 + j < p.width) p.st[col0 + j] = v[j] + p.b_state[col0 + j];
                        }
                    }
                }
                tc_fence_before();
                named_bar_sync(1, kWorkers);
                if (wtid == 0) {
                    mbar_arrive(acc_empty);
                    if (t.epi == kEpiRed) {
                        const CUtensorMap* om = maps + t.omap;
#pragma unroll
                        for (int b = 0; b < 4; ++b) tma_reduce_add_2d(om, sE + b * 8192, t.tile * 128 + 32 * b, 0);
                        bulk_commit();
                        bulk_wait_all();
                        fence_proxy_async_global();
                    }
                }
                ++gidx;
            } else if (t.kind == kAeAttn) {
                // -------------------------------------------------- attention tile
                const uint32_t ph = aidx & 1;
                const int rb = t.tile, j = t.kb0;
                const int nh = min(2, p.heads - 2 * rb);
                if (wtid == 0) {
                    const CUtensorMap* qm = maps + t.xmap;
                    mbar_arrive_expect_tx(q_full, nh * 4 * 8192);
                    for (int hh = 0; hh < nh; ++hh)
                        for (int a4 = 0; a4 < 4; ++a4)
                            tma_load_2d(sQ + a4 * 16384 + hh * 8192, qm, q_full, (2 * rb + hh) * 256 + a4 * 64, 0,
                                        kEvictLast);
                    for (int isv = 0; isv < 2; ++isv) {
                        uint64_t* bar = isv ? v_full : k_full;
                        uint8_t* dst = isv ? sV : sK;
                        mbar_arrive_expect_tx(bar, 32768);
                        for (int half = 0; half < 2; ++half) {
                            const int key = j * 64 + half * 32;
                            const bool seg0 = key < p.kv_rows0;
                            const CUtensorMap* m = maps + (seg0 ? t.wmap : t.omap);
                            const int row = seg0 ? key : key - p.kv_rows0;
                            const int col = (seg0 ? p.kcol_cache : p.kcol_own) + isv * 256;
                            for (int a4 = 0; a4 < 4; ++a4)
                                tma_load_2d(dst + a4 * 8192 + half * 4096, m, bar, col + a4 * 64, row, kEvictLast);
                        }
                    }
                }
                unsigned long long* tra = (tr && threadIdx.x == 128) ? tr : nullptr;  // warp 4 lane 0
                if (softmax) {
                    const int R = srow;
                    const int head = 2 * rb + (R >> 6);
                    const bool hv = head < p.heads;
                    const int gi = 2 * rb * 64 + R;
                    mbar_wait(s_full, ph);
                    tc_fence_after();
                    if (tra) tra[4] = gtimer();
                    float s[64];
                    tmem_ld32(tmem + kTS + tlane, reinterpret_cast<float(&)[32]>(s[0]));
                    tmem_ld32(tmem + kTS + tlane + 32, reinterpret_cast<float(&)[32]>(s[32]));
                    const int total = p.kv_rows0 + 64;
                    float mx = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 64; ++c) {
                        s[c] = j * 64 + c < total ? s[c] * p.scale_log2 : -INFINITY;
                        mx = fmaxf(mx, s[c]);
                    }
                    if (hv) atomicMax(p.mmax[t.par] + gi, fkey(mx));
                    named_bar_sync(2, 128);
                    if (R == 0) {
                        __threadfence();
                        red_release_add_u32(p.bars + t.aux, 1);
                        wait_counter(p.bars + t.aux, unsigned(p.key_blocks));
                        __threadfence();
                    }
                    named_bar_sync(2, 128);
                    if (tra) tra[5] = gtimer();
                    const float M = hv ? fdecode(ld_relaxed_u32(p.mmax[t.par] + gi)) : mx;
                    float l = 0.f;
                    uint32_t pk[32];
#pragma unroll
                    for (int c = 0; c < 64; c += 2) {
                        const float e0 = exp2f(s[c] - M), e1 = exp2f(s[c + 1] - M);
                        l += e0 + e1;
                        pk[c / 2] = pack2(e0, e1);
                    }
                    if (hv) atomicAdd(p.lacc[t.par] + gi, l);
                    uint8_t* prow = sP + R * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        *reinterpret_cast<uint4*>(prow + ((c ^ (R & 7)) << 4)) =
                            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                    fence_proxy_async_smem();
                    tc_fence_before();
                    named_bar_sync(2, 128);
                    if (R == 0) mbar_arrive(p_full);
                    mbar_wait(o_done, ph);
                    tc_fence_after();
                    if (tra) tra[6] = gtimer();
                    // un-normalised O -> fp32 boxes [head-in-pair][32-col chunk] -> reduce-add
                    const int row = R & 63;
#pragma unroll 1
                    for (int c8 = 0; c8 < 8; ++c8) {
                        float o[32];
                        tmem_ld32(tmem + kTO + tlane + c8 * 32, o);
                        uint8_t* box = sU + ((R >> 6) * 8 + c8) * 8192 + row * 128;
#pragma unroll
                        for (int q4 = 0; q4 < 8; ++q4)
                            *reinterpret_cast<float4*>(box + ((q4 ^ (row & 7)) << 4)) =
                                make_float4(o[4 * q4], o[4 * q4 + 1], o[4 * q4 + 2], o[4 * q4 + 3]);
                    }
                    fence_proxy_async_smem();
                    tc_fence_before();
                    named_bar_sync(2, 128);
                    if (R == 0) {
                        const CUtensorMap* om = maps + t.nkb;
                        for (int hh = 0; hh < nh; ++hh)
                            for (int c8 = 0; c8 < 8; ++c8)
                                tma_reduce_add_2d(om, sU + (hh * 8 + c8) * 8192, (2 * rb + hh) * 256 + c8 * 32, 0);
                        bulk_commit();
                        bulk_wait_all();
                        fence_proxy_async_global();
                        if (tra) tra[7] = gtimer();
                    }
                }
                ++aidx;
            } else if (t.kind == kAeRecY) {
                const int n4 = 64 * p.width / 4;
                const float4* s4 = reinterpret_cast<const float4*>(p.y);
                float4* d4 = reinterpret_cast<float4*>(p.rec_y + (size_t)t.aux * 64 * p.width);
                for (int q = wtid; q < n4; q += kWorkers) d4[q] = __ldcg(s4 + q);
            } else if (t.kind == kAeRecA) {
                const int n = p.chunk * p.lda;
                float* d = p.rec_a + (size_t)t.aux * n;
                for (int q = wtid; q < n; q += kWorkers) d[q] = __ldcg(p.a + q);
            }

            // -------------------------------------------------- publish completion
            // The task that completes a phase sets the phase's flag in every CTA's mailbox line.
            named_bar_sync(1, kWorkers);
            if (warp == 2) {
                unsigned old = 0;
                if (lane == 0) {
                    __threadfence();
                    old = atom_add_acqrel_u32(p.bars + t.sig_bar, 1u);
                }
                __syncwarp();
                old = __shfl_sync(0xffffffff, old, 0);
                if (old + 1 == t.sig_cnt) {
                    __threadfence();
                    for (int c = lane; c < int(gridDim.x); c += 32) st_relaxed_u32(p.mbox + size_t(c) * p.n_bars + t.sig_bar, 1u);
                }
                if (tr && lane == 0) tr[3] = gtimer();
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ====================================================================== host side

cudaError_t aemk_configure() {
    return cudaFuncSetAttribute(aemk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAeSmem);
}

cudaError_t aemk_launch(const AeParams& p, int grid, cudaStream_t stream) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kAeThreads, 1, 1);
    cfg.dynamicSmemBytes = kAeSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, aemk_kernel, p);
}

// ---------------------------------------------------------------------- planner

AePlan ae_plan(const AePlanInput& in) {
    AePlan out;
    const int W = in.width, NQ = in.n_qkv, MLP = in.mlp, NA = in.layers, FS = in.flow_steps;
    auto need = [](bool ok, const char* what) {
        if (!ok) throw std::invalid_argument(std::string("action-expert megakernel: ") + what);
    };
    need(W % 128 == 0 && NQ % 128 == 0 && (2 * MLP) % 128 == 0 && in.q_width % 256 == 0, "widths");
    need(in.rope_cols % 128 == 0, "rope columns");
    need(in.chunk + 1 <= 64, "suffix rows > 64");
    need(in.act_dim <= 32 && in.state_dim <= 64, "action/state dims");
    need(in.kv_rows0 % 32 == 0, "prefix length must be a multiple of 32");
    need(in.num_ctas >= 2 * ((in.heads + 1) / 2), "too few SMs");

    int nbar = 0;
    auto newbar = [&]() { return nbar++; };
    int phase = 0;
    struct Item {
        AeTask t;
        double cost;
    };
    std::vector<std::vector<AeTask>> lists(size_t(in.num_ctas));
    std::vector<double> load(size_t(in.num_ctas), 0.0);
    using QE = std::pair<double, int>;
    auto assign = [&](std::vector<Item>& items, bool distinct) {
        std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.cost > b.cost; });
        std::priority_queue<QE, std::vector<QE>, std::greater<QE>> pq;
        for (int c = 0; c < in.num_ctas; ++c) pq.push({load[size_t(c)], c});
        for (auto& it : items) {
            QE e = pq.top();
            pq.pop();
            load[size_t(e.second)] += it.cost;
            lists[size_t(e.second)].push_back(it.t);
            if (!distinct) pq.push({load[size_t(e.second)], e.second});
        }
        ++phase;
    };
    auto gemm = [&](uint8_t xsrc, uint8_t epi, int wmap, int xmap, int omap, int tile, int kb0, int nkb, int wbar,
                    int wcnt, int sbar) {
        AeTask t{};
        t.kind = kAeGemm;
        t.xsrc = xsrc;
        t.epi = epi;
        t.wmap = uint16_t(wmap);
        t.xmap = uint16_t(xmap);
        t.omap = uint16_t(omap);
        t.tile = uint16_t(tile);
        t.kb0 = uint16_t(kb0);
        t.nkb = uint16_t(nkb);
        t.wait_bar = uint16_t(wbar);
        t.wait_cnt = uint16_t(wcnt);
        t.sig_bar = uint16_t(sbar);
        t.phase = uint16_t(phase);
        return t;
    };
    // k-split so that tiles x splits approaches `target` tasks
    auto splits_for = [](int tiles, int kb, int target) {
        int s = std::max(1, std::min(kb, target / std::max(1, tiles)));
        const int per = (kb + s - 1) / s;
        return (kb + per - 1) / per;
    };
    const double kWB = double(kWTile);
    const int rec = in.record ? 1 : 0;
    const int kbW = W / 64;

    // ae.state_proj -> st
    const int bar_init = newbar();
    {
        std::vector<Item> it;
        for (int t = 0; t < W / 128; ++t)
            it.push_back({gemm(kXRows, kEpiInit, in.map_wst, 0, 0, t, 0, 1, 0, 0, bar_init), kWB});
        assign(it, false);
    }
    const int tiles_w = W / 128;
    const int ks_ao = splits_for(tiles_w, kbW, 32);
    const int ks_proj = splits_for(tiles_w, in.q_width / 64, 128);
    const int ks_down = splits_for(tiles_w, MLP / 64, 128);
    const int n_ao = tiles_w * ks_ao, n_proj = tiles_w * ks_proj, n_down = tiles_w * ks_down;
    const int tiles_qkv = NQ / 128, tiles_ffn = 2 * MLP / 128;
    const int pairs = (in.heads + 1) / 2;
    const int n_attn = pairs * in.key_blocks;
    int prev_bar = bar_init, prev_cnt = W / 128;
    int rec_slot = 0;
    for (int s = 0; s < FS; ++s) {
        const int bar_ap = newbar();
        {
            std::vector<Item> it;
            for (int t = 0; t < tiles_w; ++t) {
                AeTask x = gemm(kXRows, kEpiSilu, in.map_wap, 0, 0, t, 0, 1, prev_bar, prev_cnt, bar_ap);
                x.step = uint16_t(s);
                it.push_back({x, kWB});
            }
            assign(it, false);
        }
        const int bar_ao = newbar();
        {
            std::vector<Item> it;
            const int per = (kbW + ks_ao - 1) / ks_ao;
            for (int t = 0; t < tiles_w; ++t)
                for (int k = 0; k < ks_ao; ++k) {
                    const int kb0 = k * per, nkb = std::min(kbW, kb0 + per) - kb0;
                    it.push_back({gemm(kXBf16, kEpiRed, in.map_wao, in.map_ap, in.map_yh, t, kb0, nkb, bar_ap, tiles_w,
                                       bar_ao),
                                  nkb * kWB});
                }
            assign(it, false);
        }
        prev_bar = bar_ao;
        prev_cnt = n_ao;
        for (int l = 0; l < NA; ++l) {
            const int gl = s * NA + l, par = gl & 1;
            const int bar_qkv = newbar();
            {
                std::vector<Item> it;
                for (int t = 0; t < tiles_qkv; ++t) {
                    AeTask x = gemm(kXY, kEpiQkv, in.map_wqkv[size_t(l)], in.map_y, 0, t, 0, kbW, prev_bar, prev_cnt,
                                    bar_qkv);
                    x.step = uint16_t(s);
                    x.layer = uint16_t(l);
                    it.push_back({x, kbW * kWB});
                }
                assign(it, false);
            }
            const int bar_attn = newbar();
            {
                std::vector<Item> it;
                for (int rb = 0; rb < pairs; ++rb) {
                    const int bar_max = newbar();
                    for (int j = 0; j < in.key_blocks; ++j) {
                        AeTask x{};
                        x.kind = kAeAttn;
                        x.par = uint8_t(par);
                        x.wmap = uint16_t(in.map_kv[size_t(gl % int(in.map_kv.size()))]);
                        x.xmap = uint16_t(in.map_q);
                        x.omap = uint16_t(in.map_kvown);
                        x.nkb = uint16_t(in.map_oacc[size_t(par)]);
                        x.tile = uint16_t(rb);
                        x.kb0 = uint16_t(j);
                        x.wait_bar = uint16_t(bar_qkv);
                        x.wait_cnt = uint16_t(tiles_qkv);
                        x.sig_bar = uint16_t(bar_attn);
                        x.aux = uint16_t(bar_max);
                        x.step = uint16_t(s);
                        x.layer = uint16_t(l);
                        x.phase = uint16_t(phase);
                        it.push_back({x, 3.0 * kWB});
                    }
                }
                assign(it, true);
            }
            const int bar_proj = newbar();
            {
                std::vector<Item> it;
                const int kbq = in.q_width / 64, per = (kbq + ks_proj - 1) / ks_proj;
                for (int t = 0; t < tiles_w; ++t)
                    for (int k = 0; k < ks_proj; ++k) {
                        const int kb0 = k * per, nkb = std::min(kbq, kb0 + per) - kb0;
                        AeTask x = gemm(kXO, kEpiRed, in.map_wproj[size_t(l)], in.map_oacc[size_t(par)], in.map_y, t, kb0,
                                        nkb, bar_attn, n_attn, bar_proj);
                        x.par = uint8_t(par);
                        it.push_back({x, nkb * kWB});
                    }
                assign(it, false);
            }
            const int bar_ffn = newbar();
            {
                std::vector<Item> it;
                for (int t = 0; t < tiles_ffn; ++t) {
                    AeTask x = gemm(kXY, kEpiGate, in.map_wffn[size_t(l)], in.map_y, 0, t, 0, kbW, bar_proj, n_proj,
                                    bar_ffn);
                    x.par = uint8_t(par);
                    x.aux = uint16_t((std::min(tiles_ffn, 255) << 8) | std::min(t, 254));
                    if (t >= 255) x.aux = uint16_t((255 << 8) | 255);  // (never: mlp <= 8160)
                    it.push_back({x, kbW * kWB});
                }
                assign(it, false);
            }
            const int bar_down = newbar();
            {
                std::vector<Item> it;
                const int kbm = MLP / 64, per = (kbm + ks_down - 1) / ks_down;
                for (int t = 0; t < tiles_w; ++t)
                    for (int k = 0; k < ks_down; ++k) {
                        const int kb0 = k * per, nkb = std::min(kbm, kb0 + per) - kb0;
                        it.push_back({gemm(kXBf16, kEpiRed, in.map_wdown[size_t(l)], in.map_g, in.map_y, t, kb0, nkb,
                                           bar_ffn, tiles_ffn, bar_down),
                                      nkb * kWB});
                    }
                assign(it, false);
            }
            if (rec) {
                std::vector<Item> it;
                AeTask x{};
                x.kind = kAeRecY;
                x.wait_bar = uint16_t(bar_down);
                x.wait_cnt = uint16_t(n_down);
                x.sig_bar = uint16_t(bar_down);
                x.aux = uint16_t(rec_slot++);
                x.phase = uint16_t(phase);
                it.push_back({x, kWB});
                assign(it, false);
            }
            prev_bar = bar_down;
            prev_cnt = n_down + rec;
        }
        const int bar_head = newbar();
        {
            std::vector<Item> it;
            AeTask x = gemm(kXY, kEpiHead, in.map_whead, in.map_yh, 0, 0, 0, kbW, prev_bar, prev_cnt, bar_head);
            x.step = uint16_t(s);
            it.push_back({x, kbW * kWB / 4});
            assign(it, false);
        }
        if (rec) {
            std::vector<Item> it;
            AeTask x{};
            x.kind = kAeRecA;
            x.wait_bar = uint16_t(bar_head);
            x.wait_cnt = 1;
            x.sig_bar = uint16_t(bar_head);
            x.aux = uint16_t(s);
            x.phase = uint16_t(phase);
            it.push_back({x, kWB});
            assign(it, false);
        }
        prev_bar = bar_head;
        prev_cnt = 1 + rec;
    }
    need(nbar < 65535 && phase < 65535, "task table too large");
    {   // number of signallers per counter -> sig_cnt (the last one broadcasts)
        std::vector<int> cnt(size_t(nbar), 0);
        for (auto& l : lists)
            for (auto& t : l) ++cnt[t.sig_bar];
        for (auto& l : lists)
            for (auto& t : l) t.sig_cnt = uint16_t(cnt[t.sig_bar]);
    }
    size_t stride = 0;
    for (auto& l : lists) stride = std::max(stride, l.size() + 1);
    out.stride = int(stride);
    out.table.assign(size_t(in.num_ctas) * stride, AeTask{});
    for (size_t c = 0; c < lists.size(); ++c)
        std::copy(lists[c].begin(), lists[c].end(), out.table.begin() + c * stride);
    out.n_bars = nbar;
    out.n_phases = phase;
    out.n_tasks = 0;
    for (auto& l : lists) out.n_tasks += int(l.size());
    out.max_load = *std::max_element(load.begin(), load.end());
    out.min_load = *std::min_element(load.begin(), load.end());
    return out;
}

}  // namespace pi0b
