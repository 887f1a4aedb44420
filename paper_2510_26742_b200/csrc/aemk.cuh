// The action-expert megakernel (aemk.cu): the whole flow-matching loop of the pi0 action
// expert — ae.state_proj, then per flow step ae.action_proj, ae.action_out, 18 x {ae.qkv,
// ae.attn, ae.proj, ae.ffn, ae.down}, ae.head + Euler (proj/src/builder.cpp:291-363) — as ONE
// persistent launch of one CTA per SM.
//
// The host turns the fused graph into a static task table: every node instance is split into
// tasks (a 128-feature output tile over a range of 64-wide k-blocks, or one attention
// (head-pair, key-block) tile), tasks are assigned to CTAs, and each CTA walks its own list in
// global phase order.  Ordering between node instances uses monotonically increasing global
// counters (one per phase) instead of kernel boundaries: a task waits until the counter of the
// phase it reads reaches that phase's task count, and bumps its own phase counter when its
// outputs are globally visible.  Weights never depend on activations, so a dedicated TMA warp
// streams each CTA's weight tiles through a shared-memory ring ahead of all dependency waits:
// HBM keeps streaming the next layer's weights while the current layer's barriers resolve
// (the "software barrier" + weight prefetch of PAPER.md:232-242 / SURVEY.md 7.3).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <vector>

namespace pi0b {

enum AeTaskKind : uint8_t { kAeEnd = 0, kAeGemm = 1, kAeAttn = 2, kAeRecY = 3, kAeRecA = 4 };

// How the 64-row activation operand of a GEMM task reaches shared memory.
enum AeXSrc : uint8_t {
    kXBf16 = 0,  // bf16 [rows, K] tensor map, TMA straight into the swizzled operand slot
    kXY = 1,     // fp32 residual stream via TMA; workers convert to bf16 and accumulate the
                 // row sums of squares (the RmsStats node, evaluate.cpp:308-309) for the epilogue
    kXO = 2,     // fp32 un-normalised attention output O_acc via TMA, rows scaled by 1/l
    kXRows = 3,  // small fp32 rows (Euler state / robot state) loaded by the workers
};

enum AeEpi : uint8_t {
    kEpiRed = 0,   // fp32 tile -> TMA reduce-add into the residual stream (Residual epilogue)
    kEpiQkv = 1,   // RmsScale -> RoPE -> bf16 q | k | v   (ae.ln1 + ae.qkv)
    kEpiGate = 2,  // RmsScale -> up * gelu(gate) -> bf16  (ae.ln2 + ae.ffn)
    kEpiSilu = 3,  // silu(z + bias_table[step]) -> bf16; resets y = [st ; b_out] (ae.action_proj)
    kEpiHead = 4,  // a += (RmsScale z + b) / FS                      (ae.ln_out + ae.head + Euler)
    kEpiInit = 5,  // st = z + b                                       (ae.state_proj)
};

struct AeTask {
    uint8_t kind, xsrc, epi, par;  // par: layer parity of the attention accumulators
    uint16_t wmap, xmap, omap;     // tensor-map indices (weights / activation / reduce target)
    uint16_t tile;                 // GEMM: 128-feature output tile; ATTN: head pair
    uint16_t kb0, nkb;             // GEMM: k-block range; ATTN: key block in kb0
    uint16_t wait_bar, wait_cnt;   // wait until bars[wait_bar] >= wait_cnt
    uint16_t sig_bar;              // bars[sig_bar] += 1 when done
    uint16_t aux;                  // ATTN: rendezvous counter; REC: record slot
    uint16_t step, layer;          // flow step, AE layer
    uint16_t phase;                // global phase index (debug limit)
    uint16_t sig_cnt;              // tasks that signal sig_bar (the last one broadcasts)
};
static_assert(sizeof(AeTask) == 32, "AeTask layout");

struct AeParams {
    const AeTask* tasks;
    int task_stride;               // tasks per CTA row of the table
    const void* maps;              // CUtensorMap[] in global memory (64-byte aligned)
    unsigned* bars;                // phase counters, zero on entry
    unsigned* mbox;                // [ctas][n_bars] completion flags, zero on entry: the last
                                   // task of a phase sets the phase's flag in every CTA's own
                                   // line, so waiting CTAs poll disjoint L2 lines
    int n_bars;
    float* y;                      // [64, W]   residual stream (row 0 = state token)
    float* a;                      // [C, lda]  Euler state
    int lda;
    const float* state;            // [state_dim] fp32
    float* st;                     // [W] state token (ae.state_proj output)
    __nv_bfloat16* qkv;            // [64, n_qkv]
    __nv_bfloat16* ap;             // [C, W]
    __nv_bfloat16* g;              // [64, mlp]
    float* oacc[2];                // [64, q_width] un-normalised attention output, per parity
    float* lacc[2];                // [heads * 64]  softmax denominators
    unsigned* mmax[2];             // [heads * 64]  order-preserving keys of the row maxima
    const float* rope_cs;          // [positions][128] {cos, sin}
    const float* table;            // [FS, W] SiluBias table of ae.action_proj
    const float* b_state;          // [W]
    const float* b_out;            // [W]
    const float* b_head;           // [act]
    float* rec_y;                  // record mode: [slots][64, W]
    float* rec_a;                  // record mode: [slots][C, lda]
    int width, n_qkv, q_width, mlp, act_dim, state_dim, chunk, heads;
    int rope_pos0, rope_cols;      // AE RoPE positions start at the prefix length L
    int kv_rows0;                  // L: rows of the cached LLM K/V segment
    int kcol_cache, kcol_own;      // first K column in the LLM KV cache / in the AE qkv rows
    int key_blocks;                // ceil((L + 64) / 64)
    float scale_log2, inv_width, eps, euler;
    int limit_phase;               // run only tasks with phase < limit (debug / parity probes)
    int w_inflight;                // weight tiles in flight per CTA (queueing latency vs bandwidth)
    unsigned long long* trace;     // optional [ctas][stride][8] globaltimer stamps per task (pi0b.h)

};

// Host planner: dimensions + tensor-map indices in, per-CTA task table out.
struct AePlanInput {
    int num_ctas;
    int width, n_qkv, q_width, mlp, layers, flow_steps, heads, chunk, act_dim, state_dim;
    int rope_cols, kv_rows0, key_blocks;
    bool record;
    int map_wst, map_wap, map_wao, map_whead;
    std::vector<int> map_wqkv, map_wproj, map_wffn, map_wdown, map_kv;
    int map_y, map_yh, map_ap, map_g, map_q, map_kvown;
    std::array<int, 2> map_oacc;
};

struct AePlan {
    std::vector<AeTask> table;  // [num_ctas][stride]
    int stride = 0, n_bars = 0, n_phases = 0, n_tasks = 0;
    double max_load = 0, min_load = 0;  // weight bytes per CTA
};

AePlan ae_plan(const AePlanInput& in);
cudaError_t aemk_configure();
cudaError_t aemk_launch(const AeParams& p, int grid, cudaStream_t stream);

}  // namespace pi0b
