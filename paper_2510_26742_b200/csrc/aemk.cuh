// The action-expert megakernel (aemk.cu): the whole flow-matching loop of the pi0 action
// expert — ae.state_proj, then per flow step ae.action_proj, ae.action_out, 18 x {ae.qkv,
// ae.attn, ae.proj, ae.ffn, ae.down}, ae.head + Euler (proj/src/builder.cpp:291-363) — as ONE
// persistent launch of one CTA per SM.
//
// The host turns the fused graph into a static task table: every node instance is split into
// tasks (a 64-feature output tile over a range of 64-wide k-blocks, or one attention
// (head-pair, key-range) tile), tasks are assigned to CTAs, and each CTA walks its own list in
// global phase order.  Ordering between node instances uses phase counters instead of kernel
// boundaries: every task bumps its phase's counter with a release atomic, and a task waits
// until the counter of the phase it reads reaches that phase's task count.  Weights never
// depend on activations, so a dedicated producer warp streams each CTA's weight tiles through
// a shared-memory ring ahead of all dependency waits: HBM keeps streaming the next layer's
// weights while the current layer's dependencies resolve (the "software barrier" + weight
// prefetch of PAPER.md:232-242 / SURVEY.md 7.3).
//
// The kernel runs as 2-CTA clusters (cooperative launch): an ae.qkv tile is split over K between
// the two CTAs of a cluster; the helper pushes its fp32 partial and row sums of squares into the
// owner's shared memory (DSMEM) and the owner runs the epilogue.  No task ever finalises
// another task's output through global memory: the nonlinear GEMMs (ae.qkv, ae.ffn,
// ae.head) run over the full K and read the fp32 residual stream directly, computing the
// RmsStats row sums of squares while they stage it; only the residual updates (ae.proj,
// ae.down, ae.action_out) are split over K, and they add straight into the residual stream.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <vector>

namespace pi0b {

enum AeTaskKind : uint8_t { kAeEnd = 0, kAeGemm = 1, kAeAttn = 2, kAeRecY = 3, kAeRecA = 4 };

// How the 64-row activation operand of a GEMM task reaches shared memory (always cp.async).
enum AeXSrc : uint8_t {
    kXBf16 = 0,  // bf16 rows straight into the swizzled operand slot
    kXY = 1,     // fp32 residual stream (full K); workers convert to bf16 and accumulate the row
                 // sums of squares (the RmsStats node, proj/src/evaluate.cpp:308-309)
    kXO = 2,     // attention partials (bf16, per key range, with row max / sum): combined
    kXRows = 3,  // small fp32 rows (Euler state / robot state), K <= 64
};

enum AeEpi : uint8_t {
    kEpiRed = 0,   // fp32 split-K partial -> red.add into the residual stream (Residual epilogue)
    kEpiQkv = 1,   // RmsScale -> RoPE -> bf16 q | k | v   (ae.ln1 + ae.qkv)
    kEpiGate = 2,  // RmsScale -> up * gelu(gate) -> bf16  (ae.ln2 + ae.ffn)
    kEpiSilu = 3,  // silu(z + bias_table[step]) -> bf16; resets y = [st ; b_out] (ae.action_proj)
    kEpiHead = 4,  // a += (RmsScale z + b) / FS                      (ae.ln_out + ae.head + Euler)
    kEpiInit = 5,  // st = z + b                                       (ae.state_proj)
};

// A dense row-major matrix operand (device pointer + shape + pitch in elements).
struct alignas(16) AeMat {
    const void* ptr;
    int rows, cols, ld, pad_[3];
};
static_assert(sizeof(AeMat) == 32, "AeMat layout");

struct AeTask {
    uint8_t kind, xsrc, epi, rowoff;  // rowoff: kEpiRed target rows start at y row `rowoff`
    uint16_t wmat, xmat;              // AeMat indices (weights / activation)
    uint16_t ncol;                    // GEMM: output tile width, 64 or 128 (0 = 64); ATTN: 1 = one head
    uint16_t tile;                    // GEMM: output tile (ncol features); ATTN: head pair
    uint16_t kb0, nkb;                // GEMM: k-block range; ATTN: key split, #key blocks
    uint16_t wait_bar, wait_cnt;      // wait until counter wait_bar reaches wait_cnt (cnt > 0)
    uint16_t sig_bar;                 // counter of the phase this task belongs to
    uint16_t aux;                     // REC: record slot
    uint16_t step, layer;             // flow step, AE layer
    uint16_t phase;                   // global phase index (debug limit)
    uint16_t pair;                    // full-K tile split over K in a 2-CTA cluster: 1 owner / 2 helper
                                      // (owner finalises), or symmetric (each finalises half):
                                      // 3 / 4 128-wide ae.ffn tiles, 5 / 6 64-wide ae.qkv tiles
};
static_assert(sizeof(AeTask) == 32, "AeTask layout");

struct AeParams {
    const AeTask* tasks;
    int task_stride;               // tasks per CTA row of the table
    const AeMat* mats;             // operand table
    unsigned* bars;                // [n_bars] phase arrival counters, zero on entry
    int n_bars;
    float* y;                      // [64, W]   residual stream (row 0 = state token)
    float* a;                      // [C, lda]  Euler state
    int lda;
    const float* state;            // [state_dim] fp32
    float* st;                     // [W] state token (ae.state_proj output)
    __nv_bfloat16* qkv;            // [64, n_qkv]
    __nv_bfloat16* ap;             // [C, W]
    __nv_bfloat16* g;              // [64, mlp]
    __nv_bfloat16* opart;          // [splits][64, q_width] normalised attention partials
    float2* ml;                    // [splits][heads * 64] (row max (log2 units), row sum)
    const float* rope_cs;          // [positions][128] {cos, sin}
    const float* table;            // [FS, W] SiluBias table of ae.action_proj
    const float* b_state;          // [W]
    const float* b_out;            // [W]
    const float* b_head;           // [act]
    float* rec_y;                  // record mode: [slots][64, W]
    float* rec_a;                  // record mode: [slots][C, lda]
    int width, n_qkv, q_width, mlp, act_dim, state_dim, chunk, heads;
    int rope_pos0, rope_cols;      // AE RoPE positions start at the prefix length L
    int kv_rows0;                  // Lp = L rounded up to 32: first key index of the expert's own rows
    int kv_valid0;                 // L: cached keys [kv_valid0, kv_rows0) are padding (masked)
    int kcol_cache, kcol_own;      // first K column in the LLM KV cache / in the AE qkv rows
    int key_blocks;                // ceil((L + 64) / 64) key blocks of 64
    int attn_splits;               // key ranges per head pair (<= 3 key blocks each)
    float scale_log2, inv_width, eps, euler;
    int limit_phase;               // run only tasks with phase < limit (debug / parity probes)
    unsigned long long* trace;     // optional [ctas][stride][16] globaltimer stamps per task
    unsigned long long* dbg;       // optional [ctas][128] per-k-block stamps of the first ae.qkv task
    // attention V tiles by TMA (32-row boxes of 64 columns, 128-byte swizzle): [0, n) = the LLM KV
    // caches (attention task aux = index), [n] = the action expert's own q|k|v rows (32-row
    // boxes), [n + 1] = the same with 64-row boxes (Q tiles)
    const CUtensorMap* vmaps;
    int n_vmaps;
};

// Host planner: dimensions + operand indices in, per-CTA task table out.
struct AePlanInput {
    int num_ctas;
    int width, n_qkv, q_width, mlp, layers, flow_steps, heads, chunk, act_dim, state_dim;
    int rope_cols, kv_rows0, key_blocks;
    bool record;
    int ao_tasks = 64, proj_tasks = 128, down_tasks = 128;  // split-K task targets per phase
    int proj_ncol = 128, down_ncol = 64, ao_ncol = 64;     // residual-update tile widths (64 or 128)
    bool pair_qkv = true;  // ae.qkv tiles split over K between the two CTAs of a cluster (DSMEM)
    bool sym_qkv = true;      // ae.qkv pairs exchange symmetrically (each CTA finalises half)
    bool attn_single = true;  // one attention task per (head, key range) instead of (head pair, range)
    bool per_head_proj = true;  // ae.proj tasks wait only for their head's attention key ranges
    bool pair_ffn = true;  // ae.ffn as 128-wide tiles split over K, symmetric exchange (mat_wffn kTilePlain128)
    int mat_wst, mat_wap, mat_wao, mat_whead;
    std::vector<int> mat_wqkv, mat_wproj, mat_wffn, mat_wdown, mat_kv;
    int mat_y, mat_yh, mat_ap, mat_g, mat_qkv;  // fp32 y rows 0.. / rows 1.. (ae.act_rows)
};

// Weight row order of one tile of a tile-contiguous AE weight copy (64-row tiles; ae.proj uses
// plain 128-row tiles)
// (kernels_misc.cu tile_weight_kernel): plain, or "paired" — tile 2T + s of a matrix packed in
// 128-row groups [64 | 64 partners] (kPermRope qkv, kPermGate64 ffn) takes rows
// 128T + 32s + [0, 32) followed by their partners 128T + 64 + 32s + [0, 32).
enum AeTileOrder : int { kTilePlain = 0, kTilePaired = 1, kTilePlain128 = 2 };

struct AePlan {
    std::vector<AeTask> table;  // [num_ctas][stride]
    int stride = 0, n_bars = 0, n_phases = 0, n_tasks = 0, attn_splits = 1;
    double max_load = 0, min_load = 0;  // weight bytes per CTA
};

AePlan ae_plan(const AePlanInput& in);
cudaError_t aemk_configure();
// cluster: launch as 2-CTA clusters (required when the plan has pair tasks); without pair tasks
// the kernel also runs as a plain cooperative launch (e.g. under ncu, which cannot replay the
// cooperative + cluster launch).
cudaError_t aemk_launch(const AeParams& p, int grid, cudaStream_t stream, bool cluster = true);

}  // namespace pi0b
