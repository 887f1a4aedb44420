/*
 * pi0b — B200-native (sm_100a) pi0 inference engine: the C-ABI boundary.
 *
 * This is the drop-in replacement for the reference's C++ inference API
 *     rtvla::gen_weights / rtvla::gen_inputs / rtvla::evaluate
 * (proj/include/rtvla/evaluate.hpp:38-44, proj/src/evaluate.cpp:38-85,365-370) for the
 * fused pi0 graph built by rtvla::build_pi0_graph (proj/src/builder.cpp:197-367).
 * Plain C types only: no torch, no rtvla, no CUDA types in any signature.  The C++
 * adaptor that takes rtvla::Graph / WeightStore / Inputs and forwards here lives in
 * include/pi0b_rtvla.hpp; INTEGRATION.md shows how a reference caller binds it.
 *
 * Conventions:
 *   - every function returns 0 (PI0B_OK) on success, a negative PI0B_E* code or a
 *     positive cudaError_t value on failure; pi0b_last_error() describes the last
 *     failure of the calling thread;
 *   - tensors are dense row-major fp64 host arrays with the reference's shapes;
 *   - an engine is bound to one device and is not safe for concurrent calls
 *     (create one engine per thread/stream, as the reference's std::async verifiers
 *     create one Evaluator per call, proj/src/passes.cpp:864-867).
 */
#ifndef PI0B_H_
#define PI0B_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PI0B_OK 0
#define PI0B_E_INVALID (-1)     /* bad argument / unknown node id / shape mismatch (ShapeError) */
#define PI0B_E_UNSUPPORTED (-2) /* configuration outside what the kernels implement          */
#define PI0B_E_STATE (-3)       /* call out of order (e.g. run before weights are loaded)     */
#define PI0B_E_NUMERIC (-4)     /* non-finite action output (NumericError)                    */

/* Mirrors rtvla::ModelConfig field by field (proj/include/rtvla/graph.hpp:114-160). */
typedef struct pi0b_model_config {
    int views, prompt_tokens, tokens_per_view, chunk_len, flow_steps;
    int ve_layers, ve_width, ve_heads, ve_head_dim, ve_mlp, ve_patch_in;
    int llm_layers, llm_width, llm_q_heads, llm_head_dim, llm_kv_heads, llm_mlp;
    int ae_layers, ae_width, ae_q_heads, ae_head_dim, ae_kv_heads, ae_mlp, ae_action_dim,
        ae_state_dim;
} pi0b_model_config;

typedef struct pi0b_engine_options {
    int device;             /* CUDA ordinal                                              */
    int use_cuda_graph;     /* 1: capture the whole forward as one CUDA graph (default)   */
    int record_checkpoints; /* 1: keep every node instance's output for parity checks    */
    /* View-sharded vision encoder: ve_shards > 1 engines (one per GPU) each run
     * the VE for views [ve_shard*V/ve_shards, (ve_shard+1)*V/ve_shards); every layer's q|k|v rows
     * are all-gathered over peer memory before the joint attention (proj/src/builder.cpp:219-222)
     * and the llm.proj_in rows are gathered into shard 0, which runs the LLM and the action
     * expert.  Shards other than 0 serve run_prefix only.  0 or 1: no sharding. */
    int ve_shards;
    int ve_shard;
    /* CTAs of the action-expert megakernel (one per SM): 0 = every SM.  Fewer leaves SMs to work
     * running concurrently on other streams (the streaming runtime's prefix). */
    int ae_ctas;
} pi0b_engine_options;

typedef struct pi0b_engine pi0b_engine;

/* rtvla::default_config() (proj/src/builder.cpp:10-12): 2 views, empty prompt. */
void pi0b_default_config(pi0b_model_config* cfg);

/* Engine lifetime.  Allocates the weight arena (bf16), activations, KV cache. */
int pi0b_engine_create(const pi0b_model_config* cfg, const pi0b_engine_options* opt,
                       pi0b_engine** out);
void pi0b_engine_destroy(pi0b_engine* e);
/* An engine that reads `donor`'s weight arena instead of allocating its own (same config and
 * device): several KV caches / input sets over one copy of the 5.2 GB of weights, e.g. the
 * streaming runtime's double-buffered KV.  Weights are loaded through the donor only
 * (gen_weights / set_weight on this engine return PI0B_E_STATE); destroy it before the donor. */
int pi0b_engine_create_shared(const pi0b_model_config* cfg, const pi0b_engine_options* opt, pi0b_engine* donor,
                              pi0b_engine** out);

/* Device-side rtvla::gen_weights(build_pi0_graph(cfg), seed): the same SplitMix64 /
 * FNV-1a streams, rounded once to bf16 (proj/src/evaluate.cpp:38-75). */
int pi0b_engine_gen_weights(pi0b_engine* e, uint64_t seed);

/* Host weights, one WeightSet instance at a time (proj/include/rtvla/evaluate.hpp:16-27):
 * w is W[k, m] row-major, bias is [m] or NULL. */
int pi0b_engine_set_weight(pi0b_engine* e, const char* node_id, int64_t instance, const double* w,
                           int64_t k, int64_t m, const double* bias, int64_t bias_len);
/* WeightSet::bias_table of ae.action_proj, [flow_steps, m]. */
int pi0b_engine_set_bias_table(pi0b_engine* e, const char* node_id, const double* table,
                               int64_t rows, int64_t m);

/* One full inference == rtvla::evaluate(g, w, x) (proj/src/evaluate.cpp:365-370).
 * patches [views*tokens_per_view, ve_patch_in], state [1, ae_state_dim],
 * noise [chunk_len, ae_action_dim], prompt [prompt_tokens, llm_width] (NULL when 0),
 * actions_out [chunk_len, ae_action_dim]. */
int pi0b_engine_run(pi0b_engine* e, const double* patches, const double* state, const double* noise,
                    const double* prompt, double* actions_out);

/* run() from camera frames instead of patches: images [views][height][width*3]
 * fp64, channels interleaved; resized on the device to the patch grid (half-pixel-centre bilinear,
 * bit-identical to rtvla::bilinear_resize, proj/src/tensor.cpp:180-212) and cut into the
 * ve.embed patches (row view*g*g + (y/P)*g + x/P, feature ((y%P)*P + x%P)*3 + c). */
int pi0b_engine_run_images(pi0b_engine* e, const double* images, int height, int width, const double* state,
                           const double* noise, const double* prompt, double* actions_out);
/* The same resize + img2col as a device op: images (device) -> patches (device) [views*(side/patch)^2,
 * patch*patch*channels]. */
int pi0b_image_patches(const double* images, int views, int height, int width, int channels, int side,
                       int patch, double* patches, void* stream);
/* The host-side conversion run() applies to the patches before their DMA (host memory in and
 * out, no GPU needed): dst[i] = bf16(float(src[i])), round-to-nearest-even at both steps, NaN ->
 * 0x7fff -- bit-identical to the device conversion (__float2bfloat16_rn(float(x))). */
int pi0b_f64_to_bf16_host(const double* src, long long n, uint16_t* dst);
/* The RoPE table the engine uploads (host memory, no GPU): out[(p * head_dim/2 + j) * 2 + {0, 1}] =
 * fp32 {cos, sin} of p * 10000^(-2j/head_dim), computed in fp64 exactly as rtvla::make_rope_table
 * (proj/src/tensor.cpp:133-148), for positions [0, positions). */
int pi0b_rope_table_host(int positions, int head_dim, float* out);

/* ------------------------------------------------------------------ unfused checkpoints
 * Weight rules for the naive graph (rtvla::build_pi0_graph_naive, proj/src/builder.cpp:369-541),
 * host memory in and out, no GPU needed; bit-identical to rtvla::apply_weight_rules
 * (proj/src/passes.cpp:692-790).  include/pi0b_rtvla.hpp fuse_naive() applies them to a whole
 * naive WeightStore (the concatenations are plain copies there). */
/* rtvla::time_embedding(step, dim, flow_steps) (proj/src/evaluate.cpp:23-36) -> out[dim]. */
int pi0b_time_embedding(int step, int dim, int flow_steps, double* out);
/* PremultiplyDiag (passes.cpp:706-721): w[k, m] row r *= gamma[r], in place. */
int pi0b_premultiply_rows(double* w, int64_t k, int64_t m, const double* gamma);
/* ComposeTimeFold (passes.cpp:754-785): the action time MLP (ae.act_in: w_act [act, width],
 * b_act; ae.mlp_in: w_mix [t_dim + width, mix_cols], b_mix) folded into ae.action_proj:
 * w_out [act, mix_cols] and its per-flow-step bias table table_out [flow_steps, mix_cols]. */
int pi0b_fold_time_mlp(const double* w_act, int64_t act, int64_t width, const double* b_act, const double* w_mix,
                       int64_t t_dim, int64_t mix_cols, const double* b_mix, int flow_steps, double* w_out,
                       double* table_out);

/* View-sharded VE plumbing (see pi0b_engine_options): the device buffers a shard exposes to its
 * peers, and the peers' buffers mapped into this process (same process: the pointers themselves;
 * across processes: pi0b_ipc_export / pi0b_ipc_open of each buffer).  set_ve_peers must be called
 * before the first run; peers[ve_shard] is ignored. */
typedef struct pi0b_ve_buffers {
    void* qkv[2]; /* gathered ve.qkv rows, double-buffered by layer parity [T, 3 ve_width] bf16 */
    void* x;      /* llm.proj_in output rows [L, llm_width] fp32                                  */
    void* xb;     /* the same, bf16                                                               */
    void* stats;  /* prefix row-statistics arena (fp32)                                           */
    void* sync;   /* flags [8] (one per source shard) + inference counter + arrival counter       */
} pi0b_ve_buffers;
int pi0b_engine_ve_buffers(pi0b_engine* e, pi0b_ve_buffers* out);
int pi0b_engine_set_ve_peers(pi0b_engine* e, const pi0b_ve_buffers* peers, int n);
/* cudaIpcGetMemHandle / cudaIpcOpenMemHandle of a device allocation (64-byte handle). */
int pi0b_ipc_export(const void* dptr, uint8_t* handle64);
int pi0b_ipc_open(const uint8_t* handle64, void** dptr);
int pi0b_ipc_close(void* dptr);

/* Streaming split of run(): the prefix (VE + LLM, fills the KV cache) and the action
 * expert (all flow steps against the cached prefix KV). */
int pi0b_engine_run_prefix(pi0b_engine* e, const double* patches, const double* prompt);
int pi0b_engine_run_action(pi0b_engine* e, const double* state, const double* noise,
                           double* actions_out);

/* Full-streaming runtime (the real execution of what the reference only simulates,
 * proj/include/rtvla/streamsim.hpp:54-131): a camera stream at frame_rate feeds the prefix (VE + LLM)
 * into one of two KV buffers (two engines over one shared weight arena); an action-expert stream runs
 * control ticks at up to ae_rate on the KV chosen by kv_policy with the freshest sensor sample;
 * each tick writes its chunk into a trajectory buffer of trajectory_rate slots whose commit cursor
 * advances with wall time.  Runs `seconds` of synthetic frames/sensors (random patches / state /
 * noise) on one GPU and reports the reference's loop metrics (rtvla::measure_loops,
 * streamsim.hpp:166-205) measured on the real execution. */
typedef struct pi0b_stream_options {
    double frame_rate;       /* camera frames per second (30)                                  */
    int camera_latency;      /* frames between capture and availability (2)                     */
    double ae_rate;          /* target action-expert ticks per second (480)                     */
    double trajectory_rate;  /* trajectory slots per second (480)                               */
    int kv_policy;           /* 0 most_recent, 1 frame_sticky (rtvla::KvPolicy)                 */
    int device;
    int prefix_sms;          /* SMs the action-expert ticks leave to the concurrent prefix
                                (0: 20; < 0: none -- the megakernel takes every SM)             */
} pi0b_stream_options;

typedef struct pi0b_stream_report {
    double seconds;             /* wall time of the run                                         */
    int64_t frames, ticks;      /* prefixes / action-expert ticks completed                     */
    double vlm_per_s, ae_per_s;
    double quick_mean_ms, quick_best_ms, quick_worst_ms;  /* sensor sample -> first commit of its window */
    int64_t quick_count;
    double slow_mean_ms, slow_best_ms, slow_worst_ms;     /* frame capture -> first commit using its KV  */
    int64_t slow_count;
    double prefix_p50_ms, tick_p50_ms, tick_p99_ms;       /* issue -> completion, per operation           */
    int64_t committed_slots, overwritten_slots;           /* trajectory buffer                           */
} pi0b_stream_report;

/* cfg.flow_steps is the number of flow steps per tick (1 = one "AE pass" of the paper). */
int pi0b_stream_run(const pi0b_model_config* cfg, uint64_t weight_seed, const pi0b_stream_options* opt,
                    double seconds, pi0b_stream_report* report);

/* Device-resident replay of the last inputs (no host copies): 0 = full, 1 = prefix,
 * 2 = action.  `stream` is a cudaStream_t (NULL = the engine's stream).  Asynchronous. */
int pi0b_engine_replay(pi0b_engine* e, int part, void* stream);
int pi0b_engine_sync(pi0b_engine* e);
/* Number of kernels one replay of `part` launches. */
int pi0b_engine_kernel_count(pi0b_engine* e, int part);

/* Average device time (ms) of one launch of the kernels of node `node_id` (all of its
 * instances, `reps` passes, CUDA events on the engine stream).  Used for the roofline. */
int pi0b_engine_time_node(pi0b_engine* e, const char* node_id, int reps, double* ms_per_launch,
                          int* launches);

/* Debug (PI0B_AE_TRACE=1 at engine creation): the action-expert megakernel's task table
 * (32-byte records, csrc/aemk.cuh AeTask) and 16 globaltimer stamps per task from the last launch
 * (csrc/aemk.cu: worker start / dependency met / operands staged / published, weight producer,
 * MMA and epilogue / attention sub-steps).  cap = table entries. */
int pi0b_engine_ae_trace(pi0b_engine* e, void* tasks, unsigned long long* stamps, int64_t cap, int* ctas,
                         int* stride);

/* Text listing of the launch plan, one op per line (index, part, kind, node, instance, grid). */
int pi0b_engine_describe(pi0b_engine* e, char* buf, int64_t cap);

/* Parity hook (record_checkpoints=1): the output of node `node_id` instance `inst` from
 * the last run, as fp32 [rows, cols].  Node ids/instances are the reference graph's. */
int pi0b_engine_read_checkpoint(pi0b_engine* e, const char* node_id, int64_t inst, float* out,
                                int64_t rows, int64_t cols);

/* Thread-local description of the last failure. */
const char* pi0b_last_error(void);

/* ------------------------------------------------------------------ kernel level
 * Device-pointer entry points used by the unit parity tests (stream = cudaStream_t). */

typedef struct pi0b_gemm_desc {
    const void* a; int64_t lda;     /* bf16 [M, K]                                  */
    const void* w; int64_t ldw;     /* bf16 [N, K] (packed weight)                  */
    int M, N, K;
    int bn;                         /* tile width 64 / 128 / 256                    */
    int splits;                     /* split-K factor, clamped to [1, 8]: the splits of
                                       a tile run as one cluster, reduced over DSMEM  */
    int mode, flags;                /* see paper_2510_26742_b200/csrc/gemm.cuh      */
    const float* row_stats; float inv_width, eps;
    const float* bias;
    const float* table_row;
    const float* rope_cs; int rope_pos0, rope_cols;
    float resid_scale;
    void* out; int64_t ldo;
    void* outb; int64_t ldob;
    float* out_stats;
    const float* row0_src;
    float* ws; int* counters;       /* reserved (ignored; kept for ABI stability)   */
} pi0b_gemm_desc;
int pi0b_gemm(const pi0b_gemm_desc* d, void* stream);
/* Swap-AB small-M GEMM (M <= 64; the action expert's weight-streaming kernel): `w` is the
 * packed [N, K] weight, `a` the [M, K] activations, K split over a cluster of `cluster`
 * (1, 2, 4, 8) CTAs reduced through distributed shared memory.  rope_cols > 0 selects the
 * RoPE pair packing, mode 1 (gate) the 64-granule gate packing. */
int pi0b_gemm_skinny(const pi0b_gemm_desc* d, int cluster, void* stream);

typedef struct pi0b_attn_desc {
    int head_dim;                   /* 72 or 256                                    */
    const void* q; int64_t ldq; int q_rows, heads, kv_heads;
    const void* k0; const void* v0; int64_t ld0; int rows0;
    const void* k1; const void* v1; int64_t ld1; int rows1;
    void* out; int64_t ldo;
    int kv_splits;                  /* 0/1: one pass; 2, 4, 8: key splits (cluster) */
    float* ws; int* counters;       /* ws: key-split workspace, pi0b_attention_ws_floats() floats
                                       (kv_splits > 1); counters: unused, kept for ABI layout */
    int rows0_valid;                /* > 0: keys [rows0_valid, rows0) of segment 0 are padding (masked) */
} pi0b_attn_desc;
int pi0b_attention(const pi0b_attn_desc* d, void* stream);
/* Workspace floats / counters an attention launch with these dims needs. */
int64_t pi0b_attention_ws_floats(const pi0b_attn_desc* d);

/* Device SplitMix64 draw of random_tensor(rows, cols, lo, hi, seed) into fp64 (parity
 * of the parameter streams) and into the packed bf16 layout. */
int pi0b_random_f64(double* dst, int64_t n, uint64_t seed, double lo, double hi, void* stream);
/* perm: 0 identity, 1 gate (128 granule), 2 gate (64 granule), 3 RoPE pairs (rope_cols). */
int pi0b_random_packed_bf16(void* dst, int64_t ldk, int k, int m, int perm, int rope_cols, uint64_t seed,
                            double lo, double hi, void* stream);
/* FNV-1a seed derivation (proj/src/tensor.cpp:24-40). */
uint64_t pi0b_seed_hash(uint64_t seed, const char* label, uint64_t a, uint64_t b);

#ifdef __cplusplus
}
#endif

#endif /* PI0B_H_ */
