// Host runtime of the pi0 engine behind the C-ABI in include/pi0b.h.
//
// The engine turns the fused pi0 graph of rtvla::build_pi0_graph (proj/src/builder.cpp:
// 197-367) into a static launch plan: every node instance becomes one kernel launch
// (tcgen05 GEMM with its fused epilogue, or flash attention), every buffer is
// pre-allocated, the instance algebra of the reference (proj/include/rtvla/graph.hpp:3-15,
// proj/src/evaluate.cpp:120-150) is resolved at plan time into fixed device pointers,
// and the whole forward is captured once as a CUDA graph and replayed with no per-step
// host work.  The memoised demand-driven evaluator of the reference
// (proj/src/evaluate.cpp:89-361) thus becomes a straight-line schedule:
//   VE   ve.embed, 27 x {ve.qkv, ve.attn, ve.proj, ve.fc1, ve.fc2}
//   LLM  llm.proj_in (+prompt rows), 18 x llm.qkv (KV cache), 17 x {attn, proj, ffn, down}
//   AE   ae.state_proj, 10 x {action_proj, action_out+suffix, 18 x {qkv, attn, proj, ffn,
//        down}, head(+Euler)}
// RmsStats nodes have no launch: their row sums of squares are accumulated by the
// epilogue of the kernel that produced the residual stream.
#include "../../include/pi0b.h"
#include "aemk.cuh"
#include "veshard.cuh"
#include "attention.cuh"
#include "gemm.cuh"
#include "numerics.cuh"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <tuple>
#include <initializer_list>
#include <random>
#include <chrono>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace pi0b {

cudaError_t gemm_configure();
cudaError_t launch_gemm(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                        cudaStream_t stream);
cudaError_t fattn_configure();
FaMaps make_fattn_maps(const AttnParams& p, int head_dim);
cudaError_t launch_fattn(int head_dim, const FaMaps& maps, const AttnParams& p, cudaStream_t stream);
void fattn_set_pdl(bool on);
cudaError_t launch_gen_weight(__nv_bfloat16* dst, long long ldk, int k, int m, int perm, int rope_cols,
                              uint64_t seed, double lo, double hi, cudaStream_t st);
cudaError_t launch_pack_weight(__nv_bfloat16* dst, long long ldk, const double* w, int k, int m,
                               int perm, int rope_cols, cudaStream_t st);
cudaError_t launch_tile_weight(const __nv_bfloat16* src, int rows, int k, long long ldk, __nv_bfloat16* dst, int order,
                               cudaStream_t st);
cudaError_t skinny_configure();
int skinny_tiles(int n_packed);
cudaError_t launch_skinny(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p, int n_packed,
                          int cluster, bool pdl, cudaStream_t stream);
enum PackPerm { kPermNone = 0, kPermGate128 = 1, kPermGate64 = 2, kPermRope = 3 };
cudaError_t launch_gen_vector(float* dst, int n, uint64_t seed, double lo, double hi, cudaStream_t st);
cudaError_t launch_f64_to_f32(float* dst, const double* src, int n, cudaStream_t st);
cudaError_t launch_rows_to_f32(const double* src, int rows, int cols, float* dst, long long ldd,
                               __nv_bfloat16* dstb, long long lddb, float* stats, cudaStream_t st);
cudaError_t launch_f64_to_bf16_rows(const double* src, int rows, int cols, __nv_bfloat16* dst,
                                    long long ldd, cudaStream_t st,
                                    const int* host_bf16 = nullptr, const __nv_bfloat16* srcb = nullptr);
cudaError_t launch_image_patches(const double* img, int views, int H, int W, int C, int side, int P, double* patches,
                                 cudaStream_t st);
cudaError_t launch_f32_to_f64(const float* src, long long lds, int rows, int cols, double* dst,
                              cudaStream_t st);

// ------------------------------------------------------------------ errors

static thread_local std::string g_last_error;

struct EngineError : std::runtime_error {
    int code;
    EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PI0B_CUDA(x)                                                                          \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            throw EngineError(int(e_), std::string(#x) + ": " + cudaGetErrorString(e_));      \
    } while (0)

static int fail(const EngineError& e) {
    g_last_error = e.what();
    return e.code;
}

// ------------------------------------------------------------------ FNV-1a seeds

uint64_t seed_hash(uint64_t seed, const std::string& label, uint64_t a, uint64_t b) {
    uint64_t h = 0xcbf29ce484222325ULL;
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xff;
            h *= 0x100000001b3ULL;
        }
    };
    mix(seed);
    for (unsigned char c : label) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    mix(a);
    mix(b);
    return h;
}

// ------------------------------------------------------------------ tensor maps

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        PI0B_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess)
            throw EngineError(PI0B_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// bf16 [rows, cols] with row pitch `ld` elements, tiles of box_rows x 64, 128-B swizzle.
CUtensorMap make_tmap_bf16(const void* base, long long rows, long long cols, long long ld, int box_rows) {
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 2) % 16)
        throw EngineError(PI0B_E_INVALID, "TMA operand needs 16-byte aligned base and pitch");
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
    cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw EngineError(PI0B_E_INVALID, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

// [rows, cols] with row pitch `ld` elements, boxes of (128 B of columns) x box_rows, 128-B
// swizzle: 64 bf16 or 32 fp32 columns per box.
CUtensorMap make_tmap_2d(const void* base, bool f32, long long rows, long long cols, long long ld, int box_rows) {
    const int esz = f32 ? 4 : 2;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * esz) % 16)
        throw EngineError(PI0B_E_INVALID, "TMA operand needs 16-byte aligned base and pitch");
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld * esz)};
    cuuint32_t box[2] = {cuuint32_t(128 / esz), cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw EngineError(PI0B_E_INVALID, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

static int round_up(int x, int a) { return (x + a - 1) / a * a; }

// Split-K factor so that the grid approaches one wave of 148 SMs.
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

int gemm_max_active_clusters(int bn, int splits);
void gemm_set_pdl(bool on);

// K-split factor of a prefill GEMM: the splits of a tile run as one cluster (reduced over
// DSMEM), so all tiles x splits CTAs must be co-resident -- clusters are confined to a GPC,
// which the occupancy query accounts for.
static int choose_splits(int m_tiles, int n_tiles, int K, int bn, int num_sms) {
    const int ctas = m_tiles * n_tiles;
    const int kb = (K + 63) / 64;
    if (ctas * 2 > num_sms) return 1;
    // two-way splits measured best (scripts/gemm_sweep.sh): the DSMEM reduction moves (S-1)/S of
    // every tile and the cluster barriers grow with S
    int s = std::min({num_sms / ctas, kb / 2, kGemmMaxSplits, env_int("PI0B_MAX_SPLITS", 2)});
    for (; s > 1; --s) {
        const int per = (kb + s - 1) / s;
        if ((kb + per - 1) / per != s) continue;  // every split must own k-blocks
        if (gemm_max_active_clusters(bn, s) >= ctas) break;
    }
    return std::max(s, 1);
}

// The RoPE table the engine uploads: {cos, sin} of p * 10000^(-2j/d) interleaved, [positions][d/2][2],
// evaluated in fp64 with make_rope_table's operation order (proj/src/tensor.cpp:133-148) and
// rounded once to fp32 (pi0b_rope_table_host; bit-exact test against the reference in
// tests/test_capi.py).
static void rope_table_f32(int positions, int head_dim, float* out) {
    const int half = head_dim / 2;
    for (int p = 0; p < positions; ++p)
        for (int j = 0; j < half; ++j) {
            const double freq = std::pow(10000.0, -2.0 * double(j) / double(head_dim));
            const double ang = double(p) * freq;
            out[(size_t(p) * half + j) * 2 + 0] = float(std::cos(ang));
            out[(size_t(p) * half + j) * 2 + 1] = float(std::sin(ang));
        }
}

// ------------------------------------------------------------------ plan records

enum OpKind { kOpGemm, kOpAttn, kOpRowsF32, kOpF64Bf16, kOpF32F64, kOpMemset, kOpSkinny, kOpAeMega,
              kOpVeEpoch, kOpVePush, kOpVeWait };

// A checkpoint the megakernel leaves in a record buffer (record mode).
struct CkTag {
    std::string node;
    int inst;
    const void* ptr;
    int rows, cols;
    long long ld;
};

struct Op {
    OpKind kind;
    int part;  // 0 = prefix, 1 = action
    // gemm (bn = tile width; for kOpSkinny: cluster = K-split, n_packed = weight rows)
    int bn = 0;
    int cluster = 1, n_packed = 0;
    CUtensorMap ta, tb;
    GemmParams gp{};
    // attention
    int hd = 0;
    AttnParams ap{};
    FaMaps fm;
    // conversions
    const double* src64 = nullptr;
    int rows = 0, cols = 0;
    float* dst32 = nullptr;
    long long ld32 = 0;
    __nv_bfloat16* dstb = nullptr;
    long long ldb = 0;
    float* stats = nullptr;
    const float* src32 = nullptr;
    double* dst64 = nullptr;
    const int* skip = nullptr;  // kOpF64Bf16: device flag, nonzero = the rows came as bf16 in srcb
    const __nv_bfloat16* srcb = nullptr;
    void* mptr = nullptr;
    size_t mbytes = 0;
    // checkpoint tag (record mode)
    std::string node;
    int inst = -1;
    const void* ck_ptr = nullptr;
    int ck_rows = 0, ck_cols = 0;
    long long ck_ld = 0;
    int ck_bf16 = 0;
    std::vector<CkTag> extra_ck;
    // view-sharded VE: push own rows (segments: source, peer buffer, byte offset, bytes) to the
    // peers (or to shard 0 only) and signal step `ve_step`; or wait for `ve_step` from ve_mask
    int ve_step = 0, ve_nseg = 0;
    bool ve_root_only = false;
    unsigned ve_mask = 0;
    const void* ve_src[3] = {nullptr, nullptr, nullptr};
    int ve_buf[3] = {0, 0, 0};  // 0/1 qkv[parity], 2 x, 3 xb, 4 stats
    size_t ve_off[3] = {0, 0, 0}, ve_bytes[3] = {0, 0, 0};
    bool is_kernel() const { return kind != kOpMemset; }
};

struct NodeWeights {
    int k = 0, m = 0, instances = 0;
    long long ldk = 0;
    int perm = 0, rope_cols = 0;
    bool has_bias = false, has_table = false;
    std::vector<__nv_bfloat16*> w;
    std::vector<float*> b;
    float* table = nullptr;
    // what has been loaded (per instance; the bias table): launch() refuses to run on any
    // entry never written, as the reference throws NumericError("no weights for node ...")
    // (proj/src/evaluate.cpp:96-99) instead of reading zeroed / uninitialised memory
    std::vector<char> loaded;
    bool table_loaded = false;
};

struct Checkpoint {
    void* dev = nullptr;
    int rows = 0, cols = 0, bf16 = 0;
};

// Host side of the end-to-end call: the patches (2.4 MB of fp64 at 2 views) are converted to
// bf16 into pinned staging before their DMA, and one core (~10 GB/s of memory traffic) bounds
// that.  A few helper threads convert row pieces in parallel; the calling thread works too and
// issues each piece's DMA, in order, as soon as the piece is ready.
class StagingPool {
public:
    explicit StagingPool(int helpers) {
        for (int i = 0; i < helpers; ++i) th_.emplace_back([this] { loop(); });
    }
    ~StagingPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            ++gen_;
            gen_seen_.store(gen_, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // work(k) for k in [0, np) on the helpers and the calling thread; issue(k) on the calling
    // thread, in order, once work(k) has finished.
    template <class Work, class Issue>
    void run(size_t np, Work&& work, Issue&& issue) {
        if (th_.empty() || np < 2) {
            for (size_t k = 0; k < np; ++k) {
                work(k);
                issue(k);
            }
            return;
        }
        // helpers of the previous job must have left it before its fields change
        while (acks_.load(std::memory_order_acquire) != int(th_.size())) std::this_thread::yield();
        if (np > cap_) {
            done_.reset(new std::atomic<uint8_t>[np]);
            cap_ = np;
        }
        for (size_t k = 0; k < np; ++k) done_[k].store(0, std::memory_order_relaxed);
        work_ = std::function<void(size_t)>(work);
        np_ = np;
        next_.store(0, std::memory_order_relaxed);
        acks_.store(0, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> lk(m_);
            ++gen_;
            gen_seen_.store(gen_, std::memory_order_release);
        }
        cv_.notify_all();
        size_t issued = 0;
        try {
            while (issued < np) {
                if (done_[issued].load(std::memory_order_acquire)) {
                    issue(issued);
                    ++issued;
                    continue;
                }
                const size_t k = next_.fetch_add(1, std::memory_order_relaxed);
                if (k < np) do_piece(k);
            }
        } catch (...) {  // the caller's buffer must outlive every helper's work
            next_.store(np, std::memory_order_relaxed);
            while (acks_.load(std::memory_order_acquire) != int(th_.size())) std::this_thread::yield();
            throw;
        }
    }

private:
    void do_piece(size_t k) {
        work_(k);
        done_[k].store(1, std::memory_order_release);
    }
    void loop() {
        unsigned long long seen = 0;
        acks_.fetch_add(1, std::memory_order_release);  // idle
        for (;;) {
            // Optional spin before sleeping (PI0B_STAGING_SPIN_US): a condition-variable wake-up
            // costs tens of microseconds, which a back-to-back serving loop pays on every call.
            if (spin_us_ > 0) {
                const auto t0 = std::chrono::steady_clock::now();
                while (gen_seen_.load(std::memory_order_acquire) == seen &&
                       std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(spin_us_))
                    std::this_thread::yield();
            }
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            for (;;) {
                const size_t k = next_.fetch_add(1, std::memory_order_relaxed);
                if (k >= np_) break;
                do_piece(k);
            }
            acks_.fetch_add(1, std::memory_order_release);
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_;
    unsigned long long gen_ = 0;
    bool stop_ = false;
    std::atomic<size_t> next_{0};
    std::atomic<int> acks_{0};
    std::atomic<unsigned long long> gen_seen_{0};  // gen_, readable without the mutex (spinning helpers)
    const long spin_us_ = [] { const char* e = std::getenv("PI0B_STAGING_SPIN_US"); return e ? std::atol(e) : 0L; }();
    std::unique_ptr<std::atomic<uint8_t>[]> done_;
    size_t cap_ = 0;
    std::function<void(size_t)> work_;
    size_t np_ = 0;
};

static int staging_helpers() {
    const char* e = std::getenv("PI0B_STAGING_THREADS");
    const int hw = int(std::thread::hardware_concurrency());
    const int want = e ? std::atoi(e) : 3;
    return std::max(0, std::min(want, hw - 1));
}

class Engine {
public:
    // donor != nullptr: this engine reads the donor's weights (one weight arena for several
    // engines, e.g. the streaming runtime's double-buffered KV): only activations and the KV cache
    // are allocated; weights can be written only through the donor, which must outlive it.
    Engine(const pi0b_model_config& cfg, const pi0b_engine_options& opt, Engine* donor = nullptr);
    ~Engine();

    void gen_weights(uint64_t seed);
    void set_weight(const std::string& id, long long inst, const double* w, long long k, long long m,
                    const double* bias, long long blen);
    void set_bias_table(const std::string& id, const double* t, long long rows, long long m);
    void upload_inputs(const double* patches, const double* state, const double* noise,
                       const double* prompt, int which);
    // camera frames [views][height][width*3] (fp64) -> resize + img2col on the device into the
    // patch input (kernels_misc.cu image_patches_kernel), instead of host patches
    void upload_images(const double* images, int height, int width);
    void stage_patches_bf16(const double* patches);
    void launch(int part, cudaStream_t st);
    void fetch_actions(double* out);
    // asynchronous pieces for the streaming runtime (one outstanding operation per engine)
    void prefix_async(const double* patches, const double* prompt);
    void tick_async(const double* state, const double* noise);
    bool idle();                      // the last async operation completed
    const double* tick_result();      // host copy of the last tick's actions (after idle())
    void read_checkpoint(const std::string& id, long long inst, float* out, long long rows, long long cols);
    int kernel_count(int part) const;
    void prepare() {
        if (ae_mega_ && ae_tiles_dirty_) {
            for (const TiledW& tw : ae_tiled_) PI0B_CUDA(launch_tile_weight(tw.src, tw.rows, tw.k, tw.ldk, tw.dst, tw.order, stream_));
            PI0B_CUDA(cudaStreamSynchronize(stream_));
            ae_tiles_dirty_ = false;
        }
    }
    double time_node(const std::string& node, int reps, int* launches);
    std::string describe() const;
    void ae_trace(void* tasks, unsigned long long* stamps, long long cap, int* ctas, int* stride);
    cudaStream_t stream() const { return stream_; }
    bool weights_ready() const { return missing_weights().empty(); }
    std::string missing_weights() const;

private:
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        const size_t bytes = std::max<size_t>(256, (count * sizeof(T) + 255) / 256 * 256);
        PI0B_CUDA(cudaMalloc(&p, bytes));
        allocs_.push_back(p);
        return static_cast<T*>(p);
    }
    void validate_config();
    void alloc_weights();
    void alloc_activations();
    void build_plan();
    void add_gemm(int part, const std::string& node, int inst, const __nv_bfloat16* A, long long lda,
                  int M, const NodeWeights& W, int widx, int bn, GemmParams gp, bool allow_split = true,
                  int force_splits = 0);
    void add_skinny(int part, const std::string& node, int inst, const __nv_bfloat16* X, long long ldx, int M,
                    const NodeWeights& W, int widx, GemmParams gp);
    void add_attn(int part, const std::string& node, int inst, int hd, AttnParams ap);
    void tag(const std::string& node, int inst, const void* ptr, int rows, int cols, long long ld, int bf16);
    float* stats_slot(int part);
    void run_ops(int part, cudaStream_t st);
    void emit_op(const Op& op, cudaStream_t st);

    void capture(int part, int slot);

    pi0b_model_config c_;
    pi0b_engine_options o_;
    int num_sms_ = 148;
    int ae_ctas_ = 148;  // megakernel grid (PI0B_AE_CTAS: fewer leaves SMs to a concurrent prefix)
    cudaStream_t stream_ = nullptr;
    std::vector<void*> allocs_;
    std::map<std::string, NodeWeights> W_;
    bool weights_checked_ = false;

    // dims
    int T_ = 0, P_ = 0, L_ = 0, Lp_ = 0, S_ = 0, C_ = 0, FS_ = 0;  // Lp_: L_ rounded up to 32 rows
    int ve_w_ = 0, llm_w_ = 0, ae_w_ = 0, llm_q_ = 0, llm_kv_ = 0, ae_q_ = 0, ae_kv_ = 0;
    int patch_ld_ = 0, act_ld_ = 0, state_ld_ = 0, ve_mlp_ld_ = 0;

    // inputs (fp64 device staging + pinned host staging)
    double *d_patches_ = nullptr, *d_state_ = nullptr, *d_noise_ = nullptr, *d_prompt_ = nullptr,
           *d_out_ = nullptr;
    double *h_in_ = nullptr, *h_out_ = nullptr;
    std::unique_ptr<StagingPool> staging_{new StagingPool(staging_helpers())};
    // patches converted to bf16 on the host (pinned staging) + the device flag that tells the
    // graph's conversion op to skip; h_flag_[0] = 0, h_flag_[1] = 1 (pinned sources of the flag)
    uint16_t* h_pb_ = nullptr;
    int* h_flag_ = nullptr;
    int* d_patch_host_bf16_ = nullptr;
    __nv_bfloat16* d_pb_ = nullptr;  // the host-converted patches, packed
    cudaEvent_t done_ev_ = nullptr;               // streaming runtime: last async operation
    cudaEvent_t h2d_ev_ = nullptr;                // after the last H2D copy out of h_in_ / h_pb_
    double *h_img_ = nullptr, *d_img_ = nullptr;  // image front-end staging (grown on demand)
    size_t n_img_ = 0;
    size_t n_patches_ = 0, n_state_ = 0, n_noise_ = 0, n_prompt_ = 0, n_out_ = 0;

    // activations
    __nv_bfloat16 *patches_b_ = nullptr, *ve_hb_ = nullptr, *ve_qkv_ = nullptr, *ve_attn_ = nullptr,
                  *ve_mlp_ = nullptr;
    float* ve_h_ = nullptr;
    float* x_ = nullptr;
    __nv_bfloat16 *xb_ = nullptr, *llm_attn_ = nullptr, *llm_g_ = nullptr;
    std::vector<__nv_bfloat16*> kv_;  // per LLM layer [L, q+2kv]
    __nv_bfloat16 *state_b_ = nullptr, *ab_ = nullptr, *ap_b_ = nullptr, *yb_ = nullptr,
                  *aqkv_ = nullptr, *ao_ = nullptr, *ag_ = nullptr;
    float *st_ = nullptr, *y_ = nullptr, *a_ = nullptr;
    float* rope_cs_ = nullptr;
    float* stats_[2] = {nullptr, nullptr};
    int stats_rows_ = 0, stats_used_[2] = {0, 0}, stats_cap_[2] = {0, 0};

    std::vector<Op> ops_;
    cudaGraphExec_t graph_[3] = {nullptr, nullptr, nullptr};

    // action-expert megakernel (aemk.cu)
    bool ae_mega_ = true;
    AePlan ae_plan_;
    bool ae_cluster_ = true;
    AeParams ae_p_{};
    float* state32_ = nullptr;
    struct TiledW {
        const __nv_bfloat16* src;
        int rows, k;
        long long ldk;
        __nv_bfloat16* dst;
        int order;  // AeTileOrder
    };
    std::vector<TiledW> ae_tiled_;  // AE weights re-laid out as contiguous 8 KB tiles
    bool ae_tiles_dirty_ = true;
    void* ae_zero_ = nullptr;
    size_t ae_zero_bytes_ = 0;
    void build_ae_mega();
    std::map<std::pair<std::string, int>, Checkpoint> ck_;
    bool pdl_ = true;
    Engine* donor_ = nullptr;  // weights borrowed from this engine (nullptr: own arena)
    std::string ae_fallback_;  // why the per-node action expert runs instead of the megakernel
public:
    const std::string& ae_fallback() const { return ae_fallback_; }
    bool ae_megakernel() const { return ae_mega_; }
private:

    // view-sharded VE (pi0b_engine_options::ve_shards)
public:
    int ve_shards() const { return G_; }
    int ve_shard() const { return g_; }
    void ve_buffers(pi0b_ve_buffers* out) const;
    void set_ve_peers(const pi0b_ve_buffers* peers, int n);
private:
    int G_ = 1, g_ = 0, ve_r0_ = 0, ve_rows_ = 0;
    __nv_bfloat16* ve_qkv2_ = nullptr;  // second gathered q|k|v buffer (odd layers)
    unsigned* ve_sync_ = nullptr;
    std::vector<pi0b_ve_buffers> ve_peers_;
    bool ve_peers_set_ = false;
    void add_ve_push(int step, bool root_only, std::initializer_list<std::tuple<const void*, int, size_t, size_t>> segs);
    void add_ve_wait(int step, unsigned mask);
    __nv_bfloat16* ve_qkv_buf(int layer) const { return (G_ > 1 && (layer & 1)) ? ve_qkv2_ : ve_qkv_; }
};

// ------------------------------------------------------------------ construction

Engine::Engine(const pi0b_model_config& cfg, const pi0b_engine_options& opt, Engine* donor)
    : c_(cfg), o_(opt), donor_(donor) {
    if (donor_) {
        const pi0b_model_config& d = donor_->c_;
        if (std::memcmp(&d, &cfg, sizeof cfg) != 0 || donor_->o_.device != opt.device)
            throw EngineError(PI0B_E_INVALID, "shared weights: the donor engine has another config or device");
    }
    validate_config();
    PI0B_CUDA(cudaSetDevice(o_.device));
    cudaDeviceProp prop;
    PI0B_CUDA(cudaGetDeviceProperties(&prop, o_.device));
    if (prop.major != 10)
        throw EngineError(PI0B_E_UNSUPPORTED, "pi0b kernels are built for sm_100a (B200); found sm_" +
                                                  std::to_string(prop.major * 10 + prop.minor));
    num_sms_ = prop.multiProcessorCount;
    ae_ctas_ = num_sms_;
    if (const int want = env_int("PI0B_AE_CTAS", o_.ae_ctas); want > 0)
        ae_ctas_ = std::max(16, std::min(num_sms_, want & ~1));  // even: CTA pairs
    pdl_ = env_int("PI0B_PDL", 1) != 0;
    gemm_set_pdl(pdl_);
    fattn_set_pdl(pdl_);
    PI0B_CUDA(gemm_configure());
    PI0B_CUDA(fattn_configure());
    PI0B_CUDA(skinny_configure());
    PI0B_CUDA(aemk_configure());
    ae_mega_ = env_int("PI0B_AE_MEGA", 1) != 0;
    PI0B_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));

    alloc_weights();
    alloc_activations();
    build_plan();
    PI0B_CUDA(cudaStreamSynchronize(stream_));
}

Engine::~Engine() {
    for (auto& g : graph_)
        if (g) cudaGraphExecDestroy(g);
    for (auto& kv : ck_) cudaFree(kv.second.dev);
    for (void* p : allocs_) cudaFree(p);
    if (h_in_) cudaFreeHost(h_in_);
    if (h_img_) cudaFreeHost(h_img_);
    if (done_ev_) cudaEventDestroy(done_ev_);
    if (h2d_ev_) cudaEventDestroy(h2d_ev_);
    if (d_img_) cudaFree(d_img_);
    if (h_out_) cudaFreeHost(h_out_);
    if (h_pb_) cudaFreeHost(h_pb_);
    if (h_flag_) cudaFreeHost(h_flag_);
    if (stream_) cudaStreamDestroy(stream_);
}

void Engine::validate_config() {
    const auto& c = c_;
    auto need = [](bool ok, const std::string& what) {
        if (!ok) throw EngineError(PI0B_E_UNSUPPORTED, "unsupported pi0 config: " + what);
    };
    need(c.views >= 1 && c.tokens_per_view >= 1 && c.prompt_tokens >= 0, "token counts");
    need(c.chunk_len >= 1 && c.flow_steps >= 1, "chunk/flow steps");
    need(c.ve_width == c.ve_heads * c.ve_head_dim, "ve_width != ve_heads*ve_head_dim");
    need(c.ve_head_dim == 72 || c.ve_head_dim == 256, "ve_head_dim must be 72 or 256");
    need(c.llm_head_dim == 256 && c.ae_head_dim == 256, "llm/ae head_dim must be 256 (RoPE tile)");
    need(c.llm_kv_heads == c.ae_kv_heads && c.llm_kv_heads >= 1, "llm/ae kv_heads must match");
    need(c.llm_q_heads % c.llm_kv_heads == 0 && c.ae_q_heads % c.ae_kv_heads == 0, "GQA grouping");
    need(c.ae_q_heads * c.ae_head_dim > 0, "ae heads");
    need(c.llm_mlp % 128 == 0 && c.ae_mlp % 128 == 0, "mlp widths must be multiples of 128");
    for (int w : {c.ve_width, c.llm_width, c.ae_width})
        need(w % 8 == 0, "hidden widths must be multiples of 8");
    need(c.ve_layers >= 1 && c.llm_layers >= 2 && c.ae_layers >= 1, "layer counts");
}

void Engine::alloc_weights() {
    const auto& c = c_;
    if (donor_) {  // same config: the same node list, pointers into the donor's arena
        W_ = donor_->W_;
        return;
    }
    auto add = [&](const std::string& id, int k, int m, int inst, bool bias, int perm = kPermNone,
                   bool table = false, int rope_cols = 0) {
        NodeWeights nw;
        nw.k = k;
        nw.m = m;
        nw.instances = inst;
        nw.ldk = round_up(k, 8);
        nw.perm = perm;
        nw.rope_cols = rope_cols;
        nw.has_bias = bias;
        nw.has_table = table;
        const int rows = perm == kPermGate128 ? round_up(m, 256) : m;
        for (int i = 0; i < inst; ++i) {
            nw.w.push_back(alloc<__nv_bfloat16>(size_t(rows) * nw.ldk));
            PI0B_CUDA(cudaMemsetAsync(nw.w.back(), 0, size_t(rows) * nw.ldk * 2, stream_));
            if (bias) nw.b.push_back(alloc<float>(m));
        }
        if (table) nw.table = alloc<float>(size_t(c.flow_steps) * m);
        W_[id] = std::move(nw);
    };
    const int ve_w = c.ve_width, llm_w = c.llm_width, ae_w = c.ae_width;
    const int llm_qkv = (c.llm_q_heads + 2 * c.llm_kv_heads) * c.llm_head_dim;
    const int ae_q = c.ae_q_heads * c.ae_head_dim;
    const int ae_qkv = ae_q + 2 * c.ae_kv_heads * c.ae_head_dim;
    const int llm_q = c.llm_q_heads * c.llm_head_dim;
    // Weight-bearing nodes of build_pi0_graph (proj/src/builder.cpp:205-363) with their
    // binding: Shared 1, PerInstance repeat, PerLayer layer_count (evaluate.cpp:103-111).
    add("ve.embed", c.ve_patch_in, ve_w, 1, true);
    add("ve.qkv", ve_w, 3 * ve_w, c.ve_layers, true);
    add("ve.proj", ve_w, ve_w, c.ve_layers, true);
    add("ve.fc1", ve_w, c.ve_mlp, c.ve_layers, true);
    add("ve.fc2", c.ve_mlp, ve_w, c.ve_layers, true);
    add("llm.proj_in", ve_w, llm_w, 1, true);
    // llm.qkv on 128-wide tiles needs each tile to hold 64 columns of a head and their RoPE
    // partners: the kPermRope packing (PI0B_LLM_QKV_BN128=0: 256-wide head tiles, natural order)
    if (env_int("PI0B_LLM_QKV_BN128", 1))
        add("llm.qkv", llm_w, llm_qkv, c.llm_layers, false, kPermRope, false, llm_q + c.llm_kv_heads * c.llm_head_dim);
    else
        add("llm.qkv", llm_w, llm_qkv, c.llm_layers, false);
    add("llm.proj", llm_q, llm_w, c.llm_layers - 1, false);
    add("llm.ffn", llm_w, 2 * c.llm_mlp, c.llm_layers - 1, false, kPermGate128);
    add("llm.down", c.llm_mlp, llm_w, c.llm_layers - 1, false);
    add("ae.state_proj", c.ae_state_dim, ae_w, 1, true);
    add("ae.action_proj", c.ae_action_dim, ae_w, 1, false, kPermNone, true);
    add("ae.action_out", ae_w, ae_w, 1, true);
    add("ae.qkv", ae_w, ae_qkv, c.ae_layers, false, kPermRope, false, ae_q + c.ae_kv_heads * c.ae_head_dim);
    add("ae.proj", ae_q, ae_w, c.ae_layers, false);
    add("ae.ffn", ae_w, 2 * c.ae_mlp, c.ae_layers, false, kPermGate64);
    add("ae.down", c.ae_mlp, ae_w, c.ae_layers, false);
    add("ae.head", ae_w, c.ae_action_dim, 1, true);
}

void Engine::alloc_activations() {
    const auto& c = c_;
    T_ = c.views * c.tokens_per_view;
    P_ = c.prompt_tokens;
    L_ = T_ + P_;
    Lp_ = round_up(L_, 32);
    C_ = c.chunk_len;
    S_ = C_ + 1;
    FS_ = c.flow_steps;
    ve_w_ = c.ve_width;
    llm_w_ = c.llm_width;
    ae_w_ = c.ae_width;
    llm_q_ = c.llm_q_heads * c.llm_head_dim;
    llm_kv_ = c.llm_kv_heads * c.llm_head_dim;
    ae_q_ = c.ae_q_heads * c.ae_head_dim;
    ae_kv_ = c.ae_kv_heads * c.ae_head_dim;
    patch_ld_ = round_up(c.ve_patch_in, 8);
    ve_mlp_ld_ = round_up(c.ve_mlp, 8);
    act_ld_ = round_up(c.ae_action_dim, 8);
    state_ld_ = round_up(c.ae_state_dim, 8);

    n_patches_ = size_t(T_) * c.ve_patch_in;
    n_state_ = size_t(c.ae_state_dim);
    n_noise_ = size_t(C_) * c.ae_action_dim;
    n_prompt_ = size_t(P_) * llm_w_;
    n_out_ = n_noise_;
    d_patches_ = alloc<double>(n_patches_);
    d_state_ = alloc<double>(n_state_);
    d_noise_ = alloc<double>(n_noise_);
    d_prompt_ = alloc<double>(std::max<size_t>(1, n_prompt_));
    d_out_ = alloc<double>(n_out_);
    PI0B_CUDA(cudaMallocHost(&h_in_, (n_patches_ + n_state_ + n_noise_ + n_prompt_) * sizeof(double)));
    PI0B_CUDA(cudaMallocHost(&h_out_, n_out_ * sizeof(double)));
    PI0B_CUDA(cudaMallocHost(&h_pb_, n_patches_ * sizeof(uint16_t)));
    PI0B_CUDA(cudaMallocHost(&h_flag_, 2 * sizeof(int)));
    h_flag_[0] = 0;
    h_flag_[1] = 1;
    d_patch_host_bf16_ = alloc<int>(1);
    d_pb_ = alloc<__nv_bfloat16>(n_patches_);
    PI0B_CUDA(cudaMemsetAsync(d_patch_host_bf16_, 0, sizeof(int), stream_));

    patches_b_ = alloc<__nv_bfloat16>(size_t(T_) * patch_ld_);
    PI0B_CUDA(cudaMemsetAsync(patches_b_, 0, size_t(T_) * patch_ld_ * 2, stream_));
    ve_h_ = alloc<float>(size_t(T_) * ve_w_);
    ve_hb_ = alloc<__nv_bfloat16>(size_t(T_) * ve_w_);
    ve_qkv_ = alloc<__nv_bfloat16>(size_t(T_) * 3 * ve_w_);
    G_ = std::max(1, o_.ve_shards);
    g_ = G_ > 1 ? o_.ve_shard : 0;
    if (G_ > kVeMaxShards || g_ < 0 || g_ >= G_ || c.views % G_)
        throw EngineError(PI0B_E_UNSUPPORTED, "ve_shards must divide views (<= 8 shards), 0 <= ve_shard < ve_shards");
    ve_rows_ = T_ / G_;
    ve_r0_ = g_ * ve_rows_;
    if (G_ > 1) {
        ve_qkv2_ = alloc<__nv_bfloat16>(size_t(T_) * 3 * ve_w_);
        ve_sync_ = alloc<unsigned>(kVeSyncWords);
        PI0B_CUDA(cudaMemsetAsync(ve_sync_, 0, kVeSyncWords * sizeof(unsigned), stream_));
        ve_peers_.resize(size_t(G_));
    }
    ve_attn_ = alloc<__nv_bfloat16>(size_t(T_) * ve_w_);
    ve_mlp_ = alloc<__nv_bfloat16>(size_t(T_) * ve_mlp_ld_);
    PI0B_CUDA(cudaMemsetAsync(ve_mlp_, 0, size_t(T_) * ve_mlp_ld_ * 2, stream_));
    // The prefix is processed in Lp_ = round_up(L_, 32) rows (any prompt length the reference
    // accepts, proj/include/rtvla/graph.hpp:156-158): rows [L_, Lp_) start as zeros, stay finite
    // and row-local through every GEMM, and are masked out of every attention as keys.
    x_ = alloc<float>(size_t(Lp_) * llm_w_);
    xb_ = alloc<__nv_bfloat16>(size_t(Lp_) * llm_w_);
    PI0B_CUDA(cudaMemsetAsync(x_, 0, size_t(Lp_) * llm_w_ * 4, stream_));
    PI0B_CUDA(cudaMemsetAsync(xb_, 0, size_t(Lp_) * llm_w_ * 2, stream_));
    llm_attn_ = alloc<__nv_bfloat16>(size_t(Lp_) * llm_q_);
    llm_g_ = alloc<__nv_bfloat16>(size_t(Lp_) * c.llm_mlp);
    for (int l = 0; l < c.llm_layers; ++l) {
        kv_.push_back(alloc<__nv_bfloat16>(size_t(Lp_) * (llm_q_ + 2 * llm_kv_)));
        PI0B_CUDA(cudaMemsetAsync(kv_.back(), 0, size_t(Lp_) * (llm_q_ + 2 * llm_kv_) * 2, stream_));
    }
    state_b_ = alloc<__nv_bfloat16>(size_t(state_ld_));
    PI0B_CUDA(cudaMemsetAsync(state_b_, 0, size_t(state_ld_) * 2, stream_));
    ab_ = alloc<__nv_bfloat16>(size_t(C_) * act_ld_);
    PI0B_CUDA(cudaMemsetAsync(ab_, 0, size_t(C_) * act_ld_ * 2, stream_));
    a_ = alloc<float>(size_t(C_) * act_ld_);
    ap_b_ = alloc<__nv_bfloat16>(size_t(C_) * ae_w_);
    st_ = alloc<float>(size_t(ae_w_));
    y_ = alloc<float>(size_t(S_) * ae_w_);
    yb_ = alloc<__nv_bfloat16>(size_t(S_) * ae_w_);
    aqkv_ = alloc<__nv_bfloat16>(size_t(S_) * (ae_q_ + 2 * ae_kv_));
    ao_ = alloc<__nv_bfloat16>(size_t(S_) * ae_q_);
    ag_ = alloc<__nv_bfloat16>(size_t(S_) * c.ae_mlp);

    // RoPE table: cos/sin of p * 10000^(-2j/256), evaluated in fp64 as make_rope_table
    // (proj/src/tensor.cpp:133-148) and rounded to fp32. Positions [0, L+S).
    const int npos = Lp_ + S_;
    std::vector<float> cs(size_t(npos) * 128 * 2);
    rope_table_f32(npos, 256, cs.data());
    rope_cs_ = alloc<float>(cs.size());
    PI0B_CUDA(cudaMemcpyAsync(rope_cs_, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, stream_));
    PI0B_CUDA(cudaStreamSynchronize(stream_));

    // Row-stat slots: one per residual-stream producer instance, zeroed per replay.
    stats_rows_ = round_up(std::max(Lp_, S_), 64);
    stats_cap_[0] = 2 + 2 * c.ve_layers + 2 * c.llm_layers;
    stats_cap_[1] = FS_ * (2 + 2 * c.ae_layers) + 2;
    for (int p = 0; p < 2; ++p) stats_[p] = alloc<float>(size_t(stats_cap_[p]) * stats_rows_);
}

void Engine::add_ve_push(int step, bool root_only,
                         std::initializer_list<std::tuple<const void*, int, size_t, size_t>> segs) {
    Op op;
    op.kind = kOpVePush;
    op.part = 0;
    op.ve_step = step;
    op.ve_root_only = root_only;
    for (const auto& sg : segs) {
        if (op.ve_nseg == 3) throw EngineError(PI0B_E_STATE, "ve push: too many segments");
        if ((std::get<3>(sg) % 16) || (std::get<2>(sg) % 16) || (reinterpret_cast<uintptr_t>(std::get<0>(sg)) % 16))
            throw EngineError(PI0B_E_UNSUPPORTED, "ve push: rows must be 16-byte aligned");
        op.ve_src[op.ve_nseg] = std::get<0>(sg);
        op.ve_buf[op.ve_nseg] = std::get<1>(sg);
        op.ve_off[op.ve_nseg] = std::get<2>(sg);
        op.ve_bytes[op.ve_nseg] = std::get<3>(sg);
        ++op.ve_nseg;
    }
    ops_.push_back(op);
}

void Engine::add_ve_wait(int step, unsigned mask) {
    Op op;
    op.kind = kOpVeWait;
    op.part = 0;
    op.ve_step = step;
    op.ve_mask = mask;
    ops_.push_back(op);
}

void Engine::ve_buffers(pi0b_ve_buffers* out) const {
    if (G_ < 2) throw EngineError(PI0B_E_STATE, "engine is not view-sharded (ve_shards < 2)");
    out->qkv[0] = ve_qkv_;
    out->qkv[1] = ve_qkv2_;
    out->x = x_;
    out->xb = xb_;
    out->stats = stats_[0];
    out->sync = ve_sync_;
}

void Engine::set_ve_peers(const pi0b_ve_buffers* peers, int n) {
    if (G_ < 2) throw EngineError(PI0B_E_STATE, "engine is not view-sharded (ve_shards < 2)");
    if (!peers || n != G_) throw EngineError(PI0B_E_INVALID, "set_ve_peers: one entry per shard");
    for (int p = 0; p < G_; ++p) {
        if (p == g_) continue;
        const pi0b_ve_buffers& b = peers[p];
        if (!b.qkv[0] || !b.qkv[1] || !b.sync || (p == 0 && (!b.x || !b.xb || !b.stats)))
            throw EngineError(PI0B_E_INVALID, "set_ve_peers: missing peer buffer");
        ve_peers_[size_t(p)] = b;
    }
    for (auto& g : graph_)  // captured with the old peers
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
    ve_peers_set_ = true;
}

float* Engine::stats_slot(int part) {
    if (stats_used_[part] >= stats_cap_[part]) throw EngineError(PI0B_E_STATE, "stats slots exhausted");
    return stats_[part] + size_t(stats_used_[part]++) * stats_rows_;
}

void Engine::tag(const std::string& node, int inst, const void* ptr, int rows, int cols, long long ld,
                 int bf16) {
    Op& op = ops_.back();
    op.node = node;
    op.inst = inst;
    op.ck_ptr = ptr;
    op.ck_rows = rows;
    op.ck_cols = cols;
    op.ck_ld = ld;
    op.ck_bf16 = bf16;
}

void Engine::add_gemm(int part, const std::string& node, int inst, const __nv_bfloat16* A,
                      long long lda, int M, const NodeWeights& W, int widx, int bn, GemmParams gp,
                      bool allow_split, int force_splits) {
    // Tuning overrides (sweeps): PI0B_BN_<NODE> / PI0B_SPLIT_<NODE>, NODE = id with '.' -> '_',
    // upper case (e.g. PI0B_BN_VE_PROJ=64).
    std::string key = node;
    for (char& ch : key) ch = ch == '.' ? '_' : char(std::toupper(static_cast<unsigned char>(ch)));
    const int bn_env = env_int(("PI0B_BN_" + key).c_str(), 0);
    if ((bn_env == 64 || bn_env == 128 || bn_env == 256) && !(gp.flags & kFlagRope) && gp.mode != kModeGate) bn = bn_env;
    const int split_env = env_int(("PI0B_SPLIT_" + key).c_str(), 0);
    Op op;
    op.kind = kOpGemm;
    op.part = part;
    op.bn = bn;
    const int N = gp.N;
    const int K = W.k;
    const __nv_bfloat16* wptr = W.w.at(size_t(widx));
    op.ta = make_tmap_bf16(A, M, K, lda, 128);
    op.tb = make_tmap_bf16(wptr, N, K, W.ldk, bn);
    gp.M = M;
    gp.K = K;
    const int m_tiles = (M + 127) / 128, n_tiles = (N + bn - 1) / bn;
    const int kb = (K + 63) / 64;
    int splits = allow_split ? choose_splits(m_tiles, n_tiles, K, bn, num_sms_) : 1;
    if (force_splits > 0) splits = std::min({force_splits, kb, kGemmMaxSplits});
    if (split_env > 0) splits = std::min({split_env, kb, kGemmMaxSplits});
    gp.kb_per_split = (kb + splits - 1) / splits;
    gp.splits = (kb + gp.kb_per_split - 1) / gp.kb_per_split;
    // More tiles than SMs and no split-K: one persistent CTA per SM with the accumulator
    // double-buffered in TMEM (epilogue of tile j overlapped with the mainloop of tile j + 1).
    // PI0B_PERSIST_<NODE>=0/1 overrides.
    const int persist_env = env_int(("PI0B_PERSIST_" + key).c_str(), -1);
    // 256 x 256 tiles for the large unsplit bn = 256 GEMMs: a CTA pair on one tcgen05
    // cta_group::2 MMA (PI0B_CG[_<NODE>]: 0 off, 1 auto, 2 force), or else two m-tiles per CTA
    // (PI0B_MT[_<NODE>], default off: it halves L2 traffic but not the shared-memory traffic
    // that bounds a single-CTA MMA).
    {
        const bool can = bn == 256 && gp.splits == 1 && M > 128 &&
                         (gp.mode == kModeGate || gp.mode == kModeBf16 || gp.mode == kModeResid);
        const int cg_env = env_int(("PI0B_CG_" + key).c_str(), -1), cg_all = env_int("PI0B_CG", 1);
        const bool want_cg = cg_env >= 0 ? cg_env > 0 : (cg_all == 2 || (cg_all == 1 && m_tiles * n_tiles > num_sms_));
        gp.cg = can && want_cg ? 2 : 1;
        const int mt_env = env_int(("PI0B_MT_" + key).c_str(), -1), mt_all = env_int("PI0B_MT", 0);
        const bool want = mt_env >= 0 ? mt_env > 0 : (mt_all == 2 || (mt_all == 1 && m_tiles * n_tiles > num_sms_));
        gp.mt = can && want && gp.cg == 1 ? 2 : 1;
        if (gp.cg == 2) op.tb = make_tmap_bf16(wptr, N, K, W.ldk, bn / 2);
    }
    // PI0B_PERSIST: 0 off, 1 (default) when tiles > SMs, 2 every unsplit GEMM (tests).
    const int persist_all = env_int("PI0B_PERSIST", 1);
    const bool auto_p = persist_all == 2 || (persist_all == 1 && m_tiles * n_tiles > num_sms_);
    gp.persist = gp.splits == 1 && (persist_env >= 0 ? persist_env > 0 : auto_p) ? 1 : 0;
    op.gp = gp;
    ops_.push_back(op);
}

// Action-expert GEMM on the swap-AB skinny kernel: K split over a cluster of up to 8 CTAs so
// that tiles x cluster approaches one wave while every CTA keeps >= 2 k-blocks.
void Engine::add_skinny(int part, const std::string& node, int inst, const __nv_bfloat16* X, long long ldx, int M,
                        const NodeWeights& W, int widx, GemmParams gp) {
    Op op;
    op.kind = kOpSkinny;
    op.part = part;
    const int n_packed = W.perm == kPermGate64 ? W.m : gp.N;
    op.n_packed = n_packed;
    op.tb = make_tmap_bf16(X, M, W.k, ldx, 64);
    op.ta = make_tmap_bf16(W.w.at(size_t(widx)), n_packed, W.k, W.ldk, 128);
    gp.M = M;
    gp.K = W.k;
    gp.splits = 1;
    gp.kb_per_split = (W.k + 63) / 64;
    if (W.perm == kPermRope) gp.rope_cols = W.rope_cols;
    const int tiles = skinny_tiles(n_packed), kb = (W.k + 63) / 64;
    int cl = 1;
    while (cl < 8 && tiles * cl * 2 <= num_sms_ && kb >= cl * 4) cl *= 2;
    op.cluster = std::min(cl, env_int("PI0B_MAX_CLUSTER", 8));
    op.gp = gp;
    ops_.push_back(op);
}

void Engine::add_attn(int part, const std::string& node, int inst, int hd, AttnParams ap) {
    Op op;
    op.kind = kOpAttn;
    op.part = part;
    op.hd = hd;
    // Key splits (a (1, S, 1) cluster per q tile, DSMEM combine): as many as keep the grid
    // within one wave, at least two 64-key tiles per split.  PI0B_ATTN_SPLITS[_<NODE>] override.
    {
        std::string key = node;
        for (char& ch : key) ch = ch == '.' ? '_' : char(std::toupper(static_cast<unsigned char>(ch)));
        const int base = ((ap.heads / ap.kv_heads) * ap.q_rows + 127) / 128 * ap.kv_heads;
        const int tiles = (ap.rows0 + ap.rows1 + 63) / 64;
        // Measured in graph replays (scripts/ab_env.sh, scripts/attn_split_sweep.sh): llm.attn (d 256)
        // at S = 4 when the key tiles split evenly four ways (2 views, no prompt: -5 us per
        // inference), S = 2 for other prefixes of >= 8 key tiles (2v + 17/64-token prompts, 3 views:
        // -5..-18 us; S = 4 there is 150-170 us slower), unsplit below 8 tiles (1 view) and for
        // d 72 (ve.attn); always within one wave of CTAs.
        int S = 1;
        if (node == "llm.attn" && tiles >= 8) {
            if (tiles % 4 == 0 && base * 4 <= num_sms_) S = 4;
            else if (base * 2 <= num_sms_) S = 2;
        }
        S = env_int(("PI0B_ATTN_SPLITS_" + key).c_str(), env_int("PI0B_ATTN_SPLITS", S));
        ap.kv_splits = (S == 2 || S == 4 || S == 8) ? S : 1;
    }
    ap.kv_per_split = ap.rows0 + ap.rows1;
    ap.scale_log2 = float(1.4426950408889634 / std::sqrt(double(hd)));
    if ((ap.rows1 > 0 && (ap.rows0 % 32)) || (ap.rows1 % 32) || (ap.q_rows % 32))
        throw EngineError(PI0B_E_UNSUPPORTED, "attention: two key segments need 32-row multiples");
    if (ap.kv_splits > 1) ap.ws = alloc<uint8_t>(size_t(attention_ws_bytes(ap, hd)));
    op.fm = make_fattn_maps(ap, hd);
    op.ap = ap;
    ops_.push_back(op);
    (void)node;
    (void)inst;
}

void Engine::build_plan() {
    const auto& c = c_;
    auto& Wv = W_;
    const int ve_qkv_n = 3 * ve_w_;
    const int llm_qkv_n = llm_q_ + 2 * llm_kv_;
    const int ae_qkv_n = ae_q_ + 2 * ae_kv_;

    // ================================================================ prefix (part 0)
    {
        Op m;
        m.kind = kOpMemset;
        m.part = 0;
        m.mptr = stats_[0];
        m.mbytes = size_t(stats_cap_[0]) * stats_rows_ * 4;
        ops_.push_back(m);
        Op cv;
        cv.kind = kOpF64Bf16;
        cv.part = 0;
        cv.src64 = d_patches_;
        cv.rows = T_;
        cv.cols = c.ve_patch_in;
        cv.dstb = patches_b_;
        cv.ldb = patch_ld_;
        cv.skip = d_patch_host_bf16_;
        cv.srcb = d_pb_;
        ops_.push_back(cv);
    }
    // --- vision encoder (proj/src/builder.cpp:205-240).  View-sharded (G_ > 1): this engine runs
    // the rows [r0, r0 + Tg) of its own views; the joint attention reads every shard's rows,
    // all-gathered after each ve.qkv (double-buffered by layer parity: a shard can only be one
    // layer ahead of a peer, because it waits for that peer's rows of the next layer).
    const int r0 = ve_r0_, Tg = ve_rows_;
    if (G_ > 1) {
        Op e;
        e.kind = kOpVeEpoch;
        e.part = 0;
        ops_.insert(ops_.begin(), e);
    }
    float* st = stats_slot(0);
    {
        GemmParams g{};
        g.N = ve_w_;
        g.mode = kModeF32Store;
        g.flags = kFlagBias;
        g.bias = Wv["ve.embed"].b[0];
        g.out = ve_h_ + size_t(r0) * ve_w_;
        g.ldo = ve_w_;
        g.outb = ve_hb_ + size_t(r0) * ve_w_;
        g.ldob = ve_w_;
        g.out_stats = st + r0;
        add_gemm(0, "ve.embed", 0, patches_b_ + size_t(r0) * patch_ld_, patch_ld_, Tg, Wv["ve.embed"], 0, 64, g);  // bn 64: 11.8 -> 8.9 us (scripts/proj_in_probe.sh)
        tag("ve.embed", 0, ve_h_, T_, ve_w_, ve_w_, 0);
    }
    const float inv_ve = 1.0f / float(ve_w_);
    for (int i = 0; i < c.ve_layers; ++i) {
        {   // ve.ln1 + ve.qkv: (h W) * rms(h) + b
            GemmParams g{};
            g.N = ve_qkv_n;
            g.mode = kModeBf16;
            g.flags = kFlagRowScale | kFlagBias;
            g.row_stats = st + r0;
            g.inv_width = inv_ve;
            g.eps = 1e-6f;
            g.bias = Wv["ve.qkv"].b[i];
            g.out = ve_qkv_buf(i) + size_t(r0) * ve_qkv_n;
            g.ldo = ve_qkv_n;
            add_gemm(0, "ve.qkv", i, ve_hb_ + size_t(r0) * ve_w_, ve_w_, Tg, Wv["ve.qkv"], i, 128, g);
            tag("ve.qkv", i, ve_qkv_buf(i), T_, ve_qkv_n, ve_qkv_n, 1);
        }
        if (G_ > 1) {   // all-gather this layer's q|k|v rows (own rows -> every peer), then wait
            const size_t row_bytes = size_t(ve_qkv_n) * 2;
            add_ve_push(i, false, {std::make_tuple((const void*)(ve_qkv_buf(i) + size_t(r0) * ve_qkv_n), i & 1,
                                                   size_t(r0) * row_bytes, size_t(Tg) * row_bytes)});
            add_ve_wait(i, ((1u << G_) - 1u) & ~(1u << g_));
        }
        {   // ve.attn: joint over all views' tokens, no mask
            AttnParams a{};
            a.q = ve_qkv_buf(i) + size_t(r0) * ve_qkv_n;
            a.ldq = ve_qkv_n;
            a.q_rows = Tg;
            a.heads = c.ve_heads;
            a.kv_heads = c.ve_heads;
            a.k0 = ve_qkv_buf(i) + ve_w_;
            a.v0 = ve_qkv_buf(i) + 2 * ve_w_;
            a.ld0 = ve_qkv_n;
            a.rows0 = T_;
            a.out = ve_attn_ + size_t(r0) * ve_w_;
            a.ldo = ve_w_;
            add_attn(0, "ve.attn", i, c.ve_head_dim, a);
            tag("ve.attn", i, ve_attn_, T_, ve_w_, ve_w_, 1);
        }
        float* st2 = stats_slot(0);
        {   // ve.proj: h += attn W + b
            GemmParams g{};
            g.N = ve_w_;
            g.mode = kModeResid;
            g.flags = kFlagBias;
            g.bias = Wv["ve.proj"].b[i];
            g.resid_scale = 1.0f;
            g.out = ve_h_ + size_t(r0) * ve_w_;
            g.ldo = ve_w_;
            g.outb = ve_hb_ + size_t(r0) * ve_w_;
            g.ldob = ve_w_;
            g.out_stats = st2 + r0;
            // unsplit (72 CTAs at 2 views): the split-K exchange costs more than the 18 k-blocks it
            // halves (graph replay -8 us against 2-way split-K, scripts/ab_env.sh)
            add_gemm(0, "ve.proj", i, ve_attn_ + size_t(r0) * ve_w_, ve_w_, Tg, Wv["ve.proj"], i, 64, g, false);
            tag("ve.proj", i, ve_h_, T_, ve_w_, ve_w_, 0);
        }
        {   // ve.ln2 + ve.fc1: gelu((p W) * rms(p) + b)
            GemmParams g{};
            g.N = c.ve_mlp;
            g.mode = kModeBf16;
            g.flags = kFlagRowScale | kFlagBias | kFlagGelu;
            g.row_stats = st2 + r0;
            g.inv_width = inv_ve;
            g.eps = 1e-6f;
            g.bias = Wv["ve.fc1"].b[i];
            g.out = ve_mlp_ + size_t(r0) * ve_mlp_ld_;
            g.ldo = ve_mlp_ld_;
            add_gemm(0, "ve.fc1", i, ve_hb_ + size_t(r0) * ve_w_, ve_w_, Tg, Wv["ve.fc1"], i, 128, g);
            tag("ve.fc1", i, ve_mlp_, T_, c.ve_mlp, ve_mlp_ld_, 1);
        }
        st = stats_slot(0);
        {   // ve.fc2: h += mlp W + b
            GemmParams g{};
            g.N = ve_w_;
            g.mode = kModeResid;
            g.flags = kFlagBias;
            g.bias = Wv["ve.fc2"].b[i];
            g.resid_scale = 1.0f;
            g.out = ve_h_ + size_t(r0) * ve_w_;
            g.ldo = ve_w_;
            g.outb = ve_hb_ + size_t(r0) * ve_w_;
            g.ldob = ve_w_;
            g.out_stats = st + r0;
            // bn 64 split 2 while that fits one wave (1-2 views: 72 / 144 CTAs), else bn 128 split 2
            // (3 views: 108 CTAs of N = 128 MMAs, -74 us per inference against bn 64 unsplit)
            const int fmt = (Tg + 127) / 128;
            const bool f64 = fmt * ((ve_w_ + 63) / 64) * 2 <= num_sms_;
            add_gemm(0, "ve.fc2", i, ve_mlp_ + size_t(r0) * ve_mlp_ld_, ve_mlp_ld_, Tg, Wv["ve.fc2"], i, f64 ? 64 : 128, g,
                     true, f64 ? 0 : 2);
            tag("ve.fc2", i, ve_h_, T_, ve_w_, ve_w_, 0);
        }
    }
    // --- language model (proj/src/builder.cpp:242-289)
    float* xs = stats_slot(0);
    {   // ve.ln_out + llm.proj_in -> x rows [0, T)
        GemmParams g{};
        g.N = llm_w_;
        g.mode = kModeF32Store;
        g.flags = kFlagRowScale | kFlagBias;
        g.row_stats = st + r0;
        g.inv_width = inv_ve;
        g.eps = 1e-6f;
        g.bias = Wv["llm.proj_in"].b[0];
        g.out = x_ + size_t(r0) * llm_w_;
        g.ldo = llm_w_;
        g.outb = xb_ + size_t(r0) * llm_w_;
        g.ldob = llm_w_;
        g.out_stats = xs + r0;
        add_gemm(0, "llm.proj_in", 0, ve_hb_ + size_t(r0) * ve_w_, ve_w_, Tg, Wv["llm.proj_in"], 0, 64, g);  // bn 64: 18.1 -> 9.2 us
        tag("llm.proj_in", 0, x_, T_, llm_w_, llm_w_, 0);
    }
    if (G_ > 1) {
        // gather the llm.proj_in rows (fp32, bf16 shadow, row sums of squares) into shard 0, then
        // an end-of-VE barrier: shard 0 releases every peer once all rows have arrived, so no
        // shard starts the next inference's layer-0 exchange while a peer still reads layer 26
        const int kGather = c.ve_layers, kRelease = c.ve_layers + 1;
        const unsigned peers = ((1u << G_) - 1u) & ~1u;
        if (g_ != 0) {
            add_ve_push(kGather, true,
                        {std::make_tuple((const void*)(x_ + size_t(r0) * llm_w_), 2, size_t(r0) * llm_w_ * 4, size_t(Tg) * llm_w_ * 4),
                         std::make_tuple((const void*)(xb_ + size_t(r0) * llm_w_), 3, size_t(r0) * llm_w_ * 2, size_t(Tg) * llm_w_ * 2),
                         std::make_tuple((const void*)(xs + r0), 4, size_t((xs + r0) - stats_[0]) * 4, size_t(Tg) * 4)});
            add_ve_wait(kRelease, 1u);
            // shards other than 0 serve run_prefix only: no LLM, no action expert
            return;
        }
        add_ve_wait(kGather, peers);
        add_ve_push(kRelease, false, {});
    }
    if (Lp_ > L_) {  // padding rows of the prefix start each inference as zeros (engine.cu alloc_activations)
        Op m;
        m.kind = kOpMemset;
        m.part = 0;
        m.mptr = x_ + size_t(L_) * llm_w_;
        m.mbytes = size_t(Lp_ - L_) * llm_w_ * 4;
        ops_.push_back(m);
        m.mptr = xb_ + size_t(L_) * llm_w_;
        m.mbytes = size_t(Lp_ - L_) * llm_w_ * 2;
        ops_.push_back(m);
    }
    if (P_ > 0) {   // llm.tokens = concat_rows(proj_in, prompt)
        Op cv;
        cv.kind = kOpRowsF32;
        cv.part = 0;
        cv.src64 = d_prompt_;
        cv.rows = P_;
        cv.cols = llm_w_;
        cv.dst32 = x_ + size_t(T_) * llm_w_;
        cv.ld32 = llm_w_;
        cv.dstb = xb_ + size_t(T_) * llm_w_;
        cv.ldb = llm_w_;
        cv.stats = xs + T_;
        ops_.push_back(cv);
        tag("llm.tokens", 0, x_, L_, llm_w_, llm_w_, 0);
    }
    const float inv_llm = 1.0f / float(llm_w_);
    const int NL = c.llm_layers;
    for (int l = 0; l < NL; ++l) {
        {   // llm.ln1 + llm.qkv, RoPE at positions 0..L-1 -> KV cache layer l
            GemmParams g{};
            g.mode = kModeBf16;
            g.flags = kFlagRowScale | kFlagRope;
            g.row_stats = xs;
            g.inv_width = inv_llm;
            g.eps = 1e-6f;
            g.rope_cs = rope_cs_;
            g.rope_pos0 = 0;
            g.ldo = llm_qkv_n;
            const bool bn128 = Wv["llm.qkv"].perm == kPermRope;
            const int qkv_bn = bn128 ? 128 : 256;
            if (bn128) g.flags |= kFlagRopePacked;
            if (l < NL - 1) {
                g.N = llm_qkv_n;
                g.rope_cols = llm_q_ + llm_kv_;
                g.out = kv_[l];
                add_gemm(0, "llm.qkv", l, xb_, llm_w_, Lp_, Wv["llm.qkv"], l, qkv_bn, g);
            } else {
                // Last layer: only K/V feed the action expert; its Q is dead.
                NodeWeights sub = Wv["llm.qkv"];
                sub.w[l] = Wv["llm.qkv"].w[l] + size_t(llm_q_) * sub.ldk;
                g.N = 2 * llm_kv_;
                g.rope_cols = llm_kv_;
                g.out = kv_[l] + llm_q_;
                add_gemm(0, "llm.qkv", l, xb_, llm_w_, Lp_, sub, l, qkv_bn, g);
            }
            tag("llm.qkv", l, kv_[l], L_, llm_qkv_n, llm_qkv_n, 1);
        }
        if (l == NL - 1) break;
        {
            AttnParams a{};
            a.q = kv_[l];
            a.ldq = llm_qkv_n;
            a.q_rows = Lp_;
            a.heads = c.llm_q_heads;
            a.kv_heads = c.llm_kv_heads;
            a.k0 = kv_[l] + llm_q_;
            a.v0 = kv_[l] + llm_q_ + llm_kv_;
            a.ld0 = llm_qkv_n;
            a.rows0 = L_;
            a.out = llm_attn_;
            a.ldo = llm_q_;
            add_attn(0, "llm.attn", l, 256, a);
            tag("llm.attn", l, llm_attn_, L_, llm_q_, llm_q_, 1);
        }
        float* ps = stats_slot(0);
        {
            GemmParams g{};
            g.N = llm_w_;
            g.mode = kModeResid;
            g.resid_scale = 1.0f;
            g.out = x_;
            g.ldo = llm_w_;
            g.outb = xb_;
            g.ldob = llm_w_;
            g.out_stats = ps;
            // bn 64 while its tiles fit one wave (2 views: 128 CTAs), else bn 128 (a 2v + 17-token
            // prefix: 160 -> 80 tiles, -55 us per inference)
            const int pbn = ((Lp_ + 127) / 128) * (llm_w_ / 64) > num_sms_ ? 128 : 64;
            add_gemm(0, "llm.proj", l, llm_attn_, llm_q_, Lp_, Wv["llm.proj"], l, pbn, g);
            tag("llm.proj", l, x_, L_, llm_w_, llm_w_, 0);
        }
        {   // llm.ln2 + fused gated FFN: up * gelu(gate)
            GemmParams g{};
            g.N = 2 * c.llm_mlp;
            g.mode = kModeGate;
            g.flags = kFlagRowScale;
            g.row_stats = ps;
            g.inv_width = inv_llm;
            g.eps = 1e-6f;
            g.out = llm_g_;
            g.ldo = c.llm_mlp;
            add_gemm(0, "llm.ffn", l, xb_, llm_w_, Lp_, Wv["llm.ffn"], l, 256, g);
            tag("llm.ffn", l, llm_g_, L_, c.llm_mlp, c.llm_mlp, 1);
        }
        xs = stats_slot(0);
        {
            GemmParams g{};
            g.N = llm_w_;
            g.mode = kModeResid;
            g.resid_scale = 1.0f;
            g.out = x_;
            g.ldo = llm_w_;
            g.outb = xb_;
            g.ldob = llm_w_;
            g.out_stats = xs;
            // Tile width and split-K from the prefix's m-tiles (measured, scripts/down_sweep.sh:
            // 2 m-tiles -> bn 128 x 4 splits, 4 -> 128 x 2, 5 -> 256 x 3, 6 / 7 -> 256 x 2): the
            // widest split keeping <= 128 CTAs, bn 128 while that split is >= 2, else bn 256.
            const int dmt = (Lp_ + 127) / 128;
            int dbn = 128, dsp = std::min(4, 128 / (dmt * 16));
            if (dsp < 2) {
                dbn = 256;
                dsp = std::max(1, std::min(3, 128 / (dmt * 8)));
            }
            add_gemm(0, "llm.down", l, llm_g_, c.llm_mlp, Lp_, Wv["llm.down"], l, dbn, g, true, dsp);
            tag("llm.down", l, x_, L_, llm_w_, llm_w_, 0);
        }
    }

    // ================================================================ action expert (part 1)
    if (ae_mega_) {
        // the megakernel's planner covers prefixes of up to ~1200 rows (its combine of the
        // attention key ranges is bounded); any longer prefix the reference accepts runs on the
        // per-node action expert (same kernels as the prefill) instead of failing
        try {
            build_ae_mega();
        } catch (const EngineError& e) {
            if (e.code != PI0B_E_UNSUPPORTED || env_int("PI0B_AE_MEGA", 1) > 1) throw;  // 2: megakernel or fail
            ae_mega_ = false;
            ae_tiled_.clear();
            ae_fallback_ = e.what();
        }
    }
    if (!ae_mega_) {
    // (proj/src/builder.cpp:291-363)
    {
        Op m;
        m.kind = kOpMemset;
        m.part = 1;
        m.mptr = stats_[1];
        m.mbytes = size_t(stats_cap_[1]) * stats_rows_ * 4;
        ops_.push_back(m);
        Op cs;
        cs.kind = kOpF64Bf16;
        cs.part = 1;
        cs.src64 = d_state_;
        cs.rows = 1;
        cs.cols = c.ae_state_dim;
        cs.dstb = state_b_;
        cs.ldb = state_ld_;
        ops_.push_back(cs);
        Op cn;
        cn.kind = kOpRowsF32;
        cn.part = 1;
        cn.src64 = d_noise_;
        cn.rows = C_;
        cn.cols = c.ae_action_dim;
        cn.dst32 = a_;
        cn.ld32 = act_ld_;
        cn.dstb = ab_;
        cn.ldb = act_ld_;
        ops_.push_back(cn);
    }
    {
        GemmParams g{};
        g.N = ae_w_;
        g.mode = kModeF32Store;
        g.flags = kFlagBias;
        g.bias = Wv["ae.state_proj"].b[0];
        g.out = st_;
        g.ldo = ae_w_;
        add_skinny(1, "ae.state_proj", 0, state_b_, state_ld_, 1, Wv["ae.state_proj"], 0, g);
        tag("ae.state_proj", 0, st_, 1, ae_w_, ae_w_, 0);
    }
    const float inv_ae = 1.0f / float(ae_w_);
    const int NA = c.ae_layers;
    for (int s = 0; s < FS_; ++s) {
        {   // action_proj with folded time MLP: silu(a W + T[s])
            GemmParams g{};
            g.N = ae_w_;
            g.mode = kModeSiluTable;
            g.table_row = Wv["ae.action_proj"].table + size_t(s) * ae_w_;
            g.out = ap_b_;
            g.ldo = ae_w_;
            add_skinny(1, "ae.action_proj", s, ab_, act_ld_, C_, Wv["ae.action_proj"], 0, g);
            tag("ae.action_proj", s, ap_b_, C_, ae_w_, ae_w_, 1);
        }
        float* ys = stats_slot(1);
        {   // action_out + bias -> y rows 1..63, state token -> y row 0 (ae.suffix)
            GemmParams g{};
            g.N = ae_w_;
            g.mode = kModeF32Store;
            g.flags = kFlagBias;
            g.bias = Wv["ae.action_out"].b[0];
            g.out = y_ + ae_w_;
            g.ldo = ae_w_;
            g.outb = yb_ + ae_w_;
            g.ldob = ae_w_;
            g.out_stats = ys + 1;
            g.row0_src = st_;
            add_skinny(1, "ae.action_out", s, ap_b_, ae_w_, C_, Wv["ae.action_out"], 0, g);
            tag("ae.suffix", s, y_, S_, ae_w_, ae_w_, 0);
        }
        for (int l = 0; l < NA; ++l) {
            const int i = s * NA + l;
            {   // ae.ln1 + ae.qkv, RoPE at positions L..L+63
                GemmParams g{};
                g.N = ae_qkv_n;
                g.mode = kModeBf16;
                g.flags = kFlagRowScale | kFlagRope;
                g.row_stats = ys;
                g.inv_width = inv_ae;
                g.eps = 1e-6f;
                g.rope_cs = rope_cs_;
                g.rope_pos0 = L_;
                g.rope_cols = ae_q_ + ae_kv_;
                g.out = aqkv_;
                g.ldo = ae_qkv_n;
                add_skinny(1, "ae.qkv", i, yb_, ae_w_, S_, Wv["ae.qkv"], l, g);
                tag("ae.qkv", i, aqkv_, S_, ae_qkv_n, ae_qkv_n, 1);
            }
            {   // cross attention over [LLM KV_l ; own KV] (ae.kcat / ae.vcat)
                AttnParams a{};
                a.q = aqkv_;
                a.ldq = ae_qkv_n;
                a.q_rows = S_;
                a.heads = c.ae_q_heads;
                a.kv_heads = c.ae_kv_heads;
                a.k0 = kv_[i % NL] + llm_q_;  // llm.qkv@mod (instance i % R)
                a.v0 = kv_[i % NL] + llm_q_ + llm_kv_;
                a.ld0 = llm_qkv_n;
                a.rows0 = Lp_;          // 32-row aligned segment boundary ...
                a.rows0_valid = L_;     // ... cached keys [L_, Lp_) masked
                a.k1 = aqkv_ + ae_q_;
                a.v1 = aqkv_ + ae_q_ + ae_kv_;
                a.ld1 = ae_qkv_n;
                a.rows1 = S_;
                a.out = ao_;
                a.ldo = ae_q_;
                add_attn(1, "ae.attn", i, 256, a);
                tag("ae.attn", i, ao_, S_, ae_q_, ae_q_, 1);
            }
            float* ps = stats_slot(1);
            {
                GemmParams g{};
                g.N = ae_w_;
                g.mode = kModeResid;
                g.resid_scale = 1.0f;
                g.out = y_;
                g.ldo = ae_w_;
                g.outb = yb_;
                g.ldob = ae_w_;
                g.out_stats = ps;
                add_skinny(1, "ae.proj", i, ao_, ae_q_, S_, Wv["ae.proj"], l, g);
                tag("ae.proj", i, y_, S_, ae_w_, ae_w_, 0);
            }
            {
                GemmParams g{};
                g.N = 2 * c.ae_mlp;
                g.mode = kModeGate;
                g.flags = kFlagRowScale;
                g.row_stats = ps;
                g.inv_width = inv_ae;
                g.eps = 1e-6f;
                g.out = ag_;
                g.ldo = c.ae_mlp;
                add_skinny(1, "ae.ffn", i, yb_, ae_w_, S_, Wv["ae.ffn"], l, g);
                tag("ae.ffn", i, ag_, S_, c.ae_mlp, c.ae_mlp, 1);
            }
            ys = stats_slot(1);
            {
                GemmParams g{};
                g.N = ae_w_;
                g.mode = kModeResid;
                g.resid_scale = 1.0f;
                g.out = y_;
                g.ldo = ae_w_;
                g.outb = yb_;
                g.ldob = ae_w_;
                g.out_stats = ys;
                add_skinny(1, "ae.down", i, ag_, c.ae_mlp, S_, Wv["ae.down"], l, g);
                tag("ae.down", i, y_, S_, ae_w_, ae_w_, 0);
            }
        }
        {   // ae.act_rows + ae.ln_out + ae.head + Euler: a += (r W * rms(r) + b) / FS
            GemmParams g{};
            g.N = c.ae_action_dim;
            g.mode = kModeResid;
            g.flags = kFlagRowScale | kFlagBias;
            g.row_stats = ys + 1;
            g.inv_width = inv_ae;
            g.eps = 1e-6f;
            g.bias = Wv["ae.head"].b[0];
            g.resid_scale = float(1.0 / double(FS_));
            g.out = a_;
            g.ldo = act_ld_;
            g.outb = ab_;
            g.ldob = act_ld_;
            add_skinny(1, "ae.head", s, yb_ + ae_w_, ae_w_, C_, Wv["ae.head"], 0, g);
            tag("ae.head", s, a_, C_, c.ae_action_dim, act_ld_, 0);
        }
    }
    }
    {
        Op o;
        o.kind = kOpF32F64;
        o.part = 1;
        o.src32 = a_;
        o.ld32 = act_ld_;
        o.rows = C_;
        o.cols = c.ae_action_dim;
        o.dst64 = d_out_;
        ops_.push_back(o);
    }

}

// ------------------------------------------------------------------ action-expert megakernel

// The whole action expert (proj/src/builder.cpp:291-363) as one persistent launch: a zeroing
// memset (phase counters + attention accumulators), the two input conversions, the kernel.
void Engine::build_ae_mega() {
    const auto& c = c_;
    const int W = ae_w_, NQ = ae_q_ + 2 * ae_kv_, MLP = c.ae_mlp, NA = c.ae_layers;
    if (c.ae_kv_heads != 1 || c.llm_kv_heads != 1)
        throw EngineError(PI0B_E_UNSUPPORTED, "action-expert megakernel: MQA (1 kv head) only");
    state32_ = alloc<float>(size_t(std::max(c.ae_state_dim, 8)));
    std::vector<AeMat> mats;
    auto add = [&](const void* ptr, int rows, int cols, long long ld) {
        if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld % 4))
            throw EngineError(PI0B_E_INVALID, "megakernel operand needs 16-byte aligned rows");
        mats.push_back(AeMat{ptr, rows, cols, int(ld), {0, 0, 0}});
        return int(mats.size()) - 1;
    };
    auto wmat = [&](const char* node, int inst, int rows, int order = kTilePlain) {
        // tile-contiguous copy of 64-row tiles: AeMat{ptr, rows, k, k-blocks}
        const NodeWeights& nw = W_.at(node);
        const int R = order == kTilePlain128 ? 128 : 64;
        const int kb = (nw.k + 63) / 64, nt = (rows + R - 1) / R;
        __nv_bfloat16* t = nullptr;
        if (donor_) {  // the donor's tiled copy of the same weight instance
            for (const TiledW& tw : donor_->ae_tiled_)
                if (tw.src == nw.w.at(size_t(inst)) && tw.order == order && tw.rows == rows) t = tw.dst;
            if (!t) throw EngineError(PI0B_E_STATE, "shared weights: the donor has no tiled copy of " + std::string(node));
        } else {
            t = alloc<__nv_bfloat16>(size_t(nt) * kb * R * 64);
            ae_tiled_.push_back({nw.w.at(size_t(inst)), rows, nw.k, nw.ldk, t, order});
        }
        mats.push_back(AeMat{t, rows, nw.k, kb, {0, 0, 0}});
        return int(mats.size()) - 1;
    };
    AePlanInput in;
    in.num_ctas = ae_ctas_;
    in.width = W;
    in.n_qkv = NQ;
    in.q_width = ae_q_;
    in.mlp = MLP;
    in.layers = NA;
    in.flow_steps = FS_;
    in.heads = c.ae_q_heads;
    in.chunk = C_;
    in.act_dim = c.ae_action_dim;
    in.state_dim = c.ae_state_dim;
    in.rope_cols = ae_q_ + ae_kv_;
    in.kv_rows0 = Lp_;  // own keys start at the 32-aligned Lp_; cached keys [L_, Lp_) are masked
    in.key_blocks = (Lp_ + S_ + 63) / 64;
    in.record = o_.record_checkpoints != 0;
    in.ao_tasks = env_int("PI0B_AE_AO_TASKS", in.ao_tasks);
    in.proj_tasks = env_int("PI0B_AE_PROJ_TASKS", in.proj_tasks);
    in.down_tasks = env_int("PI0B_AE_DOWN_TASKS", in.down_tasks);
    in.proj_ncol = env_int("PI0B_AE_PROJ_NCOL", in.proj_ncol) == 64 ? 64 : 128;
    in.down_ncol = env_int("PI0B_AE_DOWN_NCOL", in.down_ncol) == 128 ? 128 : 64;
    in.ao_ncol = env_int("PI0B_AE_AO_NCOL", in.ao_ncol) == 128 ? 128 : 64;
    in.pair_qkv = env_int("PI0B_AE_PAIR", 1) != 0;
    in.attn_single = env_int("PI0B_AE_ATTN_SINGLE", 1) != 0;
    in.sym_qkv = env_int("PI0B_AE_SYM_QKV", 1) != 0;
    in.per_head_proj = env_int("PI0B_AE_HEAD_DEP", 1) != 0;
    in.pair_ffn = env_int("PI0B_AE_PAIR_FFN", 1) != 0 && (2 * MLP) % 128 == 0 && 2 * (2 * MLP / 128) <= ae_ctas_ &&
                  ae_ctas_ % 2 == 0;
    ae_cluster_ = in.pair_qkv || in.pair_ffn;  // pair tasks need the 2-CTA cluster launch
    in.mat_wst = wmat("ae.state_proj", 0, W);
    in.mat_wap = wmat("ae.action_proj", 0, W);
    in.mat_wao = wmat("ae.action_out", 0, W, in.ao_ncol == 128 ? kTilePlain128 : kTilePlain);
    in.mat_whead = wmat("ae.head", 0, c.ae_action_dim);
    for (int l = 0; l < NA; ++l) {
        in.mat_wqkv.push_back(wmat("ae.qkv", l, NQ, kTilePaired));
        in.mat_wproj.push_back(wmat("ae.proj", l, W, in.proj_ncol == 128 ? kTilePlain128 : kTilePlain));
        in.mat_wffn.push_back(wmat("ae.ffn", l, 2 * MLP, in.pair_ffn ? kTilePlain128 : kTilePaired));
        in.mat_wdown.push_back(wmat("ae.down", l, W, in.down_ncol == 128 ? kTilePlain128 : kTilePlain));
    }
    const int llm_qkv_n = llm_q_ + 2 * llm_kv_;
    for (int l = 0; l < c.llm_layers; ++l)  // AE instance i reads LLM layer i % llm_layers (@mod)
        in.mat_kv.push_back(add(kv_[size_t(l)], Lp_, llm_qkv_n, llm_qkv_n));
    in.mat_y = add(y_, S_, W, W);
    in.mat_yh = add(y_ + W, C_, W, W);  // ae.act_rows: rows 1..63
    in.mat_ap = add(ap_b_, C_, W, W);
    in.mat_g = add(ag_, S_, MLP, MLP);
    in.mat_qkv = add(aqkv_, S_, NQ, NQ);
    try {
        ae_plan_ = ae_plan(in);
    } catch (const std::invalid_argument& e) {
        throw EngineError(PI0B_E_UNSUPPORTED, e.what());
    }
    // zero-on-entry region: the phase counters
    ae_zero_bytes_ = size_t(round_up(ae_plan_.n_bars * 4, 256));
    uint8_t* z = alloc<uint8_t>(ae_zero_bytes_);
    ae_zero_ = z;
    __nv_bfloat16* opart = alloc<__nv_bfloat16>(size_t(ae_plan_.attn_splits) * 64 * ae_q_);
    float2* ml = alloc<float2>(size_t(ae_plan_.attn_splits) * c.ae_q_heads * 64);

    AeMat* dmats = alloc<AeMat>(mats.size());
    PI0B_CUDA(cudaMemcpyAsync(dmats, mats.data(), mats.size() * sizeof(AeMat), cudaMemcpyHostToDevice, stream_));
    AeTask* dtasks = alloc<AeTask>(ae_plan_.table.size());
    PI0B_CUDA(cudaMemcpyAsync(dtasks, ae_plan_.table.data(), ae_plan_.table.size() * sizeof(AeTask),
                              cudaMemcpyHostToDevice, stream_));
    float* rec_y = nullptr;
    float* rec_a = nullptr;
    if (in.record) {
        rec_y = alloc<float>(size_t(FS_) * NA * 64 * W);
        rec_a = alloc<float>(size_t(FS_) * C_ * act_ld_);
    }
    PI0B_CUDA(cudaStreamSynchronize(stream_));

    // V tensor maps for the attention tasks: every LLM KV cache, then the expert's q|k|v rows
    {
        std::vector<CUtensorMap> vm;
        for (int l = 0; l < c.llm_layers; ++l) vm.push_back(make_tmap_bf16(kv_[size_t(l)], L_, llm_qkv_n, llm_qkv_n, 32));
        vm.push_back(make_tmap_bf16(aqkv_, S_, NQ, NQ, 32));  // own K / V rows, 32-key boxes
        vm.push_back(make_tmap_bf16(aqkv_, S_, NQ, NQ, 64));  // own Q rows, 64-row boxes
        CUtensorMap* dvm = alloc<CUtensorMap>(vm.size());
        PI0B_CUDA(cudaMemcpy(dvm, vm.data(), vm.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
        ae_p_.vmaps = dvm;
        ae_p_.n_vmaps = int(vm.size());
    }
    AeParams& P = ae_p_;
    P.tasks = dtasks;
    P.task_stride = ae_plan_.stride;
    P.mats = dmats;
    P.bars = reinterpret_cast<unsigned*>(z);
    P.n_bars = ae_plan_.n_bars;
    P.y = y_;
    P.a = a_;
    P.lda = act_ld_;
    P.state = state32_;
    P.st = st_;
    P.qkv = aqkv_;
    P.ap = ap_b_;
    P.g = ag_;
    P.opart = opart;
    P.ml = ml;
    P.rope_cs = rope_cs_;
    P.table = W_.at("ae.action_proj").table;
    P.b_state = W_.at("ae.state_proj").b.at(0);
    P.b_out = W_.at("ae.action_out").b.at(0);
    P.b_head = W_.at("ae.head").b.at(0);
    P.rec_y = rec_y;
    P.rec_a = rec_a;
    P.width = W;
    P.n_qkv = NQ;
    P.q_width = ae_q_;
    P.mlp = MLP;
    P.act_dim = c.ae_action_dim;
    P.state_dim = c.ae_state_dim;
    P.chunk = C_;
    P.heads = c.ae_q_heads;
    P.rope_pos0 = L_;
    P.rope_cols = ae_q_ + ae_kv_;
    P.kv_rows0 = Lp_;
    P.kv_valid0 = L_;
    P.kcol_cache = llm_q_;
    P.kcol_own = ae_q_;
    P.key_blocks = in.key_blocks;
    P.attn_splits = ae_plan_.attn_splits;
    P.scale_log2 = float(1.4426950408889634 / std::sqrt(double(c.ae_head_dim)));
    P.inv_width = 1.0f / float(W);
    P.eps = 1e-6f;
    P.euler = float(1.0 / double(FS_));
    P.limit_phase = env_int("PI0B_AE_LIMIT", 1 << 30);
    P.trace = nullptr;
    P.dbg = nullptr;
    if (env_int("PI0B_AE_TRACE", 0)) {
        P.dbg = alloc<unsigned long long>(size_t(ae_ctas_) * 128);
        PI0B_CUDA(cudaMemset(P.dbg, 0, size_t(ae_ctas_) * 128 * 8));
        P.trace = alloc<unsigned long long>(ae_plan_.table.size() * 16);
        PI0B_CUDA(cudaMemset(P.trace, 0, ae_plan_.table.size() * 128));
    }

    Op m;
    m.kind = kOpMemset;
    m.part = 1;
    m.mptr = ae_zero_;
    m.mbytes = ae_zero_bytes_;
    ops_.push_back(m);
    Op cs;   // robot state -> fp32 (ae.state_proj input)
    cs.kind = kOpRowsF32;
    cs.part = 1;
    cs.src64 = d_state_;
    cs.rows = 1;
    cs.cols = c.ae_state_dim;
    cs.dst32 = state32_;
    cs.ld32 = c.ae_state_dim;
    ops_.push_back(cs);
    Op cn;   // noise -> Euler state a_0
    cn.kind = kOpRowsF32;
    cn.part = 1;
    cn.src64 = d_noise_;
    cn.rows = C_;
    cn.cols = c.ae_action_dim;
    cn.dst32 = a_;
    cn.ld32 = act_ld_;
    ops_.push_back(cn);
    Op k;
    k.kind = kOpAeMega;
    k.part = 1;
    k.node = "ae.mega";
    if (in.record) {
        for (int i = 0; i < FS_ * NA; ++i)
            k.extra_ck.push_back({"ae.down", i, rec_y + size_t(i) * 64 * W, S_, W, W});
        for (int s2 = 0; s2 < FS_; ++s2)
            k.extra_ck.push_back({"ae.head", s2, rec_a + size_t(s2) * C_ * act_ld_, C_, c.ae_action_dim, act_ld_});
    }
    ops_.push_back(k);
}

// ------------------------------------------------------------------ weights

void Engine::gen_weights(uint64_t seed) {
    if (donor_) throw EngineError(PI0B_E_STATE, "weights are shared from another engine: load them there");
    // rtvla::gen_weights (proj/src/evaluate.cpp:38-75): W ~ U(+-1/sqrt(k)) seeded by
    // (seed, node id, instance, 1); bias role 2; bias_table row s role 4.
    for (auto& kv : W_) {
        const std::string& id = kv.first;
        NodeWeights& nw = kv.second;
        const double lim = 1.0 / std::sqrt(double(std::max(1, nw.k)));
        for (int i = 0; i < nw.instances; ++i) {
            PI0B_CUDA(launch_gen_weight(nw.w[i], nw.ldk, nw.k, nw.m, nw.perm, nw.rope_cols,
                                        seed_hash(seed, id, uint64_t(i), 1), -lim, lim, stream_));
            if (nw.has_bias)
                PI0B_CUDA(launch_gen_vector(nw.b[i], nw.m, seed_hash(seed, id, uint64_t(i), 2), -lim, lim, stream_));
        }
        if (nw.has_table)
            for (int s = 0; s < FS_; ++s)
                PI0B_CUDA(launch_gen_vector(nw.table + size_t(s) * nw.m, nw.m,
                                            seed_hash(seed, id, uint64_t(s), 4), -lim, lim, stream_));
    }
    PI0B_CUDA(cudaStreamSynchronize(stream_));
    for (auto& kv : W_) {
        kv.second.loaded.assign(size_t(kv.second.instances), 1);
        kv.second.table_loaded = kv.second.has_table;
    }
    ae_tiles_dirty_ = true;
}

std::string Engine::missing_weights() const {
    if (donor_) return donor_->missing_weights();
    for (const auto& kv : W_) {
        const NodeWeights& nw = kv.second;
        for (int i = 0; i < nw.instances; ++i)
            if (size_t(i) >= nw.loaded.size() || !nw.loaded[size_t(i)])
                return "no weights for node '" + kv.first + "' instance " + std::to_string(i);
        if (nw.has_table && !nw.table_loaded) return "no bias table for node '" + kv.first + "'";
    }
    return {};
}

void Engine::set_weight(const std::string& id, long long inst, const double* w, long long k, long long m,
                        const double* bias, long long blen) {
    if (donor_) throw EngineError(PI0B_E_STATE, "weights are shared from another engine: load them there");
    auto it = W_.find(id);
    if (it == W_.end()) throw EngineError(PI0B_E_INVALID, "no weight-bearing node '" + id + "'");
    NodeWeights& nw = it->second;
    if (inst < 0 || inst >= nw.instances)
        throw EngineError(PI0B_E_INVALID, "node '" + id + "': weight instance out of range");
    if (k != nw.k || m != nw.m) throw EngineError(PI0B_E_INVALID, "node '" + id + "': weight shape mismatch");
    if (nw.has_bias && (!bias || blen != nw.m))
        throw EngineError(PI0B_E_INVALID, "node '" + id + "': bias missing or wrong length");
    double* dw = nullptr;
    PI0B_CUDA(cudaMalloc(&dw, size_t(k) * m * 8));
    // Stream-ordered upload: a pageable cudaMemcpy may return before its DMA lands, and the
    // engine stream does not synchronise with the legacy stream.
    PI0B_CUDA(cudaMemcpyAsync(dw, w, size_t(k) * m * 8, cudaMemcpyHostToDevice, stream_));
    cudaError_t e = launch_pack_weight(nw.w[size_t(inst)], nw.ldk, dw, int(k), int(m), nw.perm, nw.rope_cols, stream_);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream_);
    cudaFree(dw);
    PI0B_CUDA(e);
    if (nw.has_bias) {
        std::vector<float> b(static_cast<size_t>(m));
        for (long long j = 0; j < m; ++j) b[size_t(j)] = float(bias[j]);
        PI0B_CUDA(cudaMemcpyAsync(nw.b[size_t(inst)], b.data(), size_t(m) * 4, cudaMemcpyHostToDevice, stream_));
        PI0B_CUDA(cudaStreamSynchronize(stream_));
    }
    if (nw.loaded.size() != size_t(nw.instances)) nw.loaded.assign(size_t(nw.instances), 0);
    nw.loaded[size_t(inst)] = 1;
    ae_tiles_dirty_ = true;
}

void Engine::set_bias_table(const std::string& id, const double* t, long long rows, long long m) {
    if (donor_) throw EngineError(PI0B_E_STATE, "weights are shared from another engine: load them there");
    auto it = W_.find(id);
    if (it == W_.end() || !it->second.has_table)
        throw EngineError(PI0B_E_INVALID, "node '" + id + "' has no bias table");
    if (rows != FS_ || m != it->second.m) throw EngineError(PI0B_E_INVALID, "bias table shape mismatch");
    std::vector<float> f(size_t(rows * m));
    for (size_t i = 0; i < f.size(); ++i) f[i] = float(t[i]);
    PI0B_CUDA(cudaMemcpyAsync(it->second.table, f.data(), f.size() * 4, cudaMemcpyHostToDevice, stream_));
    PI0B_CUDA(cudaStreamSynchronize(stream_));
    it->second.table_loaded = true;
}

// ------------------------------------------------------------------ execution

void Engine::upload_inputs(const double* patches, const double* state, const double* noise,
                           const double* prompt, int which) {
    // which: 0 = all, 1 = prefix inputs, 2 = action inputs, 3 = all but the patches. Copies go through pinned
    // staging so the H2D transfers are asynchronous DMA on the engine stream.  Each input owns a
    // fixed region of h_in_ (prompt | state | noise), and no staging buffer is rewritten before
    // the DMAs of the previous upload have read it (h2d_ev_): a prefix upload followed at once by
    // an action upload (the streaming runtime) cannot overwrite bytes still queued for a DMA.
    if (!h2d_ev_) PI0B_CUDA(cudaEventCreateWithFlags(&h2d_ev_, cudaEventDisableTiming));
    PI0B_CUDA(cudaEventSynchronize(h2d_ev_));
    // Large tensors go in 256 KB pieces so that the host copy of piece i + 1 into the pinned
    // staging overlaps the DMA of piece i.
    auto stage = [&](const double* src, size_t n, double* dev, double* h) {
        if (!n) return;
        if (!src) throw EngineError(PI0B_E_INVALID, "missing input tensor");
        constexpr size_t kPiece = 32768;  // doubles (256 KB)
        for (size_t o = 0; o < n; o += kPiece) {
            const size_t m = std::min(kPiece, n - o);
            std::memcpy(h + o, src + o, m * 8);
            PI0B_CUDA(cudaMemcpyAsync(dev + o, h + o, m * 8, cudaMemcpyHostToDevice, stream_));
        }
    };
    double* h_prompt = h_in_;
    double* h_state = h_prompt + n_prompt_;
    double* h_noise = h_state + n_state_;
    if (which == 0 || which == 1) {
        stage_patches_bf16(patches);
        if (P_ > 0) stage(prompt, n_prompt_, d_prompt_, h_prompt);
    }
    if (which == 3 && P_ > 0) stage(prompt, n_prompt_, d_prompt_, h_prompt);  // image front-end: no patches
    if (which == 0 || which == 2 || which == 3) {
        stage(state, n_state_, d_state_, h_state);
        stage(noise, n_noise_, d_noise_, h_noise);
    }
    PI0B_CUDA(cudaEventRecord(h2d_ev_, stream_));
}

// bf16(float(x)) with float -> bf16 round-to-nearest-even: bit-identical to the device conversion
// (kernels_misc.cu f64_to_bf16_rows_kernel, __float2bfloat16_rn(float(x))).
static inline uint16_t host_bf16(double x) {
    const float f = float(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t(0x7fffu);  // canonical NaN, as cvt.rn.bf16.f32
    return uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

void Engine::stage_patches_bf16(const double* patches) {
    // The patches are the one large input (2.4 MB of fp64 at 2 views): converted on the host in
    // row pieces into pinned bf16 staging, each piece's (contiguous) DMA issued as soon as it is
    // converted; the graph's conversion op then only pads them into the GEMM operand.
    if (!patches) throw EngineError(PI0B_E_INVALID, "missing input tensor");
    const int cols = c_.ve_patch_in;
    constexpr int kRowsPerPiece = 32;
    const size_t np = size_t((T_ + kRowsPerPiece - 1) / kRowsPerPiece);
    constexpr size_t kDmas = 4;
    const size_t per_dma = std::max<size_t>(1, (np + kDmas - 1) / kDmas);
    uint16_t* hb = h_pb_;
    const size_t T = size_t(T_);
    staging_->run(
        np,
        [=](size_t k) {
            const size_t r0 = k * kRowsPerPiece, nr = std::min<size_t>(kRowsPerPiece, T - r0);
            const double* src = patches + r0 * cols;
            uint16_t* dst = hb + r0 * cols;
            for (size_t i = 0, n = nr * cols; i < n; ++i) dst[i] = host_bf16(src[i]);
        },
        [&](size_t k) {  // a few large DMAs: each costs ~10 us of fixed latency on the B200 boxes
            if ((k + 1) % per_dma && k + 1 != np) return;
            const size_t r0 = (k / per_dma) * per_dma * kRowsPerPiece, r1 = std::min<size_t>((k + 1) * kRowsPerPiece, T);
            PI0B_CUDA(cudaMemcpyAsync(d_pb_ + r0 * cols, hb + r0 * cols, (r1 - r0) * cols * 2, cudaMemcpyHostToDevice, stream_));
        });
    PI0B_CUDA(cudaMemcpyAsync(d_patch_host_bf16_, h_flag_ + 1, sizeof(int), cudaMemcpyHostToDevice, stream_));
}

void Engine::upload_images(const double* images, int height, int width) {
    const auto& c = c_;
    const int C = 3;
    const int P = int(std::lround(std::sqrt(double(c.ve_patch_in / C))));
    const int g = int(std::lround(std::sqrt(double(c.tokens_per_view))));
    if (P * P * C != c.ve_patch_in || g * g != c.tokens_per_view)
        throw EngineError(PI0B_E_UNSUPPORTED, "image front-end: patch_in must be P*P*3 and tokens_per_view g*g");
    if (!images || height < 2 || width < 2) throw EngineError(PI0B_E_INVALID, "image front-end: images of at least 2x2");
    const size_t n = size_t(c.views) * height * width * C;
    if (n > n_img_) {
        if (h_img_) cudaFreeHost(h_img_);
        if (d_img_) cudaFree(d_img_);
        PI0B_CUDA(cudaMallocHost(&h_img_, n * 8));
        PI0B_CUDA(cudaMalloc(&d_img_, n * 8));
        n_img_ = n;
    }
    PI0B_CUDA(cudaStreamSynchronize(stream_));  // the staging buffer may still feed the last copy
    std::memcpy(h_img_, images, n * 8);
    PI0B_CUDA(cudaMemcpyAsync(d_img_, h_img_, n * 8, cudaMemcpyHostToDevice, stream_));
    PI0B_CUDA(launch_image_patches(d_img_, c.views, height, width, C, g * P, P, d_patches_, stream_));
    PI0B_CUDA(cudaMemcpyAsync(d_patch_host_bf16_, h_flag_ + 0, sizeof(int), cudaMemcpyHostToDevice, stream_));
}

void Engine::run_ops(int part, cudaStream_t st) {
    // (The AE's input conversions forked onto a parallel graph branch cut the gap before the
    // megakernel 6.2 -> 3.8 us but made the megakernel itself ~10 us slower: kept in line.)
    for (const Op& op : ops_)
        if (part == 2 || op.part == part) emit_op(op, st);  // part 2 = everything
}

void Engine::emit_op(const Op& op, cudaStream_t st) {
    {
        switch (op.kind) {
            case kOpGemm: PI0B_CUDA(launch_gemm(op.bn, op.ta, op.tb, op.gp, st)); break;
            case kOpSkinny:
                PI0B_CUDA(launch_skinny(op.ta, op.tb, op.gp, op.n_packed, op.cluster, pdl_, st));
                break;
            case kOpAttn: PI0B_CUDA(launch_fattn(op.hd, op.fm, op.ap, st)); break;
            case kOpRowsF32:
                PI0B_CUDA(launch_rows_to_f32(op.src64, op.rows, op.cols, op.dst32, op.ld32, op.dstb, op.ldb,
                                             op.stats, st));
                break;
            case kOpF64Bf16:
                PI0B_CUDA(launch_f64_to_bf16_rows(op.src64, op.rows, op.cols, op.dstb, op.ldb, st, op.skip, op.srcb));
                break;
            case kOpF32F64: PI0B_CUDA(launch_f32_to_f64(op.src32, op.ld32, op.rows, op.cols, op.dst64, st)); break;
            case kOpMemset: PI0B_CUDA(cudaMemsetAsync(op.mptr, 0, op.mbytes, st)); break;
            case kOpAeMega: PI0B_CUDA(aemk_launch(ae_p_, ae_ctas_, st, ae_cluster_)); break;
            case kOpVeEpoch: PI0B_CUDA(launch_ve_epoch(ve_sync_ + kVeEpoch, st)); break;
            case kOpVeWait: PI0B_CUDA(launch_ve_wait(ve_sync_, op.ve_mask, ve_sync_ + kVeEpoch, unsigned(op.ve_step), st)); break;
            case kOpVePush: {
                VePushArgs a{};
                a.nseg = op.ve_nseg;
                for (int sg = 0; sg < op.ve_nseg; ++sg) {
                    a.src[sg] = static_cast<const uint4*>(op.ve_src[sg]);
                    a.n16[sg] = (long long)(op.ve_bytes[sg] / 16);
                }
                for (int p = 0; p < G_; ++p) {
                    if (p == g_ || (op.ve_root_only && p != 0)) continue;
                    const pi0b_ve_buffers& b = ve_peers_[size_t(p)];
                    for (int sg = 0; sg < op.ve_nseg; ++sg) {
                        void* base = op.ve_buf[sg] < 2 ? b.qkv[op.ve_buf[sg]]
                                                       : (op.ve_buf[sg] == 2 ? b.x : (op.ve_buf[sg] == 3 ? b.xb : b.stats));
                        a.dst[a.npeer][sg] = reinterpret_cast<uint4*>(static_cast<uint8_t*>(base) + op.ve_off[sg]);
                    }
                    a.flag[a.npeer] = static_cast<unsigned*>(b.sync) + g_;
                    ++a.npeer;
                }
                a.epoch = ve_sync_ + kVeEpoch;
                a.done = ve_sync_ + kVeDone;
                a.step = unsigned(op.ve_step);
                PI0B_CUDA(launch_ve_push(a, st));
                break;
            }
        }
        if (o_.record_checkpoints)
            for (const CkTag& tg : op.extra_ck) {
                Checkpoint& ck = ck_[std::make_pair(tg.node, tg.inst)];
                if (!ck.dev) {
                    PI0B_CUDA(cudaMalloc(&ck.dev, size_t(tg.rows) * tg.cols * 4));
                    ck.rows = tg.rows;
                    ck.cols = tg.cols;
                    ck.bf16 = 0;
                }
                PI0B_CUDA(cudaMemcpy2DAsync(ck.dev, tg.cols * 4, tg.ptr, tg.ld * 4, tg.cols * 4, tg.rows,
                                            cudaMemcpyDeviceToDevice, st));
            }
        if (o_.record_checkpoints && op.inst >= 0) {
            const auto key = std::make_pair(op.node, op.inst);
            Checkpoint& ck = ck_[key];
            const size_t esz = op.ck_bf16 ? 2 : 4;
            if (!ck.dev) {
                PI0B_CUDA(cudaMalloc(&ck.dev, size_t(op.ck_rows) * op.ck_cols * esz));
                ck.rows = op.ck_rows;
                ck.cols = op.ck_cols;
                ck.bf16 = op.ck_bf16;
            }
            PI0B_CUDA(cudaMemcpy2DAsync(ck.dev, op.ck_cols * esz, op.ck_ptr, op.ck_ld * esz,
                                        op.ck_cols * esz, op.ck_rows, cudaMemcpyDeviceToDevice, st));
        }
    }
}

void Engine::capture(int part, int slot) {
    cudaGraph_t g = nullptr;
    PI0B_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    try {
        run_ops(part, stream_);
    } catch (...) {
        cudaStreamEndCapture(stream_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    PI0B_CUDA(cudaStreamEndCapture(stream_, &g));
    cudaError_t e = cudaGraphInstantiate(&graph_[slot], g, 0);
    cudaGraphDestroy(g);
    PI0B_CUDA(e);
}

// part: 0 = full, 1 = prefix, 2 = action (C-ABI numbering)
void Engine::launch(int part, cudaStream_t st) {
    if (G_ > 1 && !ve_peers_set_) throw EngineError(PI0B_E_STATE, "view-sharded engine: set_ve_peers first");
    if (G_ > 1 && g_ != 0 && part != 1)
        throw EngineError(PI0B_E_STATE, "view-sharded engine: shards other than 0 run the prefix only");
    if (!weights_checked_) {  // every (node, instance, bias table) written at least once
        const std::string miss = missing_weights();
        if (!miss.empty()) throw EngineError(PI0B_E_STATE, "weights not loaded: " + miss);
        weights_checked_ = true;
    }
    if (ae_mega_ && ae_tiles_dirty_) {  // (re)build the tile-contiguous AE weight copies
        for (const TiledW& tw : ae_tiled_) PI0B_CUDA(launch_tile_weight(tw.src, tw.rows, tw.k, tw.ldk, tw.dst, tw.order, stream_));
        PI0B_CUDA(cudaStreamSynchronize(stream_));
        ae_tiles_dirty_ = false;
    }
    if (donor_) donor_->prepare();  // the shared tiled AE copies are the donor's
    const int internal = part == 0 ? 2 : part - 1;  // ops filter: 2 all, 0 prefix, 1 action
    const int gidx = part;
    if (o_.use_cuda_graph && !o_.record_checkpoints) {
        if (!graph_[gidx]) capture(internal, gidx);
        PI0B_CUDA(cudaGraphLaunch(graph_[gidx], st));
    } else {
        run_ops(internal, st);
    }
}

void Engine::prefix_async(const double* patches, const double* prompt) {
    if (!done_ev_) PI0B_CUDA(cudaEventCreateWithFlags(&done_ev_, cudaEventDisableTiming));
    upload_inputs(patches, nullptr, nullptr, prompt, 1);
    launch(1, stream_);
    PI0B_CUDA(cudaEventRecord(done_ev_, stream_));
}
void Engine::tick_async(const double* state, const double* noise) {
    if (!done_ev_) PI0B_CUDA(cudaEventCreateWithFlags(&done_ev_, cudaEventDisableTiming));
    upload_inputs(nullptr, state, noise, nullptr, 2);
    launch(2, stream_);
    PI0B_CUDA(cudaMemcpyAsync(h_out_, d_out_, n_out_ * 8, cudaMemcpyDeviceToHost, stream_));
    PI0B_CUDA(cudaEventRecord(done_ev_, stream_));
}
bool Engine::idle() {
    if (!done_ev_) return true;
    const cudaError_t e = cudaEventQuery(done_ev_);
    if (e == cudaErrorNotReady) return false;
    PI0B_CUDA(e);
    return true;
}
const double* Engine::tick_result() {
    for (size_t i = 0; i < n_out_; ++i)
        if (!std::isfinite(h_out_[i])) throw EngineError(PI0B_E_NUMERIC, "non-finite action output");
    return h_out_;
}

void Engine::fetch_actions(double* out) {
    PI0B_CUDA(cudaMemcpyAsync(h_out_, d_out_, n_out_ * 8, cudaMemcpyDeviceToHost, stream_));
    PI0B_CUDA(cudaStreamSynchronize(stream_));
    for (size_t i = 0; i < n_out_; ++i)
        if (!std::isfinite(h_out_[i])) throw EngineError(PI0B_E_NUMERIC, "non-finite action output");
    std::memcpy(out, h_out_, n_out_ * 8);
}

int Engine::kernel_count(int part) const {
    const int internal = part == 0 ? 2 : part - 1;
    int n = 0;
    for (const Op& op : ops_)
        if ((internal == 2 || op.part == internal) && op.is_kernel()) ++n;
    return n;
}

// One line per planned op: "<index> <part> <kind> <node> <inst> <grid> <detail>".
std::string Engine::describe() const {
    static const char* kinds[] = {"gemm", "attn", "rows_f32", "f64_bf16", "f32_f64", "memset", "skinny", "ae_mega",
                                  "ve_epoch", "ve_push", "ve_wait"};
    std::string s;
    int idx = 0;
    for (const Op& op : ops_) {
        char buf[256];
        if (op.kind == kOpGemm) {
            const int mt = (op.gp.M + 127) / 128, nt = (op.gp.N + op.bn - 1) / op.bn;
            snprintf(buf, sizeof buf, "%d %d gemm %s %d %dx%dx%d M=%d N=%d K=%d bn=%d mode=%d%s\n", idx, op.part,
                     op.node.c_str(), op.inst, mt, nt, op.gp.splits, op.gp.M, op.gp.N, op.gp.K, op.bn, op.gp.mode,
                     op.gp.cg > 1 ? (op.gp.persist ? " persistent cta-pair" : " cta-pair")
                                  : op.gp.persist ? (op.gp.mt > 1 ? " persistent mt2" : " persistent") : (op.gp.mt > 1 ? " mt2" : ""));
        } else if (op.kind == kOpSkinny) {
            snprintf(buf, sizeof buf, "%d %d skinny %s %d tiles=%d cluster=%d M=%d N=%d K=%d mode=%d\n", idx, op.part,
                     op.node.c_str(), op.inst, skinny_tiles(op.n_packed), op.cluster, op.gp.M, op.gp.N, op.gp.K,
                     op.gp.mode);
        } else if (op.kind == kOpAeMega) {
            snprintf(buf, sizeof buf, "%d %d ae_mega %s 0 ctas=%d tasks=%d phases=%d counters=%d stride=%d wload=%.0f..%.0fKB\n",
                     idx, op.part, op.node.c_str(), ae_ctas_, ae_plan_.n_tasks, ae_plan_.n_phases, ae_plan_.n_bars,
                     ae_plan_.stride, ae_plan_.min_load / 1024, ae_plan_.max_load / 1024);
        } else if (op.kind == kOpAttn) {
            snprintf(buf, sizeof buf, "%d %d attn %s %d splits=%d q=%d kv=%d hd=%d\n", idx, op.part, op.node.c_str(),
                     op.inst, op.ap.kv_splits, op.ap.q_rows, op.ap.rows0 + op.ap.rows1, op.hd);
        } else {
            snprintf(buf, sizeof buf, "%d %d %s %s %d\n", idx, op.part, kinds[op.kind], op.node.c_str(), op.inst);
        }
        s += buf;
        ++idx;
    }
    if (!ae_fallback_.empty()) s += "# action expert on per-node kernels: " + ae_fallback_ + "\n";
    return s;
}

// Average device time of one launch of `node`'s kernels, measured with CUDA events on the
// engine stream over `reps` back-to-back passes over all instances (bench roofline).
double Engine::time_node(const std::string& node, int reps, int* launches) {
    prepare();
    std::vector<const Op*> sel;
    for (const Op& op : ops_)
        if (op.node == node && (op.kind == kOpGemm || op.kind == kOpAttn || op.kind == kOpSkinny || op.kind == kOpAeMega))
            sel.push_back(&op);
    if (sel.empty()) throw EngineError(PI0B_E_INVALID, "no kernels for node '" + node + "'");
    auto fire = [&](const Op& op) {
        if (op.kind == kOpGemm) PI0B_CUDA(launch_gemm(op.bn, op.ta, op.tb, op.gp, stream_));
        else if (op.kind == kOpSkinny) PI0B_CUDA(launch_skinny(op.ta, op.tb, op.gp, op.n_packed, op.cluster, pdl_, stream_));
        else if (op.kind == kOpAeMega) {
            PI0B_CUDA(cudaMemsetAsync(ae_zero_, 0, ae_zero_bytes_, stream_));
            PI0B_CUDA(aemk_launch(ae_p_, ae_ctas_, stream_, ae_cluster_));
        }
        else PI0B_CUDA(launch_fattn(op.hd, op.fm, op.ap, stream_));
    };
    for (const Op* op : sel) fire(*op);
    cudaEvent_t a, b;
    PI0B_CUDA(cudaEventCreate(&a));
    PI0B_CUDA(cudaEventCreate(&b));
    PI0B_CUDA(cudaEventRecord(a, stream_));
    for (int r = 0; r < reps; ++r)
        for (const Op* op : sel) fire(*op);
    PI0B_CUDA(cudaEventRecord(b, stream_));
    PI0B_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    PI0B_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *launches = int(sel.size()) * reps;
    return double(ms) / double(*launches);
}

void Engine::ae_trace(void* tasks, unsigned long long* stamps, long long cap, int* ctas, int* stride) {
    if (!ae_mega_ || !ae_p_.trace) throw EngineError(PI0B_E_STATE, "no megakernel trace (set PI0B_AE_TRACE=1)");
    *ctas = ae_ctas_;
    *stride = ae_plan_.stride;
    const size_t n = ae_plan_.table.size();
    if (cap < (long long)n) throw EngineError(PI0B_E_INVALID, "trace buffer too small");
    PI0B_CUDA(cudaStreamSynchronize(stream_));
    std::memcpy(tasks, ae_plan_.table.data(), n * sizeof(AeTask));
    PI0B_CUDA(cudaMemcpy(stamps, ae_p_.trace, n * 128, cudaMemcpyDeviceToHost));
    if (ae_p_.dbg && cap >= (long long)n + ae_ctas_ * 8)  // per-k-block stamps appended after the task stamps
        PI0B_CUDA(cudaMemcpy(stamps + n * 16, ae_p_.dbg, size_t(ae_ctas_) * 128 * 8, cudaMemcpyDeviceToHost));
}

void Engine::read_checkpoint(const std::string& id, long long inst, float* out, long long rows, long long cols) {
    auto it = ck_.find(std::make_pair(id, int(inst)));
    if (it == ck_.end()) throw EngineError(PI0B_E_STATE, "no checkpoint for " + id + "[" + std::to_string(inst) + "]");
    const Checkpoint& ck = it->second;
    if (rows != ck.rows || cols != ck.cols) throw EngineError(PI0B_E_INVALID, "checkpoint shape mismatch");
    PI0B_CUDA(cudaStreamSynchronize(stream_));
    const size_t n = size_t(rows) * cols;
    if (ck.bf16) {
        std::vector<__nv_bfloat16> tmp(n);
        PI0B_CUDA(cudaMemcpy(tmp.data(), ck.dev, n * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < n; ++i) out[i] = __bfloat162float(tmp[i]);
    } else {
        PI0B_CUDA(cudaMemcpy(out, ck.dev, n * 4, cudaMemcpyDeviceToHost));
    }
}

}  // namespace pi0b

// ====================================================================== C-ABI

using pi0b::Engine;
using pi0b::EngineError;

// ---------------------------------------------------------------------- streaming runtime
// the full-streaming execution the reference simulates
// (proj/src/streamsim.cpp:280-602): camera frames -> prefix into one of two KV buffers (two engines over
// one weight arena, double-buffered KV) on one stream, action-expert ticks on the KV chosen by the policy on the other
// engine's stream, a fixed-rate trajectory buffer whose commit cursor follows wall time, and the
// reference's loop metrics (measure_loops, streamsim.cpp:520-602) on what actually ran.
namespace pi0b {
namespace {
double pctl(std::vector<double> v, double q) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    return v[std::min(v.size() - 1, size_t(q * double(v.size())))];
}
}  // namespace

void stream_run(const pi0b_model_config& cfg, uint64_t seed, const pi0b_stream_options& o, double seconds,
                pi0b_stream_report& rep) {
    using clk = std::chrono::steady_clock;
    if (o.frame_rate <= 0 || o.ae_rate <= 0 || o.trajectory_rate <= 0 || o.camera_latency < 0 || seconds <= 0)
        throw EngineError(PI0B_E_INVALID, "stream options");
    // The ticks' megakernel leaves `prefix_sms` SMs to the concurrent prefix (measured at 1440 Hz
    // 1-step ticks, 2 views: 128 of 148 SMs -> prefix p50 19.8 -> 11.3 ms, slow loop 89 -> 81 ms,
    // the megakernel itself 0.4% slower; its gated-FFN phase needs 2 x 64 CTAs, so no fewer)
    int sms = 148;
    {
        cudaDeviceProp prop;
        PI0B_CUDA(cudaGetDeviceProperties(&prop, o.device));
        sms = prop.multiProcessorCount;
    }
    const int reserve = o.prefix_sms == 0 ? 20 : std::max(0, o.prefix_sms);
    const int ffn_ctas = 2 * (2 * cfg.ae_mlp / 128);
    const int ae_ctas = reserve > 0 ? std::max(std::min(sms, ffn_ctas), (sms - reserve) & ~1) : 0;
    pi0b_engine_options eo{o.device, 1, 0, 0, 0, ae_ctas};
    // two KV buffers over ONE weight arena: the second engine borrows the first one's weights
    std::unique_ptr<Engine> eng[2];
    eng[0] = std::make_unique<Engine>(cfg, eo);
    eng[1] = std::make_unique<Engine>(cfg, eo, eng[0].get());
    eng[0]->gen_weights(seed);
    const int P = cfg.prompt_tokens, C = cfg.chunk_len, A = cfg.ae_action_dim;
    std::mt19937_64 rng(seed * 7919u + 1);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    auto rnd = [&](size_t n) {
        std::vector<double> v(n);
        for (double& x : v) x = U(rng);
        return v;
    };
    const std::vector<double> patches = rnd(size_t(cfg.views) * cfg.tokens_per_view * cfg.ve_patch_in);
    const std::vector<double> prompt = rnd(size_t(std::max(P, 1)) * cfg.llm_width);
    std::vector<double> state = rnd(size_t(cfg.ae_state_dim)), noise = rnd(size_t(C) * A);
    for (auto& e : eng) {  // CUDA-graph capture of both parts, outside the measured run
        e->prefix_async(patches.data(), P ? prompt.data() : nullptr);
        PI0B_CUDA(cudaStreamSynchronize(e->stream()));
        e->tick_async(state.data(), noise.data());
        PI0B_CUDA(cudaStreamSynchronize(e->stream()));
    }
    const double period = 1.0 / o.frame_rate, tick_dt = 1.0 / o.ae_rate, slot_dt = 1.0 / o.trajectory_rate;
    struct Op {
        int kind = 0;  // 0 idle, 1 prefix, 2 tick
        int64_t id = -1, kv = -1;
        double t_issue = 0, t_sensor = 0;
    } op[2];
    // completed frame whose KV each engine holds (kNoKv: none).  Engine 1 starts with a pre-roll
    // frame (-1, the warm-up prefix above) so control ticks run from t = 0, as in the reference's
    // simulator (its AE passes start with the run); loop metrics exclude frames < 1.
    constexpr int64_t kNoKv = -2;
    int64_t kv_frame[2] = {kNoKv, -1};
    int64_t next_frame = 0, sticky = kNoKv;
    double next_tick = 0.0;
    struct Slot {
        int64_t writer = -1, kv = -1;
        double sensor = 0;
    };
    std::map<int64_t, Slot> traj;
    std::vector<double> prefix_ms, tick_ms;
    int64_t frames = 0, ticks = 0, overwritten = 0, tick_id = 0;
    const auto t0 = clk::now();
    auto now = [&]() { return std::chrono::duration<double>(clk::now() - t0).count(); };
    auto newest = [&]() {  // engine holding the newest completed KV that is not being rewritten
        int best = -1;
        for (int e = 0; e < 2; ++e)
            if (kv_frame[e] != kNoKv && op[e].kind != 1 && (best < 0 || kv_frame[e] > kv_frame[best])) best = e;
        return best;
    };
    bool stop = false;
    while (true) {
        const double t = now();
        if (t >= seconds) stop = true;
        // completions
        for (int e = 0; e < 2; ++e) {
            if (op[e].kind == 0 || !eng[e]->idle()) continue;
            const double tc = now();
            if (op[e].kind == 1) {
                kv_frame[e] = op[e].id;
                ++frames;
                prefix_ms.push_back((tc - op[e].t_issue) * 1e3);
            } else {
                const double* act = eng[e]->tick_result();
                (void)act;  // the chunk's values are what the robot would execute; timing is the metric
                ++ticks;
                tick_ms.push_back((tc - op[e].t_issue) * 1e3);
                // write window: the chunk into the first C uncommitted slots (slot time > now)
                const int64_t first = int64_t(std::floor(tc / slot_dt)) + 1;
                for (int64_t k = first; k < first + C; ++k) {
                    auto it = traj.find(k);
                    if (it != traj.end()) ++overwritten;
                    traj[k] = Slot{op[e].id, op[e].kv, op[e].t_sensor};
                }
            }
            op[e] = Op{};
        }
        if (stop) {
            if (op[0].kind == 0 && op[1].kind == 0) break;
            continue;
        }
        // camera: frame f captured at f * period, available camera_latency frames later, prefix on
        // engine f % 2 (the other engine keeps serving the previous KV)
        if (double(next_frame + o.camera_latency) * period <= t) {
            const int e = int(next_frame % 2);
            if (op[e].kind == 0) {
                if (o.kv_policy == 1) sticky = newest() >= 0 ? kv_frame[newest()] : kNoKv;
                eng[e]->prefix_async(patches.data(), P ? prompt.data() : nullptr);
                op[e] = Op{1, next_frame, -1, now(), 0};
                kv_frame[e] = kNoKv;
                ++next_frame;
            }
        }
        // control tick: the freshest sensor sample (2 kHz grid) and fresh noise on the chosen KV
        if (t >= next_tick) {
            int e = newest();
            if (o.kv_policy == 1 && sticky != kNoKv) {  // frame_sticky: keep the KV chosen at the last VLM start
                e = -1;
                for (int k = 0; k < 2; ++k)
                    if (kv_frame[k] == sticky && op[k].kind != 1) e = k;
                if (e < 0) e = newest();
            }
            if (e >= 0 && op[e].kind == 0) {
                for (double& x : state) x = U(rng);
                for (double& x : noise) x = U(rng);
                const double ts = std::floor(t * 2000.0) / 2000.0;
                eng[e]->tick_async(state.data(), noise.data());
                op[e] = Op{2, tick_id++, kv_frame[e], now(), ts};
                // fixed-rate schedule: a tick issued late does not shift the ones after it (the
                // average rate stays at the target); only a stall of more than 4 periods is
                // dropped instead of being caught up in a burst
                next_tick += tick_dt;
                if (next_tick < t - 4.0 * tick_dt) next_tick = t;
            }
        }
    }
    const double t_end = now();
    // loop metrics on the committed slots (slot time <= end of run)
    std::map<int64_t, double> quick;  // tick -> first committed slot time - sensor time
    std::map<int64_t, double> slow;   // frame -> first committed slot time using its KV - capture time
    int64_t committed = 0;
    for (const auto& [k, sl] : traj) {
        const double ts = double(k) * slot_dt;
        if (ts > t_end) break;
        ++committed;
        if (!quick.count(sl.writer)) quick[sl.writer] = ts - sl.sensor;
        if (sl.kv >= 1 && !slow.count(sl.kv)) slow[sl.kv] = ts - double(sl.kv) * period;  // frame 0 = cold start
    }
    auto stats = [](const std::map<int64_t, double>& m, double& mean, double& best, double& worst, int64_t& n) {
        n = int64_t(m.size());
        mean = 0, best = 1e30, worst = 0;
        for (const auto& kv : m) {
            mean += kv.second;
            best = std::min(best, kv.second);
            worst = std::max(worst, kv.second);
        }
        mean = n ? mean / double(n) * 1e3 : 0.0;
        best = n ? best * 1e3 : 0.0;
        worst *= 1e3;
    };
    rep = pi0b_stream_report{};
    rep.seconds = t_end;
    rep.frames = frames;
    rep.ticks = ticks;
    rep.vlm_per_s = double(frames) / t_end;
    rep.ae_per_s = double(ticks) / t_end;
    stats(quick, rep.quick_mean_ms, rep.quick_best_ms, rep.quick_worst_ms, rep.quick_count);
    stats(slow, rep.slow_mean_ms, rep.slow_best_ms, rep.slow_worst_ms, rep.slow_count);
    rep.prefix_p50_ms = pctl(prefix_ms, 0.5);
    rep.tick_p50_ms = pctl(tick_ms, 0.5);
    rep.tick_p99_ms = pctl(tick_ms, 0.99);
    rep.committed_slots = committed;
    rep.overwritten_slots = overwritten;
}

}  // namespace pi0b

struct pi0b_engine {
    std::unique_ptr<Engine> impl;
};

#define PI0B_TRY(body)                                                         \
    try {                                                                      \
        body;                                                                  \
        return PI0B_OK;                                                        \
    } catch (const EngineError& e) {                                           \
        return pi0b::fail(e);                                                  \
    } catch (const std::exception& e) {                                        \
        return pi0b::fail(EngineError(PI0B_E_INVALID, e.what()));              \
    }

extern "C" {

void pi0b_default_config(pi0b_model_config* c) {
    *c = pi0b_model_config{2, 0, 256, 63, 10, 27, 1152, 16, 72, 4304, 588, 18, 2048, 8, 256, 1, 16384,
                           18, 1024, 8, 256, 1, 4096, 32, 32};
}

int pi0b_engine_create_shared(const pi0b_model_config* cfg, const pi0b_engine_options* opt, pi0b_engine* donor,
                              pi0b_engine** out) {
    if (!cfg || !out || !donor) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    pi0b_engine_options o{0, 1, 0, 0, 0, 0};
    if (opt) o = *opt;
    PI0B_TRY({
        auto* e = new pi0b_engine;
        try {
            e->impl.reset(new Engine(*cfg, o, donor->impl.get()));
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    })
}

int pi0b_engine_create(const pi0b_model_config* cfg, const pi0b_engine_options* opt, pi0b_engine** out) {
    if (!cfg || !out) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    pi0b_engine_options o{0, 1, 0, 0, 0, 0};
    if (opt) o = *opt;
    PI0B_TRY({
        auto* e = new pi0b_engine;
        try {
            e->impl.reset(new Engine(*cfg, o));
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    })
}

void pi0b_engine_destroy(pi0b_engine* e) { delete e; }

int pi0b_engine_gen_weights(pi0b_engine* e, uint64_t seed) { PI0B_TRY(e->impl->gen_weights(seed)) }

int pi0b_engine_set_weight(pi0b_engine* e, const char* id, int64_t inst, const double* w, int64_t k,
                           int64_t m, const double* bias, int64_t blen) {
    PI0B_TRY(e->impl->set_weight(id, inst, w, k, m, bias, blen))
}

int pi0b_engine_set_bias_table(pi0b_engine* e, const char* id, const double* t, int64_t rows, int64_t m) {
    PI0B_TRY(e->impl->set_bias_table(id, t, rows, m))
}

int pi0b_engine_run(pi0b_engine* e, const double* patches, const double* state, const double* noise,
                    const double* prompt, double* out) {
    PI0B_TRY({
        e->impl->upload_inputs(patches, state, noise, prompt, 0);
        e->impl->launch(0, e->impl->stream());
        e->impl->fetch_actions(out);
    })
}

int pi0b_engine_run_images(pi0b_engine* e, const double* images, int height, int width, const double* state,
                           const double* noise, const double* prompt, double* out) {
    PI0B_TRY({
        e->impl->upload_images(images, height, width);
        e->impl->upload_inputs(nullptr, state, noise, prompt, 3);
        e->impl->launch(0, e->impl->stream());
        e->impl->fetch_actions(out);
    })
}

int pi0b_image_patches(const double* images, int views, int height, int width, int channels, int side, int patch,
                       double* patches, void* stream) {
    return int(pi0b::launch_image_patches(images, views, height, width, channels, side, patch, patches,
                                          static_cast<cudaStream_t>(stream)));
}

int pi0b_rope_table_host(int positions, int head_dim, float* out) {
    if (!out || positions <= 0 || head_dim <= 0 || head_dim % 2)
        return pi0b::fail(EngineError(PI0B_E_INVALID, "rope table: positions > 0, even head_dim"));
    pi0b::rope_table_f32(positions, head_dim, out);
    return PI0B_OK;
}

int pi0b_f64_to_bf16_host(const double* src, long long n, uint16_t* dst) {
    if ((!src || !dst) && n > 0) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    for (long long i = 0; i < n; ++i) dst[i] = pi0b::host_bf16(src[i]);
    return PI0B_OK;
}

int pi0b_stream_run(const pi0b_model_config* cfg, uint64_t seed, const pi0b_stream_options* opt, double seconds,
                    pi0b_stream_report* report) {
    if (!cfg || !opt || !report) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    PI0B_TRY(pi0b::stream_run(*cfg, seed, *opt, seconds, *report))
}

int pi0b_engine_run_prefix(pi0b_engine* e, const double* patches, const double* prompt) {
    PI0B_TRY({
        e->impl->upload_inputs(patches, nullptr, nullptr, prompt, 1);
        e->impl->launch(1, e->impl->stream());
        PI0B_CUDA(cudaStreamSynchronize(e->impl->stream()));
    })
}

int pi0b_engine_run_action(pi0b_engine* e, const double* state, const double* noise, double* out) {
    PI0B_TRY({
        e->impl->upload_inputs(nullptr, state, noise, nullptr, 2);
        e->impl->launch(2, e->impl->stream());
        e->impl->fetch_actions(out);
    })
}

int pi0b_engine_ve_buffers(pi0b_engine* e, pi0b_ve_buffers* out) {
    if (!out) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    PI0B_TRY(e->impl->ve_buffers(out))
}

int pi0b_engine_set_ve_peers(pi0b_engine* e, const pi0b_ve_buffers* peers, int n) {
    PI0B_TRY(e->impl->set_ve_peers(peers, n))
}

int pi0b_ipc_export(const void* dptr, uint8_t* handle64) {
    if (!dptr || !handle64) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    cudaIpcMemHandle_t h;
    PI0B_TRY({
        PI0B_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
        std::memcpy(handle64, &h, 64);
    })
}

int pi0b_ipc_open(const uint8_t* handle64, void** dptr) {
    if (!dptr || !handle64) return pi0b::fail(EngineError(PI0B_E_INVALID, "null argument"));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    PI0B_TRY(PI0B_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess)))
}

int pi0b_ipc_close(void* dptr) { PI0B_TRY(PI0B_CUDA(cudaIpcCloseMemHandle(dptr))) }

int pi0b_engine_replay(pi0b_engine* e, int part, void* stream) {
    PI0B_TRY({
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : e->impl->stream();
        e->impl->launch(part, st);
    })
}

int pi0b_engine_sync(pi0b_engine* e) { PI0B_TRY(PI0B_CUDA(cudaStreamSynchronize(e->impl->stream()))) }

int pi0b_engine_kernel_count(pi0b_engine* e, int part) { return e->impl->kernel_count(part); }

int pi0b_engine_read_checkpoint(pi0b_engine* e, const char* id, int64_t inst, float* out, int64_t rows,
                                int64_t cols) {
    PI0B_TRY(e->impl->read_checkpoint(id, inst, out, rows, cols))
}

int pi0b_engine_describe(pi0b_engine* e, char* buf, int64_t cap) {
    PI0B_TRY({
        const std::string s = e->impl->describe();
        if (int64_t(s.size()) + 1 > cap) throw EngineError(PI0B_E_INVALID, "describe buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    })
}

int pi0b_engine_time_node(pi0b_engine* e, const char* id, int reps, double* ms_per_launch, int* launches) {
    PI0B_TRY(*ms_per_launch = e->impl->time_node(id, reps, launches))
}

// Debug: the megakernel task table and its per-task globaltimer stamps (PI0B_AE_TRACE=1).
int pi0b_engine_ae_trace(pi0b_engine* e, void* tasks, unsigned long long* stamps, int64_t cap, int* ctas, int* stride) {
    PI0B_TRY(e->impl->ae_trace(tasks, stamps, cap, ctas, stride))
}

const char* pi0b_last_error(void) { return pi0b::g_last_error.c_str(); }

}  // extern "C"
