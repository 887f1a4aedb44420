// TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
//
// extern "C" access to the UNMODIFIED reference implementation compiled from
// /root/reference/proj/src (see oracle/Makefile) so that Python tests can call it
// through ctypes:
//   * the inference API: gen_weights / gen_inputs / evaluate (proj/src/evaluate.cpp:38-85,
//     365-370) on build_pi0_graph(cfg) (proj/src/builder.cpp:197-367);
//   * per-node-instance values through a probe Slice node appended to the graph (the
//     reference's own Slice semantics, proj/src/evaluate.cpp:340-346), so hidden states
//     of any layer can be compared;
//   * the numerics primitives the reference tests pin (proj/src/tensor.cpp).
#include "pi0b.h"
#include "rtvla/builder.hpp"
#include "rtvla/evaluate.hpp"
#include "rtvla/passes.hpp"

#include <cstring>
#include <vector>
#include <exception>
#include <string>

namespace {

thread_local std::string g_err;

rtvla::ModelConfig to_cfg(const pi0b_model_config* c) {
    rtvla::ModelConfig m;
    m.views = c->views;
    m.prompt_tokens = c->prompt_tokens;
    m.tokens_per_view = c->tokens_per_view;
    m.chunk_len = c->chunk_len;
    m.flow_steps = c->flow_steps;
    m.ve = rtvla::VisionConfig{c->ve_layers, c->ve_width, c->ve_heads, c->ve_head_dim, c->ve_mlp,
                               c->ve_patch_in};
    m.llm = rtvla::LlmConfig{c->llm_layers, c->llm_width, c->llm_q_heads, c->llm_head_dim,
                             c->llm_kv_heads, c->llm_mlp};
    m.ae = rtvla::ActionConfig{c->ae_layers,  c->ae_width, c->ae_q_heads,    c->ae_head_dim,
                               c->ae_kv_heads, c->ae_mlp,  c->ae_action_dim, c->ae_state_dim};
    return m;
}

void from_cfg(const rtvla::ModelConfig& m, pi0b_model_config* c) {
    *c = pi0b_model_config{m.views,        m.prompt_tokens,  m.tokens_per_view, m.chunk_len,
                           m.flow_steps,   m.ve.layers,      m.ve.width,        m.ve.heads,
                           m.ve.head_dim,  m.ve.mlp,         m.ve.patch_in,     m.llm.layers,
                           m.llm.width,    m.llm.q_heads,    m.llm.head_dim,    m.llm.kv_heads,
                           m.llm.mlp,      m.ae.layers,      m.ae.width,        m.ae.q_heads,
                           m.ae.head_dim,  m.ae.kv_heads,    m.ae.mlp,          m.ae.action_dim,
                           m.ae.state_dim};
}

void copy_out(const rtvla::Tensor& t, double* out, int64_t cap) {
    if (int64_t(t.data.size()) > cap) throw std::runtime_error("output buffer too small");
    std::memcpy(out, t.data.data(), t.data.size() * sizeof(double));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_default_config(pi0b_model_config* c) { from_cfg(rtvla::default_config(), c); }
void ref_tiny_config(pi0b_model_config* c) { from_cfg(rtvla::tiny_config(), c); }

int64_t ref_count_gemm_instances(const pi0b_model_config* c) {
    return rtvla::count_gemm_instances(rtvla::build_pi0_graph(to_cfg(c)));
}

// Node ids of build_pi0_graph(cfg), '\n'-separated, with "id kind repeat n k m".
int ref_graph_listing(const pi0b_model_config* c, char* buf, int64_t cap) {
    return guarded([&] {
        const rtvla::Graph g = rtvla::build_pi0_graph(to_cfg(c));
        std::string s;
        for (const auto& n : g.nodes)
            s += n.id + " " + rtvla::to_string(n.kind) + " " + std::to_string(n.repeat) + " " +
                 std::to_string(n.shape.n) + " " + std::to_string(n.shape.k) + " " +
                 std::to_string(n.shape.m) + "\n";
        if (int64_t(s.size()) + 1 > cap) throw std::runtime_error("listing buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

int ref_gen_inputs(const pi0b_model_config* c, uint64_t seed, double* patches, double* state,
                   double* noise, double* prompt) {
    return guarded([&] {
        const rtvla::Graph g = rtvla::build_pi0_graph(to_cfg(c));
        const rtvla::Inputs in = rtvla::gen_inputs(g, seed);
        const auto& t = in.by_source;
        copy_out(t.at("patches"), patches, int64_t(t.at("patches").data.size()));
        copy_out(t.at("state"), state, int64_t(t.at("state").data.size()));
        copy_out(t.at("noise"), noise, int64_t(t.at("noise").data.size()));
        if (c->prompt_tokens > 0) copy_out(t.at("prompt"), prompt, int64_t(t.at("prompt").data.size()));
    });
}

// WeightSet of one node instance via gen_weights on a one-node graph: the reference
// seeds every tensor from (seed, node id, instance, role), so this equals the slice
// of the full gen_weights store (proj/include/rtvla/evaluate.hpp:36-38).
int ref_gen_node_weight(const pi0b_model_config* c, uint64_t seed, const char* node, int64_t inst,
                        double* w, double* bias, double* table) {
    return guarded([&] {
        const rtvla::Graph g = rtvla::build_pi0_graph(to_cfg(c));
        const rtvla::Node* n = g.find(node);
        if (!n) throw std::runtime_error(std::string("no node ") + node);
        rtvla::Graph one;
        one.config = g.config;
        one.nodes.push_back(*n);
        const rtvla::WeightStore ws = rtvla::gen_weights(one, seed);
        const rtvla::WeightSet& set = ws.by_node.at(node);
        if (w) copy_out(set.w.at(size_t(inst)), w, int64_t(set.w.at(size_t(inst)).data.size()));
        if (bias && !set.bias.empty())
            std::memcpy(bias, set.bias.at(size_t(inst)).data(), set.bias.at(size_t(inst)).size() * 8);
        if (table && n->has_bias_table) copy_out(set.bias_table, table, int64_t(set.bias_table.data.size()));
    });
}

// rtvla::evaluate on gen_weights(g, wseed) / gen_inputs(g, iseed); out = [chunk, action_dim].
int ref_evaluate(const pi0b_model_config* c, uint64_t wseed, uint64_t iseed, double* out) {
    return guarded([&] {
        const rtvla::Graph g = rtvla::build_pi0_graph(to_cfg(c));
        const rtvla::WeightStore w = rtvla::gen_weights(g, wseed);
        const rtvla::Inputs x = rtvla::gen_inputs(g, iseed);
        const rtvla::Tensor y = rtvla::evaluate(g, w, x);
        copy_out(y, out, int64_t(y.data.size()));
    });
}

// Value of node `node` instance `inst`: a probe Slice node with repeat inst+1 reads the
// node plainly, so evaluating the probe's last instance returns node[inst].
int ref_evaluate_node(const pi0b_model_config* c, uint64_t wseed, uint64_t iseed, const char* node,
                      int64_t inst, double* out, int64_t cap, int64_t* rows, int64_t* cols) {
    return guarded([&] {
        rtvla::Graph g = rtvla::build_pi0_graph(to_cfg(c));
        const rtvla::WeightStore w = rtvla::gen_weights(g, wseed);
        const rtvla::Inputs x = rtvla::gen_inputs(g, iseed);
        const rtvla::Node* n = g.find(node);
        if (!n) throw std::runtime_error(std::string("no node ") + node);
        const auto shape = rtvla::node_output_shape(g, *n);
        rtvla::Node probe;
        probe.id = "probe";
        probe.kind = rtvla::NodeKind::Slice;
        probe.stage = n->stage;
        probe.repeat = inst + 1;
        probe.lo = 0;
        probe.hi = shape.first;
        probe.inputs.push_back(rtvla::parse_input_ref(node));
        g.nodes.push_back(probe);
        g.output = "probe";
        const rtvla::Tensor y = rtvla::evaluate(g, w, x);
        copy_out(y, out, cap);
        *rows = y.rows;
        *cols = y.cols;
    });
}

// ---- persistent context: graph + WeightStore + Inputs built once, evaluate() timed alone
struct RefCtx {
    rtvla::Graph g;
    rtvla::WeightStore w;
    rtvla::Inputs x;
};
void* ref_ctx_create(const pi0b_model_config* c, uint64_t wseed, uint64_t iseed) {
    try {
        auto* ctx = new RefCtx;
        ctx->g = rtvla::build_pi0_graph(to_cfg(c));
        ctx->w = rtvla::gen_weights(ctx->g, wseed);
        ctx->x = rtvla::gen_inputs(ctx->g, iseed);
        return ctx;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int ref_ctx_evaluate(void* h, double* out) {
    return guarded([&] {
        auto* ctx = static_cast<RefCtx*>(h);
        const rtvla::Tensor y = rtvla::evaluate(ctx->g, ctx->w, ctx->x);
        std::memcpy(out, y.data.data(), y.data.size() * 8);
    });
}
void ref_ctx_destroy(void* h) { delete static_cast<RefCtx*>(h); }

// ---- numerics primitives (proj/src/tensor.cpp)
uint64_t ref_seed_hash(uint64_t seed, const char* label, uint64_t a, uint64_t b) {
    return rtvla::seed_hash(seed, label, a, b);
}
void ref_rng_stream(uint64_t seed, int64_t n, uint64_t* out) {
    rtvla::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_random_tensor(int64_t rows, int64_t cols, double lo, double hi, uint64_t seed, double* out) {
    const rtvla::Tensor t = rtvla::random_tensor(rows, cols, lo, hi, seed);
    std::memcpy(out, t.data.data(), t.data.size() * 8);
}
double ref_gelu(double x) { return rtvla::gelu(x); }
double ref_silu(double x) { return rtvla::silu(x); }
int ref_matmul(const double* a, int64_t n, int64_t k, const double* b, int64_t m, double* out) {
    return guarded([&] {
        rtvla::Tensor ta(n, k), tb(k, m);
        std::memcpy(ta.data.data(), a, size_t(n * k) * 8);
        std::memcpy(tb.data.data(), b, size_t(k * m) * 8);
        const rtvla::Tensor y = rtvla::matmul(ta, tb);
        std::memcpy(out, y.data.data(), size_t(n * m) * 8);
    });
}
int ref_rms_scales(const double* x, int64_t rows, int64_t cols, double eps, double* out) {
    return guarded([&] {
        rtvla::Tensor t(rows, cols);
        std::memcpy(t.data.data(), x, size_t(rows * cols) * 8);
        const rtvla::Tensor s = rtvla::rms_scales(t, eps);
        std::memcpy(out, s.data.data(), size_t(rows) * 8);
    });
}
int ref_bilinear_resize(const double* img, int64_t h, int64_t w, int channels, int out_h, int out_w, double* out) {
    return guarded([&] {
        rtvla::Tensor t(h, w * channels);
        std::memcpy(t.data.data(), img, size_t(h * w * channels) * 8);
        const rtvla::Tensor r = rtvla::bilinear_resize(t, channels, out_h, out_w);
        std::memcpy(out, r.data.data(), r.data.size() * 8);
    });
}
int ref_softmax_rows(const double* x, int64_t rows, int64_t cols, double* out) {
    return guarded([&] {
        rtvla::Tensor t(rows, cols);
        std::memcpy(t.data.data(), x, size_t(rows * cols) * 8);
        const rtvla::Tensor s = rtvla::softmax_rows(t);
        std::memcpy(out, s.data.data(), size_t(rows * cols) * 8);
    });
}
int ref_rope(const double* x, int64_t rows, int64_t cols, int head_dim, int pos_offset, double* out) {
    return guarded([&] {
        rtvla::Tensor t(rows, cols);
        std::memcpy(t.data.data(), x, size_t(rows * cols) * 8);
        const auto table = rtvla::make_rope_table(pos_offset + int(rows), head_dim, 10000.0);
        std::vector<int> pos(static_cast<size_t>(rows));
        for (int64_t r = 0; r < rows; ++r) pos[size_t(r)] = pos_offset + int(r);
        const rtvla::Tensor y = rtvla::rope_apply(t, table, pos);
        std::memcpy(out, y.data.data(), size_t(rows * cols) * 8);
    });
}
void ref_rope_table(int positions, int head_dim, double* cos_out, double* sin_out) {
    const auto t = rtvla::make_rope_table(positions, head_dim, 10000.0);
    std::memcpy(cos_out, t.cos_t.data.data(), t.cos_t.data.size() * 8);
    std::memcpy(sin_out, t.sin_t.data.data(), t.sin_t.data.size() * 8);
}
void ref_time_embedding(int step, int dim, int flow_steps, double* out) {
    const auto e = rtvla::time_embedding(step, dim, flow_steps);
    std::memcpy(out, e.data(), e.size() * 8);
}
double ref_max_rel_deviation(const double* a, const double* b, int64_t n) {
    rtvla::Tensor ta(1, n), tb(1, n);
    std::memcpy(ta.data.data(), a, size_t(n) * 8);
    std::memcpy(tb.data.data(), b, size_t(n) * 8);
    return rtvla::max_rel_deviation(ta, tb);
}

}  // extern "C"
