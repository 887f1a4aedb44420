// pi0b_rtvla.hpp — drop-in C++ replacement of the reference's inference API for the pi0 path,
// header-only, over the C-ABI in pi0b.h.
//
// Reference interface replaced (proj/include/rtvla/evaluate.hpp:38-44):
//     rtvla::Tensor rtvla::evaluate(const Graph&, const WeightStore&, const Inputs&);
// for graphs built by rtvla::build_pi0_graph (proj/src/builder.cpp:197-367).  Compile against the
// reference headers (-I<reference>/proj/include) and link libpi0b.so:
//
//     #include "rtvla/builder.hpp"
//     #include "pi0b_rtvla.hpp"
//     rtvla::Graph g = rtvla::build_pi0_graph(rtvla::default_config());
//     rtvla::WeightStore w = rtvla::gen_weights(g, 1);
//     rtvla::Inputs x = rtvla::gen_inputs(g, 1);
//     rtvla::Tensor a = pi0b::evaluate(g, w, x);          // was: rtvla::evaluate(g, w, x)
//
//     pi0b::Engine eng(g, w);                              // repeated inference: build once
//     rtvla::Tensor a2 = eng.run(x);                       // one CUDA-graph replay
//     eng.run_prefix(x); rtvla::Tensor a3 = eng.run_action(x);  // streaming split
//
//     // unfused checkpoint layout (rtvla::build_pi0_graph_naive): fused on the host by the
//     // reference's own passes + weight rules, then run on the GPU
//     rtvla::Tensor a4 = pi0b::evaluate_naive(gn, wn, xn);
//
// Error convention follows the reference (proj/src/evaluate.cpp:98-99,265,352-354): malformed
// graphs / shapes throw rtvla::ShapeError, non-finite outputs rtvla::NumericError, device errors
// std::runtime_error.  There is no CPU fallback: without an sm_100 GPU the Engine constructor
// throws.
#pragma once

#include "pi0b.h"
#include "rtvla/builder.hpp"
#include "rtvla/evaluate.hpp"
#include "rtvla/graph.hpp"
#include "rtvla/passes.hpp"
#include "rtvla/tensor.hpp"

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>

namespace pi0b {

inline void check(int rc, const char* what) {
    if (rc == PI0B_OK) return;
    const std::string msg = std::string(what) + ": " + pi0b_last_error();
    if (rc == PI0B_E_INVALID || rc == PI0B_E_UNSUPPORTED) throw rtvla::ShapeError(msg);
    if (rc == PI0B_E_NUMERIC) throw rtvla::NumericError(msg);
    throw std::runtime_error(msg);
}

// rtvla::ModelConfig (proj/include/rtvla/graph.hpp:114-160) -> the C-ABI mirror.
inline pi0b_model_config to_c(const rtvla::ModelConfig& c) {
    pi0b_model_config o{};
    o.views = c.views;
    o.prompt_tokens = c.prompt_tokens;
    o.tokens_per_view = c.tokens_per_view;
    o.chunk_len = c.chunk_len;
    o.flow_steps = c.flow_steps;
    o.ve_layers = c.ve.layers;
    o.ve_width = c.ve.width;
    o.ve_heads = c.ve.heads;
    o.ve_head_dim = c.ve.head_dim;
    o.ve_mlp = c.ve.mlp;
    o.ve_patch_in = c.ve.patch_in;
    o.llm_layers = c.llm.layers;
    o.llm_width = c.llm.width;
    o.llm_q_heads = c.llm.q_heads;
    o.llm_head_dim = c.llm.head_dim;
    o.llm_kv_heads = c.llm.kv_heads;
    o.llm_mlp = c.llm.mlp;
    o.ae_layers = c.ae.layers;
    o.ae_width = c.ae.width;
    o.ae_q_heads = c.ae.q_heads;
    o.ae_head_dim = c.ae.head_dim;
    o.ae_kv_heads = c.ae.kv_heads;
    o.ae_mlp = c.ae.mlp;
    o.ae_action_dim = c.ae.action_dim;
    o.ae_state_dim = c.ae.state_dim;
    return o;
}

struct EngineOptions {
    int device = 0;
    bool use_cuda_graph = true;
};

class Engine {
public:
    // Weights from a reference WeightStore (fp64 -> bf16 once, on the device).
    Engine(const rtvla::Graph& g, const rtvla::WeightStore& w, EngineOptions opt = {}) : cfg_(g.config) {
        create(g, opt);
        // isomorphism is positional and ignores node names (a graph fused from the naive one
        // by the reference's passes keeps the naive names): weights go to the engine under the
        // name of the node at the same position in build_pi0_graph
        const rtvla::Graph canon = rtvla::build_pi0_graph(g.config);
        for (size_t k = 0; k < g.nodes.size(); ++k) {
            const rtvla::Node& n = g.nodes[k];
            const std::string& cid = canon.nodes[k].id;
            auto it = w.by_node.find(n.id);
            if (it == w.by_node.end()) continue;
            const rtvla::WeightSet& ws = it->second;
            // instances beyond the node's own count (e.g. carried over from an unpruned graph by
            // rtvla::apply_weight_rules) are never read by the reference either
            const size_t n_inst = std::min(ws.w.size(), size_t(std::max<int64_t>(0, n.weight_instances())));
            for (size_t i = 0; i < n_inst; ++i) {
                const rtvla::Tensor& t = ws.w[i];
                const bool has_bias = i < ws.bias.size() && !ws.bias[i].empty();
                check(pi0b_engine_set_weight(h_.get(), cid.c_str(), int64_t(i), t.data.data(), t.rows, t.cols,
                                             has_bias ? ws.bias[i].data() : nullptr,
                                             has_bias ? int64_t(ws.bias[i].size()) : 0),
                      ("set_weight " + cid).c_str());
            }
            if (ws.bias_table.rows > 0)
                check(pi0b_engine_set_bias_table(h_.get(), cid.c_str(), ws.bias_table.data.data(), ws.bias_table.rows,
                                                 ws.bias_table.cols),
                      ("set_bias_table " + cid).c_str());
        }
    }
    // Weights generated on the device: bit-identical bf16 rounding of rtvla::gen_weights(g, seed).
    Engine(const rtvla::Graph& g, uint64_t seed, EngineOptions opt = {}) : cfg_(g.config) {
        create(g, opt);
        check(pi0b_engine_gen_weights(h_.get(), seed), "gen_weights");
    }

    rtvla::Tensor run(const rtvla::Inputs& x) {
        rtvla::Tensor out(cfg_.chunk_len, cfg_.ae.action_dim);
        check(pi0b_engine_run(h_.get(), src(x, "patches"), src(x, "state"), src(x, "noise"),
                              cfg_.prompt_tokens > 0 ? src(x, "prompt") : nullptr, out.data.data()),
              "run");
        return out;
    }
    void run_prefix(const rtvla::Inputs& x) {
        check(pi0b_engine_run_prefix(h_.get(), src(x, "patches"), cfg_.prompt_tokens > 0 ? src(x, "prompt") : nullptr),
              "run_prefix");
    }
    rtvla::Tensor run_action(const rtvla::Inputs& x) {
        rtvla::Tensor out(cfg_.chunk_len, cfg_.ae.action_dim);
        check(pi0b_engine_run_action(h_.get(), src(x, "state"), src(x, "noise"), out.data.data()), "run_action");
        return out;
    }
    pi0b_engine* handle() const { return h_.get(); }

private:
    void create(const rtvla::Graph& g, const EngineOptions& opt) {
        // Only the fused pi0 topology is implemented: reject anything else, as SURVEY 8(b) asks
        // (proj/src/passes.cpp:910-963 graphs_isomorphic).
        std::string why;
        if (!rtvla::graphs_isomorphic(g, rtvla::build_pi0_graph(g.config), &why))
            throw rtvla::ShapeError("pi0b: graph is not build_pi0_graph(config): " + why);
        const pi0b_model_config c = to_c(cfg_);
        pi0b_engine_options o{opt.device, opt.use_cuda_graph ? 1 : 0, 0};
        pi0b_engine* e = nullptr;
        check(pi0b_engine_create(&c, &o, &e), "engine_create");
        h_.reset(e);
    }
    static const double* src(const rtvla::Inputs& x, const char* id) {
        auto it = x.by_source.find(id);
        if (it == x.by_source.end()) throw rtvla::NumericError(std::string("missing input '") + id + "'");
        return it->second.data.data();
    }
    struct Del {
        void operator()(pi0b_engine* e) const { pi0b_engine_destroy(e); }
    };
    rtvla::ModelConfig cfg_;
    std::unique_ptr<pi0b_engine, Del> h_;
};

// Same signature and semantics as rtvla::evaluate for build_pi0_graph graphs.  Builds an engine
// per call (uploads and repacks every weight); keep an Engine for repeated inference.
inline rtvla::Tensor evaluate(const rtvla::Graph& g, const rtvla::WeightStore& w, const rtvla::Inputs& x) {
    Engine e(g, w);
    return e.run(x);
}

// Unfused graphs: rtvla::build_pi0_graph_naive — one node per framework-level op
// (separate q/k/v, RMSNorm with gamma, the action time-embedding MLP) — which is what a real pi0
// checkpoint maps onto.  The reference's own rewrite passes, in its standard order
// (rtvla::pass_registry, proj/src/passes.cpp), and weight rules (rtvla::apply_weight_rules,
// proj/src/passes.cpp:692-790: PremultiplyDiag gamma into W, ConcatCols q|k|v and up|gate,
// ComposeTimeFold of the time MLP into the ae.action_proj bias table) turn the naive graph and
// its WeightStore into the fused graph and weights once on the host; the engine runs those.
struct Fused {
    rtvla::Graph graph;
    rtvla::WeightStore weights;
};
inline Fused fuse(const rtvla::Graph& naive, const rtvla::WeightStore& w) {
    Fused f{naive, w};
    for (const auto& [name, fn] : rtvla::pass_registry()) {
        rtvla::PassResult r = fn(f.graph);
        f.weights = rtvla::apply_weight_rules(f.graph, r.graph, r.rules, f.weights, f.graph.config.flow_steps);
        f.graph = std::move(r.graph);
        (void)name;
    }
    return f;
}
// rtvla::evaluate on a naive-graph WeightStore (same Inputs: the source nodes are shared).
inline rtvla::Tensor evaluate_naive(const rtvla::Graph& naive, const rtvla::WeightStore& w, const rtvla::Inputs& x) {
    const Fused f = fuse(naive, w);
    return pi0b::evaluate(f.graph, f.weights, x);
}

}  // namespace pi0b
