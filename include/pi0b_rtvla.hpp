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
//     // engine's own weight rules (fuse_naive), then run on the GPU
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
#include "rtvla/passes.hpp"  // graphs_isomorphic only
#include "rtvla/tensor.hpp"

#include <algorithm>
#include <map>
#include <memory>
#include <vector>
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
    // Weights from a reference WeightStore (fp64 -> bf16 once, on the device).  Every weight
    // instance, bias and bias table the graph needs must be present: a missing one throws
    // rtvla::NumericError("no weights for node ...") as the reference's evaluator does
    // (proj/src/evaluate.cpp:96-99) instead of running on unloaded memory.
    Engine(const rtvla::Graph& g, const rtvla::WeightStore& w, EngineOptions opt = {}) : cfg_(g.config) {
        create(g, opt);
        // isomorphism is positional and ignores node names: weights go to the engine under the
        // name of the node at the same position in build_pi0_graph
        const rtvla::Graph canon = rtvla::build_pi0_graph(g.config);
        for (size_t k = 0; k < g.nodes.size(); ++k) {
            const rtvla::Node& n = g.nodes[k];
            const rtvla::Node& cn = canon.nodes[k];
            const int64_t need = std::max<int64_t>(0, cn.weight_instances());
            if (need == 0 && !cn.has_bias_table) continue;
            auto it = w.by_node.find(n.id);
            if (it == w.by_node.end()) throw rtvla::NumericError("no weights for node " + n.id);
            const rtvla::WeightSet& ws = it->second;
            // instances beyond the node's own count (e.g. carried over from an unpruned graph)
            // are never read by the reference either
            if (int64_t(ws.w.size()) < need)
                throw rtvla::NumericError("node " + n.id + ": " + std::to_string(ws.w.size()) +
                                          " weight instances, the graph reads " + std::to_string(need));
            for (int64_t i = 0; i < need; ++i) {
                const rtvla::Tensor& t = ws.w[size_t(i)];
                const bool has_bias = size_t(i) < ws.bias.size() && !ws.bias[size_t(i)].empty();
                if (cn.has_bias && !has_bias)
                    throw rtvla::NumericError("node " + n.id + ": no bias for instance " + std::to_string(i));
                check(pi0b_engine_set_weight(h_.get(), cn.id.c_str(), i, t.data.data(), t.rows, t.cols,
                                             cn.has_bias ? ws.bias[size_t(i)].data() : nullptr,
                                             cn.has_bias ? int64_t(ws.bias[size_t(i)].size()) : 0),
                      ("set_weight " + cn.id).c_str());
            }
            if (cn.has_bias_table) {
                if (ws.bias_table.rows == 0) throw rtvla::NumericError("node " + n.id + ": no bias_table");
                check(pi0b_engine_set_bias_table(h_.get(), cn.id.c_str(), ws.bias_table.data.data(), ws.bias_table.rows,
                                                 ws.bias_table.cols),
                      ("set_bias_table " + cn.id).c_str());
            }
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
        pi0b_engine_options o{opt.device, opt.use_cuda_graph ? 1 : 0, 0, 0, 0, 0};
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

// Unfused graphs: rtvla::build_pi0_graph_naive (proj/src/builder.cpp:369-541) —
// one node per framework-level op (separate q/k/v and up/gate, RMSNorm with gamma, the action
// time-embedding MLP) — which is what a real pi0 checkpoint maps onto.  fuse_naive() turns its
// WeightStore into the fused graph's with the repo's own weight rules (libpi0b, csrc/naive.cu:
// PremultiplyDiag, ComposeTimeFold + time_embedding; ConcatCols is the column copy below), which
// reproduce rtvla::apply_weight_rules (proj/src/passes.cpp:692-790) bit for bit
// (tests/test_adaptor_cpu.py, oracle/naive_fuse_check.cpp).  The reference is used only to check the naive topology
// (rtvla::graphs_isomorphic) and to name the fused graph (rtvla::build_pi0_graph).
struct Fused {
    rtvla::Graph graph;
    rtvla::WeightStore weights;
};

namespace detail {

inline const rtvla::WeightSet& naive_set(const rtvla::WeightStore& w, const std::map<std::string, std::string>& id,
                                         const std::string& canon_id) {
    const std::string& nid = id.at(canon_id);
    auto it = w.by_node.find(nid);
    if (it == w.by_node.end()) throw rtvla::NumericError("no weights for node " + nid);
    return it->second;
}

// gamma of instance wi of an RMSNorm (shared when the norm has one instance), passes.cpp:709-714
inline const std::vector<double>& gamma_of(const rtvla::WeightSet& norm, size_t wi, size_t insts, const std::string& id) {
    if (norm.gamma.size() != insts && norm.gamma.size() != 1)
        throw rtvla::NumericError("premultiply: instance counts disagree for " + id);
    return norm.gamma[norm.gamma.size() == 1 ? 0 : wi];
}

// fused[c] = [gamma (.) W_part0 | gamma (.) W_part1 | ...] per instance, biases concatenated
inline rtvla::WeightSet concat_scaled(const rtvla::WeightStore& w, const std::map<std::string, std::string>& id,
                                      const std::vector<std::string>& parts, const char* norm, bool bias,
                                      int64_t insts) {
    const rtvla::WeightSet* g = norm ? &naive_set(w, id, norm) : nullptr;
    std::vector<const rtvla::WeightSet*> ps;
    for (const auto& p : parts) ps.push_back(&naive_set(w, id, p));
    rtvla::WeightSet out;
    for (int64_t wi = 0; wi < insts; ++wi) {
        int64_t k = -1, m = 0;
        for (size_t q = 0; q < ps.size(); ++q) {
            if (int64_t(ps[q]->w.size()) <= wi)
                throw rtvla::NumericError("node " + id.at(parts[q]) + ": missing weight instance " + std::to_string(wi));
            const rtvla::Tensor& t = ps[q]->w[size_t(wi)];
            if (k >= 0 && t.rows != k) throw rtvla::ShapeError("concat: row counts differ for " + id.at(parts[q]));
            k = t.rows;
            m += t.cols;
        }
        rtvla::Tensor f(k, m);
        std::vector<double> b;
        int64_t off = 0;
        for (size_t q = 0; q < ps.size(); ++q) {
            const rtvla::Tensor& t = ps[q]->w[size_t(wi)];
            rtvla::Tensor part = t;
            if (g) {
                const auto& gm = gamma_of(*g, size_t(wi), ps[q]->w.size(), id.at(parts[q]));
                if (int64_t(gm.size()) != t.rows) throw rtvla::NumericError("premultiply: scale length mismatch for " + id.at(parts[q]));
                check(pi0b_premultiply_rows(part.data.data(), part.rows, part.cols, gm.data()), "premultiply_rows");
            }
            for (int64_t r = 0; r < k; ++r)
                std::copy(part.data.begin() + r * t.cols, part.data.begin() + (r + 1) * t.cols,
                          f.data.begin() + r * m + off);
            if (bias) {
                if (ps[q]->bias.size() <= size_t(wi)) throw rtvla::NumericError("node " + id.at(parts[q]) + ": missing bias");
                const auto& pb = ps[q]->bias[size_t(wi)];
                b.insert(b.end(), pb.begin(), pb.end());
            }
            off += t.cols;
        }
        out.w.push_back(std::move(f));
        if (bias) out.bias.push_back(std::move(b));
    }
    return out;
}

}  // namespace detail

inline Fused fuse_naive(const rtvla::Graph& naive, const rtvla::WeightStore& w) {
    const rtvla::ModelConfig& c = naive.config;
    const rtvla::Graph canon_naive = rtvla::build_pi0_graph_naive(c);
    std::string why;
    if (!rtvla::graphs_isomorphic(naive, canon_naive, &why))
        throw rtvla::ShapeError("pi0b: graph is not build_pi0_graph_naive(config): " + why);
    std::map<std::string, std::string> id;  // canonical naive id -> the caller's node id (positional)
    for (size_t k = 0; k < naive.nodes.size(); ++k) id[canon_naive.nodes[k].id] = naive.nodes[k].id;

    Fused f{rtvla::build_pi0_graph(c), {}};
    auto insts = [&](const char* fused_id) {
        const rtvla::Node* n = f.graph.find(fused_id);
        if (!n) throw rtvla::ShapeError(std::string("pi0b: fused graph lacks ") + fused_id);
        return std::max<int64_t>(0, n->weight_instances());
    };
    using detail::concat_scaled;
    struct Rule {
        const char* fused;
        std::vector<std::string> parts;
        const char* norm;  // RMSNorm whose gamma is absorbed, or nullptr
    };
    const Rule rules[] = {
        {"ve.embed", {"ve.embed"}, nullptr},
        {"ve.qkv", {"ve.q", "ve.k", "ve.v"}, "ve.ln1"},
        {"ve.proj", {"ve.proj"}, nullptr},
        {"ve.fc1", {"ve.fc1"}, "ve.ln2"},
        {"ve.fc2", {"ve.fc2"}, nullptr},
        {"llm.proj_in", {"llm.proj_in"}, "ve.ln_out"},
        {"llm.qkv", {"llm.q", "llm.k", "llm.v"}, "llm.ln1"},
        {"llm.proj", {"llm.proj"}, nullptr},
        {"llm.ffn", {"llm.up", "llm.gate"}, "llm.ln2"},
        {"llm.down", {"llm.down"}, nullptr},
        {"ae.state_proj", {"ae.state_proj"}, nullptr},
        {"ae.action_out", {"ae.mlp_out"}, nullptr},
        {"ae.qkv", {"ae.q", "ae.k", "ae.v"}, "ae.ln1"},
        {"ae.proj", {"ae.proj"}, nullptr},
        {"ae.ffn", {"ae.up", "ae.gate"}, "ae.ln2"},
        {"ae.down", {"ae.down"}, nullptr},
        {"ae.head", {"ae.head"}, "ae.ln_out"},
    };
    for (const Rule& r : rules)
        f.weights.by_node[r.fused] = concat_scaled(w, id, r.parts, r.norm, f.graph.find(r.fused)->has_bias, insts(r.fused));

    // ae.act_in (+ time embedding) -> ae.mlp_in -> SiLU  ==>  ae.action_proj + bias table
    const rtvla::WeightSet& act = detail::naive_set(w, id, "ae.act_in");
    const rtvla::WeightSet& mix = detail::naive_set(w, id, "ae.mlp_in");
    const rtvla::Node* time = canon_naive.find("ae.time");
    if (act.w.empty() || mix.w.empty() || act.bias.empty() || mix.bias.empty() || !time)
        throw rtvla::NumericError("no weights for the action time MLP (ae.act_in / ae.mlp_in)");
    const rtvla::Tensor& wa = act.w[0];
    const rtvla::Tensor& wm = mix.w[0];
    const int64_t d_t = time->cols;
    if (wm.rows != d_t + wa.cols) throw rtvla::ShapeError("ae.mlp_in rows != time dim + ae.act_in cols");
    rtvla::WeightSet ap;
    ap.w.emplace_back(wa.rows, wm.cols);
    ap.bias_table = rtvla::Tensor(c.flow_steps, wm.cols);
    check(pi0b_fold_time_mlp(wa.data.data(), wa.rows, wa.cols, act.bias[0].data(), wm.data.data(), d_t, wm.cols,
                             mix.bias[0].data(), c.flow_steps, ap.w[0].data.data(), ap.bias_table.data.data()),
          "fold_time_mlp");
    f.weights.by_node["ae.action_proj"] = std::move(ap);
    return f;
}

// rtvla::evaluate on a naive-graph WeightStore (same Inputs: the source nodes are shared).
inline rtvla::Tensor evaluate_naive(const rtvla::Graph& naive, const rtvla::WeightStore& w, const rtvla::Inputs& x) {
    const Fused f = fuse_naive(naive, w);
    return pi0b::evaluate(f.graph, f.weights, x);
}

}  // namespace pi0b
