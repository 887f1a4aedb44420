// CPU check (test infrastructure) of pi0b::fuse_naive (include/pi0b_rtvla.hpp + libpi0b's host
// weight rules, csrc/naive.cu): the naive pi0 graph (rtvla::build_pi0_graph_naive) and its
// WeightStore, fused by the ENGINE's own rules, against the reference's own pipeline
// (rtvla::pass_registry + rtvla::apply_weight_rules, proj/src/passes.cpp:665-790):
//   1. every fused weight instance, bias and the ae.action_proj bias table are BITWISE equal;
//   2. rtvla::evaluate on the engine-fused graph+weights equals the reference-fused one bitwise
//      and the naive graph within the reference's own tolerance (1e-9, passes.hpp:80).
// No GPU involved (only libpi0b's host functions run).
//   usage: naive_fuse_check [tiny|mid] [views] [prompt]
#include "pi0b_rtvla.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

static bool same(const rtvla::Tensor& a, const rtvla::Tensor& b) {
    return a.rows == b.rows && a.cols == b.cols &&
           std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(double)) == 0;
}

int main(int argc, char** argv) {
    const std::string which = argc > 1 ? argv[1] : "tiny";
    rtvla::ModelConfig c = rtvla::tiny_config();
    if (which == "mid") {  // full-scale head geometry (paper_2510_26742_b200/config.py mid_config)
        c.tokens_per_view = 256;
        c.chunk_len = 63;
        c.flow_steps = 3;
        c.ve = rtvla::VisionConfig{2, 288, 4, 72, 1076, 588};
        c.llm = rtvla::LlmConfig{3, 512, 2, 256, 1, 1024};
        c.ae = rtvla::ActionConfig{2, 256, 2, 256, 1, 512, 32, 32};
    }
    c.views = argc > 2 ? std::atoi(argv[2]) : 1;
    c.prompt_tokens = argc > 3 ? std::atoi(argv[3]) : 0;
    const rtvla::Graph gn = rtvla::build_pi0_graph_naive(c);
    const rtvla::WeightStore wn = rtvla::gen_weights(gn, 1);
    const rtvla::Inputs x = rtvla::gen_inputs(gn, 1);

    // the reference's pipeline (standard pass order) and weight rules
    rtvla::Graph gr = gn;
    rtvla::WeightStore wr = wn;
    for (const auto& [name, fn] : rtvla::pass_registry()) {
        rtvla::PassResult r = fn(gr);
        wr = rtvla::apply_weight_rules(gr, r.graph, r.rules, wr, c.flow_steps);
        gr = std::move(r.graph);
        (void)name;
    }
    // the engine's
    const pi0b::Fused f = pi0b::fuse_naive(gn, wn);
    std::string why;
    if (!rtvla::graphs_isomorphic(gr, f.graph, &why)) {
        std::printf("reference-fused graph not isomorphic to build_pi0_graph: %s\n", why.c_str());
        return 1;
    }
    long checked = 0, bad = 0;
    for (size_t k = 0; k < gr.nodes.size(); ++k) {
        const rtvla::Node& rn = gr.nodes[k];
        const rtvla::Node& on = f.graph.nodes[k];
        const int64_t need = std::max<int64_t>(0, on.weight_instances());
        if (need == 0 && !on.has_bias_table) continue;
        const rtvla::WeightSet& a = f.weights.by_node.at(on.id);
        const rtvla::WeightSet& b = wr.by_node.at(rn.id);
        for (int64_t i = 0; i < need; ++i) {
            ++checked;
            bool ok = same(a.w.at(size_t(i)), b.w.at(size_t(i)));
            if (on.has_bias) ok = ok && a.bias.at(size_t(i)) == b.bias.at(size_t(i));
            if (!ok) {
                ++bad;
                std::printf("MISMATCH %s[%lld] (reference node %s)\n", on.id.c_str(), (long long)i, rn.id.c_str());
            }
        }
        if (on.has_bias_table) {
            ++checked;
            if (!same(a.bias_table, b.bias_table)) {
                ++bad;
                std::printf("MISMATCH %s bias_table\n", on.id.c_str());
            }
        }
    }
    const rtvla::Tensor yn = rtvla::evaluate(gn, wn, x);
    const rtvla::Tensor yr = rtvla::evaluate(gr, wr, x);
    const rtvla::Tensor yo = rtvla::evaluate(f.graph, f.weights, x);
    const double dev = rtvla::max_rel_deviation(yo, yn);
    const bool bit = same(yo, yr);
    std::printf("%s %dv+%dp: %ld fused weight entries compared, %ld differ; evaluate(engine-fused) == "
                "evaluate(reference-fused) bitwise: %s; max_rel_deviation vs naive graph %.3e\n",
                which.c_str(), c.views, c.prompt_tokens, checked, bad, bit ? "yes" : "no", dev);
    return bad == 0 && bit && dev < 1e-9 ? 0 : 1;
}
