// Drop-in demonstration (test infrastructure): the reference's own C++ types and generators
// (rtvla::build_pi0_graph / gen_weights / gen_inputs, compiled read-only from /root/reference into
// oracle/_ref/librtvla_ref.so) feed pi0b::evaluate / pi0b::Engine (include/pi0b_rtvla.hpp over
// libpi0b.so), and the result is compared with rtvla::evaluate (the fp64 oracle) on a reduced-width
// twin with full-scale head geometry (paper_2510_26742_b200/config.py mid_config).
//   usage: pi0b_rtvla_demo [views] [prompt]      exit 0 when max |gpu - fp64| < 0.05
//          pi0b_rtvla_demo naive [views] [prompt] : the unfused graph (build_pi0_graph_naive) and its
//          WeightStore through pi0b::evaluate_naive (host-side fusion by the reference's passes)
//          vs rtvla::evaluate on the naive graph
#include "pi0b_rtvla.hpp"
#include "rtvla/builder.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

int main(int argc, char** argv) {
    const bool naive = argc > 1 && std::string(argv[1]) == "naive";
    if (naive) {
        --argc;
        ++argv;
    }
    rtvla::ModelConfig c;
    c.views = argc > 1 ? std::atoi(argv[1]) : 1;
    c.prompt_tokens = argc > 2 ? std::atoi(argv[2]) : 0;
    c.tokens_per_view = 256;
    c.chunk_len = 63;
    c.flow_steps = 3;
    c.ve = rtvla::VisionConfig{2, 288, 4, 72, 1076, 588};
    c.llm = rtvla::LlmConfig{3, 512, 2, 256, 1, 1024};
    c.ae = rtvla::ActionConfig{2, 256, 2, 256, 1, 512, 32, 32};
    if (naive) {
        const rtvla::Graph gn = rtvla::build_pi0_graph_naive(c);
        const rtvla::WeightStore wn = rtvla::gen_weights(gn, 1);
        const rtvla::Inputs xn = rtvla::gen_inputs(gn, 1);
        const rtvla::Tensor refn = rtvla::evaluate(gn, wn, xn);
        try {
            const rtvla::Tensor an = pi0b::evaluate_naive(gn, wn, xn);
            double d = 0, rms = 0;
            for (size_t i = 0; i < refn.data.size(); ++i) {
                d = std::fmax(d, std::fabs(an.data[i] - refn.data[i]));
                rms += refn.data[i] * refn.data[i];
            }
            std::printf("pi0b::evaluate_naive vs rtvla::evaluate(naive graph) max|d| = %.3e (rms %.3f)\n", d,
                        std::sqrt(rms / refn.data.size()));
            return d < 0.05 ? 0 : 1;
        } catch (const std::exception& e) {
            std::printf("pi0b error: %s\n", e.what());
            return 2;
        }
    }
    const rtvla::Graph g = rtvla::build_pi0_graph(c);
    const rtvla::WeightStore w = rtvla::gen_weights(g, 1);
    const rtvla::Inputs x = rtvla::gen_inputs(g, 1);
    const rtvla::Tensor ref = rtvla::evaluate(g, w, x);
    try {
        const rtvla::Tensor a = pi0b::evaluate(g, w, x);  // drop-in: same signature
        pi0b::Engine eng(g, 1);                           // device-side gen_weights(g, 1)
        const rtvla::Tensor b = eng.run(x);
        eng.run_prefix(x);
        const rtvla::Tensor s = eng.run_action(x);
        double da = 0, db = 0, ds = 0;
        for (size_t i = 0; i < ref.data.size(); ++i) {
            da = std::fmax(da, std::fabs(a.data[i] - ref.data[i]));
            db = std::fmax(db, std::fabs(b.data[i] - ref.data[i]));
            ds = std::fmax(ds, std::fabs(s.data[i] - b.data[i]));
        }
        std::printf("pi0b::evaluate vs rtvla::evaluate max|d| = %.3e; Engine(seed) %.3e; run_prefix+run_action vs run %.3e\n",
                    da, db, ds);
        bool threw = false;
        try {
            rtvla::Graph bad = g;
            bad.nodes.pop_back();
            pi0b::Engine e2(bad, 1);
        } catch (const rtvla::ShapeError&) {
            threw = true;
        }
        std::printf("non-pi0 graph rejected with rtvla::ShapeError: %s\n", threw ? "yes" : "no");
        // a WeightStore missing a node / an instance / the bias table is refused with
        // rtvla::NumericError, as rtvla::evaluate refuses it (proj/src/evaluate.cpp:96-99)
        int refused = 0;
        for (int v = 0; v < 3; ++v) {
            rtvla::WeightStore bad = w;
            if (v == 0) bad.by_node.erase("ae.ffn");
            if (v == 1) bad.by_node.at("llm.down").w.pop_back();
            if (v == 2) bad.by_node.at("ae.action_proj").bias_table = rtvla::Tensor();
            try {
                pi0b::Engine e3(g, bad);
            } catch (const rtvla::NumericError&) {
                ++refused;
            }
        }
        std::printf("incomplete WeightStores refused with rtvla::NumericError: %d of 3\n", refused);
        return (da < 0.05 && db < 0.05 && ds < 0.02 && threw && refused == 3) ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("pi0b error: %s\n", e.what());
        return 2;
    }
}
