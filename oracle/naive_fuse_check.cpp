// CPU check (test infrastructure) of pi0b::fuse (include/pi0b_rtvla.hpp): the naive pi0 graph
// (rtvla::build_pi0_graph_naive) + its WeightStore, fused by the reference's own passes and weight
// rules, give a graph isomorphic to rtvla::build_pi0_graph and the same fp64 outputs as evaluating
// the naive graph directly (reference tolerance 1e-9, proj/include/rtvla/passes.hpp:80).  No GPU
// involved: only the header's host-side fuse() runs.   usage: naive_fuse_check [views] [prompt]
#include "pi0b_rtvla.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
    rtvla::ModelConfig c = rtvla::tiny_config();
    c.views = argc > 1 ? std::atoi(argv[1]) : 1;
    c.prompt_tokens = argc > 2 ? std::atoi(argv[2]) : 0;
    const rtvla::Graph gn = rtvla::build_pi0_graph_naive(c);
    const rtvla::WeightStore wn = rtvla::gen_weights(gn, 1);
    const rtvla::Inputs x = rtvla::gen_inputs(gn, 1);
    const pi0b::Fused f = pi0b::fuse(gn, wn);
    std::string why;
    const bool iso = rtvla::graphs_isomorphic(f.graph, rtvla::build_pi0_graph(c), &why);
    const rtvla::Tensor a = rtvla::evaluate(gn, wn, x);
    const rtvla::Tensor b = rtvla::evaluate(f.graph, f.weights, x);
    const double dev = rtvla::max_rel_deviation(b, a);
    std::printf("fused graph isomorphic to build_pi0_graph: %s %s; max_rel_deviation(fused, naive) = %.3e\n",
                iso ? "yes" : "no", why.c_str(), dev);
    return iso && dev < 1e-9 ? 0 : 1;
}
