// Measurement infrastructure (not product): the reference's own roofline / cost model and report
// (proj/src/costmodel.cpp, report.cpp, compiled unmodified) run on the fused pi0 graph with a B200
// HardwareSpec and a calibration table of this engine's measured per-node times -- the B200
// version of the paper's Table 2 (proj/include/rtvla/costmodel.hpp:83-105).
//
//   analyze_driver views prompt hw.json                  -> JSON list of the graph's cost rows
//   analyze_driver views prompt hw.json calib.json [fmt] -> rendered report (markdown|csv|json)
#include "rtvla/builder.hpp"
#include "rtvla/costmodel.hpp"
#include "rtvla/report.hpp"

#include <cstdio>
#include <cstdlib>
#include <string>

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s views prompt hw.json [calib.json [format]]\n", argv[0]);
        return 2;
    }
    rtvla::ModelConfig cfg = rtvla::default_config();
    cfg.views = std::atoi(argv[1]);
    cfg.prompt_tokens = std::atoi(argv[2]);
    const rtvla::Graph g = rtvla::build_pi0_graph(cfg);
    const rtvla::HardwareSpec hw = rtvla::load_hardware(argv[3]);
    if (argc < 5) {
        const rtvla::Breakdown b = rtvla::analyze(g, hw, "none", nullptr);
        std::printf("[");
        for (size_t i = 0; i < b.rows.size(); ++i)
            std::printf("%s{\"node\": \"%s\", \"shape\": \"%s\", \"repeat\": %lld, \"roofline_ms\": %.6f}", i ? ", " : "",
                        b.rows[i].node_id.c_str(), b.rows[i].shape_str.c_str(), (long long)b.rows[i].times,
                        b.rows[i].roofline_ms);
        std::printf("]\n");
        return 0;
    }
    const rtvla::CalibrationTable cal = rtvla::load_calibration(argv[4]);
    const rtvla::Breakdown b = rtvla::analyze(g, hw, "none", &cal);
    std::printf("%s", rtvla::render_report(b, argc > 5 ? argv[5] : "markdown").c_str());
    return 0;
}
