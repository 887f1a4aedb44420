// Test/measurement infrastructure (not product): runs the reference's own full-streaming event
// simulator (proj/src/streamsim.cpp, compiled unmodified) on B200-measured stream times, so the
// paper's streaming analysis can be redone with this engine's numbers.
//
//   streamsim_driver vlm_s ae_s rate horizon policy [t_a t_b measured]...
//     vlm_s / ae_s  : measured prefix time per frame / action-expert time per pass (seconds)
//     rate          : target AE pass rate (Hz, e.g. 480)
//     policy        : most_recent | frame_sticky (rtvla::KvPolicy)
//     t_a t_b meas  : concurrent-run points for rtvla::calibrate_eta (streamsim.hpp:35-45); none ->
//                     the reference's built-in 4090 calibration
// Prints one JSON object: the fitted eta, the reference's closed-form frame makespan and the
// rtvla::measure_loops report (streamsim.hpp:166-205) of the simulated trace.
#include "rtvla/streamsim.hpp"

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

int main(int argc, char** argv) {
    if (argc < 6 || (argc - 6) % 3 != 0) {
        std::fprintf(stderr, "usage: %s vlm_s ae_s rate horizon policy [t_a t_b measured]...\n", argv[0]);
        return 2;
    }
    rtvla::SimConfig cfg;
    cfg.vlm_time = std::atof(argv[1]);
    cfg.ae_time = std::atof(argv[2]);
    cfg.ae_rate_target = std::atof(argv[3]);
    cfg.horizon = std::atof(argv[4]);
    cfg.kv_policy = rtvla::kv_policy_from(argv[5]);
    std::vector<rtvla::EtaPoint> pts;
    for (int i = 6; i + 2 < argc; i += 3) pts.push_back({std::atof(argv[i]), std::atof(argv[i + 1]), std::atof(argv[i + 2])});
    rtvla::EtaFit fit{cfg.overlap_eta, false};
    if (!pts.empty()) fit = rtvla::calibrate_eta(pts);
    cfg.overlap_eta = fit.eta;
    cfg.validate();
    const rtvla::StreamTrace tr = rtvla::simulate(cfg);
    const rtvla::LoopReport rep = rtvla::measure_loops(tr);
    const int passes = int(cfg.ae_rate_target / cfg.frame_rate + 0.5);
    std::printf("{\"eta\": %.6f, \"eta_clamped\": %s, \"eta_points\": %d, \"sim_config\": %s, "
                "\"closed_form_frame_makespan_s\": %.9f, \"passes_per_frame\": %d, \"loops\": %s}\n",
                fit.eta, fit.clamped ? "true" : "false", int(pts.size()), rtvla::serialize_sim_config(cfg).c_str(),
                rtvla::concurrent_makespan(cfg.vlm_time, passes * cfg.ae_time, cfg.overlap_eta), passes,
                rtvla::loop_report_json(rep).c_str());
    return 0;
}
