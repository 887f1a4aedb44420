// Host-side weight rules for unfused (naive-graph) checkpoints — SURVEY.md 8(f) f1 / 8(a) a17.
//
// A real pi0 checkpoint maps onto rtvla::build_pi0_graph_naive (proj/src/builder.cpp:369-541):
// separate q/k/v and up/gate matrices, RMSNorm gammas, and the action time-embedding MLP
// (ae.act_in -> concat(time, .) -> ae.mlp_in -> SiLU).  The fused graph the engine runs
// (build_pi0_graph) needs those weights transformed exactly as the reference's
// rtvla::apply_weight_rules does (proj/src/passes.cpp:692-790):
//   PremultiplyDiag  W[r, c] *= gamma[r]                                    (:706-721)
//   ConcatCols       [W_q | W_k | W_v], [W_up | W_gate], biases likewise    (:723-752)
//   ComposeTimeFold  W = W_act . W_mix[d_t:, :]; bias_table[s, c] =
//                    b_mix[c] + sum_j emb_s[j] W_mix[j, c] + sum_r b_act[r] W_mix[d_t + r, c]
//                    with emb_s = time_embedding(s, d_t, flow_steps)        (:754-785)
// These are the repo's own implementations of those rules (the concatenation itself is a
// plain copy done by the C++ adaptor, include/pi0b_rtvla.hpp fuse_naive).  Every operation
// follows the reference's order — i-p-j matmul with its zero skip, sequential sums,
// separately rounded multiply and add — so the results are bit-identical to the reference
// (tests/test_adaptor_cpu.py, oracle/naive_fuse_check.cpp).  Host code only: no device is needed.
#include "../../include/pi0b.h"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// one fp64 multiply-add, never contracted into an FMA (the reference's baseline-x86 build
// rounds the product and the sum separately)
#if defined(__GNUC__) && !defined(__clang__)
__attribute__((optimize("fp-contract=off")))
#endif
inline double mul_add(double acc, double a, double b) {
    volatile double p = a * b;
    return acc + p;
}

}  // namespace

extern "C" {

// rtvla::time_embedding (proj/src/evaluate.cpp:23-36): tau = step / flow_steps, frequencies
// 0.25 .. 250 geometric over dim/2, [sin | cos].
int pi0b_time_embedding(int step, int dim, int flow_steps, double* out) {
    if (dim % 2 != 0 || dim <= 0 || !out) return PI0B_E_INVALID;
    const int half = dim / 2;
    const double tau = flow_steps > 0 ? double(step) / flow_steps : 0.0;
    const double f_lo = 0.25, f_hi = 250.0;
    for (int j = 0; j < half; ++j) {
        const double t = half > 1 ? double(j) / (half - 1) : 0.0;
        const double f = f_lo * std::pow(f_hi / f_lo, t);
        out[j] = std::sin(tau * f);
        out[half + j] = std::cos(tau * f);
    }
    return PI0B_OK;
}

// PremultiplyDiag: w[k, m] row r scaled by gamma[r], in place.
int pi0b_premultiply_rows(double* w, int64_t k, int64_t m, const double* gamma) {
    if (!w || !gamma || k < 0 || m < 0) return PI0B_E_INVALID;
    for (int64_t r = 0; r < k; ++r) {
        const double g = gamma[r];
        double* row = w + r * m;
        for (int64_t c = 0; c < m; ++c) row[c] *= g;
    }
    return PI0B_OK;
}

// ComposeTimeFold of the action time MLP into ae.action_proj:
//   w_act [act, width], b_act [width]; w_mix [t_dim + width, mix_cols], b_mix [mix_cols]
//   -> w_out [act, mix_cols] = w_act . w_mix[t_dim:, :]   (rtvla::matmul order, zero skip)
//      table_out [flow_steps, mix_cols]                   (the per-step bias table)
int pi0b_fold_time_mlp(const double* w_act, int64_t act, int64_t width, const double* b_act, const double* w_mix,
                       int64_t t_dim, int64_t mix_cols, const double* b_mix, int flow_steps, double* w_out,
                       double* table_out) {
    if (!w_act || !b_act || !w_mix || !b_mix || !w_out || !table_out || act <= 0 || width <= 0 || t_dim <= 0 ||
        mix_cols <= 0 || flow_steps <= 0 || t_dim % 2 != 0)
        return PI0B_E_INVALID;
    const double* wm_act = w_mix + t_dim * mix_cols;  // rows t_dim.. of the mix matrix
    std::memset(w_out, 0, size_t(act * mix_cols) * sizeof(double));
    for (int64_t i = 0; i < act; ++i) {
        double* yrow = w_out + i * mix_cols;
        for (int64_t p = 0; p < width; ++p) {
            const double av = w_act[i * width + p];
            if (av == 0.0) continue;
            const double* brow = wm_act + p * mix_cols;
            for (int64_t j = 0; j < mix_cols; ++j) yrow[j] = mul_add(yrow[j], av, brow[j]);
        }
    }
    std::vector<double> emb(static_cast<size_t>(t_dim));
    for (int s = 0; s < flow_steps; ++s) {
        pi0b_time_embedding(s, int(t_dim), flow_steps, emb.data());
        for (int64_t c = 0; c < mix_cols; ++c) {
            double v = b_mix[c];
            for (int64_t j = 0; j < t_dim; ++j) v = mul_add(v, emb[size_t(j)], w_mix[j * mix_cols + c]);
            for (int64_t r = 0; r < width; ++r) v = mul_add(v, b_act[r], wm_act[r * mix_cols + c]);
            table_out[s * mix_cols + c] = v;
        }
    }
    return PI0B_OK;
}

}  // extern "C"
