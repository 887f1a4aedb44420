// TEST INFRASTRUCTURE ONLY — the parity checker, never the product.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this library.
//
// pi0_oracle: an independent fp64 CPU restatement of the reference forward pass,
// rtvla::evaluate(build_pi0_graph(cfg), gen_weights(g, seed), x), written as the
// straight-line schedule of SURVEY.md Appendix A instead of the reference's memoised
// graph interpreter, and multi-threaded.  Every output element is produced by exactly
// the reference's sequence of IEEE operations, so the result is bitwise identical:
//   * parameters: SplitMix64 stream per tensor, seed = FNV-1a(seed, node id, instance,
//     role), value lo + (hi-lo)*u                      (proj/src/tensor.cpp:7-47,
//                                                      proj/src/evaluate.cpp:38-85)
//   * matmul: y[i,j] = sum_p a[i,p]*b[p,j] in ascending p, zero a skipped
//                                                      (proj/src/tensor.cpp:49-67)
//     — threads split rows/columns and chunk p, which never reorders one element's sum;
//   * rms scale 1/sqrt(mean(x^2)+eps)                  (proj/src/tensor.cpp:81-93)
//   * epilogue order RmsScale, Bias, Rope, Gelu/GeluGate/SiluBias, Residual
//                                                      (proj/src/evaluate.cpp:160-223)
//   * RoPE half-split pairs, table pow/cos/sin in fp64  (proj/src/tensor.cpp:133-178)
//   * attention per head, scores*(1/sqrt d), max-subtracted softmax, P*V in key order
//                                                      (proj/src/evaluate.cpp:225-252,
//                                                      proj/src/tensor.cpp:95-112)
//   * dataflow / instance algebra of the fused graph   (proj/src/builder.cpp:197-367)
// Bitwise equality with the compiled reference is asserted by tests/test_oracle.py.
#include "pi0b.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct Mat {
    int64_t r = 0, c = 0;
    std::vector<double> d;
    Mat() = default;
    Mat(int64_t rows, int64_t cols) : r(rows), c(cols), d(size_t(rows * cols), 0.0) {}
    double* row(int64_t i) { return d.data() + i * c; }
    const double* row(int64_t i) const { return d.data() + i * c; }
};

int g_threads = 1;

template <typename F>
void par_for(int64_t n, F&& f) {
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(g_threads, n));
    if (nt == 1) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(size_t(nt));
    for (int64_t t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int64_t i = t; i < n; i += nt) f(i);
        });
    for (auto& x : th) x.join();
}

// ------------------------------------------------------------------ parameter streams

uint64_t fnv_seed(uint64_t seed, const std::string& label, uint64_t a, uint64_t b) {
    uint64_t h = 0xcbf29ce484222325ULL;
    auto eat = [&h](uint64_t v) {
        for (int i = 0; i < 64; i += 8) {
            h ^= (v >> i) & 0xffu;
            h *= 0x100000001b3ULL;
        }
    };
    eat(seed);
    for (unsigned char ch : label) {
        h ^= ch;
        h *= 0x100000001b3ULL;
    }
    eat(a);
    eat(b);
    return h;
}

inline uint64_t splitmix_nth(uint64_t seed, uint64_t n) {
    uint64_t z = seed + (n + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline double draw(uint64_t seed, uint64_t n, double lo, double hi) {
    const double u = double(splitmix_nth(seed, n) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

Mat uniform(int64_t rows, int64_t cols, double lo, double hi, uint64_t seed) {
    Mat m(rows, cols);
    par_for((rows * cols + 4095) / 4096, [&](int64_t blk) {
        const int64_t e = std::min<int64_t>(rows * cols, (blk + 1) * 4096);
        for (int64_t n = blk * 4096; n < e; ++n) m.d[size_t(n)] = draw(seed, uint64_t(n), lo, hi);
    });
    return m;
}

enum Role : uint64_t { kW = 1, kB = 2, kTab = 4, kIn = 5 };

double limit_for(int64_t fan_in) { return 1.0 / std::sqrt(double(std::max<int64_t>(1, fan_in))); }

struct Params {
    uint64_t seed;
    Mat w(const std::string& id, int64_t inst, int64_t k, int64_t m) const {
        const double lim = limit_for(k);
        return uniform(k, m, -lim, lim, fnv_seed(seed, id, uint64_t(inst), kW));
    }
    std::vector<double> b(const std::string& id, int64_t inst, int64_t k, int64_t m) const {
        const double lim = limit_for(k);
        return uniform(1, m, -lim, lim, fnv_seed(seed, id, uint64_t(inst), kB)).d;
    }
    Mat table(const std::string& id, int64_t steps, int64_t k, int64_t m) const {
        const double lim = limit_for(k);
        Mat t(steps, m);
        for (int64_t s = 0; s < steps; ++s) {
            Mat r = uniform(1, m, -lim, lim, fnv_seed(seed, id, uint64_t(s), kTab));
            std::copy(r.d.begin(), r.d.end(), t.row(s));
        }
        return t;
    }
};

// ------------------------------------------------------------------ numerics

// y = a * b with the reference's per-element summation order.
Mat matmul(const Mat& a, const Mat& b) {
    if (a.c != b.r) throw std::runtime_error("matmul: inner dims differ");
    Mat y(a.r, b.c);
    const int64_t RB = 8, CB = 256, PB = 256;
    const int64_t nrb = (a.r + RB - 1) / RB, ncb = (b.c + CB - 1) / CB;
    par_for(nrb * ncb, [&](int64_t t) {
        const int64_t i0 = (t / ncb) * RB, i1 = std::min(a.r, i0 + RB);
        const int64_t j0 = (t % ncb) * CB, j1 = std::min(b.c, j0 + CB);
        for (int64_t p0 = 0; p0 < a.c; p0 += PB) {
            const int64_t p1 = std::min(a.c, p0 + PB);
            for (int64_t i = i0; i < i1; ++i) {
                double* yr = y.row(i);
                const double* ar = a.row(i);
                for (int64_t p = p0; p < p1; ++p) {
                    const double av = ar[p];
                    if (av == 0.0) continue;
                    const double* br = b.row(p);
                    for (int64_t j = j0; j < j1; ++j) yr[j] += av * br[j];
                }
            }
        }
    });
    return y;
}

std::vector<double> rms_of(const Mat& x, double eps) {
    std::vector<double> s(size_t(x.r));
    for (int64_t i = 0; i < x.r; ++i) {
        double acc = 0.0;
        const double* xr = x.row(i);
        for (int64_t j = 0; j < x.c; ++j) {
            if (!std::isfinite(xr[j])) throw std::runtime_error("rms: non-finite input");
            acc += xr[j] * xr[j];
        }
        s[size_t(i)] = 1.0 / std::sqrt(acc / double(x.c) + eps);
    }
    return s;
}

double gelu_t(double x) {
    const double k = 0.7978845608028654;
    return 0.5 * x * (1.0 + std::tanh(k * (x + 0.044715 * x * x * x)));
}
double silu_t(double x) { return x / (1.0 + std::exp(-x)); }

void scale_rows(Mat& z, const std::vector<double>& s) {
    for (int64_t i = 0; i < z.r; ++i)
        for (int64_t j = 0; j < z.c; ++j) z.row(i)[j] *= s[size_t(i)];
}
void add_bias(Mat& z, const std::vector<double>& b) {
    for (int64_t i = 0; i < z.r; ++i)
        for (int64_t j = 0; j < z.c; ++j) z.row(i)[j] += b[size_t(j)];
}
void residual(Mat& z, const Mat& base, double scale) {
    for (size_t i = 0; i < z.d.size(); ++i) z.d[i] = base.d[i] + scale * z.d[i];
}

// Rotary embedding on columns [lo, hi) (whole heads of `dh`), rows at positions off+r.
void rotate(Mat& z, int64_t lo, int64_t hi, int dh, int off) {
    const int half = dh / 2;
    const int npos = off + int(z.r);
    std::vector<double> cs(size_t(npos) * half), sn(size_t(npos) * half);
    for (int p = 0; p < npos; ++p)
        for (int j = 0; j < half; ++j) {
            const double f = std::pow(10000.0, -2.0 * double(j) / double(dh));
            const double ang = double(p) * f;
            cs[size_t(p) * half + j] = std::cos(ang);
            sn[size_t(p) * half + j] = std::sin(ang);
        }
    for (int64_t i = 0; i < z.r; ++i) {
        const int p = off + int(i);
        double* zr = z.row(i);
        for (int64_t h0 = lo; h0 < hi; h0 += dh)
            for (int j = 0; j < half; ++j) {
                const double c = cs[size_t(p) * half + j], s = sn[size_t(p) * half + j];
                const double a = zr[h0 + j], b = zr[h0 + j + half];
                zr[h0 + j] = a * c - b * s;
                zr[h0 + j + half] = a * s + b * c;
            }
    }
}

Mat cols_of(const Mat& x, int64_t lo, int64_t hi) {
    Mat o(x.r, hi - lo);
    for (int64_t i = 0; i < x.r; ++i) std::copy(x.row(i) + lo, x.row(i) + hi, o.row(i));
    return o;
}
Mat stack_rows(const Mat& a, const Mat& b) {
    Mat o(a.r + b.r, a.c);
    std::copy(a.d.begin(), a.d.end(), o.d.begin());
    std::copy(b.d.begin(), b.d.end(), o.d.begin() + a.d.size());
    return o;
}

Mat attention(const Mat& q, const Mat& k, const Mat& v, int heads, int kv_heads, int dh) {
    Mat out(q.r, int64_t(heads) * dh);
    const double inv = 1.0 / std::sqrt(double(dh));
    par_for(int64_t(heads) * q.r, [&](int64_t t) {
        const int h = int(t / q.r);
        const int64_t i = t % q.r;
        const int kvh = h % kv_heads;
        std::vector<double> sc(size_t(k.r));
        for (int64_t j = 0; j < k.r; ++j) {
            double acc = 0;
            for (int c = 0; c < dh; ++c) acc += q.row(i)[int64_t(h) * dh + c] * k.row(j)[int64_t(kvh) * dh + c];
            sc[size_t(j)] = acc * inv;
        }
        double mx = -HUGE_VAL;
        for (double x : sc) {
            if (!std::isfinite(x)) throw std::runtime_error("softmax: non-finite input");
            mx = std::max(mx, x);
        }
        double sum = 0.0;
        for (auto& x : sc) {
            x = std::exp(x - mx);
            sum += x;
        }
        for (auto& x : sc) x /= sum;
        for (int c = 0; c < dh; ++c) {
            double acc = 0;
            for (int64_t j = 0; j < k.r; ++j) acc += sc[size_t(j)] * v.row(j)[int64_t(kvh) * dh + c];
            out.row(i)[int64_t(h) * dh + c] = acc;
        }
    });
    return out;
}

// ------------------------------------------------------------------ recording hooks

struct Recorder {
    std::map<std::pair<std::string, int64_t>, std::pair<double*, int64_t>> want;
    void put(const std::string& node, int64_t inst, const Mat& m) {
        auto it = want.find({node, inst});
        if (it == want.end()) return;
        if (int64_t(m.d.size()) > it->second.second) throw std::runtime_error("record buffer too small: " + node);
        std::memcpy(it->second.first, m.d.data(), m.d.size() * 8);
    }
    void put_vec(const std::string& node, int64_t inst, const std::vector<double>& v) {
        Mat m(int64_t(v.size()), 1);
        m.d = v;
        put(node, inst, m);
    }
};

// ------------------------------------------------------------------ the forward

Mat forward(const pi0b_model_config& c, const Params& prm, const Mat& patches, const Mat& state,
            const Mat& noise, const Mat* prompt, Recorder& rec) {
    const double eps = 1e-6;
    const int64_t vw = c.ve_width, lw = c.llm_width, aw = c.ae_width;
    const int64_t lq = int64_t(c.llm_q_heads) * c.llm_head_dim, lkv = int64_t(c.llm_kv_heads) * c.llm_head_dim;
    const int64_t aq = int64_t(c.ae_q_heads) * c.ae_head_dim, akv = int64_t(c.ae_kv_heads) * c.ae_head_dim;
    const int L = c.views * c.tokens_per_view + c.prompt_tokens;
    const int FS = c.flow_steps;

    // ---- vision encoder
    Mat h = matmul(patches, prm.w("ve.embed", 0, c.ve_patch_in, vw));
    add_bias(h, prm.b("ve.embed", 0, c.ve_patch_in, vw));
    rec.put("ve.embed", 0, h);
    for (int i = 0; i < c.ve_layers; ++i) {
        const auto s1 = rms_of(h, eps);
        rec.put_vec("ve.ln1", i, s1);
        Mat qkv = matmul(h, prm.w("ve.qkv", i, vw, 3 * vw));
        scale_rows(qkv, s1);
        add_bias(qkv, prm.b("ve.qkv", i, vw, 3 * vw));
        rec.put("ve.qkv", i, qkv);
        Mat o = attention(cols_of(qkv, 0, vw), cols_of(qkv, vw, 2 * vw), cols_of(qkv, 2 * vw, 3 * vw), c.ve_heads,
                          c.ve_heads, c.ve_head_dim);
        rec.put("ve.attn", i, o);
        Mat p = matmul(o, prm.w("ve.proj", i, vw, vw));
        add_bias(p, prm.b("ve.proj", i, vw, vw));
        residual(p, h, 1.0);
        rec.put("ve.proj", i, p);
        const auto s2 = rms_of(p, eps);
        rec.put_vec("ve.ln2", i, s2);
        Mat f = matmul(p, prm.w("ve.fc1", i, vw, c.ve_mlp));
        scale_rows(f, s2);
        add_bias(f, prm.b("ve.fc1", i, vw, c.ve_mlp));
        for (auto& x : f.d) x = gelu_t(x);
        rec.put("ve.fc1", i, f);
        Mat y = matmul(f, prm.w("ve.fc2", i, c.ve_mlp, vw));
        add_bias(y, prm.b("ve.fc2", i, c.ve_mlp, vw));
        residual(y, p, 1.0);
        rec.put("ve.fc2", i, y);
        h = std::move(y);
    }
    // ---- language model
    const auto so = rms_of(h, eps);
    rec.put_vec("ve.ln_out", 0, so);
    Mat x = matmul(h, prm.w("llm.proj_in", 0, vw, lw));
    scale_rows(x, so);
    add_bias(x, prm.b("llm.proj_in", 0, vw, lw));
    rec.put("llm.proj_in", 0, x);
    if (c.prompt_tokens > 0) {
        x = stack_rows(x, *prompt);
        rec.put("llm.tokens", 0, x);
    }
    std::vector<Mat> kv(size_t(c.llm_layers));
    for (int l = 0; l < c.llm_layers; ++l) {
        const auto s1 = rms_of(x, eps);
        rec.put_vec("llm.ln1", l, s1);
        Mat qkv = matmul(x, prm.w("llm.qkv", l, lw, lq + 2 * lkv));
        scale_rows(qkv, s1);
        rotate(qkv, 0, lq, c.llm_head_dim, 0);
        rotate(qkv, lq, lq + lkv, c.llm_head_dim, 0);
        rec.put("llm.qkv", l, qkv);
        kv[size_t(l)] = qkv;
        if (l == c.llm_layers - 1) break;
        Mat o = attention(cols_of(qkv, 0, lq), cols_of(qkv, lq, lq + lkv), cols_of(qkv, lq + lkv, lq + 2 * lkv),
                          c.llm_q_heads, c.llm_kv_heads, c.llm_head_dim);
        rec.put("llm.attn", l, o);
        Mat p = matmul(o, prm.w("llm.proj", l, lq, lw));
        residual(p, x, 1.0);
        rec.put("llm.proj", l, p);
        const auto s2 = rms_of(p, eps);
        rec.put_vec("llm.ln2", l, s2);
        Mat g = matmul(p, prm.w("llm.ffn", l, lw, 2 * int64_t(c.llm_mlp)));
        scale_rows(g, s2);
        Mat gg(g.r, c.llm_mlp);
        for (int64_t r = 0; r < g.r; ++r)
            for (int64_t j = 0; j < c.llm_mlp; ++j) gg.row(r)[j] = g.row(r)[j] * gelu_t(g.row(r)[c.llm_mlp + j]);
        rec.put("llm.ffn", l, gg);
        Mat y = matmul(gg, prm.w("llm.down", l, c.llm_mlp, lw));
        residual(y, p, 1.0);
        rec.put("llm.down", l, y);
        x = std::move(y);
    }
    // ---- action expert
    Mat st = matmul(state, prm.w("ae.state_proj", 0, c.ae_state_dim, aw));
    add_bias(st, prm.b("ae.state_proj", 0, c.ae_state_dim, aw));
    rec.put("ae.state_proj", 0, st);
    const Mat tab = prm.table("ae.action_proj", FS, c.ae_action_dim, aw);
    const Mat w_ap = prm.w("ae.action_proj", 0, c.ae_action_dim, aw);
    const Mat w_ao = prm.w("ae.action_out", 0, aw, aw);
    const auto b_ao = prm.b("ae.action_out", 0, aw, aw);
    const Mat w_hd = prm.w("ae.head", 0, aw, c.ae_action_dim);
    const auto b_hd = prm.b("ae.head", 0, aw, c.ae_action_dim);
    std::vector<Mat> wq, wp, wf, wd;
    for (int l = 0; l < c.ae_layers; ++l) {
        wq.push_back(prm.w("ae.qkv", l, aw, aq + 2 * akv));
        wp.push_back(prm.w("ae.proj", l, aq, aw));
        wf.push_back(prm.w("ae.ffn", l, aw, 2 * int64_t(c.ae_mlp)));
        wd.push_back(prm.w("ae.down", l, c.ae_mlp, aw));
    }
    Mat a = noise;
    for (int s = 0; s < FS; ++s) {
        Mat z = matmul(a, w_ap);
        for (int64_t r = 0; r < z.r; ++r)
            for (int64_t j = 0; j < z.c; ++j) z.row(r)[j] = silu_t(z.row(r)[j] + tab.row(s)[j]);
        rec.put("ae.action_proj", s, z);
        Mat ao = matmul(z, w_ao);
        add_bias(ao, b_ao);
        rec.put("ae.action_out", s, ao);
        Mat y = stack_rows(st, ao);
        rec.put("ae.suffix", s, y);
        for (int l = 0; l < c.ae_layers; ++l) {
            const int64_t i = int64_t(s) * c.ae_layers + l;
            const auto s1 = rms_of(y, eps);
            rec.put_vec("ae.ln1", i, s1);
            Mat qkv = matmul(y, wq[size_t(l)]);
            scale_rows(qkv, s1);
            rotate(qkv, 0, aq, c.ae_head_dim, L);
            rotate(qkv, aq, aq + akv, c.ae_head_dim, L);
            rec.put("ae.qkv", i, qkv);
            const Mat& lk = kv[size_t(i % c.llm_layers)];  // llm.qkv@mod: instance i % R(llm.qkv)
            Mat kc = stack_rows(cols_of(lk, lq, lq + lkv), cols_of(qkv, aq, aq + akv));
            Mat vc = stack_rows(cols_of(lk, lq + lkv, lq + 2 * lkv), cols_of(qkv, aq + akv, aq + 2 * akv));
            Mat o = attention(cols_of(qkv, 0, aq), kc, vc, c.ae_q_heads, c.ae_kv_heads, c.ae_head_dim);
            rec.put("ae.attn", i, o);
            Mat p = matmul(o, wp[size_t(l)]);
            residual(p, y, 1.0);
            rec.put("ae.proj", i, p);
            const auto s2 = rms_of(p, eps);
            rec.put_vec("ae.ln2", i, s2);
            Mat g = matmul(p, wf[size_t(l)]);
            scale_rows(g, s2);
            Mat gg(g.r, c.ae_mlp);
            for (int64_t r = 0; r < g.r; ++r)
                for (int64_t j = 0; j < c.ae_mlp; ++j) gg.row(r)[j] = g.row(r)[j] * gelu_t(g.row(r)[c.ae_mlp + j]);
            rec.put("ae.ffn", i, gg);
            Mat d = matmul(gg, wd[size_t(l)]);
            residual(d, p, 1.0);
            rec.put("ae.down", i, d);
            y = std::move(d);
        }
        Mat r(y.r - 1, y.c);
        std::copy(y.d.begin() + y.c, y.d.end(), r.d.begin());
        rec.put("ae.act_rows", s, r);
        const auto s3 = rms_of(r, eps);
        rec.put_vec("ae.ln_out", s, s3);
        Mat v = matmul(r, w_hd);
        scale_rows(v, s3);
        add_bias(v, b_hd);
        residual(v, a, 1.0 / FS);
        rec.put("ae.head", s, v);
        a = std::move(v);
    }
    return a;
}

Mat wrap(const double* p, int64_t r, int64_t c) {
    Mat m(r, c);
    if (r * c) std::memcpy(m.d.data(), p, size_t(r * c) * 8);
    return m;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// gen_inputs (proj/src/evaluate.cpp:77-85): sources ~ U(-1, 1), role 5, instance 0.
int orc_gen_inputs(const pi0b_model_config* c, uint64_t seed, double* patches, double* state, double* noise,
                   double* prompt) {
    try {
        g_threads = std::max(1u, std::thread::hardware_concurrency());
        const int T = c->views * c->tokens_per_view;
        auto put = [&](const char* id, int64_t r, int64_t cols, double* dst) {
            Mat m = uniform(r, cols, -1.0, 1.0, fnv_seed(seed, id, 0, kIn));
            std::memcpy(dst, m.d.data(), m.d.size() * 8);
        };
        put("patches", T, c->ve_patch_in, patches);
        put("state", 1, c->ae_state_dim, state);
        put("noise", c->chunk_len, c->ae_action_dim, noise);
        if (c->prompt_tokens > 0) put("prompt", c->prompt_tokens, c->llm_width, prompt);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Full forward with parameters drawn from `wseed`; out = [chunk_len, action_dim].
// Optional recording of node instances (reference node ids) into caller buffers.
int orc_forward(const pi0b_model_config* c, uint64_t wseed, const double* patches, const double* state,
                const double* noise, const double* prompt, double* out, int nthreads, int n_rec,
                const char* const* rec_node, const int64_t* rec_inst, double* const* rec_buf,
                const int64_t* rec_cap) {
    try {
        g_threads = nthreads > 0 ? nthreads : int(std::max(1u, std::thread::hardware_concurrency()));
        const int T = c->views * c->tokens_per_view;
        Recorder rec;
        for (int i = 0; i < n_rec; ++i) rec.want[{rec_node[i], rec_inst[i]}] = {rec_buf[i], rec_cap[i]};
        Mat pr;
        if (c->prompt_tokens > 0) pr = wrap(prompt, c->prompt_tokens, c->llm_width);
        Params prm{wseed};
        Mat a = forward(*c, prm, wrap(patches, T, c->ve_patch_in), wrap(state, 1, c->ae_state_dim),
                        wrap(noise, c->chunk_len, c->ae_action_dim), c->prompt_tokens > 0 ? &pr : nullptr, rec);
        std::memcpy(out, a.d.data(), a.d.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// One weight instance W[k, m] (+ bias [m]) exactly as gen_weights draws it.
int orc_weight(uint64_t seed, const char* node, int64_t inst, int64_t k, int64_t m, double* w, double* bias) {
    try {
        g_threads = std::max(1u, std::thread::hardware_concurrency());
        Params prm{seed};
        if (w) {
            Mat x = prm.w(node, inst, k, m);
            std::memcpy(w, x.d.data(), x.d.size() * 8);
        }
        if (bias) {
            auto b = prm.b(node, inst, k, m);
            std::memcpy(bias, b.data(), b.size() * 8);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
