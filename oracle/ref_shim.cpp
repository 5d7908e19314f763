// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libspecsamp_ref.so).  Used (a) to pin the C restatement in
// oracle/ssv_oracle.c bit-for-bit, (b) to write the golden vectors under
// tests/golden/, and (c) as the CPU baseline / `bench.py --impl reference`
// arm.  Nothing in the product links this.
//
// The reference API wrapped here:
//   verify_sequential        verify_reference.hpp:12 / verify_reference.cpp:76-111
//   verify_fused             verify_fused.hpp:24-27   / verify_fused.cpp:13-105
//   materialize_softmax_into activation.hpp:12-13     / activation.cpp:20-37
//   verify_sigmoid_*         verify_sigmoid.hpp:41-51 / verify_sigmoid.cpp:50-224
//   make_bench_inputs        bench.hpp:45             / bench.cpp:46-74
//   make_model_pair, decode  toy_model.hpp, decode.hpp / toy_model.cpp:16-42, decode.cpp:45-159
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "specsamp/activation.hpp"
#include "specsamp/bench.hpp"
#include "specsamp/decode.hpp"
#include "specsamp/toy_model.hpp"
#include "specsamp/dist.hpp"
#include "specsamp/stats.hpp"
#include "specsamp/step.hpp"
#include "specsamp/tile.hpp"
#include "specsamp/verify_fused.hpp"
#include "specsamp/verify_reference.hpp"
#include "specsamp/verify_sigmoid.hpp"
#include "specsamp/worker_pool.hpp"

using namespace specsamp;

// bench.cpp's run_bench references these harness symbols (stats.cpp needs
// boost, report.cpp needs nlohmann json); they are never reached from the
// entry points below, so link-time stand-ins are enough.
namespace specsamp {
double mean(std::span<const double>) { return 0.0; }
double stddev(std::span<const double>) { return 0.0; }
double median(std::vector<double>) { return 0.0; }
uint64_t peak_rss_bytes() { return 0; }
void write_bench_report(const std::vector<BenchRow>&, const std::string&, ReportFormat) {
    throw std::logic_error("ref_shim: reporting is not wired");
}
}  // namespace specsamp

namespace {

thread_local std::string g_err;

struct RefOut {
    int32_t* accepted_len;
    double* tau;
    int32_t* final_token;
    uint8_t* resample_used;
    double* residual_denom;
};

void fill_grid(Grid3& g, const double* src) {
    auto f = g.flat();
    std::memcpy(f.data(), src, f.size() * sizeof(double));
}

LogitTensor make_grid(const double* src, size_t b, size_t s, size_t v) {
    LogitTensor g(b, s, v);
    fill_grid(g, src);
    return g;
}

template <typename T>
Matrix<T> make_matrix(const T* src, size_t r, size_t c) {
    Matrix<T> m(r, c);
    for (size_t i = 0; i < r; ++i)
        for (size_t j = 0; j < c; ++j) m(i, j) = src[i * c + j];
    return m;
}

void copy_result(const VerificationResult& r, RefOut* o) {
    const size_t B = r.accepted_len.size();
    for (size_t b = 0; b < B; ++b) {
        o->accepted_len[b] = r.accepted_len[b];
        o->final_token[b] = r.final_token[b];
        o->resample_used[b] = r.resample_used[b];
        o->residual_denom[b] = r.residual_denom[b];
        for (size_t c = 0; c < r.tau.cols(); ++c) o->tau[b * r.tau.cols() + c] = r.tau(b, c);
    }
}

StepInputs prob_inputs(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                       const int32_t* ids, const double* u) {
    StepInputs in;
    in.p = ProbTensor(B, p_steps, V);
    fill_grid(in.p.values, p);
    in.q = ProbTensor(B, gamma, V);
    fill_grid(in.q.values, q);
    in.draft_tokens = make_matrix(ids, B, gamma);
    in.uniforms = make_matrix(u, B, gamma + 1);
    return in;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;  // specbench.cpp:234-240: invalid_argument -> exit 2
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

using Clock = std::chrono::steady_clock;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_verify_sequential(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                          const int32_t* ids, const double* u, RefOut* out) {
    return guarded([&] {
        const auto in = prob_inputs(p, p_steps, q, B, gamma, V, ids, u);
        copy_result(verify_sequential(in), out);
    });
}

int ref_verify_fused(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                     const int32_t* ids, const double* u, int tile_width, unsigned workers,
                     RefOut* out) {
    return guarded([&] {
        auto in = prob_inputs(p, p_steps, q, B, gamma, V, ids, u);
        copy_result(verify_fused(in, plan_tiles(V, tile_width), workers).result, out);
    });
}

// Logits-in exact step exactly as bench.cpp:113-127 ("reference" backend).
int ref_verify_exact_logits(const double* zp, int p_steps, const double* zq, int B, int gamma,
                            int V, const int32_t* ids, const double* u, RefOut* out) {
    return guarded([&] {
        StepInputs in;
        in.draft_tokens = make_matrix(ids, B, gamma);
        in.uniforms = make_matrix(u, B, gamma + 1);
        materialize_softmax_into(make_grid(zp, B, p_steps, V), in.p);
        materialize_softmax_into(make_grid(zq, B, gamma, V), in.q);
        copy_result(verify_sequential(in), out);
    });
}

int ref_verify_sigmoid_sequential_h(const double* zp, int p_steps, const double* zq, int B,
                                    int gamma, int V, const int32_t* ids, const double* u,
                                    double alpha, double beta, int emulate_half, RefOut* out);

int ref_verify_sigmoid_sequential(const double* zp, int p_steps, const double* zq, int B,
                                  int gamma, int V, const int32_t* ids, const double* u,
                                  double alpha, double beta, RefOut* out) {
    return ref_verify_sigmoid_sequential_h(zp, p_steps, zq, B, gamma, V, ids, u, alpha, beta, 0, out);
}

int ref_verify_sigmoid_sequential_h(const double* zp, int p_steps, const double* zq, int B,
                                    int gamma, int V, const int32_t* ids, const double* u,
                                    double alpha, double beta, int emulate_half, RefOut* out) {
    return guarded([&] {
        SigmoidStepInputs in;
        in.z_p = make_grid(zp, B, p_steps, V);
        in.z_q = make_grid(zq, B, gamma, V);
        in.bounds = ScaleBounds{alpha, beta};
        in.emulate_half = emulate_half != 0;
        in.draft_tokens = make_matrix(ids, B, gamma);
        in.uniforms = make_matrix(u, B, gamma + 1);
        copy_result(verify_sigmoid_sequential(in), out);
    });
}

int ref_verify_sigmoid_fused(const double* zp, int p_steps, const double* zq, int B, int gamma,
                             int V, const int32_t* ids, const double* u, double alpha,
                             double beta, int tile_width, unsigned workers, RefOut* out) {
    return guarded([&] {
        SigmoidStepInputs in;
        in.z_p = make_grid(zp, B, p_steps, V);
        in.z_q = make_grid(zq, B, gamma, V);
        in.bounds = ScaleBounds{alpha, beta};
        in.draft_tokens = make_matrix(ids, B, gamma);
        in.uniforms = make_matrix(u, B, gamma + 1);
        copy_result(verify_sigmoid_fused(in, plan_tiles(V, tile_width), workers).result, out);
    });
}

int ref_make_bench_inputs(uint64_t seed, int gamma, int V, double* zp, double* zq, int32_t* ids,
                          double* u) {
    return guarded([&] {
        const BenchInputs in = make_bench_inputs(seed, gamma, static_cast<size_t>(V));
        std::memcpy(zp, in.z_p.flat().data(), in.z_p.size() * sizeof(double));
        std::memcpy(zq, in.z_q.flat().data(), in.z_q.size() * sizeof(double));
        for (int c = 0; c < gamma; ++c) ids[c] = in.draft_tokens(0, c);
        for (int c = 0; c <= gamma; ++c) u[c] = in.uniforms(0, c);
    });
}

// ---- CPU baseline timing (bench.cpp:85-151 semantics, B >= 1) -------------
// backend: 0 = "reference" (sequential softmax + verify_sequential, 1 core),
//          1 = "fused"     (pooled softmax + verify_fused on `workers` threads),
//          2 = "sigmoid"   (verify_sigmoid_fused on `workers` threads).
// Runs `warmup` untimed and `trials` timed steps; writes per-trial total ns to
// ns_out[trials] and the last result to out.  Inputs are converted to the
// reference's Grid3 once, outside the timed region.
int ref_time_backend(int backend, const double* zp, int p_steps, const double* zq, int B,
                     int gamma, int V, const int32_t* ids, const double* u, double alpha,
                     double beta, int tile_width, unsigned workers, int warmup, int trials,
                     double* ns_out, RefOut* out) {
    return guarded([&] {
        const LogitTensor z_p = make_grid(zp, B, p_steps, V);
        const LogitTensor z_q = make_grid(zq, B, gamma, V);
        const TilePlan plan = plan_tiles(V, std::min<size_t>(tile_width, V));
        WorkerPool pool(backend == 0 ? 1u : workers);
        VerificationResult last;
        if (backend == 2) {
            SigmoidStepInputs in;
            in.z_p = z_p;
            in.z_q = z_q;
            in.bounds = ScaleBounds{alpha, beta};
            in.draft_tokens = make_matrix(ids, B, gamma);
            in.uniforms = make_matrix(u, B, gamma + 1);
            for (int it = 0; it < warmup + trials; ++it) {
                const auto t0 = Clock::now();
                auto r = verify_sigmoid_fused(in, plan, pool);
                const auto t1 = Clock::now();
                if (it >= warmup) ns_out[it - warmup] = std::chrono::duration<double, std::nano>(t1 - t0).count();
                last = std::move(r.result);
            }
        } else {
            StepInputs in;
            in.draft_tokens = make_matrix(ids, B, gamma);
            in.uniforms = make_matrix(u, B, gamma + 1);
            for (int it = 0; it < warmup + trials; ++it) {
                const auto t0 = Clock::now();
                if (backend == 0) {
                    materialize_softmax_into(z_p, in.p);
                    materialize_softmax_into(z_q, in.q);
                    last = verify_sequential(in);
                } else {
                    materialize_softmax_into(z_p, in.p, pool);
                    materialize_softmax_into(z_q, in.q, pool);
                    last = verify_fused(in, plan, pool).result;
                }
                const auto t1 = Clock::now();
                if (it >= warmup) ns_out[it - warmup] = std::chrono::duration<double, std::nano>(t1 - t0).count();
            }
        }
        copy_result(last, out);
    });
}

// toy_model.cpp:16-42: the (target, draft) logit tables, V x V each.
int ref_make_model_pair(uint64_t seed, int V, double divergence, double logit_scale, double* target,
                        double* draft) {
    return guarded([&] {
        const ModelPair mp = make_model_pair(seed, (size_t)V, divergence, logit_scale);
        std::memcpy(target, mp.target.table.data(), sizeof(double) * (size_t)V * V);
        std::memcpy(draft, mp.draft.table.data(), sizeof(double) * (size_t)V * V);
    });
}

// decode.cpp:45-159 on given tables (temperature 1).  backend 0 reference,
// 1 fused, 2 sigmoid (emulate_half: the binary16 emulation, as ablate.cpp:66-75 runs it).  Writes max_len tokens and the gamma history (max_len
// entries at most); returns the step count through *steps.
int ref_decode(const double* target, const double* draft, int V, const int32_t* prompt, int prompt_len,
               int max_len, int gamma0, int min_gamma, int max_gamma, uint64_t seed, int backend, double alpha,
               double beta, int emulate_half, int32_t* tokens, int32_t* gamma_hist, int* steps) {
    return guarded([&] {
        ToyModel t, d;
        t.vocab_size = d.vocab_size = (size_t)V;
        t.table.assign(target, target + (size_t)V * V);
        d.table.assign(draft, draft + (size_t)V * V);
        DecodeConfig cfg;
        cfg.max_len = (size_t)max_len;
        cfg.backend = backend == 0 ? Backend::reference : (backend == 1 ? Backend::fused : Backend::sigmoid);
        cfg.gamma = GammaState{gamma0, min_gamma, max_gamma};
        cfg.workers = 2;
        cfg.bounds = ScaleBounds{alpha, beta};
        cfg.emulate_half = emulate_half != 0;
        cfg.seed = seed;
        const DecodeOutput out = decode(t, d, std::span<const int32_t>(prompt, (size_t)prompt_len), cfg);
        std::memcpy(tokens, out.tokens.data(), sizeof(int32_t) * out.tokens.size());
        *steps = (int)out.stats.steps;
        for (size_t i = 0; i < out.stats.gamma_history.size() && i < (size_t)max_len; ++i)
            gamma_hist[i] = out.stats.gamma_history[i];
    });
}

}  // extern "C"
