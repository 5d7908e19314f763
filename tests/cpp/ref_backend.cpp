// ref_backend.cpp -- TEST of the reference-side integration (INTEGRATION.md
// section 1): a translation unit of the REFERENCE (its own headers, linked
// against the reference compiled from its sources, oracle/_ref/
// libspecsamp_ref.so) that adds the two CUDA backends through
// include/ssv/specsamp_bridge.hpp and checks them against the reference's own
// backends on the reference's own inputs (make_bench_inputs, bench.cpp:46-74):
//
//   * Backend switch of bench.cpp:94-143 extended with cuda_exact /
//     cuda_sigmoid (run_backend below is the patch INTEGRATION.md shows);
//   * verify_cuda_exact vs materialize_softmax_into x2 + verify_sequential on
//     unrounded (fp64 storage) and fp32-rounded logits;
//   * verify_cuda_fused vs verify_fused: results, the residual written into q
//     (verify_fused.cpp:50), and the MemoryTrace counters (tile.cpp counting
//     rules) for two tile plans;
//   * verify_cuda_sigmoid_sequential / _fused vs the reference's, traces equal;
//   * the reference's error behaviour: a uniform outside [0, 1) throws
//     std::invalid_argument from the sequential entry points (exact and
//     sigmoid, verify_reference.cpp:28-33) and not from verify_sigmoid_fused.
//
// Built here by oracle/Makefile (needs /root/reference) into oracle/_ref/, run
// on the GPU by tests/test_gpu_cpp.py.  Exit 0 = every check passed.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "specsamp/activation.hpp"
#include "specsamp/bench.hpp"
#include "specsamp/step.hpp"
#include "specsamp/tile.hpp"
#include "specsamp/verify_fused.hpp"
#include "specsamp/verify_reference.hpp"
#include "specsamp/verify_sigmoid.hpp"
#include "ssv/specsamp_bridge.hpp"

using namespace specsamp;

namespace {

int g_fail = 0;
#define CHECK(c, ...)                                          \
    do {                                                       \
        if (!(c)) {                                            \
            std::fprintf(stderr, "FAILED %s:%d %s: ", __FILE__, __LINE__, #c); \
            std::fprintf(stderr, __VA_ARGS__);                 \
            std::fprintf(stderr, "\n");                        \
            ++g_fail;                                          \
        }                                                      \
    } while (0)

// Batch rows b = make_bench_inputs(seed + b, gamma, V) stacked into one
// B-row step (the bench's per-row recipe; rows are independent).
BenchInputs make_batch(uint64_t seed, int B, int gamma, size_t V) {
    BenchInputs out;
    const size_t g = static_cast<size_t>(gamma);
    out.z_p = LogitTensor(B, g + 1, V);
    out.z_q = LogitTensor(B, g, V);
    out.draft_tokens = Matrix<int32_t>(B, g);
    out.uniforms = Matrix<double>(B, g + 1);
    for (int b = 0; b < B; ++b) {
        const BenchInputs r = make_bench_inputs(seed + b, gamma, V);
        for (size_t c = 0; c <= g; ++c) std::copy(r.z_p.row(0, c).begin(), r.z_p.row(0, c).end(), out.z_p.row(b, c).begin());
        for (size_t c = 0; c < g; ++c) std::copy(r.z_q.row(0, c).begin(), r.z_q.row(0, c).end(), out.z_q.row(b, c).begin());
        for (size_t c = 0; c < g; ++c) out.draft_tokens(b, c) = r.draft_tokens(0, c);
        for (size_t c = 0; c <= g; ++c) out.uniforms(b, c) = r.uniforms(0, c);
    }
    return out;
}

void round_f32(Grid3& g) {
    for (double& v : g.flat()) v = static_cast<double>(static_cast<float>(v));
}

// bench.cpp:94-143 with the two CUDA backends of INTEGRATION.md section 1.
enum class BackendX { reference, fused, sigmoid, cuda_exact, cuda_sigmoid };
const char* name(BackendX b) {
    switch (b) {
        case BackendX::reference: return "reference";
        case BackendX::fused: return "fused";
        case BackendX::sigmoid: return "sigmoid";
        case BackendX::cuda_exact: return "cuda_exact";
        default: return "cuda_sigmoid";
    }
}

VerificationResult run_backend(BackendX backend, const BenchInputs& in, const TilePlan& plan, WorkerPool& pool,
                               ScaleBounds bounds, ssv::Storage storage) {
    if (backend == BackendX::sigmoid || backend == BackendX::cuda_sigmoid) {
        SigmoidStepInputs inputs;
        inputs.z_p = in.z_p;
        inputs.z_q = in.z_q;
        inputs.bounds = bounds;
        inputs.draft_tokens = in.draft_tokens;
        inputs.uniforms = in.uniforms;
        if (backend == BackendX::sigmoid) return verify_sigmoid_fused(inputs, plan, pool).result;
        return ssv::verify_cuda_sigmoid_fused(inputs, plan, pool.size(), storage).result;
    }
    if (backend == BackendX::cuda_exact)
        return ssv::verify_cuda_exact(in.z_p, in.z_q, in.draft_tokens, in.uniforms, storage);
    StepInputs inputs;
    inputs.draft_tokens = in.draft_tokens;
    inputs.uniforms = in.uniforms;
    materialize_softmax_into(in.z_p, inputs.p, pool);
    materialize_softmax_into(in.z_q, inputs.q, pool);
    if (backend == BackendX::reference) return verify_sequential(inputs);
    return verify_fused(inputs, plan, pool).result;
}

// results_match (validate.cpp:21-44): integers exact, tau / denominators 1e-6.
int compare(const VerificationResult& a, const VerificationResult& b, const std::string& what) {
    int bad = 0;
    for (size_t r = 0; r < a.accepted_len.size(); ++r) {
        if (a.accepted_len[r] != b.accepted_len[r] || a.final_token[r] != b.final_token[r] ||
            a.resample_used[r] != b.resample_used[r] ||
            std::abs(a.residual_denom[r] - b.residual_denom[r]) > 1e-6 * std::max(1.0, std::abs(a.residual_denom[r]))) {
            std::fprintf(stderr, "  %s: row %zu: accepted %d/%d token %d/%d resample %d/%d denom %.9g/%.9g\n",
                         what.c_str(), r, a.accepted_len[r], b.accepted_len[r], a.final_token[r], b.final_token[r],
                         a.resample_used[r], b.resample_used[r], a.residual_denom[r], b.residual_denom[r]);
            ++bad;
        }
        for (size_t c = 0; c < a.tau.cols(); ++c)
            if (std::abs(a.tau(r, c) - b.tau(r, c)) > 1e-6) {
                std::fprintf(stderr, "  %s: row %zu tau[%zu] %.12g vs %.12g\n", what.c_str(), r, c, a.tau(r, c),
                             b.tau(r, c));
                ++bad;
            }
    }
    return bad;
}

bool same_trace(const MemoryTrace& a, const MemoryTrace& b) {
    return a.hbm_elem_reads_p == b.hbm_elem_reads_p && a.hbm_elem_reads_q == b.hbm_elem_reads_q &&
           a.hbm_elem_writes == b.hbm_elem_writes && a.peak_tile_bytes == b.peak_tile_bytes &&
           a.kernel_invocations == b.kernel_invocations;
}

template <typename F>
bool throws_invalid(F f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    }
    return false;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int main() {
    WorkerPool pool(4);
    const ScaleBounds bounds{-1e3, 1e3};
    struct Cfg {
        uint64_t seed;
        int B, gamma;
        size_t V;
    };
    // C1 at several seeds (seed 1 only takes the bonus path), C2, and a C3-shaped slab.
    const std::vector<Cfg> cfgs = {{1, 1, 5, 32000}, {2, 1, 5, 32000}, {3, 1, 5, 32000}, {6, 1, 5, 32000},
                                   {1, 8, 5, 51865}, {1, 16, 8, 32000}};
    int rows = 0;
    for (const Cfg& cf : cfgs) {
        BenchInputs in = make_batch(cf.seed, cf.B, cf.gamma, cf.V);
        const TilePlan plan = plan_tiles(cf.V, 1024);
        char tag[96];
        std::snprintf(tag, sizeof tag, "seed=%llu B=%d gamma=%d V=%zu", (unsigned long long)cf.seed, cf.B, cf.gamma,
                      cf.V);
        rows += cf.B;
        // Backend switch: the reference's backends against the CUDA ones.
        for (ssv::Storage st : {ssv::Storage::f64, ssv::Storage::f32}) {
            BenchInputs rin = in;
            if (st == ssv::Storage::f32) {  // the device streams fp32: the reference sees the same rounded logits
                round_f32(rin.z_p);
                round_f32(rin.z_q);
            }
            const auto t0 = std::chrono::steady_clock::now();
            const VerificationResult ref = run_backend(BackendX::reference, rin, plan, pool, bounds, st);
            const double t_ref = ms_since(t0);
            const auto t1 = std::chrono::steady_clock::now();
            const VerificationResult cuda = run_backend(BackendX::cuda_exact, rin, plan, pool, bounds, st);
            const double t_cuda = ms_since(t1);
            const std::string w = std::string(tag) + (st == ssv::Storage::f32 ? " f32" : " f64") + " exact";
            CHECK(compare(ref, cuda, w) == 0, "%s", w.c_str());
            const VerificationResult rs = run_backend(BackendX::sigmoid, rin, plan, pool, bounds, st);
            const VerificationResult cs = run_backend(BackendX::cuda_sigmoid, rin, plan, pool, bounds, st);
            CHECK(compare(rs, cs, w + " sigmoid") == 0, "%s sigmoid", w.c_str());
            std::printf("%-40s %-4s %s %.2f ms, %s %.2f ms (incl. upload; %d rows)\n", tag,
                        st == ssv::Storage::f32 ? "f32" : "f64", name(BackendX::reference), t_ref,
                        name(BackendX::cuda_exact), t_cuda, cf.B);
        }
        // verify_fused on probabilities: results, residual written into q, trace.
        StepInputs pin;
        pin.draft_tokens = in.draft_tokens;
        pin.uniforms = in.uniforms;
        materialize_softmax_into(in.z_p, pin.p, pool);
        materialize_softmax_into(in.z_q, pin.q, pool);
        for (size_t tw : {size_t(1024), size_t(333)}) {
            const TilePlan pl = plan_tiles(cf.V, tw);
            StepInputs a = pin, b = pin;
            const FusedVerifyOutput rf = verify_fused(a, pl, pool);
            const FusedVerifyOutput cf2 = ssv::verify_cuda_fused(b, pl, pool.size());
            CHECK(compare(rf.result, cf2.result, std::string(tag) + " verify_fused") == 0, "%s verify_fused", tag);
            CHECK(same_trace(rf.trace, cf2.trace), "%s tile %zu: trace writes %llu vs %llu", tag, tw,
                  (unsigned long long)rf.trace.hbm_elem_writes, (unsigned long long)cf2.trace.hbm_elem_writes);
            double worst = 0.0;
            for (size_t i = 0; i < a.q.values.size(); ++i)
                worst = std::max(worst, std::abs(a.q.values.flat()[i] - b.q.values.flat()[i]));
            CHECK(worst <= 1e-15, "%s: residual written into q differs by %.3g", tag, worst);
            CHECK(compare(verify_sequential(pin), ssv::verify_cuda_sequential(pin), std::string(tag) + " seq") == 0,
                  "%s verify_sequential", tag);
        }
        // sigmoid: sequential oracle and fused, traces
        SigmoidStepInputs s;
        s.z_p = in.z_p;
        s.z_q = in.z_q;
        s.bounds = bounds;
        s.draft_tokens = in.draft_tokens;
        s.uniforms = in.uniforms;
        CHECK(compare(verify_sigmoid_sequential(s), ssv::verify_cuda_sigmoid_sequential(s, ssv::Storage::f64),
                      std::string(tag) + " sigmoid seq") == 0,
              "%s sigmoid sequential", tag);
        const FusedVerifyOutput sf = verify_sigmoid_fused(s, plan, pool);
        const FusedVerifyOutput csf = ssv::verify_cuda_sigmoid_fused(s, plan, pool.size(), ssv::Storage::f64);
        CHECK(same_trace(sf.trace, csf.trace), "%s sigmoid trace", tag);
        // error behaviour: the sequential entry points reject u = 1, the fused sigmoid does not
        SigmoidStepInputs bad = s;
        bad.uniforms(0, 0) = 1.0;
        CHECK(throws_invalid([&] { verify_sigmoid_sequential(bad); }), "reference sigmoid sequential must throw");
        CHECK(throws_invalid([&] { ssv::verify_cuda_sigmoid_sequential(bad); }), "cuda sigmoid sequential must throw");
        CHECK(!throws_invalid([&] { ssv::verify_cuda_sigmoid_fused(bad, plan, 1); }), "cuda sigmoid fused must not throw");
        CHECK(!throws_invalid([&] { verify_sigmoid_fused(bad, plan, pool); }), "reference sigmoid fused must not throw");
        CHECK(throws_invalid([&] { ssv::verify_cuda_exact(bad.z_p, bad.z_q, bad.draft_tokens, bad.uniforms); }),
              "cuda exact must throw on u = 1");
        StepInputs badp = pin;
        badp.draft_tokens(0, 0) = static_cast<int32_t>(cf.V);
        CHECK(throws_invalid([&] { ssv::verify_cuda_sequential(badp); }), "token out of range must throw");
    }
    // plan_tiles KAT: the ssv copy matches the reference's.
    const TilePlan rp = plan_tiles(50257, 1024);
    const ssv::TilePlan sp = ssv::plan_tiles(50257, 1024);
    CHECK(rp.tile_count() == 50 && sp.tile_count() == 50 && sp.tiles.back().size() == 81 &&
              rp.tiles.back().size() == sp.tiles.back().size(),
          "plan_tiles");
    std::printf("ref_backend: %d batch rows, %d failed checks\n", rows, g_fail);
    return g_fail ? 1 : 0;
}
