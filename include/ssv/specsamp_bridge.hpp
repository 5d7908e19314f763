// specsamp_bridge.hpp -- the reference-side integration of the B200 verify
// step: included by a translation unit of the reference AFTER its own headers
// (specsamp/step.hpp, tile.hpp, verify_fused.hpp, verify_sigmoid.hpp), it
// provides
//
//   * to_ssv / from_ssv: moves between the reference's Grid3 / Matrix /
//     VerificationResult / MemoryTrace / TilePlan and the identical layouts of
//     ssv.hpp (both row-major [b][c][v], tensor.hpp:28-33);
//   * CUDA backends with the REFERENCE's own signatures and types, the entry
//     points a maintainer wires into the Backend switch (decode.cpp:106-136,
//     bench.cpp:94-143) as Backend::cuda_exact / Backend::cuda_sigmoid:
//       verify_cuda_sequential(const specsamp::StepInputs&)          (verify_reference.hpp:12)
//       verify_cuda_fused(specsamp::StepInputs&, const TilePlan&, unsigned)  (verify_fused.hpp:24-27)
//       verify_cuda_exact(const LogitTensor& z_p, z_q, draft_tokens, uniforms)
//           = materialize_softmax_into x2 + verify_sequential      (bench.cpp:113-127)
//       verify_cuda_sigmoid_sequential(const specsamp::SigmoidStepInputs&) (verify_sigmoid.hpp:41)
//       verify_cuda_sigmoid_fused(const SigmoidStepInputs&, const TilePlan&, unsigned) (verify_sigmoid.hpp:48-51)
//
// The backends read the reference's containers in place (no intermediate
// ssv:: copy of the grids); errors keep the reference's classes
// (std::invalid_argument / std::runtime_error).  INTEGRATION.md section 1 is
// the patch; tests/cpp/ref_backend.cpp compiles it against the reference's
// headers and checks it against the reference's own backends.
#pragma once

#include "ssv/ssv.hpp"

#ifndef SPECSAMP_BRIDGE_NO_REFERENCE_CHECK
#if !__has_include("specsamp/step.hpp")
#error "specsamp_bridge.hpp needs the reference's include directory (proj/include) on the include path"
#endif
#endif

#include "specsamp/step.hpp"
#include "specsamp/tile.hpp"
#include "specsamp/verify_fused.hpp"
#include "specsamp/verify_sigmoid.hpp"

namespace ssv {

// ---- layout moves ------------------------------------------------------------
inline Grid3 to_ssv(const specsamp::Grid3& g) {
    Grid3 out(g.batch(), g.steps(), g.vocab());
    std::copy(g.flat().begin(), g.flat().end(), out.flat().begin());
    return out;
}
template <typename T>
Matrix<T> to_ssv(const specsamp::Matrix<T>& m) {
    Matrix<T> out(m.rows(), m.cols());
    for (size_t r = 0; r < m.rows(); ++r) std::copy(m.row(r).begin(), m.row(r).end(), out.row(r).begin());
    return out;
}
inline TilePlan to_ssv(const specsamp::TilePlan& p) {
    TilePlan out;
    out.vocab_size = p.vocab_size;
    out.tile_width = p.tile_width;
    for (const auto& t : p.tiles) out.tiles.push_back({t.begin, t.end});
    return out;
}
inline specsamp::Grid3 from_ssv(const Grid3& g) {
    specsamp::Grid3 out(g.batch(), g.steps(), g.vocab());
    std::copy(g.flat().begin(), g.flat().end(), out.flat().begin());
    return out;
}
template <typename T>
specsamp::Matrix<T> from_ssv(const Matrix<T>& m) {
    specsamp::Matrix<T> out(m.rows(), m.cols());
    for (size_t r = 0; r < m.rows(); ++r) std::copy(m.row(r).begin(), m.row(r).end(), out.row(r).begin());
    return out;
}
inline specsamp::VerificationResult from_ssv(VerificationResult r) {
    specsamp::VerificationResult out;
    out.accepted_len = std::move(r.accepted_len);
    out.tau = from_ssv(r.tau);
    out.final_token = std::move(r.final_token);
    out.resample_used = std::move(r.resample_used);
    out.residual_denom = std::move(r.residual_denom);
    return out;
}
inline specsamp::MemoryTrace from_ssv(const MemoryTrace& t) {
    specsamp::MemoryTrace out;
    out.hbm_elem_reads_p = t.hbm_elem_reads_p;
    out.hbm_elem_reads_q = t.hbm_elem_reads_q;
    out.hbm_elem_writes = t.hbm_elem_writes;
    out.peak_tile_bytes = t.peak_tile_bytes;
    out.kernel_invocations = t.kernel_invocations;
    return out;
}
inline specsamp::FusedVerifyOutput from_ssv(FusedVerifyOutput f) {
    return specsamp::FusedVerifyOutput{from_ssv(std::move(f.result)), from_ssv(f.trace)};
}

// ---- CUDA backends with the reference's signatures -----------------------------
namespace detail {
inline void check_tokens(const specsamp::Matrix<int32_t>& ids, size_t V, const char* msg) {
    for (size_t r = 0; r < ids.rows(); ++r)
        for (size_t c = 0; c < ids.cols(); ++c)
            if (ids(r, c) < 0 || static_cast<size_t>(ids(r, c)) >= V) throw std::invalid_argument(msg);
}
inline TilePlan plan_of(const specsamp::TilePlan& p) { return to_ssv(p); }
}  // namespace detail

// verify_reference.hpp:12 on the device (fp64 probabilities, as given).
inline specsamp::VerificationResult verify_cuda_sequential(const specsamp::StepInputs& in,
                                                           Device& dev = default_device()) {
    in.validate();  // the reference's own checks and messages
    return from_ssv(detail::run(ssv_verify_probs_host, dev.get(), in.p.values, in.q.values, in.draft_tokens,
                                in.uniforms, Storage::f64, 0, 0));
}

// verify_fused.hpp:24-27 on the device: consumes q like the reference (the
// clamped residual max(0, p - q) is written into it, verify_fused.cpp:50); the
// MemoryTrace is the reference's counting rule for the same plan.
inline specsamp::FusedVerifyOutput verify_cuda_fused(specsamp::StepInputs& in, const specsamp::TilePlan& plan,
                                                     unsigned workers, Device& dev = default_device()) {
    (void)workers;
    in.validate();
    if (plan.vocab_size != in.vocab() || plan.tiles.empty())
        throw std::invalid_argument("verify_fused: tile plan does not match the input vocabulary");
    std::vector<double> residual(in.q.values.size());
    VerificationResult r = detail::run(ssv_verify_probs_host, dev.get(), in.p.values, in.q.values, in.draft_tokens,
                                       in.uniforms, Storage::f64, 0, 0, SSV_WANT_RESIDUAL, residual.data());
    std::copy(residual.begin(), residual.end(), in.q.values.flat().begin());
    const MemoryTrace t = detail::analytic_trace(r, in.batch(), in.gamma(), in.vocab(), detail::plan_of(plan));
    return specsamp::FusedVerifyOutput{from_ssv(std::move(r)), from_ssv(t)};
}

// materialize_softmax_into(z_p), (z_q) + verify_sequential (bench.cpp:113-127,
// decode.cpp:121-135), logits in; `storage` is what the device streams
// (the logits are rounded to it; Storage::f64 = no rounding).
inline specsamp::VerificationResult verify_cuda_exact(const specsamp::LogitTensor& z_p,
                                                      const specsamp::LogitTensor& z_q,
                                                      const specsamp::Matrix<int32_t>& draft_tokens,
                                                      const specsamp::Matrix<double>& uniforms,
                                                      Storage storage = Storage::f32,
                                                      Device& dev = default_device()) {
    detail::check_shapes(z_p, z_q, draft_tokens, uniforms, false);
    detail::check_tokens(draft_tokens, z_q.vocab(), "StepInputs: draft token out of vocabulary range");
    detail::check_uniforms(uniforms);
    return from_ssv(
        detail::run(ssv_verify_exact_host, dev.get(), z_p, z_q, draft_tokens, uniforms, storage, 0, 0));
}

// verify_sigmoid.hpp:41: validates like the reference (SigmoidStepInputs::
// validate, then verify_sequential's uniform range check, verify_sigmoid.cpp:50-58).
inline specsamp::VerificationResult verify_cuda_sigmoid_sequential(const specsamp::SigmoidStepInputs& in,
                                                                   Storage storage = Storage::f32,
                                                                   Device& dev = default_device()) {
    in.validate();
    detail::check_uniforms(in.uniforms);
    return from_ssv(detail::run(ssv_verify_sigmoid_host, dev.get(), in.z_p, in.z_q, in.draft_tokens, in.uniforms,
                                storage, in.bounds.alpha, in.bounds.beta, in.emulate_half ? SSV_EMULATE_HALF : 0u));
}

// verify_sigmoid.hpp:48-51: inputs untouched, uniforms not range-checked.
inline specsamp::FusedVerifyOutput verify_cuda_sigmoid_fused(const specsamp::SigmoidStepInputs& in,
                                                             const specsamp::TilePlan& plan, unsigned workers,
                                                             Storage storage = Storage::f32,
                                                             Device& dev = default_device()) {
    (void)workers;
    in.validate();
    if (plan.vocab_size != in.vocab() || plan.tiles.empty())
        throw std::invalid_argument("verify_sigmoid_fused: tile plan does not match the vocabulary");
    VerificationResult r = detail::run(ssv_verify_sigmoid_host, dev.get(), in.z_p, in.z_q, in.draft_tokens,
                                       in.uniforms, storage, in.bounds.alpha, in.bounds.beta,
                                       in.emulate_half ? SSV_EMULATE_HALF : 0u);
    const MemoryTrace t = detail::analytic_trace(r, in.batch(), in.gamma(), in.vocab(), detail::plan_of(plan));
    return specsamp::FusedVerifyOutput{from_ssv(std::move(r)), from_ssv(t)};
}

}  // namespace ssv
