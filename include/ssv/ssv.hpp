// ssv.hpp -- header-only C++ drop-in over the C-ABI (ssv.h), with the
// reference's types and calling conventions (namespace specsamp in
// /root/reference/proj/include/specsamp).  A caller of the reference swaps
//
//   specsamp::verify_sequential / verify_fused / verify_sigmoid_fused /
//   verify_sigmoid_sequential / materialize_softmax_into + verify_sequential
//
// for the same-named functions here (namespace ssv), linking libssv.so.  Errors
// keep the reference's classes: std::invalid_argument where the reference's
// validate() throws, std::runtime_error for CUDA failures.
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ssv/ssv.h"

namespace ssv {

inline constexpr double kZeroEps = 1e-12;  // dist.hpp:9
inline constexpr int32_t kNoToken = -1;    // step.hpp:11

// ---- tensor.hpp:13-89 ------------------------------------------------------
class Grid3 {
public:
    Grid3() = default;
    Grid3(size_t batch, size_t steps, size_t vocab)
        : batch_(batch), steps_(steps), vocab_(vocab), data_(batch * steps * vocab, 0.0) {
        if (batch == 0 || steps == 0 || vocab == 0) throw std::invalid_argument("Grid3: all dimensions must be >= 1");
    }
    size_t batch() const { return batch_; }
    size_t steps() const { return steps_; }
    size_t vocab() const { return vocab_; }
    size_t size() const { return data_.size(); }
    std::span<double> row(size_t b, size_t c) { return {data_.data() + (b * steps_ + c) * vocab_, vocab_}; }
    std::span<const double> row(size_t b, size_t c) const { return {data_.data() + (b * steps_ + c) * vocab_, vocab_}; }
    std::span<double> flat() { return data_; }
    std::span<const double> flat() const { return data_; }
    bool operator==(const Grid3&) const = default;

private:
    size_t batch_ = 0, steps_ = 0, vocab_ = 0;
    std::vector<double> data_;
};
using LogitTensor = Grid3;

struct ProbTensor {
    Grid3 values;
    bool normalized = true;
    ProbTensor() = default;
    ProbTensor(size_t batch, size_t steps, size_t vocab, bool normalized_ = true)
        : values(batch, steps, vocab), normalized(normalized_) {}
    size_t batch() const { return values.batch(); }
    size_t steps() const { return values.steps(); }
    size_t vocab() const { return values.vocab(); }
    std::span<double> row(size_t b, size_t c) { return values.row(b, c); }
    std::span<const double> row(size_t b, size_t c) const { return values.row(b, c); }
    bool operator==(const ProbTensor&) const = default;
};

template <typename T>
class Matrix {
public:
    Matrix() = default;
    Matrix(size_t rows, size_t cols, T fill = T{}) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    size_t rows() const { return rows_; }
    size_t cols() const { return cols_; }
    T& operator()(size_t r, size_t c) { return data_[r * cols_ + c]; }
    const T& operator()(size_t r, size_t c) const { return data_[r * cols_ + c]; }
    std::span<T> row(size_t r) { return {data_.data() + r * cols_, cols_}; }
    std::span<const T> row(size_t r) const { return {data_.data() + r * cols_, cols_}; }
    const T* data() const { return data_.data(); }
    T* data() { return data_.data(); }
    bool operator==(const Matrix&) const = default;

private:
    size_t rows_ = 0, cols_ = 0;
    std::vector<T> data_;
};

// ---- dist.hpp:25-32 --------------------------------------------------------
struct ScaleBounds {
    double alpha;
    double beta;
    void validate() const {
        if (!std::isfinite(alpha) || !std::isfinite(beta) || !(alpha < 0.0) || !(beta > 0.0))
            throw std::invalid_argument("ScaleBounds: require alpha < 0 < beta, both finite");
    }
    double width() const { return beta - alpha; }
};

// ---- step.hpp:24-51 ----------------------------------------------------------
struct StepInputs {
    ProbTensor p;  // B x gamma(+1) x V
    ProbTensor q;  // B x gamma x V
    Matrix<int32_t> draft_tokens;
    Matrix<double> uniforms;
    size_t batch() const { return q.batch(); }
    size_t gamma() const { return q.steps(); }
    size_t vocab() const { return q.vocab(); }
    bool has_bonus_row() const { return p.steps() == q.steps() + 1; }
};

// Logits-in exact step: the inputs of materialize_softmax_into(z_p), (z_q)
// followed by verify_sequential (bench.cpp:113-127, decode.cpp:121-135).
struct LogitStepInputs {
    LogitTensor z_p;  // B x gamma(+1) x V
    LogitTensor z_q;  // B x gamma x V
    Matrix<int32_t> draft_tokens;
    Matrix<double> uniforms;
    size_t batch() const { return z_q.batch(); }
    size_t gamma() const { return z_q.steps(); }
    size_t vocab() const { return z_q.vocab(); }
    bool has_bonus_row() const { return z_p.steps() == z_q.steps() + 1; }
};

// verify_sigmoid.hpp:15-29
struct SigmoidStepInputs {
    LogitTensor z_p;
    LogitTensor z_q;
    ScaleBounds bounds;
    bool emulate_half = false;  // binary16 emulation (dist.cpp:64-69): SSV_EMULATE_HALF
    Matrix<int32_t> draft_tokens;
    Matrix<double> uniforms;
    size_t batch() const { return z_q.batch(); }
    size_t gamma() const { return z_q.steps(); }
    size_t vocab() const { return z_q.vocab(); }
    bool has_bonus_row() const { return z_p.steps() == z_q.steps() + 1; }
};

struct VerificationResult {
    std::vector<int32_t> accepted_len;
    Matrix<double> tau;
    std::vector<int32_t> final_token;
    std::vector<uint8_t> resample_used;
    std::vector<double> residual_denom;
    bool operator==(const VerificationResult&) const = default;
};

// ---- tile.hpp:10-48 (host bookkeeping; the device picks its own tiling) ----
struct TileRange {
    size_t begin = 0, end = 0;
    size_t size() const { return end - begin; }
    bool operator==(const TileRange&) const = default;
};
struct TilePlan {
    size_t vocab_size = 0;
    size_t tile_width = 0;
    std::vector<TileRange> tiles;
    size_t tile_count() const { return tiles.size(); }
};
inline TilePlan plan_tiles(size_t vocab_size, size_t tile_width) {  // tile.cpp:11-23
    if (vocab_size == 0 || tile_width == 0)
        throw std::invalid_argument("plan_tiles: vocab_size and tile_width must be >= 1");
    TilePlan plan;
    plan.vocab_size = vocab_size;
    plan.tile_width = tile_width;
    for (size_t b = 0; b < vocab_size; b += tile_width) plan.tiles.push_back({b, std::min(b + tile_width, vocab_size)});
    return plan;
}

// The reference's modeled counters, reported analytically for the same plan
// (the device's real traffic is measured by ncu).
struct MemoryTrace {
    uint64_t hbm_elem_reads_p = 0, hbm_elem_reads_q = 0, hbm_elem_writes = 0, peak_tile_bytes = 0,
             kernel_invocations = 0;
    bool operator==(const MemoryTrace&) const = default;
};
struct FusedVerifyOutput {
    VerificationResult result;
    MemoryTrace trace;
};

enum class Storage { f32 = SSV_F32, bf16 = SSV_BF16, f64 = SSV_F64 };

// ---- device context -------------------------------------------------------
class Device {
public:
    explicit Device(int device = 0) {
        const int rc = ssv_create(device, &ctx_);
        if (rc != SSV_OK) throw std::runtime_error("ssv_create failed (no CUDA device?)");
    }
    ~Device() { ssv_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    ssv_ctx* get() const { return ctx_; }

private:
    ssv_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
    thread_local Device dev(0);
    return dev;
}

namespace detail {

inline void check(ssv_ctx* ctx, int rc) {
    if (rc == SSV_OK) return;
    const std::string msg = ssv_last_error(ctx);
    if (rc == SSV_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// Device storage of a double grid.
struct Staged {
    std::vector<float> f;
    std::vector<uint16_t> h;
    const void* ptr = nullptr;
};

inline uint16_t to_bf16(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

inline Staged stage(std::span<const double> x, Storage s) {
    Staged out;
    if (s == Storage::f64) {
        out.ptr = x.data();
    } else if (s == Storage::f32) {
        out.f.resize(x.size());
        for (size_t i = 0; i < x.size(); ++i) out.f[i] = static_cast<float>(x[i]);
        out.ptr = out.f.data();
    } else {
        out.h.resize(x.size());
        for (size_t i = 0; i < x.size(); ++i) out.h[i] = to_bf16(static_cast<float>(x[i]));
        out.ptr = out.h.data();
    }
    return out;
}

// Pointer to a row-major matrix's storage (ssv::Matrix or the reference's
// specsamp::Matrix, whose rows are contiguous).
template <typename M>
auto mat_ptr(const M& m) -> decltype(m.row(0).data()) {
    return m.rows() && m.cols() ? m.row(0).data() : nullptr;
}

// Shape checks with the reference's messages: StepInputs::validate
// (verify_reference.cpp:12-21) or SigmoidStepInputs::validate
// (verify_sigmoid.cpp:14-23).
template <typename G, typename MI, typename MU>
void check_shapes(const G& zp, const G& zq, const MI& ids, const MU& u, bool sigmoid) {
    const size_t B = zq.batch(), Gm = zq.steps(), V = zq.vocab();
    if (zp.batch() != B || zp.vocab() != V || (zp.steps() != Gm && zp.steps() != Gm + 1))
        throw std::invalid_argument(sigmoid ? "SigmoidStepInputs: z_p must be B x gamma(+1) x V matching z_q"
                                            : "StepInputs: p must be B x gamma(+1) x V matching q");
    if (ids.rows() != B || ids.cols() != Gm)
        throw std::invalid_argument(sigmoid ? "SigmoidStepInputs: draft_tokens must be B x gamma"
                                            : "StepInputs: draft_tokens must be B x gamma");
    if (u.rows() != B || u.cols() != Gm + 1)
        throw std::invalid_argument(sigmoid ? "SigmoidStepInputs: uniforms must be B x (gamma+1)"
                                            : "StepInputs: uniforms must be B x (gamma+1)");
}

// The uniform range check of StepInputs::validate (verify_reference.cpp:28-33),
// which the sigmoid SEQUENTIAL oracle inherits through verify_sequential
// (verify_sigmoid.cpp:50-58) and the fused sigmoid path does not.
template <typename MU>
void check_uniforms(const MU& u) {
    for (size_t r = 0; r < u.rows(); ++r)
        for (size_t c = 0; c < u.cols(); ++c) {
            const double x = u(r, c);
            if (!(x >= 0.0) || !(x < 1.0)) throw std::invalid_argument("StepInputs: uniforms must lie in [0, 1)");
        }
}

// One host-entry call (ssv_verify_*_host): stage the double grids in the
// storage type, run on the device, results into a VerificationResult.  G is
// ssv::Grid3 or specsamp::Grid3; MI / MU ssv:: or specsamp::Matrix.
template <typename Fn, typename G, typename MI, typename MU>
VerificationResult run(Fn fn, ssv_ctx* ctx, const G& zp, const G& zq, const MI& ids, const MU& u, Storage s,
                       double alpha, double beta, uint32_t flags = 0, void* residual = nullptr) {
    const size_t B = zq.batch(), Gm = zq.steps(), V = zq.vocab();
    const Staged sp = stage(zp.flat(), s), sq = stage(zq.flat(), s);
    VerificationResult r;
    r.accepted_len.assign(B, 0);
    r.tau = Matrix<double>(B, Gm);
    r.final_token.assign(B, kNoToken);
    r.resample_used.assign(B, 0);
    r.residual_denom.assign(B, 0.0);
    ssv_verify_args a{static_cast<int32_t>(B), static_cast<int32_t>(Gm), static_cast<int32_t>(V),
                      static_cast<int32_t>(zp.steps()), static_cast<int32_t>(s), sp.ptr, sq.ptr, mat_ptr(ids),
                      mat_ptr(u), alpha, beta, flags};
    ssv_verify_out o{r.accepted_len.data(), r.final_token.data(), r.resample_used.data(), r.tau.data(),
                     r.residual_denom.data(), nullptr, nullptr, residual, nullptr};
    check(ctx, fn(ctx, &a, &o));
    return r;
}

inline MemoryTrace analytic_trace(const VerificationResult& r, size_t B, size_t G, size_t V, const TilePlan& plan) {
    // tile.cpp:73-100 and verify_fused.cpp:88-92 counting rules.
    MemoryTrace t;
    const uint64_t K = plan.tile_count();
    t.hbm_elem_reads_p = t.hbm_elem_reads_q = static_cast<uint64_t>(B) * G * V;
    t.kernel_invocations = static_cast<uint64_t>(B) * G * K;
    t.hbm_elem_writes = static_cast<uint64_t>(B) * G * V + static_cast<uint64_t>(B) * G * K + static_cast<uint64_t>(B) * G;
    for (size_t b = 0; b < B; ++b)
        if (r.resample_used[b] && r.residual_denom[b] > 0.0) t.hbm_elem_writes += V;
    const size_t n = plan.tiles.empty() ? 0 : plan.tiles.front().size();
    t.peak_tile_bytes = (2 * n + std::bit_ceil(n)) * sizeof(double);
    return t;
}

}  // namespace detail

// ---- drop-ins ----------------------------------------------------------------
// materialize_softmax_into(z_p), (z_q) + verify_sequential, logits in
// (bench.cpp:113-127, decode.cpp:121-135).
inline VerificationResult verify_exact(const LogitStepInputs& in, Storage storage = Storage::f32,
                                       Device& dev = default_device()) {
    detail::check_shapes(in.z_p, in.z_q, in.draft_tokens, in.uniforms, false);
    return detail::run(ssv_verify_exact_host, dev.get(), in.z_p, in.z_q, in.draft_tokens, in.uniforms, storage, 0, 0);
}

// verify_reference.hpp:12 -- probabilities in, fp64 storage (the reference's own type).
inline VerificationResult verify_sequential(const StepInputs& in, Device& dev = default_device()) {
    detail::check_shapes(in.p.values, in.q.values, in.draft_tokens, in.uniforms, false);
    return detail::run(ssv_verify_probs_host, dev.get(), in.p.values, in.q.values, in.draft_tokens, in.uniforms,
                       Storage::f64, 0, 0);
}

// verify_fused.hpp:24-27 -- same signature; like the reference, q is consumed:
// the clamped residual max(0, p - q) of every drafted row is written back into
// it (verify_fused.cpp:50).  `workers` and the tile plan shape only the
// analytic MemoryTrace (the device picks its own tiling).
inline FusedVerifyOutput verify_fused(StepInputs& in, const TilePlan& plan, unsigned workers,
                                      Device& dev = default_device()) {
    (void)workers;
    detail::check_shapes(in.p.values, in.q.values, in.draft_tokens, in.uniforms, false);
    if (plan.vocab_size != in.vocab() || plan.tiles.empty())
        throw std::invalid_argument("verify_fused: tile plan does not match the input vocabulary");
    std::vector<double> residual(in.q.values.size());
    FusedVerifyOutput out;
    out.result = detail::run(ssv_verify_probs_host, dev.get(), in.p.values, in.q.values, in.draft_tokens, in.uniforms,
                             Storage::f64, 0, 0, SSV_WANT_RESIDUAL, residual.data());
    std::copy(residual.begin(), residual.end(), in.q.values.flat().begin());
    out.trace = detail::analytic_trace(out.result, in.batch(), in.gamma(), in.vocab(), plan);
    return out;
}

// verify_sigmoid.hpp:41.  Like the reference, the sequential oracle rejects
// uniforms outside [0, 1) (it validates through verify_sequential,
// verify_sigmoid.cpp:50-58 -> verify_reference.cpp:28-33).
inline VerificationResult verify_sigmoid_sequential(const SigmoidStepInputs& in, Storage storage = Storage::f32,
                                                    Device& dev = default_device()) {
    in.bounds.validate();
    detail::check_shapes(in.z_p, in.z_q, in.draft_tokens, in.uniforms, true);
    detail::check_uniforms(in.uniforms);
    return detail::run(ssv_verify_sigmoid_host, dev.get(), in.z_p, in.z_q, in.draft_tokens, in.uniforms, storage,
                       in.bounds.alpha, in.bounds.beta, in.emulate_half ? SSV_EMULATE_HALF : 0u);
}

// verify_sigmoid.hpp:48-51.  Inputs untouched; uniforms not range-checked
// (SigmoidStepInputs::validate, verify_sigmoid.cpp:13-33).
inline FusedVerifyOutput verify_sigmoid_fused(const SigmoidStepInputs& in, const TilePlan& plan, unsigned workers,
                                              Storage storage = Storage::f32, Device& dev = default_device()) {
    (void)workers;
    in.bounds.validate();
    detail::check_shapes(in.z_p, in.z_q, in.draft_tokens, in.uniforms, true);
    if (plan.vocab_size != in.vocab() || plan.tiles.empty())
        throw std::invalid_argument("verify_sigmoid_fused: tile plan does not match the vocabulary");
    FusedVerifyOutput out;
    out.result = detail::run(ssv_verify_sigmoid_host, dev.get(), in.z_p, in.z_q, in.draft_tokens, in.uniforms,
                             storage, in.bounds.alpha, in.bounds.beta, in.emulate_half ? SSV_EMULATE_HALF : 0u);
    out.trace = detail::analytic_trace(out.result, in.batch(), in.gamma(), in.vocab(), plan);
    return out;
}

}  // namespace ssv
