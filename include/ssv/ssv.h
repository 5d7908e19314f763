/*
 * ssv.h -- C-ABI of the B200-native speculative-sampling verification step
 * (arXiv 2406.11016).  Plain C: pointers, sizes and POD structs only.
 *
 * The reference (/root/reference/proj) is a C++ library whose verify API is a
 * set of free functions over std::vector-backed grids; it has no FFI.  Each
 * entry point below names the reference interface it replaces.  A host
 * program keeps the reference's C++ API by including <ssv/ssv.hpp>, a
 * header-only wrapper over this ABI with the reference's types and error
 * behaviour (std::invalid_argument / std::runtime_error).
 *
 * Semantics (identical for every entry point):
 *   inputs   z_p  B x p_steps x V  (p_steps = gamma, or gamma+1 with a bonus row)
 *            z_q  B x gamma   x V  (row-major [b][c][v], row pitch = V elements)
 *            draft_tokens B x gamma int32, uniforms B x (gamma+1) double
 *   outputs  accepted_len[B], final_token[B] (-1 = kNoToken), resample_used[B],
 *            tau[B x gamma] (clamped ratio at EVERY drafted position),
 *            residual_denom[B] (0 unless a non-degenerate resample happened),
 *            optional p / q / residual grids (flags below).
 *   rules    accept while u[b][c] <= tau[b][c] (inclusive); q <= 1e-12 gives
 *            tau = (p > 1e-12); residual max(0, p - q) sampled by the ascending
 *            inverse CDF with u[b][gamma]; residual mass <= 1e-12 falls back to
 *            sampling p (residual_denom reported 0); full acceptance samples the
 *            bonus row gamma when present.
 */
#ifndef SSV_H
#define SSV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror the reference's exception classes) -------------- */
#define SSV_OK 0
#define SSV_ECUDA 1  /* reference: any other std::exception -> exit 1 (specbench.cpp:234-240) */
#define SSV_EINVAL 2 /* reference: std::invalid_argument    -> exit 2 */

/* Device-side input-error bits, written to ssv_verify_out.status when non-NULL
 * (the stream-ordered entry points cannot throw; the host entry points turn
 * any set bit into SSV_EINVAL, as the reference's validate() would). */
#define SSV_STATUS_NONFINITE 1u     /* stable_softmax require_finite, dist.cpp:27-36 */
#define SSV_STATUS_TOKEN_RANGE 2u   /* StepInputs::validate, verify_reference.cpp:22-27 */
#define SSV_STATUS_UNIFORM_RANGE 4u /* StepInputs::validate, verify_reference.cpp:28-33 */
#define SSV_STATUS_NEGATIVE 8u      /* ratio_clamped, dist.cpp:105-107 */

typedef enum { SSV_F32 = 0, SSV_BF16 = 1, SSV_F64 = 2 } ssv_dtype;

/* Optional materialized outputs.  P: B x p_steps x V, Q: B x gamma x V,
 * RESIDUAL: B x gamma x V = max(0, p - q) for every drafted row -- the values
 * verify_fused leaves in q (verify_fused.hpp:18-22).  Element type is float
 * for SSV_F32/SSV_BF16 inputs and double for SSV_F64 inputs. */
#define SSV_WANT_P 1u
#define SSV_WANT_Q 2u
#define SSV_WANT_RESIDUAL 4u
/* Sigmoid entry points only: binary16 emulation of the activation, exactly
 * SigmoidStepInputs::emulate_half (dist.cpp:64-69 sigmoid_scaled_value_half:
 * z, alpha, 1/width, the shifted value, the scaled argument and sigma each
 * rounded to half) -- the paper's FP16 scale-limit study. */
#define SSV_EMULATE_HALF 8u

typedef struct ssv_ctx ssv_ctx; /* one per (host thread, device): stream + scratch */

typedef struct {
    int32_t B, gamma, V;
    int32_t p_steps;     /* gamma or gamma+1 (StepInputs::has_bonus_row, step.hpp:33) */
    int32_t dtype;       /* ssv_dtype of z_p / z_q */
    const void* z_p;     /* logits (exact/sigmoid) or probabilities (probs entry) */
    const void* z_q;
    const int32_t* draft_tokens;
    const double* uniforms;
    double alpha, beta;  /* sigmoid bounds, alpha < 0 < beta (ScaleBounds, dist.hpp:25-32) */
    uint32_t flags;      /* SSV_WANT_* */
} ssv_verify_args;

typedef struct {
    int32_t* accepted_len;   /* [B] */
    int32_t* final_token;    /* [B] */
    uint8_t* resample_used;  /* [B] */
    double* tau;             /* [B x gamma] */
    double* residual_denom;  /* [B] */
    void* p;                 /* optional, see SSV_WANT_P */
    void* q;
    void* residual;
    uint32_t* status;        /* optional [1], SSV_STATUS_* bits (device entry points) */
} ssv_verify_out;

/* ---- context ----------------------------------------------------------------- */
int ssv_create(int device, ssv_ctx** out);
void ssv_destroy(ssv_ctx* ctx);
/* Launch on a caller-owned cudaStream_t (NULL = the legacy default stream, as
 * everywhere in CUDA).  A new context uses its own non-blocking stream, whose
 * handle ssv_get_stream returns until the first ssv_set_stream. */
int ssv_set_stream(ssv_ctx* ctx, void* cuda_stream);
void* ssv_get_stream(const ssv_ctx* ctx);
const char* ssv_last_error(const ssv_ctx* ctx);
/* Number of kernels the last verify/sample/generate call launched. */
int ssv_last_launch_count(const ssv_ctx* ctx);
/* The plan the last verify call launched: info[0] = SSV_PLAN_*, then cluster
 * size, threads per CTA, shared-memory slots, statistics rows per cluster,
 * pieces per row slice (the first n of these).  Diagnostics for tests and the
 * bench; no reference counterpart (the reference has one CPU code path). */
#define SSV_PLAN_STREAMING 0
#define SSV_PLAN_CLUSTER_RESIDENT 1
#define SSV_PLAN_CLUSTER_RING 2
#define SSV_PLAN_SLAB 3
#define SSV_PLAN_SIGMOID_STREAM 4
int ssv_last_plan(const ssv_ctx* ctx, int32_t* info, int32_t n);

/* Kernel selection for the verify entry points: AUTO
 * picks the cluster kernel when every batch row can get a resident thread-
 * block cluster, else the streaming kernel.  All give identical results up to
 * the summation order of the fp32 partial sums (same parity bar). */
#define SSV_PATH_AUTO 0
#define SSV_PATH_STREAMING 1
#define SSV_PATH_CLUSTER 2 /* falls back to streaming where the cluster kernel cannot run */
#define SSV_PATH_CLUSTER_RING 3 /* cluster kernel, two-CTAs-per-SM ring plan only (no resident plan) */
#define SSV_PATH_SLAB 4 /* exact variant: the slab kernel (experimental; falls back to streaming where it cannot run) */
int ssv_set_path(ssv_ctx* ctx, int32_t path);
const char* ssv_version(void);

/* Kernel timing.  While enabled, each kernel launch of this context (up to
 * `capacity` launches after enable/reset) is bracketed by a pair of CUDA
 * events on the launching stream -- also under stream capture, where the
 * records become graph nodes and are re-recorded on every replay.
 * ssv_profile_read sums the bracketed durations of one kernel id
 * (0 = verify, 2 = materialize, 3 = generator) after the
 * stream has been synchronized. */
int ssv_profile_enable(ssv_ctx* ctx, int capacity);
int ssv_profile_disable(ssv_ctx* ctx);
int ssv_profile_reset(ssv_ctx* ctx);
int ssv_profile_read(ssv_ctx* ctx, int32_t kernel_id, double* total_ms, int32_t* count);

/* Diagnostics.  capacity > 0 with host_out == NULL attaches a device buffer
 * of `capacity` globaltimer stamps (ns) that verify launches fill when it holds
 * at least 8 * B + 26 slots: [8 * B] per-batch-row phase stamps, then kernel
 * start / end and finer stamps of batch row 0 (layout: tools/trace_step.py).
 * host_out != NULL copies the buffer out (after a stream sync); capacity 0
 * detaches it. */
int ssv_debug_trace(ssv_ctx* ctx, int capacity, unsigned long long* host_out, int* grid_out);

/* ---- stream-ordered entry points: every pointer is DEVICE memory ----------- */
/* Exact step, logits in.  Replaces materialize_softmax_into(z_p) and (z_q)
 * (activation.hpp:12-13 / activation.cpp:20-37) followed by verify_sequential
 * (verify_reference.hpp:12) or verify_fused (verify_fused.hpp:24-27); the
 * sequence bench.cpp:113-141 and decode.cpp:121-135 run. */
int ssv_verify_exact(ssv_ctx* ctx, const ssv_verify_args* args, ssv_verify_out* out);

/* Sigmoid-approximation step, logits in.  Replaces verify_sigmoid_fused /
 * verify_sigmoid_sequential (verify_sigmoid.hpp:41-51), emulate_half = false. */
int ssv_verify_sigmoid(ssv_ctx* ctx, const ssv_verify_args* args, ssv_verify_out* out);

/* Exact step, probabilities in (no softmax).  Replaces verify_sequential /
 * verify_fused on StepInputs{p, q} (verify_reference.hpp:12,
 * verify_fused.hpp:24-27) for callers that already hold probabilities. */
int ssv_verify_probs(ssv_ctx* ctx, const ssv_verify_args* args, ssv_verify_out* out);

/* ---- host entry points: every pointer is HOST memory ------------------------- */
/* Validate on the host exactly like StepInputs::validate (verify_reference.cpp:
 * 11-36) / SigmoidStepInputs::validate (verify_sigmoid.cpp:13-33), copy the
 * inputs to the device (pinned host memory recommended, see ssv_host_alloc),
 * run the step, copy every output back, synchronize.  Returns SSV_EINVAL for
 * the cases the reference throws std::invalid_argument on. */
int ssv_verify_exact_host(ssv_ctx* ctx, const ssv_verify_args* args, ssv_verify_out* out);
int ssv_verify_sigmoid_host(ssv_ctx* ctx, const ssv_verify_args* args, ssv_verify_out* out);
int ssv_verify_probs_host(ssv_ctx* ctx, const ssv_verify_args* args, ssv_verify_out* out);

/* Pinned host memory for the host entry points. */
void* ssv_host_alloc(size_t bytes);
void ssv_host_free(void* p);

/* ---- callers on either side of the path ---------------------------------------- */
/* Categorical draw from softmax(logits row) with one uniform per row, by the
 * ascending inverse CDF: stable_softmax_into + detail::sample_row, the draft
 * sampling step of decode.cpp:85-91 and bench.cpp:66-69.  Device pointers. */
int ssv_sample_softmax(ssv_ctx* ctx, int32_t dtype, const void* logits, int32_t rows, int32_t V,
                       const double* uniforms, int32_t* tokens_out, uint32_t* status);

/* Synthetic inputs by the reference bench recipe, make_bench_inputs
 * (bench.cpp:46-74), batch row b seeded with seed + b: z_p = 4 N(0,1),
 * z_q = z_p + N(0,1), counter-RNG uniforms, drafts sampled from softmax(z_q).
 * Writes z_p (B x (gamma+1) x V), z_q (B x gamma x V) in `dtype`, draft_tokens
 * and uniforms.  Device pointers. */
int ssv_make_bench_inputs(ssv_ctx* ctx, uint64_t seed, int32_t B, int32_t gamma, int32_t V,
                          int32_t dtype, void* z_p, void* z_q, int32_t* draft_tokens,
                          double* uniforms);

#ifdef __cplusplus
}
#endif

#endif /* SSV_H */
