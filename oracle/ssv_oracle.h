/*
 * ssv_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's speculative-sampling verification
 * path (arXiv 2406.11016 artifact, /root/reference/proj).  It is the checker
 * the parity tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * compare the CUDA product against.  Nothing in the product
 * (paper_2406_11016_b200/, include/) links, loads or calls it.
 *
 * Parity of this restatement is PINNED two ways ("Oracle"):
 *   1. the SPEC.md worked examples (known-answer tests in tests/test_oracle.py);
 *   2. the reference itself, compiled from /root/reference/proj/src by
 *      oracle/Makefile into oracle/_ref/ and compared bit-for-bit on seeded
 *      instances (tests/test_oracle.py), plus committed golden vectors
 *      (tests/golden/, written by tests/golden/make_golden.py from oracle/_ref).
 *
 * All arithmetic is double, as in the reference.  Every function
 * cites the reference file:line it restates.
 */
#ifndef SSV_ORACLE_H
#define SSV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_EINVAL 2   /* the reference throws std::invalid_argument here */

#define ORC_ZERO_EPS 1e-12   /* dist.hpp:9 kZeroEps */
#define ORC_NO_TOKEN (-1)    /* step.hpp:11 kNoToken */

/* ---- counter RNG (rng.cpp:12-33) ---------------------------------------- */
uint64_t orc_word_at(uint64_t seed, uint64_t index);
typedef struct {
    uint64_t seed;
    uint64_t counter;
} orc_rng;
uint64_t orc_next_u64(orc_rng* r);
double orc_next_uniform(orc_rng* r);
double orc_next_normal(orc_rng* r);

/* ---- distribution primitives (dist.cpp) --------------------------------- */
double orc_stable_sigmoid(double t);
int orc_stable_softmax_into(const double* z, size_t n, double* out);
double orc_sigmoid_scaled_value(double z, double alpha, double beta);
int orc_ratio_clamped(double p, double q, double* out);
double orc_sequential_sum(const double* v, size_t n);
size_t orc_scan_categorical(const double* v, size_t n, double denom, double u);
int32_t orc_sample_row(const double* row, size_t n, double u);
double orc_tree_reduce(const double* v, size_t n);

/* ---- verification ------------------------------------------------------- */
/* Outputs mirror VerificationResult (step.hpp:43-51): accepted_len[B],
 * tau[B*gamma], final_token[B], resample_used[B], residual_denom[B]. */
typedef struct {
    int32_t* accepted_len;
    double* tau;
    int32_t* final_token;
    uint8_t* resample_used;
    double* residual_denom;
} orc_result;

/* verify_reference.cpp:76-111 on probability grids.  p is B x p_steps x V
 * with p_steps in {gamma, gamma+1}; q is B x gamma x V. */
int orc_verify_sequential(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                          const int32_t* draft_tokens, const double* uniforms, orc_result* out);

/* verify_fused.cpp:13-105 (tree-reduced residual mass over tile_width tiles). */
int orc_verify_fused(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                     const int32_t* draft_tokens, const double* uniforms, int tile_width,
                     orc_result* out);

/* Logits-in exact step = materialize_softmax_into (activation.cpp:20-27) on
 * both grids followed by verify_sequential; the north star's exact API. */
int orc_verify_exact_logits(const double* z_p, int p_steps, const double* z_q, int B, int gamma,
                            int V, const int32_t* draft_tokens, const double* uniforms,
                            orc_result* out);

/* verify_sigmoid.cpp:50-58 (materialize_sigmoid + verify_sequential),
 * emulate_half = false. */
int orc_verify_sigmoid_sequential(const double* z_p, int p_steps, const double* z_q, int B,
                                  int gamma, int V, const int32_t* draft_tokens,
                                  const double* uniforms, double alpha, double beta,
                                  orc_result* out);

/* Materialized activations (for the optional p/q/residual outputs). */
int orc_softmax_grid(const double* z, size_t rows, int V, double* out);
void orc_sigmoid_grid(const double* z, size_t n, double alpha, double beta, double* out);

/* ---- input generators ----------------------------------------------------- */
/* bench.cpp:46-74 make_bench_inputs(seed, gamma, V) for ONE batch row:
 * z_p (gamma+1) x V, z_q gamma x V, ids [gamma], uniforms [gamma+1]. */
void orc_make_bench_inputs(uint64_t seed, int gamma, int V, double* z_p, double* z_q,
                           int32_t* ids, double* uniforms);
/* Same recipe for B batch rows (row b uses seed + b), threads > 1 splits rows. */
void orc_make_bench_batch(uint64_t seed, int B, int gamma, int V, int threads, double* z_p,
                          double* z_q, int32_t* ids, double* uniforms);

/* validate.cpp:57-82 make_instance: probability grids. */
void orc_make_instance(orc_rng* rng, int B, int gamma, int V, int bonus_row, double logit_scale,
                       double* p, double* q, int32_t* ids, double* uniforms);
/* Logit-space variant of make_instance: the same draws, but the softmax of
 * the logits is NOT taken for p (used for logits-in parity grids). */
void orc_make_logit_instance(orc_rng* rng, int B, int gamma, int V, int bonus_row,
                             double logit_scale, double* z_p, double* z_q, int32_t* ids,
                             double* uniforms);
/* validate.cpp:84-109 make_sigmoid_instance (emulate_half = false). */
void orc_make_sigmoid_instance(orc_rng* rng, int B, int gamma, int V, int bonus_row,
                               double logit_scale, double* z_p, double* z_q, int32_t* ids,
                               double* uniforms);

/* ---- storage rounding (RNE), so the oracle sees the device's exact bits --- */
void orc_round_f32(double* x, size_t n);
void orc_round_bf16(double* x, size_t n);
void orc_to_f32(const double* x, size_t n, float* out);
void orc_to_bf16(const double* x, size_t n, uint16_t* out);

#ifdef __cplusplus
}
#endif

#endif
