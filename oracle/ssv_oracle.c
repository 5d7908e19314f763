/*
 * ssv_oracle.c -- TEST INFRASTRUCTURE ONLY (see ssv_oracle.h).
 *
 * Plain-C restatement of the reference's verification path.  Each function
 * cites the file:line under /root/reference/proj it follows.  Arithmetic is
 * double throughout and the evaluation order of every sum matches the
 * reference, so results are bit-identical to it (checked against the compiled
 * reference in tests/test_oracle.py).
 */
#include "ssv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.cpp:12-33 ------------------------------------------------------- */
static uint64_t mix64(uint64_t z) { /* rng.cpp:14-18 SplitMix64 finalizer */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

uint64_t orc_word_at(uint64_t seed, uint64_t index) { /* rng.cpp:20-22 */
    return mix64(seed + (index + 1) * 0x9e3779b97f4a7c15ull);
}

uint64_t orc_next_u64(orc_rng* r) { return orc_word_at(r->seed, r->counter++); } /* rng.hpp:18 */

double orc_next_uniform(orc_rng* r) { /* rng.cpp:24-26 */
    return (double)(orc_next_u64(r) >> 11) * 0x1.0p-53;
}

double orc_next_normal(orc_rng* r) { /* rng.cpp:28-33 */
    const double u1 = ((double)(orc_next_u64(r) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = orc_next_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* ---- dist.cpp ------------------------------------------------------------ */
double orc_stable_sigmoid(double t) { /* dist.cpp:17-23 */
    if (t >= 0.0) return 1.0 / (1.0 + exp(-t));
    const double e = exp(t);
    return e / (1.0 + e);
}

int orc_stable_softmax_into(const double* z, size_t n, double* out) { /* dist.cpp:40-51 */
    if (n == 0) return ORC_EINVAL; /* require_finite, dist.cpp:27-36 */
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(z[i])) return ORC_EINVAL;
    double mx = z[0]; /* std::max_element: first maximum */
    for (size_t i = 1; i < n; ++i)
        if (mx < z[i]) mx = z[i];
    double denom = 0.0;
    for (size_t i = 0; i < n; ++i) {
        out[i] = exp(z[i] - mx);
        denom += out[i];
    }
    for (size_t i = 0; i < n; ++i) out[i] /= denom;
    return ORC_OK;
}

double orc_sigmoid_scaled_value(double z, double alpha, double beta) { /* dist.cpp:60-62 */
    return orc_stable_sigmoid((z - alpha) / (beta - alpha));
}

int orc_ratio_clamped(double p, double q, double* out) { /* dist.cpp:104-112 */
    if (p < 0.0 || q < 0.0) return ORC_EINVAL;
    if (q <= ORC_ZERO_EPS) {
        *out = p > ORC_ZERO_EPS ? 1.0 : 0.0;
        return ORC_OK;
    }
    const double r = p / q;
    *out = r < 1.0 ? r : 1.0; /* std::min(1.0, p / q) */
    return ORC_OK;
}

double orc_sequential_sum(const double* v, size_t n) { /* dist.cpp:114-120 */
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += v[i];
    return s;
}

size_t orc_scan_categorical(const double* v, size_t n, double denom, double u) { /* dist.cpp:122-137 */
    double cum = 0.0;
    size_t last_positive = 0;
    int saw_positive = 0;
    for (size_t i = 0; i < n; ++i) {
        if (v[i] > 0.0) {
            last_positive = i;
            saw_positive = 1;
        }
        cum += v[i] / denom;
        if (u < cum) return i;
    }
    return saw_positive ? last_positive : 0;
}

int32_t orc_sample_row(const double* row, size_t n, double u) { /* verify_reference.cpp:40-43 */
    const double denom = orc_sequential_sum(row, n);
    return (int32_t)orc_scan_categorical(row, n, denom, u);
}

static size_t bit_ceil(size_t n) {
    size_t m = 1;
    while (m < n) m <<= 1;
    return m;
}

double orc_tree_reduce(const double* v, size_t n) { /* tile.cpp:33-44 */
    if (n == 0) return 0.0;
    const size_t m = bit_ceil(n);
    double* s = (double*)calloc(m, sizeof(double));
    memcpy(s, v, n * sizeof(double));
    for (size_t stride = m >> 1; stride >= 1; stride >>= 1)
        for (size_t i = 0; i < stride; ++i) s[i] += s[i + stride];
    const double r = s[0];
    free(s);
    return r;
}

/* ---- verify_reference.cpp ---------------------------------------------- */
static int validate_common(int B, int gamma, int V, int p_steps, const int32_t* ids,
                           const double* uniforms, int check_uniforms) {
    /* StepInputs::validate, verify_reference.cpp:11-36 (and the sigmoid
     * variant verify_sigmoid.cpp:13-33, which skips the uniform check). */
    if (B < 1 || gamma < 1 || V < 1) return ORC_EINVAL;
    if (p_steps != gamma && p_steps != gamma + 1) return ORC_EINVAL;
    for (int b = 0; b < B; ++b) {
        for (int c = 0; c < gamma; ++c) {
            const int32_t t = ids[(size_t)b * gamma + c];
            if (t < 0 || t >= V) return ORC_EINVAL;
        }
        if (check_uniforms) {
            for (int c = 0; c <= gamma; ++c) {
                const double u = uniforms[(size_t)b * (gamma + 1) + c];
                if (!(u >= 0.0) || !(u < 1.0)) return ORC_EINVAL;
            }
        }
    }
    return ORC_OK;
}

/* verify_reference.cpp:45-65 resample_with_denom */
static void resample_with_denom(const double* p_row, const double* q_row, size_t n, double u,
                                int32_t* token, double* denom_out, int* used_fallback) {
    double* residual = (double*)malloc(n * sizeof(double));
    double denom = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = p_row[i] - q_row[i];
        const double a = d > 0.0 ? d : 0.0; /* std::max(0.0, d) */
        residual[i] = a;
        denom += a;
    }
    *denom_out = denom;
    if (denom <= ORC_ZERO_EPS) {
        *used_fallback = 1;
        *token = orc_sample_row(p_row, n, u);
    } else {
        *used_fallback = 0;
        *token = (int32_t)orc_scan_categorical(residual, n, denom, u);
    }
    free(residual);
}

int orc_verify_sequential(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                          const int32_t* ids, const double* uniforms, orc_result* out) {
    /* verify_reference.cpp:76-111 */
    int rc = validate_common(B, gamma, V, p_steps, ids, uniforms, 1);
    if (rc) return rc;
    const size_t Vs = (size_t)V;
    for (int b = 0; b < B; ++b) {
        for (int c = 0; c < gamma; ++c) {
            const size_t tok = (size_t)ids[(size_t)b * gamma + c];
            const double pv = p[((size_t)b * p_steps + c) * Vs + tok];
            const double qv = q[((size_t)b * gamma + c) * Vs + tok];
            rc = orc_ratio_clamped(pv, qv, &out->tau[(size_t)b * gamma + c]);
            if (rc) return rc;
        }
    }
    for (int b = 0; b < B; ++b) {
        const double* u = uniforms + (size_t)b * (gamma + 1);
        const double* tau = out->tau + (size_t)b * gamma;
        int accepted = 0;
        while (accepted < gamma && u[accepted] <= tau[accepted]) ++accepted;
        out->accepted_len[b] = accepted;
        out->final_token[b] = ORC_NO_TOKEN;
        out->resample_used[b] = 0;
        out->residual_denom[b] = 0.0;
        const double u_final = u[gamma];
        if (accepted < gamma) {
            int32_t tok;
            double denom;
            int fb;
            resample_with_denom(p + ((size_t)b * p_steps + accepted) * Vs,
                                q + ((size_t)b * gamma + accepted) * Vs, Vs, u_final, &tok, &denom,
                                &fb);
            out->final_token[b] = tok;
            out->resample_used[b] = 1;
            out->residual_denom[b] = fb ? 0.0 : denom;
        } else if (p_steps == gamma + 1) {
            out->final_token[b] = orc_sample_row(p + ((size_t)b * p_steps + gamma) * Vs, Vs, u_final);
        }
    }
    return ORC_OK;
}

int orc_verify_fused(const double* p, int p_steps, const double* q, int B, int gamma, int V,
                     const int32_t* ids, const double* uniforms, int tile_width,
                     orc_result* out) {
    /* verify_fused.cpp:13-100 with plan_tiles (tile.cpp:11-23) and the
     * per-tile tree_reduce of tile_pass_core (tile.cpp:93-96).  The residual
     * is kept in a private buffer instead of overwriting q. */
    int rc = validate_common(B, gamma, V, p_steps, ids, uniforms, 1);
    if (rc) return rc;
    if (tile_width < 1) return ORC_EINVAL;
    const size_t Vs = (size_t)V, n = (size_t)tile_width;
    const size_t K = (Vs + n - 1) / n;
    double* partials = (double*)malloc(K * sizeof(double));
    double* a = (double*)malloc(Vs * sizeof(double));
    for (int b = 0; b < B; ++b) {
        for (int c = 0; c < gamma; ++c) {
            const size_t tok = (size_t)ids[(size_t)b * gamma + c];
            rc = orc_ratio_clamped(p[((size_t)b * p_steps + c) * Vs + tok],
                                   q[((size_t)b * gamma + c) * Vs + tok],
                                   &out->tau[(size_t)b * gamma + c]);
            if (rc) goto done;
        }
        const double* u = uniforms + (size_t)b * (gamma + 1);
        const double* tau = out->tau + (size_t)b * gamma;
        int accepted = 0;
        while (accepted < gamma && u[accepted] <= tau[accepted]) ++accepted;
        out->accepted_len[b] = accepted;
        out->final_token[b] = ORC_NO_TOKEN;
        out->resample_used[b] = 0;
        out->residual_denom[b] = 0.0;
        const double u_final = u[gamma];
        if (accepted < gamma) {
            const double* pr = p + ((size_t)b * p_steps + accepted) * Vs;
            const double* qr = q + ((size_t)b * gamma + accepted) * Vs;
            for (size_t i = 0; i < Vs; ++i) {
                const double d = pr[i] - qr[i];
                a[i] = d > 0.0 ? d : 0.0;
            }
            for (size_t k = 0; k < K; ++k) {
                const size_t beg = k * n, end = beg + n < Vs ? beg + n : Vs;
                partials[k] = orc_tree_reduce(a + beg, end - beg);
            }
            out->resample_used[b] = 1;
            const double denom = orc_tree_reduce(partials, K); /* verify_fused.cpp:84 */
            if (denom > ORC_ZERO_EPS) {
                out->residual_denom[b] = denom;
                out->final_token[b] = (int32_t)orc_scan_categorical(a, Vs, denom, u_final);
            } else {
                out->final_token[b] = orc_sample_row(pr, Vs, u_final);
            }
        } else if (p_steps == gamma + 1) {
            out->final_token[b] = orc_sample_row(p + ((size_t)b * p_steps + gamma) * Vs, Vs, u_final);
        }
    }
done:
    free(partials);
    free(a);
    return rc;
}

int orc_softmax_grid(const double* z, size_t rows, int V, double* out) { /* activation.cpp:20-27 */
    for (size_t r = 0; r < rows; ++r) {
        const int rc = orc_stable_softmax_into(z + r * (size_t)V, (size_t)V, out + r * (size_t)V);
        if (rc) return rc;
    }
    return ORC_OK;
}

void orc_sigmoid_grid(const double* z, size_t n, double alpha, double beta, double* out) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_sigmoid_scaled_value(z[i], alpha, beta); /* verify_sigmoid.cpp:39-48 */
}

int orc_verify_exact_logits(const double* z_p, int p_steps, const double* z_q, int B, int gamma,
                            int V, const int32_t* ids, const double* uniforms, orc_result* out) {
    const size_t np = (size_t)B * p_steps * V, nq = (size_t)B * gamma * V;
    double* p = (double*)malloc(np * sizeof(double));
    double* q = (double*)malloc(nq * sizeof(double));
    int rc = validate_common(B, gamma, V, p_steps, ids, uniforms, 1);
    if (!rc) rc = orc_softmax_grid(z_p, (size_t)B * p_steps, V, p);
    if (!rc) rc = orc_softmax_grid(z_q, (size_t)B * gamma, V, q);
    if (!rc) rc = orc_verify_sequential(p, p_steps, q, B, gamma, V, ids, uniforms, out);
    free(p);
    free(q);
    return rc;
}

int orc_verify_sigmoid_sequential(const double* z_p, int p_steps, const double* z_q, int B,
                                  int gamma, int V, const int32_t* ids, const double* uniforms,
                                  double alpha, double beta, orc_result* out) {
    /* verify_sigmoid.cpp:50-58; bounds.validate() dist.cpp:11-15 */
    if (!isfinite(alpha) || !isfinite(beta) || !(alpha < 0.0) || !(beta > 0.0)) return ORC_EINVAL;
    int rc = validate_common(B, gamma, V, p_steps, ids, uniforms, 0);
    if (rc) return rc;
    const size_t np = (size_t)B * p_steps * V, nq = (size_t)B * gamma * V;
    double* p = (double*)malloc(np * sizeof(double));
    double* q = (double*)malloc(nq * sizeof(double));
    orc_sigmoid_grid(z_p, np, alpha, beta, p);
    orc_sigmoid_grid(z_q, nq, alpha, beta, q);
    rc = orc_verify_sequential(p, p_steps, q, B, gamma, V, ids, uniforms, out);
    free(p);
    free(q);
    return rc;
}

/* ---- generators -------------------------------------------------------- */
void orc_make_bench_inputs(uint64_t seed, int gamma, int V, double* z_p, double* z_q,
                           int32_t* ids, double* uniforms) {
    /* bench.cpp:46-74: kBenchLogitScale = 4, kBenchDraftJitter = 1 (35-36). */
    orc_rng rng = {seed, 0};
    const size_t Vs = (size_t)V, g = (size_t)gamma;
    for (size_t i = 0; i < (g + 1) * Vs; ++i) z_p[i] = 4.0 * orc_next_normal(&rng);
    for (size_t c = 0; c < g; ++c)
        for (size_t i = 0; i < Vs; ++i)
            z_q[c * Vs + i] = z_p[c * Vs + i] + 1.0 * orc_next_normal(&rng);
    double* prob = (double*)malloc(Vs * sizeof(double));
    for (size_t c = 0; c < g; ++c) {
        orc_stable_softmax_into(z_q + c * Vs, Vs, prob);
        ids[c] = orc_sample_row(prob, Vs, orc_next_uniform(&rng));
    }
    for (size_t c = 0; c <= g; ++c) uniforms[c] = orc_next_uniform(&rng);
    free(prob);
}

typedef struct {
    uint64_t seed;
    int b0, b1, gamma, V;
    double *z_p, *z_q, *u;
    int32_t* ids;
} bench_job;

static void* bench_worker(void* arg) {
    bench_job* j = (bench_job*)arg;
    const size_t Vs = (size_t)j->V, g = (size_t)j->gamma;
    for (int b = j->b0; b < j->b1; ++b)
        orc_make_bench_inputs(j->seed + (uint64_t)b, j->gamma, j->V, j->z_p + (size_t)b * (g + 1) * Vs,
                              j->z_q + (size_t)b * g * Vs, j->ids + (size_t)b * g,
                              j->u + (size_t)b * (g + 1));
    return NULL;
}

void orc_make_bench_batch(uint64_t seed, int B, int gamma, int V, int threads, double* z_p,
                          double* z_q, int32_t* ids, double* uniforms) {
    if (threads < 1) threads = 1;
    if (threads > B) threads = B;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    bench_job* jobs = (bench_job*)malloc(sizeof(bench_job) * threads);
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (bench_job){seed, (int)((long)B * t / threads), (int)((long)B * (t + 1) / threads),
                              gamma, V, z_p, z_q, uniforms, ids};
        pthread_create(&th[t], NULL, bench_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
}

void orc_make_instance(orc_rng* rng, int B, int gamma, int V, int bonus_row, double logit_scale,
                       double* p, double* q, int32_t* ids, double* uniforms) {
    /* validate.cpp:57-82 */
    const size_t Vs = (size_t)V, g = (size_t)gamma, ps = g + (bonus_row ? 1 : 0);
    double* logits = (double*)malloc(Vs * sizeof(double));
    for (int b = 0; b < B; ++b) {
        for (size_t c = 0; c < ps; ++c) {
            for (size_t i = 0; i < Vs; ++i) logits[i] = logit_scale * orc_next_normal(rng);
            orc_stable_softmax_into(logits, Vs, p + ((size_t)b * ps + c) * Vs);
        }
        for (size_t c = 0; c < g; ++c) {
            for (size_t i = 0; i < Vs; ++i) logits[i] = logit_scale * orc_next_normal(rng);
            double* qr = q + ((size_t)b * g + c) * Vs;
            orc_stable_softmax_into(logits, Vs, qr);
            ids[(size_t)b * g + c] = orc_sample_row(qr, Vs, orc_next_uniform(rng));
        }
        for (size_t c = 0; c <= g; ++c) uniforms[(size_t)b * (g + 1) + c] = orc_next_uniform(rng);
    }
    free(logits);
}

void orc_make_logit_instance(orc_rng* rng, int B, int gamma, int V, int bonus_row,
                             double logit_scale, double* z_p, double* z_q, int32_t* ids,
                             double* uniforms) {
    const size_t Vs = (size_t)V, g = (size_t)gamma, ps = g + (bonus_row ? 1 : 0);
    double* prob = (double*)malloc(Vs * sizeof(double));
    for (int b = 0; b < B; ++b) {
        for (size_t c = 0; c < ps; ++c)
            for (size_t i = 0; i < Vs; ++i)
                z_p[((size_t)b * ps + c) * Vs + i] = logit_scale * orc_next_normal(rng);
        for (size_t c = 0; c < g; ++c) {
            double* zr = z_q + ((size_t)b * g + c) * Vs;
            for (size_t i = 0; i < Vs; ++i) zr[i] = logit_scale * orc_next_normal(rng);
            orc_stable_softmax_into(zr, Vs, prob);
            ids[(size_t)b * g + c] = orc_sample_row(prob, Vs, orc_next_uniform(rng));
        }
        for (size_t c = 0; c <= g; ++c) uniforms[(size_t)b * (g + 1) + c] = orc_next_uniform(rng);
    }
    free(prob);
}

void orc_make_sigmoid_instance(orc_rng* rng, int B, int gamma, int V, int bonus_row,
                               double logit_scale, double* z_p, double* z_q, int32_t* ids,
                               double* uniforms) {
    /* validate.cpp:84-109 */
    const size_t Vs = (size_t)V, g = (size_t)gamma, ps = g + (bonus_row ? 1 : 0);
    for (size_t i = 0; i < (size_t)B * ps * Vs; ++i) z_p[i] = logit_scale * orc_next_normal(rng);
    for (size_t i = 0; i < (size_t)B * g * Vs; ++i) z_q[i] = logit_scale * orc_next_normal(rng);
    double* prob = (double*)malloc(Vs * sizeof(double));
    for (int b = 0; b < B; ++b) {
        for (size_t c = 0; c < g; ++c) {
            orc_stable_softmax_into(z_q + ((size_t)b * g + c) * Vs, Vs, prob);
            ids[(size_t)b * g + c] = orc_sample_row(prob, Vs, orc_next_uniform(rng));
        }
        for (size_t c = 0; c <= g; ++c) uniforms[(size_t)b * (g + 1) + c] = orc_next_uniform(rng);
    }
    free(prob);
}

/* ---- rounding ------------------------------------------------------------ */
void orc_round_f32(double* x, size_t n) {
    for (size_t i = 0; i < n; ++i) x[i] = (double)(float)x[i];
}

static uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40);
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

static double bf16_to_double(uint16_t h) {
    const uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

void orc_round_bf16(double* x, size_t n) {
    /* double -> float (RNE) -> bf16 (RNE).  Double rounding can differ from a
     * direct double->bf16 RNE only on exact float ties; the device consumes
     * exactly these bits, so the oracle stays consistent with it. */
    for (size_t i = 0; i < n; ++i) x[i] = bf16_to_double(f32_to_bf16_rne((float)x[i]));
}

void orc_to_f32(const double* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = (float)x[i];
}

void orc_to_bf16(const double* x, size_t n, uint16_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = f32_to_bf16_rne((float)x[i]);
}
