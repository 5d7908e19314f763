/*
 * benchgen.c -- synthetic benchmark inputs for bench.py (harness code, not the
 * verification path).
 *
 * Batch row b of a benchmark batch is the reference's make_bench_inputs(seed +
 * b, gamma, V) (/root/reference/proj/src/bench.cpp:46-74): z_p ~ 4 N(0,1) over
 * gamma + 1 rows, z_q = z_p + N(0,1) over gamma rows, draft ids sampled from
 * softmax(z_q) with sample_row, then gamma + 1 uniforms, all from the counter
 * RNG of rng.cpp:12-33 in that order.  The logits are stored rounded to the
 * benchmark's storage type (fp32 RNE, or fp32 -> bf16 RNE); the draft ids are
 * sampled from the unrounded double logits exactly as the reference does.
 *
 * Both benchmark arms consume these bits: the GPU arm copies them to the
 * device, the reference arm (bench.py --impl reference) widens the same rows to
 * double for the compiled reference.  tests/test_benchgen.py pins this file
 * bit for bit against the compiled reference's own make_bench_inputs.
 *
 * Batch rows are independent, so they are generated in parallel (pthreads),
 * straight into the caller's (pinned) buffers.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint64_t seed, counter;
} bg_rng;

static uint64_t bg_mix64(uint64_t z) { /* rng.cpp:14-18 */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static uint64_t bg_next(bg_rng* r) { /* rng.cpp:20-22: word at index counter++ */
    const uint64_t i = r->counter++;
    return bg_mix64(r->seed + (i + 1) * 0x9e3779b97f4a7c15ull);
}
static double bg_uniform(bg_rng* r) { return (double)(bg_next(r) >> 11) * 0x1.0p-53; } /* rng.cpp:24-26 */
static double bg_normal(bg_rng* r) {                                                    /* rng.cpp:28-33 */
    const double u1 = ((double)(bg_next(r) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = bg_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* stable_softmax_into (dist.cpp:40-51) + detail::sample_row (verify_reference.cpp:40-43,
 * dist.cpp:114-137) on one row; `prob` is scratch of n doubles. */
static int32_t bg_sample_softmax(const double* z, size_t n, double* prob, double u) {
    double mx = z[0];
    for (size_t i = 1; i < n; ++i)
        if (mx < z[i]) mx = z[i];
    double denom = 0.0;
    for (size_t i = 0; i < n; ++i) {
        prob[i] = exp(z[i] - mx);
        denom += prob[i];
    }
    for (size_t i = 0; i < n; ++i) prob[i] /= denom;
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += prob[i];
    double cum = 0.0;
    size_t last = 0;
    int saw = 0;
    for (size_t i = 0; i < n; ++i) {
        if (prob[i] > 0.0) {
            last = i;
            saw = 1;
        }
        cum += prob[i] / s;
        if (u < cum) return (int32_t)i;
    }
    return (int32_t)(saw ? last : 0);
}

static uint16_t bg_bf16(float f) { /* fp32 -> bf16 round to nearest even */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

static void bg_store(void* dst, size_t i, double v, int dtype) {
    if (dtype == 0) ((float*)dst)[i] = (float)v;
    else if (dtype == 1) ((uint16_t*)dst)[i] = bg_bf16((float)v);
    else ((double*)dst)[i] = v;
}

/* One batch row: make_bench_inputs(seed, gamma, V) -> stored logits (dtype 0
 * fp32, 1 bf16, 2 fp64), ids[gamma], uniforms[gamma + 1]. */
static void bg_row(uint64_t seed, int gamma, int V, int dtype, void* zp, void* zq, int32_t* ids, double* u,
                   double* zpd, double* zqd, double* prob) {
    bg_rng rng = {seed, 0};
    const size_t Vs = (size_t)V, g = (size_t)gamma;
    for (size_t i = 0; i < (g + 1) * Vs; ++i) zpd[i] = 4.0 * bg_normal(&rng); /* kBenchLogitScale */
    for (size_t c = 0; c < g; ++c)
        for (size_t i = 0; i < Vs; ++i) zqd[c * Vs + i] = zpd[c * Vs + i] + 1.0 * bg_normal(&rng); /* kBenchDraftJitter */
    for (size_t c = 0; c < g; ++c) ids[c] = bg_sample_softmax(zqd + c * Vs, Vs, prob, bg_uniform(&rng));
    for (size_t c = 0; c <= g; ++c) u[c] = bg_uniform(&rng);
    for (size_t i = 0; i < (g + 1) * Vs; ++i) bg_store(zp, i, zpd[i], dtype);
    for (size_t i = 0; i < g * Vs; ++i) bg_store(zq, i, zqd[i], dtype);
}

typedef struct {
    uint64_t seed;
    int B, gamma, V, dtype, t, nt;
    char *zp, *zq;
    int32_t* ids;
    double* u;
} bg_job;

static void* bg_worker(void* arg) {
    bg_job* j = (bg_job*)arg;
    const size_t Vs = (size_t)j->V, g = (size_t)j->gamma;
    const size_t es = j->dtype == 0 ? 4 : (j->dtype == 1 ? 2 : 8);
    double* zpd = (double*)malloc((g + 1) * Vs * sizeof(double));
    double* zqd = (double*)malloc((g ? g : 1) * Vs * sizeof(double));
    double* prob = (double*)malloc(Vs * sizeof(double));
    for (int b = j->t; b < j->B; b += j->nt) /* interleaved: rows cost the same */
        bg_row(j->seed + (uint64_t)b, j->gamma, j->V, j->dtype, j->zp + (size_t)b * (g + 1) * Vs * es,
               j->zq + (size_t)b * g * Vs * es, j->ids + (size_t)b * g, j->u + (size_t)b * (g + 1), zpd, zqd, prob);
    free(zpd);
    free(zqd);
    free(prob);
    return NULL;
}

/* B batch rows, row b seeded seed + b.  z_p [B][gamma+1][V], z_q [B][gamma][V]
 * in the storage type, ids [B][gamma], uniforms [B][gamma+1].  Returns 0. */
int bg_make_bench_batch(uint64_t seed, int B, int gamma, int V, int dtype, int threads, void* z_p, void* z_q,
                        int32_t* ids, double* uniforms) {
    if (B < 1 || gamma < 1 || V < 1 || dtype < 0 || dtype > 2) return 2;
    if (threads < 1) threads = 1;
    if (threads > B) threads = B;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    bg_job* jobs = (bg_job*)malloc(sizeof(bg_job) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (bg_job){seed, B, gamma, V, dtype, t, threads, (char*)z_p, (char*)z_q, ids, uniforms};
        pthread_create(&th[t], NULL, bg_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}

/* toy_model.cpp:16-42 make_model_pair: target table = logit_scale * N(0,1)
 * from stream `seed`, draft = target + divergence * N(0,1) from stream
 * seed ^ 0xd1f (row-major [V][V], doubles).  The ablation's input tables. */
int bg_make_model_pair(uint64_t seed, int V, double divergence, double logit_scale, double* target, double* draft) {
    if (V < 2 || divergence < 0.0) return 1;
    const size_t n = (size_t)V * (size_t)V;
    bg_rng t = {seed, 0};
    for (size_t i = 0; i < n; ++i) target[i] = logit_scale * bg_normal(&t);
    bg_rng d = {seed ^ 0xd1fu, 0};
    for (size_t i = 0; i < n; ++i) draft[i] = target[i] + divergence * bg_normal(&d);
    return 0;
}
