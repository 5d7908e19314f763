// ssv_kernels.cu -- sm_100a kernels of the speculative-sampling verification step.
//
// Path (DESIGN.md has the full derivation):
//   K1 k_row_stats   exact variant only.  One CTA per (row, 8K-element chunk) of
//                    the 2*gamma drafted rows (+ the bonus row when p is
//                    materialized): 128-bit streaming loads into registers, CTA
//                    max, fp32 ex2 sums with fp64 carries -> chunk partial
//                    (m, s).  The LAST CTA of each batch row (completion counter)
//                    folds the partials into row statistics, evaluates tau at
//                    every drafted position in fp64, runs the first-rejection
//                    scan and records what the batch row still needs.
//   K2 k_row_pass    every variant.  One warp per 512-element granule of the
//                    ONE row (bonus) or row PAIR (rejected position) a batch row
//                    still needs; granule masses of max(0, p - q) (or of p) with
//                    fp64 carries.  The LAST CTA of each batch row does the
//                    inverse CDF: granule prefix in fp64, then an fp64 element
//                    scan inside the selected granule -- dist.cpp:122-137
//                    semantics including the last-positive fallback.  For the
//                    sigmoid and probability variants K2 is the whole step: its
//                    CTAs evaluate tau from the B*gamma gathered logits
//                    themselves (no row reductions).
//   K3 k_materialize optional p / q / residual grids.
//   generator / sampler kernels for the callers either side of the path.
#include <type_traits>

#include "ssv_launch.h"
#include "ssv_device.cuh"

namespace ssv {

// ---------------------------------------------------------------------------
// Row addressing.  Stat rows of batch row b: r < G -> p row r, G <= r < 2G ->
// q row r-G, r == 2G -> p row G (bonus, only when p is materialized).
template <typename T>
__device__ __forceinline__ const T* p_row(const StepParams& P, int b, int c) {
    return reinterpret_cast<const T*>(P.zp) + ((size_t)b * P.PS + c) * (size_t)P.V;
}
template <typename T>
__device__ __forceinline__ const T* q_row(const StepParams& P, int b, int c) {
    return reinterpret_cast<const T*>(P.zq) + ((size_t)b * P.G + c) * (size_t)P.V;
}
template <typename T>
__device__ __forceinline__ const T* stat_row(const StepParams& P, int b, int r) {
    if (r < P.G) return p_row<T>(P, b, r);
    if (r < 2 * P.G) return q_row<T>(P, b, r - P.G);
    return p_row<T>(P, b, P.G);
}

__device__ __forceinline__ void flag(const StepParams& P, uint32_t bits) { atomicOr(P.status, bits); }

__device__ __forceinline__ double ratio_clamped(double p, double q) {  // dist.cpp:104-112
    if (q <= kZeroEps) return p > kZeroEps ? 1.0 : 0.0;
    return fmin(1.0, p / q);
}

// ---------------------------------------------------------------------------
// Register tile of one warp over [lo, hi) of one row: NV 16-byte vectors per
// lane plus at most one peeled scalar (head to the first 16-byte boundary,
// lanes 0..; tail, lanes 16..).
template <typename T, int NV>
struct WarpTile {
    using A = typename Elem<T>::acc;
    static constexpr int VEC = Elem<T>::VEC;
    uint4 v[NV];
    int nvec;
    A xs;
    bool has_x;

    __device__ __forceinline__ void load(const T* row, int lo, int hi) {
        const int lane = threadIdx.x & 31;
        const Span16<T> s = split16(row, lo, hi);
        nvec = s.nvec;
        const T* vb = row + s.vec_begin;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int idx = j * 32 + lane;
            if (idx < nvec) v[j] = ldg_stream(vb + (size_t)idx * VEC);
        }
        has_x = false;
        const int nh = s.head_end - lo, nt = hi - s.tail_begin;
        if (lane < nh) {
            xs = load_elem(row + lo + lane);
            has_x = true;
        } else if (lane >= 16 && lane - 16 < nt) {
            xs = load_elem(row + s.tail_begin + (lane - 16));
            has_x = true;
        }
    }

    __device__ __forceinline__ void minmax(A& mx, A& mn) const {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            if (j * 32 + lane < nvec) {
                A x[VEC];
                unpack(v[j], x);
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    mx = fmax(mx, x[e]);
                    mn = fmin(mn, x[e]);
                }
            }
        }
        if (has_x) {
            mx = fmax(mx, xs);
            mn = fmin(mn, xs);
        }
    }

    // sum of e^(x - m): fp32 within a 16-byte vector, fp64 across vectors.
    __device__ __forceinline__ double sum_exp(A m) const {
        const int lane = threadIdx.x & 31;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            if (j * 32 + lane < nvec) {
                A x[VEC];
                unpack(v[j], x);
                A t = 0;
#pragma unroll
                for (int e = 0; e < VEC; ++e) t += exp_rel(x[e], m);
                s += (double)t;
            }
        }
        if (has_x) s += (double)exp_rel(xs, m);
        return s;
    }

    template <typename F>
    __device__ __forceinline__ double sum_map(F f) const {
        const int lane = threadIdx.x & 31;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            if (j * 32 + lane < nvec) {
                A x[VEC];
                unpack(v[j], x);
                A t = 0;
#pragma unroll
                for (int e = 0; e < VEC; ++e) t += f(x[e]);
                s += (double)t;
            }
        }
        if (has_x) s += (double)f(xs);
        return s;
    }
};

// ---------------------------------------------------------------------------
// K1 epilogue: the last CTA of batch row b.  Row statistics from the chunk
// partials (fixed order, fp64), tau at every drafted position (fp64, from the
// gathered logits -- activation.cpp:20-27 + verify_reference.cpp:87-92),
// first rejection (verify_reference.cpp:93-96, inclusive u <= tau).
template <typename T>
__device__ void decide_softmax(const StepParams& P, int b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = P.G;
    for (int r = warp; r < P.NR; r += kWarps) {
        const double2* part = P.part + ((size_t)b * P.NR + r) * P.K;
        double m = -CUDART_INF;
        for (int k = lane; k < P.K; k += 32) m = fmax(m, __ldcg(&part[k].x));
        m = warp_max(m);
        double s = 0.0;
        for (int k = lane; k < P.K; k += 32) {
            const double2 pk = __ldcg(&part[k]);
            if (pk.y > 0.0) s += pk.y * exp(pk.x - m);
        }
        s = warp_sum(s);
        if (lane == 0) P.rowstat[(size_t)b * P.NR + r] = make_double2(m, s);
    }
    __syncthreads();
    const double2* rs = P.rowstat + (size_t)b * P.NR;
    for (int c = threadIdx.x; c < G; c += kThreads) {
        int x = P.ids[(size_t)b * G + c];
        if (x < 0 || x >= P.V) {
            flag(P, SSV_STATUS_TOKEN_RANGE);
            x = x < 0 ? 0 : P.V - 1;
        }
        const double2 sp = rs[c], sq = rs[G + c];
        const double zp = load_exact(p_row<T>(P, b, c) + x);
        const double zq = load_exact(q_row<T>(P, b, c) + x);
        const double p = exp(zp - sp.x) / sp.y;
        const double q = exp(zq - sq.x) / sq.y;
        P.tau[(size_t)b * G + c] = ratio_clamped(p, q);
    }
    if (P.check_uniforms) {
        for (int c = threadIdx.x; c <= G; c += kThreads) {
            const double u = P.u[(size_t)b * (G + 1) + c];
            if (!(u >= 0.0) || !(u < 1.0)) flag(P, SSV_STATUS_UNIFORM_RANGE);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double* u = P.u + (size_t)b * (G + 1);
        const double* tau = P.tau + (size_t)b * G;
        int a = 0;
        while (a < G && u[a] <= tau[a]) ++a;
        P.acc[b] = a;
        Decision d{};
        if (a < G) {
            d.mode = MODE_REJECT;
            d.row = a;
            d.Mp = rs[a].x;
            d.Sp = rs[a].y;
            d.Mq = rs[G + a].x;
            d.Sq = rs[G + a].y;
        } else if (P.PS == G + 1) {
            d.mode = MODE_BONUS;
            d.row = G;
        } else {
            d.mode = MODE_NONE;
            P.fin[b] = -1;  // kNoToken, step.hpp:11
            P.rsu[b] = 0;
            P.rden[b] = 0.0;
        }
        P.dec[b] = d;
    }
}

template <typename T, int NV>
__global__ void __launch_bounds__(kThreads) k_row_stats(StepParams P) {
    using A = typename Elem<T>::acc;
    constexpr int W = 32 * NV * Elem<T>::VEC;  // elements per warp
    const int warp = threadIdx.x >> 5;
    const int task = blockIdx.x;
    const int k = task % P.K;
    const int br = task / P.K;
    const int r = br % P.NR;
    const int b = br / P.NR;
    const T* row = stat_row<T>(P, b, r);
    const int lo = min(k * P.CH + warp * W, P.V);
    const int hi = min(lo + W, P.V);

    WarpTile<T, NV> t;
    t.load(row, lo, hi);
    A mx = -CUDART_INF_F, mn = CUDART_INF_F;
    if constexpr (sizeof(A) == 8) {
        mx = -CUDART_INF;
        mn = CUDART_INF;
    }
    t.minmax(mx, mn);

    __shared__ A s_mx[kWarps], s_mn[kWarps];
    __shared__ double s_sum[kWarps];
    __shared__ bool s_last;
    mx = warp_max(mx);
    mn = warp_min(mn);
    if ((threadIdx.x & 31) == 0) {
        s_mx[warp] = mx;
        s_mn[warp] = mn;
    }
    __syncthreads();
    A M = s_mx[0], MN = s_mn[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
        M = fmax(M, s_mx[w]);
        MN = fmin(MN, s_mn[w]);
    }
    double s = warp_sum(t.sum_exp(M));
    if ((threadIdx.x & 31) == 0) s_sum[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double S = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) S += s_sum[w];
        P.part[task] = make_double2((double)M, S);
        if (!isfinite((double)M) || isnan(S) || !isfinite((double)MN)) flag(P, SSV_STATUS_NONFINITE);
        __threadfence();
        const unsigned prev = atomicAdd(&P.cnt1[b], 1u);
        s_last = (prev == (unsigned)(P.NR * P.K - 1));
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) P.cnt1[b] = 0;  // self-resetting for the next call
    decide_softmax<T>(P, b);
}

// ---------------------------------------------------------------------------
// Gathered-logit decision for the sigmoid / probability variants (one warp).
// verify_sigmoid.cpp:50-58 -> verify_reference.cpp:87-96; the sigmoid is
// evaluated in fp64 exactly as dist.cpp:60-62 does.
template <typename T, int ACT>
__device__ void decide_gather(const StepParams& P, int b, bool write, int& mode, int& row) {
    const int lane = threadIdx.x & 31;
    const int G = P.G;
    int accepted = G;
    for (int c0 = 0; c0 < G; c0 += 32) {
        const int c = c0 + lane;
        bool rej = false;
        if (c < G) {
            int x = P.ids[(size_t)b * G + c];
            if (x < 0 || x >= P.V) {
                if (write) flag(P, SSV_STATUS_TOKEN_RANGE);
                x = x < 0 ? 0 : P.V - 1;
            }
            const double zp = load_exact(p_row<T>(P, b, c) + x);
            const double zq = load_exact(q_row<T>(P, b, c) + x);
            double p, q;
            if (ACT == ACT_SIGMOID) {
                p = sigmoid_scaled_d(zp, P.alpha, P.width);
                q = sigmoid_scaled_d(zq, P.alpha, P.width);
            } else {
                p = zp;
                q = zq;
                if (write && (p < 0.0 || q < 0.0)) flag(P, SSV_STATUS_NEGATIVE);
            }
            const double tau = ratio_clamped(p, q);
            if (write) P.tau[(size_t)b * G + c] = tau;
            rej = !(P.u[(size_t)b * (G + 1) + c] <= tau);
        }
        const unsigned m = __ballot_sync(kFull, rej);
        if (m) {
            accepted = c0 + __ffs(m) - 1;
            break;
        }
    }
    if (write && P.check_uniforms) {
        for (int c = lane; c <= G; c += 32) {
            const double u = P.u[(size_t)b * (G + 1) + c];
            if (!(u >= 0.0) || !(u < 1.0)) flag(P, SSV_STATUS_UNIFORM_RANGE);
        }
    }
    if (accepted < G) {
        mode = MODE_REJECT;
        row = accepted;
    } else if (P.PS == G + 1) {
        mode = MODE_BONUS;
        row = G;
    } else {
        mode = MODE_NONE;
        row = -1;
    }
    if (write && lane == 0) {
        P.acc[b] = accepted;
        if (mode == MODE_NONE) {
            P.fin[b] = -1;
            P.rsu[b] = 0;
            P.rden[b] = 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// Per-element values.  Streaming (acc precision) and exact (fp64) forms.
struct RowCtx {
    int mode;         // MODE_REJECT / MODE_BONUS
    bool useA;        // reject: sample the residual (else the degenerate fallback on p)
    double Mp, Sp, Mq, Sq;
    double denom;
};

template <typename T, int ACT>
__device__ __forceinline__ double exact_p(const StepParams& P, const RowCtx& R, double z) {
    if (ACT == ACT_SOFTMAX) return exp(z - R.Mp) / R.Sp;     // dist.cpp:46-50
    if (ACT == ACT_SIGMOID) return sigmoid_scaled_d(z, P.alpha, P.width);
    return z;
}
template <typename T, int ACT>
__device__ __forceinline__ double exact_q(const StepParams& P, const RowCtx& R, double z) {
    if (ACT == ACT_SOFTMAX) return exp(z - R.Mq) / R.Sq;
    if (ACT == ACT_SIGMOID) return sigmoid_scaled_d(z, P.alpha, P.width);
    return z;
}

// Value the inverse CDF scans at element i (fp64): residual max(0, p - q)
// (verify_reference.cpp:51-55) or the p row itself (fallback / bonus).
template <typename T, int ACT>
__device__ __forceinline__ double exact_value(const StepParams& P, const RowCtx& R, const T* pr,
                                              const T* qr, int i) {
    const double p = exact_p<T, ACT>(P, R, load_exact(pr + i));
    if (R.mode == MODE_REJECT && R.useA) {
        const double q = exact_q<T, ACT>(P, R, load_exact(qr + i));
        const double d = p - q;
        return d > 0.0 ? d : 0.0;
    }
    return p;
}

// ---------------------------------------------------------------------------
// K2 epilogue: inverse CDF of batch row b over the granule partials, then an
// exact fp64 scan inside the selected granule (dist.cpp:122-137).
template <typename T, int ACT>
__device__ void locate(const StepParams& P, int b, int mode, int row, const double* st) {
    __shared__ double s_red[kWarps];
    __shared__ int s_ired[kWarps];
    const int NG = P.NG;
    const double2* gp = P.gpart + (size_t)b * NG;
    const T* pr = p_row<T>(P, b, row);
    const T* qr = (mode == MODE_REJECT) ? q_row<T>(P, b, row) : nullptr;
    const double u = P.u[(size_t)b * (P.G + 1) + P.G];  // u_final, verify_reference.cpp:98

    RowCtx R;
    R.mode = mode;
    R.Mp = st[0];
    R.Sp = st[1];
    R.Mq = st[2];
    R.Sq = st[3];
    R.useA = false;
    double gM = 0.0, gS = 1.0;  // softmax bonus: row max / sum from the granule partials

    if (mode == MODE_REJECT) {
        double sa = 0.0, sp = 0.0;
        for (int g = threadIdx.x; g < NG; g += kThreads) {
            const double2 v = __ldcg(&gp[g]);
            sa += v.x;
            sp += v.y;
        }
        sa = block_reduce(sa, s_red, OpSum());
        sp = block_reduce(sp, s_red, OpSum());
        R.useA = sa > kZeroEps;  // verify_reference.cpp:57-62
        R.denom = R.useA ? sa : sp;
        if (threadIdx.x == 0) {
            if (P.rsu) P.rsu[b] = 1;
            if (P.rden) P.rden[b] = R.useA ? sa : 0.0;
        }
    } else {
        if (ACT == ACT_SOFTMAX) {
            double m = -CUDART_INF;
            for (int g = threadIdx.x; g < NG; g += kThreads) m = fmax(m, __ldcg(&gp[g].x));
            gM = block_reduce(m, s_red, OpMax());
            double s = 0.0;
            for (int g = threadIdx.x; g < NG; g += kThreads) {
                const double2 v = __ldcg(&gp[g]);
                if (v.y > 0.0) s += v.y * exp(v.x - gM);
            }
            gS = block_reduce(s, s_red, OpSum());
            R.Mp = gM;
            R.Sp = gS;
        }
        if (threadIdx.x == 0) {
            if (P.rsu) P.rsu[b] = 0;
            if (P.rden) P.rden[b] = 0.0;
        }
    }
    // Granule mass in the units the scan uses.
    auto gmass = [&](int g) -> double {
        const double2 v = __ldcg(&gp[g]);
        if (mode == MODE_REJECT) return R.useA ? v.x : v.y;
        if (ACT == ACT_SOFTMAX) return v.y > 0.0 ? v.y * exp(v.x - gM) / gS : 0.0;
        return v.y;
    };
    if (mode == MODE_BONUS) {
        double s = 0.0;
        for (int g = threadIdx.x; g < NG; g += kThreads) s += gmass(g);
        R.denom = block_reduce(s, s_red, OpSum());  // sample_row's sequential_sum, ~1 for softmax
    }

    // Level 1: first granule whose normalized prefix exceeds u.
    double carry = 0.0;
    int gstar = -1;
    for (int g0 = 0; g0 < NG && gstar < 0; g0 += kThreads) {
        const int g = g0 + threadIdx.x;
        const double w = g < NG ? gmass(g) / R.denom : 0.0;
        double total;
        const double incl = carry + block_scan_incl(w, s_red, total);
        const int hit = (g < NG && u < incl) ? g : 0x7fffffff;
        const int first = block_reduce(hit, s_ired, OpMin());
        if (first != 0x7fffffff) {
            gstar = first;
            // carry before gstar = incl(gstar) - w(gstar); recompute exactly
            if (threadIdx.x == first - g0) s_red[0] = incl - w;
            __syncthreads();
            carry = s_red[0];
            __syncthreads();
        } else {
            carry += total;
        }
    }

    // Level 2: exact element scan, continuing into later granules on rounding.
    constexpr int E2 = kGranule / kThreads;
    int token = -1;
    while (gstar >= 0 && gstar < NG) {
        const int lo = gstar * kGranule;
        const int base = lo + threadIdx.x * E2;
        double vals[E2];
        double tsum = 0.0;
#pragma unroll
        for (int e = 0; e < E2; ++e) {
            const int i = base + e;
            vals[e] = (i < P.V) ? exact_value<T, ACT>(P, R, pr, qr, i) / R.denom : 0.0;
            tsum += vals[e];
        }
        double total;
        const double incl = block_scan_incl(tsum, s_red, total);
        double cum = carry + (incl - tsum);
        int hit = 0x7fffffff;
#pragma unroll
        for (int e = 0; e < E2; ++e) {
            cum += vals[e];
            if (hit == 0x7fffffff && base + e < P.V && u < cum) hit = base + e;
        }
        const int first = block_reduce(hit, s_ired, OpMin());
        if (first != 0x7fffffff) {
            token = first;
            break;
        }
        carry += total;
        ++gstar;
    }
    if (token < 0) {
        // dist.cpp:135-136: last index with positive mass, else 0.
        int glast = -1;
        for (int g = threadIdx.x; g < NG; g += kThreads)
            if (gmass(g) > 0.0) glast = max(glast, g);
        glast = block_reduce(glast, s_ired, OpMax());
        token = 0;
        if (glast >= 0) {
            int last = -1;
            for (int i = glast * kGranule + threadIdx.x; i < min((glast + 1) * kGranule, P.V); i += kThreads)
                if (exact_value<T, ACT>(P, R, pr, qr, i) > 0.0) last = max(last, i);
            last = block_reduce(last, s_ired, OpMax());
            if (last >= 0) token = last;
        }
    }
    if (threadIdx.x == 0) P.fin[b] = token;
}

// ---------------------------------------------------------------------------
// Granule partials of one warp.
template <typename T, int ACT>
__device__ __forceinline__ double2 granule_partial(const StepParams& P, const RowCtx& R,
                                                   const T* pr, const T* qr, int lo, int hi) {
    using A = typename Elem<T>::acc;
    constexpr int VEC = Elem<T>::VEC;
    constexpr int NV = kGranule / (32 * VEC);
    const int lane = threadIdx.x & 31;
    const A alpha = (A)P.alpha, invw = (A)(1.0 / P.width);

    // streaming value of p (acc precision)
    auto vp_of = [&](A x) -> A {
        if (ACT == ACT_SOFTMAX) return exp_rel(x, (A)R.Mp) * (A)(1.0 / R.Sp);
        if (ACT == ACT_SIGMOID) return (A)1 / ((A)1 + exp_neg((x - alpha) * invw));
        return x;
    };

    if (R.mode == MODE_BONUS) {
        WarpTile<T, NV> t;
        t.load(pr, lo, hi);
        if (ACT == ACT_SOFTMAX) {
            A mx = -INFINITY, mn = INFINITY;
            t.minmax(mx, mn);
            mx = warp_max(mx);
            const double s = warp_sum(t.sum_exp(mx));
            return make_double2((double)mx, s);
        }
        const double s = warp_sum(t.sum_map(vp_of));
        return make_double2(0.0, s);
    }

    // Residual pair: a = max(0, p - q) and the fallback mass sum p.
    auto pair = [&](A xp, A xq, A& a, A& vp) {
        if (ACT == ACT_SOFTMAX) {
            vp = exp_rel(xp, (A)R.Mp) * (A)(1.0 / R.Sp);
            const A vq = exp_rel(xq, (A)R.Mq) * (A)(1.0 / R.Sq);
            a = vp - vq > (A)0 ? vp - vq : (A)0;
        } else if (ACT == ACT_SIGMOID) {
            // sigma(tp) - sigma(tq) = sigma(tp) * sigma(-tq) * (1 - e^-(tp-tq)), no cancellation.
            const A tp = (xp - alpha) * invw, tq = (xq - alpha) * invw;
            const A d = (xp - xq) * invw;
            vp = (A)1 / ((A)1 + exp_neg(tp));
            const A sq_neg = (A)1 / ((A)1 + exp_neg(-tq));
            a = d > (A)0 ? vp * sq_neg * (-expm1_acc(-d)) : (A)0;
        } else {
            vp = xp;
            a = xp - xq > (A)0 ? xp - xq : (A)0;
        }
    };

    double sa = 0.0, sp = 0.0;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(qr)) & 15) == 0 &&
                        (P.V % VEC) == 0;
    if (vec_ok) {
        const int nvec = (hi - lo) / VEC;  // lo and V are multiples of VEC
        uint4 vp4[NV], vq4[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int idx = j * 32 + lane;
            if (idx < nvec) {
                vp4[j] = ldg_stream(pr + lo + (size_t)idx * VEC);
                vq4[j] = ldg_stream(qr + lo + (size_t)idx * VEC);
            }
        }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            if (j * 32 + lane < nvec) {
                A xp[VEC], xq[VEC];
                unpack(vp4[j], xp);
                unpack(vq4[j], xq);
                A ta = 0, tp = 0;
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    A a, v;
                    pair(xp[e], xq[e], a, v);
                    ta += a;
                    tp += v;
                }
                sa += (double)ta;
                sp += (double)tp;
            }
        }
    } else {
        constexpr int NS = kGranule / 32;
        A xp[NS], xq[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const int i = lo + j * 32 + lane;
            if (i < hi) {
                xp[j] = load_elem(pr + i);
                xq[j] = load_elem(qr + i);
            }
        }
        A ta = 0, tp = 0;
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            if (lo + j * 32 + lane < hi) {
                A a, v;
                pair(xp[j], xq[j], a, v);
                ta += a;
                tp += v;
            }
            if ((j & 7) == 7) {
                sa += (double)ta;
                sp += (double)tp;
                ta = 0;
                tp = 0;
            }
        }
        sa += (double)ta;
        sp += (double)tp;
    }
    return make_double2(warp_sum(sa), warp_sum(sp));
}

template <typename T, int ACT>
__global__ void __launch_bounds__(kThreads) k_row_pass(StepParams P) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5;
    __shared__ int s_mode, s_row;
    __shared__ double s_st[4];
    __shared__ bool s_last;

    if (P.sample_mode) {
        if (threadIdx.x == 0) {
            s_mode = MODE_BONUS;
            s_row = 0;
        }
    } else if (ACT == ACT_SOFTMAX) {
        if (threadIdx.x == 0) {
            const Decision d = P.dec[b];
            s_mode = d.mode;
            s_row = d.row;
            s_st[0] = d.Mp;
            s_st[1] = d.Sp;
            s_st[2] = d.Mq;
            s_st[3] = d.Sq;
        }
    } else if (warp == 0) {
        int mode, row;
        decide_gather<T, ACT>(P, b, blockIdx.x == 0, mode, row);
        if (threadIdx.x == 0) {
            s_mode = mode;
            s_row = row;
            s_st[0] = s_st[2] = 0.0;
            s_st[1] = s_st[3] = 1.0;
        }
    }
    __syncthreads();
    const int mode = s_mode, row = s_row;
    if (mode == MODE_NONE) return;

    RowCtx R;
    R.mode = mode;
    R.Mp = s_st[0];
    R.Sp = s_st[1];
    R.Mq = s_st[2];
    R.Sq = s_st[3];
    const T* pr = p_row<T>(P, b, row);
    const T* qr = mode == MODE_REJECT ? q_row<T>(P, b, row) : nullptr;

    const int g = blockIdx.x * kWarps + warp;
    if (g < P.NG) {
        const int lo = g * kGranule;
        const int hi = min(lo + kGranule, P.V);
        const double2 part = granule_partial<T, ACT>(P, R, pr, qr, lo, hi);
        if ((threadIdx.x & 31) == 0) P.gpart[(size_t)b * P.NG + g] = part;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&P.cnt2[b], 1u);
        s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) P.cnt2[b] = 0;
    double st[4] = {s_st[0], s_st[1], s_st[2], s_st[3]};
    locate<T, ACT>(P, b, mode, row, st);
}

// ---------------------------------------------------------------------------
// K3: optional materialized grids (activation.cpp:20-49; verify_fused.cpp:50
// residual-in-q semantics; verify_sigmoid.cpp:39-48).
template <typename T, int ACT>
__global__ void __launch_bounds__(kThreads) k_materialize(StepParams P, void* outp, void* outq, void* outr) {
    using A = typename Elem<T>::acc;
    using O = typename std::conditional<sizeof(A) == 8, double, float>::type;
    const size_t V = (size_t)P.V;
    const size_t np = (size_t)P.B * P.PS * V, nq = (size_t)P.B * P.G * V;
    const A alpha = (A)P.alpha, invw = (A)(1.0 / P.width);
    auto act = [&](A x, const double2& st) -> A {
        if (ACT == ACT_SOFTMAX) return exp_rel(x, (A)st.x) * (A)(1.0 / st.y);
        if (ACT == ACT_SIGMOID) return (A)1 / ((A)1 + exp_neg((x - alpha) * invw));
        return x;
    };
    auto stat_of = [&](int b, int r) -> double2 {
        if (ACT != ACT_SOFTMAX) return make_double2(0.0, 1.0);
        return P.rowstat[(size_t)b * P.NR + r];
    };
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const size_t rowi = i / V;
        const int b = (int)(rowi / P.PS), c = (int)(rowi % P.PS);
        const A x = load_elem(reinterpret_cast<const T*>(P.zp) + i);
        const A pv = act(x, stat_of(b, c < P.G ? c : 2 * P.G));
        if (outp) reinterpret_cast<O*>(outp)[i] = (O)pv;
    }
    if (!outq && !outr) return;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += stride) {
        const size_t rowi = i / V, e = i % V;
        const int b = (int)(rowi / P.G), c = (int)(rowi % P.G);
        const A xq = load_elem(reinterpret_cast<const T*>(P.zq) + i);
        const A qv = act(xq, stat_of(b, P.G + c));
        if (outq) reinterpret_cast<O*>(outq)[i] = (O)qv;
        if (outr) {
            const A xp = load_elem(p_row<T>(P, b, c) + e);
            const A pv = act(xp, stat_of(b, c));
            reinterpret_cast<O*>(outr)[i] = (O)(pv - qv > (A)0 ? pv - qv : (A)0);
        }
    }
}

// ---------------------------------------------------------------------------
// Synthetic inputs: bench.cpp:46-74 per batch row (seed + b), using the
// counter RNG of rng.cpp:12-33 (SplitMix64 at index i, Box-Muller in fp64).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t word_at(uint64_t seed, uint64_t index) {
    return mix64(seed + (index + 1) * 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t index) {
    return (double)(word_at(seed, index) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t n) {  // n-th normal = words 2n, 2n+1
    const double u1 = ((double)(word_at(seed, 2 * n) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (double)(word_at(seed, 2 * n + 1) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

template <typename T>
__device__ __forceinline__ T to_store(double v);
template <>
__device__ __forceinline__ float to_store<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ double to_store<double>(double v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_store<__nv_bfloat16>(double v) {
    return __float2bfloat16_rn((float)v);  // double -> fp32 -> bf16, like orc_round_bf16
}

template <typename T>
__global__ void k_gen_logits(uint64_t seed, int B, int G, int V, T* zp, T* zq) {
    const size_t per_b = (size_t)(2 * G + 1) * V;
    const size_t n = (size_t)B * per_b;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int b = (int)(i / per_b);
        const size_t j = i % per_b;
        const uint64_t s = seed + (uint64_t)b;
        const size_t np = (size_t)(G + 1) * V;
        if (j < np) {
            zp[(size_t)b * np + j] = to_store<T>(4.0 * normal_at(s, j));
        } else {
            const size_t jq = j - np;  // q row c element e: z_p[c][e] + N at index np + jq
            const double v = 4.0 * normal_at(s, jq) + 1.0 * normal_at(s, np + jq);
            zq[(size_t)b * G * V + jq] = to_store<T>(v);
        }
    }
}

// Draft draws (index 2(2G+1)V + c) and acceptance/final uniforms
// (index 2(2G+1)V + G + c) of bench.cpp:66-73.
__global__ void k_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int per = 2 * G + 1;
    if (i >= B * per) return;
    const int b = i / per, c = i % per;
    const uint64_t base = 2ull * (uint64_t)(2 * G + 1) * (uint64_t)V;
    const double v = uniform_at(seed + (uint64_t)b, base + (uint64_t)c);
    if (c < G) draft_u[(size_t)b * G + c] = v;
    else u[(size_t)b * (G + 1) + (c - G)] = v;
}

// ---------------------------------------------------------------------------
// Host-side launchers.
template <typename T, int NV>
static void launch_stats_nv(const StepParams& P, const Launch& L) {
    const long tasks = (long)P.B * P.NR * P.K;
    const int h = L.begin(KID_ROW_STATS);
    k_row_stats<T, NV><<<(unsigned)tasks, kThreads, 0, L.st>>>(P);
    L.end(h);
}

template <typename T>
static int stats_nv_for(const StepParams& P, int& CH) {
    constexpr int VEC = Elem<T>::VEC;
    const int nvs[3] = {8, 4, 2};
    for (int i = 0; i < 3; ++i) {
        const int ch = kWarps * 32 * nvs[i] * VEC;
        const long tasks = (long)P.B * P.NR * ((P.V + ch - 1) / ch);
        if (tasks >= 148L * 8 || i == 2) {
            CH = ch;
            return nvs[i];
        }
    }
    return 2;
}

template <typename T>
static void launch_stats_t(StepParams P, const Launch& L) {
    int CH;
    const int nv = stats_nv_for<T>(P, CH);
    P.CH = CH;
    P.K = (P.V + CH - 1) / CH;
    if (nv == 8) launch_stats_nv<T, 8>(P, L);
    else if (nv == 4) launch_stats_nv<T, 4>(P, L);
    else launch_stats_nv<T, 2>(P, L);
}

int stats_chunks(int dtype, const StepParams& P) {
    int CH = 0;
    if (dtype == DT_F32) stats_nv_for<float>(P, CH);
    else if (dtype == DT_BF16) stats_nv_for<__nv_bfloat16>(P, CH);
    else stats_nv_for<double>(P, CH);
    return (P.V + CH - 1) / CH;
}

template <typename T, int ACT>
static void launch_pass_t(const StepParams& P, const Launch& L) {
    dim3 grid((unsigned)((P.NG + kWarps - 1) / kWarps), (unsigned)P.B);
    const int h = L.begin(KID_ROW_PASS);
    k_row_pass<T, ACT><<<grid, kThreads, 0, L.st>>>(P);
    L.end(h);
}

template <typename T, int ACT>
static void launch_mat_t(const StepParams& P, void* p, void* q, void* r, const Launch& L) {
    const int h = L.begin(KID_MATERIALIZE);
    k_materialize<T, ACT><<<148 * 8, kThreads, 0, L.st>>>(P, p, q, r);
    L.end(h);
}

template <typename T>
static void dispatch_verify(int act, StepParams P, void* outp, void* outq, void* outr, const Launch& L) {
    const bool mat = outp || outq || outr;
    if (act == ACT_SOFTMAX) {
        launch_stats_t<T>(P, L);
        launch_pass_t<T, ACT_SOFTMAX>(P, L);
        if (mat) launch_mat_t<T, ACT_SOFTMAX>(P, outp, outq, outr, L);
    } else if (act == ACT_SIGMOID) {
        launch_pass_t<T, ACT_SIGMOID>(P, L);
        if (mat) launch_mat_t<T, ACT_SIGMOID>(P, outp, outq, outr, L);
    } else {
        launch_pass_t<T, ACT_PROBS>(P, L);
        if (mat) launch_mat_t<T, ACT_PROBS>(P, outp, outq, outr, L);
    }
}

void launch_verify(int dtype, int act, const StepParams& P, void* outp, void* outq, void* outr, const Launch& L) {
    StepParams Q = P;
    if (act == ACT_SOFTMAX) Q.K = stats_chunks(dtype, P);
    if (dtype == DT_F32) dispatch_verify<float>(act, Q, outp, outq, outr, L);
    else if (dtype == DT_BF16) dispatch_verify<__nv_bfloat16>(act, Q, outp, outq, outr, L);
    else dispatch_verify<double>(act, Q, outp, outq, outr, L);
}

void launch_sample_softmax(int dtype, const StepParams& P, const Launch& L) {
    if (dtype == DT_F32) launch_pass_t<float, ACT_SOFTMAX>(P, L);
    else if (dtype == DT_BF16) launch_pass_t<__nv_bfloat16, ACT_SOFTMAX>(P, L);
    else launch_pass_t<double, ACT_SOFTMAX>(P, L);
}

void launch_gen_logits(int dtype, uint64_t seed, int B, int G, int V, void* zp, void* zq, const Launch& L) {
    const int blocks = 148 * 16;
    const int h = L.begin(KID_GEN);
    if (dtype == DT_F32) k_gen_logits<float><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (float*)zp, (float*)zq);
    else if (dtype == DT_BF16)
        k_gen_logits<__nv_bfloat16><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (__nv_bfloat16*)zp, (__nv_bfloat16*)zq);
    else k_gen_logits<double><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (double*)zp, (double*)zq);
    L.end(h);
}

void launch_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u, const Launch& L) {
    const int n = B * (2 * G + 1);
    const int h = L.begin(KID_GEN);
    k_gen_uniforms<<<(n + kThreads - 1) / kThreads, kThreads, 0, L.st>>>(seed, B, G, V, draft_u, u);
    L.end(h);
}

}  // namespace ssv
