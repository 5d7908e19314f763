// ssv_device.cuh -- device building blocks for the sm_100a verification kernels.
//
// Element traits (fp32 / bf16 / fp64 logits), 128-bit streaming loads with
// misaligned-row peeling, the fp32-in-register / fp64-carry arithmetic the
// parity contract needs ("Bit-exact tokens need fp64
// carries"), and warp / block reductions and scans with a FIXED topology, so
// every result is bit-identical run to run (the reference's guarantee across
// worker counts, verify_fused.hpp:23).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace ssv {

constexpr double kZeroEps = 1e-12;  // dist.hpp:9
constexpr int kThreads = 256;       // 8 warps per CTA for every kernel
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

// ---- element traits --------------------------------------------------------
// Every element is widened to `acc` (fp32 for fp32/bf16 storage, fp64 for
// fp64 storage) before any arithmetic; one 16-byte vector holds VEC elements.
template <typename T>
struct Elem;
template <>
struct Elem<float> {
    using acc = float;
    static constexpr int VEC = 4;
};
template <>
struct Elem<__nv_bfloat16> {
    using acc = float;
    static constexpr int VEC = 8;
};
template <>
struct Elem<double> {
    using acc = double;
    static constexpr int VEC = 2;
};

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void unpack(const uint4& v, float (&x)[4]) {
    x[0] = __uint_as_float(v.x);
    x[1] = __uint_as_float(v.y);
    x[2] = __uint_as_float(v.z);
    x[3] = __uint_as_float(v.w);
}
__device__ __forceinline__ void unpack(const uint4& v, float (&x)[8]) {
    // bf16 -> fp32 is exact: the bf16 bits are the high half of the fp32 word.
    x[0] = __uint_as_float(v.x << 16);
    x[1] = __uint_as_float(v.x & 0xffff0000u);
    x[2] = __uint_as_float(v.y << 16);
    x[3] = __uint_as_float(v.y & 0xffff0000u);
    x[4] = __uint_as_float(v.z << 16);
    x[5] = __uint_as_float(v.z & 0xffff0000u);
    x[6] = __uint_as_float(v.w << 16);
    x[7] = __uint_as_float(v.w & 0xffff0000u);
}
__device__ __forceinline__ void unpack(const uint4& v, double (&x)[2]) {
    x[0] = __hiloint2double((int)v.y, (int)v.x);
    x[1] = __hiloint2double((int)v.w, (int)v.z);
}

__device__ __forceinline__ float load_elem(const float* p) { return __ldg(p); }
__device__ __forceinline__ float load_elem(const __nv_bfloat16* p) {
    return __uint_as_float(((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p))) << 16);
}
__device__ __forceinline__ double load_elem(const double* p) { return __ldg(p); }

__device__ __forceinline__ float load_smem_elem(const float* p) { return *p; }
__device__ __forceinline__ float load_smem_elem(const __nv_bfloat16* p) {
    return __uint_as_float(((uint32_t)*reinterpret_cast<const unsigned short*>(p)) << 16);
}
__device__ __forceinline__ double load_smem_elem(const double* p) { return *p; }

// Exact (fp64) value of a stored element.
template <typename T>
__device__ __forceinline__ double load_exact(const T* p) {
    return (double)load_elem(p);
}

// ---- exponentials ---------------------------------------------------------
// e^(x - m) for x <= m.  fp32 path: one subtraction, one multiply, one MUFU
// ex2 -- the per-element hot op.  The relative error is ~1e-7 for the terms
// that carry the row mass and is absorbed by the fp64 carries (DESIGN.md,
// "Numerics").  fp64 path: libdevice exp.
__device__ __forceinline__ float exp_rel(float x, float m) {
    const float t = (x - m) * 1.4426950408889634f;
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
    return r;
}
__device__ __forceinline__ double exp_rel(double x, double m) { return exp(x - m); }

// e^(x - m) to ~3e-7 relative for the materialized p / q / residual grids
// (north star: 1e-5 relative, and residual elements where p ~ q cancel need
// both terms far more accurate than exp_rel's ~2e-6 at |x - m| ~ 40): the
// difference as an exact float pair (TwoSum), times log2(e) as hi + lo, then
// 2^n * 2^f with |f| <= 0.5 from MUFU ex2.
__device__ __forceinline__ float exp_rel_acc(float x, float m) {
    const float s = x - m;
    const float bv = s - x;
    const float e = (x - (s - bv)) + (-m - bv);
    constexpr float L = 1.44269502162933349609375f;  // log2(e), fp32 head
    constexpr float Ll = 1.925962991126617468e-8f;   // log2(e) - L
    const float yh = s * L;
    const float yl = fmaf(s, L, -yh) + fmaf(s, Ll, e * L);
    const float n = rintf(yh);
    float r;
    asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"((yh - n) + yl));
    return scalbnf(r, (int)n);
}
__device__ __forceinline__ double exp_rel_acc(double x, double m) { return exp(x - m); }

// dist.cpp:17-23 stable_sigmoid, fp64 (exact path).
__device__ __forceinline__ double stable_sigmoid_d(double t) {
    if (t >= 0.0) return 1.0 / (1.0 + exp(-t));
    const double e = exp(t);
    return e / (1.0 + e);
}
// dist.cpp:60-62 sigmoid_scaled_value: t = (z - alpha) / (beta - alpha).
__device__ __forceinline__ double sigmoid_scaled_d(double z, double alpha, double width) {
    return stable_sigmoid_d((z - alpha) / width);
}

// dist.cpp:64-69 sigmoid_scaled_value_half with half.cpp's round_to_half
// (double -> float -> binary16 RNE -> back): z, alpha, 1/width, the shifted
// value, the scaled argument and sigma each rounded to half.
__device__ __forceinline__ double round_half_d(double x) { return (double)__half2float(__float2half_rn((float)x)); }
__device__ __forceinline__ double sigmoid_half_d(double z, double alpha, double width) {
    const double inv_w = round_half_d(1.0 / width);
    const double shifted = round_half_d(round_half_d(z) - round_half_d(alpha));
    const double arg = round_half_d(shifted * inv_w);
    return round_half_d(stable_sigmoid_d(arg));
}

// Streaming-path sigmoid pieces (fp32 or fp64 `acc`).  The sigmoid variant
// touches only the rows a batch row still needs, so it affords the accurate
// (<= 2 ulp, unbiased) expf: its masses are sums of ~V values near 0.5-1 whose
// rounding must not accumulate a bias (residual_denom parity).
__device__ __forceinline__ float exp_neg(float t) { return expf(-t); }
__device__ __forceinline__ double exp_neg(double t) { return exp(-t); }

__device__ __forceinline__ float ex2f(float t) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
    return r;
}

// Streaming sigmoid 1 / (1 + e^-t): MUFU ex2 + MUFU rcp (~2 ulp each), the
// per-element op of the sigmoid variant's granule sums.  Its relative error
// (< 5e-7, no systematic sign) stays well inside the 1e-6 relative tolerance of
// the denominators and moves CDF boundaries by < 1e-6 (explained mismatches).
__device__ __forceinline__ float sigmoid_fast(float t) {
    const float e = ex2f(-t * 1.4426950408889634f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    return r;
}
__device__ __forceinline__ double sigmoid_fast(double t) { return 1.0 / (1.0 + exp(-t)); }
// e^x - 1 for the sigmoid residual's 1 - e^-(tp - tq) factor, to ~3e-7
// relative without libm's branches: a degree-7 Taylor polynomial below
// |x| = 0.5 (truncation <= x^7 / 40320 relative), MUFU ex2 above (the result
// is then >= 0.39 in magnitude, so the ex2's 2 ulp do not cancel).
__device__ __forceinline__ float expm1_acc(float x) {
    if (fabsf(x) < 0.5f) {
        float p = 1.0f / 5040.0f;
        p = fmaf(p, x, 1.0f / 720.0f);
        p = fmaf(p, x, 1.0f / 120.0f);
        p = fmaf(p, x, 1.0f / 24.0f);
        p = fmaf(p, x, 1.0f / 6.0f);
        p = fmaf(p, x, 0.5f);
        p = fmaf(p, x, 1.0f);
        return p * x;
    }
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * 1.4426950408889634f));
    return r - 1.0f;
}
__device__ __forceinline__ double expm1_acc(double x) { return expm1(x); }

// ---- sm_100a three-input min/max (FMNMX3) and packed fp32x2 arithmetic ------
// (FADD2 / FMUL2): the per-element hot ops of the row-statistics pass.
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// NaN-propagating minimum: the running minimum of a statistics pass doubles as
// its non-finite detector (require_finite, dist.cpp:27-36) -- a NaN anywhere in
// the inputs makes it NaN even where max / sum drop NaN operands.
__device__ __forceinline__ float fmin3f_nan(float a, float b, float c) {
    float r;
    asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ double fmin_nan(double a, double b) { return (a != a || b != b) ? a + b : fmin(a, b); }

// ---- warp / block reductions (fixed topology) ------------------------------
template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
template <typename V>
__device__ __forceinline__ V warp_max(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    return v;
}
template <typename V>
__device__ __forceinline__ V warp_min(V v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// Block reductions over NW warps (default: kThreads threads); `sm` needs NW
// slots.  All threads receive the result.  Ends with the scratch free for reuse.
template <int NW, typename V, typename Op>
__device__ __forceinline__ V block_reduce_n(V v, V* sm, Op op) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
    __syncthreads();
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    V r = sm[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) r = op(r, sm[w]);
    return r;
}
template <typename V, typename Op>
__device__ __forceinline__ V block_reduce(V v, V* sm, Op op) {
    return block_reduce_n<kWarps>(v, sm, op);
}
struct OpSum {
    template <typename V>
    __device__ V operator()(V a, V b) const { return a + b; }
};
struct OpMax {
    template <typename V>
    __device__ V operator()(V a, V b) const { return a > b ? a : b; }
};
struct OpMin {
    template <typename V>
    __device__ V operator()(V a, V b) const { return a < b ? a : b; }
};

// Inclusive warp scan (Hillis-Steele, fixed order).
__device__ __forceinline__ double warp_scan_incl(double v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Block inclusive scan over NW warps; returns the inclusive prefix and writes
// the block total.  `sm` needs NW slots.
template <int NW>
__device__ __forceinline__ double block_scan_incl_n(double v, double* sm, double& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double incl = warp_scan_incl(v);
    __syncthreads();
    if (lane == 31) sm[warp] = incl;
    __syncthreads();
    double off = 0.0;
    for (int w = 0; w < warp; ++w) off += sm[w];
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += sm[w];
    total = tot;
    return off + incl;
}
__device__ __forceinline__ double block_scan_incl(double v, double* sm, double& total) {
    return block_scan_incl_n<kWarps>(v, sm, total);
}

// ---- misaligned-row peeling ---------------------------------------------------
// A range [lo, hi) of elements starting at `base` is split into a scalar head
// (to the first 16-byte boundary), an aligned run of 16-byte vectors, and a
// scalar tail.  Rows of odd length (V = 51865) start at arbitrary offsets.
template <typename T>
struct Span16 {
    int head_end;  // [lo, head_end) scalar
    int vec_begin; // == head_end
    int nvec;      // vectors in [vec_begin, vec_begin + nvec*VEC)
    int tail_begin;// [tail_begin, hi) scalar
};

template <typename T>
__device__ __forceinline__ Span16<T> split16(const T* base, int lo, int hi) {
    constexpr int VEC = Elem<T>::VEC;
    Span16<T> s;
    if (hi <= lo) {
        s.head_end = s.vec_begin = s.tail_begin = lo;
        s.nvec = 0;
        return s;
    }
    const uintptr_t a = reinterpret_cast<uintptr_t>(base + lo);
    int head = (int)(((16 - (a & 15)) & 15) / sizeof(T));
    if (head > hi - lo) head = hi - lo;
    s.head_end = lo + head;
    s.vec_begin = s.head_end;
    s.nvec = (hi - s.vec_begin) / VEC;
    s.tail_begin = s.vec_begin + s.nvec * VEC;
    return s;
}

}  // namespace ssv
