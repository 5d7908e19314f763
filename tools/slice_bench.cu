// Micro-benchmark of the cluster kernel's per-warp slice statistics loop
// (design check): 8 warps per SM, each reducing a 2048-float slice held in
// shared memory (max + sum of e^(x - max)), with parts of the work removed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2406_11016_b200/csrc -o tools/slice_bench tools/slice_bench.cu
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdio>

#include "ssv_device.cuh"

using namespace ssv;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_slice(const float* in, float* out, long long* cyc, int reps) {
    extern __shared__ uint4 sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NV = 512;  // vectors per warp slice (2048 floats)
    for (int i = tid; i < 8 * NV; i += 256) sm[i] = reinterpret_cast<const uint4*>(in)[i];
    __syncthreads();
    const uint4* rv = sm + warp * NV;
    float acc = 0.f;
    const long long c0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        float m = -FLT_MAX;
        double sd = 0.0;
        float fs = 0.f;
        for (int v0 = lane; v0 < NV; v0 += 128) {
            uint4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] = rv[v0 + 32 * u];
            float cm = -FLT_MAX;
            if (MODE != 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    cm = fmax3f(cm, __uint_as_float(w[u].x), __uint_as_float(w[u].y));
                    cm = fmax3f(cm, __uint_as_float(w[u].z), __uint_as_float(w[u].w));
                }
                if (cm > m) {
                    if (MODE == 0 && sd != 0.0) sd *= exp((double)m - (double)cm);
                    if (MODE != 0) fs *= ex2f((m - cm) * 1.44f);
                    m = cm;
                }
            }
            if (MODE == 3) continue;
            const float2 negM = make_float2(-m, -m), l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
            float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float2 t0 = __fmul2_rn(__fadd2_rn(make_float2(__uint_as_float(w[u].x), __uint_as_float(w[u].y)), negM), l2e);
                float2 t1 = __fmul2_rn(__fadd2_rn(make_float2(__uint_as_float(w[u].z), __uint_as_float(w[u].w)), negM), l2e);
                float2& s = (u & 1) ? s1 : s0;
                if (MODE == 1 || MODE == 4) {
                    s = __fadd2_rn(s, t0);
                    s = __fadd2_rn(s, t1);
                } else {
                    s = __fadd2_rn(s, make_float2(ex2f(t0.x), ex2f(t0.y)));
                    s = __fadd2_rn(s, make_float2(ex2f(t1.x), ex2f(t1.y)));
                }
            }
            const float2 t = __fadd2_rn(s0, s1);
            if (MODE == 0) sd += (double)t.x + (double)t.y;
            else fs += t.x + t.y;
        }
        acc += (float)sd + fs + m;
    }
    const long long c1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 8 + warp] = (c1 - c0) / reps;
    out[blockIdx.x * 256 + tid] = acc;
}

// fp64 / conversion throughput: 8 warps per SM, 8 independent chains per lane
template <int OP>
__global__ void __launch_bounds__(256, 1) k_op(float* out, long long* cyc, float seed) {
    double d[8];
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        d[i] = seed + i + threadIdx.x;
        f[i] = seed * i + threadIdx.x;
    }
    const long long c0 = clock64();
    for (int k = 0; k < 256; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) d[i] = d[i] + 1.000001;                 // DADD
            if (OP == 1) d[i] = fma(d[i], 0.999999, 1e-3);       // DFMA
            if (OP == 2) d[i] += (double)f[i], f[i] += 1.0f;     // F2F.F64.F32 + DADD (+FADD)
            if (OP == 3) d[i] = exp(d[i] * 1e-9);                // fp64 exp
            if (OP == 4) f[i] = ex2f(f[i] * 0.999f);             // MUFU.EX2
        }
    }
    const long long c1 = clock64();
    double acc = 0;
    for (int i = 0; i < 8; ++i) acc += d[i] + f[i];
    out[blockIdx.x * 256 + threadIdx.x] = (float)acc;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 8 + (threadIdx.x >> 5)] = (c1 - c0);
}

template <int OP>
static void run_op(const char* name, float* out, long long* cyc, int sms) {
    k_op<OP><<<sms, 256>>>(out, cyc, 1.5f);
    k_op<OP><<<sms, 256>>>(out, cyc, 1.5f);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    // 2048 ops per lane; 8 warps -> per SM ops = 8 * 32 * 2048
    printf("%-28s %lld cycles for 2048 ops/lane, 8 warps/SM: %.2f lane-ops/clk/SM\n", name, h[0],
           8.0 * 32 * 2048 / h[0]);
}

template <int MODE>
static void run(const char* name, const float* in, float* out, long long* cyc, int sms) {
    cudaFuncSetAttribute(k_slice<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 512 * 16);
    k_slice<MODE><<<sms, 256, 8 * 512 * 16>>>(in, out, cyc, 50);
    k_slice<MODE><<<sms, 256, 8 * 512 * 16>>>(in, out, cyc, 50);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s warp0 %lld cycles per 2048-element slice (%.1f per element per lane)\n", name, h[0], h[0] / 64.0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *out;
    long long* cyc;
    cudaMalloc(&in, 8 * 2048 * 4);
    cudaMalloc(&out, sms * 256 * 4);
    cudaMalloc(&cyc, sms * 8 * 8);
    float h[8 * 2048];
    for (int i = 0; i < 8 * 2048; ++i) h[i] = (float)((i * 7919) % 1000) * 0.01f - 5.f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0>("full (minmax, ex2, fp64 sum)", in, out, cyc, sms);
    run<2>("fp32 running sum", in, out, cyc, sms);
    run<1>("no ex2 (fp32 sum)", in, out, cyc, sms);
    run<3>("minmax only", in, out, cyc, sms);
    run<4>("loads + adds only", in, out, cyc, sms);
    run_op<0>("DADD", out, cyc, sms);
    run_op<1>("DFMA", out, cyc, sms);
    run_op<2>("F2F.F64.F32 + DADD", out, cyc, sms);
    run_op<3>("exp() fp64", out, cyc, sms);
    run_op<4>("MUFU.EX2 (+FMUL)", out, cyc, sms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
