// lat_bench.cu -- single-warp dependent-chain latencies (cycles) of the ops
// on the verify kernels' latency-bound paths (decision, locate): fp64 add /
// fma / div / exp, fp32 ex2, double shuffles, shared loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_bench lat_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int OP>
__global__ void k(double* out, long long* cyc, double seed) {
    __shared__ double sm[64];
    sm[threadIdx.x] = seed + threadIdx.x;
    __syncthreads();
    double x = seed + threadIdx.x * 1e-3;
    float f = (float)x;
    const int N = 256;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        if (OP == 0) x = x + 1e-9;
        if (OP == 1) x = fma(x, 1.0000001, 1e-9);
        if (OP == 2) x = 1.0 / (x + 1.0);
        if (OP == 3) x = exp(-x) + 0.5;
        if (OP == 4) x += __shfl_xor_sync(0xffffffffu, x, 1);
        if (OP == 5) x = sm[((int)x) & 31] + 1e-9;
        if (OP == 6) {
            float r;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
            f = r * 0.5f;
        }
        if (OP == 7) f = f * 1.0000001f + 1e-9f;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[OP] = (t1 - t0) / N;
    out[threadIdx.x] = x + f;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMallocManaged(&cyc, 16 * 8);
    k<0><<<1, 32>>>(out, cyc, 1.0);
    k<1><<<1, 32>>>(out, cyc, 1.0);
    k<2><<<1, 32>>>(out, cyc, 1.0);
    k<3><<<1, 32>>>(out, cyc, 1.0);
    k<4><<<1, 32>>>(out, cyc, 1.0);
    k<5><<<1, 32>>>(out, cyc, 1.0);
    k<6><<<1, 32>>>(out, cyc, 1.0);
    k<7><<<1, 32>>>(out, cyc, 1.0);
    cudaDeviceSynchronize();
    const char* names[] = {"DADD", "DFMA", "fp64 1/x", "fp64 exp", "SHFL f64+DADD", "LDS f64", "MUFU.EX2", "FFMA"};
    for (int i = 0; i < 8; ++i) printf("%-16s %lld cycles\n", names[i], cyc[i]);
}
