// fp64_bench.cu -- design microbenchmark: DADD/DFMA latency and throughput and
// the cost of exp(double) on this B200 (decides how much fp64 the decision /
// locate chains can afford).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_bench fp64_bench.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_lat(double* out, int n, double a) {  // one dependent chain per thread
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / n;
    if (x == 12345.0) out[1] = x;
}
__global__ void k_tput(double* out, int n, double a) {  // 8 independent chains per thread
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, 1e-9);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.0) out[1] = s;
}
__global__ void k_exp(double* out, int n) {
    double s = 0, x = threadIdx.x * -1e-3;
    for (int i = 0; i < n; ++i) { s += exp(x); x -= 1e-4; }
    if (s == 12345.0) out[1] = s;
}
__global__ void k_f32tput(float* out, int n, float a) {
    float x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, 1e-9f);
    float s = 0;
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.0f) out[1] = s;
}
int main() {
    double* d; cudaMalloc(&d, 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k_lat<<<1, 32>>>(d, 100000, 0.999); cudaDeviceSynchronize();
    double lat; cudaMemcpy(&lat, d, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", lat);
    const int n = 20000;
    float ms;
    k_tput<<<sms * 4, 256>>>(d, n, 0.999); cudaDeviceSynchronize();
    cudaEventRecord(a); k_tput<<<sms * 4, 256>>>(d, n, 0.999); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DFMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * n * sms * 4 * 256 / (ms * 1e-3) / 1e12);
    k_f32tput<<<sms * 4, 256>>>((float*)d, n, 0.999f); cudaDeviceSynchronize();
    cudaEventRecord(a); k_f32tput<<<sms * 4, 256>>>((float*)d, n, 0.999f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("FFMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * n * sms * 4 * 256 / (ms * 1e-3) / 1e12);
    cudaEventRecord(a); k_exp<<<sms * 4, 256>>>(d, 2000); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("exp(double): %.2f Gexp/s (%.0f per SM per us)\n", 2000.0 * sms * 4 * 256 / (ms * 1e-3) / 1e9, 2000.0 * 4 * 256 / (ms * 1e3));
    return 0;
}
