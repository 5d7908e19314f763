// PCIe host->device probe for the host entry points (design check):
//   (a) cudaMemcpyAsync of 18.26 MB (the C2 step's logits) split over 1..4 streams;
//   (b) a kernel reading the pinned buffer directly (zero-copy over PCIe) and
//       writing it to HBM, at several grid sizes / vector widths.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pcie_bw tools/pcie_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void zc_copy(const uint4* __restrict__ h, uint4* __restrict__ d, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x * 4;
    for (size_t i = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; i < n; i += stride) {
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j * blockDim.x < n) v[j] = h[i + j * blockDim.x];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j * blockDim.x < n) d[i + j * blockDim.x] = v[j];
    }
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? (size_t)atoll(argv[1]) : 18257024;  // bytes (default: the C2 step's logits)
    void* h;
    void* dptr;
    CK(cudaMallocHost(&h, n));
    CK(cudaMalloc(&dptr, n));
    memset(h, 1, n);
    std::vector<cudaStream_t> st(4);
    for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int split = 1; split <= 4; ++split) {
        float best = 1e30f, sum = 0;
        const int iters = n > 500000000 ? 5 : 30;
        for (int it = 0; it < iters + 3; ++it) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0, st[0]));
            for (int i = 1; i < split; ++i) CK(cudaStreamWaitEvent(st[i], e0, 0));
            const size_t k = (n / split + 255) & ~size_t(255);
            for (int i = 0; i < split; ++i) {
                const size_t a = i * k, b = i + 1 < split ? (i + 1) * k : n;
                CK(cudaMemcpyAsync((char*)dptr + a, (char*)h + a, b - a, cudaMemcpyHostToDevice, st[i]));
            }
            cudaEvent_t j[4];
            for (int i = 1; i < split; ++i) {
                CK(cudaEventCreateWithFlags(&j[i], cudaEventDisableTiming));
                CK(cudaEventRecord(j[i], st[i]));
                CK(cudaStreamWaitEvent(st[0], j[i], 0));
            }
            CK(cudaEventRecord(e1, st[0]));
            CK(cudaEventSynchronize(e1));
            for (int i = 1; i < split; ++i) cudaEventDestroy(j[i]);
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (it >= 3) { sum += ms; if (ms < best) best = ms; }
        }
        printf("memcpy %d stream(s): mean %.1f us  best %.1f us  = %.1f GB/s (mean)\n", split, sum / iters * 1e3,
               best * 1e3, n / (sum / iters * 1e-3) / 1e9);
    }
    if (n > 500000000) return 0;  // large transfers: the copy-engine split only
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int grid : {sms, 2 * sms, 4 * sms, 8 * sms}) {
        for (int threads : {256, 512}) {
            float sum = 0;
            const int iters = 30;
            for (int it = 0; it < iters + 3; ++it) {
                CK(cudaEventRecord(e0, st[0]));
                zc_copy<<<grid, threads, 0, st[0]>>>((const uint4*)h, (uint4*)dptr, n / 16);
                CK(cudaEventRecord(e1, st[0]));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (it >= 3) sum += ms;
            }
            printf("zero-copy kernel grid %4d x %3d: mean %.1f us = %.1f GB/s\n", grid, threads, sum / iters * 1e3,
                   n / (sum / iters * 1e-3) / 1e9);
        }
    }
    return 0;
}
