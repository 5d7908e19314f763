// tma_lat.cu -- design microbenchmark for the small-batch cluster path: how
// long does one SM take to stage R row slices of S bytes from HBM into shared
// memory, by (a) one TMA bulk copy per slice (mbarrier per slice), (b) per-
// thread cp.async 16 B, (c) plain 128-bit loads into registers?  One CTA per SM
// (NB CTAs), globaltimer stamps per CTA; prints the median / max CTA latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_lat tma_lat.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2406_11016_b200/csrc/ssv_pipe.cuh"

using namespace ssv;

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const uint8_t* src, size_t cta_stride, size_t row_stride, int R, int S,
                                              unsigned long long* out, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bar[32];
    const uint8_t* base = src + (size_t)blockIdx.x * cta_stride;
    unsigned long long t0 = gt();
    float acc = 0.f;
    if (MODE == 0) {
        if (threadIdx.x == 0) {
            for (int r = 0; r < R; ++r) mbar_init(&bar[r], 1);
            mbar_fence_init();
            for (int r = 0; r < R; ++r) {
                mbar_arrive_expect_tx(&bar[r], S);
                bulk_g2s(sm + (size_t)r * S, base + (size_t)r * row_stride, S, &bar[r]);
            }
        }
        __syncthreads();
        for (int r = 0; r < R; ++r) mbar_wait(&bar[r], 0);
        const float* f = reinterpret_cast<const float*>(sm);
        for (int i = threadIdx.x; i < R * S / 4; i += blockDim.x) acc += f[i];
    } else if (MODE == 1) {
        for (int r = 0; r < R; ++r)
            for (int i = threadIdx.x; i < S / 16; i += blockDim.x) {
                const uint32_t d = smem_u32(sm + (size_t)r * S + i * 16);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(base + (size_t)r * row_stride + i * 16)
                             : "memory");
            }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        const float* f = reinterpret_cast<const float*>(sm);
        for (int i = threadIdx.x; i < R * S / 4; i += blockDim.x) acc += f[i];
    } else {
        for (int r = 0; r < R; ++r) {
            const uint4* p = reinterpret_cast<const uint4*>(base + (size_t)r * row_stride);
            uint4 v[4];
            for (int i = threadIdx.x; i < S / 16; i += 4 * blockDim.x) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i + u * blockDim.x < S / 16) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i + u * blockDim.x < S / 16) acc += __uint_as_float(v[u].x);
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = gt();
    if (threadIdx.x == 0) {
        out[2 * blockIdx.x] = t0;
        out[2 * blockIdx.x + 1] = t1;
    }
    if (acc == 1.2345f) sink[0] = acc;
}

int main() {
    const size_t bytes = 4ull << 30;
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    unsigned long long* out;
    cudaMalloc(&out, 2 * 1024 * sizeof(unsigned long long));
    float* sink;
    cudaMalloc(&sink, 4);
    uint8_t* flush;
    cudaMalloc(&flush, 512 << 20);
    for (auto fn : {k<0>, k<1>, k<2>}) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg {
        int nb, R, S;
    } cfgs[] = {{128, 10, 14336}, {128, 10, 8192}, {128, 1, 8192}, {16, 10, 8192}, {128, 16, 8192}, {148, 4, 32768}};
    const char* names[] = {"tma-bulk", "cp.async", "ldg-reg"};
    for (auto c : cfgs) {
        for (int mode = 0; mode < 3; ++mode) {
            std::vector<double> lat;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(flush, rep, 512 << 20);  // evict L2
                const size_t row_stride = 207472, cta_stride = (size_t)c.R * row_stride + 4096;
                const size_t smem = mode == 2 ? 0 : (size_t)c.R * c.S;
                if (mode == 0) k<0><<<c.nb, 256, smem>>>(src, cta_stride, row_stride, c.R, c.S, out, sink);
                if (mode == 1) k<1><<<c.nb, 256, smem>>>(src, cta_stride, row_stride, c.R, c.S, out, sink);
                if (mode == 2) k<2><<<c.nb, 256, smem>>>(src, cta_stride, row_stride, c.R, c.S, out, sink);
                cudaDeviceSynchronize();
                std::vector<unsigned long long> h(2 * c.nb);
                cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
                unsigned long long mn = ~0ull, mx = 0;
                for (int i = 0; i < c.nb; ++i) {
                    mn = std::min(mn, h[2 * i]);
                    mx = std::max(mx, h[2 * i + 1]);
                }
                if (rep) lat.push_back((mx - mn) / 1e3);
            }
            std::sort(lat.begin(), lat.end());
            printf("%-9s CTAs=%3d rows=%2d slice=%6d B (%4d KB/CTA): span %6.2f us (min %6.2f)\n", names[mode], c.nb, c.R,
                   c.S, c.R * c.S / 1024, lat[lat.size() / 2], lat[0]);
        }
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
