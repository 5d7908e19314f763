// stream_bench.cu -- design microbenchmark: how fast can an SM stream HBM into
// the consumer warps?  (a) TMA bulk-copy ring (producer warp + consumer warps,
// mbarriers), stage size / depth / CTAs-per-SM swept, consumers only touch the
// stage; (b) the same ring with an fp32 max + exp-sum consumer; (c) plain
// 128-bit LDG streaming with a grid-stride loop.  Prints GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_bench stream_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2406_11016_b200/csrc/ssv_pipe.cuh"

using namespace ssv;

__device__ __forceinline__ void red_rel(unsigned* p) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned* p) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// WORK: 0 touch, 1 max+exp-sum (per-warp arrive), 2 = 1 + last-warp fold (smem
// counter, fp64 exp) + global store + red.release, last warp frees the stage,
// 3 = 2 with a relaxed red, 4 = 2 but every warp frees the stage (count 8),
// 5 = 2 without the global store / red.
template <int STAGES, int SBYTES, int CONS_WARPS, int WORK, int RUN = 1>
__global__ void __launch_bounds__((CONS_WARPS + 2) * 32) k_ring(const float* __restrict__ src, size_t nchunks,
                                                                 unsigned* next, float* sink) {
    __shared__ double2 wpart[STAGES][CONS_WARPS];
    __shared__ unsigned icnt[STAGES];
    constexpr int Q = 64;
    __shared__ double qv[Q];
    __shared__ unsigned qkey[Q];
    __shared__ volatile unsigned qready[Q];
    __shared__ unsigned qtail;
    __shared__ volatile unsigned qhead, qdone;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * SBYTES);
    uint64_t* empty = full + STAGES;
    unsigned* slot = reinterpret_cast<unsigned*>(empty + STAGES);
    struct Big { int a[14]; double d[4]; };
    __shared__ Big big[STAGES];
    constexpr int NC = CONS_WARPS * 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (WORK >= 2 && WORK != 4) ? 1 : CONS_WARPS);
            icnt[s] = 0;
        }
        for (int q = 0; q < Q; ++q) qready[q] = 0xffffffffu;
        qtail = 0;
        qhead = 0;
        qdone = 0;
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= NC + 32) {  // publisher warp (WORK 6)
        if (WORK == 6) {
            const int lane = threadIdx.x & 31;
            unsigned head = 0;
            for (;;) {
                const unsigned tail = *(volatile unsigned*)&qtail;
                if (head == tail) {
                    if (qdone) {
                        if (head == *(volatile unsigned*)&qtail) break;
                        continue;
                    }
                    __nanosleep(64);
                    continue;
                }
                const unsigned n = min(tail - head, 32u);
                unsigned key = 0;
                if (lane < n) {
                    const unsigned e = (head + lane) % Q;
                    while (qready[e] != head + lane) {}
                    __threadfence_block();
                    key = qkey[e];
                    reinterpret_cast<double*>(sink)[1 + (key & 1023)] = qv[e];
                    __threadfence();
                }
                __syncwarp();
                if (lane < n) red_rlx(next + 64 + (key & 255));
                head += n;
                if (lane == 0) qhead = head;
                __syncwarp();
            }
        }
    } else if (threadIdx.x >= NC) {
        if (threadIdx.x == NC) {
            unsigned n = 0;
            unsigned base = 0, left = 0;
            for (;;) {
                if (left == 0) {
                    base = atomicAdd(next, 1u) * RUN;
                    left = RUN;
                }
                const unsigned i = base++;
                --left;
                const unsigned s = n % STAGES, ph = (n / STAGES) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                slot[s] = i;
                if (WORK == 7) {
                    Big bg;
                    for (int q = 0; q < 14; ++q) bg.a[q] = i + q;
                    for (int q = 0; q < 4; ++q) bg.d[q] = i * 0.5 + q;
                    big[s] = bg;
                }
                if (i >= nchunks) {
                    mbar_arrive(&full[s]);
                    break;
                }
                mbar_arrive_expect_tx(&full[s], SBYTES);
                bulk_g2s(smem + (size_t)s * SBYTES, reinterpret_cast<const char*>(src) + (size_t)i * SBYTES, SBYTES,
                         &full[s]);
                ++n;
            }
        }
    } else {
        unsigned n = 0;
        float acc = 0.f;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (;;) {
            const unsigned s = n % STAGES, ph = (n / STAGES) & 1u;
            mbar_wait(&full[s], ph);
            const unsigned i = slot[s];
            ++n;
            if (i >= nchunks) break;
            if (WORK == 7) {
                const Big bg = big[s];
                int z = 0;
                for (int q = 0; q < 14; ++q) z += bg.a[q];
                acc += z * 1e-30f + (float)(bg.d[0] + bg.d[1] + bg.d[2] + bg.d[3]) * 1e-30f;
            }
            const float4* st = reinterpret_cast<const float4*>(smem + (size_t)s * SBYTES);
            constexpr int WPW = SBYTES / 16 / CONS_WARPS;
            if (WORK == 0) {
                acc += st[warp * WPW + lane].x;
            } else {
                float mx = -INFINITY;
                float4 v[WPW / 32];
#pragma unroll
                for (int m = 0; m < WPW / 32; ++m) {
                    v[m] = st[warp * WPW + lane + 32 * m];
                    mx = fmaxf(mx, fmaxf(fmaxf(v[m].x, v[m].y), fmaxf(v[m].z, v[m].w)));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                float t = 0.f;
#pragma unroll
                for (int m = 0; m < WPW / 32; ++m)
                    t += exp2f((v[m].x - mx) * 1.4427f) + exp2f((v[m].y - mx) * 1.4427f) +
                         exp2f((v[m].z - mx) * 1.4427f) + exp2f((v[m].w - mx) * 1.4427f);
                acc += t;
                if (WORK >= 2) {
                    double sum = t;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    unsigned old = 0;
                    if (lane == 0) {
                        wpart[s][warp] = make_double2((double)mx, sum);
                        __threadfence_block();
                        old = atomicAdd(&icnt[s], 1u);
                        __threadfence_block();
                    }
                    old = __shfl_sync(0xffffffffu, old, 0);
                    if (old == CONS_WARPS - 1) {
                        const double2 wp = lane < CONS_WARPS ? wpart[s][lane] : make_double2(-1e300, 0.0);
                        double M = wp.x;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
                        double S = wp.y * exp(wp.x - M);
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
                        if (lane == 0 && WORK == 6) {
                            icnt[s] = 0;
                            mbar_arrive(&empty[s]);
                            const unsigned slotq = atomicAdd(&qtail, 1u);
                            while (slotq - qhead >= (unsigned)Q) {}
                            qv[slotq % Q] = S;
                            qkey[slotq % Q] = i;
                            __threadfence_block();
                            qready[slotq % Q] = slotq;
                        } else if (lane == 0) {
                            icnt[s] = 0;
                            if (WORK != 4) mbar_arrive(&empty[s]);
                            if (WORK != 5 && WORK != 7) {
                                reinterpret_cast<double*>(sink)[1 + (i & 1023)] = S;
                                if (WORK == 3) red_rlx(next + 64 + (i & 255));
                                else red_rel(next + 64 + (i & 255));
                            }
                        }
                    }
                    if (WORK == 4) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                    }
                    continue;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 12345.f) sink[0] = acc;
        if (WORK == 6) {
            asm volatile("bar.sync 2, %0;" ::"n"(NC));
            if (threadIdx.x == 0) qdone = 1;
        }
    }
}

template <int UNROLL>
__global__ void k_ldg(const float4* __restrict__ src, size_t n4, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride * UNROLL) {
        float4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            if (i + u * stride < n4) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            if (i + u * stride < n4) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 12345.f) sink[0] = acc;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

template <int STAGES, int SBYTES, int CONS_WARPS, int WORK, int RUN = 1>
void run_ring(const float* src, size_t bytes, unsigned* next, float* sink, int ctas_per_sm, int sms) {
    const size_t nchunks = bytes / SBYTES;
    const size_t smem = (size_t)STAGES * SBYTES + 2 * STAGES * 8 + STAGES * 4;
    cudaFuncSetAttribute(k_ring<STAGES, SBYTES, CONS_WARPS, WORK, RUN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
        cudaMemset(next, 0, 4);
        cudaEventRecord(a);
        k_ring<STAGES, SBYTES, CONS_WARPS, WORK, RUN><<<sms * ctas_per_sm, (CONS_WARPS + 2) * 32, smem>>>(src, nchunks, next, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        best = fminf(best, time_ms(a, b));
    }
    cudaError_t e = cudaGetLastError();
    printf("ring stages=%d sbytes=%d cons_warps=%d work=%d run=%d ctas/sm=%d: %.0f GB/s %s\n", STAGES, SBYTES, CONS_WARPS, WORK,
           RUN, ctas_per_sm, nchunks * (double)SBYTES / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int UNROLL>
void run_ldg(const float* src, size_t bytes, float* sink, int blocks, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        k_ldg<UNROLL><<<blocks, threads>>>(reinterpret_cast<const float4*>(src), bytes / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        best = fminf(best, time_ms(a, b));
    }
    printf("ldg unroll=%d blocks=%d threads=%d: %.0f GB/s\n", UNROLL, blocks, threads, bytes / (best * 1e-3) / 1e9);
}

int main() {
    const size_t bytes = 2ull << 30;  // 2 GiB
    float* src;
    float* sink;
    unsigned* next;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 0, bytes);
    cudaMalloc(&sink, 16384);
    cudaMalloc(&next, 4096);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run_ring<4, 16384, 8, 5, 38>(src, bytes, next, sink, 2, sms);
    run_ring<4, 16384, 8, 7, 38>(src, bytes, next, sink, 2, sms);
    return 0;
}
