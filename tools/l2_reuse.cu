// l2_reuse.cu -- design microbenchmark: how much of a region read X MB ago is
// still in this B200's L2 (decides whether a re-read of the rejected row pair
// can be served from L2).  Three launches: read A (a MB), read B (d MB of other
// data), re-read A; run under
//   ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:k_read
// and compare the third launch's DRAM bytes with a MB.
//   mode 0: ld.global.nc (L1::no_allocate)   mode 1: cp.async.cg (the kernels' A-loads)
//   mode 2: ld.global with L2::evict_last for A
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_reuse l2_reuse.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_last(const uint4* p, unsigned long long pol) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

__global__ void k_read(const uint4* __restrict__ src, size_t n, int mode, float* sink) {
    __shared__ uint4 st[256 * 4];
    float acc = 0.f;
    unsigned long long pol = 0;
    if (mode == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint4 v;
        if (mode == 1) {
            const unsigned d = (unsigned)__cvta_generic_to_shared(&st[threadIdx.x]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\ncp.async.wait_all;" ::"r"(d), "l"(src + i) : "memory");
            v = st[threadIdx.x];
        } else if (mode == 2) {
            v = ld_last(src + i, pol);
        } else {
            v = ld_nc(src + i);
        }
        acc += __uint_as_float(v.x);
    }
    if (acc == 1234.5f) *sink = acc;
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    float* sink;
    cudaMalloc(&sink, 4);
    const size_t total = 1ull << 30;
    uint4* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int as[] = {16, 32, 48, 64, 96};
    const int ds[] = {0, 16, 32, 64, 96, 128};
    for (int a : as)
        for (int d : ds) {
            const size_t na = (size_t)a << 20, nd = (size_t)d << 20;
            // flush: read 512 MB elsewhere
            k_read<<<sms * 4, 256>>>(buf + ((size_t)512 << 20) / 16, ((size_t)400 << 20) / 16, 0, sink);
            k_read<<<sms * 4, 256>>>(buf, na / 16, mode, sink);                       // A
            if (d) k_read<<<sms * 4, 256>>>(buf + ((size_t)128 << 20) / 16, nd / 16, 0, sink);  // B
            k_read<<<sms * 4, 256>>>(buf, na / 16, 0, sink);                          // A again
            cudaDeviceSynchronize();
            printf("a=%d d=%d\n", a, d);
        }
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
