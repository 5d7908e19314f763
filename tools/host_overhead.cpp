// Fixed cost of one host-entry call (design check for ssv_verify_*_host):
// breaks a tiny and a C2-sized call into its pieces, timed on the host.
// g++ -O2 -std=c++17 -I include -I /usr/local/cuda/include tools/host_overhead.cpp \
//     -L paper_2406_11016_b200 -lssv -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2406_11016_b200 -o tools/host_overhead
#include <ssv/ssv.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <vector>

static double time_us(const std::function<void()>& f, int iters = 200) {
    for (int i = 0; i < 10; ++i) f();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
}

int main() {
    ssv_ctx* ctx;
    if (ssv_create(0, &ctx)) return 1;
    cudaStream_t s = (cudaStream_t)ssv_get_stream(ctx);
    for (auto shape : {std::vector<int>{1, 1, 7}, std::vector<int>{1, 5, 32000}, std::vector<int>{8, 5, 51865}}) {
        const int B = shape[0], G = shape[1], V = shape[2];
        const size_t np = (size_t)B * (G + 1) * V, nq = (size_t)B * G * V;
        float *hzp, *hzq;
        int32_t* hids;
        double* hu;
        hzp = (float*)ssv_host_alloc(np * 4);
        hzq = (float*)ssv_host_alloc(nq * 4);
        hids = (int32_t*)ssv_host_alloc(B * G * 4);
        hu = (double*)ssv_host_alloc(B * (G + 1) * 8);
        std::mt19937 rng(1);
        std::normal_distribution<float> nd;
        for (size_t i = 0; i < np; ++i) hzp[i] = 4 * nd(rng);
        for (size_t i = 0; i < nq; ++i) hzq[i] = hzp[i] + nd(rng);
        for (int i = 0; i < B * G; ++i) hids[i] = i % V;
        for (int i = 0; i < B * (G + 1); ++i) hu[i] = 0.5;
        std::vector<int32_t> acc(B), fin(B);
        std::vector<uint8_t> rsu(B);
        std::vector<double> tau(B * G), rden(B);
        ssv_verify_args a{};
        a.B = B; a.gamma = G; a.V = V; a.p_steps = G + 1; a.dtype = SSV_F32;
        a.z_p = hzp; a.z_q = hzq; a.draft_tokens = hids; a.uniforms = hu;
        ssv_verify_out o{};
        o.accepted_len = acc.data(); o.final_token = fin.data(); o.resample_used = rsu.data();
        o.tau = tau.data(); o.residual_denom = rden.data();
        printf("B=%d gamma=%d V=%d (%.2f MB logits)\n", B, G, V, (np + nq) * 4 / 1e6);
        printf("  host entry (exact)          %8.1f us\n", time_us([&] { ssv_verify_exact_host(ctx, &a, &o); }));
        printf("  host entry (sigmoid)        %8.1f us\n", time_us([&] {
                   a.alpha = -1e3; a.beta = 1e3; ssv_verify_sigmoid_host(ctx, &a, &o); }));
        // device pieces
        void *dzp, *dzq, *dsm;
        cudaMalloc(&dzp, np * 4); cudaMalloc(&dzq, nq * 4); cudaMalloc(&dsm, 1 << 20);
        cudaMemcpy(dzp, hzp, np * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dzq, hzq, nq * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dsm, hids, B * G * 4, cudaMemcpyHostToDevice);
        cudaMemcpy((char*)dsm + 4096, hu, B * (G + 1) * 8, cudaMemcpyHostToDevice);
        ssv_verify_args da = a;
        da.z_p = dzp; da.z_q = dzq; da.draft_tokens = (int32_t*)dsm; da.uniforms = (double*)((char*)dsm + 4096);
        char* d = (char*)dsm + 65536;
        ssv_verify_out dout{};
        dout.accepted_len = (int32_t*)d; dout.final_token = (int32_t*)(d + 8192); dout.resample_used = (uint8_t*)(d + 16384);
        dout.tau = (double*)(d + 24576); dout.residual_denom = (double*)(d + 32768);
        printf("  device entry + sync         %8.1f us\n", time_us([&] { ssv_verify_exact(ctx, &da, &dout); cudaStreamSynchronize(s); }));
        printf("  device entry, launch only   %8.1f us\n", time_us([&] { ssv_verify_exact(ctx, &da, &dout); }) );
        cudaStreamSynchronize(s);
        static char hbuf[65536];
        void* hp = ssv_host_alloc(65536);
        printf("  empty sync                  %8.1f us\n", time_us([&] { cudaStreamSynchronize(s); }));
        printf("  small H2D + sync            %8.1f us\n", time_us([&] { cudaMemcpyAsync(dsm, hp, 512, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); }));
        printf("  small D2H + sync            %8.1f us\n", time_us([&] { cudaMemcpyAsync(hp, dsm, 512, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }));
        printf("  H2D + kernel + D2H + sync   %8.1f us\n", time_us([&] {
                   cudaMemcpyAsync(dsm, hp, 512, cudaMemcpyHostToDevice, s);
                   ssv_verify_exact(ctx, &da, &dout);
                   cudaMemcpyAsync(hp, d, 512, cudaMemcpyDeviceToHost, s);
                   cudaStreamSynchronize(s); }));
        printf("  logits H2D (1 stream)+sync  %8.1f us\n", time_us([&] {
                   cudaMemcpyAsync(dzp, hzp, np * 4, cudaMemcpyHostToDevice, s);
                   cudaMemcpyAsync(dzq, hzq, nq * 4, cudaMemcpyHostToDevice, s);
                   cudaStreamSynchronize(s); }, 50));
        (void)hbuf;
        ssv_host_free(hp);
        cudaFree(dzp); cudaFree(dzq); cudaFree(dsm);
        ssv_host_free(hzp); ssv_host_free(hzq); ssv_host_free(hids); ssv_host_free(hu);
    }
    ssv_destroy(ctx);
    return 0;
}
