// Exercises the reference-typed C++ drop-in (include/ssv/ssv.hpp) on the
// SPEC.md worked examples.  Compiled by tests/test_abi.py on any host; run by
// tests/test_gpu_cpp.py on the GPU (which also runs tests/cpp/ref_backend.cpp,
// the same drop-in checked against the reference's own backends).  Exit 0 =
// all checks passed.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "ssv/ssv.hpp"

#define EXPECT(c)                                                   \
    do {                                                            \
        if (!(c)) {                                                 \
            std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                               \
        }                                                           \
    } while (0)

int main() {
    // |V|=2, gamma=1, p=[0.5,0.5], q=[0.9,0.1], token 0, r=0.6
    ssv::StepInputs in;
    in.p = ssv::ProbTensor(1, 1, 2);
    in.q = ssv::ProbTensor(1, 1, 2);
    in.p.row(0, 0)[0] = 0.5;
    in.p.row(0, 0)[1] = 0.5;
    in.q.row(0, 0)[0] = 0.9;
    in.q.row(0, 0)[1] = 0.1;
    in.draft_tokens = ssv::Matrix<int32_t>(1, 1, 0);
    in.uniforms = ssv::Matrix<double>(1, 2);
    in.uniforms(0, 0) = 0.6;
    in.uniforms(0, 1) = 0.3;
    const auto r = ssv::verify_sequential(in);
    EXPECT(r.accepted_len[0] == 0 && r.final_token[0] == 1 && r.resample_used[0] == 1);
    EXPECT(std::abs(r.tau(0, 0) - 5.0 / 9.0) < 1e-15 && std::abs(r.residual_denom[0] - 0.4) < 1e-15);
    in.uniforms(0, 0) = 0.5;
    auto f = ssv::verify_fused(in, ssv::plan_tiles(2, 1024), 2);
    EXPECT(f.result.accepted_len[0] == 1 && f.result.final_token[0] == ssv::kNoToken);
    EXPECT(f.trace.hbm_elem_reads_p == 2 && f.trace.kernel_invocations == 1);
    EXPECT(in.q.row(0, 0)[0] == 0.0 && std::abs(in.q.row(0, 0)[1] - 0.4) < 1e-15);  // residual written into q

    // sigmoid tau ~ 0.7614
    ssv::SigmoidStepInputs s;
    s.z_p = ssv::LogitTensor(1, 1, 2);
    s.z_q = ssv::LogitTensor(1, 1, 2);
    s.z_q.row(0, 0)[0] = 2000.0;
    s.z_q.row(0, 0)[1] = -2000.0;
    s.bounds = {-1e3, 1e3};
    s.draft_tokens = ssv::Matrix<int32_t>(1, 1, 0);
    s.uniforms = ssv::Matrix<double>(1, 2, 0.9);
    const auto rs = ssv::verify_sigmoid_sequential(s);
    EXPECT(std::abs(rs.tau(0, 0) - 0.761349) < 1e-6);

    // logits in: softmax([0, ln 3]) = [0.25, 0.75] for p, q uniform -> tau(token 1) = 1
    ssv::LogitStepInputs li;
    li.z_p = ssv::LogitTensor(1, 2, 2);
    li.z_q = ssv::LogitTensor(1, 1, 2);
    li.z_p.row(0, 0)[1] = std::log(3.0);
    li.draft_tokens = ssv::Matrix<int32_t>(1, 1, 1);
    li.uniforms = ssv::Matrix<double>(1, 2, 0.5);
    const auto re = ssv::verify_exact(li, ssv::Storage::f64);
    EXPECT(re.accepted_len[0] == 1 && re.tau(0, 0) == 1.0 && re.final_token[0] == 1);

    // plan_tiles (tile.cpp:11-23; SPEC.md:184 KAT) and the analytic trace of
    // verify_fused (tile.cpp:73-100 counting rules): B*gamma*V reads of each
    // grid, one invocation per (b, c, tile), writes a + partial + tau + resample
    {
        const auto plan = ssv::plan_tiles(50257, 1024);
        EXPECT(plan.tile_count() == 50 && plan.tiles.back().size() == 81 && plan.tiles[1].begin == 1024);
        ssv::StepInputs big;
        const size_t B = 2, G = 3, V = 2500;
        big.p = ssv::ProbTensor(B, G + 1, V);
        big.q = ssv::ProbTensor(B, G, V);
        for (size_t b = 0; b < B; ++b)
            for (size_t c = 0; c <= G; ++c)
                for (size_t i = 0; i < V; ++i) {
                    big.p.row(b, c)[i] = (1.0 + (double)((i * 7 + c) % 13)) / (7.0 * V);
                    if (c < G) big.q.row(b, c)[i] = (1.0 + (double)((i * 5 + b) % 11)) / (6.0 * V);
                }
        big.draft_tokens = ssv::Matrix<int32_t>(B, G, 17);
        big.uniforms = ssv::Matrix<double>(B, G + 1, 0.999);
        const ssv::StepInputs keep = big;
        const auto tp = ssv::plan_tiles(V, 1024);
        const auto fo = ssv::verify_fused(big, tp, 4);
        EXPECT(fo.trace.hbm_elem_reads_p == B * G * V && fo.trace.hbm_elem_reads_q == B * G * V);
        EXPECT(fo.trace.kernel_invocations == B * G * 3);
        uint64_t writes = B * G * V + B * G * 3 + B * G;
        for (size_t b = 0; b < B; ++b)
            if (fo.result.resample_used[b] && fo.result.residual_denom[b] > 0.0) writes += V;
        EXPECT(fo.trace.hbm_elem_writes == writes && fo.trace.peak_tile_bytes == (2 * 1024 + 1024) * 8);
        for (size_t b = 0; b < B; ++b)  // the residual max(0, p - q) replaced q (verify_fused.cpp:50)
            for (size_t c = 0; c < G; ++c)
                for (size_t i = 0; i < V; ++i)
                    EXPECT(big.q.row(b, c)[i] == std::max(0.0, keep.p.row(b, c)[i] - keep.q.row(b, c)[i]));
        EXPECT(fo.result == ssv::verify_sequential(keep));
    }

    // the sigmoid SEQUENTIAL entry point range-checks uniforms like the
    // reference (verify_sigmoid.cpp:50-58 -> verify_reference.cpp:28-33); the
    // fused one does not (SigmoidStepInputs::validate)
    {
        ssv::SigmoidStepInputs bad = s;
        bad.uniforms(0, 0) = 1.0;
        bool t1 = false;
        try {
            ssv::verify_sigmoid_sequential(bad);
        } catch (const std::invalid_argument&) {
            t1 = true;
        }
        EXPECT(t1);
        const auto fused = ssv::verify_sigmoid_fused(bad, ssv::plan_tiles(2, 1024), 1);
        EXPECT(fused.result.accepted_len[0] == 0);  // u = 1 > tau: rejected, no throw
    }

    // error behaviour: std::invalid_argument, as the reference's validate()
    bool threw = false;
    try {
        in.draft_tokens(0, 0) = 7;
        ssv::verify_sequential(in);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    std::printf("wrapper_demo ok\n");
    return 0;
}
