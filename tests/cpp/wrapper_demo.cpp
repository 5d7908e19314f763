// Exercises the reference-typed C++ drop-in (include/ssv/ssv.hpp) on the
// SPEC.md worked examples.  Compiled by tests/test_abi.py on any host; run by
// tests/test_gpu_misc.py on the GPU.  Exit 0 = all checks passed.
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
