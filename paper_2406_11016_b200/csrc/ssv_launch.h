// ssv_launch.h -- internal contract between the C-ABI host layer (ssv_api.cpp)
// and the kernels (ssv_kernels.cu).  Not installed; include/ssv/ssv.h is the
// public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssv/ssv.h"

namespace ssv {

enum DType : int { DT_F32 = SSV_F32, DT_BF16 = SSV_BF16, DT_F64 = SSV_F64 };
enum Act : int { ACT_SOFTMAX = 0, ACT_SIGMOID = 1, ACT_PROBS = 2 };
enum Mode : int { MODE_NONE = 0, MODE_REJECT = 1, MODE_BONUS = 2 };

// Elements per K2 granule (one warp); the inverse-CDF's first level.
constexpr int kGranule = 512;

// What batch row b still needs after the acceptance scan (K1 -> K2).
struct Decision {
    int mode;  // Mode
    int row;   // rejected position c*, or gamma for the bonus row
    int pad0, pad1;
    double Mp, Sp, Mq, Sq;  // softmax statistics of the rejected pair
};

struct StepParams {
    const void* zp;
    const void* zq;
    const int32_t* ids;
    const double* u;
    int B, G, V, PS;  // batch, gamma, vocab, p steps (gamma or gamma+1)
    int NR, K, CH;    // K1: stat rows per batch row, chunks per row, chunk elements
    int NG;           // K2: granules per row
    double alpha, width;
    int sample_mode;    // K2 only: sample softmax(z_p row b) with u[b] (draft sampling)
    int check_uniforms; // StepInputs::validate checks u in [0,1); the sigmoid variant does not
    // scratch
    double2* part;     // [B][NR][K]  K1 chunk partials (max, sum e^(x-max))
    double2* rowstat;  // [B][NR]     row (max, sum)
    Decision* dec;     // [B]
    double2* gpart;    // [B][NG]     K2 granule partials
    unsigned* cnt1;    // [B] self-resetting completion counters
    unsigned* cnt2;    // [B]
    // outputs
    int32_t* acc;
    int32_t* fin;
    uint8_t* rsu;
    double* tau;
    double* rden;
    uint32_t* status;
};

// Kernel ids for the profiling hook (ssv_profile_*).
enum KernelId : int { KID_ROW_STATS = 0, KID_ROW_PASS = 1, KID_MATERIALIZE = 2, KID_GEN = 3, KID_COUNT = 4 };

// Optional per-launch CUDA-event bracketing (works inside stream capture: the
// records become graph event nodes).  Owned by the context.
struct ProfileHook {
    cudaEvent_t* ev = nullptr;  // 2 * capacity events
    int* kid = nullptr;         // kernel id of each bracketed launch
    int capacity = 0;
    int used = 0;
};

// Counts launches and brackets them with events when profiling is on.
struct Launch {
    cudaStream_t st;
    int* launches;
    ProfileHook* prof;
    int begin(int id) const {
        if (!prof || prof->used >= prof->capacity) return -1;
        const int i = prof->used++;
        prof->kid[i] = id;
        cudaEventRecord(prof->ev[2 * i], st);
        return i;
    }
    void end(int i) const {
        ++*launches;
        if (i >= 0) cudaEventRecord(prof->ev[2 * i + 1], st);
    }
};

int stats_chunks(int dtype, const StepParams& P);
void launch_verify(int dtype, int act, const StepParams& P, void* outp, void* outq, void* outr,
                   const Launch& L);
void launch_sample_softmax(int dtype, const StepParams& P, const Launch& L);
void launch_gen_logits(int dtype, uint64_t seed, int B, int G, int V, void* zp, void* zq,
                       const Launch& L);
void launch_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u,
                         const Launch& L);

}  // namespace ssv
