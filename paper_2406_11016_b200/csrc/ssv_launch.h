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

// Persistent-kernel geometry: a ring of kStages shared-memory stages of
// kStageBytes each, filled by TMA bulk copies.  A-items (row statistics) take
// one chunk of kStageBytes; B-items (the rejected pair / bonus row) take half a
// stage per row; one consumer warp owns one granule (B-item / 8) of a B-item.
constexpr int kStages = 4;
constexpr int kStageBytes = 16384;
constexpr int kStageStride = kStageBytes + 64;  // room for the 16-byte-aligned superset
constexpr int kHalfStride = kStageStride / 2;   // 16-byte aligned
constexpr int kLocCap = 1024;                   // granule partials cached in SMEM by locate

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
    int NR, K, CH;    // stat rows per batch row, A-chunks per row, A-chunk elements
    int NG;           // granules per row
    int CB, GW;       // B-item elements per row, granule elements (CB / 8)
    int nA, nBi, lag; // per batch row: A-items, B-items; lag = segments between a row's A- and D-items
    int nph[4];       // items per batch row of each phase (A, D, B, L)
    int off[4];       // segment offset of each phase
    int bp[9], nbp;   // sorted segment breakpoints (piecewise-constant segment sizes)
    int claim;        // items claimed per atomic by a producer
    int runA, RPR;    // chunks per A-run, A-runs (= partials) per stat row
    int runB;         // slices per B-run
    unsigned long long* trace;  // diagnostics: [2*grid] CTA start/end, [4*B] decide/locate start/end
    unsigned n_items;
    unsigned epoch;   // per-launch tag of the decision flags (never reset)
    double alpha, width;
    int sample_mode;    // K2 only: sample softmax(z_p row b) with u[b] (draft sampling)
    int check_uniforms; // StepInputs::validate checks u in [0,1); the sigmoid variant does not
    // scratch
    double2* part;     // [B][NR][RPR] run partials (max, sum e^(x-max))
    double2* rowstat;  // [B][NR]     row (max, sum)
    Decision* dec;     // [B]
    double2* gpart;    // [B][NG]     granule partials
    double* gat;       // [B][NR]     logit at the drafted token of each stat row
    unsigned* cnt1;    // [B] self-resetting completion counters (A-items)
    unsigned* cnt2;    // [B]                                      (B-items)
    unsigned* flag;    // [B] decision published (== epoch)
    unsigned* next;    // [1] work counter, reset by the last CTA to exit
    unsigned* exit_cnt;// [1]
    // outputs
    int32_t* acc;
    int32_t* fin;
    uint8_t* rsu;
    double* tau;
    double* rden;
    uint32_t* status;
};

// Kernel ids for the profiling hook (ssv_profile_*).
enum KernelId : int { KID_VERIFY = 0, KID_MATERIALIZE = 2, KID_GEN = 3, KID_COUNT = 4 };

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
        cudaEventRecordWithFlags(prof->ev[2 * i], st, cudaEventRecordExternal);
        return i;
    }
    void end(int i) const {
        ++*launches;
        if (i >= 0) cudaEventRecordWithFlags(prof->ev[2 * i + 1], st, cudaEventRecordExternal);
    }
};

void plan_geometry(int dtype, int act, StepParams& P);
int verify_grid(const StepParams& P);
void launch_verify(int dtype, int act, const StepParams& P, void* outp, void* outq, void* outr,
                   const Launch& L);
void launch_sample_softmax(int dtype, const StepParams& P, const Launch& L);
void launch_gen_logits(int dtype, uint64_t seed, int B, int G, int V, void* zp, void* zq,
                       const Launch& L);
void launch_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u,
                         const Launch& L);

}  // namespace ssv
