// ssv_launch.h -- internal contract between the C-ABI host layer (ssv_api.cpp)
// and the kernels (ssv_kernels.cu).  Not installed; include/ssv/ssv.h is the
// public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssv/ssv.h"

namespace ssv {

enum DType : int { DT_F32 = SSV_F32, DT_BF16 = SSV_BF16, DT_F64 = SSV_F64 };
enum Act : int { ACT_SOFTMAX = 0, ACT_SIGMOID = 1, ACT_PROBS = 2, ACT_SIGMOID_HALF = 3 };
// The binary16-emulated sigmoid (SSV_EMULATE_HALF) is its own instantiation so
// its fp64 emulation code stays out of the fast sigmoid kernels.
constexpr bool is_sigmoid(int act) { return act == ACT_SIGMOID || act == ACT_SIGMOID_HALF; }
enum Mode : int { MODE_NONE = 0, MODE_REJECT = 1, MODE_BONUS = 2 };

// Work-item geometry of k_verify (one CTA of kCtaThreads threads per item):
//   A-item  a run of runA consecutive 32 KB chunks (16-byte aligned) of one
//           statistics row, streamed through a kAStages-deep cp.async ring of
//           per-thread shared-memory slots (kAVec 16-byte vectors per thread
//           per chunk).
//   D-item  the decision of one batch row (exact only).
//   B-item  kCB consecutive elements of the rejected row pair (or the bonus
//           row) of one batch row; warp w of the CTA owns granule w of kGW
//           elements.
//   L-item  the inverse CDF (locate) of one batch row.
constexpr int kCtaThreads = 256;
constexpr int kWarpsPerCta = kCtaThreads / 32;
#ifndef SSV_AVEC
#define SSV_AVEC 8
#endif
#ifndef SSV_ASTAGES
#define SSV_ASTAGES 2
#endif
constexpr int kAVec = SSV_AVEC;                          // 16-byte vectors per thread per chunk
constexpr int kAStages = SSV_ASTAGES;                    // cp.async ring depth
constexpr int kAChunkBytes = kCtaThreads * kAVec * 16;   // 32 KB
constexpr int kDynSmem = kAStages * kAChunkBytes;        // 64 KB (aliased by locate's granule cache)
constexpr int kCB = 4096;
constexpr int kGW = kCB / (kCtaThreads / 32);  // 512
constexpr int kLocCap = 1024;                  // granule partials a locate caches in SMEM

// What batch row b still needs after the acceptance scan (decide -> B-items).
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
    int B, G, V, PS;   // batch, gamma, vocab, p steps (gamma or gamma+1)
    int NR;            // statistics rows per batch row (0: no A phase)
    int Kc;            // kAChunkBytes chunks per statistics row (any alignment)
    int runA;          // chunks per A-item
    int K;             // A-items (= partials) per statistics row
    int nA, nB;        // A- and B-items per batch row
    int NG;            // granules per row
    int nph[4];        // items per batch row of each phase (A, D, B, L)
    int off[4];        // segment offset of each phase: segment t holds phase p of row t - off[p]
    int nrange;        // segment ranges of constant composition
    int rseg[9];       // first segment of each range (+ end)
    unsigned ritem[9]; // first item of each range (+ total)
    int rsize[8];      // items per segment in each range
    unsigned n_items;  // work items
    int claim_ahead;   // claim the next item before processing the current one (set at launch)
    // Cluster path (small batches, see k_verify_cluster): one cluster of cl_size
    // CTAs per batch row, rank k stages elements [k*cl_se, (k+1)*cl_se) of every
    // row it needs in its shared memory.
    int cl_size, cl_se, cl_gps, cl_rows, cl_slots, cl_rowbytes, cl_smem;
    int cl_threads;  // 256, or 512 for all-resident slices with more rows than 8 warps
    int cl_resident;  // 1: the resident plan (every row slice in shared memory), 0: the ring plan
    int cl_pieces, cl_pe;  // ring units: each row slice in cl_pieces pieces of cl_pe elements
    // Slab path (exact, large batches, see k_verify_slab): one persistent CTA
    // per SM; unit u = (b, s) is slice s (kSlabVec 16-byte vectors) of all
    // 2*gamma drafted rows of batch row b, held in a shared-memory buffer until
    // b's decision is known.
    int sl_on, sl_ns, sl_nbuf, sl_dp, sl_lag, sl_ub, sl_smem, sl_grid, sl_dbg;
    // Sigmoid-stream path (large batches, see k_verify_sig): tiles of sg_te
    // elements of each batch row's needed row, sg_nt per row, a ring of sg_nbuf
    // tile buffers of sg_tb bytes per CTA.
    int sg_on, sg_te, sg_nt, sg_nbuf, sg_tb, sg_smem, sg_grid;
    int sg_warp;  // 1: k_verify_sigw (16-byte-aligned rows, barrier-free warp units)
    int sg_dw;    // k_verify_sigw: a deciding warp's share of the stream, in 16ths of the others'
    // Optional grids written by the verify kernel itself (resident cluster plan:
    // every row slice is still in shared memory after the decision), else by
    // k_materialize as a second pass.
    int fuse_grids;
    void* grid_p;
    void* grid_q;
    void* grid_r;
    int dbg;  // experiment bits (SSV_DBG_MODE), 0 in production
    double alpha, width;
    int sample_mode;     // sample softmax(z_p row b) with u[b] (draft sampling)
    int check_uniforms;  // StepInputs::validate checks u in [0,1); the sigmoid variant does not
    int emulate_half;    // sigmoid: binary16 emulation (SSV_EMULATE_HALF)
    unsigned long long* trace;  // diagnostics: [8*B] per-row phase stamps (tools/trace_step.py), [8*B..+2) kernel start/end
    // scratch
    // Slots (streaming kernel): each written once per launch with relaxed
    // stores, polled by its consumer until neither word holds kSlotEmpty, then
    // reset to kSlotEmpty -- the value is its own completion flag, so the
    // producers need no release fence (a MEMBAR that would drain their
    // in-flight cp.async ring).  The slot region is all-empty between launches.
    double2* part;     // [B][NR][KP] partials (max, sum e^(x-max)): A-item warps / slab slices
    double2* gpart;    // [B][NG]    granule partials
    double2* dslot;    // [B][3]     decision: (mode, row), (Mp, Sp), (Mq, Sq)
    int KP;            // partial slots per statistics row
    double2* rowstat;  // [B][NR]    row (max, sum)
    double2* cgpart;   // [B][NG]    cluster path: granule partials (last-positive fallback)
    unsigned* next;     // [1] item claim counter   (reset by the last CTA to exit)
    unsigned* exit_cnt; // [1] CTAs done            (reset by the last CTA to exit)
    unsigned* rej_cnt;  // [1] k_verify_sigw: rejected rows listed (reset by the last CTA to exit)
    unsigned* dec_cnt;  // [1] k_verify_sigw: decisions made      (reset by the last CTA to exit)
    int* rej_list;      // [B] k_verify_sigw: the rejected rows
    // outputs
    int32_t* acc;
    int32_t* fin;
    uint8_t* rsu;
    double* tau;
    double* rden;
    uint32_t* status;
    uint32_t* status_mirror;  // host entry points: pinned host copy of *status (no D2H copy)
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

// Empty-slot pattern: a NaN whose low word no computed partial can carry
// (partials are fp32-derived or fp64 sums: their NaN payloads have zero low bits).
constexpr unsigned long long kSlotEmpty = 0xFFF0DEADFFF0DEADull;

void plan_geometry(int dtype, int act, StepParams& P);
void launch_fill_slots(void* p, size_t n_u64, cudaStream_t st);
bool plan_cluster(int dtype, int act, StepParams& P, bool allow_resident = true);  // small-batch cluster path (sets cl_*)
bool plan_slab(int dtype, int act, StepParams& P);  // exact, large batches (sets sl_*)
bool plan_sig(int dtype, int act, StepParams& P);   // sigmoid, large batches (sets sg_*)
int trace_slots(const StepParams& P);
void launch_verify(int dtype, int act, const StepParams& P, void* outp, void* outq, void* outr,
                   const Launch& L);
void launch_sample_softmax(int dtype, const StepParams& P, const Launch& L);
void launch_gen_logits(int dtype, uint64_t seed, int B, int G, int V, void* zp, void* zq,
                       const Launch& L);
void launch_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u,
                         const Launch& L);

}  // namespace ssv
