// ssv_api.cpp -- the C-ABI host layer (include/ssv/ssv.h): context, argument
// validation with the reference's error behaviour, scratch management, and
// the host-buffer entry points.  No computation happens here: every result is
// produced by the sm_100a kernels in ssv_kernels.cu, and there is no CPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "ssv_launch.h"

using namespace ssv;

struct ssv_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    int launches = 0;
    // stream-ordered scratch
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    unsigned* counters = nullptr;  // [4]: next, exit, rejected rows, decisions (kernels leave them 0)
    void* slots = nullptr;  // streaming kernel's self-flagging slots (part, gpart): all kSlotEmpty between launches
    size_t slots_bytes = 0;
    uint32_t* status_dev = nullptr;  // default status word
    // host-entry staging
    void* stage = nullptr;
    size_t stage_bytes = 0;
    uint32_t* status_host = nullptr;  // pinned
    void* hstage = nullptr;           // pinned mirror of the small host-entry inputs / outputs
    size_t hstage_bytes = 0;
    ProfileHook prof;
    bool profiling = false;
    int path = SSV_PATH_AUTO;
    int32_t plan[6] = {0, 0, 0, 0, 0, 0};  // ssv_last_plan
    unsigned long long* trace = nullptr;  // diagnostics (ssv_debug_trace)
    int trace_cap = 0;
    uint32_t* status_mirror = nullptr;    // set by run_host for the duration of its launch
    // Stream hand-over: the scratch and counters are shared by every launch of
    // the context, so a launch on a new stream must follow the last launch on
    // the previous one (ssv_set_stream records / waits on this event).
    cudaEvent_t handover = nullptr;
    bool dirty = false;  // a launch was issued on `stream` since the last hand-over
    Launch launcher() {
        dirty = true;
        return Launch{stream, &launches, profiling ? &prof : nullptr};
    }
};

namespace {

const char* kVersion = "ssv 0.1.0 (sm_100a)";

int fail(ssv_ctx* ctx, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    return code;
}

int cuda_fail(ssv_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, SSV_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                              \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

size_t dtype_size(int dt) { return dt == SSV_F64 ? 8 : (dt == SSV_BF16 ? 2 : 4); }
size_t out_elem_size(int dt) { return dt == SSV_F64 ? 8 : 4; }
size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

enum Variant { V_EXACT = ACT_SOFTMAX, V_SIGMOID = ACT_SIGMOID, V_PROBS = ACT_PROBS };

const char* variant_name(int v) {
    return v == V_EXACT ? "verify_exact" : (v == V_SIGMOID ? "verify_sigmoid" : "verify_probs");
}

// Shape checks shared by every entry point: StepInputs::validate
// (verify_reference.cpp:12-21), SigmoidStepInputs::validate
// (verify_sigmoid.cpp:14-24) and ScaleBounds::validate (dist.cpp:11-15).
int check_shape(ssv_ctx* ctx, int variant, const ssv_verify_args* a, const ssv_verify_out* o) {
    if (!ctx) return SSV_EINVAL;
    if (!a || !o) return fail(ctx, SSV_EINVAL, "%s: null args/out", variant_name(variant));
    if (a->B < 1 || a->gamma < 1 || a->V < 1)
        return fail(ctx, SSV_EINVAL, "Grid3: all dimensions must be >= 1");
    if (a->p_steps != a->gamma && a->p_steps != a->gamma + 1)
        return fail(ctx, SSV_EINVAL, "StepInputs: p must be B x gamma(+1) x V matching q");
    if (a->dtype != SSV_F32 && a->dtype != SSV_BF16 && a->dtype != SSV_F64)
        return fail(ctx, SSV_EINVAL, "%s: unknown dtype %d", variant_name(variant), a->dtype);
    if (variant == V_SIGMOID) {
        if (!std::isfinite(a->alpha) || !std::isfinite(a->beta) || !(a->alpha < 0.0) || !(a->beta > 0.0))
            return fail(ctx, SSV_EINVAL, "ScaleBounds: require alpha < 0 < beta, both finite");
    }
    if (!a->z_p || !a->z_q || !a->draft_tokens || !a->uniforms)
        return fail(ctx, SSV_EINVAL, "%s: null input pointer", variant_name(variant));
    if (!o->accepted_len || !o->final_token || !o->resample_used || !o->tau || !o->residual_denom)
        return fail(ctx, SSV_EINVAL, "%s: null output pointer", variant_name(variant));
    if ((a->flags & SSV_WANT_P) && !o->p) return fail(ctx, SSV_EINVAL, "SSV_WANT_P without out->p");
    if ((a->flags & SSV_WANT_Q) && !o->q) return fail(ctx, SSV_EINVAL, "SSV_WANT_Q without out->q");
    if ((a->flags & SSV_WANT_RESIDUAL) && !o->residual)
        return fail(ctx, SSV_EINVAL, "SSV_WANT_RESIDUAL without out->residual");
    const long rows = (long)a->B * (2L * a->gamma + 1);
    if (rows * 64L > 0x7fffffffL) return fail(ctx, SSV_EINVAL, "%s: B*gamma too large", variant_name(variant));
    return SSV_OK;
}

// Grow the stream-ordered scratch; counters start at zero and the kernels
// leave them at zero; slots start empty and the kernels leave them empty.
int ensure_scratch(ssv_ctx* ctx, size_t bytes, size_t slot_bytes) {
    if (bytes <= ctx->scratch_bytes && ctx->counters && slot_bytes <= ctx->slots_bytes) return SSV_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    if (bytes > ctx->scratch_bytes) {
        if (ctx->scratch) CK(cudaFree(ctx->scratch));
        ctx->scratch = nullptr;
        const size_t nb = std::max(bytes, ctx->scratch_bytes * 2);
        CK(cudaMalloc(&ctx->scratch, nb));
        ctx->scratch_bytes = nb;
    }
    if (!ctx->counters) {
        CK(cudaMalloc(&ctx->counters, 4 * sizeof(unsigned)));
        // on the context's stream: the kernels that read the counters follow it
        CK(cudaMemsetAsync(ctx->counters, 0, 4 * sizeof(unsigned), ctx->stream));
    }
    if (slot_bytes > ctx->slots_bytes) {
        if (ctx->slots) CK(cudaFree(ctx->slots));
        ctx->slots = nullptr;
        const size_t nb = align_up(std::max(slot_bytes, ctx->slots_bytes * 2));
        CK(cudaMalloc(&ctx->slots, nb));
        launch_fill_slots(ctx->slots, nb / sizeof(unsigned long long), ctx->stream);
        CK(cudaGetLastError());
        ctx->slots_bytes = nb;
    }
    return SSV_OK;
}

struct Layout {
    size_t rowstat, cgpart, rejl, extra, total;  // scratch
    size_t part, gpart, dslot, slots;      // slot region
};

Layout plan_scratch(const StepParams& P, size_t extra_bytes) {
    Layout L;
    size_t off = 0;
    L.rowstat = off;
    off = align_up(off + (size_t)P.B * std::max(P.NR, 1) * sizeof(double2));
    L.cgpart = off;
    off = align_up(off + (size_t)P.B * P.NG * sizeof(double2));
    L.rejl = off;
    off = align_up(off + (size_t)P.B * sizeof(int));
    L.extra = off;
    off = align_up(off + extra_bytes);
    L.total = off;
    off = 0;
    L.part = off;
    off = align_up(off + (size_t)P.B * std::max(P.NR, 1) * std::max(P.KP, 1) * sizeof(double2));
    L.gpart = off;
    off = align_up(off + (size_t)P.B * P.NG * sizeof(double2));
    L.dslot = off;
    off = align_up(off + (size_t)P.B * 3 * sizeof(double2));
    L.slots = off;
    return L;
}

void bind_scratch(ssv_ctx* ctx, StepParams& P, const Layout& L) {
    char* s = static_cast<char*>(ctx->scratch);
    char* z = static_cast<char*>(ctx->slots);
    P.part = reinterpret_cast<double2*>(z + L.part);
    P.gpart = reinterpret_cast<double2*>(z + L.gpart);
    P.rowstat = reinterpret_cast<double2*>(s + L.rowstat);
    P.dslot = reinterpret_cast<double2*>(z + L.dslot);
    P.cgpart = reinterpret_cast<double2*>(s + L.cgpart);
    P.next = ctx->counters;
    P.exit_cnt = ctx->counters + 1;
    P.rej_cnt = ctx->counters + 2;
    P.dec_cnt = ctx->counters + 3;
    P.rej_list = reinterpret_cast<int*>(s + L.rejl);
}

int run_device(ssv_ctx* ctx, int variant, const ssv_verify_args* a, ssv_verify_out* o) {
    int rc = check_shape(ctx, variant, a, o);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    StepParams P{};
    P.zp = a->z_p;
    P.zq = a->z_q;
    P.ids = a->draft_tokens;
    P.u = a->uniforms;
    P.B = a->B;
    P.G = a->gamma;
    P.V = a->V;
    P.PS = a->p_steps;
    const bool want_p = a->flags & SSV_WANT_P;
    P.NR = 2 * P.G + ((want_p && P.PS == P.G + 1) ? 1 : 0);
    P.alpha = a->alpha;
    P.width = a->beta - a->alpha;
    P.check_uniforms = variant != V_SIGMOID;
    P.emulate_half = variant == V_SIGMOID && (a->flags & SSV_EMULATE_HALF) ? 1 : 0;
    const int act = P.emulate_half ? ACT_SIGMOID_HALF : variant;  // the emulation has its own kernels
    plan_geometry(a->dtype, act, P);
    const bool mat = a->flags & (SSV_WANT_P | SSV_WANT_Q | SSV_WANT_RESIDUAL);
    if (ctx->path != SSV_PATH_STREAMING && ctx->path != SSV_PATH_SLAB)
        plan_cluster(a->dtype, act, P, ctx->path != SSV_PATH_CLUSTER_RING);
    // The slab kernel is selected only on request (measured slower than the
    // streaming kernel on every shape so far).
    if (P.cl_size == 0 && !mat && ctx->path == SSV_PATH_SLAB) plan_slab(a->dtype, act, P);
    if (P.cl_size == 0 && ctx->path != SSV_PATH_STREAMING) plan_sig(a->dtype, act, P);
    const Layout L = plan_scratch(P, 0);
    rc = ensure_scratch(ctx, L.total, L.slots);
    if (rc) return rc;
    bind_scratch(ctx, P, L);
    P.acc = o->accepted_len;
    P.fin = o->final_token;
    P.rsu = o->resample_used;
    P.tau = o->tau;
    P.rden = o->residual_denom;
    P.status = o->status ? o->status : ctx->status_dev;
    P.status_mirror = ctx->status_mirror;
    P.trace = (ctx->trace && trace_slots(P) <= ctx->trace_cap) ? ctx->trace : nullptr;
    ctx->launches = 0;
    // kernel, cluster size, threads, slots, rows, pieces (ssv_last_plan)
    ctx->plan[0] = P.cl_size > 0 ? (P.cl_resident ? SSV_PLAN_CLUSTER_RESIDENT : SSV_PLAN_CLUSTER_RING)
                                 : (P.sl_on ? SSV_PLAN_SLAB : (P.sg_on ? SSV_PLAN_SIGMOID_STREAM : SSV_PLAN_STREAMING));
    ctx->plan[1] = P.cl_size;
    ctx->plan[2] = P.cl_size > 0 ? P.cl_threads : kCtaThreads;
    ctx->plan[3] = P.cl_slots;
    ctx->plan[4] = P.cl_rows;
    ctx->plan[5] = P.cl_pieces;
    launch_verify(a->dtype, act, P, want_p ? o->p : nullptr, (a->flags & SSV_WANT_Q) ? o->q : nullptr,
                  (a->flags & SSV_WANT_RESIDUAL) ? o->residual : nullptr, ctx->launcher());
    CK(cudaGetLastError());
    return SSV_OK;
}

// StepInputs::validate (verify_reference.cpp:22-33) on host data, with the
// reference's messages.  The sigmoid variant does not check the uniforms
// (verify_sigmoid.cpp:25-31).
int check_host_values(ssv_ctx* ctx, int variant, const ssv_verify_args* a) {
    const int B = a->B, G = a->gamma;
    for (int b = 0; b < B; ++b) {
        for (int c = 0; c < G; ++c) {
            const int32_t t = a->draft_tokens[(size_t)b * G + c];
            if (t < 0 || t >= a->V)
                return fail(ctx, SSV_EINVAL,
                            variant == V_SIGMOID ? "SigmoidStepInputs: draft token out of range"
                                                 : "StepInputs: draft token out of vocabulary range");
        }
        if (variant != V_SIGMOID) {
            for (int c = 0; c <= G; ++c) {
                const double u = a->uniforms[(size_t)b * (G + 1) + c];
                if (!(u >= 0.0) || !(u < 1.0))
                    return fail(ctx, SSV_EINVAL, "StepInputs: uniforms must lie in [0, 1)");
            }
        }
    }
    return SSV_OK;
}

int status_to_rc(ssv_ctx* ctx, uint32_t st) {
    if (st & SSV_STATUS_NONFINITE) return fail(ctx, SSV_EINVAL, "logit row contains a non-finite value");
    if (st & SSV_STATUS_TOKEN_RANGE) return fail(ctx, SSV_EINVAL, "StepInputs: draft token out of vocabulary range");
    if (st & SSV_STATUS_UNIFORM_RANGE) return fail(ctx, SSV_EINVAL, "StepInputs: uniforms must lie in [0, 1)");
    if (st & SSV_STATUS_NEGATIVE) return fail(ctx, SSV_EINVAL, "ratio_clamped: inputs must be non-negative");
    return SSV_OK;
}

int run_host(ssv_ctx* ctx, int variant, const ssv_verify_args* a, ssv_verify_out* o) {
    int rc = check_shape(ctx, variant, a, o);
    if (rc) return rc;
    rc = check_host_values(ctx, variant, a);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    const size_t es = dtype_size(a->dtype), os = out_elem_size(a->dtype);
    const size_t B = a->B, G = a->gamma, V = a->V, PS = a->p_steps;
    const size_t np = B * PS * V, nq = B * G * V;
    struct Piece {
        size_t off, bytes;
    };
    // Device staging: the logits, then ONE block of small inputs (ids,
    // uniforms, a zeroed status word).  The small outputs are written by the
    // kernels straight into pinned host memory (mapped, UVA), so a call costs
    // the logits copies + one small H2D and no D2H copy (a D2H costs ~8 us of
    // copy-engine latency on the critical path, tools/host_overhead.cpp).
    size_t off = 0;
    auto take = [&](size_t bytes) {
        Piece p{off, bytes};
        off = align_up(off + bytes);
        return p;
    };
    const Piece zp = take(np * es), zq = take(nq * es);
    const size_t small0 = off;
    const Piece ids = take(B * G * 4), u = take(B * (G + 1) * 8), st = take(4);
    const size_t small_in = off - small0;
    const bool wp = a->flags & SSV_WANT_P, wq = a->flags & SSV_WANT_Q, wr = a->flags & SSV_WANT_RESIDUAL;
    const Piece pp = take(wp ? np * os : 0), pq = take(wq ? nq * os : 0), pr = take(wr ? nq * os : 0);
    // pinned host block: [small inputs][status mirror][small outputs]
    size_t hoff = small_in;
    auto htake = [&](size_t bytes) {
        Piece p{hoff, bytes};
        hoff = align_up(hoff + bytes);
        return p;
    };
    const Piece hst = htake(4), acc = htake(B * 4), fin = htake(B * 4), rsu = htake(B), tau = htake(B * G * 8),
                rden = htake(B * 8);
    const size_t hbytes = hoff;
    if (off > ctx->stage_bytes) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->stage) CK(cudaFree(ctx->stage));
        ctx->stage = nullptr;
        CK(cudaMalloc(&ctx->stage, off));
        ctx->stage_bytes = off;
    }
    if (hbytes > ctx->hstage_bytes) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->hstage) CK(cudaFreeHost(ctx->hstage));
        ctx->hstage = nullptr;
        CK(cudaMallocHost(&ctx->hstage, hbytes));
        ctx->hstage_bytes = hbytes;
    }
    char* d = static_cast<char*>(ctx->stage);
    char* h = static_cast<char*>(ctx->hstage);  // [0, small_in) mirrors d + small0
    std::memcpy(h + (ids.off - small0), a->draft_tokens, ids.bytes);
    std::memcpy(h + (u.off - small0), a->uniforms, u.bytes);
    std::memset(h + (st.off - small0), 0, 4);
    std::memset(h + hst.off, 0, 4);
    cudaStream_t s = ctx->stream;
    // One stream: measured on B200 / PCIe 5, C2's 18.26 MB cross in 336 us as
    // two copies on one stream, 343 us split over two streams (copy engines),
    // and every extra copy costs ~4 us (tools/pcie_bw.cu, tools/host_overhead.cpp).
    CK(cudaMemcpyAsync(d + small0, h, small_in, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d + zp.off, a->z_p, zp.bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d + zq.off, a->z_q, zq.bytes, cudaMemcpyHostToDevice, s));
    ssv_verify_args da = *a;
    da.z_p = d + zp.off;
    da.z_q = d + zq.off;
    da.draft_tokens = reinterpret_cast<const int32_t*>(d + ids.off);
    da.uniforms = reinterpret_cast<const double*>(d + u.off);
    ssv_verify_out dout{};
    dout.accepted_len = reinterpret_cast<int32_t*>(h + acc.off);
    dout.final_token = reinterpret_cast<int32_t*>(h + fin.off);
    dout.resample_used = reinterpret_cast<uint8_t*>(h + rsu.off);
    dout.tau = reinterpret_cast<double*>(h + tau.off);
    dout.residual_denom = reinterpret_cast<double*>(h + rden.off);
    dout.status = reinterpret_cast<uint32_t*>(d + st.off);
    dout.p = wp ? d + pp.off : nullptr;
    dout.q = wq ? d + pq.off : nullptr;
    dout.residual = wr ? d + pr.off : nullptr;
    ctx->status_mirror = reinterpret_cast<uint32_t*>(h + hst.off);
    rc = run_device(ctx, variant, &da, &dout);
    ctx->status_mirror = nullptr;
    if (rc) return rc;
    if (wp) CK(cudaMemcpyAsync(o->p, dout.p, pp.bytes, cudaMemcpyDeviceToHost, s));
    if (wq) CK(cudaMemcpyAsync(o->q, dout.q, pq.bytes, cudaMemcpyDeviceToHost, s));
    if (wr) CK(cudaMemcpyAsync(o->residual, dout.residual, pr.bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::memcpy(o->accepted_len, h + acc.off, acc.bytes);
    std::memcpy(o->final_token, h + fin.off, fin.bytes);
    std::memcpy(o->resample_used, h + rsu.off, rsu.bytes);
    std::memcpy(o->tau, h + tau.off, tau.bytes);
    std::memcpy(o->residual_denom, h + rden.off, rden.bytes);
    uint32_t status;
    std::memcpy(&status, h + hst.off, 4);
    if (o->status) *o->status = status;
    return status_to_rc(ctx, status);
}

}  // namespace

extern "C" {

const char* ssv_version(void) { return kVersion; }

int ssv_create(int device, ssv_ctx** out) {
    if (!out) return SSV_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return SSV_ECUDA;
    if (device < 0 || device >= n) return SSV_EINVAL;
    ssv_ctx* ctx = new (std::nothrow) ssv_ctx();
    if (!ctx) return SSV_ECUDA;
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->status_dev, sizeof(uint32_t)) != cudaSuccess ||
        cudaMemsetAsync(ctx->status_dev, 0, sizeof(uint32_t), ctx->own) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->handover, cudaEventDisableTiming) != cudaSuccess ||
        cudaMallocHost(&ctx->status_host, sizeof(uint32_t)) != cudaSuccess) {
        ssv_destroy(ctx);
        return SSV_ECUDA;
    }
    ctx->stream = ctx->own;
    *out = ctx;
    return SSV_OK;
}

static void free_profile(ssv_ctx* ctx) {
    for (int i = 0; i < 2 * ctx->prof.capacity; ++i) cudaEventDestroy(ctx->prof.ev[i]);
    delete[] ctx->prof.ev;
    delete[] ctx->prof.kid;
    ctx->prof = ProfileHook{};
    ctx->profiling = false;
}

void ssv_destroy(ssv_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    free_profile(ctx);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->counters) cudaFree(ctx->counters);
    if (ctx->slots) cudaFree(ctx->slots);
    if (ctx->status_dev) cudaFree(ctx->status_dev);
    if (ctx->stage) cudaFree(ctx->stage);
    if (ctx->hstage) cudaFreeHost(ctx->hstage);
    if (ctx->status_host) cudaFreeHost(ctx->status_host);
    if (ctx->handover) cudaEventDestroy(ctx->handover);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
}

int ssv_set_stream(ssv_ctx* ctx, void* stream) {
    if (!ctx) return SSV_EINVAL;
    cudaStream_t next = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream, as in CUDA
    if (next != ctx->stream && ctx->dirty) {
        // Order the new stream after the context's last launch on the old one
        // (they share scratch and counters).  Under graph capture on either
        // side there is nothing to order here: captured work runs when the
        // graph is launched, on the stream it is launched on.
        CK(cudaSetDevice(ctx->device));
        cudaStreamCaptureStatus a = cudaStreamCaptureStatusNone, b = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(ctx->stream, &a));
        CK(cudaStreamIsCapturing(next, &b));
        if (a == cudaStreamCaptureStatusNone && b == cudaStreamCaptureStatusNone) {
            CK(cudaEventRecord(ctx->handover, ctx->stream));
            CK(cudaStreamWaitEvent(next, ctx->handover, 0));
        }
        ctx->dirty = false;
    }
    ctx->stream = next;
    return SSV_OK;
}

void* ssv_get_stream(const ssv_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

const char* ssv_last_error(const ssv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int ssv_last_launch_count(const ssv_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ssv_last_plan(const ssv_ctx* ctx, int32_t* info, int32_t n) {
    if (!ctx || !info || n < 1) return SSV_EINVAL;
    for (int i = 0; i < n && i < 6; ++i) info[i] = ctx->plan[i];
    return SSV_OK;
}

int ssv_set_path(ssv_ctx* ctx, int32_t path) {
    if (!ctx) return SSV_EINVAL;
    if (path != SSV_PATH_AUTO && path != SSV_PATH_STREAMING && path != SSV_PATH_CLUSTER && path != SSV_PATH_CLUSTER_RING &&
        path != SSV_PATH_SLAB)
        return fail(ctx, SSV_EINVAL, "ssv_set_path: unknown path %d", path);
    ctx->path = path;
    return SSV_OK;
}

int ssv_profile_enable(ssv_ctx* ctx, int capacity) {
    if (!ctx || capacity < 1) return SSV_EINVAL;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    free_profile(ctx);
    ctx->prof.ev = new cudaEvent_t[2 * capacity];
    ctx->prof.kid = new int[capacity];
    for (int i = 0; i < 2 * capacity; ++i) {
        const cudaError_t e = cudaEventCreate(&ctx->prof.ev[i]);
        if (e != cudaSuccess) {
            ctx->prof.capacity = i / 2;
            free_profile(ctx);
            return cuda_fail(ctx, e, "cudaEventCreate");
        }
    }
    ctx->prof.capacity = capacity;
    ctx->prof.used = 0;
    ctx->profiling = true;
    return SSV_OK;
}

int ssv_profile_disable(ssv_ctx* ctx) {
    if (!ctx) return SSV_EINVAL;
    ctx->profiling = false;
    return SSV_OK;
}

int ssv_profile_reset(ssv_ctx* ctx) {
    if (!ctx) return SSV_EINVAL;
    ctx->prof.used = 0;
    return SSV_OK;
}

int ssv_profile_read(ssv_ctx* ctx, int32_t kernel_id, double* total_ms, int32_t* count) {
    if (!ctx || !total_ms || !count) return SSV_EINVAL;
    double tot = 0.0;
    int n = 0;
    for (int i = 0; i < ctx->prof.used; ++i) {
        if (ctx->prof.kid[i] != kernel_id) continue;
        float ms = 0.f;
        const cudaError_t e = cudaEventElapsedTime(&ms, ctx->prof.ev[2 * i], ctx->prof.ev[2 * i + 1]);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaEventElapsedTime");
        tot += ms;
        ++n;
    }
    *total_ms = tot;
    *count = n;
    return SSV_OK;
}

int ssv_debug_trace(ssv_ctx* ctx, int capacity, unsigned long long* host_out, int* grid_out) {
    if (!ctx) return SSV_EINVAL;
    CK(cudaSetDevice(ctx->device));
    if (host_out) {
        if (!ctx->trace) return fail(ctx, SSV_EINVAL, "ssv_debug_trace: tracing not enabled");
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaMemcpy(host_out, ctx->trace, (size_t)ctx->trace_cap * 8, cudaMemcpyDeviceToHost));
        return SSV_OK;
    }
    if (ctx->trace) CK(cudaFree(ctx->trace));
    ctx->trace = nullptr;
    ctx->trace_cap = 0;
    if (capacity > 0) {
        CK(cudaMalloc(&ctx->trace, (size_t)capacity * 8));
        CK(cudaMemsetAsync(ctx->trace, 0, (size_t)capacity * 8, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->trace_cap = capacity;
    }
    (void)grid_out;
    return SSV_OK;
}

int ssv_verify_exact(ssv_ctx* ctx, const ssv_verify_args* a, ssv_verify_out* o) {
    return run_device(ctx, V_EXACT, a, o);
}
int ssv_verify_sigmoid(ssv_ctx* ctx, const ssv_verify_args* a, ssv_verify_out* o) {
    return run_device(ctx, V_SIGMOID, a, o);
}
int ssv_verify_probs(ssv_ctx* ctx, const ssv_verify_args* a, ssv_verify_out* o) {
    return run_device(ctx, V_PROBS, a, o);
}
int ssv_verify_exact_host(ssv_ctx* ctx, const ssv_verify_args* a, ssv_verify_out* o) {
    return run_host(ctx, V_EXACT, a, o);
}
int ssv_verify_sigmoid_host(ssv_ctx* ctx, const ssv_verify_args* a, ssv_verify_out* o) {
    return run_host(ctx, V_SIGMOID, a, o);
}
int ssv_verify_probs_host(ssv_ctx* ctx, const ssv_verify_args* a, ssv_verify_out* o) {
    return run_host(ctx, V_PROBS, a, o);
}

void* ssv_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}
void ssv_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int ssv_sample_softmax(ssv_ctx* ctx, int32_t dtype, const void* logits, int32_t rows, int32_t V,
                       const double* uniforms, int32_t* tokens_out, uint32_t* status) {
    if (!ctx) return SSV_EINVAL;
    if (rows < 1 || V < 1) return fail(ctx, SSV_EINVAL, "sample_softmax: rows and V must be >= 1");
    if (dtype != SSV_F32 && dtype != SSV_BF16 && dtype != SSV_F64)
        return fail(ctx, SSV_EINVAL, "sample_softmax: unknown dtype %d", dtype);
    if (!logits || !uniforms || !tokens_out) return fail(ctx, SSV_EINVAL, "sample_softmax: null pointer");
    CK(cudaSetDevice(ctx->device));
    StepParams P{};
    P.zp = logits;
    P.zq = logits;
    P.u = uniforms;
    P.B = rows;
    P.G = 0;
    P.PS = 1;
    P.V = V;
    P.sample_mode = 1;
    plan_geometry(dtype, ACT_SOFTMAX, P);
    const Layout L = plan_scratch(P, 0);
    int rc = ensure_scratch(ctx, L.total, L.slots);
    if (rc) return rc;
    bind_scratch(ctx, P, L);
    P.fin = tokens_out;
    P.trace = (ctx->trace && trace_slots(P) <= ctx->trace_cap) ? ctx->trace : nullptr;
    P.status = status ? status : ctx->status_dev;
    ctx->launches = 0;
    launch_sample_softmax(dtype, P, ctx->launcher());
    CK(cudaGetLastError());
    return SSV_OK;
}

int ssv_make_bench_inputs(ssv_ctx* ctx, uint64_t seed, int32_t B, int32_t gamma, int32_t V, int32_t dtype,
                          void* z_p, void* z_q, int32_t* draft_tokens, double* uniforms) {
    if (!ctx) return SSV_EINVAL;
    if (B < 1 || gamma < 1 || V < 1) return fail(ctx, SSV_EINVAL, "make_bench_inputs: bad shape");
    if (dtype != SSV_F32 && dtype != SSV_BF16 && dtype != SSV_F64)
        return fail(ctx, SSV_EINVAL, "make_bench_inputs: unknown dtype %d", dtype);
    if (!z_p || !z_q || !draft_tokens || !uniforms) return fail(ctx, SSV_EINVAL, "make_bench_inputs: null pointer");
    CK(cudaSetDevice(ctx->device));
    // draft-draw uniforms live past the sampler's scratch
    StepParams P{};
    P.B = B * gamma;
    P.G = 0;
    P.PS = 1;
    P.V = V;
    P.sample_mode = 1;
    plan_geometry(dtype, ACT_SOFTMAX, P);
    const Layout L = plan_scratch(P, (size_t)B * gamma * sizeof(double));
    int rc = ensure_scratch(ctx, L.total, L.slots);
    if (rc) return rc;
    double* draft_u = reinterpret_cast<double*>(static_cast<char*>(ctx->scratch) + L.extra);
    int launches = 0;
    ctx->dirty = true;
    const Launch lau{ctx->stream, &launches, ctx->profiling ? &ctx->prof : nullptr};
    launch_gen_logits(dtype, seed, B, gamma, V, z_p, z_q, lau);
    launch_gen_uniforms(seed, B, gamma, V, draft_u, uniforms, lau);
    CK(cudaGetLastError());
    rc = ssv_sample_softmax(ctx, dtype, z_q, B * gamma, V, draft_u, draft_tokens, nullptr);
    ctx->launches += launches;
    return rc;
}

}  // extern "C"
