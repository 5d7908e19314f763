// ssv_kernels.cu -- sm_100a kernels of the speculative-sampling verification step.
//
// Single-launch implementations of the whole step (DESIGN.md 3 has the
// derivation and the roofline); the host picks one per call (plan_cluster,
// plan_sig, plan_slab):
//
// k_verify<T, ACT> -- streaming path (any size; C4 exact).  Persistent
// 256-thread CTAs claim work items in order from a global counter; every wait
// is on an item with a smaller claim index (held by a running CTA), so any
// grid size is deadlock-free.  Items of batch row b:
//   A-item  (exact only) a run of 32 KB chunks of one drafted p / q row through
//           a 2-deep cp.async ring of per-thread 16-byte slots (no barrier);
//           per thread a running max (FMNMX3 / packed bf16 max) and
//           sum e^(x - max) (FADD2/FMUL2 + MUFU ex2 in fp32 pairs of <= 16
//           terms, fp64 across); one fp64 partial per warp, stored into its
//           self-flagging slot (no release fence).  The next claimed run's
//           first chunk streams while this run drains.
//   D-item  exact: folds b's partial slots into row statistics, tau at every
//           drafted position in fp64 (activation.cpp:20-27 +
//           verify_reference.cpp:87-92), first rejection (93-96); sigmoid /
//           probabilities: the decision from the B*gamma gathered values alone
//           (paper section 3.2.2).  Publishes the decision slots.
//   B-item  8192 elements of the ONE row (bonus) or row PAIR (rejected
//           position) b still needs -> 512-element granule masses (re-read of
//           the rejected pair) into the granule slots.
//   L-item  inverse CDF: fp64 granule prefix, then the exact fp64 element scan
//           (locate_scan; dist.cpp:122-137 incl. its fallbacks); clears b's
//           slots.
//
// k_verify_cluster<T, ACT> -- cluster path (batches whose rows each get a
// co-resident thread-block cluster; C1-C3), described above the kernel.
// k_verify_sigw / k_verify_sig<T> -- the sigmoid variant beyond the cluster
// path (C4 sigmoid): decisions from the gathers first, then the bonus rows
// streamed once (barrier-free warp units for aligned rows, TMA tiles else).
// k_verify_slab<T> -- experimental exact kernel keeping every drafted row
// slice in shared memory until its decision (SSV_PATH_SLAB only).
//
// Every reduction has a fixed topology, so results are bit-identical run to
// run.  k_materialize (optional p / q / residual grids when the verify kernel
// does not write them itself) and the synthetic-input generator follow.
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "ssv_launch.h"
#include "ssv_device.cuh"
#include "ssv_pipe.cuh"
#include "ssv_exptab.h"

#include <cooperative_groups.h>

namespace ssv {

constexpr int kMaxRowsSmem = 96;  // row statistics a decide keeps in SMEM (gamma <= 47)
constexpr int kBG = 2;            // granules per warp per B-item (a B-item covers kBG * 4096 elements per row)
constexpr int kCtaMinBlocks = (227 * 1024) / (kDynSmem + 4096);  // resident CTAs per SM (3 with the 64 KB ring)
static_assert(kLocCap * sizeof(double2) <= (size_t)kDynSmem, "granule cache aliases the ring");

struct ItemRef {
    int type, b, idx;
};

constexpr int kMaxWarps = 16;  // block-reduction scratch: 512-thread cluster CTAs
struct Shared {
    float fred[kMaxWarps];
    double dred[kMaxWarps];
    int ired[kMaxWarps];
    int last;
    unsigned item, item_next;
    Decision dec;
    double2 wpart[kWarps];
    double2 rs[kMaxRowsSmem];
    double loc_d[4];  // locate: carry, denominator, bonus-row max / sum
    int loc_g, loc_useA;
};

// ---------------------------------------------------------------------------
// Row addressing.  Stat rows of batch row b: r < G -> p row r, G <= r < 2G ->
// q row r-G, r == 2G -> p row G (bonus, only when p is materialized).
template <typename T>
__device__ __forceinline__ const T* p_row(const StepParams& P, int b, int c) {
    return reinterpret_cast<const T*>(P.zp) + ((size_t)b * P.PS + c) * (size_t)P.V;
}
template <typename T>
__device__ __forceinline__ const T* q_row(const StepParams& P, int b, int c) {
    return reinterpret_cast<const T*>(P.zq) + ((size_t)b * P.G + c) * (size_t)P.V;
}
template <typename T>
__device__ __forceinline__ const T* stat_row(const StepParams& P, int b, int r) {
    if (r < P.G) return p_row<T>(P, b, r);
    if (r < 2 * P.G) return q_row<T>(P, b, r - P.G);
    return p_row<T>(P, b, P.G);
}

// Programmatic dependent launch: the verify kernels are launched with
// programmatic stream serialization, so the next kernel's CTAs may be
// scheduled while this grid drains (its launch latency overlaps our tail).
// Every CTA releases its dependents at entry and waits for its own
// predecessor's completion (and memory flush) before touching anything.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void flag(const StepParams& P, uint32_t bits) {
    uint32_t v = atomicOr(P.status, bits) | bits;
    if (P.status_mirror) {
        // Pinned host mirror (host entry points): bits only accumulate, so
        // rewrite until the mirror holds the device word's current value.
        for (;;) {
            *reinterpret_cast<volatile uint32_t*>(P.status_mirror) = v;
            __threadfence_system();
            const uint32_t w = *reinterpret_cast<volatile uint32_t*>(P.status);
            if (w == v) break;
            v = w;
        }
    }
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace(const StepParams& P, int idx) {
    if (P.trace) P.trace[idx] = gtime();
}

// The sigmoid activation as the reference evaluates it (verify_sigmoid.cpp:35-37).
template <int ACT>
__device__ __forceinline__ double sigmoid_act(const StepParams& P, double z) {
    if constexpr (ACT == ACT_SIGMOID_HALF) return sigmoid_half_d(z, P.alpha, P.width);
    return sigmoid_scaled_d(z, P.alpha, P.width);
}

__device__ __forceinline__ double ratio_clamped(double p, double q) {  // dist.cpp:104-112
    if (q <= kZeroEps) return p > kZeroEps ? 1.0 : 0.0;
    return fmin(1.0, p / q);
}

// Decision of batch row b as three self-flagging slots (StepParams::dslot):
// (mode, row), (Mp, Sp), (Mq, Sq).  Written once by the decide step, polled
// by every consumer, cleared by the row's locate once all consumers are done.
__device__ __forceinline__ void publish_decision(const StepParams& P, int b, const Decision& d) {
    st_slot(&P.dslot[3 * b + 1], make_double2(d.Mp, d.Sp));
    st_slot(&P.dslot[3 * b + 2], make_double2(d.Mq, d.Sq));
    st_slot(&P.dslot[3 * b + 0], make_double2((double)d.mode, (double)d.row));
}
__device__ __forceinline__ bool try_decision(const StepParams& P, int b, Decision& d) {
    double2 a, x, y;
    const bool ok = ld_slot(&P.dslot[3 * b + 0], a, kSlotEmpty) & ld_slot(&P.dslot[3 * b + 1], x, kSlotEmpty) &
                    ld_slot(&P.dslot[3 * b + 2], y, kSlotEmpty);
    d.mode = (int)a.x;
    d.row = (int)a.y;
    d.Mp = x.x;
    d.Sp = x.y;
    d.Mq = y.x;
    d.Sq = y.y;
    return ok;
}
__device__ __forceinline__ Decision wait_decision(const StepParams& P, int b) {
    Decision d;
    while (!try_decision(P, b, d)) __nanosleep(32);
    return d;
}

// ---------------------------------------------------------------------------
// Item order.  Segment t holds, in order, the A-items of batch row t - off[A],
// the D-item of t - off[D], the B-items of t - off[B] and the L-item of
// t - off[L] (each only if that row exists and the phase has items).  Every
// item waits only on items of an earlier phase of the same row, i.e. on
// smaller block indices.  The segment composition is piecewise constant over
// at most 8 ranges the host tabulates.
enum ItemType : int { IT_A = 0, IT_D = 1, IT_B = 2, IT_L = 3 };

__device__ __forceinline__ ItemRef decode_item(const StepParams& P, unsigned i) {
    int k = 0;
    while (k + 1 < P.nrange && i >= P.ritem[k + 1]) ++k;
    const unsigned rel = i - P.ritem[k], sz = (unsigned)P.rsize[k];
    const int t = P.rseg[k] + (int)(rel / sz);
    int o = (int)(rel % sz);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int b = t - P.off[p];
        if (P.nph[p] == 0 || b < 0 || b >= P.B) continue;
        if (o < P.nph[p]) return {p, b, o};
        o -= P.nph[p];
    }
    return {IT_L, 0, 0};  // unreachable
}

// ---------------------------------------------------------------------------
// A-item helpers.  Elements outside the row inside an edge vector are padded
// with -max (finite: neutral for the max, e^(pad - max) = 0, and invisible to
// the -inf check).
template <typename T>
__device__ __forceinline__ uint4 pad_vec();
template <>
__device__ __forceinline__ uint4 pad_vec<float>() { return make_uint4(0xff7fffffu, 0xff7fffffu, 0xff7fffffu, 0xff7fffffu); }
template <>
__device__ __forceinline__ uint4 pad_vec<__nv_bfloat16>() {
    return make_uint4(0xff7fff7fu, 0xff7fff7fu, 0xff7fff7fu, 0xff7fff7fu);
}
template <>
__device__ __forceinline__ uint4 pad_vec<double>() { return make_uint4(0xffffffffu, 0xffefffffu, 0xffffffffu, 0xffefffffu); }

// Keep elements [lo, hi) of the vector, pad the rest.
template <typename T>
__device__ __forceinline__ void mask_vec(uint4& w, int lo, int hi) {
    constexpr int VEC = Elem<T>::VEC;
    constexpr int EPW = VEC / 4 > 0 ? VEC / 4 : 1;  // elements per 32-bit word (1 or 2); fp64: 1/2
    const uint4 pad = pad_vec<T>();
    uint32_t* wv = reinterpret_cast<uint32_t*>(&w);
    const uint32_t* pv = reinterpret_cast<const uint32_t*>(&pad);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (sizeof(T) == 8) {
            const int e = q / 2;
            if (e < lo || e >= hi) wv[q] = pv[q];
        } else if (EPW == 1) {
            if (q < lo || q >= hi) wv[q] = pv[q];
        } else {
            const int e0 = 2 * q, e1 = 2 * q + 1;
            const uint32_t keep = ((e0 >= lo && e0 < hi) ? 0x0000ffffu : 0u) | ((e1 >= lo && e1 < hi) ? 0xffff0000u : 0u);
            wv[q] = (wv[q] & keep) | (pv[q] & ~keep);
        }
    }
}

// Thread partials over the loaded vectors: max / min (pass 1) and
// sum e^(x - M) (pass 2).  fp32 / bf16: FMNMX3, FADD2/FMUL2, MUFU ex2, fp32
// pair sums (<= 16 terms each) widened to fp64.  fp64 storage: libdevice exp.
template <typename T>
struct AStat;

template <>
struct AStat<float> {
    static __device__ __forceinline__ void minmax(const uint4& v, float& m, float& n) {
        const float a = __uint_as_float(v.x), b = __uint_as_float(v.y), c = __uint_as_float(v.z),
                    d = __uint_as_float(v.w);
        m = fmax3f(m, a, b);
        m = fmax3f(m, c, d);
        n = fmin3f_nan(n, a, b);
        n = fmin3f_nan(n, c, d);
    }
    static __device__ __forceinline__ void expsum(const uint4& v, float2 negM, float2& s) {
        const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
        float2 t0 = __fmul2_rn(__fadd2_rn(make_float2(__uint_as_float(v.x), __uint_as_float(v.y)), negM), l2e);
        float2 t1 = __fmul2_rn(__fadd2_rn(make_float2(__uint_as_float(v.z), __uint_as_float(v.w)), negM), l2e);
        s = __fadd2_rn(s, make_float2(ex2f(t0.x), ex2f(t0.y)));
        s = __fadd2_rn(s, make_float2(ex2f(t1.x), ex2f(t1.y)));
    }
};

template <>
struct AStat<__nv_bfloat16> {
    // max / min are exact in bf16: reduce the 8 packed values with VHMNMX.BF16_V2
    // (two per instruction, three inputs) and widen only the two survivors.
    static __device__ __forceinline__ uint32_t max2(uint32_t a, uint32_t b) {
        uint32_t r;
        asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
        return r;
    }
    static __device__ __forceinline__ uint32_t min2(uint32_t a, uint32_t b) {  // NaN-propagating (detector)
        uint32_t r;
        asm("min.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
        return r;
    }
    static __device__ __forceinline__ void minmax(const uint4& v, float& m, float& n) {
        const uint32_t mx = max2(max2(v.x, v.y), max2(v.z, v.w));
        const uint32_t mi = min2(min2(v.x, v.y), min2(v.z, v.w));
        m = fmax3f(m, __uint_as_float(mx << 16), __uint_as_float(mx & 0xffff0000u));
        n = fmin3f_nan(n, __uint_as_float(mi << 16), __uint_as_float(mi & 0xffff0000u));
    }
    static __device__ __forceinline__ void expsum(const uint4& v, float2 negM, float2& s) {
        const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
        float x[8];
        unpack(v, x);
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            const float2 t = __fmul2_rn(__fadd2_rn(make_float2(x[e], x[e + 1]), negM), l2e);
            s = __fadd2_rn(s, make_float2(ex2f(t.x), ex2f(t.y)));
        }
    }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Geometry of one A-run (a run of chunks of one statistics row).  Chunk c of
// a row is vectors [c * CV, (c + 1) * CV) of the 16-byte-aligned superset of
// the row; thread t owns vectors t + 256 j (j < kAVec) of every chunk.
template <typename T>
struct ARun {
    const uint4* vb;  // aligned row base
    int nvec_row, shift, tail;
    int c0, n;        // first chunk, chunks in the run
    __device__ __forceinline__ void init(const StepParams& P, int b, int idx) {
        constexpr int VEC = Elem<T>::VEC;
        const int r = idx / P.K, q = idx - r * P.K;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(stat_row<T>(P, b, r));
        shift = (int)((a0 & 15) / sizeof(T));
        nvec_row = (shift + P.V + VEC - 1) / VEC;
        tail = (shift + P.V) % VEC;
        vb = reinterpret_cast<const uint4*>(a0 - (a0 & 15));
        c0 = q * P.runA;
        n = min(c0 + P.runA, P.Kc) - c0;
    }
    // cp.async this thread's vectors of chunk c0 + k into ring slot `slot`
    __device__ __forceinline__ void issue(int k, uint4* ring, unsigned slot) const {
        constexpr int CV = kCtaThreads * kAVec;
        uint4* st = ring + (size_t)slot * CV;
#pragma unroll
        for (int j = 0; j < kAVec; ++j) {
            const int v = (c0 + k) * CV + threadIdx.x + kCtaThreads * j;
            if (v < nvec_row) cp_async16(st + j * kCtaThreads + threadIdx.x, vb + v);
        }
        cp_async_commit();
    }
};

// The CTA's cp.async stream: every issued chunk is one commit group and owns
// ring slot (position % kAStages); at most kAStages are outstanding.
struct AStream {
    unsigned issued = 0, consumed = 0;
    int next_pre = 0;  // chunks of the NEXT run already issued
};

__device__ __forceinline__ void cp_async_wait_pending(unsigned n) {  // wait until <= n groups pending
    static_assert(kAStages >= 2 && kAStages <= 8, "wait switch covers up to 7 pending groups");
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        default: cp_async_wait<6>(); break;
    }
}

// A-item: run q of statistics row r of batch row b.  The run's chunks stream
// through the ring kAStages - 1 ahead, and its tail already streams the first
// chunks of the next claimed item when that is an A-run too, so the loads of
// consecutive runs overlap (no drain / refill per run).  Per thread: running
// max (fp32) and sum e^(x - max) (fp64, the chunk's 16-32 terms summed in fp32
// pairs); an fp64 exp only when the max grows.  End of run: warp fold, CTA
// fold (fixed order) -> one partial.
template <typename T>
__device__ void item_A(const StepParams& P, int b, int idx, const ItemRef& nxt, Shared& sh, uint4* ring,
                       AStream& as) {
    constexpr int VEC = Elem<T>::VEC;
    constexpr int CV = kCtaThreads * kAVec;  // vectors per chunk
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = idx / P.K, q = idx - r * P.K;
    ARun<T> cur;
    cur.init(P, b, idx);
    ARun<T> nr;
    const bool pre = nxt.type == IT_A;
    if (pre) nr.init(P, nxt.b, nxt.idx);
    int cur_issued = as.next_pre;  // the previous run already issued these
    int nxt_issued = 0;
    const int shift = cur.shift, tail = cur.tail, nvec_row = cur.nvec_row;
    using A = typename Elem<T>::acc;
    A m = -FLT_MAX, mn = FLT_MAX;
    uint32_t mnp = 0x7f7f7f7fu;  // bf16: packed running minimum (largest finite pair)
    if constexpr (sizeof(T) == 8) {
        m = -DBL_MAX;
        mn = DBL_MAX;
    }
    double s = 0.0;
    for (int k = 0; k < cur.n; ++k) {
        while (as.issued - as.consumed < (unsigned)kAStages) {  // top up the ring
            if (cur_issued < cur.n) {
                cur.issue(cur_issued++, ring, as.issued % kAStages);
            } else if (pre && nxt_issued < min(nr.n, kAStages - 1)) {
                nr.issue(nxt_issued++, ring, as.issued % kAStages);
            } else {
                break;
            }
            ++as.issued;
        }
        cp_async_wait_pending(as.issued - as.consumed - 1);  // chunk k has landed (this thread's copies)
        const int c = cur.c0 + k;
        const uint4* st = ring + (size_t)(as.consumed % kAStages) * CV;
        ++as.consumed;
        uint4 w[kAVec];
        // CTA-uniform: only a row's first chunk (misaligned start) and its last
        // (partial / past-the-end vectors) need masking.
        const bool edge = (c == 0 && shift) || (c + 1) * CV > nvec_row - (tail ? 1 : 0);
        if (!edge) {
#pragma unroll
            for (int j = 0; j < kAVec; ++j) w[j] = st[j * kCtaThreads + tid];
        } else {
#pragma unroll
            for (int j = 0; j < kAVec; ++j) {
                const int v = c * CV + tid + kCtaThreads * j;
                w[j] = v < nvec_row ? st[j * kCtaThreads + tid] : pad_vec<T>();
                if (v == 0 && shift) mask_vec<T>(w[j], shift, VEC);        // the row's first vector
                if (v == nvec_row - 1 && tail) mask_vec<T>(w[j], 0, tail);  // and its last
            }
        }
        if constexpr (sizeof(T) == 8) {
            double cm = -DBL_MAX;
#pragma unroll
            for (int j = 0; j < kAVec; ++j) {
                double x[2];
                unpack(w[j], x);
                cm = fmax(cm, fmax(x[0], x[1]));
                mn = fmin_nan(mn, fmin_nan(x[0], x[1]));
            }
            if (cm > m) {
                if (s != 0.0) s *= exp(m - cm);
                m = cm;
            }
            if (m != -DBL_MAX) {
#pragma unroll
                for (int j = 0; j < kAVec; ++j) {
                    double x[2];
                    unpack(w[j], x);
                    s += exp(x[0] - m) + exp(x[1] - m);
                }
            }
        } else {
            float cm = -FLT_MAX;
            if constexpr (sizeof(T) == 2) {
                // bf16: packed VHMNMX over the chunk's words (4 per vector), one
                // running packed minimum for the whole run, a single widening of
                // the chunk maximum -- ~0.5 fewer instructions per element than
                // widening per vector.
                uint32_t mx = AStat<T>::max2(AStat<T>::max2(w[0].x, w[0].y), AStat<T>::max2(w[0].z, w[0].w));
                uint32_t mi = AStat<T>::min2(AStat<T>::min2(w[0].x, w[0].y), AStat<T>::min2(w[0].z, w[0].w));
#pragma unroll
                for (int j = 1; j < kAVec; ++j) {
                    mx = AStat<T>::max2(mx, AStat<T>::max2(AStat<T>::max2(w[j].x, w[j].y), AStat<T>::max2(w[j].z, w[j].w)));
                    mi = AStat<T>::min2(mi, AStat<T>::min2(AStat<T>::min2(w[j].x, w[j].y), AStat<T>::min2(w[j].z, w[j].w)));
                }
                cm = fmaxf(__uint_as_float(mx << 16), __uint_as_float(mx & 0xffff0000u));
                mnp = AStat<T>::min2(mnp, mi);
            } else {
#pragma unroll
                for (int j = 0; j < kAVec; ++j) AStat<T>::minmax(w[j], cm, mn);
            }
            // Warp-uniform running max: when the warp's max grows (rarely, after
            // the first chunks) every lane rescales its fp64 sum by the same
            // factor, and the end-of-run fold needs no exp at all.
            cm = warp_max(cm);
            if (cm > m) {
                if (s != 0.0) s *= exp((double)m - (double)cm);
                m = cm;
            }
            if (m != -FLT_MAX) {  // a thread that has seen pads only contributes nothing
                const float2 negM = make_float2(-m, -m);
#pragma unroll
                for (int j0 = 0; j0 < kAVec; j0 += 4) {  // <= 16 fp32 terms per pair lane, then fp64
                    float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = j0; j < j0 + 4 && j < kAVec; ++j) {
                        if (j & 1) AStat<T>::expsum(w[j], negM, s1);
                        else AStat<T>::expsum(w[j], negM, s0);
                    }
                    const float2 t = __fadd2_rn(s0, s1);
                    s += (double)t.x + (double)t.y;
                }
            }
        }
    }
    as.next_pre = nxt_issued;
    if constexpr (sizeof(T) == 2) mn = fmin3f_nan(FLT_MAX, __uint_as_float(mnp << 16), __uint_as_float(mnp & 0xffff0000u));
    // -inf or NaN logit (require_finite, dist.cpp:27-36; the running minimum
    // propagates NaN even where the max and the sum skip it); +inf surfaces in the sum
    if (__any_sync(kFull, !isfinite(mn)) && lane == 0) flag(P, SSV_STATUS_NONFINITE);
    // Warp fold (fixed order, fp64) -> one partial per warp; no CTA barrier, so
    // the warps of a CTA drift freely between runs.
    double M = (double)m;  // warp-uniform (fp32 path); fp64 storage keeps per-lane maxima
    double S;
    if constexpr (sizeof(T) == 8) {
        M = warp_max((double)m);
        S = warp_sum(s != 0.0 ? s * exp((double)m - M) : s);  // NaN propagates
    } else {
        S = warp_sum(s);
    }
    if (lane == 0) {
        if (isnan(S) || M == CUDART_INF) flag(P, SSV_STATUS_NONFINITE);
        if (S == 0.0) M = -CUDART_INF;  // a warp that saw pads only
        st_slot(&P.part[(((size_t)b * P.NR + r) * P.K + q) * kWarps + warp], make_double2(M, S));
    }
}

// ---------------------------------------------------------------------------
// Decisions.  Exact: row statistics from the A-item partials (fixed order,
// fp64), tau at every drafted position from the gathered logits (fp64;
// activation.cpp:20-27 + verify_reference.cpp:87-92), first rejection
// (verify_reference.cpp:93-96, inclusive u <= tau).  Runs on the CTA that
// completed the row's last A-item; publishes Decision + release flag.
// e^-n for an integer n >= 0 (table; 0 past fp64 underflow).
__device__ __forceinline__ double exp_neg_int(double n) {
    return n < (double)kExpNegN ? __ldg(&kExpNeg[(int)n]) : 0.0;
}

// Slab partials carry integer references R = ceil(slice max): two rows'
// slots folded per warp with every load of a chunk in flight, the rescale
// factors e^(R_s - R) read from kExpNeg (no fp64 exp on the decision path).
__device__ __forceinline__ void fold_int_ref2(double2* pa, double2* pb, int KP, double2& ra, double2& rb) {
    constexpr int NPL = 6;  // slots per lane per row per chunk (12 loads in flight)
    const int lane = threadIdx.x & 31;
    double m[2] = {-CUDART_INF, -CUDART_INF}, sm[2] = {0.0, 0.0};
    double2* pr[2] = {pa, pb};
    for (int k0 = 0; k0 < KP; k0 += NPL * 32) {
        double2 v[2][NPL];
        bool ok[2][NPL];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < NPL; ++i) {
                const int k = k0 + lane + 32 * i;
                const bool in = pr[h] != nullptr && k < KP;
                ok[h][i] = in ? ld_slot(&pr[h][k], v[h][i], kSlotEmpty) : true;
                if (!in) v[h][i] = make_double2(-CUDART_INF, 0.0);
            }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double cm = -CUDART_INF;
#pragma unroll
            for (int i = 0; i < NPL; ++i) {
                if (!ok[h][i]) v[h][i] = ld_slot_wait(&pr[h][k0 + lane + 32 * i], kSlotEmpty);
                cm = fmax(cm, v[h][i].x);
            }
            if (cm > m[h]) {
                if (sm[h] != 0.0) sm[h] *= exp_neg_int(cm - m[h]);
                m[h] = cm;
            }
#pragma unroll
            for (int i = 0; i < NPL; ++i)
                if (v[h][i].y != 0.0) sm[h] += v[h][i].y * exp_neg_int(m[h] - v[h][i].x);  // NaN propagates
        }
    }
    double2 r[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const double M = warp_max(m[h]);
        if (sm[h] != 0.0) sm[h] *= exp_neg_int(M - m[h]);
        r[h] = make_double2(M, warp_sum(sm[h]));
    }
    ra = r[0];
    rb = r[1];
}

template <typename T, bool SLAB = false>
__device__ void item_D(const StepParams& P, int b, Shared& sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = P.G;
    // The gathers and uniforms do not depend on the row statistics: issue
    // them before waiting so their latency overlaps the A-items' tail.
    double zp = 0.0, zq = 0.0, u = 0.0;
    if (tid < G) {
        int x = P.ids[(size_t)b * G + tid];
        if (x < 0 || x >= P.V) {
            flag(P, SSV_STATUS_TOKEN_RANGE);
            x = x < 0 ? 0 : P.V - 1;
        }
        zp = load_exact(p_row<T>(P, b, tid) + x);
        zq = load_exact(q_row<T>(P, b, tid) + x);
    }
    if (tid <= G) u = P.u[(size_t)b * (G + 1) + tid];
    const int KP = P.KP;  // partial slots per statistics row
    if constexpr (SLAB) {  // slab partials: integer references, two rows per pass
        for (int r0 = warp; r0 < P.NR; r0 += 2 * kWarps) {
            const int r1 = r0 + kWarps;
            double2* pa = P.part + ((size_t)b * P.NR + r0) * KP;
            double2* pb = r1 < P.NR ? P.part + ((size_t)b * P.NR + r1) * KP : nullptr;
            double2 st[2];
            fold_int_ref2(pa, pb, KP, st[0], st[1]);
            for (int k = lane; k < KP; k += 32) {
                clear_slot(&pa[k], kSlotEmpty);
                if (pb) clear_slot(&pb[k], kSlotEmpty);
            }
            if (lane == 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = h ? r1 : r0;
                    if (r >= P.NR) continue;
                    if (!isfinite(st[h].x) || !isfinite(st[h].y)) flag(P, SSV_STATUS_NONFINITE);  // NaN / +inf logit
                    P.rowstat[(size_t)b * P.NR + r] = st[h];
                    if (r < kMaxRowsSmem) sh.rs[r] = st[h];
                }
            }
        }
    }
    for (int r = SLAB ? P.NR : warp; r < P.NR; r += kWarps) {
        // Each partial slot is its own completion flag (written once by its
        // A-item, no counter): wait for the row's slots, fold, and leave
        // them empty for the next launch.
        double2* part = P.part + ((size_t)b * P.NR + r) * KP;
        // Chunks of 8 slots per lane with every load in flight (the slab
        // path folds ~300 slots per row), merged into a per-lane running
        // (max, sum) in fp64, then the warp fold.
        double m = -CUDART_INF, sm = 0.0;
        for (int k0 = 0; k0 < KP; k0 += 8 * 32) {
            double2 v[8];
            bool ok[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = k0 + lane + 32 * i;
                ok[i] = k < KP ? ld_slot(&part[k], v[i], kSlotEmpty) : true;
                if (k >= KP) v[i] = make_double2(-CUDART_INF, 0.0);
            }
            double cm = -CUDART_INF;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (!ok[i]) v[i] = ld_slot_wait(&part[k0 + lane + 32 * i], kSlotEmpty);
                cm = fmax(cm, v[i].x);
            }
            if (cm > m) {
                if (sm != 0.0) sm *= exp(m - cm);
                m = cm;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (v[i].y != 0.0) sm += v[i].y * exp(v[i].x - m);  // NaN propagates
        }
        for (int k = lane; k < KP; k += 32) clear_slot(&part[k], kSlotEmpty);
        {
            const double M = warp_max(m);
            sm = sm != 0.0 ? sm * exp(m - M) : sm;
            m = M;
        }
        sm = warp_sum(sm);
        if (lane == 0) {
            if (!isfinite(m) || !isfinite(sm)) flag(P, SSV_STATUS_NONFINITE);  // NaN / +inf logit
            P.rowstat[(size_t)b * P.NR + r] = make_double2(m, sm);
            if (r < kMaxRowsSmem) sh.rs[r] = make_double2(m, sm);
        }
    }
    __syncthreads();
    if (tid == 0) trace(P, 8 * b + 1);
    auto rs = [&](int r) -> double2 { return r < kMaxRowsSmem ? sh.rs[r] : __ldcg(&P.rowstat[(size_t)b * P.NR + r]); };
    auto tau_at = [&](int c, double zpc, double zqc) -> double {
        const double2 sp = rs(c), sq = rs(G + c);
        const double p = exp(zpc - sp.x) / sp.y;  // activation.cpp:20-27, dist.cpp:46-50
        const double q = exp(zqc - sq.x) / sq.y;
        return ratio_clamped(p, q);
    };
    int rej = 0x7fffffff;
    if (tid < G) {
        const double tau = tau_at(tid, zp, zq);
        P.tau[(size_t)b * G + tid] = tau;
        if (!(u <= tau)) rej = tid;  // verify_reference.cpp:93-96 (inclusive)
    }
    for (int c = tid + kCtaThreads; c < G; c += kCtaThreads) {  // gamma > 256
        int x = P.ids[(size_t)b * G + c];
        if (x < 0 || x >= P.V) {
            flag(P, SSV_STATUS_TOKEN_RANGE);
            x = x < 0 ? 0 : P.V - 1;
        }
        const double tau = tau_at(c, load_exact(p_row<T>(P, b, c) + x), load_exact(q_row<T>(P, b, c) + x));
        P.tau[(size_t)b * G + c] = tau;
        if (!(P.u[(size_t)b * (G + 1) + c] <= tau)) rej = min(rej, c);
    }
    if (P.check_uniforms) {
        if (tid <= G && (!(u >= 0.0) || !(u < 1.0))) flag(P, SSV_STATUS_UNIFORM_RANGE);
        for (int c = tid + kCtaThreads; c <= G; c += kCtaThreads) {
            const double uc = P.u[(size_t)b * (G + 1) + c];
            if (!(uc >= 0.0) || !(uc < 1.0)) flag(P, SSV_STATUS_UNIFORM_RANGE);
        }
    }
    const int a = min(block_reduce(rej, sh.ired, OpMin()), G);
    if (tid == 0) {
        P.acc[b] = a;
        Decision d{};
        if (a < G) {
            const double2 sp = rs(a), sq = rs(G + a);
            d.mode = MODE_REJECT;
            d.row = a;
            d.Mp = sp.x;
            d.Sp = sp.y;
            d.Mq = sq.x;
            d.Sq = sq.y;
        } else if (P.PS == G + 1) {
            d.mode = MODE_BONUS;
            d.row = G;
        } else {
            d.mode = MODE_NONE;
            P.fin[b] = -1;  // kNoToken, step.hpp:11
            P.rsu[b] = 0;
            P.rden[b] = 0.0;
        }
        publish_decision(P, b, d);
    }
}

// Sigmoid / probability decision from the gathered values only (warp 0 of a
// B-item).  verify_sigmoid.cpp:50-58 -> verify_reference.cpp:87-96; the
// sigmoid is evaluated in fp64 exactly as dist.cpp:60-62 does.  Only the
// row's first B-item writes the outputs; the others recompute identically.
template <typename T, int ACT>
__device__ void decide_gather(const StepParams& P, int b, bool write, Decision& out) {
    const int lane = threadIdx.x & 31;
    const int G = P.G;
    int accepted = G;
    for (int c0 = 0; c0 < G; c0 += 32) {
        const int c = c0 + lane;
        bool rej = false;
        if (c < G) {
            int x = P.ids[(size_t)b * G + c];
            if (x < 0 || x >= P.V) {
                if (write) flag(P, SSV_STATUS_TOKEN_RANGE);
                x = x < 0 ? 0 : P.V - 1;
            }
            const double zp = load_exact(p_row<T>(P, b, c) + x);
            const double zq = load_exact(q_row<T>(P, b, c) + x);
            double p, q;
            if (is_sigmoid(ACT)) {
                p = sigmoid_act<ACT>(P, zp);
                q = sigmoid_act<ACT>(P, zq);
            } else {
                p = zp;
                q = zq;
                if (write && (p < 0.0 || q < 0.0)) flag(P, SSV_STATUS_NEGATIVE);
            }
            const double tau = ratio_clamped(p, q);
            if (write) P.tau[(size_t)b * G + c] = tau;
            rej = !(P.u[(size_t)b * (G + 1) + c] <= tau);
        }
        const unsigned m = __ballot_sync(kFull, rej);
        if (m) {
            accepted = c0 + __ffs(m) - 1;
            if (write) {  // tau past the first rejection is still reported (step.hpp:39-41)
                for (int c2 = c0 + 32 + lane; c2 < G; c2 += 32) {
                    int x = P.ids[(size_t)b * G + c2];
                    if (x < 0 || x >= P.V) {
                        flag(P, SSV_STATUS_TOKEN_RANGE);
                        x = x < 0 ? 0 : P.V - 1;
                    }
                    const double zp = load_exact(p_row<T>(P, b, c2) + x);
                    const double zq = load_exact(q_row<T>(P, b, c2) + x);
                    double p = zp, q = zq;
                    if (is_sigmoid(ACT)) {
                        p = sigmoid_act<ACT>(P, zp);
                        q = sigmoid_act<ACT>(P, zq);
                    } else if (p < 0.0 || q < 0.0) {
                        flag(P, SSV_STATUS_NEGATIVE);
                    }
                    P.tau[(size_t)b * G + c2] = ratio_clamped(p, q);
                }
            }
            break;
        }
    }
    if (write && P.check_uniforms) {
        for (int c = lane; c <= G; c += 32) {
            const double u = P.u[(size_t)b * (G + 1) + c];
            if (!(u >= 0.0) || !(u < 1.0)) flag(P, SSV_STATUS_UNIFORM_RANGE);
        }
    }
    if (lane == 0) {
        Decision d{};
        d.Sp = d.Sq = 1.0;
        if (accepted < G) {
            d.mode = MODE_REJECT;
            d.row = accepted;
        } else if (P.PS == G + 1) {
            d.mode = MODE_BONUS;
            d.row = G;
        } else {
            d.mode = MODE_NONE;
        }
        if (write) {
            P.acc[b] = accepted;
            if (d.mode == MODE_NONE) {
                P.fin[b] = -1;
                P.rsu[b] = 0;
                P.rden[b] = 0.0;
            }
        }
        out = d;
    }
}

// ---------------------------------------------------------------------------
// Per-element values.  Streaming (acc precision) and exact (fp64) forms.
struct RowCtx {
    int mode;   // MODE_REJECT / MODE_BONUS
    bool useA;  // reject: sample the residual (else the degenerate fallback on p)
    double Mp, Sp, Mq, Sq;
    double denom;
};

template <int ACT>
__device__ __forceinline__ double exact_act(const StepParams& P, double z, double M, double S) {
    if (ACT == ACT_SOFTMAX) return exp(z - M) / S;  // dist.cpp:46-50
    if (is_sigmoid(ACT)) return sigmoid_act<ACT>(P, z);
    return z;
}

// Value the inverse CDF scans at element i (fp64): residual max(0, p - q)
// (verify_reference.cpp:51-55) or the p row itself (fallback / bonus).
// A shared-memory copy of elements [lo, hi) of the p and q rows (cluster path,
// every row slice resident): p[i - lo], q[i - lo]; hi = 0 when there is none.
template <typename T>
struct RowSlice {
    const T* p = nullptr;
    const T* q = nullptr;
    int lo = 0, hi = 0;
};

template <typename T>
__device__ __forceinline__ double row_elem(const T* g, const T* s, const RowSlice<T>& S, int i) {
    return i >= S.lo && i < S.hi ? (double)load_smem_elem(s + (i - S.lo)) : load_exact(g + i);
}

template <typename T, int ACT>
__device__ __forceinline__ double exact_value(const StepParams& P, const RowCtx& R, const T* pr, const T* qr,
                                              int i, const RowSlice<T>& S = RowSlice<T>()) {
    const double p = exact_act<ACT>(P, row_elem(pr, S.p, S, i), R.Mp, R.Sp);
    if (R.mode == MODE_REJECT && R.useA) {
        const double q = exact_act<ACT>(P, row_elem(qr, S.q, S, i), R.Mq, R.Sq);
        const double d = p - q;
        return d > 0.0 ? d : 0.0;
    }
    return p;
}

// ---------------------------------------------------------------------------
// Granules: a warp reduces one 512-element granule of the needed row(s)
// (coalesced element loads; rows of odd length have arbitrary alignment) to
//   reject:  (sum max(0, p - q), sum p)          -- residual / fallback masses
//   bonus:   (max, sum e^(x - max)) [softmax]  or  (0, sum value)
// Split into load and reduce so a B-item can keep two granules' loads in flight.
template <typename T>
struct GranuleData {
    using A = typename Elem<T>::acc;
    static constexpr int EPL = kGW / 32;  // elements per lane per row (16)
    A xs[EPL], xq[EPL];
    int n;
};

// SM: sp / sq point at the granule's first element in shared memory (the
// cluster path's resident slices) instead of the rows in global memory.
template <typename T, bool SM = false>
__device__ __forceinline__ void granule_load(const StepParams& P, int b, int g, const Decision& d, GranuleData<T>& D,
                                             const T* sp = nullptr, const T* sq = nullptr) {
    using A = typename Elem<T>::acc;
    const int lane = threadIdx.x & 31;
    const int lo = g * kGW;
    D.n = g < P.NG ? min(kGW, P.V - lo) : 0;
    const bool reject = d.mode == MODE_REJECT;
    const T* pr = SM ? sp : p_row<T>(P, b, d.row) + lo;
    const T* qr = SM ? sq : (reject ? q_row<T>(P, b, d.row) + lo : pr);
    constexpr int EPL = GranuleData<T>::EPL;
    if constexpr (sizeof(T) == 2) {
        // bf16, full granule of 16-byte-aligned rows: each lane takes 16
        // consecutive elements with two 128-bit loads (the sums only need the
        // granule's set).  (fp32 keeps the coalesced scalar loads: with two
        // granules in flight the vector temporaries spill at 80 registers.)
        constexpr int NV = EPL * (int)sizeof(T) / 16;  // vectors per lane per row (4 fp32, 2 bf16)
        const bool vec = D.n == kGW && ((reinterpret_cast<uintptr_t>(pr) | reinterpret_cast<uintptr_t>(qr)) & 15) == 0;
        if (vec) {
            const uint4* vp = reinterpret_cast<const uint4*>(pr) + lane * NV;
            const uint4* vq = reinterpret_cast<const uint4*>(qr) + lane * NV;
            uint4 wp[NV], wq[NV];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                wp[k] = SM ? vp[k] : __ldg(vp + k);
                if (reject) wq[k] = SM ? vq[k] : __ldg(vq + k);
            }
            constexpr int VEC = Elem<T>::VEC;
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                A xp[VEC], xq[VEC];
                unpack(wp[k], xp);
                if (reject) unpack(wq[k], xq);
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    D.xs[k * VEC + e] = xp[e];
                    D.xq[k * VEC + e] = reject ? xq[e] : (A)0;
                }
            }
            return;
        }
    }
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
        const int e = t * 32 + lane;
        D.xs[t] = e < D.n ? (SM ? load_smem_elem(pr + e) : load_elem(pr + e)) : (A)0;
        D.xq[t] = (reject && e < D.n) ? (SM ? load_smem_elem(qr + e) : load_elem(qr + e)) : (A)0;
    }
}

template <typename T, int ACT>
__device__ __forceinline__ double2 granule_reduce(const StepParams& P, const Decision& d, const GranuleData<T>& D) {
    using A = typename Elem<T>::acc;
    constexpr int EPL = GranuleData<T>::EPL;
    const int lane = threadIdx.x & 31;
    const int n = D.n;
    const A alpha = (A)P.alpha, invw = (A)(1.0 / P.width);
    if (d.mode != MODE_REJECT) {
        if (ACT == ACT_SOFTMAX) {
            A mx = -INFINITY, mn = INFINITY;
#pragma unroll
            for (int t = 0; t < EPL; ++t)
                if (t * 32 + lane < n) {
                    mx = fmax(mx, D.xs[t]);
                    mn = fmin(mn, D.xs[t]);
                }
            mx = warp_max(mx);
            mn = warp_min(mn);
            A sm = 0;
#pragma unroll
            for (int t = 0; t < EPL; ++t)
                if (t * 32 + lane < n) sm += exp_rel(D.xs[t], mx);
            const double S = warp_sum((double)sm);
            if (n > 0 && lane == 0 && (!isfinite((double)mx) || isnan(S) || !isfinite((double)mn)))
                flag(P, SSV_STATUS_NONFINITE);
            return make_double2((double)mx, S);
        }
        if (ACT == ACT_SIGMOID_HALF) {  // binary16 emulation: the reference's values, fp64
            double sh = 0.0;
#pragma unroll
            for (int t = 0; t < EPL; ++t)  // (unrolled: D stays in registers)
                if (t * 32 + lane < n) sh += sigmoid_act<ACT>(P, (double)D.xs[t]);
            return make_double2(0.0, warp_sum(sh));
        }
        A sm = 0;
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
            if (t * 32 + lane < n) {
                if (is_sigmoid(ACT)) sm += sigmoid_fast((D.xs[t] - alpha) * invw);
                else sm += D.xs[t];
            }
        }
        return make_double2(0.0, warp_sum((double)sm));
    }
    if (ACT == ACT_SIGMOID_HALF) {
        double ta = 0.0, tp = 0.0;
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
            if (t * 32 + lane < n) {
                const double vp = sigmoid_act<ACT>(P, (double)D.xs[t]), vq = sigmoid_act<ACT>(P, (double)D.xq[t]);
                ta += vp - vq > 0.0 ? vp - vq : 0.0;
                tp += vp;
            }
        }
        return make_double2(warp_sum(ta), warp_sum(tp));
    }
    const A Mp = (A)d.Mp, Mq = (A)d.Mq, iSp = (A)(1.0 / d.Sp), iSq = (A)(1.0 / d.Sq);
    if constexpr (ACT == ACT_SOFTMAX && sizeof(A) == 4) {
        if (n == kGW) {  // full granule (warp-uniform): packed pairs, FADD2 / FMUL2 (the same roundings per term)
            const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
            const float2 nMp = make_float2(-Mp, -Mp), nMq = make_float2(-Mq, -Mq);
            const float2 sP = make_float2(iSp, iSp), sQ = make_float2(iSq, iSq);
            float2 ta2 = make_float2(0.f, 0.f), tp2 = make_float2(0.f, 0.f);  // 8 terms per chain
#pragma unroll
            for (int t = 0; t < EPL; t += 2) {
                const float2 ap = __fmul2_rn(__fadd2_rn(make_float2(D.xs[t], D.xs[t + 1]), nMp), l2e);
                const float2 aq = __fmul2_rn(__fadd2_rn(make_float2(D.xq[t], D.xq[t + 1]), nMq), l2e);
                const float2 vp = __fmul2_rn(make_float2(ex2f(ap.x), ex2f(ap.y)), sP);
                const float2 vq = __fmul2_rn(make_float2(ex2f(aq.x), ex2f(aq.y)), sQ);
                const float2 dv = __fadd2_rn(vp, make_float2(-vq.x, -vq.y));
                ta2 = __fadd2_rn(ta2, make_float2(dv.x > 0.f ? dv.x : 0.f, dv.y > 0.f ? dv.y : 0.f));
                tp2 = __fadd2_rn(tp2, vp);
            }
            return make_double2(warp_sum((double)ta2.x + (double)ta2.y), warp_sum((double)tp2.x + (double)tp2.y));
        }
    }
    A ta = 0, tp = 0;
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
        if (t * 32 + lane < n) {
            const A xp = D.xs[t], xqq = D.xq[t];
            A a, vp;
            if (ACT == ACT_SOFTMAX) {
                vp = exp_rel(xp, Mp) * iSp;
                const A vq = exp_rel(xqq, Mq) * iSq;
                a = vp - vq > (A)0 ? vp - vq : (A)0;
            } else if (is_sigmoid(ACT)) {
                // sigma(tp) - sigma(tq) = sigma(tp) sigma(-tq) (1 - e^-(tp-tq)): no cancellation.
                const A tp_ = (xp - alpha) * invw, tq_ = (xqq - alpha) * invw;
                const A dd = (xp - xqq) * invw;
                vp = sigmoid_fast(tp_);
                const A sqn = sigmoid_fast(-tq_);
                a = dd > (A)0 ? vp * sqn * (-expm1_acc(-dd)) : (A)0;
            } else {
                vp = xp;
                a = xp - xqq > (A)0 ? xp - xqq : (A)0;
            }
            ta += a;
            tp += vp;
        }
    }
    return make_double2(warp_sum((double)ta), warp_sum((double)tp));
}

template <typename T, int ACT>
__device__ void granule(const StepParams& P, int b, int g, const Decision& d, double2* gp) {
    GranuleData<T> D;
    granule_load<T>(P, b, g, d, D);
    const double2 out = granule_reduce<T, ACT>(P, d, D);
    if ((threadIdx.x & 31) == 0) *gp = out;
}

// ---------------------------------------------------------------------------
// Inverse CDF, element level (whole CTA): exact fp64 scan from granule gstar
// with the cumulative mass `carry` before it, continuing into later granules
// on rounding; no hit -> dist.cpp:135-136 (last index with positive mass,
// else 0), with gmass(g) the normalized mass of granule g.  Returns the token.
template <typename T, int ACT, int NT, typename GMass>
__device__ int locate_scan(const StepParams& P, const RowCtx& R, const T* pr, const T* qr, int gstar, double carry,
                           double u, const GMass& gmass, Shared& sh, bool tl, const RowSlice<T>& S = RowSlice<T>()) {
    const int NG = P.NG, GW = kGW;
    int token = -1;
    constexpr int E = (kGW + NT - 1) / NT;  // elements per thread (2 at 256 threads, 1 at 512)
    static_assert(E == 1 || E == 2, "level-2 scan takes one or two elements per thread");
    while (gstar >= 0 && gstar < NG) {
        const int lo = gstar * GW;
        const int hi = min(lo + GW, P.V);
        const int base = lo + threadIdx.x * E;
        double v0 = 0.0, v1 = 0.0;
        if (base < hi) v0 = exact_value<T, ACT>(P, R, pr, qr, base, S) / R.denom;
        if (E > 1 && base + 1 < hi) v1 = exact_value<T, ACT>(P, R, pr, qr, base + 1, S) / R.denom;
        const double ts = v0 + v1;
        if (tl) trace(P, 8 * P.B + 19);
        double tot;
        const double incl = block_scan_incl_n<NT / 32>(ts, sh.dred, tot);
        double cum = carry + (incl - ts);
        int h = 0x7fffffff;
        cum += v0;
        if (base < hi && u < cum) h = base;
        cum += v1;
        if (h == 0x7fffffff && E > 1 && base + 1 < hi && u < cum) h = base + 1;
        const int first = block_reduce_n<NT / 32>(h, sh.ired, OpMin());
        if (first != 0x7fffffff) {
            token = first;
            break;
        }
        carry += tot;
        ++gstar;
    }
    if (token < 0) {
        // dist.cpp:135-136: last index with positive mass, else 0.
        int glast = -1;
        for (int g = threadIdx.x; g < NG; g += NT)
            if (gmass(g) > 0.0) glast = max(glast, g);
        glast = block_reduce_n<NT / 32>(glast, sh.ired, OpMax());
        token = 0;
        if (glast >= 0) {
            int last = -1;
            for (int i = glast * GW + threadIdx.x; i < min((glast + 1) * GW, P.V); i += NT)
                if (exact_value<T, ACT>(P, R, pr, qr, i) > 0.0) last = max(last, i);
            last = block_reduce_n<NT / 32>(last, sh.ired, OpMax());
            if (last >= 0) token = last;
        }
    }
    return token;
}

// ---------------------------------------------------------------------------
// Inverse CDF of batch row b (whole CTA): granule partials -> SMEM -> fp64
// granule prefix (contiguous ownership, one scan) -> exact fp64 scan inside
// the selected granule (dist.cpp:122-137, incl. both fallbacks).
template <typename T, int ACT, int NT = kCtaThreads>
__device__ void locate(const StepParams& P, int b, const Decision& d, Shared& sh, double2* gcache, double u) {
    const int NG = P.NG;
    const double2* gp = P.gpart + (size_t)b * NG;
    const T* pr = p_row<T>(P, b, d.row);
    const T* qr = d.mode == MODE_REJECT ? q_row<T>(P, b, d.row) : nullptr;
    // u = u_final (verify_reference.cpp:98), loaded by the caller ahead of time
    if (P.trace && b == 0 && threadIdx.x == 0) trace(P, 8 * P.B + 21);
    // (the caller has cached granules [0, kLocCap) in gcache)
    const long long cyc0 = clock64();
    auto raw = [&](int g) -> double2 { return g < kLocCap ? gcache[g] : __ldcg(&gp[g]); };

    // Level 1 on warp 0 alone (no block barriers): the denominators, then the
    // fp64 granule prefix (verify_reference.cpp:51-62 / dist.cpp:122-137 at
    // granule resolution); lane 0 publishes.  Lane l takes granules l, l + 32,
    // ... (conflict-free shared-memory reads; a lane-contiguous layout made
    // every read an 8-way bank conflict and the search a serial chain: ~4700
    // cycles at NG = 297), one warp scan per 32-granule round in the search.
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int rounds = (NG + 31) / 32;
        bool useA = false;
        double denom = 1.0, gM = 0.0, gS = 1.0;
        auto wraw = [&](int g) -> double {  // unnormalized granule mass
            const double2 v = raw(g);
            if (d.mode == MODE_REJECT) return useA ? v.x : v.y;
            if (ACT == ACT_SOFTMAX) return v.y > 0.0 ? (g < kLocCap ? v.y : v.y * exp(v.x - gM)) : 0.0;
            return v.y;
        };
        if (d.mode == MODE_REJECT) {
            double a1 = 0.0, a2 = 0.0;
            for (int g = lane; g < NG; g += 32) {
                const double2 v = raw(g);
                a1 += v.x;
                a2 += v.y;
            }
            if (P.trace && b == 0 && lane == 0) P.trace[8 * P.B + 23] = (unsigned long long)(clock64() - cyc0);
            const double sa = warp_sum(a1), sp = warp_sum(a2);
            useA = sa > kZeroEps;  // verify_reference.cpp:57-62
            denom = useA ? sa : sp;
            if (lane == 0) {
                if (P.rsu) P.rsu[b] = 1;
                if (P.rden) P.rden[b] = useA ? sa : 0.0;
            }
        } else {
            double sm = 0.0;
            if (ACT == ACT_SOFTMAX) {  // the bonus row's statistics from its granules
                double m = -CUDART_INF;
                for (int g = lane; g < NG; g += 32) m = fmax(m, raw(g).x);
                gM = warp_max(m);
                for (int g = lane; g < NG; g += 32) {
                    const double2 v = raw(g);
                    const double w = v.y > 0.0 ? v.y * exp(v.x - gM) : 0.0;
                    sm += w;
                    // rebase the cached granule to the row max: (gM, w) is the same
                    // mass, and the search below needs no further exp
                    if (g < kLocCap) gcache[g] = make_double2(gM, w);
                }
                __syncwarp();
            } else {
                for (int g = lane; g < NG; g += 32) sm += raw(g).y;
            }
            const double tot = warp_sum(sm);
            if (ACT == ACT_SOFTMAX) gS = tot;
            else denom = tot;
            if (lane == 0) {
                if (P.rsu) P.rsu[b] = 0;
                if (P.rden) P.rden[b] = 0.0;
            }
        }
        if (P.trace && b == 0 && lane == 0) P.trace[8 * P.B + 24] = (unsigned long long)(clock64() - cyc0);
        const double norm = d.mode != MODE_REJECT && ACT == ACT_SOFTMAX ? gS : denom;
        const double thr = u * norm;
        int gst = -1;
        double car = 0.0, carry = 0.0;
        for (int j = 0; j < rounds; ++j) {  // first granule whose inclusive prefix passes u * norm
            const int g = lane + 32 * j;
            const double w = g < NG ? wraw(g) : 0.0;
            const double incl = warp_scan_incl(w);
            const unsigned hm = __ballot_sync(kFull, g < NG && thr < carry + incl);
            if (hm) {
                const int src = __ffs(hm) - 1;
                gst = 32 * j + src;
                car = (carry + __shfl_sync(kFull, incl - w, src)) / norm;
                break;
            }
            carry += __shfl_sync(kFull, incl, 31);
        }
        const unsigned hm = gst >= 0 ? 1u : 0u;
        if (lane == 0) {
            if (P.trace && b == 0) {
                P.trace[8 * P.B + 22] = (unsigned long long)(clock64() - cyc0);
            }
            sh.loc_g = hm ? gst : -1;
            sh.loc_useA = useA;
            sh.loc_d[0] = car;
            sh.loc_d[1] = denom;
            sh.loc_d[2] = gM;
            sh.loc_d[3] = gS;
        }
    }
    __syncthreads();
    RowCtx R;
    R.mode = d.mode;
    R.Mp = d.Mp;
    R.Sp = d.Sp;
    R.Mq = d.Mq;
    R.Sq = d.Sq;
    R.useA = sh.loc_useA;
    R.denom = sh.loc_d[1];
    const double gM = sh.loc_d[2], gS = sh.loc_d[3];
    if (d.mode != MODE_REJECT && ACT == ACT_SOFTMAX) {
        R.Mp = gM;
        R.Sp = gS;
        R.denom = 1.0;  // sample_row's sequential_sum of a softmax row (1 within rounding)
    }
    auto gmass = [&](int g) -> double {  // normalized granule mass (fallback path)
        const double2 v = raw(g);
        if (R.mode == MODE_REJECT) return (R.useA ? v.x : v.y) / R.denom;
        if (ACT == ACT_SOFTMAX) return v.y > 0.0 ? v.y * exp(v.x - gM) / gS : 0.0;
        return v.y / R.denom;
    };
    int gstar = sh.loc_g;
    double carry = sh.loc_d[0];
    const bool tl = P.trace && b == 0 && threadIdx.x == 0;  // locate stamps: trace[8B + 18 ..]
    if (tl) trace(P, 8 * P.B + 18);

    const int token = locate_scan<T, ACT, NT>(P, R, pr, qr, gstar, carry, u, gmass, sh, tl);
    if (tl) trace(P, 8 * P.B + 20);
    if (threadIdx.x == 0) P.fin[b] = token;
}

// The decision a B- or L-item works from: the D-item's (release flag), or,
// when sampling, the bonus row 0.
template <typename T, int ACT>
__device__ void get_decision(const StepParams& P, int b, bool write, Shared& sh) {
    const int tid = threadIdx.x;
    if (P.sample_mode) {
        if (tid == 0) {
            Decision d{};
            d.mode = MODE_BONUS;
            d.row = 0;
            d.Sp = d.Sq = 1.0;
            sh.dec = d;
        }
    } else {
        if (tid == 0) sh.dec = wait_decision(P, b);
    }
    (void)write;
    __syncthreads();
}

// Sigmoid / probability D-item: the decision from the gathered values alone
// (warp 0, paper section 3.2.2), published like the exact one.
template <typename T, int ACT>
__device__ void item_D_gather(const StepParams& P, int b, Shared& sh) {
    if (threadIdx.x >= 32) return;
    if (threadIdx.x == 0) trace(P, 8 * b);
    decide_gather<T, ACT>(P, b, true, sh.dec);
    __syncwarp();
    if (threadIdx.x == 0) {
        publish_decision(P, b, sh.dec);
        trace(P, 8 * b + 2);
    }
}

// B-item j of batch row b: granules kBG*8*j .. +kBG*8-1 of the needed row(s),
// kBG per warp with both granules' loads in flight; thread 0 publishes the
// partials, then counts the item (release).
template <typename T, int ACT>
__device__ void item_B(const StepParams& P, int b, int j, Shared& sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (j == 0 && tid == 0) trace(P, 8 * b + 3);
    const int g0 = j * kWarps * kBG;
    // Sigmoid / probabilities (no A phase): while the row's gathers-only
    // decision is pending, pull this item's slice of the bonus row into L2 --
    // the likely case (high acceptance); a rejection reads the pair instead.
    if (ACT != ACT_SOFTMAX && !P.sample_mode && P.PS == P.G + 1) {
        const size_t e0 = (size_t)g0 * kGW, e1 = min((size_t)P.V, e0 + (size_t)kWarps * kBG * kGW);
        const char* row = reinterpret_cast<const char*>(p_row<T>(P, b, P.G));
        const size_t lo = (e0 * sizeof(T)) & ~size_t(127), hi = e1 * sizeof(T);
        const size_t at = lo + (size_t)tid * 128;
        if (at < hi) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + at));
    }
    get_decision<T, ACT>(P, b, false, sh);
    if (j == 0 && tid == 0) trace(P, 8 * b + 4);
    const Decision d = sh.dec;
    // Each warp stores its granule partials straight into their slots (the
    // value is the completion flag; with no row left to sample the slots
    // still carry zeros, so the L-item knows every B-item has read the flag).
    double2* out = P.gpart + (size_t)b * P.NG;
    if (d.mode != MODE_NONE) {
        GranuleData<T> D[kBG];
#pragma unroll
        for (int k = 0; k < kBG; ++k) granule_load<T>(P, b, g0 + k * kWarps + warp, d, D[k]);
#pragma unroll
        for (int k = 0; k < kBG; ++k) {
            const double2 gp = granule_reduce<T, ACT>(P, d, D[k]);
            const int g = g0 + k * kWarps + warp;
            if (lane == 0 && g < P.NG) st_slot(&out[g], gp);
        }
    } else if (lane == 0) {
#pragma unroll
        for (int k = 0; k < kBG; ++k) {
            const int g = g0 + k * kWarps + warp;
            if (g < P.NG) st_slot(&out[g], make_double2(0.0, 0.0));
        }
    }
}

// L-item of batch row b: waits for the row's B-items, runs the inverse CDF,
// and leaves b's counters at zero for the next launch.
template <typename T, int ACT>
__device__ void item_L(const StepParams& P, int b, Shared& sh, double2* gcache) {
    const int tid = threadIdx.x;
    if (tid == 0) trace(P, 8 * b + 5);
    const double u = __ldcg(&P.u[(size_t)b * (P.G + 1) + P.G]);  // u_final, issued before the waits
    get_decision<T, ACT>(P, b, true, sh);
    const Decision d = sh.dec;
    // Wait for every granule slot of b (each B-item fills its own), caching
    // the first kLocCap for the locate.
    double2* gp = P.gpart + (size_t)b * P.NG;
    for (int g = tid; g < P.NG; g += kCtaThreads) {
        const double2 v = ld_slot_wait(&gp[g], kSlotEmpty);
        if (g < kLocCap) gcache[g] = v;
    }
    __syncthreads();
    if (tid == 0) trace(P, 8 * b + 6);
    if (d.mode != MODE_NONE) {
        locate<T, ACT>(P, b, d, sh, gcache, u);
        if (tid == 0) trace(P, 8 * b + 7);
    }
    __syncthreads();  // the locate has read the slots
    for (int g = tid; g < P.NG; g += kCtaThreads) clear_slot(&gp[g], kSlotEmpty);
    if (tid < 3) clear_slot(&P.dslot[3 * b + tid], kSlotEmpty);  // every B-item has read it (its slots are filled)
}

// ---------------------------------------------------------------------------
template <typename T, int ACT>
__global__ void __launch_bounds__(kCtaThreads, kCtaMinBlocks) k_verify(StepParams P) {
    __shared__ Shared sh;
    extern __shared__ __align__(128) uint4 dsm[];
    const int tid = threadIdx.x;
    pdl_enter();
    if (P.trace && blockIdx.x == 0 && tid == 0) trace(P, 8 * P.B);
    // Claims run two ahead: the item after the current one is known while the
    // current one runs (an A-run streams its first chunks early), and the
    // claim after that is in flight.
    // (With few items per CTA the claim-ahead would hand two items to half the
    // CTAs and none to the rest: then claim one at a time.)
    unsigned q1 = 0, q2 = 0;
    if (tid == 0) {
        q1 = atomicAdd(P.next, 1u);
        q2 = P.claim_ahead ? atomicAdd(P.next, 1u) : P.n_items;
    }
    AStream as;
    for (;;) {
        if (tid == 0) {
            sh.item = q1;
            sh.item_next = q2;
            if (P.claim_ahead) {
                q1 = q2;
                q2 = atomicAdd(P.next, 1u);
            } else {
                q1 = atomicAdd(P.next, 1u);
            }
        }
        __syncthreads();
        const unsigned i = sh.item, inext = sh.item_next;
        if (i >= P.n_items) break;
        const ItemRef it = decode_item(P, i);
        if (it.type == IT_B) {
            item_B<T, ACT>(P, it.b, it.idx, sh);
        } else if (it.type == IT_L) {
            item_L<T, ACT>(P, it.b, sh, reinterpret_cast<double2*>(dsm));
        } else if constexpr (ACT == ACT_SOFTMAX) {
            if (it.type == IT_A) {
                const ItemRef nx = inext < P.n_items ? decode_item(P, inext) : ItemRef{-1, 0, 0};
                item_A<T>(P, it.b, it.idx, nx, sh, dsm, as);
            } else {
                if (tid == 0) trace(P, 8 * it.b);
                item_D<T>(P, it.b, sh);
                if (tid == 0) trace(P, 8 * it.b + 2);
            }
        } else {
            item_D_gather<T, ACT>(P, it.b, sh);  // (the only other item type without an A phase)
        }
        __syncthreads();  // the item's shared state is dead before the next one
    }
    if (tid == 0) {
        if (P.trace) atomicMax(&P.trace[8 * P.B + 1], gtime());
        __threadfence();
        if (atomicAdd(P.exit_cnt, 1u) == gridDim.x - 1) {  // last CTA out resets the claim counter
            *P.exit_cnt = 0;
            *P.next = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// K1s k_verify_slab<T>: the slab path (exact variant, large batches; DESIGN.md
// 3.3).  One persistent CTA per SM, units assigned statically: CTA c takes
// units c, c + grid, c + 2 grid, ...  Unit u = (b, s) is slice s (kSlabVec
// 16-byte vectors: 512 fp32 / 1024 bf16 elements) of ALL 2*gamma drafted rows
// of batch row b, copied once into a shared-memory buffer and kept there until
// b's decision is known, so the rejected pair is never re-read from HBM.
// Step k of a CTA:
//   1. cp.async the unit of step k + Dp into its buffer (Dp units in flight);
//   2. statistics of step k: one warp per row slice -> (max, sum e^(x-max))
//      into its self-flagging partial slot; the CTA holding the LAST slice of
//      b then folds b's partials (item_D: fixed order, fp64), computes tau at
//      every position and the first rejection, and publishes the decision;
//   3. residual of step k - L (its buffer still resident): granule masses of
//      the rejected pair (from shared memory) or the bonus row (global), into
//      granule slots; the CTA that decided b runs b's inverse CDF (locate)
//      once all of b's granule slots are filled.
// Every wait is on work of an earlier step, or of the same step's earlier
// phase (statistics never wait), so with all CTAs co-resident (cooperative
// launch) the schedule cannot deadlock; L >= ceil((NS - 1) / grid) keeps a
// residual from waiting on a decision of a later step.
constexpr int kSlabVec = 128;                 // 16-byte vectors per row slice (2 KB)
constexpr int kSlabVPR = kSlabVec + 2;        // shared-memory vectors per row slice (aligned superset)
constexpr int kSlabRowBytes = kSlabVPR * 16;  // 2080 B
constexpr int kSlabGcache = kLocCap * (int)sizeof(double2);  // locate's granule cache (16 KB)

template <typename T>
struct SlabSlice {
    const uint4* a0;  // 16-byte-aligned start of the slice's superset
    int shift;        // elements of a0's first vector before the slice
    int len;          // elements in the slice
    int nvec;         // vectors of the superset
};

template <typename T>
__device__ __forceinline__ SlabSlice<T> slab_slice(const StepParams& P, int b, int r, int s) {
    constexpr int VEC = Elem<T>::VEC;
    constexpr int SE = kSlabVec * VEC;
    const T* row = r < P.G ? p_row<T>(P, b, r) : q_row<T>(P, b, r - P.G);
    const int e0 = s * SE;
    const uintptr_t g = reinterpret_cast<uintptr_t>(row + e0);
    SlabSlice<T> x;
    x.a0 = reinterpret_cast<const uint4*>(g & ~uintptr_t(15));
    x.shift = (int)((g & 15) / sizeof(T));
    x.len = min(SE, P.V - e0);
    x.nvec = (x.shift + x.len + VEC - 1) / VEC;
    return x;
}

// cp.async every drafted row slice of unit (b, s) into buffer `buf`: warp w
// copies rows w, w + 8, ... (slice geometry once per row, then one 16-byte
// copy per lane and vector).
template <typename T>
__device__ __forceinline__ void slab_issue(const StepParams& P, int b, int s, uint8_t* buf) {
    const int lane = threadIdx.x & 31;
    for (int r = threadIdx.x >> 5; r < 2 * P.G; r += kWarps) {
        const SlabSlice<T> x = slab_slice<T>(P, b, r, s);
        uint8_t* dst = buf + r * kSlabRowBytes;
#pragma unroll
        for (int t = 0; t < (kSlabVPR + 31) / 32; ++t) {
            const int j = lane + 32 * t;
            if (j < x.nvec) cp_async16(dst + j * 16, x.a0 + j);
        }
    }
}

// One warp: (R, sum e^(x - R)) of row slice x staged at `rowp`, R = ceil of
// the slice max.  fp32 pair sums of <= 8 terms widened to fp64,
// fp64 warp fold.
template <typename T>
__device__ __forceinline__ double2 slab_row_stats(const StepParams& P, const uint4* rowp, const SlabSlice<T>& x) {
    constexpr int VEC = Elem<T>::VEC;
    constexpr int NV = (kSlabVPR + 31) / 32;  // 5 vectors per lane (the 5th only on lanes 0, 1)
    constexpr int GRP = VEC == 4 ? 4 : 2;     // vectors per fp32 group: 8 terms per pair lane
    const int lane = threadIdx.x & 31;
    uint4 w[NV];
    float m = -FLT_MAX, mn = FLT_MAX;
#pragma unroll
    for (int t = 0; t < NV; ++t) {
        const int j = lane + 32 * t;
        w[t] = j < x.nvec ? rowp[j] : pad_vec<T>();
    }
    if (x.shift != 0 || x.len != kSlabVec * VEC) {  // misaligned or short slice: pad the edge vectors (warp-uniform)
#pragma unroll
        for (int t = 0; t < NV; ++t) {
            const int j = lane + 32 * t;
            if (j < x.nvec && (j == 0 || j == x.nvec - 1))
                mask_vec<T>(w[t], max(0, x.shift - j * VEC), min(VEC, x.shift + x.len - j * VEC));
        }
    }
#pragma unroll
    for (int t = 0; t < NV; ++t) AStat<T>::minmax(w[t], m, mn);
    m = ceilf(warp_max(m));  // integer reference >= the slice max (fold: e^(R_s - R) from kExpNeg)
    double S = 0.0;
    const float2 negM = make_float2(-m, -m);
#pragma unroll
    for (int t0 = 0; t0 < NV; t0 += GRP) {
        float2 a = make_float2(0.f, 0.f);
#pragma unroll
        for (int t = t0; t < t0 + GRP && t < NV; ++t) AStat<T>::expsum(w[t], negM, a);
        S += (double)a.x + (double)a.y;
    }
    S = warp_sum(S);
    if (__any_sync(kFull, !isfinite(mn)) && lane == 0) flag(P, SSV_STATUS_NONFINITE);  // -inf / NaN logit
    return make_double2((double)m, S);
}

// Raw loads of b's decision slots, issued a step before they are needed (the
// words are decoded -- and the load latency paid -- only at the next step).
struct DecRaw {
    unsigned long long w[6];
};
__device__ __forceinline__ void dec_issue(const StepParams& P, int b, DecRaw& r) {
    const double2* p = P.dslot + 3 * b;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.w[2 * i]), "=l"(r.w[2 * i + 1]) : "l"(p + i)
                     : "memory");
}
__device__ __forceinline__ bool dec_decode(const DecRaw& r, Decision& d) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 6; ++i) ok &= r.w[i] != kSlotEmpty;
    d.mode = (int)__longlong_as_double((long long)r.w[0]);
    d.row = (int)__longlong_as_double((long long)r.w[1]);
    d.Mp = __longlong_as_double((long long)r.w[2]);
    d.Sp = __longlong_as_double((long long)r.w[3]);
    d.Mq = __longlong_as_double((long long)r.w[4]);
    d.Sq = __longlong_as_double((long long)r.w[5]);
    return ok;
}

// Inverse CDF of batch row b once all of its granule slots are filled (slab
// and sigmoid-stream kernels); then b's granule and decision slots are left
// empty for the next launch.
template <typename T, int ACT>
__device__ void locate_row(const StepParams& P, int b, Shared& sh, double2* gcache) {
    const int tid = threadIdx.x, G = P.G;
    const double uf = __ldcg(&P.u[(size_t)b * (G + 1) + G]);
    DecRaw dr;
    if (tid == 0) dec_issue(P, b, dr);  // in flight with the granule slots below
    double2* gp = P.gpart + (size_t)b * P.NG;
    for (int g0 = 0; g0 < P.NG; g0 += 4 * kCtaThreads) {  // four slots per thread in flight
        double2 v[4];
        bool ok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int g = g0 + tid + i * kCtaThreads;
            ok[i] = g < P.NG ? ld_slot(&gp[g], v[i], kSlotEmpty) : true;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int g = g0 + tid + i * kCtaThreads;
            if (!ok[i]) v[i] = ld_slot_wait(&gp[g], kSlotEmpty);
            if (g < P.NG && g < kLocCap) gcache[g] = v[i];
        }
    }
    if (tid == 0) {
        Decision d;
        if (!dec_decode(dr, d)) d = wait_decision(P, b);
        sh.dec = d;
    }
    __syncthreads();
    const Decision d = sh.dec;
    if (tid == 0) trace(P, 8 * b + 6);
    if (d.mode != MODE_NONE) locate<T, ACT>(P, b, d, sh, gcache, uf);
    if (tid == 0) trace(P, 8 * b + 7);
    __syncthreads();
    for (int g = tid; g < P.NG; g += kCtaThreads) clear_slot(&gp[g], kSlotEmpty);
    if (tid < 3) clear_slot(&P.dslot[3 * b + tid], kSlotEmpty);
    __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(kCtaThreads, 1) k_verify_slab(StepParams P) {
    __shared__ Shared sh;
    extern __shared__ __align__(128) uint8_t slab_smem[];
    constexpr int VEC = Elem<T>::VEC;
    constexpr int SE = kSlabVec * VEC;
    constexpr int GPSL = SE / kGW;  // granules per slice (1 fp32, 2 bf16)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = P.G, NRd = 2 * G, NS = P.sl_ns, nbuf = P.sl_nbuf, Dp = P.sl_dp, L = P.sl_lag;
    double2* gcache = reinterpret_cast<double2*>(slab_smem + (size_t)nbuf * P.sl_ub);
    pdl_enter();
    const int NU = P.B * NS;
    const int grid = gridDim.x, c = blockIdx.x;
    const int nsteps = c < NU ? (NU - c + grid - 1) / grid : 0;
    auto bufp = [&](int slot) { return slab_smem + (size_t)slot * P.sl_ub; };
    if (P.trace && c == 0 && tid == 0) trace(P, 8 * P.B);
    // Unit of step k: u = c + k * grid = (b, s); tracked incrementally.
    auto unit_bs = [&](int k, int& b, int& s) {
        const int u = c + k * grid;
        b = u / NS;
        s = u - b * NS;
    };
    for (int k = 0; k < Dp; ++k) {
        if (k < nsteps) {
            int b, s;
            unit_bs(k, b, s);
            slab_issue<T>(P, b, s, bufp(k % nbuf));
        }
        cp_async_commit();
    }
    DecRaw pre;  // thread 0: the next residual step's decision words, in flight (issued at step k - 1)
    int slot_k = 0;                         // buffer of step k
    int slot_i = Dp % nbuf;                 // buffer of step k + Dp
    int slot_r = (nbuf - L % nbuf) % nbuf;  // buffer of step k - L
    for (int k = 0; k < nsteps + L; ++k) {
        if (k + Dp < nsteps) {
            int b, s;
            unit_bs(k + Dp, b, s);
            slab_issue<T>(P, b, s, bufp(slot_i));
        }
        cp_async_commit();  // (possibly empty: one group per step keeps the wait count fixed)
        if (k < nsteps) {
            int b, s;
            unit_bs(k, b, s);
            cp_async_wait_pending((unsigned)Dp);
            __syncthreads();  // unit k has landed (every thread's copies)
            const uint8_t* buf = bufp(slot_k);
            for (int r = warp; r < NRd && !(P.dbg & 2); r += kWarps) {
                const SlabSlice<T> x = slab_slice<T>(P, b, r, s);
                const double2 st = slab_row_stats<T>(P, reinterpret_cast<const uint4*>(buf + r * kSlabRowBytes), x);
                if (lane == 0) st_slot(&P.part[((size_t)b * NRd + r) * NS + s], st);
            }
            if (s == 0 && tid == 0) trace(P, 8 * b + 3);
            if (P.trace && tid == 0 && k < 6 && P.sl_dbg) P.trace[8 * P.B + 26 + c * 8 + k] = gtime();
            if (s == NS - 1 && !(P.dbg & 1)) {  // this CTA decides b (item_D waits for b's other partial slots)
                if (tid == 0) trace(P, 8 * b);
                item_D<T, true>(P, b, sh);
                if (tid == 0) trace(P, 8 * b + 2);
            }
        }
        if (k >= L && !(P.dbg & 1)) {
            const int kr = k - L;
            int b, s;
            unit_bs(kr, b, s);
            if (tid == 0) {
                Decision d;
                if (!dec_decode(pre, d)) d = wait_decision(P, b);
                sh.dec = d;
                if (s == 0) trace(P, 8 * b + 4);
            }
            __syncthreads();
            const Decision d = sh.dec;
            const uint8_t* buf = bufp(slot_r);
            const int e0 = s * SE;
            const int ng = min(GPSL, (P.V - e0 + kGW - 1) / kGW);
            if (warp < ng) {
                const int g = s * GPSL + warp;
                double2 out = make_double2(0.0, 0.0);
                if (d.mode == MODE_REJECT) {
                    const SlabSlice<T> xp = slab_slice<T>(P, b, d.row, s), xq = slab_slice<T>(P, b, G + d.row, s);
                    const T* sp = reinterpret_cast<const T*>(buf + d.row * kSlabRowBytes) + xp.shift + warp * kGW;
                    const T* sq = reinterpret_cast<const T*>(buf + (G + d.row) * kSlabRowBytes) + xq.shift + warp * kGW;
                    GranuleData<T> D;
                    granule_load<T, true>(P, b, g, d, D, sp, sq);
                    out = granule_reduce<T, ACT_SOFTMAX>(P, d, D);
                } else if (d.mode == MODE_BONUS) {
                    granule<T, ACT_SOFTMAX>(P, b, g, d, &out);
                }
                if (lane == 0) st_slot(&P.gpart[(size_t)b * P.NG + g], out);
            }
            if (s == 0 && tid == 0) trace(P, 8 * b + 5);
            if (P.trace && tid == 0 && kr < 2 && P.sl_dbg) P.trace[8 * P.B + 26 + c * 8 + 6 + kr] = gtime();
        }
        if (tid == 0 && k + 1 >= L && k + 1 - L < nsteps) dec_issue(P, (c + (k + 1 - L) * grid) / NS, pre);
        __syncthreads();  // buffer of step k - L is free; shared state dead
        slot_k = slot_k + 1 == nbuf ? 0 : slot_k + 1;
        slot_i = slot_i + 1 == nbuf ? 0 : slot_i + 1;
        slot_r = slot_r + 1 == nbuf ? 0 : slot_r + 1;
    }
    // Inverse CDFs, spread over the CTAs once every residual is in.
    for (int b = c; b < P.B && !(P.dbg & 1); b += grid) locate_row<T, ACT_SOFTMAX>(P, b, sh, gcache);
    if (P.trace && tid == 0) atomicMax(&P.trace[8 * P.B + 1], gtime());
}


// ---------------------------------------------------------------------------
// K2s k_verify_sig<T>: the sigmoid variant for batches the cluster path cannot
// hold.  The paper's approximation needs no row statistics
// (section 3.2.2), so one launch streams each batch row's needed row once:
//   1. every warp decides its batch rows from the gathered logits alone
//      (decide_gather: tau in fp64, first rejection) and publishes the
//      decision slots -- while the first tiles already stream in;
//   2. persistent CTAs take tiles (b, j) = elements [j*TE, (j+1)*TE) in a
//      static round-robin; the bonus row's tile (the likely case: sigmoid
//      acceptance is ~1 at the bench bounds) is copied into a shared-memory
//      ring nbuf - 1 tiles ahead by cp.async, independent of the decision; a
//      rejected row reads its pair from global instead.  Each warp reduces
//      512-element granules (MUFU ex2 + rcp sigmoid, fp32 lanes, fp64 warp
//      sum) into the granule slots;
//   3. once every tile is in, CTA c runs the inverse CDF of rows c, c + grid,
//      ... (locate: fp64 granule prefix, exact fp64 element scan).
// One TMA bulk copy (cp.async.bulk, completion on the slot's mbarrier) of the
// 16-byte-aligned superset of tile j of b's bonus row; thread 0 only.
template <typename T>
__device__ __forceinline__ void sig_issue(const StepParams& P, int b, int j, uint8_t* buf, uint64_t* bar) {
    constexpr int VEC = Elem<T>::VEC;
    const int TE = P.sg_te;
    const T* row = p_row<T>(P, b, P.G) + (size_t)j * TE;
    const uintptr_t g = reinterpret_cast<uintptr_t>(row);
    const int shift = (int)((g & 15) / sizeof(T));
    const int len = min(TE, P.V - j * TE);
    const uint32_t bytes = (uint32_t)((shift + len + VEC - 1) / VEC) * 16u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's previous reads came first
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(buf, reinterpret_cast<const void*>(g & ~uintptr_t(15)), bytes, bar);
}

// Bonus-row granules of tile j (staged in shared memory at element offset
// `shift`): warp w reduces granules w, w + 8, ...  Per element one FFMA for
// -(z - alpha) / width * log2(e), MUFU ex2, one add, MUFU rcp, one add (fp32
// lanes of 16 terms), then an fp64 warp sum -- the two granules' chains
// interleaved.  Aligned full granules read 128-bit vectors.
template <typename T, int ACT>
__device__ __forceinline__ void sig_bonus_granules(const StepParams& P, int b, int j, const T* tb, int shift) {
    constexpr int VEC = Elem<T>::VEC;
    constexpr int NVL = kGW / VEC / 32;  // 16-byte vectors per lane per granule (4 fp32, 2 bf16)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int GPT = P.sg_te / kGW;
    const float sc = (float)(-1.4426950408889634 / P.width);
    const float off = (float)(P.alpha * 1.4426950408889634 / P.width);
    for (int t0 = warp; t0 < GPT; t0 += 2 * kWarps) {
        double acc[2] = {0.0, 0.0};  // lane partials (fp32 chains of 16 terms)
        int gg[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = t0 + h * kWarps;
            const int g = j * GPT + t;
            gg[h] = t < GPT && g < P.NG ? g : -1;
            if (gg[h] < 0) continue;
            const int n = min(kGW, P.V - g * kGW);
            const T* base = tb + shift + t * kGW;
            if (ACT == ACT_SIGMOID && shift == 0 && n == kGW) {
                const uint4* v = reinterpret_cast<const uint4*>(base) + lane;
                float a = 0.f;
#pragma unroll
                for (int i = 0; i < NVL; ++i) {
                    float x[VEC];
                    unpack(v[32 * i], x);
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        const float ex = ex2f(fmaf(x[e], sc, off));
                        float r;
                        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + ex));
                        a += r;
                    }
                }
                acc[h] = a;
            } else {  // misaligned / short granule: the generic path (already warp-summed)
                GranuleData<T> D;
                Decision d{};
                d.mode = MODE_BONUS;
                granule_load<T, true>(P, b, g, d, D, base, base);
                const double gs = granule_reduce<T, ACT>(P, d, D).y;
                acc[h] = lane == 0 ? gs : 0.0;
            }
        }
        double s0 = acc[0], s1 = acc[1];  // fixed-order fp64 warp sums, both chains interleaved
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(kFull, s0, o);
            s1 += __shfl_xor_sync(kFull, s1, o);
        }
        if (lane == 0) {
            if (gg[0] >= 0) st_slot(&P.gpart[(size_t)b * P.NG + gg[0]], make_double2(0.0, s0));
            if (gg[1] >= 0) st_slot(&P.gpart[(size_t)b * P.NG + gg[1]], make_double2(0.0, s1));
        }
    }
}

template <typename T, int ACT>
__global__ void __launch_bounds__(kCtaThreads, 2) k_verify_sig(StepParams P) {
    __shared__ Shared sh;
    extern __shared__ __align__(128) uint8_t sig_smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int TE = P.sg_te, GPT = TE / kGW, NT = P.sg_nt, nbuf = P.sg_nbuf;
    pdl_enter();
    const int grid = gridDim.x, c = blockIdx.x;
    const int NU = P.B * NT;
    const int nsteps = c < NU ? (NU - c + grid - 1) / grid : 0;
    const bool spec = P.PS == P.G + 1;  // a bonus row exists: stream it speculatively
    auto bufp = [&](int slot) { return sig_smem + (size_t)slot * P.sg_tb; };
    uint64_t* bars = reinterpret_cast<uint64_t*>(sig_smem + (size_t)nbuf * P.sg_tb);  // one mbarrier per slot
    double2* gcache = reinterpret_cast<double2*>(sig_smem + (size_t)nbuf * P.sg_tb + 64);  // locate's granule cache
    if (P.trace && c == 0 && tid == 0) trace(P, 8 * P.B);
    if (tid == 0) {
        for (int i = 0; i < nbuf; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // 1. decisions from the gathers (warp per batch row), before the tile
    // stream starts: the two dependent round trips (ids, then logits) see an
    // idle memory system.
    for (int b = c * kWarps + warp; b < P.B; b += grid * kWarps) {
        Decision d;
        decide_gather<T, ACT>(P, b, true, d);
        __syncwarp();
        if (lane == 0) {
            publish_decision(P, b, d);
            trace(P, 8 * b + 2);
        }
    }
    if (tid == 0) {
        for (int k = 0; k < nbuf - 1 && spec && k < nsteps; ++k) {
            const int u = c + k * grid, b = u / NT;
            sig_issue<T>(P, b, u - b * NT, bufp(k), &bars[k]);
        }
    }
    __syncthreads();  // barriers initialized
    // 2. tiles.  Thread 0 keeps the decision words of the next kDecAhead
    // tiles in flight (a loaded L2 round trip is ~2 us, a tile ~0.7 us).
    constexpr int kDecAhead = 4;
    DecRaw pre[kDecAhead];
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < kDecAhead; ++i)
            if (i < nsteps) dec_issue(P, (c + i * grid) / NT, pre[i]);
    }
    // One CTA barrier per tile: it publishes the tile's decision (double-
    // buffered, so thread 0 may run one tile ahead) and proves every warp is
    // done with the slot tile k - 1 used, which thread 0 then refills.
    __shared__ Decision sdec[2];
    int slot_k = 0, slot_i = (nbuf - 1) % nbuf;
    for (int k = 0; k < nsteps; ++k) {
        const int u = c + k * grid, b = u / NT, j = u - b * NT;
        if (tid == 0) {
            Decision d;
            if (!dec_decode(pre[0], d)) d = wait_decision(P, b);
            sdec[k & 1] = d;
#pragma unroll
            for (int i = 0; i + 1 < kDecAhead; ++i) pre[i] = pre[i + 1];
            if (k + kDecAhead < nsteps) dec_issue(P, (u + kDecAhead * grid) / NT, pre[kDecAhead - 1]);
        }
        __syncthreads();  // decision of tile k published; tile k - 1's slot is free
        if (tid == 0 && spec && k + nbuf - 1 < nsteps) {
            const int ui = c + (k + nbuf - 1) * grid, bi = ui / NT;
            sig_issue<T>(P, bi, ui - bi * NT, bufp(slot_i), &bars[slot_i]);
        }
        const Decision d = sdec[k & 1];
        if (spec) mbar_wait(&bars[slot_k], (uint32_t)((k / nbuf) & 1));  // tile k has landed
        const T* tb = reinterpret_cast<const T*>(bufp(slot_k));
        const int shift = (int)((reinterpret_cast<uintptr_t>(p_row<T>(P, b, P.G) + (size_t)j * TE) & 15) / sizeof(T));
        if (d.mode == MODE_BONUS) {
            sig_bonus_granules<T, ACT>(P, b, j, tb, shift);
        } else {
            for (int t = warp; t < GPT; t += kWarps) {
                const int g = j * GPT + t;
                if (g >= P.NG) break;
                double2 out = make_double2(0.0, 0.0);
                if (d.mode == MODE_REJECT) granule<T, ACT>(P, b, g, d, &out);
                if (lane == 0) st_slot(&P.gpart[(size_t)b * P.NG + g], out);
            }
        }
        if (j == 0 && tid == 0) trace(P, 8 * b + 3);
        slot_k = slot_k + 1 == nbuf ? 0 : slot_k + 1;
        slot_i = slot_i + 1 == nbuf ? 0 : slot_i + 1;
    }
    __syncthreads();  // every warp's tiles are done
    // 3. inverse CDFs once every tile is in (a locate inside the stream stalls
    // its CTA for ~4 us of dependent round trips, and a locate waiting on a CTA
    // busy with its own chains the stalls: measured slower either way).
    for (int b = c; b < P.B; b += grid) locate_row<T, ACT>(P, b, sh, gcache);
    if (P.trace && tid == 0) atomicMax(&P.trace[8 * P.B + 1], gtime());
}

// K2w k_verify_sigw<T>: the sigmoid-stream kernel for 16-byte-aligned rows
// (every row start and V * sizeof(T) a multiple of 16 -- C4), with no CTA
// barrier in the stream: every warp owns whole units of the bonus row (256
// 16-byte vectors = 2 fp32 / 4 bf16 granules), every thread cp.asyncs and later
// reads only its own vectors through a kSigWStages-deep ring (the A-item
// scheme), and lane 0 of each warp polls the decisions of its
// next units.  Decisions first and the inverse CDFs last, as k_verify_sig.
// Warp reduce-scatter of GU (2 or 4) per-lane partials: the first log2(GU)
// butterfly levels exchange only the half each lane does not keep, so lane l
// ends with the warp sum of value l / (32 / GU) after 5 (GU = 2) or 6 (GU = 4)
// shuffles instead of 5 GU.
template <int GU>
__device__ __forceinline__ double warp_reduce_scatter(const double (&acc)[GU], int lane) {
    static_assert(GU == 2 || GU == 4, "two or four values per lane");
    double keep;
    if constexpr (GU == 2) {
        const bool up = lane & 16;
        keep = (up ? acc[1] : acc[0]) + __shfl_xor_sync(kFull, up ? acc[0] : acc[1], 16);
    } else {
        const bool up = lane & 16;
        const double k0 = (up ? acc[2] : acc[0]) + __shfl_xor_sync(kFull, up ? acc[0] : acc[2], 16);
        const double k1 = (up ? acc[3] : acc[1]) + __shfl_xor_sync(kFull, up ? acc[1] : acc[3], 16);
        const bool up8 = lane & 8;
        keep = (up8 ? k1 : k0) + __shfl_xor_sync(kFull, up8 ? k0 : k1, 8);
    }
#pragma unroll
    for (int o = 32 / GU / 2; o > 0; o >>= 1) keep += __shfl_xor_sync(kFull, keep, o);
    return keep;
}

constexpr int kSigWNJ = 8;      // vectors per lane per unit
constexpr int kSigWStages = 3;  // ring depth (2 units in flight per warp)
constexpr int kSigWUnitVec = 32 * kSigWNJ;

template <typename T, int ACT>
__global__ void __launch_bounds__(kCtaThreads, 2) k_verify_sigw(StepParams P) {
    __shared__ Shared sh;
    extern __shared__ __align__(128) uint8_t sigw_smem[];
    constexpr int VEC = Elem<T>::VEC;
    constexpr int EU = kSigWUnitVec * VEC;  // elements per unit (1024 fp32, 2048 bf16)
    constexpr int GU = EU / kGW;            // granules per unit (2, 4)
    constexpr int JPG = kSigWNJ / GU;       // lane vectors per granule (4, 2)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_enter();
    const int grid = gridDim.x, c = blockIdx.x;
    const int NTW = (P.V + EU - 1) / EU;   // units per row
    const int NU = P.B * NTW;
    const int nwarps = grid * kWarps, gw = c * kWarps + warp;
    // Each warp takes a contiguous range of units (one or two rows): the
    // decision changes only at a row boundary, and no division per unit.
    // A warp that computes a decision first (phase 1: row b on warp (b / grid)
    // % 8 of CTA b % grid) starts streaming ~5 us late, so its range is
    // shorter: weight sg_dw / 16 against 16 / 16 (the deciding warps had been
    // the last to finish at C4).  pos(w) = weighted warps before warp w.
    // CTA c decides on min(8, ceil((B - c) / grid)) warps: with B = q grid + r,
    // min(8, q + 1) for c < r and min(8, q) after (closed form, no loop).
    const int dq = P.B / grid, dr = P.B - dq * grid, dhi = min(kWarps, dq + 1), dlo = min(kWarps, dq);
    auto ndec_before = [&](int w) -> long {  // deciding warps among warps [0, w)
        const int cw = w / kWarps, ww = w - cw * kWarps;
        return (long)min(cw, dr) * dhi + (long)max(0, cw - dr) * dlo + min(ww, cw < dr ? dhi : dlo);
    };
    const int dw = P.sg_dw;
    auto pos = [&](int w) -> long { return 16L * w - (16 - dw) * ndec_before(w); };
    const long tot = pos(nwarps);
    const int u0 = (int)(pos(gw) * NU / tot), u1 = (int)(pos(gw + 1) * NU / tot);
    const int nsteps = u1 - u0;
    const int nvec_row = (P.V + VEC - 1) / VEC;
    uint4* ring = reinterpret_cast<uint4*>(sigw_smem);  // [stage][j][thread]
    double2* gcache = reinterpret_cast<double2*>(sigw_smem + (size_t)kSigWStages * kSigWNJ * kCtaThreads * 16);
    if (P.trace && c == 0 && tid == 0) trace(P, 8 * P.B);
    const bool spec = P.PS == P.G + 1;  // a bonus row exists: stream it speculatively
    int ib = u0 / NTW, ij = u0 - ib * NTW;  // unit of the next issue
    int cur_b = -1, cur_mode = MODE_NONE, cur_row = 0;  // the consumed row's decision, once known
    auto issue = [&](int stage) {
        if (ib == cur_b && cur_mode == MODE_REJECT) {
            // a rejected row: no bonus tile (its pair is reduced in the reject phase)
        } else if (spec && ib < P.B && ib * NTW + ij < u1) {
            const uint4* rowv = reinterpret_cast<const uint4*>(p_row<T>(P, ib, P.G)) + ij * kSigWUnitVec + lane;
            uint4* dst = ring + (size_t)stage * kSigWNJ * kCtaThreads + tid;
            const int nv = nvec_row - ij * kSigWUnitVec - lane;  // vectors left in the row from this lane's first
#pragma unroll
            for (int j = 0; j < kSigWNJ; ++j)
                if (j * 32 < nv) cp_async16(dst + j * kCtaThreads, rowv + j * 32);
        }
        cp_async_commit();
        if (++ij == NTW) {
            ij = 0;
            ++ib;
        }
    };
    // 1. decisions from the gathers: row b on warp (b / grid) % 8 of CTA b % grid,
    // so most CTAs lose one warp for ~4 us instead of a few CTAs all eight
    for (int b = c + grid * warp; b < P.B; b += grid * kWarps) {
        Decision d;
        decide_gather<T, ACT>(P, b, true, d);
        __syncwarp();
        if (lane == 0) {
            publish_decision(P, b, d);
            if (d.mode == MODE_REJECT) P.rej_list[atomicAdd(P.rej_cnt, 1u)] = b;
            __threadfence();  // the list entry before the count
            atomicAdd(P.dec_cnt, 1u);
            trace(P, 8 * b + 2);
        }
    }
    for (int k = 0; k < kSigWStages - 1; ++k) issue(k);
    int b = u0 / NTW, jw = u0 - b * NTW;
    DecRaw pre;
    if (lane == 0 && nsteps > 0) dec_issue(P, b, pre);
    int mode = 0, row = 0;
    const float sc = (float)(-1.4426950408889634 / P.width);
    const float off = (float)(P.alpha * 1.4426950408889634 / P.width);
    int stage = 0;
    for (int k = 0; k < nsteps; ++k) {
        if (k == 0 || jw == 0) {  // a new row: its decision (the next row's words go in flight)
            if (lane == 0) {
                Decision dd;
                if (!dec_decode(pre, dd)) dd = wait_decision(P, b);
                mode = dd.mode;
                row = dd.row;
                if (b + 1 < P.B && (b + 1) * NTW < u1) dec_issue(P, b + 1, pre);
            }
            mode = __shfl_sync(kFull, mode, 0);
            row = __shfl_sync(kFull, row, 0);
            cur_b = b;
            cur_mode = mode;
            cur_row = row;
        }
        issue((stage + kSigWStages - 1) % kSigWStages);
        cp_async_wait<kSigWStages - 1>();  // this thread's vectors of unit k have landed
        const int g0 = jw * GU;
        double2* out = P.gpart + (size_t)b * P.NG;
        if (mode == MODE_BONUS) {
            const int nv = nvec_row - jw * kSigWUnitVec - lane;
            const uint4* src = ring + (size_t)stage * kSigWNJ * kCtaThreads + tid;
            double acc[GU];
#pragma unroll
            for (int h = 0; h < GU; ++h) {
                float a = 0.f;
#pragma unroll
                for (int jj = 0; jj < JPG; ++jj) {
                    const int j = h * JPG + jj;
                    if (j * 32 < nv) {  // (rows are whole vectors: no element mask)
                        float x[VEC];
                        unpack(src[j * kCtaThreads], x);
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            const float ex = ex2f(fmaf(x[e], sc, off));
                            float r;
                            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + ex));
                            a += r;
                        }
                    }
                }
                acc[h] = a;
            }
            // reduce-scatter: lane l ends with granule l / (32 / GU)'s sum (half the shuffles)
            const double gs = warp_reduce_scatter<GU>(acc, lane);
            const int hh = lane / (32 / GU);
            if (lane % (32 / GU) == 0 && g0 + hh < P.NG) st_slot(&out[g0 + hh], make_double2(0.0, gs));
        } else if (mode == MODE_NONE) {  // nothing to sample: the slots only flag completion
            if (lane == 0) {
#pragma unroll
                for (int h = 0; h < GU; ++h)
                    if (g0 + h < P.NG) st_slot(&out[g0 + h], make_double2(0.0, 0.0));
            }
        }  // MODE_REJECT: the reject phase below
        if (jw == 0 && lane == 0) trace(P, 8 * b + 3);
        stage = stage + 1 == kSigWStages ? 0 : stage + 1;
        if (++jw == NTW) {
            jw = 0;
            ++b;
        }
    }
    cp_async_wait<0>();
    if (P.trace && P.sl_dbg && lane == 0) P.trace[8 * P.B + 26 + gw] = gtime();  // experiment: warp loop end
    // 3. rejected rows (rare at the sigmoid's acceptance): their pair granules,
    // spread over every warp of the grid once all decisions are in, two
    // granules' loads in flight per warp (a rejected row reduced only by the
    // warps that own its units made them stragglers: +15 us at B=256 V=32000).
    if (tid == 0) {
        while (ld_acquire(P.dec_cnt) < (unsigned)P.B) __nanosleep(64);
        sh.last = (int)ld_acquire(P.rej_cnt);
    }
    __syncthreads();
    const int R = sh.last;
    for (int i = gw; i < R * NTW; i += nwarps) {
        const int rb = __ldcg(&P.rej_list[i / NTW]), jr = i % NTW, g0 = jr * GU;
        Decision d{};
        d.mode = MODE_REJECT;
        int rr = 0;
        if (lane == 0) rr = wait_decision(P, rb).row;
        d.row = __shfl_sync(kFull, rr, 0);
        d.Sp = d.Sq = 1.0;
        double2* out = P.gpart + (size_t)rb * P.NG;
        for (int h = 0; h < GU; h += 2) {
            GranuleData<T> D[2];
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (g0 + h + q < P.NG) granule_load<T>(P, rb, g0 + h + q, d, D[q]);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (g0 + h + q >= P.NG) break;
                const double2 gv = granule_reduce<T, ACT>(P, d, D[q]);
                if (lane == 0) st_slot(&out[g0 + h + q], gv);
            }
        }
    }
    __syncthreads();
    for (int b = grid - 1 - c; b < P.B; b += grid) locate_row<T, ACT>(P, b, sh, gcache);
    if (tid == 0) {
        if (P.trace) atomicMax(&P.trace[8 * P.B + 1], gtime());
        __threadfence();
        if (atomicAdd(P.exit_cnt, 1u) == gridDim.x - 1) {  // the last CTA out resets the counters
            *P.rej_cnt = 0;
            *P.dec_cnt = 0;
            *P.exit_cnt = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// K1c/K2c k_verify_cluster<T, ACT>: the cluster path.  One
// thread-block cluster of cl_size (16 down to 4) CTAs per batch row; rank k
// owns the element slice [k*SE, (k+1)*SE) of every row.  Two plans
// (plan_cluster_t): resident -- one CTA per SM holding every drafted row
// slice (small B); ring -- two CTAs per SM streaming the slices (in pieces of
// >= 12 KB) through cl_slots shared-memory slots.
//   1. exact: one TMA bulk copy per drafted p / q row slice (or piece) stages
//      it in a slot, while all threads gather the drafted logits and the
//      uniforms; one warp per row folds the slice to (max, sum e^(x - max)) as
//      it lands (FMNMX3; four fp32 sum chains, fp64 in the folds) and restages
//      the slot it consumed with a later unit; the slice partials are pushed
//      into every rank's shared memory;
//   2. cluster barrier; every CTA folds the cl_size slice partials of every row
//      in the same fixed order, so all ranks reach the identical decision (tau
//      in fp64, first rejection) without another exchange; sigmoid /
//      probabilities: the decision comes from the gathers alone;
//   3. each rank reduces its slice of the rejected pair (from shared memory
//      when resident, else L2-hot) / bonus row (bulk-prefetched into L2) to
//      512-element granule masses and pushes its slice total into every
//      rank's shared memory (DSMEM stores);
//   4. cluster barrier; every rank combines the totals in the same order, and
//      the rank whose slice holds u * denominator runs the inverse CDF over its
//      own granules and elements (no DSMEM access after the barrier).
// Cluster CTAs: 8 warps, or 16 when one CTA per SM keeps every row slice
// resident and the rows outnumber 8 warps (one warp per row: no second round
// of row folds on the critical path; plan_cluster_t).
constexpr int kClThreads = 256;
// Rows x cluster ranks up to which every rank pushes its slice partials into
// every rank's shared memory before the barrier (the fold after it then reads
// only local shared memory); beyond it the fold reads the owners' partials
// through DSMEM.
constexpr int kClPushMax = 256;

template <typename T, int ACT, int NT = kClThreads>
__global__ void __launch_bounds__(NT, 1) k_verify_cluster(StepParams P) {
    constexpr int kClWarps = NT / 32;
    namespace cg = cooperative_groups;
    constexpr int VEC = Elem<T>::VEC;
    constexpr bool EXACT = ACT == ACT_SOFTMAX;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ Shared sh;
    extern __shared__ __align__(128) uint8_t csm[];
    pdl_enter();
    const int CS = P.cl_size, SE = P.cl_se, GPS = P.cl_gps, RB = P.cl_rowbytes;
    const int rank = (int)cl.block_rank();
    const int b = blockIdx.x / CS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = P.G, V = P.V;
    const int e0 = min(V, rank * SE), n = min(V, e0 + SE) - e0;  // this rank's slice
    const int NRc = EXACT ? P.cl_rows : 0;
    const int NS = EXACT ? P.cl_slots : 1;  // ring slots (NS == NRc: every row resident at once)
    // Ring units: each row slice in H pieces of PE elements (H == 1: whole slices)
    const int H = EXACT ? P.cl_pieces : 1, PE = H > 1 ? P.cl_pe : SE, NU = NRc * H;
    const bool whole = H == 1;
    // shared-memory carve-up (host: cluster_smem)
    uint8_t* slots = csm;                                                       // NS x RB
    const int NSp = (NS + 1) & ~1;
    uint64_t* full = reinterpret_cast<uint64_t*>(slots + (size_t)NS * RB);      // NS (even-padded)
    const int PM = NRc * CS <= kClPushMax ? CS : 1;                             // pushed partials per row
    double2* part = reinterpret_cast<double2*>(full + NSp);                     // [NRc][PM] slice partials
    double2* gloc = part + NRc * PM;                                            // [GPS] granule partials (DSMEM)
    double2* rtot = gloc + GPS;                                                 // [16] slice totals (pushed by the ranks)
    double* zg = reinterpret_cast<double*>(rtot + 16);                          // [3G + 1] gathers, uniforms
    int* offs = reinterpret_cast<int*>(zg + 3 * G + 1);                         // [NS]
    int* fills = offs + NS;                                                     // [NS] fills issued per slot - 1

    // Every rank pushes its slice partials (exact) or its slice totals (every
    // variant) into the other ranks' shared memory before the first full
    // cluster barrier, which needs every CTA of the cluster to have started:
    // arrive now, wait just before the first push (exact: the row folds;
    // sigmoid / probabilities: the granule pass).
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    const bool tr = P.trace && rank == 0 && tid == 0;  // per-row stamps (tools/trace_step.py)
    if (tr) {
        trace(P, 8 * b);
        if (b == 0) trace(P, 8 * P.B);
    }
    auto piece_n = [&](int h) { return max(0, min(n, (h + 1) * PE) - h * PE); };  // elements of piece h
    auto stage_row = [&](int u) {  // one thread: bulk-copy the 16-byte superset of unit u (row u / H, piece u % H) into slot u % NS
        const int sl = u % NS, r = u / H, h = u % H;
        const T* row = r < G ? p_row<T>(P, b, r) : (r < 2 * G ? q_row<T>(P, b, r - G) : p_row<T>(P, b, G));
        const int pn = piece_n(h);
        if (pn == 0) {  // nothing of this piece in the slice: complete the phase without a copy
            offs[sl] = 0;
            mbar_arrive(&full[sl]);
            return;
        }
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(row + e0 + h * PE), a1 = a0 + (uintptr_t)pn * sizeof(T);
        const uintptr_t s0 = a0 & ~uintptr_t(15), s1 = (a1 + 15) & ~uintptr_t(15);
        offs[sl] = (int)((a0 - s0) / sizeof(T));
        mbar_arrive_expect_tx(&full[sl], (uint32_t)(s1 - s0));
        bulk_g2s(slots + (size_t)sl * RB, reinterpret_cast<const void*>(s0), (uint32_t)(s1 - s0), &full[sl]);
    };
    // This rank's slice of the bonus row (16-byte superset), pulled into L2
    // ahead of a possible bonus sample: the sigmoid / probabilities decision
    // needs only the gathers (likely bonus); exact waits until its slices have
    // landed (resident plan only -- a ring still streams) so the prefetch does
    // not compete with them.
    auto prefetch_bonus = [&]() {
        const T* row = p_row<T>(P, b, G);
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(row + e0), a1 = reinterpret_cast<uintptr_t>(row + e0 + n);
        const uintptr_t s0 = a0 & ~uintptr_t(15), s1 = (a1 + 15) & ~uintptr_t(15);
        bulk_prefetch_l2(reinterpret_cast<const void*>(s0), (uint32_t)(s1 - s0));
    };
    const bool want_bonus_pf = P.PS == G + 1 && n > 0 && !(P.dbg & 4) &&
                               (EXACT ? (whole && NS == NRc && NRc == 2 * G) : true);
    if (!EXACT && want_bonus_pf && tid == 0) prefetch_bonus();
    const bool tx = tr && b == 0;  // finer stamps for batch row 0: trace[8B + 2 + k]
    if (EXACT && warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < NS; ++i) {
                mbar_init(&full[i], 1);
                fills[i] = 0;
            }
            mbar_fence_init();
        }
        __syncwarp();
        // first fills, one row per lane: a bulk-copy issue costs ~250 cycles, so
        // one thread issuing them all delays the last one by ~1 us
        if (n > 0)
            for (int u = lane; u < NS; u += 32) stage_row(u);
    }
    if (tx) trace(P, 8 * P.B + 2);
    // gathers and uniforms (needed by every rank for the decision)
    for (int c = tid; c < G; c += NT) {
        int x = P.ids[(size_t)b * G + c];
        if (x < 0 || x >= V) {
            if (rank == 0) flag(P, SSV_STATUS_TOKEN_RANGE);
            x = x < 0 ? 0 : V - 1;
        }
        zg[c] = load_exact(p_row<T>(P, b, c) + x);
        zg[G + c] = load_exact(q_row<T>(P, b, c) + x);
    }
    for (int c = tid; c <= G; c += NT) {
        const double u = P.u[(size_t)b * (G + 1) + c];
        zg[2 * G + c] = u;
        if (rank == 0 && P.check_uniforms && (!(u >= 0.0) || !(u < 1.0))) flag(P, SSV_STATUS_UNIFORM_RANGE);
    }
    __syncthreads();
    if (tx) trace(P, 8 * P.B + 3);

    if constexpr (EXACT) {
        // One warp per row slice (rows in flight in parallel): per-lane online
        // max / sum of e^(x - max) in one pass over the slot; the warp that
        // consumed a slot restages it with row r + NS.  (Tried: the whole CTA
        // on one row at a time, rows in ring order -- ~1.5x slower at C1/C2:
        // the per-row warp folds then sit on the critical path.)
        float mn = FLT_MAX;
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        for (int r = warp; r < NRc; r += kClWarps) {
            float m = -FLT_MAX;
            double sd = 0.0;
            float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
            float2 s2 = make_float2(0.f, 0.f), s3 = make_float2(0.f, 0.f);
            for (int h = 0; h < H && n > 0; ++h) {
                const int u = r * H + h, sl = u % NS, pn = piece_n(h);
                // Slot reuse: unit u is the (u / NS)-th fill of its slot.  Parity
                // waits only tell the current phase from the one before, so first
                // make sure the slot's previous unit has been consumed (and unit u
                // issued) -- a fresh barrier would otherwise pass a parity-1 wait.
                if (u >= NS) {
                    if (lane == 0)
                        while (ld_volatile_s32(&fills[sl]) < u / NS) __nanosleep(20);
                    __syncwarp();
                }
                mbar_wait(&full[sl], (unsigned)(u / NS) & 1u);
                if (u == NU - 1 && want_bonus_pf && lane == 0) prefetch_bonus();  // last slice landed
                const bool txw = P.trace && rank == 0 && b == 0 && lane == 0 && h == 0;
                if (txw && r < 8) trace(P, 8 * P.B + 4 + r);
                if (pn == 0) {  // (no copy was issued; the slot is free again)
                    __syncwarp();
                    if (lane == 0 && u + NS < NU) {
                        stage_row(u + NS);
                        st_volatile_s32(&fills[sl], (u + NS) / NS);
                    }
                    continue;
                }
                const int off = offs[sl], nv = (off + pn + VEC - 1) / VEC;
                const uint4* rv = reinterpret_cast<const uint4*>(slots + (size_t)sl * RB);
                // A step loads 4 vectors per lane (unguarded in the interior, so
                // the 4 shared-memory loads are in flight together), takes their
                // max, rescales the lane's sums if the max grew, and adds the
                // step's terms.  The sums stay fp32 (four chains per lane, <= 4
                // terms per chain per step; fp64 only in the lane / slice /
                // cluster folds): fp64 adds in the loop cost ~1.8x the slice
                // time (tools/slice_bench.cu).  The two edge vectors are masked
                // and join the last step.
                auto edge = [&](int v) {
                    uint4 w = rv[v];
                    if (v == 0 && off) mask_vec<T>(w, off, VEC);
                    if (v == nv - 1 && (off + pn) % VEC) mask_vec<T>(w, 0, (off + pn) % VEC);
                    return w;
                };
                const int vi1 = max(1, nv - 1);
                auto step = [&](const uint4* w, int nw) {  // nw <= 9 vectors, four sum chains
                    float cm = -FLT_MAX;
#pragma unroll
                    for (int u = 0; u < 9; ++u)
                        if (u < nw) AStat<T>::minmax(w[u], cm, mn);
                    if (cm > m) {
                        const float f = ex2f((m - cm) * 1.4426950408889634f);  // 0 on the first step
                        const float2 ff = make_float2(f, f);
                        s0 = __fmul2_rn(s0, ff);
                        s1 = __fmul2_rn(s1, ff);
                        s2 = __fmul2_rn(s2, ff);
                        s3 = __fmul2_rn(s3, ff);
                        m = cm;
                    }
                    if (m != -FLT_MAX) {  // a lane that has seen pads only adds nothing
                        const float2 negM = make_float2(-m, -m);
#pragma unroll
                        for (int u = 0; u < 9; ++u)
                            if (u < nw) AStat<T>::expsum(w[u], negM, (u & 3) == 0 ? s0 : (u & 3) == 1 ? s1 : (u & 3) == 2 ? s2 : s3);
                    }
                };
                // fp32: steps of eight vectors per lane (the per-step max /
                // rescale latency amortized over twice the terms; bf16 vectors
                // already hold eight terms), then four, then the remainder with
                // the two edge vectors.
                int v0 = 1 + lane;
                for (; sizeof(T) == 4 && v0 + 224 < vi1; v0 += 256) {
                    uint4 w[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) w[u] = rv[v0 + 32 * u];
                    step(w, 8);
                }
                for (; v0 + 96 < vi1; v0 += 128) {
                    uint4 w[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) w[u] = rv[v0 + 32 * u];
                    step(w, 4);
                }
                {  // the remainder (< 4 vectors per lane) and the edge vectors
                    uint4 w[5];
#pragma unroll
                    for (int u = 0; u < 4; ++u) w[u] = v0 + 32 * u < vi1 ? rv[v0 + 32 * u] : pad_vec<T>();
                    w[4] = lane == 0 ? edge(0) : (lane == 1 && nv > 1 ? edge(nv - 1) : pad_vec<T>());
                    step(w, 5);
                }
                __syncwarp();
                if (txw && r < 6) trace(P, 8 * P.B + 12 + r);
                if (lane == 0 && u + NS < NU) {  // this warp was the slot's only reader
                    stage_row(u + NS);
                    st_volatile_s32(&fills[sl], (u + NS) / NS);  // unit u + NS is in flight
                }
            }
            {
                const float2 a = __fadd2_rn(s0, s2), c = __fadd2_rn(s1, s3);
                sd = ((double)a.x + (double)a.y) + ((double)c.x + (double)c.y);
            }
            // fold the lanes: M = max, S = sum of s_l e^(m_l - M) (fp64)
            const float M = warp_max(m);
            double S = sd != 0.0 ? sd * exp((double)m - (double)M) : sd;  // NaN propagates
            S = warp_sum(S);
            const double2 pv = S != 0.0 ? make_double2((double)M, S) : make_double2(-CUDART_INF, 0.0);
            if (lane == 0 && (isnan(S) || M == INFINITY)) flag(P, SSV_STATUS_NONFINITE);
            if (PM > 1) {
                if (lane < CS) *cl.map_shared_rank(&part[r * PM + rank], lane) = pv;
            } else if (lane == 0) {
                part[r] = pv;
            }
        }
        if (__any_sync(kFull, !isfinite(mn)) && lane == 0) flag(P, SSV_STATUS_NONFINITE);
        if (tr) trace(P, 8 * b + 1);
        cl.sync();  // slice partials visible to the cluster
        if (tr) trace(P, 8 * b + 2);
        // Half a warp per row (cl_size <= 16): every row of a small step in one
        // round, 4-step segmented shuffles, the same fold order on every rank.
        const int half = lane >> 4, hl = lane & 15;
        for (int r0 = 2 * warp; r0 < NRc; r0 += 2 * kClWarps) {
            const int r = r0 + half;
            double2 v = make_double2(-CUDART_INF, 0.0);
            if (r < NRc && hl < CS) v = PM > 1 ? part[r * PM + hl] : *cl.map_shared_rank(&part[r], hl);
            double M = v.x;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(kFull, M, o, 16));
            double S = v.y != 0.0 ? v.y * exp(v.x - M) : 0.0;  // NaN propagates
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) S += __shfl_xor_sync(kFull, S, o, 16);
            if (hl == 0 && r < NRc) {
                if (!isfinite(M) || !isfinite(S)) flag(P, SSV_STATUS_NONFINITE);
                if (r < kMaxRowsSmem) sh.rs[r] = make_double2(M, S);
                if (rank == 0 && r < P.NR) P.rowstat[(size_t)b * P.NR + r] = make_double2(M, S);
            }
        }
        __syncthreads();
    }
    // decision (warp 0; every rank computes the same one)
    if (warp == 0) {
        int accepted = G;
        for (int c0 = 0; c0 < G; c0 += 32) {
            const int c = c0 + lane;
            bool rej = false;
            if (c < G) {
                double p, q;
                if (EXACT) {
                    const double2 sp = sh.rs[c], sq = sh.rs[G + c];
                    p = exp(zg[c] - sp.x) / sp.y;  // activation.cpp:20-27, dist.cpp:46-50
                    q = exp(zg[G + c] - sq.x) / sq.y;
                } else if (is_sigmoid(ACT)) {
                    p = sigmoid_act<ACT>(P, zg[c]);  // dist.cpp:60-69
                    q = sigmoid_act<ACT>(P, zg[G + c]);
                } else {
                    p = zg[c];
                    q = zg[G + c];
                    if (rank == 0 && (p < 0.0 || q < 0.0)) flag(P, SSV_STATUS_NEGATIVE);
                }
                const double tau = ratio_clamped(p, q);
                if (rank == 0) P.tau[(size_t)b * G + c] = tau;
                rej = !(zg[2 * G + c] <= tau);  // verify_reference.cpp:93-96 (inclusive)
            }
            const unsigned msk = __ballot_sync(kFull, rej);
            if (msk && accepted == G) accepted = c0 + __ffs(msk) - 1;
        }
        if (lane == 0) {
            Decision dd{};
            dd.Sp = dd.Sq = 1.0;
            if (accepted < G) {
                dd.mode = MODE_REJECT;
                dd.row = accepted;
                if (EXACT) {
                    dd.Mp = sh.rs[accepted].x;
                    dd.Sp = sh.rs[accepted].y;
                    dd.Mq = sh.rs[G + accepted].x;
                    dd.Sq = sh.rs[G + accepted].y;
                }
            } else if (P.PS == G + 1) {
                dd.mode = MODE_BONUS;
                dd.row = G;
            } else {
                dd.mode = MODE_NONE;
            }
            sh.dec = dd;
            if (rank == 0) {
                P.acc[b] = accepted;
                if (dd.mode == MODE_NONE) {
                    P.fin[b] = -1;  // kNoToken, step.hpp:11
                    P.rsu[b] = 0;
                    P.rden[b] = 0.0;
                }
            }
        }
    }
    __syncthreads();
    if (tr) trace(P, 8 * b + 3);
    const Decision d = sh.dec;
    if (!EXACT) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every rank has started
    // Granule masses of this rank's slice of the needed row(s) (L2-hot re-read),
    // also stored to global for the rare last-positive fallback.  The slice
    // total (fixed order) is pushed into every rank's rtot[rank] so that after
    // the barrier each rank holds all totals locally (no DSMEM reads after it).
    const int nloc = max(0, min(GPS, P.NG - rank * GPS));  // this rank's granules
    // Every row slice resident (exact): the rejected pair's slices are still in
    // this rank's shared memory -- granules and the element scan read them there.
    RowSlice<T> rs;
    if (EXACT && whole && NS == NRc && d.mode == MODE_REJECT && n > 0) {
        const int sp = d.row, sq = G + d.row;
        rs.p = reinterpret_cast<const T*>(slots + (size_t)sp * RB) + offs[sp];
        rs.q = reinterpret_cast<const T*>(slots + (size_t)sq * RB) + offs[sq];
        rs.lo = e0;
        rs.hi = e0 + n;
    }
    if (d.mode != MODE_NONE) {
        for (int j = warp; j < GPS; j += kClWarps) {
            const int g = rank * GPS + j;
            double2 out = make_double2(0.0, 0.0);
            if (g < P.NG) {
                if (rs.hi > 0) {
                    GranuleData<T> D;
                    granule_load<T, true>(P, b, g, d, D, rs.p + (g * kGW - e0), rs.q + (g * kGW - e0));
                    out = granule_reduce<T, ACT>(P, d, D);
                } else {
                    granule<T, ACT>(P, b, g, d, &out);
                }
            }
            if (lane == 0) {
                gloc[j] = out;
                if (g < P.NG) P.cgpart[(size_t)b * P.NG + g] = out;
            }
        }
        __syncthreads();
        if (warp == 0) {
            double2 t;
            if (d.mode == MODE_BONUS && ACT == ACT_SOFTMAX) {  // (max, sum e^(x - max)) of the slice
                double m = -CUDART_INF;
                for (int j = lane; j < nloc; j += 32)
                    if (gloc[j].y > 0.0) m = fmax(m, gloc[j].x);
                m = warp_max(m);
                double sm = 0.0;
                for (int j = lane; j < nloc; j += 32)
                    if (gloc[j].y > 0.0) sm += gloc[j].y * exp(gloc[j].x - m);
                t = make_double2(m, warp_sum(sm));
            } else {
                double a1 = 0.0, a2 = 0.0;
                for (int j = lane; j < nloc; j += 32) {
                    a1 += gloc[j].x;
                    a2 += gloc[j].y;
                }
                t = make_double2(warp_sum(a1), warp_sum(a2));
            }
            if (lane < CS) *cl.map_shared_rank(&rtot[rank], lane) = t;
        }
    }
    if (tr) trace(P, 8 * b + 4);
    cl.sync();  // rank totals delivered; granule masses visible in global memory
    if (tr) trace(P, 8 * b + 5);
    // Optional p / q / residual grids straight from the resident slices (no
    // second pass over the logits): every rank writes its slice of every row
    // -- the locator after its scan, the others instead of exiting early.
    auto write_grids = [&]() {
        if constexpr (EXACT) {
            if (!P.fuse_grids || n <= 0) return;
            float* gp = reinterpret_cast<float*>(P.grid_p);
            float* gq = reinterpret_cast<float*>(P.grid_q);
            float* gr = reinterpret_cast<float*>(P.grid_r);
            for (int c = 0; c <= G; ++c) {
                const bool pair = c < G;
                if (!pair && (!gp || NRc <= 2 * G)) break;
                const int rp = pair ? c : 2 * G;
                const T* xp = reinterpret_cast<const T*>(slots + (size_t)rp * RB) + offs[rp];
                const T* xq = pair ? reinterpret_cast<const T*>(slots + (size_t)(G + c) * RB) + offs[G + c] : xp;
                const float Mp = (float)sh.rs[rp].x, iSp = (float)(1.0 / sh.rs[rp].y);
                const float Mq = pair ? (float)sh.rs[G + c].x : 0.f, iSq = pair ? (float)(1.0 / sh.rs[G + c].y) : 0.f;
                float* op = gp ? gp + ((size_t)b * P.PS + c) * (size_t)V + e0 : nullptr;
                float* oq = gq && pair ? gq + ((size_t)b * G + c) * (size_t)V + e0 : nullptr;
                float* orr = gr && pair ? gr + ((size_t)b * G + c) * (size_t)V + e0 : nullptr;
                for (int i = tid; i < n; i += NT) {
                    const float pv = exp_rel_acc(load_smem_elem(xp + i), Mp) * iSp;
                    if (op) op[i] = pv;
                    if (oq || orr) {
                        const float qv = exp_rel_acc(load_smem_elem(xq + i), Mq) * iSq;
                        if (oq) oq[i] = qv;
                        if (orr) orr[i] = pv - qv > 0.f ? pv - qv : 0.f;
                    }
                }
            }
        }
    };
    if (d.mode == MODE_NONE) {
        write_grids();
        return;
    }
    const double u = zg[2 * G + G];  // u_final (verify_reference.cpp:98)
    // Every rank combines the totals in the same order: denominators
    // (verify_reference.cpp:51-62 / dist.cpp:114-121 at slice resolution) and
    // the rank whose slice holds u * denominator (the locator).
    if (warp == 0) {
        const double2 t = lane < CS ? rtot[lane] : make_double2(0.0, 0.0);
        bool useA = false;
        double denom = 1.0, gM = 0.0, gS = 1.0, w;
        if (d.mode == MODE_REJECT) {
            const double sa = warp_sum(t.x), sp = warp_sum(t.y);
            useA = sa > kZeroEps;  // verify_reference.cpp:57-62
            denom = useA ? sa : sp;
            w = useA ? t.x : t.y;
        } else if (ACT == ACT_SOFTMAX) {
            gM = warp_max(lane < CS && t.y > 0.0 ? t.x : -CUDART_INF);
            w = lane < CS && t.y > 0.0 ? t.y * exp(t.x - gM) : 0.0;
            gS = warp_sum(w);
        } else {
            w = t.y;
            denom = warp_sum(w);
        }
        const double norm = d.mode != MODE_REJECT && ACT == ACT_SOFTMAX ? gS : denom;
        const double incl = warp_scan_incl(w), run = incl - w;
        const double thr = u * norm;
        const unsigned hm = __ballot_sync(kFull, lane < CS && thr < run + w);
        const int owner = hm ? __ffs(hm) - 1 : -1;
        if (lane == 0) {
            sh.loc_g = owner;
            sh.loc_useA = useA;
            sh.loc_d[0] = __shfl_sync(kFull, run, owner >= 0 ? owner : 0);
            sh.loc_d[1] = denom;
            sh.loc_d[2] = gM;
            sh.loc_d[3] = gS;
            if (rank == 0) {
                if (P.rsu) P.rsu[b] = d.mode == MODE_REJECT ? 1 : 0;
                if (P.rden) P.rden[b] = d.mode == MODE_REJECT && useA ? denom : 0.0;
            }
        } else {
            (void)__shfl_sync(kFull, run, owner >= 0 ? owner : 0);
        }
    }
    __syncthreads();
    const int owner = sh.loc_g;
    if (rank != (owner >= 0 ? owner : 0)) {  // one locator per batch row
        write_grids();
        return;
    }
    const bool tl = P.trace && b == 0 && tid == 0;  // locate stamps: trace[8B + 18 ..]
    if (tr) trace(P, 8 * b + 6);
    if (tl) trace(P, 8 * P.B + 21);
    RowCtx R;
    R.mode = d.mode;
    R.Mp = d.Mp;
    R.Sp = d.Sp;
    R.Mq = d.Mq;
    R.Sq = d.Sq;
    R.useA = sh.loc_useA;
    R.denom = sh.loc_d[1];
    const double gM = sh.loc_d[2], gS = sh.loc_d[3];
    const bool soft_bonus = d.mode != MODE_REJECT && ACT == ACT_SOFTMAX;
    if (soft_bonus) {
        R.Mp = gM;
        R.Sp = gS;
        R.denom = 1.0;  // sample_row's sequential_sum of a softmax row (1 within rounding)
    }
    const double norm = soft_bonus ? gS : R.denom;
    // granule level inside the locator's slice (warp 0): contiguous lane ranges,
    // one warp scan, first granule whose prefix passes u * norm
    if (warp == 0) {
        int gst = -1;
        double car = 0.0;
        if (owner >= 0) {
            auto wloc = [&](int j) -> double {  // unnormalized granule mass
                const double2 v = gloc[j];
                if (d.mode == MODE_REJECT) return R.useA ? v.x : v.y;
                if (ACT == ACT_SOFTMAX) return v.y > 0.0 ? v.y * exp(v.x - gM) : 0.0;
                return v.y;
            };
            const int gpl = (nloc + 31) / 32;
            const int ja = min(nloc, lane * gpl), jb = min(nloc, ja + gpl);
            double sm = 0.0;
            for (int j = ja; j < jb; ++j) sm += wloc(j);
            const double incl = warp_scan_incl(sm), tot = __shfl_sync(kFull, incl, 31);
            double run = sh.loc_d[0] + (incl - sm);
            const double thr = u * norm;
            int hit = 0x7fffffff;
            double hit_carry = 0.0;
            for (int j = ja; j < jb; ++j) {
                const double w = wloc(j);
                if (thr < run + w) {
                    hit = j;
                    hit_carry = run / norm;
                    break;
                }
                run += w;
            }
            const unsigned hm = __ballot_sync(kFull, hit != 0x7fffffff);
            const int src = hm ? __ffs(hm) - 1 : 0;
            const int jh = __shfl_sync(kFull, hit, src);
            car = __shfl_sync(kFull, hit_carry, src);
            if (hm) {
                gst = rank * GPS + jh;
            } else {  // rounding between the slice total and its granules: continue after the slice
                gst = rank * GPS + nloc;
                car = (sh.loc_d[0] + tot) / norm;
            }
        }
        if (lane == 0) {
            sh.loc_g = gst;
            sh.loc_d[0] = car;
        }
    }
    __syncthreads();
    if (tl) trace(P, 8 * P.B + 18);
    const double2* gp = P.cgpart + (size_t)b * P.NG;
    auto gmass = [&](int g) -> double {  // normalized granule mass (fallback path)
        const double2 v = __ldcg(&gp[g]);
        if (R.mode == MODE_REJECT) return (R.useA ? v.x : v.y) / R.denom;
        if (ACT == ACT_SOFTMAX) return v.y > 0.0 ? v.y * exp(v.x - gM) / gS : 0.0;
        return v.y / R.denom;
    };
    const T* pr = p_row<T>(P, b, d.row);
    const T* qr = d.mode == MODE_REJECT ? q_row<T>(P, b, d.row) : nullptr;
    const int token = locate_scan<T, ACT, NT>(P, R, pr, qr, sh.loc_g, sh.loc_d[0], u, gmass, sh, tl, rs);
    if (tl) trace(P, 8 * P.B + 20);
    if (tid == 0) {
        P.fin[b] = token;
        if (P.trace) {
            trace(P, 8 * b + 7);
            atomicMax(&P.trace[8 * P.B + 1], gtime());
        }
    }
    write_grids();
}

// ---------------------------------------------------------------------------
// K3: optional materialized grids (activation.cpp:20-49; verify_fused.cpp:50
// residual-in-q semantics; verify_sigmoid.cpp:39-48), after the verify launch
// that produced the row statistics (a normalized softmax row cannot be written
// before its row's statistics exist, so this is a second pass over the logits;
// it reads every logit once and writes each requested grid once).
// Work unit = (row, 4096-element segment): a drafted pair (b, c < gamma)
// writes p, q and residual from one read of both rows; the bonus row (b, gamma)
// writes p.  Row-major addressing (no per-element division), coalesced
// element loads (rows of odd V start at any alignment).  Values: fp32 via
// exp_rel_acc (~3e-7) / sigmoid_fast, fp64 storage in fp64.
constexpr int kMatSeg = 4096;
template <typename T, int ACT>
__global__ void __launch_bounds__(kThreads) k_materialize(StepParams P, void* outp, void* outq, void* outr) {
    using A = typename Elem<T>::acc;
    using O = typename std::conditional<sizeof(A) == 8, double, float>::type;
    const int V = P.V, G = P.G;
    const int nseg = (V + kMatSeg - 1) / kMatSeg;
    const int pairs = P.B * G, bonus = P.PS == G + 1 && outp ? P.B : 0;
    const long units = (long)(pairs + bonus) * nseg;
    const A alpha = (A)P.alpha, invw = (A)(1.0 / P.width);
    const bool want_q = outq || outr;
    for (long w = blockIdx.x; w < units; w += gridDim.x) {
        const int row = (int)(w / nseg), seg = (int)(w - (long)row * nseg);
        const bool is_pair = row < pairs;
        const int b = is_pair ? row / G : row - pairs;
        const int c = is_pair ? row - b * G : G;
        const int lo = seg * kMatSeg, hi = min(V, lo + kMatSeg);
        double2 sp = make_double2(0.0, 1.0), sq = sp;
        if (ACT == ACT_SOFTMAX) {
            sp = __ldcg(&P.rowstat[(size_t)b * P.NR + (is_pair ? c : 2 * G)]);
            if (is_pair && want_q) sq = __ldcg(&P.rowstat[(size_t)b * P.NR + G + c]);
        }
        const A Mp = (A)sp.x, iSp = (A)(1.0 / sp.y), Mq = (A)sq.x, iSq = (A)(1.0 / sq.y);
        auto act = [&](A x, A M, A iS) -> A {
            if (ACT == ACT_SOFTMAX) return exp_rel_acc(x, M) * iS;
            if (ACT == ACT_SIGMOID_HALF) return (A)sigmoid_act<ACT>(P, (double)x);
            if (is_sigmoid(ACT)) return sigmoid_fast((x - alpha) * invw);
            return x;
        };
        const T* __restrict__ pr = p_row<T>(P, b, c);
        const T* __restrict__ qr = is_pair ? q_row<T>(P, b, c) : nullptr;
        O* __restrict__ op = outp ? reinterpret_cast<O*>(outp) + ((size_t)b * P.PS + c) * (size_t)V : nullptr;
        O* __restrict__ oq = (outq && is_pair) ? reinterpret_cast<O*>(outq) + ((size_t)b * G + c) * (size_t)V : nullptr;
        O* __restrict__ orr = (outr && is_pair) ? reinterpret_cast<O*>(outr) + ((size_t)b * G + c) * (size_t)V : nullptr;
        const bool need_p = op || orr, need_q = is_pair && want_q;
        // All of the segment's loads first (kMatSeg / kThreads per thread in
        // flight), then the values and the stores: one memory latency per unit
        // instead of one per element (the stores could alias the loads).
        constexpr int EPT = kMatSeg / kThreads;
        A xp[EPT], xq[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int i = lo + threadIdx.x + e * kThreads;
            xp[e] = need_p && i < hi ? load_elem(pr + i) : (A)0;
            xq[e] = need_q && i < hi ? load_elem(qr + i) : (A)0;
        }
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int i = lo + threadIdx.x + e * kThreads;
            if (i >= hi) break;
            const A pv = need_p ? act(xp[e], Mp, iSp) : (A)0;
            if (op) op[i] = (O)pv;
            if (need_q) {
                const A qv = act(xq[e], Mq, iSq);
                if (oq) oq[i] = (O)qv;
                if (orr) orr[i] = (O)(pv - qv > (A)0 ? pv - qv : (A)0);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Synthetic inputs: bench.cpp:46-74 per batch row (seed + b), using the
// counter RNG of rng.cpp:12-33 (SplitMix64 at index i, Box-Muller in fp64).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t word_at(uint64_t seed, uint64_t index) {
    return mix64(seed + (index + 1) * 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t index) {
    return (double)(word_at(seed, index) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t n) {  // n-th normal = words 2n, 2n+1
    const double u1 = ((double)(word_at(seed, 2 * n) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (double)(word_at(seed, 2 * n + 1) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

template <typename T>
__device__ __forceinline__ T to_store(double v);
template <>
__device__ __forceinline__ float to_store<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ double to_store<double>(double v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_store<__nv_bfloat16>(double v) {
    return __float2bfloat16_rn((float)v);  // double -> fp32 -> bf16, like orc_round_bf16
}

template <typename T>
__global__ void k_gen_logits(uint64_t seed, int B, int G, int V, T* zp, T* zq) {
    const size_t per_b = (size_t)(2 * G + 1) * V;
    const size_t n = (size_t)B * per_b;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int b = (int)(i / per_b);
        const size_t j = i % per_b;
        const uint64_t s = seed + (uint64_t)b;
        const size_t np = (size_t)(G + 1) * V;
        if (j < np) {
            zp[(size_t)b * np + j] = to_store<T>(4.0 * normal_at(s, j));
        } else {
            const size_t jq = j - np;  // q row c element e: z_p[c][e] + N at index np + jq
            const double v = 4.0 * normal_at(s, jq) + 1.0 * normal_at(s, np + jq);
            zq[(size_t)b * G * V + jq] = to_store<T>(v);
        }
    }
}

// Draft draws (index 2(2G+1)V + c) and acceptance/final uniforms
// (index 2(2G+1)V + G + c) of bench.cpp:66-73.
__global__ void k_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int per = 2 * G + 1;
    if (i >= B * per) return;
    const int b = i / per, c = i % per;
    const uint64_t base = 2ull * (uint64_t)(2 * G + 1) * (uint64_t)V;
    const double v = uniform_at(seed + (uint64_t)b, base + (uint64_t)c);
    if (c < G) draft_u[(size_t)b * G + c] = v;
    else u[(size_t)b * (G + 1) + (c - G)] = v;
}

// ---------------------------------------------------------------------------
// Host-side launchers.
//
// Experiment knobs (SSV_* environment variables) exist only in experiment
// builds (make EXPERIMENTS=1 -> -DSSV_EXPERIMENTS); the product library always
// uses the defaults, so no environment variable can change what it computes.
static int knob(const char* name, int dflt) {
#ifdef SSV_EXPERIMENTS
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
#else
    (void)name;
    return dflt;
#endif
}
static bool knob_set(const char* name) {
#ifdef SSV_EXPERIMENTS
    return getenv(name) != nullptr;
#else
    (void)name;
    return false;
#endif
}
static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static size_t elem_size(int dtype) { return dtype == DT_F64 ? 8 : (dtype == DT_BF16 ? 2 : 4); }

void plan_geometry(int dtype, int act, StepParams& P) {
    const int s = (int)elem_size(dtype);
    const int VEC = 16 / s;
    P.nB = (P.V + kCB * kBG - 1) / (kCB * kBG);
    P.NG = (P.V + kGW - 1) / kGW;
    const long resident = (long)sm_count() * kCtaMinBlocks;
    const bool exact = act == ACT_SOFTMAX && !P.sample_mode;
    if (!exact) {
        P.NR = 0;
        P.Kc = P.runA = P.K = 0;
        P.nA = 0;
    } else {
        // chunks per row (any alignment) and the run length: long enough to
        // amortize a partial over many chunks, short enough that the A phase
        // still spreads over ~4 items per resident CTA.
        const long nvec = (P.V + 2L * VEC - 2) / VEC;
        const long CV = (long)kCtaThreads * kAVec;
        P.Kc = (int)((nvec + CV - 1) / CV);
        // Runs as long as load balance allows (up to 64 chunks = 1 MB): every
        // run ends in a warp fold and a claim, so long runs keep the ring busy
        // (measured: 38-chunk runs stream at ~100% of the copy roofline, 4-chunk
        // runs at ~70%).  The lags below scale with the run length.
        static const int run_cap = std::max(1, knob("SSV_RUNA", 64));
        long want = ((long)P.Kc * P.B * P.NR + 4 * resident - 1) / (4 * resident);
        want = std::max<long>(1, std::min<long>({want, (long)P.Kc, (long)run_cap}));
        static const int run_force = knob("SSV_RUNA_FORCE", 0);
        if (run_force > 0) want = std::min<long>(run_force, P.Kc);
        const long runs = (P.Kc + want - 1) / want;
        P.runA = (int)((P.Kc + runs - 1) / runs);
        P.K = (P.Kc + P.runA - 1) / P.runA;
        P.nA = P.NR * P.K;
    }
    P.KP = P.K * kWarps;
    P.nph[IT_A] = P.nA;
    P.nph[IT_D] = P.sample_mode ? 0 : 1;  // exact: row statistics + decision; sigmoid / probs: gathers only
    P.nph[IT_B] = P.nB;
    P.nph[IT_L] = 1;
    // Phase offsets, in segments of one batch row each: a phase of row b is
    // dispatched about one resident wave after the phase it waits on, so the
    // wait is short and the rejected pair (read by the A-items a few rows
    // earlier) is still in L2 when its B-items re-read it.
    // items in progress at any time: one per resident CTA plus one claimed ahead
    const long seg = (long)P.nph[0] + P.nph[1] + P.nph[2] + P.nph[3];
    static const int lag_mult = std::max(0, knob("SSV_LAG_MULT", 0));  // 0: default by run length
    const int wave = (int)((2 * resident + seg - 1) / seg);
    // A D-item waits for its row's runs, which take ~runA/8 "waves" of
    // claims to complete; B- and L-items follow one wave after that.
    const int mD = lag_mult ? lag_mult : std::max(1, (P.runA + 7) / 8);
    auto clampB = [&](long x) { return (int)std::min<long>(P.B, std::max<long>(0, x)); };
    P.off[IT_A] = 0;
    if (exact) {
        P.off[IT_D] = clampB((long)mD * wave);
        P.off[IT_B] = clampB(P.off[IT_D] + (long)std::max(1, mD / 2) * wave);
        P.off[IT_L] = clampB(P.off[IT_B] + (long)std::max(1, mD) * wave);
    } else {  // a gathers-only D-item takes ~2 us: B-items one wave later, L one wave after them
        P.off[IT_D] = 0;
        P.off[IT_B] = P.sample_mode ? 0 : clampB(wave);
        P.off[IT_L] = clampB(P.off[IT_B] + wave);
    }
    // Ranges of constant segment composition.
    int pts[10], n = 0;
    pts[n++] = 0;
    for (int p = 0; p < 4; ++p) {
        if (P.nph[p] == 0) continue;
        pts[n++] = P.off[p];
        pts[n++] = P.off[p] + P.B;
    }
    for (int i = 1; i < n; ++i)  // insertion sort of <= 9 points, then dedupe
        for (int j = i; j > 0 && pts[j - 1] > pts[j]; --j) std::swap(pts[j - 1], pts[j]);
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (m == 0 || pts[i] != pts[m - 1]) pts[m++] = pts[i];
    n = m;
    const int tend = P.B + P.off[IT_L];
    P.nrange = 0;
    unsigned item = 0;
    for (int i = 0; i < n && pts[i] < tend; ++i) {
        const int t0 = pts[i], t1 = i + 1 < n ? std::min(pts[i + 1], tend) : tend;
        int sz = 0;
        for (int p = 0; p < 4; ++p)
            if (P.nph[p] > 0 && t0 - P.off[p] >= 0 && t0 - P.off[p] < P.B) sz += P.nph[p];
        if (sz == 0 || t1 <= t0) continue;
        P.rseg[P.nrange] = t0;
        P.ritem[P.nrange] = item;
        P.rsize[P.nrange] = sz;
        ++P.nrange;
        item += (unsigned)sz * (unsigned)(t1 - t0);
    }
    P.ritem[P.nrange] = item;
    P.rseg[P.nrange] = tend;
    P.n_items = item;
}

int trace_slots(const StepParams& P) { return 8 * P.B + 26; }

// Programmatic stream serialization for the verify launches (see pdl_enter).
static int pdl_attr(cudaLaunchAttribute& a) {
    static const bool off = knob_set("SSV_NO_PDL");
    if (off) return 0;
    a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a.val.programmaticStreamSerializationAllowed = 1;
    return 1;
}

template <typename T, int ACT>
static void launch_verify_t(const StepParams& P, const Launch& L) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_verify<T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
        attr = true;
    }
    static int per_sm = 0;
    if (per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_verify<T, ACT>, kCtaThreads, kDynSmem);
        per_sm = std::max(1, per_sm);
    }
    // Persistent: one CTA per resident slot, items claimed in order.  (Any
    // grid size is deadlock-free -- items only wait on earlier claims.)
    const unsigned grid = std::min<unsigned>(P.n_items, (unsigned)(sm_count() * per_sm));
    StepParams Q = P;
    Q.claim_ahead = P.n_items > 2u * grid;
    static const int dbgm = knob("SSV_DBG_MODE", 0);
    Q.dbg = dbgm;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kCtaThreads, 1, 1);
    cfg.dynamicSmemBytes = kDynSmem;
    cfg.stream = L.st;
    cudaLaunchAttribute at[1];
    cfg.attrs = at;
    cfg.numAttrs = pdl_attr(at[0]);
    const int h = L.begin(KID_VERIFY);
    cudaLaunchKernelEx(&cfg, k_verify<T, ACT>, Q);
    L.end(h);
}

// Cluster path geometry (cl_size 0 = not applicable: use the streaming kernel).
constexpr int kClusterSmemMax = 227 * 1024 - 4096;  // dynamic budget (static Shared + slack)

constexpr int kClusterSmemTwoPerSm = 100 * 1024;  // two CTAs per SM (twice the resident clusters)

static int cluster_smem(const StepParams& P, int s, int NRc, int NS, int SE, int GPS, int cs, int PE = 0) {
    const int VEC = 16 / s;
    const int RB = (((PE ? PE : SE) + 2 * VEC) * s + 15) & ~15;
    const int PM = NRc * cs <= kClPushMax ? cs : 1;  // slice partials pushed to every rank
    long bytes = (long)NS * RB + 8L * ((NS + 1) & ~1) + 16L * (NRc * PM + GPS + 16) + 8L * (3 * P.G + 1) + 8L * NS + 64;
    return bytes > kClusterSmemMax ? -1 : (int)bytes;
}

template <typename T, int ACT, int NT>
static int max_active_clusters(int cs, int smem) {
    struct Entry {
        int cs, smem, n;
    };
    static Entry cache[16];  // the plans a serving loop alternates between
    static int n_cached = 0, next = 0;
    for (int i = 0; i < n_cached; ++i)
        if (cache[i].cs == cs && cache[i].smem == smem) return cache[i].n;
    auto k = k_verify_cluster<T, ACT, NT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kClusterSmemMax);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[next] = Entry{cs, smem, n};
    next = (next + 1) % 16;
    n_cached = n_cached < 16 ? n_cached + 1 : 16;
    return n;
}

// Small batches: one cluster per batch row, all clusters resident at once.
// Largest cluster (most SMs per row) whose slices fit in shared memory and of
// which B fit on the GPU together.
template <typename T, int ACT>
static bool plan_cluster_t(StepParams& P, int s, bool allow_resident) {
    static const bool off = knob_set("SSV_NO_CLUSTER");
    static const bool dbg = knob_set("SSV_DEBUG");
    if (off || P.sample_mode || P.G > 256) return false;
    const int NRc = ACT == ACT_SOFTMAX ? 2 * P.G + (P.NR > 2 * P.G ? 1 : 0) : 0;  // bonus stats only if materialized
    if (NRc > kMaxRowsSmem) return false;  // the decision reads every row's statistics from SMEM
    // (two-CTA clusters measured slower than the streaming kernel at B = 64)
    static const int res_env = knob("SSV_RES_MODE", 2);
    const int res_mode = allow_resident ? res_env : 0;
    static const int force_cs = knob("SSV_FORCE_CS", 0);
    static const bool res_nopad = knob_set("SSV_RES_NOPAD");
    for (int pass = res_mode == 2 ? 0 : 1; pass < 2; ++pass)
    for (int cs : {16, 12, 11, 10, 9, 8, 4}) {
        if (force_cs && cs != force_cs) continue;
        if (pass == 1 && cs > 8 && cs < 12) continue;  // odd sizes only for the resident plan
        const bool no_resident = res_mode == 0 || (res_mode == 2 && pass == 1);
        const int SE = ((P.V + cs - 1) / cs + kGW - 1) / kGW * kGW;
        const int GPS = SE / kGW;
        const int RB = NRc > 0 ? ((SE + 2 * (16 / s)) * s + 15) & ~15 : 0;
        // Small batches first try one CTA per SM with every row slice resident
        // (no ring restaging on the critical path), 16 warps when the rows
        // outnumber 8 (one row fold per warp); used only if all B clusters
        // are still co-resident.
        if constexpr (ACT == ACT_SOFTMAX) {
          if (!no_resident && (long)P.B * cs <= sm_count()) {
            int smem1 = cluster_smem(P, s, NRc, NRc, SE, GPS, cs);
            // Slices that would fit two CTAs per SM: padded to one CTA per SM
            // (C1 bf16 17.7 -> 14.8 us, B=1 gamma=2 16.4 -> 13.4 us).
            if (!res_nopad && smem1 >= 0 && smem1 <= kClusterSmemTwoPerSm) smem1 = kClusterSmemTwoPerSm + 16 * 1024;
            if (smem1 > kClusterSmemTwoPerSm) {
                const int nt = NRc > 8 ? 512 : 256;
                const int mac = nt == 512 ? max_active_clusters<T, ACT, 512>(cs, smem1)
                                          : max_active_clusters<T, ACT, 256>(cs, smem1);
                if (dbg)
                    fprintf(stderr, "ssv: cluster plan (resident) act=%d B=%d V=%d rows=%d cs=%d SE=%d smem=%d threads=%d max_active=%d\n",
                            ACT, P.B, P.V, NRc, cs, SE, smem1, nt, mac);
                if (mac >= P.B) {
                    P.cl_size = cs;
                    P.cl_se = SE;
                    P.cl_gps = GPS;
                    P.cl_rows = NRc;
                    P.cl_slots = NRc;
                    P.cl_rowbytes = RB;
                    P.cl_smem = smem1;
                    P.cl_threads = nt;
                    P.cl_pieces = 1;
                    P.cl_resident = 1;
                    P.cl_pe = SE;
                    static const int dbgm = knob("SSV_DBG_MODE", 0);
                    P.dbg = dbgm;  // experiment bits (4: no bonus-row prefetch)
                    P.NR = NRc;
                    return true;
                }
            }
          }
        }
        if (pass == 0) continue;
        // every row resident if that still leaves two CTAs per SM, else a ring
        int NS = NRc;
        const int all_rows = NS > 0 ? cluster_smem(P, s, NRc, NS, SE, GPS, cs) : 0;  // -1: beyond one SM
        if (all_rows < 0 || all_rows > kClusterSmemTwoPerSm) {
            const int base = cluster_smem(P, s, NRc, 0, SE, GPS, cs);
            NS = std::max(2, std::min(NRc, (kClusterSmemTwoPerSm - base) / std::max(RB + 20, 1)));
        }
        // Measured crossover vs the streaming kernel (tools/sweep.py, gamma 1-16 x
        // B 1-64 x V 32000-151936, fp32 / bf16): a CTA's slices of all its rows
        // must stay small for its shared-memory ring -- up to ~300 KB; ~600 KB
        // with a ring of >= 4 slots; ~520 KB at B >= 48, where the streaming
        // kernel's per-row tail costs more.
        const long cta_bytes = (long)NRc * RB;
        // Since the pieced ring (below): also up to 600 KB at B >= 32 and V <= 64K when
        // the ring holds >= 3 slices or streams pieces (B=64 gamma=5 V=51865:
        // 59.5 -> 53.8 us; B=32 gamma=8 V=51865: 52.3 -> 44.4 us; the V = 151936
        // shapes stay on the streaming kernel, 6-60 % faster there).
        // pieces of >= 12 KB (measured: 12 KB beats 16 KB on every ring shape,
        // e.g. B=64 gamma=8 V=51865 bf16 67.0 -> 59.6 us; 10 KB loses C3 f32)
        static const int piece_min = knob("SSV_PIECE_KB", 12) * 1024;
        const bool pieced = NS < NRc && SE * s >= 2 * piece_min;
        static const bool no_gate = knob_set("SSV_NO_GATE");
        if (!no_gate && !(cta_bytes <= 300L * 1024 || (NS >= 4 && cta_bytes <= 600L * 1024) || (P.B >= 48 && cta_bytes <= 520L * 1024) ||
                          (P.B >= 32 && P.V <= 65536 && cta_bytes <= 600L * 1024 && (NS >= 3 || pieced))))
            continue;
        // A true ring streams pieces of the slices (H per slice, >= 12 KB each):
        // a slot is refilled after a piece's fold, not a whole slice's
        // (C3 f32, 32 KB slices in 16 KB pieces: 48.4 -> 44.7 us; 8 KB pieces
        // measured slower than whole 16 KB slices).
        static const int pieces_env = knob("SSV_PIECES", 0);
        int H = 1, PE = SE, NSu = NS;
        const int want_h = pieces_env > 0 ? pieces_env : std::max(1, std::min(4, SE * s / piece_min));
        if (NS < NRc && want_h > 1) {
            H = want_h;
            PE = ((SE + H - 1) / H + kGW - 1) / kGW * kGW;
            H = (SE + PE - 1) / PE;
            const int RBp = ((PE + 2 * (16 / s)) * s + 15) & ~15;
            const int base = cluster_smem(P, s, NRc, 0, SE, GPS, cs, PE);
            NSu = std::max(2, std::min(NRc * H, (kClusterSmemTwoPerSm - base) / std::max(RBp + 20, 1)));
        }
        const int smem = cluster_smem(P, s, NRc, NSu, SE, GPS, cs, PE);
        if (smem < 0) continue;
        const int mac = max_active_clusters<T, ACT, kClThreads>(cs, smem);
        if (dbg)
            fprintf(stderr, "ssv: cluster plan act=%d B=%d V=%d rows=%d slots=%d pieces=%d cs=%d SE=%d smem=%d max_active=%d\n",
                    ACT, P.B, P.V, NRc, NSu, H, cs, SE, smem, mac);
        if (mac < P.B) continue;
        P.cl_size = cs;
        P.cl_se = SE;
        P.cl_gps = GPS;
        P.cl_rows = NRc;
        P.cl_slots = NSu;
        P.cl_rowbytes = H > 1 ? (((PE + 2 * (16 / s)) * s + 15) & ~15) : RB;
        P.cl_smem = smem;
        P.cl_threads = kClThreads;
        P.cl_pieces = H;
        P.cl_resident = 0;
        P.cl_pe = PE;
        static const int dbgm = knob("SSV_DBG_MODE", 0);
        P.dbg = dbgm;
        if (ACT == ACT_SOFTMAX) P.NR = NRc;  // rowstat rows the cluster path writes
        return true;
    }
    return false;
}

bool plan_cluster(int dtype, int act, StepParams& P, bool allow_resident) {
    P.cl_size = 0;
    if (dtype == DT_F32) {
        if (act == ACT_SOFTMAX) return plan_cluster_t<float, ACT_SOFTMAX>(P, 4, allow_resident);
        if (act == ACT_SIGMOID) return plan_cluster_t<float, ACT_SIGMOID>(P, 4, allow_resident);
        if (act == ACT_SIGMOID_HALF) return plan_cluster_t<float, ACT_SIGMOID_HALF>(P, 4, allow_resident);
        return plan_cluster_t<float, ACT_PROBS>(P, 4, allow_resident);
    }
    if (dtype == DT_BF16) {
        if (act == ACT_SOFTMAX) return plan_cluster_t<__nv_bfloat16, ACT_SOFTMAX>(P, 2, allow_resident);
        if (act == ACT_SIGMOID) return plan_cluster_t<__nv_bfloat16, ACT_SIGMOID>(P, 2, allow_resident);
        if (act == ACT_SIGMOID_HALF) return plan_cluster_t<__nv_bfloat16, ACT_SIGMOID_HALF>(P, 2, allow_resident);
        return plan_cluster_t<__nv_bfloat16, ACT_PROBS>(P, 2, allow_resident);
    }
    return false;
}

template <typename T, int ACT>
static void launch_cluster_t(const StepParams& P, const Launch& L) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P.B * P.cl_size), 1, 1);
    cfg.blockDim = dim3((unsigned)P.cl_threads, 1, 1);
    cfg.dynamicSmemBytes = P.cl_smem;
    cfg.stream = L.st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P.cl_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1 + pdl_attr(at[1]);
    const int h = L.begin(KID_VERIFY);
    if constexpr (ACT == ACT_SOFTMAX) {
        if (P.cl_threads == 512) {
            cudaLaunchKernelEx(&cfg, k_verify_cluster<T, ACT, 512>, P);
            L.end(h);
            return;
        }
    }
    cudaLaunchKernelEx(&cfg, k_verify_cluster<T, ACT>, P);
    L.end(h);
}

// Slab path geometry (sl_on 0 = not applicable).  One CTA per SM (shared
// memory sized so), nbuf unit buffers: Dp in flight, one in use, L awaiting
// their batch row's decision.
constexpr int kSlabSmemMax = 227 * 1024 - 4096;  // dynamic budget (static Shared + slack)

template <typename T>
static bool plan_slab_t(StepParams& P) {
    P.sl_on = 0;
    if (P.sample_mode || 2 * P.G > kMaxRowsSmem) return false;
    const int NRd = 2 * P.G;
    const int ub = NRd * kSlabRowBytes;
    const int nbuf = std::min((kSlabSmemMax - kSlabGcache) / ub, 16);
    const int SE = kSlabVec * (int)(16 / sizeof(T));
    const int NS = (P.V + SE - 1) / SE;
    const int smem = nbuf * ub + kSlabGcache;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_verify_slab<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlabSmemMax);
        attr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_verify_slab<T>, kCtaThreads, smem);
    if (per_sm < 1) return false;
    const int grid = sm_count() * per_sm;
    const int Lmin = std::max(1, (NS - 1 + grid - 1) / grid);
    if (nbuf < Lmin + 2) return false;
    static const int dp_env = knob("SSV_SLAB_DP", 0);
    int Dp = dp_env > 0 ? dp_env : (64 * 1024 + ub - 1) / ub;
    Dp = std::max(1, std::min(Dp, nbuf - 1 - Lmin));
    P.sl_on = 1;
    P.sl_ns = NS;
    P.sl_nbuf = nbuf;
    P.sl_dp = Dp;
    P.sl_lag = P.sl_nbuf - 1 - Dp;
    P.sl_ub = ub;
    P.sl_smem = P.sl_nbuf * ub + kSlabGcache;
    P.sl_grid = grid;
    static const int sl_dbg = knob("SSV_SLAB_TRACE", 0);
    P.sl_dbg = sl_dbg;
    static const int dbgm = knob("SSV_DBG_MODE", 0);
    P.dbg = dbgm;  // experiment bits (slab: 1 statistics only, 2 loads only; results invalid)
    P.NR = NRd;
    P.KP = NS;
    static const bool dbg = knob_set("SSV_DEBUG");
    if (dbg)
        fprintf(stderr, "ssv: slab plan B=%d G=%d V=%d NS=%d nbuf=%d Dp=%d L=%d ub=%d smem=%d grid=%d\n", P.B, P.G,
                P.V, NS, P.sl_nbuf, Dp, P.sl_lag, ub, P.sl_smem, grid);
    return true;
}

bool plan_slab(int dtype, int act, StepParams& P) {
    P.sl_on = 0;
    if (act != ACT_SOFTMAX) return false;
    if (dtype == DT_F32) return plan_slab_t<float>(P);
    if (dtype == DT_BF16) return plan_slab_t<__nv_bfloat16>(P);
    return false;
}

template <typename T>
static void launch_slab_t(const StepParams& P, const Launch& L) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P.sl_grid, 1, 1);
    cfg.blockDim = dim3(kCtaThreads, 1, 1);
    cfg.dynamicSmemBytes = P.sl_smem;
    cfg.stream = L.st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident (the schedule's waits need it)
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1 + pdl_attr(at[1]);
    const int h = L.begin(KID_VERIFY);
    cudaLaunchKernelEx(&cfg, k_verify_slab<T>, P);
    L.end(h);
}

// Sigmoid-stream geometry (sg_on 0 = not applicable): tiles of TE elements
// (48 KB of one row), a ring of nbuf tiles per CTA, two CTAs per SM.
template <typename T, int ACT>
static bool plan_sig_t(StepParams& P) {
    P.sg_on = 0;
    if (P.sample_mode) return false;
    static const int te_kb = knob("SSV_SIG_TE_KB", 48);  // 48 KB tiles: 32 KB 55 us, 64 KB (one CTA per SM) 67 us at C4
    static const int sg_dw_env = knob("SSV_SIGW_DW16", 0);  // deciding warps' share (16ths); 0: by the stream length
    const int TE = te_kb * 1024 / (int)sizeof(T) / (kGW * kWarps) * (kGW * kWarps);  // multiple of kGW * kWarps
    const int tb = ((TE + 2 * (16 / (int)sizeof(T))) * (int)sizeof(T) + 127) & ~127;
    // Two CTAs per SM (16 warps to hide the per-element MUFU chains), each a
    // ring of two 48 KB tiles (three measured no faster) plus the locate's
    // granule cache.
    static const int nb_env = knob("SSV_SIG_NBUF", 0);
    const int nbuf = nb_env > 1 ? nb_env : 2;
    const int smem = nbuf * tb + 64 + std::min(P.NG, kLocCap) * (int)sizeof(double2);
    if (smem > kSlabSmemMax || nbuf < 2) return false;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_verify_sig<T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlabSmemMax);
        attr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_verify_sig<T, ACT>, kCtaThreads, smem);
    if (per_sm < 1) return false;
    P.sg_on = 1;
    P.sg_warp = 0;
    static const int sl_dbg = knob("SSV_SLAB_TRACE", 0);
    P.sl_dbg = sl_dbg;
    {  // 16-byte-aligned rows: the barrier-free warp kernel
        const bool aligned = (reinterpret_cast<uintptr_t>(P.zp) & 15) == 0 && ((size_t)P.V * sizeof(T)) % 16 == 0;
        static const int no_warp = knob("SSV_SIG_NO_WARP", 0);
        if (aligned && !no_warp) {
            const int smemw = kSigWStages * kSigWNJ * kCtaThreads * 16 + std::min(P.NG, kLocCap) * (int)sizeof(double2);
            static bool attrw = false;
            if (!attrw) {
                cudaFuncSetAttribute(k_verify_sigw<T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlabSmemMax);
                attrw = true;
            }
            int pw = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pw, k_verify_sigw<T, ACT>, kCtaThreads, smemw);
            if (pw >= 1) {
                P.sg_warp = 1;
                // A decision costs a warp ~5 us of the stream (B * V * s bytes at ~6 TB/s):
                // C4 43.7 -> 43.0 us at 13/16; B = 1024 loses 4 us at a fixed 13/16.
                const double t_us = (double)P.B * P.V * sizeof(T) / 6.0e6;
                const int dw = sg_dw_env > 0 ? sg_dw_env : (int)lround(16.0 * std::max(0.0, 1.0 - 5.0 / t_us));
                P.sg_dw = std::max(1, std::min(16, dw));
                P.sg_smem = smemw;
                P.sg_grid = sm_count() * pw;
                P.sg_te = TE;
                P.sg_nt = (P.V + TE - 1) / TE;
                return true;
            }
        }
    }
    P.sg_te = TE;
    P.sg_nt = (P.V + TE - 1) / TE;
    P.sg_nbuf = nbuf;
    P.sg_tb = tb;
    P.sg_smem = smem;
    P.sg_grid = sm_count() * per_sm;
    return true;
}

bool plan_sig(int dtype, int act, StepParams& P) {
    P.sg_on = 0;
    if (act != ACT_SIGMOID) return false;
    if (dtype == DT_F32) return plan_sig_t<float, ACT_SIGMOID>(P);
    if (dtype == DT_BF16) return plan_sig_t<__nv_bfloat16, ACT_SIGMOID>(P);
    return false;
}

template <typename T, int ACT>
static void launch_sig_t(const StepParams& P, const Launch& L) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P.sg_grid, 1, 1);
    cfg.blockDim = dim3(kCtaThreads, 1, 1);
    cfg.dynamicSmemBytes = P.sg_smem;
    cfg.stream = L.st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;  // the locates wait on every CTA's tiles
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1 + pdl_attr(at[1]);
    const int h = L.begin(KID_VERIFY);
    if (P.sg_warp) cudaLaunchKernelEx(&cfg, k_verify_sigw<T, ACT>, P);
    else cudaLaunchKernelEx(&cfg, k_verify_sig<T, ACT>, P);
    L.end(h);
}

template <typename T, int ACT>
static void launch_mat_t(const StepParams& P, void* p, void* q, void* r, const Launch& L) {
    const int h = L.begin(KID_MATERIALIZE);
    k_materialize<T, ACT><<<sm_count() * 8, kThreads, 0, L.st>>>(P, p, q, r);  // grid-stride over units
    L.end(h);
}

template <typename T, int ACT>
static void launch_step_t(const StepParams& P, const Launch& L) {
    if constexpr (sizeof(T) != 8) {
        if (P.cl_size > 0) return launch_cluster_t<T, ACT>(P, L);
        if constexpr (ACT == ACT_SOFTMAX) {
            if (P.sl_on) return launch_slab_t<T>(P, L);
        }
        if constexpr (ACT == ACT_SIGMOID) {
            if (P.sg_on) return launch_sig_t<T, ACT>(P, L);
        }
    }
    launch_verify_t<T, ACT>(P, L);
}

template <typename T>
static void dispatch_verify(int act, const StepParams& P0, void* outp, void* outq, void* outr, const Launch& L) {
    const bool mat = outp || outq || outr;
    if (act == ACT_SOFTMAX) {
        // Resident cluster plan: the verify kernel writes the grids from the
        // slices it still holds; otherwise k_materialize is a second pass.
        StepParams P = P0;
        static const bool no_fuse = knob_set("SSV_NO_FUSE_GRIDS");
        const bool fuse = mat && sizeof(T) != 8 && P.cl_size > 0 && P.cl_resident && !no_fuse;
        if (fuse) {
            P.fuse_grids = 1;
            P.grid_p = outp;
            P.grid_q = outq;
            P.grid_r = outr;
        }
        launch_step_t<T, ACT_SOFTMAX>(P, L);
        if (mat && !fuse) launch_mat_t<T, ACT_SOFTMAX>(P, outp, outq, outr, L);
    } else if (act == ACT_SIGMOID) {
        launch_step_t<T, ACT_SIGMOID>(P0, L);
        if (mat) launch_mat_t<T, ACT_SIGMOID>(P0, outp, outq, outr, L);
    } else if (act == ACT_SIGMOID_HALF) {
        launch_step_t<T, ACT_SIGMOID_HALF>(P0, L);
        if (mat) launch_mat_t<T, ACT_SIGMOID_HALF>(P0, outp, outq, outr, L);
    } else {
        launch_step_t<T, ACT_PROBS>(P0, L);
        if (mat) launch_mat_t<T, ACT_PROBS>(P0, outp, outq, outr, L);
    }
}

void launch_verify(int dtype, int act, const StepParams& P, void* outp, void* outq, void* outr, const Launch& L) {
    if (dtype == DT_F32) dispatch_verify<float>(act, P, outp, outq, outr, L);
    else if (dtype == DT_BF16) dispatch_verify<__nv_bfloat16>(act, P, outp, outq, outr, L);
    else dispatch_verify<double>(act, P, outp, outq, outr, L);
}

void launch_sample_softmax(int dtype, const StepParams& P, const Launch& L) {
    if (dtype == DT_F32) launch_verify_t<float, ACT_SOFTMAX>(P, L);
    else if (dtype == DT_BF16) launch_verify_t<__nv_bfloat16, ACT_SOFTMAX>(P, L);
    else launch_verify_t<double, ACT_SOFTMAX>(P, L);
}

void launch_gen_logits(int dtype, uint64_t seed, int B, int G, int V, void* zp, void* zq, const Launch& L) {
    const int blocks = sm_count() * 16;
    const int h = L.begin(KID_GEN);
    if (dtype == DT_F32) k_gen_logits<float><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (float*)zp, (float*)zq);
    else if (dtype == DT_BF16)
        k_gen_logits<__nv_bfloat16><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (__nv_bfloat16*)zp, (__nv_bfloat16*)zq);
    else k_gen_logits<double><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (double*)zp, (double*)zq);
    L.end(h);
}

__global__ void k_fill_slots(unsigned long long* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = kSlotEmpty;
}

void launch_fill_slots(void* p, size_t n_u64, cudaStream_t st) {
    k_fill_slots<<<sm_count() * 4, kThreads, 0, st>>>(static_cast<unsigned long long*>(p), n_u64);
}

void launch_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u, const Launch& L) {
    const int n = B * (2 * G + 1);
    const int h = L.begin(KID_GEN);
    k_gen_uniforms<<<(n + kThreads - 1) / kThreads, kThreads, 0, L.st>>>(seed, B, G, V, draft_u, u);
    L.end(h);
}

}  // namespace ssv
